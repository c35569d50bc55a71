/*
 * otprg.h — C ABI of the B200-native push-relabel assignment solver.
 *
 * Drop-in boundary for the reference's assignment path
 * (/root/reference/proj, namespace otpr):
 *
 *   otprg_solve_assignment   replaces  otpr::solve_assignment
 *                            (include/otpr/assignment.hpp:137-138,
 *                             src/assignment.cpp:368-400), including the
 *                            cost rounding it performs first
 *                            (otpr::scale_round_costs, include/otpr/core.hpp:105,
 *                             src/core.cpp:34-53) and the final
 *                            otpr::matching_cost (core.hpp:147, core.cpp:95-102).
 *   otprg_scale_round_costs  replaces  otpr::scale_round_costs (core.hpp:105)
 *                            for callers that only need the rounded matrix.
 *   otprg_scaled_floor       replaces  otpr::scaled_floor (core.hpp:101).
 *
 * Plain pointers and sizes only.  All host buffers are caller-owned; the
 * context owns its device buffers and reuses them across solves.  Calls block
 * until results are on the host.  A context is single-owner (not re-entrant),
 * like the reference solver.
 *
 * Status codes mirror the reference exception taxonomy
 * (include/otpr/errors.hpp:9-37) and otbench's exit codes
 * (tools/otbench.cpp:187-209):
 *   0 ok, 2 ParameterError, 3 InputError/FormatError, 4 NumericalError,
 *   5 InvariantViolation, 6 CUDA/NCCL failure.
 * otprg_last_error() returns the message of the last failing call.
 *
 * Semantics follow the reference with threads = 1 (the deterministic
 * sequential greedy); results are bit-identical to it: same matching, same
 * integer duals, same phase count / free_counts, same cost bits.
 */
#ifndef OTPRG_H_
#define OTPRG_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum otprg_status {
  OTPRG_OK = 0,
  OTPRG_PARAMETER = 2,
  OTPRG_INPUT = 3,
  OTPRG_NUMERICAL = 4,
  OTPRG_INVARIANT = 5,
  OTPRG_DEVICE = 6,
  OTPRG_ABORTED = 7 /* an observer callback returned nonzero (its exception, in a wrapper) */
};

/* How the cost of edge (a, b) is given. */
enum otprg_cost_kind {
  /* c(a,b) = cost[a*n_b + b], row-major doubles in [0,1]
   * (AssignmentInstance::cost, core.hpp:69-81). */
  OTPRG_COST_DENSE_F64 = 0,
  /* c(a,b) = sqrt(dx*dx+dy*dy)/sqrt(2) of 2-D points pts_a[2a..2a+1],
   * pts_b[2b..2b+1] — gen_uniform_square's formula
   * (src/instances.cpp:70-75), evaluated in non-fused IEEE doubles. */
  OTPRG_COST_POINTS2D = 1,
  /* c(a,b) = 0.5 * sum_p |img_a[a][p]/tot_a - img_b[b][p]/tot_b| over
   * `dim` uint8 pixels, ascending p — load_mnist_pair's formula
   * (src/instances.cpp:114-142). */
  OTPRG_COST_L1_U8 = 2
};

/* Storage width of the rounded cost matrix on the device.  AUTO: uint16 when
 * ceil(1/eps) + 2 <= 65533, else uint32 (eps down to the reference's own
 * limit, unit_floor + 4 <= INT32_MAX, core.cpp:36-41). */
enum otprg_storage {
  OTPRG_STORAGE_AUTO = 0,
  OTPRG_STORAGE_U8 = 1,
  OTPRG_STORAGE_U16 = 2,
  OTPRG_STORAGE_U32 = 3
};

typedef struct otprg_problem {
  int32_t n_a; /* demand side A (rows)   */
  int32_t n_b; /* supply side B (columns) */
  double eps;  /* AssignmentOptions::eps, must lie in (0,1) */
  int32_t cost_kind;
  int32_t storage; /* otprg_storage */
  const double* cost;   /* DENSE_F64: n_a*n_b, host */
  const double* pts_a;  /* POINTS2D: n_a*2 (x,y interleaved), host */
  const double* pts_b;  /* POINTS2D: n_b*2 */
  const uint8_t* img_a; /* L1_U8: n_a*dim */
  const uint8_t* img_b; /* L1_U8: n_b*dim */
  int32_t dim;          /* L1_U8 pixels per image */
  int32_t flags;        /* OTPRG_FLAG_* (0 = none) */
} otprg_problem;

/* Caller-allocated results (SolveStats, assignment.hpp:35-53 + Matching,
 * core.hpp:117-138).  Duals are reported like SolveStats::duals_final: in
 * the solver's internal orientation (swapped when n_b > n_a), before the
 * completion step. */
/* The device keeps free_counts for at most this many phases; a solve that
 * reaches it (only possible for eps below ~2.4e-4, where the reference's own
 * phase cap ceil((1+2eps)/eps^2)+8 is larger) stops with OTPRG_INVARIANT. */
#define OTPRG_MAX_PHASES (1 << 24)

typedef struct otprg_result {
  int32_t* match_of_a;   /* n_a entries, -1 = unmatched (kUnmatched) */
  int32_t* match_of_b;   /* n_b entries */
  int64_t* y_a;          /* max(n_a,n_b) entries (internal demand side) or NULL */
  int64_t* y_b;          /* min(n_a,n_b) entries (internal supply side) or NULL */
  int64_t* free_counts;  /* n_i per executed phase, up to free_cap entries, or NULL */
  int64_t free_cap;
  /* outputs */
  int64_t phases;
  int64_t sum_ni;
  int32_t swapped;
  int32_t full_match_termination;
  double cost;            /* matching_cost of the final matching */
  /* device-side measurements */
  double build_ms;        /* cost build/rounding kernels (CUDA events) */
  double solve_ms;        /* phase loop + completion kernels (CUDA events) */
  double phase1_ms;       /* the phase-1 propose scan kernel (device %globaltimer span) */
  double loop_ms;         /* the phase-loop launch (every phase's chains, phases >= 2 scans) */
  double solve_d2h_ms;    /* solve_ms + D2H of the results into pinned staging */
  int64_t bytes_touched;  /* cost-matrix bytes the scan kernels loaded */
  int64_t bytes_alg;      /* sum_i n_i * n_a * width (Lemma-5 schedule) */
  int32_t width;          /* bytes per rounded cost entry on the device */
  int32_t gpu_launches;   /* kernels launched by this call */
  /* proposal-chain statistics: fresh chains, takeovers, proposals from the
   * low-set cache, exhaustions by a complete cache, scans past the cache,
   * full rescans, rowmin skips, proposals (atomicMin) */
  int64_t chain_stats[8];
  /* sharded solves: refill rounds (rescans of truncated candidate lists) and
   * the shard count; 0 for the single-GPU solver */
  int32_t refill_rounds;
  int32_t n_shards;
} otprg_result;

typedef struct otprg_ctx otprg_ctx;

int otprg_create(int device, otprg_ctx** out);
void otprg_destroy(otprg_ctx* ctx);
const char* otprg_last_error(const otprg_ctx* ctx);
int otprg_version(void);

/* Run this context's work on the caller's CUDA stream (NULL: its own stream
 * again).  Used to put several contexts and an NCCL exchange on one stream so
 * the sharded protocol needs no host sync between scan, exchange and DA. */
int otprg_set_stream(otprg_ctx* ctx, void* stream);

/* scaled_floor(c, eps) (core.cpp:26-32), evaluated on the host. */
int64_t otprg_scaled_floor(double c, double eps);

/* Exact threshold table of the 2-D point cost: for the cost
 * c = sqrt(d2) / sqrt(2) of gen_uniform_square (instances.cpp:70-75, IEEE
 * round-to-nearest, no FMA) and k = scaled_floor(c, eps), thr[j] is the
 * smallest double d2 >= 0 with k(d2) >= j, j = 0..unit_floor+1 (thr[0] = 0,
 * +inf where unreachable for d2 <= 2): k(d2) = max{j : thr[j] <= d2}, so
 * k(a,b) needs no sqrt or division.  Writes unit_floor + 2 doubles (cap
 * permitting) and returns that count, or -1 for a bad eps.  Host-only. */
int32_t otprg_points_threshold_table(double eps, double* thr, int32_t cap);

/* otprg_problem.flags */
#define OTPRG_FLAG_ON_THE_FLY 1 /* sharded 2-D points: no kT slab; the scans compute k(a,b) from
                                 * the points with the threshold table above */

/* Full solve: H2D of the problem's host buffers, cost build + rounding on
 * the device, device-resident phase loop, completion, D2H of the results,
 * matching cost.  Mirrors otpr::solve_assignment. */
int otprg_solve_assignment(otprg_ctx* ctx, const otprg_problem* prob, otprg_result* res);

/* Two-step form used by benchmarks: prepare() uploads + builds the rounded
 * matrix and keeps it resident in the context; solve_prepared() runs the
 * phase loop on it (results as above).  solve_prepared() may be called
 * repeatedly on the same prepared problem. */
int otprg_prepare(otprg_ctx* ctx, const otprg_problem* prob, otprg_result* res);
int otprg_solve_prepared(otprg_ctx* ctx, otprg_result* res);

/* Stepping form (host-synced; used for per-phase observation like the
 * reference's PhaseObserver, assignment.hpp:55-67, and for debugging):
 *   otprg_begin     init_state on the prepared problem (assignment.cpp:54-60)
 *   otprg_step      run phases until `max_phases` phases have executed in
 *                   total (<= 0: until termination); reports the phase count
 *                   and whether the termination test (:330-334) has passed
 *   otprg_snapshot  copy the current state (matching, duals, free_counts,
 *                   phases) without completing the matching
 *   otprg_finish    run the remaining phases, complete the matching
 *                   (:253-262) and return the final results. */
int otprg_begin(otprg_ctx* ctx);
int otprg_step(otprg_ctx* ctx, int64_t max_phases, int64_t* phases_done, int32_t* finished);
int otprg_snapshot(otprg_ctx* ctx, otprg_result* res);
int otprg_finish(otprg_ctx* ctx, otprg_result* res);

/* ---- copy mode ---------------------------------------
 * solve_assignment with AssignmentOptions::demand_groups / supply_groups
 * (assignment.hpp:81-89; scan order assignment.cpp:81-103, supply-copy dual
 * lift :241-250): every phase visits the admissible demand copies of a free
 * b in group order (free copies first, then matched copies by their
 * partner's supply group), and free supply copies are raised to their
 * group's maximum dual.  Requires n_b <= n_a (ParameterError otherwise, as
 * the reference).  Host-synced phases (copy mode serves the reference's
 * OT-equivalence checks, not the benchmark path):
 *   otprg_groups_begin   prepare + init_state with the group maps
 *   otprg_groups_step    run one phase (finished once the termination test passed)
 *   otprg_snapshot / otprg_verify_feasibility / otprg_admissible work between steps
 *   otprg_groups_finish  remaining phases, completion, results (as otprg_solve_assignment) */
int otprg_groups_begin(otprg_ctx* ctx, const otprg_problem* prob, const int32_t* demand_groups,
                       const int32_t* supply_groups);
int otprg_groups_step(otprg_ctx* ctx, int64_t* phases_done, int32_t* finished);
int otprg_groups_finish(otprg_ctx* ctx, otprg_result* res);

/* ---- invariant suite (reference A12) ----------------
 * verify_feasibility (assignment.cpp:264-312) evaluated on the device.  The
 * result is the number of violations and the FIRST one in the reference's
 * order of checks (Matching::validate core.cpp:69-86 a then b; per demand a:
 * positive dual, free with nonzero dual, |Y| > dual_bound; per supply b:
 * negative dual, |Y| > dual_bound; every edge a-major: matched edge not
 * tight, else Y(a)+Y(b) > k+1), i.e. report.violations.front().  When the
 * matching itself is inconsistent the reference stops there: violations = 1.
 * Indices are in the orientation of the checked state (the solver's
 * internal one for otprg_verify_feasibility). */
enum {
  OTPRG_VIOL_NONE = 0,
  OTPRG_VIOL_MATCH_A = 1,         /* matching is not mutually consistent at a= */
  OTPRG_VIOL_MATCH_B = 2,         /* ... at b= */
  OTPRG_VIOL_DEMAND_POSITIVE = 3, /* demand dual positive at a= */
  OTPRG_VIOL_FREE_NONZERO = 4,    /* free demand vertex with nonzero dual at a= */
  OTPRG_VIOL_DEMAND_BOUND = 5,    /* demand dual magnitude exceeds bound at a= */
  OTPRG_VIOL_SUPPLY_NEGATIVE = 6, /* supply dual negative at b= */
  OTPRG_VIOL_SUPPLY_BOUND = 7,    /* supply dual magnitude exceeds bound at b= */
  OTPRG_VIOL_NOT_TIGHT = 8,       /* matching edge not tight at (a,b) */
  OTPRG_VIOL_EXCEEDS = 9          /* dual sum exceeds rounded cost allowance at (a,b) */
};
typedef struct otprg_feasibility {
  int64_t violations;
  int32_t kind;        /* OTPRG_VIOL_* of the first violation */
  int32_t a, b;        /* its vertices (-1 when not applicable) */
  int32_t pad;
  int64_t sum;         /* Y(a)+Y(b) for edge kinds, else the offending dual */
  int64_t k;           /* k(a,b) for edge kinds */
} otprg_feasibility;

/* The context's current solver state (between phases of the stepping API,
 * i.e. what check_invariants sees after apply_phase, assignment.cpp:344-349). */
int otprg_verify_feasibility(otprg_ctx* ctx, otprg_feasibility* out);
/* Arbitrary state, the reference's verify_feasibility(sc, duals, m):
 * k row-major n_a x n_b int32 (ScaledCosts::k), dual bound unit_ceil + 2. */
int otprg_verify_host(otprg_ctx* ctx, int32_t n_a, int32_t n_b, const int32_t* k,
                      int32_t unit_ceil, const int64_t* y_a, const int64_t* y_b,
                      const int32_t* match_of_a, const int32_t* match_of_b,
                      otprg_feasibility* out);
/* verify_feasibility of a solver result (internal orientation, pre-completion
 * matching, e.g. from otprg_snapshot of another context — a sharded or
 * on-the-fly solve of the same instance) against this context's prepared
 * rounded costs: the check for sizes where no host k matrix fits (n = 100k). */
int otprg_verify_result(otprg_ctx* ctx, const int64_t* y_a, const int64_t* y_b,
                        const int32_t* match_of_a, const int32_t* match_of_b, otprg_feasibility* out);
/* collect_workset's B' and E' for the current state (assignment.cpp:107-147,
 * internal orientation): b_free ascending (n_free entries, caller buffer of
 * n_b), offsets[n_free + 1] and the admissible a of every free b ascending in
 * a_list.  a_list == NULL or a_cap < n_edges: only n_free / n_edges / b_free
 * / offsets are written (call again with a larger buffer). */
int otprg_admissible(otprg_ctx* ctx, int32_t* b_free, int64_t* offsets, int32_t* a_list,
                     int64_t a_cap, int64_t* n_free, int64_t* n_edges);

/* Rounded costs k(a,b) = scaled_floor(c(a,b), eps) computed on the device
 * and returned row-major (n_a x n_b int32, like ScaledCosts::k), plus
 * unit_floor / unit_ceil (core.hpp:89-92).  Mirrors otpr::scale_round_costs. */
int otprg_scale_round_costs(otprg_ctx* ctx, const otprg_problem* prob, int32_t* k,
                            int32_t* unit_floor, int32_t* unit_ceil);

/* Point sets of otpr::gen_uniform_square(n, seed) (src/instances.cpp:48-62):
 * std::mt19937_64 streams seeded with splitmix64(seed) (A) and
 * splitmix64(seed ^ 0x9E3779B97F4A7C15) (B), x then y per point, 53-bit
 * uniforms.  Writes interleaved (x, y) pairs, n per side.  Host-only. */
int otprg_uniform_square_points(int32_t n, uint64_t seed, double* pts_a, double* pts_b);

/* The image pair of otpr::load_mnist_pair(path, n, seed)
 * (src/instances.cpp:80-144): parses the IDX3 file, draws the seeded sample of
 * 2n distinct images (mt19937_64(splitmix64(seed ^ 0xD1B54A32D192ED03)),
 * partial Fisher-Yates) and writes the first n raw 28x28 images to img_a and
 * the next n to img_b (n*784 bytes each).  The L1/2 cost of the pair is then
 * computed on the device with OTPRG_COST_L1_U8.  Errors: 3 for unreadable /
 * malformed files (FormatError / InputError), message in err.  Host-only. */
int otprg_load_mnist_pair(const char* path, int32_t n, uint64_t seed, uint8_t* img_a,
                          uint8_t* img_b, char* err, int32_t err_cap);

/* ---- A-row-sharded solve over several GPUs ---------------
 * Shard g of G owns the demand range [bounds[g], bounds[g+1]) of every
 * rounded-cost row (built from the problem's 2-D point sets on its GPU, or no
 * slab at all with OTPRG_FLAG_ON_THE_FLY); matching, duals and DA holders are
 * replicated and every shard computes the identical result, bit-identical for
 * every G (and to otprg_solve_assignment / the reference).  A round is: scan
 * (first K admissible a of every proposer in the slab) -> exchange of the
 * candidate slots -> deferred acceptance over the merged lists; chains that
 * reach a truncated list park and the next round rescans them; a phase ends
 * with its top (apply M', termination, next free list).
 *
 * Easiest: a multi-device context.  otprg_create_multi(devices, n) makes one
 * shard per listed device (the same device may be listed several times:
 * logical shards sharing it); otprg_solve_assignment / otprg_prepare +
 * otprg_solve_prepared on it run the resident loop below for point instances
 * (other cost kinds run on the first device).  K: otprg_set_shard_k (16). */
int otprg_create_multi(const int32_t* devices, int32_t ndev, otprg_ctx** out);
int otprg_set_shard_k(otprg_ctx* ctx, int32_t K);

/* Shard contexts (one per shard and device; created with otprg_create): */
int otprg_shard_prepare(otprg_ctx* ctx, const otprg_problem* prob, int32_t n_shards,
                        int32_t shard, int32_t K, int32_t* bounds_out);
/* Resident solve of the shards this process holds: every round of every phase
 * runs inside one CUDA graph per device (a conditional WHILE node: scan ->
 * NVLink peer push of the candidate slots + epoch flags -> DA -> top ->
 * round bookkeeping, which sets the loop condition), one host sync per solve.
 * Shards on one device run in stream order and exchange nothing; each device
 * appears once (its shards consecutive).  When the shards do not cover all
 * n_shards (one process per GPU), attach the other processes' exchange blocks
 * first with otprg_shard_ipc_export / otprg_shard_ipc_attach.  Results as
 * otprg_solve_assignment (from the lowest local shard; all must agree). */
int otprg_shard_solve_resident(otprg_ctx** shards, int32_t n, otprg_result* res);
/* Multi-process resident mode (one process per GPU; this process's shard
 * forms group my_group of n_groups): export writes the CUDA IPC handle
 * (OTPRG_IPC_HANDLE_BYTES) of this shard's exchange block; the caller
 * all-gathers the handles (e.g. torch.distributed) and attaches them all
 * (handles[q] of group q, group q holding shards [group_shard_lo[q],
 * group_shard_lo[q+1])).  Then otprg_shard_solve_resident(&ctx, 1, res). */
#define OTPRG_IPC_HANDLE_BYTES 64
/* Self-test of the resident loop's peer exchange on one device: n_groups
 * groups (shards_per_group shards each) push varying round slots into each
 * other's exchange blocks and wait on the epoch flags, emulated as one
 * cooperative grid (co-resident blocks; the multi-GPU push proper needs one
 * GPU per group).  *mismatches counts wrong slots / flags over `rounds`. */
int otprg_selftest_exchange(int32_t device, int32_t n_groups, int32_t shards_per_group, int32_t ib,
                            int32_t K, int32_t rounds, int64_t* mismatches);
int otprg_shard_ipc_export(otprg_ctx* ctx, int32_t n_groups, int32_t my_group, void* handle_out);
int otprg_shard_ipc_attach(otprg_ctx* ctx, const void* handles, int32_t n_groups,
                           const int32_t* group_shard_lo);
/* Host-driven protocol (the caller exchanges the slots between scan and DA,
 * e.g. with an NCCL / gloo all-gather; one host sync per round):
 *   otprg_shard_begin  init_state + the phase-0 top;
 *   otprg_shard_top    n_i of the coming phase and whether the solve finished;
 *   otprg_shard_scan   this shard's first-K candidates of every proposer into
 *                      its slot of cand[n_shards][cap][K] / meta[n_shards][cap]
 *                      (device buffers; refill = 1 for a rescan round);
 *   otprg_shard_da     deferred acceptance over the merged slots; reports the
 *                      parked chains (> 0: scan(refill=1), exchange,
 *                      da(resume=1) again);
 *   otprg_shard_finish completes the matching and returns the results. */
int otprg_shard_begin(otprg_ctx* ctx);
int otprg_shard_top(otprg_ctx* ctx, int32_t* n_out, int32_t* finished);
int otprg_shard_scan(otprg_ctx* ctx, int32_t* cand, int32_t* meta, int32_t cap, int32_t refill);
int otprg_shard_da(otprg_ctx* ctx, const int32_t* cand, const int32_t* meta, int32_t cap,
                   int32_t resume, int32_t* parked);
int otprg_shard_finish(otprg_ctx* ctx, otprg_result* res);

/* ---- optimal transport (config 5) ---------------------------------------
 * otprg_solve_ot replaces otpr::solve_ot (include/otpr/ot.hpp:161-163,
 * src/ot.cpp:705-732): theta-scaling of the masses at eps/3
 * (scale_and_round, ot.cpp:109-128), the copy/cluster phase algorithm
 * (solve_copy_matching, ot.cpp:418-637) and plan_from_flow (ot.cpp:639-703).
 * Plan entries are written row-major (as TransportPlan::entries) up to
 * entry_cap; n_entries reports the full count.  Masses and costs as the
 * reference sees them (no renormalisation here). */
typedef struct otprg_ot_problem {
  int32_t n_a, n_b;
  double eps;
  const double* mu;    /* n_a demand masses, host */
  const double* nu;    /* n_b supply masses, host */
  const double* cost;  /* n_a*n_b row-major in [0,1], host */
  int32_t flags;       /* reserved, 0 */
  int32_t pad;
} otprg_ot_problem;

typedef struct otprg_ot_result {
  int32_t* ent_a;
  int32_t* ent_b;
  double* ent_mass;
  int64_t entry_cap;
  int64_t* free_counts; /* free supply copies per phase, or NULL */
  int64_t free_cap;
  /* outputs */
  int64_t n_entries;
  double cost;           /* TransportPlan::cost */
  int64_t phases;
  int64_t sum_ni;
  int32_t full_match_termination;
  int32_t gpu_launches;
  double theta;          /* ScaledMasses::theta */
  int64_t total_d, total_s;
  double build_ms, loop_ms, scan_ms, solve_ms;  /* host-clock ms around the stages */
  int64_t bytes_touched; /* kT bytes covered by the device scans */
} otprg_ot_result;

int otprg_solve_ot(otprg_ctx* ctx, const otprg_ot_problem* prob, otprg_ot_result* res);

/* ---- OT phase primitives and debug mode ----------------------------------
 * The copy/cluster solver's types (include/otpr/ot.hpp:52-95) in flat form.
 * A CopyInstance: rounded costs over the original vertices plus a copy count
 * per vertex (ot.hpp:52-63).  unit_ceil is ScaledCosts::unit_ceil, so the
 * dual bound of the checks is unit_ceil + 2 (core.hpp:95). */
typedef struct otprg_copy_instance {
  int32_t n_a, n_b;
  const int32_t* k;              /* n_a*n_b row-major ScaledCosts::k */
  int64_t unit_ceil;
  const int64_t* demand_copies;  /* n_a */
  const int64_t* supply_copies;  /* n_b */
} otprg_copy_instance;

/* ClusterState (ot.hpp:65-95): demand vertex a owns clusters
 * [dem_off[a], dem_off[a+1]) (dual, free copies, flow entries
 * [flow_off[c], flow_off[c+1]) of (b, copies) ascending b); supply vertex b
 * owns [sup_off[b], sup_off[b+1]).  Clusters are in descending dual order, as
 * normalize_demand / normalize_supply leave them (ot.cpp:362-414). */
typedef struct otprg_cluster_state {
  int32_t n_a, n_b;
  const int32_t* dem_off;   /* n_a + 1 */
  const int64_t* dem_y;
  const int64_t* dem_free;
  const int64_t* flow_off;  /* clusters + 1 */
  const int32_t* flow_b;
  const int64_t* flow_cnt;
  const int32_t* sup_off;   /* n_b + 1 */
  const int64_t* sup_y;
  const int64_t* sup_free;
  const int64_t* sup_matched;
} otprg_cluster_state;

/* ClusterPhaseSnapshot (ot.hpp:115-122); every pointer is valid only during
 * the observer call (the reference's references have the same lifetime). */
typedef struct otprg_cluster_snapshot {
  int64_t phase; /* 1-based */
  int64_t n_i;   /* free supply copies at phase start */
  int64_t sum_abs_before, sum_abs_after;
  otprg_copy_instance inst;
  otprg_cluster_state state;
} otprg_cluster_snapshot;

typedef int (*otprg_cluster_observer)(const otprg_cluster_snapshot* snap, void* user);

/* OTOptions / ClusterOptions (ot.hpp:124-129, 153-156).  check_invariants:
 * after every phase the greedy-maximality, cluster-invariant and
 * cluster-feasibility checks of ot.cpp:524-533, 594-603 (host; the first
 * violation is OTPRG_INVARIANT with the reference's message).  observer:
 * called after every phase; a nonzero return stops the solve (OTPRG_ABORTED). */
typedef struct otprg_ot_options {
  int32_t check_invariants;
  int32_t pad;
  otprg_cluster_observer observer;
  void* user;
} otprg_ot_options;

/* solve_ot with options (opt may be NULL = otprg_solve_ot). */
int otprg_solve_ot_opts(otprg_ctx* ctx, const otprg_ot_problem* prob, const otprg_ot_options* opt,
                        otprg_ot_result* res);

/* solve_copy_matching (ot.hpp:135-141, ot.cpp:418-637) on a copy instance:
 * the k matrix goes to the device as the scan's kT, the claim step and the
 * cluster bookkeeping are those of otprg_solve_ot.  eps is the solve's
 * accuracy (termination eps * total supply copies, phase cap).  Errors as
 * CopyInstance::validate (ot.cpp:142-152) -> OTPRG_PARAMETER; in addition k
 * must lie in [0, 2^31 - 16) (device storage).  flow: the n_a*n_b dense
 * ClusterSolveResult::flow (completion included) or NULL.  The final state
 * before completion stays readable through otprg_copy_state until the next
 * solve on the context. */
typedef struct otprg_copy_result {
  int64_t* flow;
  int64_t* free_counts;  /* n_i per phase, up to free_cap entries, or NULL */
  int64_t free_cap;
  int64_t phases;
  int64_t sum_ni;
  int32_t full_match_termination;
  int32_t gpu_launches;
} otprg_copy_result;

int otprg_solve_copy_matching(otprg_ctx* ctx, const otprg_copy_instance* inst, double eps,
                              const otprg_ot_options* opt, otprg_copy_result* res);
/* ClusterSolveResult::state of the last otprg_solve_copy_matching /
 * otprg_solve_ot_opts on ctx (pointers owned by ctx). */
int otprg_copy_state(otprg_ctx* ctx, otprg_cluster_state* out);

/* check_cluster_invariant (which = 0, ot.cpp:190-265) and
 * check_cluster_feasibility (which = 1, ot.cpp:267-315) on a flat state:
 * *count = number of violations (ClusterReport::violations.size()), their
 * messages newline-separated into msgs (NUL-terminated, truncated to
 * msgs_cap).  Host-only. */
int otprg_check_cluster_state(const otprg_cluster_state* state, const otprg_copy_instance* inst,
                              int32_t which, int64_t* count, char* msgs, int32_t msgs_cap);

/* plan_from_flow (ot.hpp:143-151, ot.cpp:639-703): dense integer copy flow
 * (n_a*n_b row-major) + ScaledMasses (theta, d, s) + the OT instance ->
 * plan entries / cost in res (the plan fields of otprg_ot_result).  Host-only. */
int otprg_plan_from_flow(const otprg_ot_problem* prob, const int64_t* flow, double theta,
                         const int64_t* d, const int64_t* s, otprg_ot_result* res);

/* ---- Sinkhorn baseline -------------------------------
 * otprg_sinkhorn replaces otpr::sinkhorn (include/otpr/sinkhorn.hpp:13-31,
 * src/sinkhorn.cpp:69-151): kernel exp(-c/reg), alternating scaling until the
 * L1 row-marginal violation <= tol (or max_iters / the time budget), then
 * round_to_marginals (:12-66).  FP64 on the device; deterministic reductions
 * (not the reference's sequential sums bit for bit).  Errors: 2 for reg/tol
 * <= 0 or costs outside [0,1], 3 for masses not summing to 1, 4 when the
 * kernel or a scaling vector underflows / diverges (NumericalError). */
typedef struct otprg_sinkhorn_config {
  double reg;            /* > 0 */
  int32_t max_iters;
  int32_t pad;
  double tol;            /* > 0 */
  double time_budget_ms; /* 0 = none */
} otprg_sinkhorn_config;

typedef struct otprg_sinkhorn_result {
  int32_t* ent_a;        /* plan entries (p > 0, row-major) up to entry_cap, or NULL */
  int32_t* ent_b;
  double* ent_mass;
  int64_t entry_cap;
  /* outputs */
  int64_t n_entries;
  double cost;           /* SinkhornResult::cost = plan.cost */
  int32_t iters;
  int32_t converged;
  double marginal_violation;
  double build_ms, loop_ms, round_ms;
} otprg_sinkhorn_result;

int otprg_sinkhorn(otprg_ctx* ctx, const otprg_ot_problem* prob, const otprg_sinkhorn_config* cfg,
                   otprg_sinkhorn_result* res);

/* scale_and_round (ot.cpp:109-128): d = exact_ceil(mu*theta),
 * s = exact_floor(nu*theta), theta = 4 max(n_a,n_b) / eps.  Host-only. */
int otprg_ot_scale_and_round(int32_t n_a, int32_t n_b, const double* mu, const double* nu,
                             double eps, int64_t* d, int64_t* s, double* theta);

/* otpr::gen_random_ot_rational(n_a, n_b, seed) (instances.cpp:159-191)
 * including OTInstance::renormalize (ot.cpp:91-100).  Host-only. */
int otprg_random_ot_rational(int32_t n_a, int32_t n_b, uint64_t seed, double* mu, double* nu,
                             double* cost);

/* Free and total device memory of `device` (cudaMemGetInfo), for callers that
 * choose between the materialised matrix and on-the-fly costs
 * (AssignmentOptions costs = auto) without a CUDA runtime of their own. */
int otprg_mem_info(int device, uint64_t* free_bytes, uint64_t* total_bytes);

/* Writes a buffer larger than L2 on the context's stream (benchmark hygiene). */
int otprg_flush_l2(otprg_ctx* ctx);

/* Device timeline (tracing): when enabled, every phase-loop phase records 16
 * u64 (%globaltimer ns) per phase — see solve_kernels.cu for the slot map —
 * for up to max_phases phases (0 = off).  otprg_get_trace copies them out
 * (max_phases * 16 u64). */
int otprg_set_trace(otprg_ctx* ctx, int64_t max_phases);
int otprg_get_trace(otprg_ctx* ctx, uint64_t* out, int64_t max_phases);

/* CUDA-event timer on the context's stream: start, ..., stop -> elapsed ms. */
int otprg_timer_start(otprg_ctx* ctx);
int otprg_timer_stop(otprg_ctx* ctx, double* ms);

#ifdef __cplusplus
}
#endif

#endif /* OTPRG_H_ */
