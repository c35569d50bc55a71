// kernels.h — host-side launchers of the sm_100a kernels (internal to
// libotprg.so; the public boundary is include/otprg.h).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "device_common.cuh"

namespace otprg {

// Raises (never lowers) a kernel's opt-in dynamic shared-memory limit on the
// current device: the attribute is per function, so contexts prepared with
// different sizes must not shrink it under each other (kernel_attrs.cpp).
cudaError_t smem_attr_raise(const void* fn, size_t bytes);
template <typename F>
inline cudaError_t smem_attr_raise(F* fn, size_t bytes) {
  return smem_attr_raise(reinterpret_cast<const void*>(fn), bytes);
}

// Low-set cache per supply vertex b (see solve_kernels.cu): the ascending
// positions a < cov with k(a,b) + t(a) <= upto at the time of the scan that
// built it, up to kLowCap entries, each packed as (k << 32) | a.
#ifndef OTPRG_LOWCAP
#define OTPRG_LOWCAP 16
#endif
#ifndef OTPRG_LOWLEVELS
#define OTPRG_LOWLEVELS 2
#endif
constexpr int kLowCap = OTPRG_LOWCAP;        // <= 32 (one entry per lane)
constexpr int kTraceSlots = 16;  // u64 timeline slots per phase (see solve_kernels.cu)
constexpr int kLowLevels = OTPRG_LOWLEVELS;  // upto = target + kLowLevels when (re)built

// Device state of one prepared assignment problem, in the solver's internal
// orientation (n_a >= n_b; rows of kT are supply vertices b, contiguous over
// demand vertices a).  Lists rotate over three phases (written in phase p,
// consumed in p+1, reset in p+2).
struct SolveArgs {
  const void* kT;               // T[n_b][lda], pad entries = type max
  void* t;                      // T[lda]  : t(a) = -Y(a) >= 0, pad = 0
  int32_t* yb;                  // [n_b]   : Y(b) >= 1
  int32_t* match_a;             // [n_a]
  int32_t* match_b;             // [n_b]
  // [n_a] x2 : DA holder keys (~phase << 32 | b); phase p proposes into
  // holder[p & 1] while the top of phase p+1 still reads phase p's winners.
  unsigned long long* holder[2];
  void* rowmin;                 // T[n_b]  : lower bound on min_a k(a,b)+t(a)
  int4* lmeta;                  // [n_b]   : low set (upto, cov, cnt, -)
  unsigned long long* lent;     // [n_b * kLowCap] low-set entries
  int32_t* list[3];             // [n_b]   : free b's of the next phase
  int2* mp[3];                  // [n_b]   : (a, previous partner) first held this phase
  int64_t* free_counts;         // [phase_cap + 1]
  Ctl* ctl;
  uint32_t max_phase;           // run phases up to and including this one
  int32_t pre_scanned;          // phase-1 lists/rowmin built by launch_propose_stream
  int32_t tail_switch;          // (full loop) stop where the tail-specialised loop takes over
  // Optional device timeline (%globaltimer ns), kTraceSlots u64 per phase, indexed by
  // phase - 1; nullptr disables tracing.
  unsigned long long* trace;
  uint32_t trace_cap;           // phases the trace buffer holds
};

// Rounding kernels (K1/K2): write kT in the internal orientation.
// width = sizeof(T) of kT (1 or 2).
cudaError_t launch_round_dense(const double* cost, int n_a, int n_b, bool swapped, double eps,
                               void* kT, int lda, int width, int* status, cudaStream_t s);
// thr: exact threshold table (thr_n entries, <= 8192) or nullptr (exact
// division form); absmax: the largest |coordinate| of either point set;
// fix_buf: scratch of round_points_fix_bytes() for the rows deferred to the
// exact fix-up pass (nullptr: the exact division form).
size_t round_points_fix_bytes(int n_ai, int n_bi, int lda, int width, double eps, double absmax);
cudaError_t launch_round_points2d(const double* pa, const double* pb, int n_ai, int n_bi,
                                  double eps, double sqrt2, const double* thr, int thr_n, double absmax,
                                  void* kT, int lda, int width, void* fix_buf, size_t fix_bytes, cudaStream_t s);
// First (a, b) (row-major, original orientation) whose point cost is outside
// [0, 1]: atomicMin into *first (initialise to ~0).
cudaError_t launch_points_range(const double* pa, const double* pb, int n_a, int n_b, double d2_max,
                                unsigned long long* first, cudaStream_t s);
// K3: L1/2 cost of per-image-normalised uint8 vectors (load_mnist_pair).
// normalize: out[i][p] = img[i][p] / sum_p img[i][p] (status 3 on a zero image);
// round: kT[b][a] = scaled_floor(sum_p |xa[a][p] - yb[b][p]| / 2, eps) (status 2
// when a cost leaves [0,1]).  lda must be a multiple of 64.
cudaError_t launch_l1_normalize(const uint8_t* img, int count, int dim, double* out, int* status,
                                cudaStream_t s);
// masks: scratch of l1_mask_bytes() for the tiles' pixel-support masks (the
// sums skip pixels that are zero in every image of both tiles; nullptr: every
// pixel is summed).
size_t l1_mask_bytes(int n_ai, int n_bi, int lda, int dim);
cudaError_t launch_l1_round(const double* xa, const double* yb, int n_ai, int n_bi, int dim,
                            double eps, void* kT, int lda, int width, int* status, cudaStream_t s,
                            uint32_t* masks);
// The range check of K3 alone (status 2 when a cost leaves [0,1]), no kT.
cudaError_t launch_l1_check(const double* xa, const double* yb, int n_ai, int n_bi, int dim, int* status,
                            cudaStream_t s, uint32_t* masks);
// out[p * n + i] = in[i * dim + p] (pixels of the on-the-fly L1 scans).
cudaError_t launch_transpose_f64(const double* in, int n, int dim, double* out, cudaStream_t s);
// Costs of the matched pairs of an L1 image instance (thread per original a).
cudaError_t launch_l1_matched_cost(const double* xa, const double* yb, int dim, const int32_t* match, int n,
                                   bool self_is_a, double* out, cudaStream_t s);
// Matched-pair costs for matching_cost (core.cpp:95-102), one per caller a
// (0 where unmatched): 2-D points (instances.cpp:70-75, sqrt(dx*dx+dy*dy)/sqrt(2)
// in IEEE round-to-nearest, no FMA) or a gather from the dense f64 matrix on the device.
cudaError_t launch_points_matched_cost(const double* xa, const double* yb, const int32_t* match, int n,
                                       double* out, cudaStream_t s);
cudaError_t launch_dense_matched_cost(const double* cost, int n_b, const int32_t* match, int n, double* out,
                                      cudaStream_t s);
// Rounded matrix back to int32 row-major in the ORIGINAL orientation (for
// otprg_scale_round_costs).
cudaError_t launch_k_to_kT(const int32_t* k, int n_a, int n_b, void* kT, int lda, int width,
                           cudaStream_t s);
cudaError_t launch_export_k(const void* kT, int n_ai, int n_bi, int lda, int width, bool swapped,
                            int32_t* k_out, cudaStream_t s);

// A-row-sharded phase step (shard_kernels.cu).  This rank owns demand range
// [lo, hi) of every kT row; everything else is replicated.
struct ShardArgs {
  const void* kT;          // T[n_b][lda] : columns lo..hi-1 (local index a - lo)
  int lda, lo, hi, shard, n_shards;
  const int* bounds;       // [n_shards + 1] shard boundaries (device)
  int K, cap;              // candidates per (shard, proposer); slot stride of the exchange buffers
  int ib;                  // supply vertices (stride of the mps halves)
  void* t;                 // T[n_a] replicated t(a) = -Y(a)
  int width;               // sizeof(T)
  int32_t* yb;
  int32_t* match_a;
  int32_t* match_b;
  unsigned long long* holder;  // [n_a] replicated DA holders
  const int32_t* list_in;  // free b's of the running phase (ascending)
  int2* mps;               // [2][ib] (a, partner) first held in phase p, half p & 1
  int32_t* pos_of_b;       // [n_b] b -> index in list_in
  int4* park[2];           // parked chains (list index, b, restart); ctl->sh_park_cur holds the current
  int64_t* free_counts;
  Ctl* ctl;
  int* scratch;            // [>= 148] compaction block counts
  // Segmented scans (few requests): per-work-item first hits [kSegWarps][K],
  // per-item hit counts [kSegWarps], per-request arrival counters [n_b]
  // (zero between launches).  seg_hits == nullptr: one warp per request.
  int32_t* seg_hits;
  int32_t* seg_cnt;
  int32_t* row_cnt;
  // On-the-fly costs (thr != nullptr): demand / supply points (global
  // indices) and the exact threshold table of thr_n doubles.
  const double2* pa;
  const double2* pb;
  const double* thr;
  int thr_n;
  int otf_tiled;           // the tiled on-the-fly kernel fits shared memory (else the per-row kernel)
  // On-the-fly L1 image costs (l1x != nullptr): normalised demand pixels
  // transposed [dim][n_a] (global a), supply pixels row-major [n_b][dim], eps.
  const double* l1x;
  const double* l1y;
  int dim, na_full;
  double eps;
  // pixel-support masks ((dim + 31) / 32 words each): of the slab's 32-image
  // demand groups (group g = images lo + 32 g ..) and of every supply image;
  // the sums walk the union only (a pixel zero on both sides adds +0)
  const uint32_t* l1_gmask;
  const uint32_t* l1_bmask;
};
// Pixel-support masks of groups of `rows` consecutive images of x (n images
// of dim pixels): bit p of group g when any image of the group has pixel p
// != 0; (dim + 31) / 32 words per group.
cudaError_t launch_l1_group_masks(const double* x, int n, int dim, int rows, uint32_t* mask, cudaStream_t s);
constexpr int kSegWarps = 32768;
constexpr int kMaxSegs = 32;
constexpr int kMaxShardPeers = 8;  // device groups one group pushes to (<= 8 GPUs per node + slack)

// Peer exchange of a device group (one resident loop per device): after the
// local scans, the group's slots are pushed into every other group's exchange
// buffers over NVLink peer memory and each group signals its flag there; a
// group proceeds to DA once every peer's flag reached this round's epoch.
struct ShardPeers {
  int n;                              // peer groups
  int32_t* cand[kMaxShardPeers];      // their exchange buffers (same layout as ours)
  int2* meta[kMaxShardPeers];
  uint32_t* flag[kMaxShardPeers];     // their flag arrays, indexed by group
  uint32_t* my_flags;                 // ours, written by the peers
  int my_group, n_groups;
  int shard_lo, shard_hi;             // local shards [lo, hi): their slots are pushed
  unsigned* arrive;                   // block arrival counter (zero between launches)
};

// Device-driven round kernels: every per-round quantity (mode, request count,
// phase, park buffer, segment split) is read from ctl, so the same launches
// serve the host-driven protocol and the resident graph loop.
// grid: resident-sized (shard_scan_grid); cap = slot stride (S.cap).
int shard_scan_grid(const ShardArgs& a, int num_sms);
bool shard_otf_tiled_fits(int width, int thr_n, int device);
cudaError_t launch_shard_scan(const ShardArgs& a, int32_t* cand, int2* meta, int grid, cudaStream_t s);
cudaError_t launch_shard_push(const ShardArgs& a, const int32_t* cand, const int2* meta,
                              const ShardPeers& p, cudaStream_t s);
// Self-test: n_groups pushes (device arrays of their args) as one cooperative grid.
cudaError_t launch_shard_push_emulated(const ShardArgs* a, const int32_t* const* cand, const int2* const* meta,
                                       const ShardPeers* p, int n_groups, int nblk, cudaStream_t s);
cudaError_t launch_shard_da(const ShardArgs& a, const int32_t* cand, const int2* meta, int grid,
                            cudaStream_t s);
// After the DA: when no chain parked, apply M' / termination / next free
// list (top + compaction); then the round bookkeeping (ctl kernel), which
// sets the resident loop's condition `cond` when use_cond.
cudaError_t launch_shard_after_da(const ShardArgs& a, cudaStream_t s);
cudaError_t launch_shard_ctl(const ShardArgs& a, cudaGraphConditionalHandle cond, bool use_cond,
                             cudaStream_t s);
// top + compaction + bookkeeping as one cooperative launch (148 blocks, grid barriers)
cudaError_t launch_shard_round_end(const ShardArgs& a, cudaGraphConditionalHandle cond, bool use_cond,
                                   cudaStream_t s);
// Before the first round: phase 0 top (termination test, first free list) and ctl.
cudaError_t launch_shard_first_top(const ShardArgs& a, cudaStream_t s);

// OT admissible-cluster scan (ot_kernels.cu): per request (b, target, start)
// the first K admissible (a, ci), encoded a*2+ci, and (count, resume).
cudaError_t launch_ot_scan(const void* kT, int lda, int width, const void* t0, const void* t1,
                           const int4* req, int nreq, int K, int32_t* out, int2* meta,
                           cudaStream_t s);

// ---- OT copy/cluster phase on the device (ot_device.cu) ---------------------
constexpr int32_t kFreeB = 0x7fffffff;  // flow-entry "b" of a demand cluster's free copies
// kCtrTouch..kCtrBig: the device-sized DA rounds (ot_dev_da_rounds): clusters
// proposed to this round, segment space handed out, rounds over (1) or a
// segment too large for the warp resolve (2), entries this round.  kCtrHold:
// the device-sized phase (ot_host.cpp) stopped at a step the host must
// finish (1 admissible lists beyond adm_cap, 2 claim rounds not over, 3 more
// records than one block sorts); every later kernel of the phase returns at
// once while it is set.  kCtrNFlows: records after the merge.
enum OtCtr {
  kCtrNi = 0, kCtrFree = 1, kCtrNew = 2, kCtrE = 3, kCtrRec = 4,
  kCtrTouch = 5, kCtrAlloc = 6, kCtrDone = 7, kCtrN = 8, kCtrBig = 9, kCtrRounds = 10,
  kCtrHold = 11, kCtrNFlows = 12, kCtrCount = 14
};
struct OtDev {
  int n_a, n_b, lda, width;
  const void* kT;      // [n_b][lda] rounded costs at eps/3
  void* t;             // [2][lda] width-typed: t_ci(a) = -y(a, ci), type max if absent
  // demand clusters: code 2a + slot (slot 0 the higher dual), count 0 = absent
  int32_t* dy;
  int64_t* dfree;
  int64_t* dmatched;
  int64_t* consumed;   // copies given this phase
  int32_t* cl_cut;     // DA: highest holder list index of a full cluster (INT_MAX: room)
  // flows: CSR by code, entries ascending b then the free-copy sentinel (b = kFreeB)
  int64_t* fl_off;     // [2 n_a + 1]
  int32_t* fl_code;
  int32_t* fl_b;
  int64_t* fl_cnt;
  int64_t* fl_pre;     // matched copies of the cluster before this entry
  // supply clusters: 2b + slot (slot 0 the higher dual)
  int32_t* sy;
  int64_t* sfree;
  int64_t* smatched;
  int64_t* sfreed;     // displaced copies returning free this phase
  // the phase's free supply vertices (list index i, ascending b)
  int32_t* fb;
  int32_t* fy;
  int32_t* fpos;       // frontier index in the admissible list
  int32_t* fidx;       // [n_b] list index or -1
  int64_t* fu0;        // free copies at phase start
  int64_t* fu;         // copies not (yet) placed
  int64_t* adm_len;
  int64_t* adm_off;
  int32_t* adm;        // admissible cluster codes, ascending a
  int64_t adm_cap;     // entries adm holds (the device-sized phase checks it)
  int64_t e_cap, r_cap;  // DA entries / records the buffers hold (the persistent loop checks them)
  unsigned* bar;       // [2] persistent loop: grid barrier count, count at the last exit
  int64_t* loop;       // [4] persistent loop: phases this launch, claim rounds
  unsigned long long* steptime;  // [32] persistent loop timeline (OTPRG_OT_STEPTIME) or nullptr
  int64_t* fcounts;    // [fc_cap] persistent loop: n_i of the phases of this launch
  int64_t* rec_off;    // [n_a + 1] persistent loop: merged records per demand vertex, scanned
  int small_rec;       // persistent loop: records merged by one block up to this many (else buckets)
  int in_loop;         // set inside the persistent loop: the steps skip their own hold / done checks
  unsigned long long* r_key2;  // [r_cap] records scratch (the bucket merge; the host sort's output)
  int64_t* r_val2;
  int64_t fc_cap;
  // DA entries (key = code << 32 | i) and next-state records
  unsigned long long* e_key;
  int64_t* e_val;
  unsigned long long* s_key;  // the round's entries grouped by cluster (segment per code)
  int64_t* s_val;
  int32_t* da_cnt;     // [2 n_a] entries per cluster this round (0 between rounds)
  int32_t* da_fill;    // [2 n_a] scatter cursor (0 between rounds)
  int64_t* da_off;     // [2 n_a] segment start
  int32_t* da_touch;   // [2 n_a] clusters proposed to this round
  unsigned long long* r_key;
  int64_t* r_val;
  int64_t* ctr;        // [kCtrCount]
  int* status;
  int32_t* err;        // [3]
};
cudaError_t ot_dev_free_list(OtDev& D, int* scratch, cudaStream_t s);
cudaError_t ot_dev_t(OtDev& D, cudaStream_t s);
cudaError_t ot_dev_adm(OtDev& D, int pass, cudaStream_t s);
cudaError_t ot_dev_cut_init(OtDev& D, cudaStream_t s);
cudaError_t ot_dev_propose(OtDev& D, cudaStream_t s);
// R device-sized DA rounds (no host sizes): propose, count per cluster,
// segment allocation, scatter, warp-per-cluster resolve.  ctr[kCtrDone] = 1
// once a round finds no proposal; 2 when a cluster got more than
// kDaWarpMax entries (that round's entries stay in e_key[0, ctr[kCtrN]) for
// the sorted path, ot_dev_da_clear resets the per-cluster counts).
constexpr int kDaWarpMax = 256;
cudaError_t ot_dev_da_rounds(OtDev& D, int rounds, cudaStream_t s);
cudaError_t ot_dev_da_clear(OtDev& D, cudaStream_t s);
// The device-sized phase (no host sizes; see kCtrHold): counters of the
// phase to zero (all but n_i / n_free), the admissible offsets by one
// block, the claim-rounds gate, the updates, the record merge in one block
// (<= kOtSmallRec records), the CSR rebuild; n < 0 in ot_dev_consumed /
// ot_dev_records / ot_dev_rebuild reads the size from the counters.
constexpr int kOtSmallRec = 8192;
cudaError_t ot_dev_phase_begin(OtDev& D, cudaStream_t s);
cudaError_t ot_dev_adm_scan(OtDev& D, cudaStream_t s);
cudaError_t ot_dev_da_gate(OtDev& D, cudaStream_t s);
cudaError_t ot_dev_small_merge(OtDev& D, unsigned long long* key, int64_t* val, cudaStream_t s);
// The whole phase loop as one cooperative launch (a grid barrier between the
// steps above): from `stage` (0 phase start, 1 admissible fill, 2 claim
// rounds, 3 updates, 4 CSR rebuild) through every phase until it stops with
// ctr[kCtrHold] = 9 (n_i <= threshold), 10 (fcounts full), 1-4 (as above; 4:
// records beyond r_cap) or 11 (status set).  Records go to r_key / r_val.
cudaError_t ot_dev_phase_loop(OtDev& D, int stage, double threshold, int* scratch, cudaStream_t s);
cudaError_t ot_dev_resolve(OtDev& D, const unsigned long long* key, const int64_t* val, long long n,
                           unsigned long long* out_key, int64_t* out_val, cudaStream_t s);
cudaError_t ot_dev_consumed(OtDev& D, const unsigned long long* key, const int64_t* val, long long n,
                            cudaStream_t s);
cudaError_t ot_dev_records(OtDev& D, const unsigned long long* key, const int64_t* val, long long n,
                           cudaStream_t s);
cudaError_t ot_dev_rebuild(OtDev& D, const unsigned long long* key, const int64_t* val, long long n,
                           cudaStream_t s);
cudaError_t ot_sort_pairs(void* temp, size_t& temp_bytes, const unsigned long long* kin, unsigned long long* kout,
                          const int64_t* vin, int64_t* vout, long long n, int end_bit, cudaStream_t s);
cudaError_t ot_reduce_by_key(void* temp, size_t& temp_bytes, const unsigned long long* kin,
                             unsigned long long* kout, const int64_t* vin, int64_t* vout, long long* nout,
                             long long n, cudaStream_t s);
cudaError_t ot_exclusive_sum(void* temp, size_t& temp_bytes, const int64_t* in, int64_t* out, int n,
                             cudaStream_t s);

// Phase loop.
cudaError_t launch_init_state(const SolveArgs& a, int n_a, int n_b, int lda, int width,
                              cudaStream_t s);
cudaError_t launch_phase_loop(const SolveArgs& a, int width, bool smem_t, int lda, int grid,
                              cudaStream_t s);
// Launches launch_phase_loop issues (2 when the tail-specialised loop follows).
int phase_loop_launches(int width, bool smem_t, int lda, int grid);
int phase_loop_grid(int width, bool smem_t, int lda, int num_sms);
size_t phase_loop_smem(int width, bool smem_t, int lda);
// Phase-1 propose scan (propose_kernels.cu): every row's k == 0 positions
// (low-set level 0) and row minimum, streamed once with TMA bulk copies.
int propose_stream_chunk(int width, int lda);
cudaError_t launch_propose_stream(const void* kT, int lda, int n_b, int width, int4* lmeta,
                                  unsigned long long* lent, void* rowmin, Ctl* ctl, int num_sms,
                                  cudaStream_t s);
bool smem_t_fits(int width, int lda);

// Largest t(a) / Y(b) the device state may hold: below the saturation value
// of the packed k + t sums (u8/u16) and inside int32 (u32).
inline uint32_t storage_tmax(int width) {
  return width == 1 ? 253u : width == 2 ? 65533u : 0x7ffffff0u;
}
// Bytes per kT entry for |Y| <= need (= unit_ceil + 2, core.hpp:94-95), or -1
// when the requested storage cannot hold it.  storage: 0 auto, 1 u8, 2 u16,
// 3 u32 (otprg_storage).  Auto picks uint16 whenever it fits (measured faster
// than uint8 end to end on B200 for config 2, profiles/r01_variants.txt, even
// though a phase-1 scan reads twice the bytes), else uint32.
inline int storage_width(int64_t need, int storage) {
  auto fits = [&](int w) { return need <= (int64_t)storage_tmax(w) ? w : -1; };
  switch (storage) {
    case 1: return fits(1);
    case 2: return fits(2);
    case 3: return fits(4);
    default: return fits(2) > 0 ? 2 : fits(4);
  }
}

// Device invariant suite (verify_kernels.cu): first violation key
// (section << 60 | index << 4 | kind, minimum over the grid) and count.
struct VerifyOut {
  unsigned long long first;  // ~0 = none
  unsigned long long count;
};
enum VerifyKind : unsigned {
  kMatchA = 1, kMatchB = 2, kDemandPositive = 3, kFreeNonzero = 4, kDemandBound = 5,
  kSupplyNegative = 6, kSupplyBound = 7, kNotTight = 8, kExceeds = 9
};
cudaError_t launch_verify_state(const void* kT, int lda, int width, const void* t,
                                const int32_t* yb, const int32_t* ma, const int32_t* mb, int n_a,
                                int n_b, long long bound, VerifyOut* out, cudaStream_t s);
cudaError_t launch_verify_host(const int32_t* k, const long long* ya, const long long* yb,
                               const int32_t* ma, const int32_t* mb, int n_a, int n_b,
                               long long bound, VerifyOut* out, cudaStream_t s);
// Sinkhorn baseline (sinkhorn_kernels.cu).
cudaError_t sk_build(const double* cost, int n_a, int n_b, double reg, double* K, int* row_ok,
                     int* col_ok, int* bad_cost, cudaStream_t s);
cudaError_t sk_row(const double* K, int n_a, int n_b, const double* u, const double* v,
                   const double* mu, double* term, double* u_next, int* err, cudaStream_t s);
cudaError_t sk_col(const double* K, int n_a, int n_b, const double* w, const double* nu, double* v,
                   double* partial, int* err, cudaStream_t s);
size_t sk_partial_elems(int n_a, int n_b);
cudaError_t sk_sum(const double* x, int n, double* out, cudaStream_t s);
cudaError_t sk_plan(const double* K, int n_a, int n_b, const double* u, const double* v,
                    const double* rs, const double* cs, double* P, cudaStream_t s);
cudaError_t sk_prow(const double* P, int n_a, int n_b, const double* mu, double* row, double* scale,
                    cudaStream_t s);
cudaError_t sk_pcol(const double* P, int n_a, int n_b, double* ones_a, double* partial, double* col,
                    cudaStream_t s);
cudaError_t sk_colscale(const double* col, const double* nu, int n_b, double* scale, cudaStream_t s);
cudaError_t sk_adds(double* P, int n_b, const int2* ab, const double* add, int n, cudaStream_t s);
cudaError_t sk_rowcost(const double* P, const double* cost, int n_a, int n_b, double* rcost,
                       long long* rcnt, cudaStream_t s);
cudaError_t sk_entries(const double* P, int n_a, int n_b, const long long* offs, int32_t* ea,
                       int32_t* eb, double* em, cudaStream_t s);

// Copy mode (copy_kernels.cu).
size_t copy_sort_temp_bytes(int n_a);
cudaError_t copy_order(const int32_t* dgroup, const int32_t* sgroup, const int32_t* ma, int n_a,
                       unsigned long long* keys, unsigned long long* keys_sorted, int32_t* vals,
                       int32_t* pi, int32_t* rank, void* temp, size_t temp_bytes, cudaStream_t s);
cudaError_t copy_da(const void* kT, int lda, int width, const void* t, int32_t* yb, const int32_t* ma,
                    unsigned long long* holder, const int32_t* pi, const int32_t* rank,
                    const int32_t* bfree, int nfree, int n_a, uint32_t phase, int2* mp, int* mp_cnt,
                    Ctl* ctl, cudaStream_t s);
cudaError_t copy_apply(const int2* mp, const int* mp_cnt, const unsigned long long* holder, int32_t* ma,
                       int32_t* mb, void* t, int width, uint32_t phase, Ctl* ctl, cudaStream_t s);
cudaError_t copy_lift(int32_t* yb, const int32_t* mb, const int32_t* sgroup, int n_b, int n_groups,
                      int* gmax, cudaStream_t s);

cudaError_t launch_free_list(const int32_t* mb, int n_b, int32_t* out, int* count, cudaStream_t s);
cudaError_t launch_admissible(const void* kT, int lda, int width, const void* t, const int32_t* yb,
                              const int32_t* bfree, int nfree, int n_a, long long* counts,
                              const long long* offs, int32_t* out, cudaStream_t s);
cudaError_t launch_complete(int32_t* match_a, int32_t* match_b, int n_a, int n_b,
                            int32_t* scratch_a, int32_t* scratch_b, cudaStream_t s);
cudaError_t launch_flush(void* buf, size_t bytes, cudaStream_t s);

}  // namespace otprg
