// shard_host.cpp — host side of the A-row-sharded solve.
//
// Shard g of G owns the demand range [bounds[g], bounds[g+1]) of every rounded
// cost row (its kT slab, built on its device from the 2-D point sets, or no
// slab at all with on-the-fly costs); the matching, the integer duals and the
// deferred-acceptance holders are replicated and every shard runs the same
// deterministic rounds, so only candidate lists are exchanged.  The loop is
// the reference's solve_oriented (assignment.cpp:316-364) with the phase step
// of :157-235; the round kernels are in shard_kernels.cu and read every
// per-round quantity from the device control block.
//
// Two drivers over the same kernels:
//   * host-driven (otprg_shard_top/scan/da): one host sync per round, the
//     caller exchanges the slots (torch.distributed all-gather, sharded.py);
//   * resident (otprg_shard_solve_resident, otprg_create_multi): every round of
//     every phase runs inside one CUDA graph per device — a conditional WHILE
//     node whose body is scan -> peer push + flag wait -> DA -> top/compaction ->
//     round bookkeeping, the last kernel setting the loop condition — so a
//     solve costs one host sync.  Shards on one device form a group that runs
//     its shards' kernels in stream order (no exchange needed inside a group);
//     groups on different devices push their slots into each other's exchange
//     blocks over NVLink peer memory (cudaDeviceEnablePeerAccess in one
//     process, CUDA IPC handles across processes) and wait on per-group epoch
//     flags.  Groups never share a device, so no kernel waits on another kernel
//     of the same GPU.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <memory>
#include <string>
#include <vector>

#include "capi_internal.h"

using otprg::Ctl;
using otprg::DevBuf;
using otprg::host_scaled_floor;
using namespace otprg_capi;

namespace {

otprg::ShardArgs shard_args(otprg_ctx* ctx) {
  otprg::ShardArgs S{};
  S.kT = ctx->kT.p;
  S.lda = ctx->lda;
  S.lo = ctx->sh_lo;
  S.hi = ctx->sh_hi;
  S.shard = ctx->sh_shard;
  S.n_shards = ctx->sh_n_shards;
  S.bounds = ctx->sh_bounds.as<int>();
  S.K = ctx->sh_K;
  S.cap = ctx->sh_cap;
  S.ib = ctx->ib;
  S.t = ctx->t.p;
  S.width = ctx->width;
  S.yb = ctx->yb.as<int32_t>();
  S.match_a = ctx->ma.as<int32_t>();
  S.match_b = ctx->mb.as<int32_t>();
  S.holder = ctx->holder.as<unsigned long long>();
  S.list_in = ctx->sh_list.as<int32_t>();
  S.mps = ctx->mps.as<int2>();
  S.pos_of_b = ctx->sh_pos.as<int32_t>();
  S.park[0] = ctx->sh_park[0].as<int4>();
  S.park[1] = ctx->sh_park[1].as<int4>();
  S.free_counts = ctx->fc.as<int64_t>();
  S.ctl = ctx->ctl.as<Ctl>();
  S.scratch = ctx->fa.as<int>();  // (completion scratch, free during the phases)
  S.seg_hits = ctx->sh_seg.as<int32_t>();
  S.seg_cnt = S.seg_hits + static_cast<size_t>(otprg::kSegWarps) * ctx->sh_K;
  S.row_cnt = S.seg_cnt + otprg::kSegWarps;
  if (ctx->sh_otf && ctx->cost_kind == OTPRG_COST_L1_U8) {
    const size_t dim = ctx->img_dim;
    S.l1x = reinterpret_cast<const double*>(static_cast<const char*>(ctx->pts.p) + ctx->sh_l1_xt);
    S.l1y = ctx->pts.as<double>() + static_cast<size_t>(ctx->ia) * dim;
    S.dim = ctx->img_dim;
    S.na_full = ctx->ia;
    S.eps = ctx->eps;
    S.l1_gmask = ctx->l1_otf_mask.as<uint32_t>();
    S.l1_bmask = S.l1_gmask + static_cast<size_t>((ctx->sh_hi - ctx->sh_lo + 31) / 32) * ((dim + 31) / 32);
  } else if (ctx->sh_otf) {
    S.pa = ctx->pts.as<double2>();
    S.pb = S.pa + ctx->ia;
    S.thr = ctx->thr_dev.as<double>();
    S.thr_n = ctx->sh_thr_n;
    S.otf_tiled = ctx->sh_otf_tiled ? 1 : 0;
  }
  return S;
}

int read_ctl(otprg_ctx* ctx, Ctl* h) {
  CK(cudaMemcpyAsync(h, ctx->ctl.p, sizeof(Ctl), cudaMemcpyDeviceToHost, ctx->stream), "D2H ctl");
  CK(cudaStreamSynchronize(ctx->stream), "shard step");
  return check_status(ctx, *h, false);
}

// The round state the host-driven protocol reports (otprg_shard_top / _da).
void cache_round(otprg_ctx* ctx, const Ctl& h) {
  ctx->sh_have = true;
  ctx->sh_done = h.done;
  if (h.sh_mode == 1) {
    ctx->sh_parked = h.sh_nreq;
  } else {
    ctx->sh_parked = 0;
    ctx->sh_n = h.sh_nreq;
  }
  ctx->sh_epoch = h.sh_epoch;
}

// init_state (assignment.cpp:54-60), control block, phase-0 top (termination
// test, first free list) and round bookkeeping; no host sync.
int shard_begin_launch(otprg_ctx* ctx, uint32_t epoch) {
  CK(cudaSetDevice(ctx->device), "cudaSetDevice");
  Ctl h{};
  h.n_a = ctx->ia;
  h.n_b = ctx->ib;
  h.lda = ctx->lda;
  // (double)n_i <= eps * m  <=>  n_i <= floor(eps * m)   (assignment.cpp:324-331)
  h.thresh = static_cast<int32_t>(std::floor(ctx->eps * static_cast<double>(std::min(ctx->n_a, ctx->n_b))));
  h.phase_cap = static_cast<int32_t>(ctx->fc_cap - 1);
  h.tmax = otprg::storage_tmax(ctx->width);
  h.cnt[0] = ctx->ib;
  h.sh_epoch = epoch;
  CK(cudaMemcpyAsync(ctx->ctl.p, &h, sizeof(Ctl), cudaMemcpyHostToDevice, ctx->stream), "H2D ctl");
  otprg::SolveArgs A{};
  A.t = ctx->t.p;
  A.yb = ctx->yb.as<int32_t>();
  A.match_a = ctx->ma.as<int32_t>();
  A.match_b = ctx->mb.as<int32_t>();
  A.holder[0] = ctx->holder.as<unsigned long long>();
  A.holder[1] = A.holder[0] + ctx->ia;
  A.rowmin = ctx->rowmin.p;
  A.lmeta = ctx->lmeta.as<int4>();
  A.list[0] = ctx->lists.as<int32_t>();
  const int full = (ctx->ia + 511) / 512 * 512;
  CK(otprg::launch_init_state(A, ctx->ia, ctx->ib, full, ctx->width, ctx->stream), "init launch");
  CK(otprg::launch_shard_first_top(shard_args(ctx), ctx->stream), "shard top launch");
  ctx->begun = true;
  ctx->completed = false;
  ctx->sh_have = false;
  return OTPRG_OK;
}

// ---- resident loop ----------------------------------------------------------

// Exchange block of one group (one allocation, so one IPC handle covers it):
// cand [G][ib][K] int32 | meta [G][ib] int2 | flags [kMaxGroups] u32 | arrive u32.
constexpr int kMaxGroups = 64;
struct XLayout {
  size_t cand = 0, meta = 0, flags = 0, arrive = 0, bytes = 0;
  XLayout() = default;
  XLayout(int n_shards, int ib, int K) {
    cand = 0;
    meta = ((size_t)n_shards * ib * K * 4 + 255) / 256 * 256;
    flags = meta + ((size_t)n_shards * ib * 8 + 255) / 256 * 256;
    arrive = flags + kMaxGroups * 4;
    bytes = arrive + 256;
  }
};

struct ResGroup {
  int device = 0;
  bool local = true;
  int shard_lo = 0, shard_hi = 0;  // global shard indices of the group
  std::vector<otprg_ctx*> shards;  // local groups: their contexts, ascending shard index
  char* base = nullptr;            // exchange block (own allocation, peer or IPC mapping)
  DevBuf own;
  bool ipc_mapped = false;
  cudaStream_t cap_stream = nullptr;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaEvent_t ev[2] = {nullptr, nullptr};
  ~ResGroup() {
    if (local || ipc_mapped) cudaSetDevice(device);
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    if (cap_stream) cudaStreamDestroy(cap_stream);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    if (ipc_mapped && base) cudaIpcCloseMemHandle(base);
  }
};

struct ResPlan {
  std::vector<otprg_ctx*> key;
  std::vector<uint64_t> gens;
  int n_shards = 0, ib = 0, K = 0, my_group = -1;
  XLayout lay;
  std::vector<std::unique_ptr<ResGroup>> groups;  // every group of the solve (local and remote)
  bool built = false;
};

int plan_fail(otprg_ctx* ctx, const std::string& m) { return fail(ctx, OTPRG_PARAMETER, m); }

// Groups of the local shards: consecutive shard indices on one device.  A
// device may appear in one group only (two groups on one GPU would make its
// kernels wait on each other).
int make_local_groups(otprg_ctx* err_ctx, otprg_ctx** shards, int n, ResPlan& P) {
  std::vector<otprg_ctx*> v(shards, shards + n);
  std::sort(v.begin(), v.end(), [](otprg_ctx* a, otprg_ctx* b) { return a->sh_shard < b->sh_shard; });
  for (size_t i = 0; i < v.size(); ++i) {
    otprg_ctx* c = v[i];
    if (!c || !c->sharded || !c->prepared) return plan_fail(err_ctx, "shard context not prepared (otprg_shard_prepare)");
    if (c->sh_n_shards != v[0]->sh_n_shards || c->ib != v[0]->ib || c->ia != v[0]->ia || c->sh_K != v[0]->sh_K ||
        c->width != v[0]->width || c->eps != v[0]->eps || c->sh_otf != v[0]->sh_otf)
      return plan_fail(err_ctx, "shard contexts were prepared for different problems");
    if (i > 0 && c->sh_shard == v[i - 1]->sh_shard) return plan_fail(err_ctx, "shard index given twice");
    if (i > 0 && c->sh_shard != v[i - 1]->sh_shard + 1 && c->device == v[i - 1]->device)
      return plan_fail(err_ctx, "the shards of one device must be consecutive");
    if (P.groups.empty() || P.groups.back()->device != c->device || c->sh_shard != P.groups.back()->shard_hi) {
      for (auto& g : P.groups)
        if (g->device == c->device) return plan_fail(err_ctx, "the shards of one device must be consecutive");
      P.groups.emplace_back(new ResGroup());
      P.groups.back()->device = c->device;
      P.groups.back()->shard_lo = c->sh_shard;
      P.groups.back()->shard_hi = c->sh_shard;
    }
    P.groups.back()->shards.push_back(c);
    P.groups.back()->shard_hi = c->sh_shard + 1;
  }
  P.n_shards = v[0]->sh_n_shards;
  P.ib = v[0]->ib;
  P.K = v[0]->sh_K;
  P.lay = XLayout(P.n_shards, P.ib, P.K);
  return OTPRG_OK;
}

int alloc_block(otprg_ctx* ctx, ResGroup& g, const XLayout& lay) {
  CK(cudaSetDevice(g.device), "cudaSetDevice");
  CK(g.own.ensure(lay.bytes), "alloc exchange block");
  CK(cudaMemset(g.own.p, 0, lay.bytes), "memset exchange block");
  g.base = static_cast<char*>(g.own.p);
  return OTPRG_OK;
}

// Captures one group's loop body into a WHILE node and instantiates it.
int build_graph(otprg_ctx* ctx, ResPlan& P, ResGroup& g, int gi) {
  CK(cudaSetDevice(g.device), "cudaSetDevice");
  if (!g.cap_stream) CK(cudaStreamCreateWithFlags(&g.cap_stream, cudaStreamNonBlocking), "stream");
  for (auto& e : g.ev)
    if (!e) CK(cudaEventCreate(&e), "event");
  int32_t* xcand = reinterpret_cast<int32_t*>(g.base + P.lay.cand);
  int2* xmeta = reinterpret_cast<int2*>(g.base + P.lay.meta);
  otprg::ShardPeers peers{};
  const int n_groups = static_cast<int>(P.groups.size());
  if (n_groups > 1) {
    if (n_groups - 1 > otprg::kMaxShardPeers || n_groups > kMaxGroups)
      return plan_fail(ctx, "too many device groups for the peer exchange");
    for (int q = 0; q < n_groups; ++q) {
      if (q == gi) continue;
      char* pb = P.groups[q]->base;
      peers.cand[peers.n] = reinterpret_cast<int32_t*>(pb + P.lay.cand);
      peers.meta[peers.n] = reinterpret_cast<int2*>(pb + P.lay.meta);
      peers.flag[peers.n] = reinterpret_cast<uint32_t*>(pb + P.lay.flags);
      ++peers.n;
    }
    peers.my_flags = reinterpret_cast<uint32_t*>(g.base + P.lay.flags);
    peers.arrive = reinterpret_cast<unsigned*>(g.base + P.lay.arrive);
    peers.my_group = gi;
    peers.n_groups = n_groups;
    peers.shard_lo = g.shard_lo;
    peers.shard_hi = g.shard_hi;
  }
  CK(cudaGraphCreate(&g.graph, 0), "graph create");
  cudaGraphConditionalHandle cond;
  CK(cudaGraphConditionalHandleCreate(&cond, g.graph, 1, cudaGraphCondAssignDefault), "conditional handle");
  cudaGraphNodeParams cp{};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = cond;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  CK(cudaGraphAddNode(&node, g.graph, nullptr, 0, &cp), "conditional node");
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  CK(cudaStreamBeginCaptureToGraph(g.cap_stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed),
     "capture");
  int st = OTPRG_OK;
  auto args = [&](otprg_ctx* c) {
    otprg::ShardArgs S = shard_args(c);
    S.cap = P.ib;  // fixed slot stride
    return S;
  };
  for (otprg_ctx* c : g.shards)
    if (otprg::launch_shard_scan(args(c), xcand, xmeta, c->sh_grid, g.cap_stream) != cudaSuccess) st = OTPRG_DEVICE;
  if (n_groups > 1 && otprg::launch_shard_push(args(g.shards[0]), xcand, xmeta, peers, g.cap_stream) != cudaSuccess)
    st = OTPRG_DEVICE;
  for (size_t i = 0; i < g.shards.size(); ++i) {
    otprg_ctx* c = g.shards[i];
    const otprg::ShardArgs S = args(c);
    if (otprg::launch_shard_da(S, xcand, xmeta, c->sh_da_grid, g.cap_stream) != cudaSuccess ||
        otprg::launch_shard_round_end(S, cond, i + 1 == g.shards.size(), g.cap_stream) != cudaSuccess)
      st = OTPRG_DEVICE;
  }
  cudaGraph_t captured = nullptr;
  const cudaError_t ce = cudaStreamEndCapture(g.cap_stream, &captured);
  if (st) return fail(ctx, st, "kernel launch failed during graph capture");
  CK(ce, "end capture");
  CK(cudaGraphInstantiate(&g.exec, g.graph, 0), "graph instantiate");
  return OTPRG_OK;
}

int enable_peers(otprg_ctx* ctx, const ResPlan& P) {
  for (auto& a : P.groups) {
    if (!a->local) continue;
    for (auto& b : P.groups) {
      if (!b->local || a->device == b->device) continue;
      int can = 0;
      CK(cudaDeviceCanAccessPeer(&can, a->device, b->device), "peer query");
      if (!can)
        return fail(ctx, OTPRG_DEVICE, "GPU " + std::to_string(a->device) + " cannot access GPU " +
                                           std::to_string(b->device) + " (no peer path)");
      CK(cudaSetDevice(a->device), "cudaSetDevice");
      const cudaError_t e = cudaDeviceEnablePeerAccess(b->device, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      else if (e != cudaSuccess) return cuda_fail(ctx, e, "enable peer access");
    }
  }
  return OTPRG_OK;
}

std::shared_ptr<ResPlan> plan_of(otprg_ctx* c) { return std::static_pointer_cast<ResPlan>(c->sh_plan); }

bool plan_matches(const ResPlan& P, otprg_ctx** shards, int n) {
  if (!P.built || (int)P.key.size() != n) return false;
  for (int i = 0; i < n; ++i)
    if (P.key[i] != shards[i] || P.gens[i] != shards[i]->sh_gen) return false;
  return true;
}

// One solve on a built plan: begin every local shard, launch every local
// group's graph, complete, export the first shard's results; every local
// shard must end in the same state.
int run_plan(otprg_ctx* ctx, ResPlan& P, otprg_result* res) {
  // every local group runs on its first shard's stream (its other shards'
  // contexts are switched to it for the solve)
  std::vector<ResGroup*> local;
  for (auto& g : P.groups)
    if (g->local) local.push_back(g.get());
  uint32_t epoch = 0;
  for (ResGroup* g : local)
    for (otprg_ctx* c : g->shards) epoch = std::max(epoch, c->sh_epoch);
  struct StreamSwap {  // restores the contexts' own streams on every exit path
    std::vector<std::pair<otprg_ctx*, cudaStream_t>> saved;
    ~StreamSwap() {
      for (auto& s : saved) s.first->stream = s.second;
    }
  } swap;
  for (ResGroup* g : local) {
    cudaStream_t s = g->shards[0]->stream;
    for (otprg_ctx* c : g->shards) {
      if (c->stream != s) {
        CK(cudaSetDevice(c->device), "cudaSetDevice");
        CK(cudaStreamSynchronize(c->stream), "stream");
      }
      swap.saved.emplace_back(c, c->stream);
      c->stream = s;
    }
  }
  int st = OTPRG_OK;
  for (ResGroup* g : local) {
    CK(cudaSetDevice(g->device), "cudaSetDevice");
    CK(cudaEventRecord(g->ev[0], g->shards[0]->stream), "event");
    for (otprg_ctx* c : g->shards)
      if ((st = shard_begin_launch(c, epoch))) return st;
  }
  for (ResGroup* g : local) {
    CK(cudaSetDevice(g->device), "cudaSetDevice");
    CK(cudaGraphLaunch(g->exec, g->shards[0]->stream), "graph launch");
  }
  for (ResGroup* g : local) {
    CK(cudaSetDevice(g->device), "cudaSetDevice");
    for (otprg_ctx* c : g->shards)
      if ((st = launch_finish(c))) return st;
    CK(cudaEventRecord(g->ev[1], g->shards[0]->stream), "event");
  }
  // results of the lowest local shard (its export syncs its group's stream)
  otprg_ctx* first = local[0]->shards[0];
  CK(cudaSetDevice(first->device), "cudaSetDevice");
  Ctl h0{};
  if ((st = export_state(first, res, &h0))) return st;
  double ms = 0.0;
  for (ResGroup* g : local) {
    CK(cudaSetDevice(g->device), "cudaSetDevice");
    CK(cudaEventSynchronize(g->ev[1]), "solve");
    float f = 0.f;
    cudaEventElapsedTime(&f, g->ev[0], g->ev[1]);
    ms = std::max(ms, static_cast<double>(f));
    for (otprg_ctx* c : g->shards) {
      Ctl h{};
      CK(cudaMemcpy(&h, c->ctl.p, sizeof(Ctl), cudaMemcpyDeviceToHost), "D2H ctl");
      if ((st = check_status(c, h, true))) return fail(ctx, st, "shard " + std::to_string(c->sh_shard) + ": " + c->err);
      if (h.phase != h0.phase || h.sum_ni != h0.sum_ni || h.sh_rounds != h0.sh_rounds || h.done != h0.done)
        return fail(ctx, OTPRG_INVARIANT,
                    "shards ended in different states: shard " + std::to_string(c->sh_shard) + " [phase,sum_ni,rounds,done]=" +
                        std::to_string(h.phase) + "," + std::to_string(h.sum_ni) + "," + std::to_string(h.sh_rounds) + "," +
                        std::to_string(h.done) + " vs " + std::to_string(h0.phase) + "," + std::to_string(h0.sum_ni) + "," +
                        std::to_string(h0.sh_rounds) + "," + std::to_string(h0.done) + " [mode,nreq,epoch,live,park,w1,st]=" +
                        std::to_string(h.sh_mode) + "," + std::to_string(h.sh_nreq) + "," + std::to_string(h.sh_epoch) + "," +
                        std::to_string(h.sh_live) + "," + std::to_string(h.sh_park_cur) + "," + std::to_string(h.work[1]) + "," +
                        std::to_string(h.status) + " vs " +
                        std::to_string(h0.sh_mode) + "," + std::to_string(h0.sh_nreq) + "," + std::to_string(h0.sh_epoch) + "," +
                        std::to_string(h0.sh_live) + "," + std::to_string(h0.sh_park_cur) + "," + std::to_string(h0.work[1]) + "," +
                        std::to_string(h0.status) + " sizeof(Ctl)=" + std::to_string(sizeof(Ctl)));
      c->sh_epoch = h.sh_epoch;
    }
  }
  if ((st = check_status(first, h0, true))) return fail(ctx, st, first->err);
  res->solve_ms = ms;
  res->loop_ms = ms;
  res->solve_d2h_ms = ms;
  res->phase1_ms = 0.0;
  res->refill_rounds = h0.sh_rounds;
  res->n_shards = P.n_shards;
  // launches per local shard: init + phase-0 top (top, 2 compaction, ctl) +
  // complete, and per round: scan (1 slab / 2 on the fly) + DA + the
  // cooperative round end; + one push per group and round when there are peers
  int launches = 0;
  const int rounds = static_cast<int>(h0.phase) + h0.sh_rounds;
  for (ResGroup* g : local) {
    for (otprg_ctx* c : g->shards) launches += 6 + rounds * ((c->sh_otf ? 2 : 1) + 2);
    if (P.groups.size() > 1) launches += rounds;
  }
  res->gpu_launches = launches;
  return OTPRG_OK;
}

}  // namespace

extern "C" {

int otprg_shard_prepare(otprg_ctx* ctx, const otprg_problem* p, int32_t n_shards, int32_t shard,
                        int32_t K, int32_t* bounds_out) {
  if (!ctx) return OTPRG_PARAMETER;
  int st = validate_problem(ctx, p);
  if (st) return st;
  if (p->cost_kind != OTPRG_COST_POINTS2D && p->cost_kind != OTPRG_COST_L1_U8)
    return fail(ctx, OTPRG_PARAMETER, "sharded mode builds its slab from 2-D point sets or L1 images");
  if (n_shards < 1 || shard < 0 || shard >= n_shards)
    return fail(ctx, OTPRG_PARAMETER, "bad shard index");
  if (K < 1 || K > 32) return fail(ctx, OTPRG_PARAMETER, "K must lie in [1, 32]");
  CK(cudaSetDevice(ctx->device), "cudaSetDevice");
  ctx->prepared = false;
  ctx->sh_plan.reset();
  ctx->sh_gen += 1;
  ctx->n_a = p->n_a;
  ctx->n_b = p->n_b;
  ctx->swapped = p->n_b > p->n_a;
  ctx->ia = ctx->swapped ? p->n_b : p->n_a;
  ctx->ib = ctx->swapped ? p->n_a : p->n_b;
  ctx->eps = p->eps;
  ctx->cost_kind = p->cost_kind;
  const int64_t uf = host_scaled_floor(1.0, p->eps);
  ctx->unit_floor = static_cast<int32_t>(uf);
  ctx->unit_ceil = static_cast<int32_t>(static_cast<double>(uf) * p->eps == 1.0 ? uf : uf + 1);
  const int64_t need = static_cast<int64_t>(ctx->unit_ceil) + 2;
  const int width = otprg::storage_width(need, p->storage);
  if (width < 0) return fail(ctx, OTPRG_PARAMETER, "eps too small for the device cost storage");
  ctx->width = width;
  // shard boundaries: multiples of 512 elements (aligned t / kT vectors)
  std::vector<int> bounds(n_shards + 1);
  for (int g = 0; g < n_shards; ++g)
    bounds[g] = static_cast<int>((static_cast<int64_t>(ctx->ia) * g / n_shards) / 512 * 512);
  bounds[n_shards] = ctx->ia;
  if (bounds_out)
    for (int g = 0; g <= n_shards; ++g) bounds_out[g] = bounds[g];
  ctx->sharded = true;
  ctx->sh_n_shards = n_shards;
  ctx->sh_shard = shard;
  ctx->sh_lo = bounds[shard];
  ctx->sh_hi = bounds[shard + 1];
  ctx->sh_K = K;
  ctx->sh_cap = ctx->ib;
  const int align = 512 / width;
  const size_t ia = ctx->ia, ib = ctx->ib;
  const int local = std::max(ctx->sh_hi - ctx->sh_lo, 1);
  ctx->lda = (local + align - 1) / align * align;
  const size_t full = (ia + 511) / 512 * 512;
  ctx->sh_otf = (p->flags & OTPRG_FLAG_ON_THE_FLY) != 0;
  if (!ctx->sh_otf) CK(ctx->kT.ensure(ib * ctx->lda * width), "alloc kT slab");
  CK(ctx->t.ensure(full * width), "alloc t");
  CK(ctx->yb.ensure(ib * 4), "alloc yb");
  CK(ctx->ma.ensure(ia * 4), "alloc match_a");
  CK(ctx->mb.ensure(ib * 4), "alloc match_b");
  CK(ctx->holder.ensure(2 * ia * 8), "alloc holder");
  CK(ctx->rowmin.ensure(ib * width), "alloc rowmin");
  CK(ctx->lmeta.ensure(ib * 16), "alloc low-set meta");
  CK(ctx->lists.ensure(3 * ib * 4), "alloc lists");
  CK(ctx->mps.ensure(2 * ib * 8), "alloc mp lists");
  // completion scratch, and the compaction's per-block counts during the phases (>= 148 ints)
  CK(ctx->fa.ensure(std::max<size_t>(ia, 1024) * 4), "alloc scratch");
  CK(ctx->fb.ensure(ib * 4), "alloc scratch");
  CK(ctx->ctl.ensure(sizeof(Ctl)), "alloc ctl");
  CK(ctx->sh_bounds.ensure((n_shards + 1) * sizeof(int)), "alloc bounds");
  CK(ctx->sh_pos.ensure(ib * 4), "alloc pos");
  CK(ctx->sh_list.ensure(ib * 4), "alloc list");
  for (auto& pk : ctx->sh_park) CK(pk.ensure(ib * 16), "alloc park");
  {  // segmented-scan merge buffers; the per-request counters start (and stay) zero
    const size_t seg_words = static_cast<size_t>(otprg::kSegWarps) * (K + 1) + ib;
    CK(ctx->sh_seg.ensure(seg_words * 4), "alloc segment buffers");
    CK(cudaMemsetAsync(ctx->sh_seg.p, 0, seg_words * 4, ctx->stream), "memset segment buffers");
  }
  const double capd = std::ceil((1.0 + 2.0 * p->eps) / (p->eps * p->eps)) + 8.0;
  ctx->fc_cap = static_cast<int64_t>(std::min(capd + 1.0, double(OTPRG_MAX_PHASES)));
  CK(ctx->fc.ensure(ctx->fc_cap * 8), "alloc free_counts");
  CK(cudaMemcpyAsync(ctx->sh_bounds.p, bounds.data(), (n_shards + 1) * sizeof(int),
                     cudaMemcpyHostToDevice, ctx->stream), "H2D bounds");
  if (p->cost_kind == OTPRG_COST_L1_U8) {
    // load_mnist_pair's cost (instances.cpp:114-142): normalised pixels (K3a) of
    // both sides; the slab by K3b, or on the fly (the scans sum the pixel
    // differences themselves) after a device pass of the reference's range check
    const size_t dim = static_cast<size_t>(p->dim);
    const uint8_t* ia_img = ctx->swapped ? p->img_b : p->img_a;
    const uint8_t* ib_img = ctx->swapped ? p->img_a : p->img_b;
    const size_t raw_off = (ia + ib) * dim * sizeof(double);
    const size_t xt_off = (raw_off + (ia + ib) * dim + 255) / 256 * 256;
    CK(ctx->pts.ensure(xt_off + (ctx->sh_otf ? ia * dim * sizeof(double) : 0)), "alloc images");
    double* xa = ctx->pts.as<double>();
    double* yb = xa + ia * dim;
    uint8_t* raw = static_cast<uint8_t*>(ctx->pts.p) + raw_off;
    CK(cudaEventRecord(ctx->ev[4], ctx->stream), "event");
    CK(cudaMemcpyAsync(raw, ia_img, ia * dim, cudaMemcpyHostToDevice, ctx->stream), "H2D images");
    CK(cudaMemcpyAsync(raw + ia * dim, ib_img, ib * dim, cudaMemcpyHostToDevice, ctx->stream), "H2D images");
    CK(cudaMemsetAsync(ctx->ctl.p, 0, sizeof(Ctl), ctx->stream), "memset");
    int* status = &ctx->ctl.as<Ctl>()->status;
    CK(otprg::launch_l1_normalize(raw, static_cast<int>(ia + ib), p->dim, xa, status, ctx->stream), "l1 normalize");
    if (ctx->sh_otf) {
      CK(ctx->l1_mask.ensure(otprg::l1_mask_bytes(ctx->ia, ctx->ib, ctx->ia, p->dim)), "alloc masks");
      CK(otprg::launch_l1_check(xa, yb, ctx->ia, ctx->ib, p->dim, status, ctx->stream, ctx->l1_mask.as<uint32_t>()),
         "l1 check");
      CK(otprg::launch_transpose_f64(xa, ctx->ia, p->dim,
                                     reinterpret_cast<double*>(static_cast<char*>(ctx->pts.p) + xt_off), ctx->stream),
         "transpose");
      const size_t nw = (dim + 31) / 32, groups = (ctx->sh_hi - ctx->sh_lo + 31) / 32;
      CK(ctx->l1_otf_mask.ensure((groups + ib) * nw * 4 + 4), "alloc masks");
      uint32_t* gm = ctx->l1_otf_mask.as<uint32_t>();
      CK(otprg::launch_l1_group_masks(xa + static_cast<size_t>(ctx->sh_lo) * dim, ctx->sh_hi - ctx->sh_lo, p->dim, 32,
                                      gm, ctx->stream),
         "group masks");
      CK(otprg::launch_l1_group_masks(yb, static_cast<int>(ib), p->dim, 1, gm + groups * nw, ctx->stream),
         "image masks");
    } else if (ctx->sh_hi > ctx->sh_lo) {
      CK(ctx->l1_mask.ensure(otprg::l1_mask_bytes(ctx->sh_hi - ctx->sh_lo, ctx->ib, ctx->lda, p->dim)), "alloc masks");
      CK(otprg::launch_l1_round(xa + static_cast<size_t>(ctx->sh_lo) * dim, yb, ctx->sh_hi - ctx->sh_lo, ctx->ib,
                                p->dim, p->eps, ctx->kT.p, ctx->lda, width, status, ctx->stream,
                                ctx->l1_mask.as<uint32_t>()),
         "l1 round");
    }
    int dstatus = 0;
    CK(cudaMemcpyAsync(&dstatus, status, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream), "D2H status");
    CK(cudaStreamSynchronize(ctx->stream), "image slab build");
    if (dstatus == OTPRG_PARAMETER) return fail(ctx, OTPRG_PARAMETER, "cost entry outside [0,1]");
    if (dstatus == OTPRG_INPUT) return fail(ctx, OTPRG_INPUT, "image has zero total intensity");
    if (dstatus) return fail(ctx, dstatus, "cost build failed");
    ctx->img_dim = p->dim;
    ctx->sh_l1_xt = xt_off;
    ctx->sh_thr_n = 0;
  } else {
    // this shard's slab of kT from the points (K2 on the demand range)
    const double* pa = ctx->swapped ? p->pts_b : p->pts_a;
    const double* pb = ctx->swapped ? p->pts_a : p->pts_b;
    CK(ctx->pts.ensure((ia + ib) * 2 * sizeof(double)), "alloc points");
    double* dpa = ctx->pts.as<double>();
    double* dpb = dpa + ia * 2;
    CK(cudaMemcpyAsync(dpa, pa, ia * 2 * sizeof(double), cudaMemcpyHostToDevice, ctx->stream), "H2D");
    CK(cudaMemcpyAsync(dpb, pb, ib * 2 * sizeof(double), cudaMemcpyHostToDevice, ctx->stream), "H2D");
    CK(cudaEventRecord(ctx->ev[4], ctx->stream), "event");
    if ((st = check_points_range(ctx, p, ctx->swapped ? dpb : dpa, ctx->swapped ? dpa : dpb))) return st;
    int thr_n = 0;
    if ((st = points_table(ctx, p->eps, &thr_n))) return st;
    if (ctx->sh_otf) {  // the exact threshold table replaces the slab
      if (thr_n == 0)
        return fail(ctx, OTPRG_PARAMETER, "on-the-fly costs need 1/eps <= 8190 (threshold table in shared memory)");
      ctx->sh_thr_n = thr_n;
      ctx->sh_otf_tiled = otprg::shard_otf_tiled_fits(width, thr_n, ctx->device);
    } else if (ctx->sh_hi > ctx->sh_lo) {
      const size_t fix_bytes = otprg::round_points_fix_bytes(ctx->sh_hi - ctx->sh_lo, ctx->ib, ctx->lda, width,
                                                             p->eps, ctx->pts_absmax);
      CK(ctx->k2_fix.ensure(fix_bytes), "alloc K2 fix-up list");
      CK(otprg::launch_round_points2d(dpa + static_cast<size_t>(ctx->sh_lo) * 2, dpb, ctx->sh_hi - ctx->sh_lo,
                                      ctx->ib, p->eps, std::sqrt(2.0), thr_n ? ctx->thr_dev.as<double>() : nullptr,
                                      thr_n, ctx->pts_absmax, ctx->kT.p, ctx->lda, width, ctx->k2_fix.p, fix_bytes,
                                      ctx->stream),
         "round_points launch");
    }
  }
  CK(cudaEventRecord(ctx->ev[5], ctx->stream), "event");
  CK(cudaStreamSynchronize(ctx->stream), "slab build");
  float ms = 0.f;
  cudaEventElapsedTime(&ms, ctx->ev[4], ctx->ev[5]);
  ctx->build_ms = ms;
  if (p->cost_kind == OTPRG_COST_POINTS2D) {
    ctx->pts_a.assign(p->pts_a, p->pts_a + 2 * static_cast<size_t>(p->n_a));
    ctx->pts_b.assign(p->pts_b, p->pts_b + 2 * static_cast<size_t>(p->n_b));
  }
  {
    const otprg::ShardArgs S = shard_args(ctx);
    ctx->sh_grid = otprg::shard_scan_grid(S, ctx->num_sms);
    ctx->sh_da_grid = ctx->num_sms * 8;
  }
  ctx->prepared = true;
  return OTPRG_OK;
}

int otprg_shard_begin(otprg_ctx* ctx) {
  if (!ctx) return OTPRG_PARAMETER;
  if (!ctx->prepared || !ctx->sharded) return fail(ctx, OTPRG_PARAMETER, "otprg_shard_prepare() first");
  return shard_begin_launch(ctx, ctx->sh_epoch);
}

int otprg_shard_top(otprg_ctx* ctx, int32_t* n_out, int32_t* finished) {
  if (!ctx) return OTPRG_PARAMETER;
  if (!ctx->begun || !ctx->sharded) return fail(ctx, OTPRG_PARAMETER, "otprg_shard_begin() first");
  if (!ctx->sh_have) {
    Ctl h{};
    const int st = read_ctl(ctx, &h);
    if (st) return st;
    cache_round(ctx, h);
  }
  if (ctx->sh_parked) return fail(ctx, OTPRG_PARAMETER, "chains are parked: rescan and resume first");
  if (n_out) *n_out = ctx->sh_n;
  if (finished) *finished = ctx->sh_done;
  return OTPRG_OK;
}

int otprg_shard_scan(otprg_ctx* ctx, int32_t* cand, int32_t* meta_words, int32_t cap, int32_t refill) {
  int2* meta = reinterpret_cast<int2*>(meta_words);
  if (!ctx) return OTPRG_PARAMETER;
  if (!ctx->begun || !ctx->sharded || !ctx->sh_have) return fail(ctx, OTPRG_PARAMETER, "otprg_shard_top() first");
  if ((refill != 0) != (ctx->sh_parked > 0)) return fail(ctx, OTPRG_PARAMETER, "refill flag does not match the round");
  // cap = slots per shard in the exchange buffers: >= the round's requests
  // (the caller passes n_i so the all-gather moves only the used prefix)
  if (cap < ctx->sh_n || cap > ctx->sh_cap) return fail(ctx, OTPRG_PARAMETER, "bad exchange slot count");
  otprg::ShardArgs S = shard_args(ctx);
  S.cap = cap;
  CK(otprg::launch_shard_scan(S, cand, meta, ctx->sh_grid, ctx->stream), "shard_scan launch");
  // no sync: the exchange and the DA are ordered after the scan on the
  // context's stream (otprg_set_stream puts every rank of a process and the
  // NCCL all-gather on one stream)
  return OTPRG_OK;
}

int otprg_shard_da(otprg_ctx* ctx, const int32_t* cand, const int32_t* meta_words, int32_t cap,
                   int32_t resume, int32_t* parked) {
  const int2* meta = reinterpret_cast<const int2*>(meta_words);
  if (!ctx) return OTPRG_PARAMETER;
  if (!ctx->begun || !ctx->sharded || !ctx->sh_have) return fail(ctx, OTPRG_PARAMETER, "otprg_shard_top() first");
  if ((resume != 0) != (ctx->sh_parked > 0)) return fail(ctx, OTPRG_PARAMETER, "resume flag does not match the round");
  otprg::ShardArgs S = shard_args(ctx);
  S.cap = cap;
  CK(otprg::launch_shard_da(S, cand, meta, ctx->sh_da_grid, ctx->stream), "shard_da launch");
  // complete phase -> its top (apply M', termination, next free list); then
  // the round bookkeeping — all decided on the device
  CK(otprg::launch_shard_round_end(S, cudaGraphConditionalHandle{}, false, ctx->stream), "shard round-end launch");
  Ctl h{};
  const int st = read_ctl(ctx, &h);
  if (st) return st;
  cache_round(ctx, h);
  if (parked) *parked = ctx->sh_parked;
  return OTPRG_OK;
}

int otprg_shard_finish(otprg_ctx* ctx, otprg_result* res) {
  if (!ctx) return OTPRG_PARAMETER;
  if (!res || !res->match_of_a || !res->match_of_b)
    return fail(ctx, OTPRG_PARAMETER, "result buffers are null");
  int st = launch_finish(ctx);
  if (st) return st;
  Ctl h{};
  if ((st = export_state(ctx, res, &h))) return st;
  res->build_ms = ctx->build_ms;
  ctx->sh_epoch = h.sh_epoch;
  return check_status(ctx, h, true);
}

int otprg_shard_solve_resident(otprg_ctx** shards, int32_t n, otprg_result* res) {
  if (!shards || n < 1 || !shards[0]) return OTPRG_PARAMETER;
  otprg_ctx* ctx = shards[0];
  if (!res || !res->match_of_a || !res->match_of_b) return fail(ctx, OTPRG_PARAMETER, "result buffers are null");
  std::shared_ptr<ResPlan> P = plan_of(ctx);
  if (!P || !(plan_matches(*P, shards, n) || (P->my_group >= 0 && n == 1 && P->built))) {
    // in-process plan: the local shards must cover every shard
    P = std::make_shared<ResPlan>();
    int st = make_local_groups(ctx, shards, n, *P);
    if (st) return st;
    if (n != P->n_shards)
      return fail(ctx, OTPRG_PARAMETER, "the shards of this process do not cover all " +
                                            std::to_string(P->n_shards) + " shards (multi-process: "
                                            "otprg_shard_ipc_export / otprg_shard_ipc_attach first)");
    if ((st = enable_peers(ctx, *P))) return st;
    for (auto& g : P->groups)
      if ((st = alloc_block(ctx, *g, P->lay))) return st;
    for (size_t gi = 0; gi < P->groups.size(); ++gi)
      if ((st = build_graph(ctx, *P, *P->groups[gi], static_cast<int>(gi)))) return st;
    for (int i = 0; i < n; ++i) {
      P->key.push_back(shards[i]);
      P->gens.push_back(shards[i]->sh_gen);
    }
    P->built = true;
    ctx->sh_plan = P;
  }
  const int st = run_plan(ctx, *P, res);
  res->build_ms = ctx->build_ms;
  return st;
}

// ---- multi-process resident mode (one process per GPU, CUDA IPC) -----------

int otprg_shard_ipc_export(otprg_ctx* ctx, int32_t n_groups, int32_t my_group, void* handle_out) {
  if (!ctx || !handle_out) return OTPRG_PARAMETER;
  if (!ctx->prepared || !ctx->sharded) return fail(ctx, OTPRG_PARAMETER, "otprg_shard_prepare() first");
  if (n_groups < 1 || n_groups > kMaxGroups || my_group < 0 || my_group >= n_groups)
    return fail(ctx, OTPRG_PARAMETER, "bad group count / index");
  auto P = std::make_shared<ResPlan>();
  P->n_shards = ctx->sh_n_shards;
  P->ib = ctx->ib;
  P->K = ctx->sh_K;
  P->lay = XLayout(P->n_shards, P->ib, P->K);
  P->my_group = my_group;
  for (int q = 0; q < n_groups; ++q) P->groups.emplace_back(new ResGroup());
  ResGroup& me = *P->groups[my_group];
  me.device = ctx->device;
  me.shards.push_back(ctx);
  me.shard_lo = ctx->sh_shard;
  me.shard_hi = ctx->sh_shard + 1;
  int st = alloc_block(ctx, me, P->lay);
  if (st) return st;
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, me.base), "IPC handle");
  static_assert(sizeof(cudaIpcMemHandle_t) == OTPRG_IPC_HANDLE_BYTES, "IPC handle size");
  std::memcpy(handle_out, &h, sizeof(h));
  P->key.push_back(ctx);
  P->gens.push_back(ctx->sh_gen);
  ctx->sh_plan = P;
  return OTPRG_OK;
}

int otprg_shard_ipc_attach(otprg_ctx* ctx, const void* handles, int32_t n_groups, const int32_t* group_shard_lo) {
  if (!ctx || !handles || !group_shard_lo) return OTPRG_PARAMETER;
  std::shared_ptr<ResPlan> P = plan_of(ctx);
  if (!P || P->my_group < 0 || (int)P->groups.size() != n_groups || P->gens[0] != ctx->sh_gen)
    return fail(ctx, OTPRG_PARAMETER, "otprg_shard_ipc_export() first (same group count)");
  CK(cudaSetDevice(ctx->device), "cudaSetDevice");
  for (int q = 0; q < n_groups; ++q) {
    ResGroup& g = *P->groups[q];
    g.shard_lo = group_shard_lo[q];
    g.shard_hi = q + 1 < n_groups ? group_shard_lo[q + 1] : P->n_shards;
    if (q == P->my_group) {
      if (g.shard_lo != ctx->sh_shard || g.shard_hi != ctx->sh_shard + 1)
        return fail(ctx, OTPRG_PARAMETER, "group shard ranges do not match this context's shard");
      continue;
    }
    g.local = false;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, static_cast<const char*>(handles) + (size_t)q * OTPRG_IPC_HANDLE_BYTES, sizeof(h));
    void* p = nullptr;
    CK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess), "IPC open");
    g.base = static_cast<char*>(p);
    g.ipc_mapped = true;
    g.device = ctx->device;  // (mapping lives in this process's context on our device)
  }
  int st = build_graph(ctx, *P, *P->groups[P->my_group], P->my_group);
  if (st) return st;
  P->built = true;
  return OTPRG_OK;
}

int otprg_create_multi(const int32_t* devices, int32_t ndev, otprg_ctx** out) {
  if (!out || !devices || ndev < 1) return OTPRG_PARAMETER;
  *out = nullptr;
  otprg_ctx* root = nullptr;
  int st = otprg_create(devices[0], &root);
  if (st) return st;
  for (int i = 0; i < ndev; ++i) {
    otprg_ctx* c = nullptr;
    if ((st = otprg_create(devices[i], &c))) {
      otprg_destroy(root);
      return st;
    }
    root->multi.push_back(c);
  }
  *out = root;
  return OTPRG_OK;
}

int otprg_selftest_exchange(int32_t device, int32_t n_groups, int32_t shards_per_group, int32_t ib, int32_t K,
                            int32_t rounds, int64_t* mismatches) {
  if (!mismatches || n_groups < 2 || n_groups > 1 + otprg::kMaxShardPeers || shards_per_group < 1 || ib < 1 ||
      K < 1 || rounds < 1)
    return OTPRG_PARAMETER;
  *mismatches = 0;
  if (cudaSetDevice(device) != cudaSuccess) return OTPRG_DEVICE;
  const int G = n_groups * shards_per_group;
  const XLayout lay(G, ib, K);
  std::vector<DevBuf> blocks(n_groups), ctls(n_groups);
  DevBuf dS, dP, dC, dM;
  auto pat = [](int r, int g, int i, int k) { return static_cast<int32_t>((r * 7919 + g * 131 + i) * 33 + k); };
  auto mpat = [](int r, int g, int i) { return make_int2(r * 1000 + g, i * 3 + 1); };
  for (int q = 0; q < n_groups; ++q) {
    if (blocks[q].ensure(lay.bytes) != cudaSuccess || ctls[q].ensure(sizeof(Ctl)) != cudaSuccess) return OTPRG_DEVICE;
    cudaMemset(blocks[q].p, 0, lay.bytes);
  }
  if (dS.ensure(n_groups * sizeof(otprg::ShardArgs)) || dP.ensure(n_groups * sizeof(otprg::ShardPeers)) ||
      dC.ensure(n_groups * sizeof(void*)) || dM.ensure(n_groups * sizeof(void*)))
    return OTPRG_DEVICE;
  std::vector<int32_t> hc(static_cast<size_t>(G) * ib * K);
  std::vector<int2> hm(static_cast<size_t>(G) * ib);
  for (int r = 0; r < rounds; ++r) {
    const int nreq = std::max(1, ib - r * (ib / (rounds + 1)));
    std::vector<otprg::ShardArgs> S(n_groups);
    std::vector<otprg::ShardPeers> P(n_groups);
    std::vector<const int32_t*> C(n_groups);
    std::vector<const int2*> M(n_groups);
    for (int q = 0; q < n_groups; ++q) {
      char* base = static_cast<char*>(blocks[q].p);
      // this group's local slots (shards [q*spg, (q+1)*spg)); the rest of its block is stale
      for (int g = q * shards_per_group; g < (q + 1) * shards_per_group; ++g)
        for (int i = 0; i < ib; ++i) {
          for (int k = 0; k < K; ++k) hc[((size_t)g * ib + i) * K + k] = pat(r, g, i, k);
          hm[(size_t)g * ib + i] = mpat(r, g, i);
        }
      const size_t g0 = (size_t)q * shards_per_group;
      cudaMemcpy(base + lay.cand + g0 * ib * K * 4, hc.data() + g0 * ib * K, (size_t)shards_per_group * ib * K * 4,
                 cudaMemcpyHostToDevice);
      cudaMemcpy(base + lay.meta + g0 * ib * 8, hm.data() + g0 * ib, (size_t)shards_per_group * ib * 8,
                 cudaMemcpyHostToDevice);
      Ctl h{};
      h.sh_nreq = nreq;
      h.sh_live = 1;
      h.sh_epoch = static_cast<uint32_t>(r);
      cudaMemcpy(ctls[q].p, &h, sizeof(h), cudaMemcpyHostToDevice);
      S[q].ctl = ctls[q].as<Ctl>();
      S[q].K = K;
      S[q].cap = ib;
      C[q] = reinterpret_cast<const int32_t*>(base + lay.cand);
      M[q] = reinterpret_cast<const int2*>(base + lay.meta);
      P[q].my_group = q;
      P[q].n_groups = n_groups;
      P[q].shard_lo = q * shards_per_group;
      P[q].shard_hi = (q + 1) * shards_per_group;
      P[q].my_flags = reinterpret_cast<uint32_t*>(base + lay.flags);
      P[q].arrive = reinterpret_cast<unsigned*>(base + lay.arrive);
      for (int o = 0; o < n_groups; ++o) {
        if (o == q) continue;
        char* ob = static_cast<char*>(blocks[o].p);
        P[q].cand[P[q].n] = reinterpret_cast<int32_t*>(ob + lay.cand);
        P[q].meta[P[q].n] = reinterpret_cast<int2*>(ob + lay.meta);
        P[q].flag[P[q].n] = reinterpret_cast<uint32_t*>(ob + lay.flags);
        ++P[q].n;
      }
    }
    cudaMemcpy(dS.p, S.data(), n_groups * sizeof(S[0]), cudaMemcpyHostToDevice);
    cudaMemcpy(dP.p, P.data(), n_groups * sizeof(P[0]), cudaMemcpyHostToDevice);
    cudaMemcpy(dC.p, C.data(), n_groups * sizeof(void*), cudaMemcpyHostToDevice);
    cudaMemcpy(dM.p, M.data(), n_groups * sizeof(void*), cudaMemcpyHostToDevice);
    if (otprg::launch_shard_push_emulated(dS.as<otprg::ShardArgs>(), dC.as<const int32_t*>(), dM.as<const int2*>(),
                                          dP.as<otprg::ShardPeers>(), n_groups, 4, nullptr) != cudaSuccess ||
        cudaDeviceSynchronize() != cudaSuccess)
      return OTPRG_DEVICE;
    // every group's block must now hold every shard's slots of this round
    std::vector<int32_t> gc(hc.size());
    std::vector<int2> gm(hm.size());
    std::vector<uint32_t> gf(n_groups);
    for (int q = 0; q < n_groups; ++q) {
      const char* base = static_cast<const char*>(blocks[q].p);
      cudaMemcpy(gc.data(), base + lay.cand, gc.size() * 4, cudaMemcpyDeviceToHost);
      cudaMemcpy(gm.data(), base + lay.meta, gm.size() * 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(gf.data(), base + lay.flags, n_groups * 4, cudaMemcpyDeviceToHost);
      Ctl h{};
      cudaMemcpy(&h, ctls[q].p, sizeof(h), cudaMemcpyDeviceToHost);
      if (h.status) ++*mismatches;
      for (int g = 0; g < G; ++g)
        for (int i = 0; i < nreq; ++i) {
          for (int k = 0; k < K; ++k)
            if (gc[((size_t)g * ib + i) * K + k] != pat(r, g, i, k)) ++*mismatches;
          const int2 m = gm[(size_t)g * ib + i], w = mpat(r, g, i);
          if (m.x != w.x || m.y != w.y) ++*mismatches;
        }
      for (int o = 0; o < n_groups; ++o)
        if (o != q && gf[o] != static_cast<uint32_t>(r + 1)) ++*mismatches;
    }
  }
  return cudaGetLastError() == cudaSuccess ? OTPRG_OK : OTPRG_DEVICE;
}

int otprg_set_shard_k(otprg_ctx* ctx, int32_t K) {
  if (!ctx) return OTPRG_PARAMETER;
  if (K < 1 || K > 32) return fail(ctx, OTPRG_PARAMETER, "K must lie in [1, 32]");
  ctx->multi_K = K;
  return OTPRG_OK;
}

}  // extern "C"

// ---- multi-device context (otprg_create_multi) -------------------------------
namespace otprg_capi {

// Point instances are sharded over the context's devices; anything else runs
// on its first device (the root context itself).
int multi_prepare(otprg_ctx* ctx, const otprg_problem* p) {
  ctx->multi_prepared = false;
  if (!p || p->cost_kind != OTPRG_COST_POINTS2D) return OTPRG_OK;
  const int G = static_cast<int>(ctx->multi.size());
  for (int g = 0; g < G; ++g) {
    otprg_ctx* c = ctx->multi[g];
    const int st = otprg_shard_prepare(c, p, G, g, ctx->multi_K, nullptr);
    if (st) return fail(ctx, st, c->err);
  }
  ctx->multi_prepared = true;
  ctx->build_ms = 0.0;
  for (otprg_ctx* c : ctx->multi) ctx->build_ms = std::max(ctx->build_ms, c->build_ms);
  return OTPRG_OK;
}

int multi_solve(otprg_ctx* ctx, otprg_result* res) {
  const int st = otprg_shard_solve_resident(ctx->multi.data(), static_cast<int32_t>(ctx->multi.size()), res);
  if (st) return fail(ctx, st, ctx->multi[0]->err);
  res->build_ms = ctx->build_ms;
  return OTPRG_OK;
}

}  // namespace otprg_capi
