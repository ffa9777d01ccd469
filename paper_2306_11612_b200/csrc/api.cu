// api.cu -- the C ABI (include/dvl.h): argument validation, context state, device memory,
// stream ordering and per-phase CUDA-event timing.  Every compute step is a kernel from
// hilbert.cu / sort.cu / build.cu / update.cu; this file only orchestrates them.
#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include "dvl_common.cuh"
#include "dvl_internal.h"

using namespace dvl;

namespace {

enum Phase { PH_INGEST, PH_ENCODE, PH_SORT, PH_GATHER, PH_MAXV, PH_WSCAN, PH_BREDUCE, PH_EPI,
             PH_BOUND, PH_N };

struct Dataset {
  int64_t n = 0, n_pad = 0;
  int M = 0, b = 0, Lmax = 0, key_bytes = 4, passes = 0, items = 16, tiles = 0;
  uint32_t E = 0;
  void* keys = nullptr;                 // sorted codes (n x key_bytes)
  uint32_t* perm = nullptr;             // input id of each sorted cell
  unsigned long long* gids = nullptr;   // distributed build: global input id of each cell
  uint8_t* level_s = nullptr;           // n_pad
  float* scal_s = nullptr;              // M x n_pad
  std::vector<float> vmin, vmax;        // member data ranges (finite values)
  // per-dataset update state
  float* d_vmin = nullptr;              // M
  float* d_vmax = nullptr;
  float* d_lo = nullptr;                // M
  float* d_inv = nullptr;
  float4* d_rgba = nullptr;             // M x N
  float2* d_tab = nullptr;              // M x N
  unsigned long long* status1 = nullptr;  // tiles
  unsigned long long* tile_prefix = nullptr;
  // persistent TMA path (M <= 16)
  bool tma = false;
  TmaPlan plan{};
  int grid = 0;                           // pass-2 chunks = CTAs
  int grid1 = 0;                          // pass-1 chunks = CTAs (look-back granularity)
  // edit-cache pass 1 at M > 8: its stage holds 13 B per cell, not 4M + 1, so it runs as
  // several CTAs per SM (as many consumer warps per SM as the M <= 4 configuration), with
  // its own chunks; pass 2 takes the chunking of the pass 1 that ran last
  TmaPlan plan_c{};
  int grid1_c = 0;
  bool plan_c_ok = false;
  bool last_c = false;
  int planN = 0;                          // TF size the plan was made for
  int chunk_cap = 0;
  unsigned long long* chunk_status = nullptr;   // grid + 1 (last slot: chunk counter)
  unsigned long long* chunk_prefix = nullptr;   // grid
  unsigned long long* tile_meta = nullptr;      // n_pad / 128: pass-1 q sum of every warp tile
  unsigned long long* meta2 = nullptr;          // n_pad / 128: the warp's running q sum in its
                                                // pass-1 chunk before the warp tile's tile
  void* agg = nullptr;                          // D3: per warp tile and member t statistics
  unsigned long long* blist = nullptr;          // 2 x n_pad / 128: listed boundary warp tiles (+ the job list)
  uint32_t* bctr = nullptr;                     // their counts + done counters (self-resetting)
  // edit cache (TMA path, M >= 3): per cell the min / max of the alpha bits of the members
  // other than cache_member, valid while their TFs and the domains stay as they were
  uint32_t* cmin = nullptr;
  uint32_t* cmax = nullptr;
  int cache_member = -1;
};

}  // namespace

struct dvl_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  dvl_alloc_fn alloc = nullptr;
  dvl_free_fn free = nullptr;
  void* user = nullptr;
  uint32_t flags = 0;
  std::string err;
  std::unordered_map<void*, size_t> live;
  size_t bytes = 0;

  bool built = false;
  Dataset ds;
  std::vector<float> lo_h, hi_h, inv_h;  // domains
  int N = 256;
  float P = 1.0f, eps = 0.025f;
  int mode = DVL_MAXV_CONSERVATIVE;
  int shift = 0;

  // small persistent device state
  float* d_maxv = nullptr;
  unsigned long long* d_qtot = nullptr;
  uint32_t* d_ctr1 = nullptr;
  uint32_t* d_err = nullptr;
  float* h_stage = nullptr;          // pinned + mapped: two TF buffers (kMaxN x 4 floats each)
  float* d_hstage = nullptr;         // its device alias (read by the prologue kernel)
  cudaEvent_t stage_ev[2] = {nullptr, nullptr};   // staging buffer i is free once this completes
  int stage_par = 0;
  uint16_t* d_t1 = nullptr;
  uint16_t* d_t2 = nullptr;
  int nstates = 0;

  // accumulators / outputs
  uint32_t accW = 0;
  int accM = 0;
  Acc acc{};
  dvl_vertex* d_out = nullptr;
  unsigned long long* d_bin_lo = nullptr;
  unsigned long long* d_bin_hi = nullptr;
  uint32_t last_W = 0;

  cudaEvent_t ev[PH_N][2] = {};
  bool ev_used[PH_N] = {};
  int sort_passes = 0;
  int launches = 0;
  int num_sms = 148;
  int acc_par = 0;                        // which lo / hi copy the next call uses
  uint32_t acc_dirty[2] = {0, 0};         // per lo / hi copy: pixels [0, w) not yet restored
  bool volume = false;                    // dvl_set_level_scale: weights by cell volume
  // dvl_set_comm / dvl_set_local_comm: the context's own communicator over the shards;
  // dvl_build then runs the distributed sample sort and dvl_get_polylines the sharded edit
  // (both exchanges) itself
  Comm* comm = nullptr;
  int comm_ranks = 0, comm_rank = 0;
  unsigned long long* d_totals = nullptr;   // [comm_ranks]
  int64_t* d_export = nullptr;              // the accumulator export, merged in place
  uint64_t export_cap = 0;
  bool edit_cache = true;                 // DVL_FLAG_NO_EDIT_CACHE: every edit reads every member
  int pass2_mode = 0;                     // 0 auto, 1 boundary tiles inline, 2 listed, 3 jobs (flags)
  uint32_t prod_sleep = 1000000;          // producer wait hint (ns)
  int stages_override = 0;
  int dbg = 0;                // experiment: pass-2 ring depth

  // sharding (dvl_set_global_bits / dvl_set_shard)
  int global_bits = 0;
  bool sharded = false;
  uint64_t cell_offset = 0, n_global = 0;
  int lmax_global = 0;
  unsigned long long* d_offset = nullptr;      // global scan offset of this shard
  unsigned long long* d_qtot_glob = nullptr;   // global Qtot
};

namespace {

struct Fail {
  dvl_status s;
};

void set_err(dvl_ctx* c, const std::string& m) {
  if (c) c->err = m;
}

#define CK(expr)                                                                     \
  do {                                                                               \
    cudaError_t _e = (expr);                                                         \
    if (_e != cudaSuccess) {                                                         \
      set_err(ctx, std::string(#expr) + ": " + cudaGetErrorString(_e));              \
      throw Fail{DVL_E_CUDA};                                                        \
    }                                                                                \
  } while (0)

#define CKLAUNCH()                                                                   \
  do {                                                                               \
    cudaError_t _e = cudaGetLastError();                                             \
    if (_e != cudaSuccess) {                                                         \
      set_err(ctx, std::string("kernel launch: ") + cudaGetErrorString(_e));         \
      throw Fail{DVL_E_CUDA};                                                        \
    }                                                                                \
    ++ctx->launches;                                                                 \
  } while (0)

[[noreturn]] void fail(dvl_ctx* ctx, dvl_status s, const std::string& m) {
  set_err(ctx, m);
  throw Fail{s};
}

void* dmalloc(dvl_ctx* ctx, size_t bytes) {
  if (bytes == 0) bytes = 16;
  bytes = (bytes + 255) & ~(size_t)255;
  void* p = nullptr;
  if (ctx->alloc) {
    p = ctx->alloc(bytes, (void*)ctx->stream, ctx->user);
    if (!p) fail(ctx, DVL_E_NOMEM, "device allocation of " + std::to_string(bytes) + " B failed");
  } else {
    cudaError_t e = cudaMallocAsync(&p, bytes, ctx->stream);   // stream-ordered pool
    if (e != cudaSuccess) {
      cudaGetLastError();
      fail(ctx, DVL_E_NOMEM, "cudaMalloc(" + std::to_string(bytes) + "): " + cudaGetErrorString(e));
    }
  }
  ctx->live[p] = bytes;
  ctx->bytes += bytes;
  return p;
}

template <typename T>
T* dalloc(dvl_ctx* ctx, size_t count) {
  return static_cast<T*>(dmalloc(ctx, count * sizeof(T)));
}

void dfree(dvl_ctx* ctx, void* p) {
  if (!p) return;
  auto it = ctx->live.find(p);
  size_t bytes = it == ctx->live.end() ? 0 : it->second;
  if (it != ctx->live.end()) {
    ctx->live.erase(it);
    ctx->bytes -= bytes;
  }
  if (ctx->free)
    ctx->free(p, bytes, (void*)ctx->stream, ctx->user);
  else
    cudaFreeAsync(p, ctx->stream);
}

void free_dataset(dvl_ctx* ctx, Dataset& d) {
  void* ps[] = {d.keys, d.perm, d.gids, d.level_s, d.scal_s, d.d_vmin, d.d_vmax, d.d_lo, d.d_inv,
                d.d_rgba, d.d_tab, d.status1, d.tile_prefix, d.chunk_status, d.chunk_prefix,
                d.tile_meta, d.meta2, d.agg, d.cmin, d.cmax, d.blist, d.bctr};
  for (void* p : ps) dfree(ctx, p);
  d = Dataset();
}

void tic(dvl_ctx* ctx, Phase ph) {
  if (!(ctx->flags & DVL_FLAG_TIMING)) return;
  cudaEventRecord(ctx->ev[ph][0], ctx->stream);
}

void toc(dvl_ctx* ctx, Phase ph) {
  if (!(ctx->flags & DVL_FLAG_TIMING)) return;
  cudaEventRecord(ctx->ev[ph][1], ctx->stream);
  ctx->ev_used[ph] = true;
}

int ceil_log2_u64(uint64_t n) {
  int c = 0;
  while (c < 63 && (1ull << c) < n) ++c;
  return c;
}

int ceil_lmax_p(int Lmax, float P) { return (int)std::ceil((double)Lmax * (double)P); }

PowParams pow_params(float P) {
  PowParams pw{};
  if (P == 0.0f) {
    pw.kind = kPow0;
  } else if (P == 1.0f) {
    pw.kind = kPow1;
  } else if (P == std::floor(P) && P >= 2.0f && P <= 8.0f) {
    pw.kind = kPowInt;
    pw.k = (int)P;
  } else {
    pw.kind = kPowDet;
  }
  pw.P = P;
  return pw;
}

int items_for(int M, bool tma) {
  if (tma) return tma_items_for(M);
  if (M <= 4) return 16;
  if (M <= 8) return 8;
  if (M <= 16) return 4;
  if (M <= 32) return 2;
  return 1;
}

bool smem_tab_ok(const dvl_ctx* ctx) {
  return (size_t)ctx->ds.M * ctx->N * sizeof(float2) <= 64 * 1024;
}

// the level factor of Eq. 3: 1 (cell width 2^L) or 3 (cell volume 2^3L)
int lscale(const dvl_ctx* ctx) { return ctx->volume ? 3 : 1; }

UpdParams upd_params(dvl_ctx* ctx) {
  UpdParams p{};
  const Dataset& d = ctx->ds;
  p.n = d.n;
  p.n_pad = d.n_pad;
  p.M = d.M;
  p.N = ctx->N;
  p.level = d.level_s;
  p.scal = d.scal_s;
  p.lo = d.d_lo;
  p.inv = d.d_inv;
  p.tab = d.d_tab;
  p.maxv = ctx->d_maxv;
  p.eps = ctx->eps;
  p.pw = pow_params(ctx->P);
  p.scale = pow2f(ctx->shift);
  p.shift = ctx->shift;
  p.lscale = lscale(ctx);
  p.offset = 0;
  p.prod_sleep = ctx->prod_sleep;
  p.dbg = ctx->dbg;
  p.pass2_mode = ctx->pass2_mode;
  p.cmin = d.cmin;
  p.cmax = d.cmax;
  p.cmember = -1;
  return p;
}

int lmax_eff(const dvl_ctx* ctx) {
  return ctx->sharded ? std::max(ctx->lmax_global, ctx->ds.Lmax) : ctx->ds.Lmax;
}

// O11: s = 61 - ceil(log2 n) - ceil(Lmax P), over the whole (possibly sharded) dataset
int compute_shift(dvl_ctx* ctx) {
  const uint64_t n = ctx->sharded ? ctx->n_global : (uint64_t)ctx->ds.n;
  return 61 - ceil_log2_u64(n) - ceil_lmax_p(lscale(ctx) * lmax_eff(ctx), ctx->P);
}

void upload_domains(dvl_ctx* ctx) {
  const int M = ctx->ds.M;
  ctx->ds.cache_member = -1;   // the alphas depend on the domains
  CK(cudaMemcpyAsync(ctx->ds.d_lo, ctx->lo_h.data(), sizeof(float) * M, cudaMemcpyHostToDevice,
                     ctx->stream));
  CK(cudaMemcpyAsync(ctx->ds.d_inv, ctx->inv_h.data(), sizeof(float) * M,
                     cudaMemcpyHostToDevice, ctx->stream));
  // D3: the per-warp-tile statistics of t depend on the domains (not on the TFs)
  if (ctx->ds.tma && ctx->ds.agg) {
    launch_agg_build(upd_params(ctx), ctx->ds.agg, ctx->ds.n_pad / tma_warp_tile_cells(),
                     ctx->num_sms, ctx->stream);
    CKLAUNCH();
  }
}

// Put one N x 4 TF into the pinned, mapped staging buffer (after the previous reader of the
// buffer has finished); the prologue kernel reads it over PCIe.
// Two buffers alternate.  The event of buffer b is recorded when the edit before the one that
// will use b is staged (before its prologue is enqueued), so it completes once the prologue of
// the edit before that -- b's last reader -- has run: the host can enqueue an edit while the
// GPU still runs the last, and no event sits between two kernels of one edit (an event
// between a kernel and its programmatic dependent would serialise them).
void stage_tf(dvl_ctx* ctx, const float* rgba, int N) {
  ctx->stage_par ^= 1;
  CK(cudaEventSynchronize(ctx->stage_ev[ctx->stage_par]));
  memcpy(ctx->h_stage + (size_t)ctx->stage_par * 4 * kMaxN, rgba, sizeof(float) * 4 * N);
  CK(cudaEventRecord(ctx->stage_ev[ctx->stage_par ^ 1], ctx->stream));
}

// The fused prologue: optional TF install of `member`, pass-1 state reset, max(V_h).
void launch_prologue(dvl_ctx* ctx, int member, int mode, unsigned long long* zero, int zero_words) {
  Dataset& d = ctx->ds;
  launch_tf_prologue(ctx->d_hstage + (size_t)ctx->stage_par * 4 * kMaxN, member, mode, d.M, ctx->N, d.d_rgba, d.d_tab, d.d_vmin,
                     d.d_vmax, d.d_lo, d.d_inv, ctx->d_maxv, zero, zero_words, ctx->stream);
  CKLAUNCH();
}

// Work split of the TMA path for the current TF size: tile size from M, stage ring depth
// from the shared-memory budget (2 CTAs/SM when two stages fit in half an SM), chunks =
// resident CTAs.
void ensure_plan(dvl_ctx* ctx) {
  Dataset& d = ctx->ds;
  if (!d.tma || d.planN == ctx->N) return;
  TmaPlan pl{};
  const int64_t T1 = (int64_t)kBlock * d.items;        // pass-1 tile (n_pad is a multiple)
  const int64_t T2 = tma_tile2_cells(d.M);             // pass-2 tile
  auto round128 = [](size_t b) { return (uint32_t)((b + 127) & ~(size_t)127); };
  pl.tiles1 = (int)(d.n_pad / T1);
  pl.tiles = (int)(d.n_pad / T2);
  pl.stage_bytes1 = round128((size_t)d.M * T1 * 4 + T1);
  pl.stage_bytes = round128((size_t)d.M * T2 * 4 + T2 + 8 * (T2 / tma_warp_tile_cells()));
  pl.tab_bytes = smem_tab_ok(ctx) ? round128((size_t)d.M * ctx->N * 8) : 0;
  // Ring depths (at most 4) from per-CTA shared-memory budgets: pass 1 runs one CTA per SM
  // (the whole budget, which is the kernels' dynamic shared-memory limit set in
  // prepare_tma_kernels) with the TF slope table; pass 2 runs 3 / 2 / 1 CTAs per SM for
  // M <= 4 / 8 / 16 and keeps no table (only its boundary warps sample the TF, through L1).
  const size_t full = 225 * 1024, half = 110 * 1024, third = 74 * 1024;
  auto fit = [&](size_t budget, size_t tab, uint32_t stage) -> int {
    return tab < budget ? std::min(4, (int)((budget - tab) / stage)) : 0;
  };
  pl.stages1 = fit(full, pl.tab_bytes, pl.stage_bytes1);
  const int c2 = tma_pass2_ctas_per_sm(d.M);
  const size_t b2 = c2 >= 4 ? 55 * 1024 : c2 == 3 ? third : c2 == 2 ? half : full;
  pl.stages = fit(b2, 0, pl.stage_bytes);
  if (pl.stages < 2) pl.stages = fit(full, 0, pl.stage_bytes);
  if (ctx->stages_override) pl.stages = ctx->stages_override;
  if (pl.stages < 2 || pl.stages1 < 2)
    fail(ctx, DVL_E_INVAL, "TMA plan: two stages do not fit in shared memory");
  pl.tpc1 = pl.tpc = 1;
  const int bps = tma_blocks_per_sm(d.M, false, pl, 2);
  const int bps1 = tma_blocks_per_sm(d.M, pl.tab_bytes > 0, pl, 1);
  int G = std::min(pl.tiles, ctx->num_sms * bps);
  pl.tpc = (pl.tiles + G - 1) / G;
  G = (pl.tiles + pl.tpc - 1) / pl.tpc;
  int G1 = std::min(pl.tiles1, ctx->num_sms * bps1);
  pl.tpc1 = (pl.tiles1 + G1 - 1) / G1;
  G1 = (pl.tiles1 + pl.tpc1 - 1) / pl.tpc1;
  // the edit-cache plan (M > 8): 3 CTAs per SM, stages of 13 B per cell, the TF table read
  // through L1 (the edited member's only)
  TmaPlan pc = pl;
  int G1c = 0;
  bool pc_ok = false;
  if (d.M > 8 && d.M >= 3) {
    pc.tab_bytes = 0;
    pc.stage_bytes1 = round128((size_t)T1 * 13);
    pc.stages1 = fit(third, 0, pc.stage_bytes1);
    if (pc.stages1 >= 2 && tma_blocks_per_sm_cache(d.M, pc) >= 3) {
      G1c = std::min(pl.tiles1, ctx->num_sms * 3);
      pc.tpc1 = (pl.tiles1 + G1c - 1) / G1c;
      G1c = (pl.tiles1 + pc.tpc1 - 1) / pc.tpc1;
      pc_ok = true;
    }
  }
  const int cap = std::max(G1, G1c) + 1;   // chunk status words + the chunk counters' word
  if (cap > d.chunk_cap) {
    unsigned long long* cs = dalloc<unsigned long long>(ctx, cap);
    unsigned long long* cp = dalloc<unsigned long long>(ctx, cap);
    // the last word holds pass 1's self-resetting chunk counters: zero once here
    CK(cudaMemsetAsync(cs, 0, sizeof(unsigned long long) * cap, ctx->stream));
    dfree(ctx, d.chunk_status);
    dfree(ctx, d.chunk_prefix);
    d.chunk_status = cs;
    d.chunk_prefix = cp;
    d.chunk_cap = cap;
  }
  d.plan = pl;
  d.plan_c = pc;
  d.plan_c_ok = pc_ok;
  d.grid1_c = G1c;
  d.last_c = false;
  d.grid = G;
  d.grid1 = G1;
  d.planN = ctx->N;
}

// the pass-1 chunking pass 2 must use: that of the last pass 1
const TmaPlan& pass2_plan(const Dataset& d) { return d.last_c ? d.plan_c : d.plan; }

// U0-U2: (member >= 0: install the staged TF of that member), maxV, pass 1 (weights +
// decoupled look-back scan).
void run_weights(dvl_ctx* ctx, bool export_q, unsigned long long* q_out, int member = -1) {
  Dataset& d = ctx->ds;
  ctx->shift = compute_shift(ctx);
  ensure_plan(ctx);
  UpdParams p = upd_params(ctx);
  tic(ctx, PH_MAXV);
  const bool exact = ctx->mode == DVL_MAXV_EXACT;
  launch_prologue(ctx, member, exact ? -1 : ctx->mode, d.tma ? d.chunk_status : nullptr,
                  d.tma ? d.chunk_cap - 1 : 0);
  if (exact) {
    // 4 cells per thread on the TMA layout (tiles of 4 * 256 * k cells), else the tile's
    const int per = d.tma ? 4 : d.items;
    int grid = (int)(d.n_pad / ((int64_t)kBlock * per));
    launch_maxv_exact(p, ctx->d_maxv, grid, ctx->stream);
    CKLAUNCH();
    // a shard's exact max(V_h) is the max over every shard's cells: one MAX all_reduce of
    // the bits (maxV >= +0, so the u32 order is the float order); collective
    if (ctx->sharded) {
      if (!ctx->comm) fail(ctx, DVL_E_STATE, "exact max(V_h) on a shard needs the context's communicator");
      if (const char* e = ctx->comm->allreduce(ctx->d_maxv, 1, kU32, kMax, ctx->stream))
        fail(ctx, DVL_E_NCCL, std::string("all_reduce MAX of maxV: ") + e);
    }
  }
  toc(ctx, PH_MAXV);
  // the edit cache: an edit of member e reads only e's scalars and the cached alpha range
  // of the others when the cache holds them (kCache), else pass 1 reads every member and
  // (re)writes the cache for e (kWrite).  Any other TF or domain change invalidates it.
  int cmode = 0;
  if (member >= 0) {
    if (d.tma && d.M >= 3 && ctx->edit_cache && !export_q) {
      if (!d.cmin) {
        try {
          d.cmin = dalloc<uint32_t>(ctx, (size_t)d.n_pad);
          d.cmax = dalloc<uint32_t>(ctx, (size_t)d.n_pad);
        } catch (Fail&) {   // no room for it: every edit reads every member
          dfree(ctx, d.cmin);
          d.cmin = nullptr;
          ctx->edit_cache = false;
        }
      }
      if (d.cmin) {
        cmode = d.cache_member == member ? 1 : 2;
        p.cmin = d.cmin;
        p.cmax = d.cmax;
        p.cmember = member;
      }
    }
    d.cache_member = cmode ? member : -1;
  }
  tic(ctx, PH_WSCAN);
  if (d.tma) {
    uint32_t* ctr = reinterpret_cast<uint32_t*>(d.chunk_status + d.chunk_cap - 1);
    d.last_c = cmode == 1 && d.plan_c_ok;
    if (d.last_c)
      launch_weights_reduce_tma(false, p, d.plan_c, d.grid1_c, d.chunk_status, ctr, d.chunk_prefix,
                                ctx->d_qtot, d.tile_meta, d.meta2, cmode, ctx->stream);
    else
      launch_weights_reduce_tma(d.plan.tab_bytes > 0, p, d.plan, d.grid1, d.chunk_status, ctr,
                                d.chunk_prefix, ctx->d_qtot, d.tile_meta, d.meta2, cmode, ctx->stream);
    CKLAUNCH();
    if (export_q) {
      launch_q_export_tma(false, p, d.plan, d.grid, d.chunk_prefix, ctx->d_qtot, ctx->d_err, q_out,
                          d.tile_meta, ctx->stream);
      CKLAUNCH();
    }
  } else {
    CK(cudaMemsetAsync(d.status1, 0, sizeof(unsigned long long) * d.tiles, ctx->stream));
    CK(cudaMemsetAsync(ctx->d_ctr1, 0, sizeof(uint32_t), ctx->stream));
    launch_weights_scan(d.items, smem_tab_ok(ctx), export_q, p, d.status1, ctx->d_ctr1,
                        d.tile_prefix, ctx->d_qtot, q_out, d.tiles, ctx->stream);
    CKLAUNCH();
  }
  toc(ctx, PH_WSCAN);
}

// the accumulators of this call: lo / hi from the copy of the current parity
Acc cur_acc(const dvl_ctx* ctx) {
  Acc a = ctx->acc;
  if (ctx->acc_par) {
    std::swap(a.lo, a.lo2);
    std::swap(a.hi, a.hi2);
  }
  return a;
}

void ensure_acc(dvl_ctx* ctx, uint32_t W) {
  const int M = ctx->ds.M;
  if (ctx->accW >= W && ctx->accM == M) return;
  uint32_t cap = std::max(W, ctx->accW);
  if (ctx->accM != M) cap = W;
  Acc a{};
  a.lo = dalloc<unsigned long long>(ctx, cap);
  a.hi = dalloc<unsigned long long>(ctx, cap);
  a.lo2 = dalloc<unsigned long long>(ctx, cap);
  a.hi2 = dalloc<unsigned long long>(ctx, cap);
  a.tmin = dalloc<uint32_t>(ctx, (size_t)cap * M);
  a.tmax = dalloc<uint32_t>(ctx, (size_t)cap * M);
  a.slo = dalloc<unsigned long long>(ctx, (size_t)cap * M);
  a.shi = dalloc<unsigned long long>(ctx, (size_t)cap * M);
  dvl_vertex* out = dalloc<dvl_vertex>(ctx, (size_t)cap * M);
  unsigned long long* blo = dalloc<unsigned long long>(ctx, cap);
  unsigned long long* bhi = dalloc<unsigned long long>(ctx, cap);
  dfree(ctx, ctx->acc.lo);
  dfree(ctx, ctx->acc.hi);
  dfree(ctx, ctx->acc.lo2);
  dfree(ctx, ctx->acc.hi2);
  dfree(ctx, ctx->acc.tmin);
  dfree(ctx, ctx->acc.tmax);
  dfree(ctx, ctx->acc.slo);
  dfree(ctx, ctx->acc.shi);
  dfree(ctx, ctx->d_out);
  dfree(ctx, ctx->d_bin_lo);
  dfree(ctx, ctx->d_bin_hi);
  ctx->acc = a;
  ctx->acc_par = 0;
  ctx->acc_dirty[0] = ctx->acc_dirty[1] = 0;
  ctx->d_out = out;
  ctx->d_bin_lo = blo;
  ctx->d_bin_hi = bhi;
  ctx->accW = cap;
  ctx->accM = M;
  ctx->last_W = 0;
  // identity of every accumulator plane (the epilogue restores it after each use);
  // planes are laid out with the capacity as member stride, so init the whole capacity
  launch_acc_init(a, cap, M, ctx->stream);
  CKLAUNCH();
}

void identity_tf_host(std::vector<float>& tf, int N) {
  tf.resize((size_t)N * 4);
  for (int i = 0; i < N; ++i) {
    float a = (float)((double)i / (double)(N - 1));
    tf[4 * i] = tf[4 * i + 1] = tf[4 * i + 2] = 0.5f;
    tf[4 * i + 3] = a;
  }
}

void set_all_tfs(dvl_ctx* ctx, const std::vector<float>& tf, int N) {
  ctx->ds.cache_member = -1;   // every member's TF changes
  for (int m = 0; m < ctx->ds.M; ++m) {
    stage_tf(ctx, tf.data(), N);
    launch_prologue(ctx, m, -1, nullptr, 0);
  }
}

bool maybe_degenerate(const dvl_ctx* ctx) {
  if (ctx->eps <= 0.0f) return true;
  // smallest possible weight: V = 0 -> r = eps, L = 0 -> f = eps^P (approximately)
  double fmin = std::pow((double)ctx->eps, (double)ctx->P);
  return fmin * std::ldexp(1.0, ctx->shift) < 4.0;
}

}  // namespace

// ============================================================================== C ABI
extern "C" {

const char* dvl_status_string(dvl_status s) {
  switch (s) {
    case DVL_OK: return "DVL_OK";
    case DVL_E_INVAL: return "DVL_E_INVAL";
    case DVL_E_STATE: return "DVL_E_STATE";
    case DVL_E_RANGE: return "DVL_E_RANGE";
    case DVL_E_OVERLAP: return "DVL_E_OVERLAP";
    case DVL_E_DEGENERATE: return "DVL_E_DEGENERATE";
    case DVL_E_NOMEM: return "DVL_E_NOMEM";
    case DVL_E_CUDA: return "DVL_E_CUDA";
    case DVL_E_NCCL: return "DVL_E_NCCL";
  }
  return "DVL_E_UNKNOWN";
}

const char* dvl_last_error(const dvl_ctx* ctx) { return ctx ? ctx->err.c_str() : ""; }

void* dvl_stream(dvl_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

int dvl_hilbert_states(void) { return hilbert_num_states(); }

dvl_status dvl_hilbert_encode_host(uint64_t n, const uint32_t* xyz, int bits, uint64_t* codes) {
  if ((n && (!xyz || !codes)) || bits < 1 || bits > 21) return DVL_E_INVAL;
  for (uint64_t i = 0; i < n; ++i) {
    uint32_t x = xyz[3 * i], y = xyz[3 * i + 1], z = xyz[3 * i + 2];
    if ((x | y | z) >> bits) return DVL_E_INVAL;
  }
  for (uint64_t i = 0; i < n; ++i)
    codes[i] = hilbert_encode_host(xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2], bits);
  return DVL_OK;
}

dvl_status dvl_create(const dvl_init* init, dvl_ctx** out) {
  if (!init || !out) return DVL_E_INVAL;
  *out = nullptr;
  dvl_ctx* ctx = new dvl_ctx();
  try {
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (init->device < 0 || init->device >= ndev) fail(ctx, DVL_E_INVAL, "bad device ordinal");
    if ((init->alloc == nullptr) != (init->free == nullptr))
      fail(ctx, DVL_E_INVAL, "alloc and free must both be set or both be NULL");
    ctx->device = init->device;
    ctx->alloc = init->alloc;
    ctx->free = init->free;
    ctx->user = init->user;
    ctx->flags = init->flags;
    CK(cudaSetDevice(ctx->device));
    {
      // keep freed blocks in the device's default pool (rebuilds reuse them)
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, ctx->device) == cudaSuccess) {
        uint64_t thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
      }
    }
    if (init->cuda_stream) {
      ctx->stream = (cudaStream_t)init->cuda_stream;
    } else {
      CK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
      ctx->own_stream = true;
    }
    static bool prepared = false;
    if (!prepared) {
      CK(prepare_onesweep());
      CK(prepare_update_kernels());
      CK(prepare_tma_kernels());
      prepared = true;
    }
    CK(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, ctx->device));
    // experiment knobs
    ctx->edit_cache = !(init->flags & DVL_FLAG_NO_EDIT_CACHE);
    ctx->pass2_mode = (init->flags & DVL_FLAG_PASS2_JOBS)   ? 3
                      : (init->flags & DVL_FLAG_PASS2_LIST)   ? 2
                      : (init->flags & DVL_FLAG_PASS2_INLINE) ? 1
                                                              : 0;
#ifdef DVL_PROF
    // experiment knobs of the profiling build only
    if (const char* e = getenv("DVL_PROD_SLEEP")) ctx->prod_sleep = (uint32_t)atoi(e);
    if (const char* e = getenv("DVL_STAGES2")) ctx->stages_override = atoi(e);
    if (const char* e = getenv("DVL_DBG")) ctx->dbg = atoi(e);
#endif
    ctx->d_maxv = dalloc<float>(ctx, 1);
    ctx->d_qtot = dalloc<unsigned long long>(ctx, 1);
    ctx->d_ctr1 = dalloc<uint32_t>(ctx, 1);
    ctx->d_err = dalloc<uint32_t>(ctx, 1);
    ctx->d_offset = dalloc<unsigned long long>(ctx, 1);
    ctx->d_qtot_glob = dalloc<unsigned long long>(ctx, 1);
    CK(cudaHostAlloc(&ctx->h_stage, sizeof(float) * (2 * 4 * kMaxN + 32), cudaHostAllocMapped));
    CK(cudaHostGetDevicePointer((void**)&ctx->d_hstage, ctx->h_stage, 0));
    for (int i = 0; i < 2; ++i) {
      CK(cudaEventCreateWithFlags(&ctx->stage_ev[i], cudaEventDisableTiming));
      CK(cudaEventRecord(ctx->stage_ev[i], ctx->stream));
    }
    for (int i = 0; i < PH_N; ++i) {
      CK(cudaEventCreate(&ctx->ev[i][0]));
      CK(cudaEventCreate(&ctx->ev[i][1]));
    }
    std::vector<uint16_t> t1, t2;
    hilbert_tables_host(&t1, &t2, &ctx->nstates);
    ctx->d_t1 = dalloc<uint16_t>(ctx, t1.size());
    ctx->d_t2 = dalloc<uint16_t>(ctx, t2.size());
    CK(cudaMemcpyAsync(ctx->d_t1, t1.data(), t1.size() * 2, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->d_t2, t2.data(), t2.size() * 2, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemsetAsync(ctx->d_err, 0, 4, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  } catch (Fail& f) {
    // keep the message visible through a process-wide fallback
    fprintf(stderr, "dvl_create: %s\n", ctx->err.c_str());
    dvl_destroy(ctx);
    return f.s;
  }
  *out = ctx;
  return DVL_OK;
}

void dvl_destroy(dvl_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  delete ctx->comm;
  free_dataset(ctx, ctx->ds);
  std::vector<void*> ps;
  for (auto& kv : ctx->live) ps.push_back(kv.first);
  for (void* p : ps) dfree(ctx, p);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  if (ctx->h_stage) cudaFreeHost(ctx->h_stage);
  for (int i = 0; i < 2; ++i)
    if (ctx->stage_ev[i]) cudaEventDestroy(ctx->stage_ev[i]);
  for (int i = 0; i < PH_N; ++i)
    for (int j = 0; j < 2; ++j)
      if (ctx->ev[i][j]) cudaEventDestroy(ctx->ev[i][j]);
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

// ------------------------------------------------------------------ build helpers
namespace {

using Tmp = std::vector<void*>;

// device copies of the inputs (host inputs are staged into temporaries) and the device
// array of the member row pointers
struct Inputs {
  const uint32_t* lower = nullptr;
  const uint8_t* level = nullptr;
  const float** d_ptrs = nullptr;
};

Inputs stage_inputs(dvl_ctx* ctx, int64_t nn, const uint32_t* lower_xyz, const uint8_t* level,
                    int M, const float* const* scalars, dvl_mem where, Tmp& tmp) {
  cudaStream_t st = ctx->stream;
  Inputs in;
  in.lower = lower_xyz;
  in.level = level;
  std::vector<const float*> ptrs(M, nullptr);
  if (scalars)
    for (int m = 0; m < M; ++m) ptrs[m] = scalars[m];
  if (where == DVL_MEM_HOST && nn > 0) {
    uint32_t* l = dalloc<uint32_t>(ctx, 3 * (size_t)nn);
    tmp.push_back(l);
    uint8_t* lv = dalloc<uint8_t>(ctx, nn);
    tmp.push_back(lv);
    float* sc = dalloc<float>(ctx, (size_t)M * nn);
    tmp.push_back(sc);
    CK(cudaMemcpyAsync(l, lower_xyz, 12 * (size_t)nn, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(lv, level, nn, cudaMemcpyHostToDevice, st));
    for (int m = 0; m < M; ++m) {
      CK(cudaMemcpyAsync(sc + (size_t)m * nn, scalars[m], 4 * (size_t)nn, cudaMemcpyHostToDevice, st));
      ptrs[m] = sc + (size_t)m * nn;
    }
    in.lower = l;
    in.level = lv;
  }
  in.d_ptrs = (const float**)dmalloc(ctx, sizeof(float*) * M);
  tmp.push_back((void*)in.d_ptrs);
  CK(cudaMemcpyAsync(in.d_ptrs, ptrs.data(), sizeof(float*) * M, cudaMemcpyHostToDevice, st));
  return in;
}

IngestOut* new_ingest(dvl_ctx* ctx, Tmp& tmp) {
  IngestOut h;
  memset(&h, 0, sizeof h);
  for (int m = 0; m < 64; ++m) h.vmin[m] = 0xffffffffu;
  IngestOut* d = (IngestOut*)dmalloc(ctx, sizeof(IngestOut));
  tmp.push_back(d);
  CK(cudaMemcpyAsync(d, &h, sizeof h, cudaMemcpyHostToDevice, ctx->stream));
  return d;
}

void read_ingest(dvl_ctx* ctx, const IngestOut* d, IngestOut* h) {
  CK(cudaMemcpyAsync(h, d, sizeof(IngestOut), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
}

struct Sorted {
  void* keys = nullptr;      // n sorted codes (key_bytes each)
  uint32_t* perm = nullptr;  // source index of each sorted code
};

// B2 on codes already in `keys` (n of them, b bits): the bucket sort of distinct codes for
// 3b <= 36 (bsort.cu) or the onesweep LSD sort; with lower/level given, B1 (the Hilbert
// encode) runs first and writes `keys` itself.  The returned arrays are owned by the
// caller (the codes may end in `keys` or in a new buffer); the other temporaries go to tmp.
Sorted sort_codes(dvl_ctx* ctx, const uint32_t* lower, const uint8_t* level, void* keys,
                  int64_t nn, int b, int kb, Tmp& tmp) {
  cudaStream_t st = ctx->stream;
  const bool encode = lower != nullptr;
  void* kA = keys;
  void* kB = dmalloc(ctx, (size_t)kb * nn);
  uint32_t* iA = dalloc<uint32_t>(ctx, nn);
  uint32_t* iB = dalloc<uint32_t>(ctx, nn);
  Sorted out;
  const bool bucket = 3 * b <= 36 && !(ctx->flags & DVL_FLAG_LSD_SORT);
  if (bucket) {
    int lb = 0;
    const int64_t nb = bucket_count(b, &lb);
    const int64_t nblk = (nb + 4095) / 4096;
    uint32_t* bcnt = dalloc<uint32_t>(ctx, (size_t)nb);
    uint32_t* bstart = dalloc<uint32_t>(ctx, (size_t)nb + 1);
    uint16_t* slot = dalloc<uint16_t>(ctx, (size_t)nn);
    uint32_t* bsum = dalloc<uint32_t>(ctx, (size_t)nblk + 1);
    uint32_t* work = dalloc<uint32_t>(ctx, 1);
    for (void* q : {(void*)bcnt, (void*)bstart, (void*)slot, (void*)bsum, (void*)work}) tmp.push_back(q);
    CK(cudaMemsetAsync(bcnt, 0, sizeof(uint32_t) * nb, st));
    CK(cudaMemsetAsync(work, 0, sizeof(uint32_t), st));
    tic(ctx, PH_ENCODE);
    if (encode)
      launch_encode_bucket(lower, level, nn, b, lb, kb, ctx->d_t1, ctx->d_t2, ctx->nstates, kA,
                           slot, bcnt, ctx->num_sms, st);
    else
      launch_bucket_slot(kA, kb, nn, lb, slot, bcnt, ctx->num_sms, st);
    CKLAUNCH();
    toc(ctx, PH_ENCODE);
    tic(ctx, PH_SORT);
    launch_bucket_scan(bcnt, nb, lb, bsum, bstart, (uint32_t)nn, ctx->d_err, st);
    CKLAUNCH();
    launch_bucket_sort(kA, slot, kb, nn, lb, nb, bstart, kB, iB, kA, iA, work, ctx->d_err,
                       ctx->num_sms, st);
    CKLAUNCH();
    toc(ctx, PH_SORT);
    ctx->sort_passes = 2;
    out.keys = kA;
    out.perm = iA;
    tmp.push_back(kB);
    tmp.push_back(iB);
    return out;
  }
  const int passes = (3 * b + 7) / 8;
  uint32_t* hist = dalloc<uint32_t>(ctx, (size_t)passes * 256);
  uint32_t* base = dalloc<uint32_t>(ctx, (size_t)passes * 256);
  const int64_t stiles = (nn + kSortTile - 1) / kSortTile;
  uint32_t* status = dalloc<uint32_t>(ctx, (size_t)passes * stiles * 256);
  uint32_t* ctrs = dalloc<uint32_t>(ctx, passes);
  for (void* q : {(void*)hist, (void*)base, (void*)status, (void*)ctrs}) tmp.push_back(q);
  CK(cudaMemsetAsync(hist, 0, sizeof(uint32_t) * passes * 256, st));
  CK(cudaMemsetAsync(status, 0, sizeof(uint32_t) * passes * stiles * 256, st));
  CK(cudaMemsetAsync(ctrs, 0, sizeof(uint32_t) * passes, st));
  tic(ctx, PH_ENCODE);
  const int grid = (int)std::min<int64_t>((nn + kBlock - 1) / kBlock, 148 * 8);
  if (encode)
    launch_encode_hist(lower, level, nn, b, kb, passes, ctx->d_t1, ctx->d_t2, ctx->nstates, kA,
                       iA, hist, grid, st);
  else
    launch_key_hist(kA, kb, nn, passes, hist, ctx->num_sms, st);
  CKLAUNCH();
  toc(ctx, PH_ENCODE);
  // onesweep passes (a pass whose digit is constant is the identity: skipped)
  tic(ctx, PH_SORT);
  launch_hist_scan(hist, base, passes, st);
  CKLAUNCH();
  std::vector<uint32_t> h_hist((size_t)passes * 256);
  CK(cudaMemcpyAsync(h_hist.data(), hist, 4 * h_hist.size(), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  void* kin = kA;
  void* kout = kB;
  uint32_t* vin = iA;
  uint32_t* vout = iB;
  int done = 0;
  for (int p = 0; p < passes; ++p) {
    uint32_t mx = *std::max_element(h_hist.begin() + p * 256, h_hist.begin() + (p + 1) * 256);
    if ((int64_t)mx == nn) continue;
    // the first pass generates the ids (iota) instead of reading them
    launch_onesweep(kin, done == 0 ? nullptr : vin, kout, vout, nn, kb, 8 * p, base + p * 256,
                    status + (size_t)p * stiles * 256, ctrs + p, st);
    CKLAUNCH();
    std::swap(kin, kout);
    std::swap(vin, vout);
    ++done;
  }
  if (done == 0) {   // every digit constant (n == 1): the identity permutation
    launch_iota(vin, nn, st);
    CKLAUNCH();
  }
  ctx->sort_passes = done;
  toc(ctx, PH_SORT);
  out.keys = kin;
  out.perm = vin;
  if (kout != keys) tmp.push_back(kout);   // the caller's buffer stays the caller's
  tmp.push_back(vout);
  return out;
}

// B3: level_s / scal_s (rows of n_pad) in sorted order from the source arrays through
// `perm`, the overlap check along the run (error word) and the member ranges (into ing)
void gather_sorted(dvl_ctx* ctx, Dataset& d, const uint8_t* level_in, const float* const* d_ptrs,
                   IngestOut* ing) {
  cudaStream_t st = ctx->stream;
  d.level_s = dalloc<uint8_t>(ctx, d.n_pad);
  d.scal_s = dalloc<float>(ctx, (size_t)d.M * d.n_pad);
  CK(cudaMemsetAsync(d.level_s, 0, d.n_pad, st));
  CK(cudaMemsetAsync(d.scal_s, 0, sizeof(float) * d.M * d.n_pad, st));
  tic(ctx, PH_GATHER);
  launch_gather_validate4(d.keys, d.key_bytes, d.perm, level_in, d_ptrs, d.n, d.M, d.n_pad,
                          d.level_s, d.scal_s, ctx->d_err, ing, ctx->num_sms, st);
  CKLAUNCH();
  toc(ctx, PH_GATHER);
}

// tile geometry of a dataset of d.n cells and d.M members
void set_geometry(dvl_ctx* ctx, Dataset& d) {
  d.key_bytes = 3 * d.b <= 32 ? 4 : 8;
  d.passes = (3 * d.b + 7) / 8;
  d.tma = d.M <= 16 && !(ctx->flags & DVL_FLAG_GENERIC);
  d.items = items_for(d.M, d.tma);
  const int64_t T = (int64_t)kBlock * d.items;
  d.tiles = (int)((d.n + T - 1) / T);
  d.n_pad = (int64_t)d.tiles * T;
}

void ranges_from(Dataset& d, const IngestOut& h) {
  d.vmin.resize(d.M);
  d.vmax.resize(d.M);
  for (int m = 0; m < d.M; ++m) {
    d.vmin[m] = h.any[m] ? ordered_to_float(h.vmin[m]) : 0.0f;
    d.vmax[m] = h.any[m] ? ordered_to_float(h.vmax[m]) : 0.0f;
  }
}

// the per-dataset update state (TF tables, look-back state, D3 statistics, lists)
void alloc_update_state(dvl_ctx* ctx, Dataset& d) {
  cudaStream_t st = ctx->stream;
  const int M = d.M;
  d.d_vmin = dalloc<float>(ctx, M);
  d.d_vmax = dalloc<float>(ctx, M);
  d.d_lo = dalloc<float>(ctx, M);
  d.d_inv = dalloc<float>(ctx, M);
  d.d_rgba = dalloc<float4>(ctx, (size_t)M * kMaxN);
  d.d_tab = dalloc<float2>(ctx, (size_t)M * kMaxN);
  d.status1 = dalloc<unsigned long long>(ctx, d.tiles);
  d.tile_prefix = dalloc<unsigned long long>(ctx, d.tiles);
  if (d.tma) {
    d.tile_meta = dalloc<unsigned long long>(ctx, (size_t)(d.n_pad / tma_warp_tile_cells()));
    d.meta2 = dalloc<unsigned long long>(ctx, (size_t)(d.n_pad / tma_warp_tile_cells()));
    d.agg = dalloc<unsigned char>(ctx, agg_bytes(M, d.n_pad / tma_warp_tile_cells()));
    // the boundary-tile list (2 words per warp tile), then the job list (u32 per job, at
    // most nwt / 24 + 1 jobs); counters: boundary list count + done, job list count + done
    const size_t nwt = (size_t)(d.n_pad / tma_warp_tile_cells());
    d.blist = dalloc<unsigned long long>(ctx, 2 * nwt + nwt / 32 + 2);
    d.bctr = dalloc<uint32_t>(ctx, 4);
    CK(cudaMemsetAsync(d.bctr, 0, 4 * sizeof(uint32_t), st));
  }
  CK(cudaMemcpyAsync(d.d_vmin, d.vmin.data(), 4 * M, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d.d_vmax, d.vmax.data(), 4 * M, cudaMemcpyHostToDevice, st));
}

// replace the context's dataset with d; default domains = the data ranges, identity TFs,
// the first weights
dvl_status commit_dataset(dvl_ctx* ctx, Dataset& d, bool sharded, uint64_t cell_offset,
                          uint64_t n_global, int lmax_global) {
  free_dataset(ctx, ctx->ds);
  ctx->ds = d;
  ctx->built = true;
  ctx->sharded = sharded;
  ctx->cell_offset = cell_offset;
  ctx->n_global = n_global;
  ctx->lmax_global = lmax_global;
  ctx->N = 256;
  ctx->lo_h = ctx->ds.vmin;
  ctx->hi_h = ctx->ds.vmax;
  ctx->inv_h.resize(ctx->ds.M);
  for (int m = 0; m < ctx->ds.M; ++m) {
    float lo = ctx->lo_h[m], hi = ctx->hi_h[m];
    ctx->inv_h[m] = hi > lo ? 1.0f / (hi - lo) : 0.0f;
  }
  if (ctx->accM != ctx->ds.M) ctx->accW = 0;
  ctx->last_W = 0;
  try {
    upload_domains(ctx);
    std::vector<float> tf;
    identity_tf_host(tf, ctx->N);
    set_all_tfs(ctx, tf, ctx->N);
    run_weights(ctx, false, nullptr);
    CK(cudaStreamSynchronize(ctx->stream));
  } catch (Fail& f) {
    ctx->built = false;
    return f.s;
  }
  return DVL_OK;
}

uint32_t read_err(dvl_ctx* ctx) {
  uint32_t herr = 0;
  CK(cudaMemcpyAsync(&herr, ctx->d_err, 4, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return herr;
}

dvl_status dist_build(dvl_ctx* ctx, uint64_t n, const uint32_t* lower_xyz, const uint8_t* level,
                      uint32_t members, const float* const* scalars, dvl_mem where);

}  // namespace

dvl_status dvl_build(dvl_ctx* ctx, uint64_t n, const uint32_t* lower_xyz, const uint8_t* level,
                     uint32_t members, const float* const* scalars, dvl_mem where) {
  if (!ctx) return DVL_E_INVAL;
  ctx->err.clear();
  if (ctx->comm) return dist_build(ctx, n, lower_xyz, level, members, scalars, where);

  Dataset d;
  Tmp tmp;   // temporaries freed on every exit
  auto cleanup = [&]() {
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    for (void* p : tmp) dfree(ctx, p);
  };
  try {
    if (n == 0) fail(ctx, DVL_E_INVAL, "n must be >= 1");
    if (n >= (1ull << 30)) fail(ctx, DVL_E_RANGE, "n must be < 2^30 per device");
    if (members < 1 || members > (uint32_t)kMaxM) fail(ctx, DVL_E_INVAL, "members must be in [1, 64]");
    if (!lower_xyz || !level || !scalars) fail(ctx, DVL_E_INVAL, "NULL input pointer");
    for (uint32_t m = 0; m < members; ++m)
      if (!scalars[m]) fail(ctx, DVL_E_INVAL, "NULL scalar pointer");
    if (where != DVL_MEM_HOST && where != DVL_MEM_DEVICE) fail(ctx, DVL_E_INVAL, "bad dvl_mem");
    CK(cudaSetDevice(ctx->device));
    const int M = (int)members;
    const int64_t nn = (int64_t)n;
    cudaStream_t st = ctx->stream;

    // ---- stage inputs; B0: ingest reduction over the geometry
    tic(ctx, PH_INGEST);
    Inputs in = stage_inputs(ctx, nn, lower_xyz, level, M, scalars, where, tmp);
    IngestOut* d_ing = new_ingest(ctx, tmp);
    launch_ingest_geom(in.lower, in.level, nn, d_ing, ctx->num_sms, st);
    CKLAUNCH();
    toc(ctx, PH_INGEST);
    IngestOut h_ing;
    read_ingest(ctx, d_ing, &h_ing);
    if (h_ing.err & kErrInval) fail(ctx, DVL_E_INVAL, "a cell has L > 20 or a lower corner not a multiple of 2^L");
    if (h_ing.extent > (1ull << 21)) fail(ctx, DVL_E_RANGE, "logical extent E > 2^21");
    if (ceil_lmax_p(lscale(ctx) * (int)h_ing.lmax, ctx->P) > 100)
      fail(ctx, DVL_E_RANGE, "ceil(Lmax * P) > 100 (fp32 weight overflow)");
    d.n = nn;
    d.M = M;
    d.E = (uint32_t)h_ing.extent;
    d.b = std::max(1, ceil_log2_u64(h_ing.extent));
    if (ctx->global_bits > 0) {
      if (d.b > ctx->global_bits) fail(ctx, DVL_E_RANGE, "shard extent exceeds 2^global_bits");
      d.b = ctx->global_bits;
    }
    d.Lmax = (int)h_ing.lmax;
    set_geometry(ctx, d);

    // ---- B1 + B2: Hilbert encode and sort
    CK(cudaMemsetAsync(ctx->d_err, 0, 4, st));
    void* keys = dmalloc(ctx, (size_t)d.key_bytes * nn);
    tmp.push_back(keys);
    Sorted srt = sort_codes(ctx, in.lower, in.level, keys, nn, d.b, d.key_bytes, tmp);
    if (srt.keys == keys) tmp.erase(std::find(tmp.begin(), tmp.end(), keys));
    d.keys = srt.keys;
    d.perm = srt.perm;

    // ---- B3: permute into curve order + overlap validation + member ranges
    gather_sorted(ctx, d, in.level, in.d_ptrs, d_ing);
    const uint32_t herr = read_err(ctx);
    read_ingest(ctx, d_ing, &h_ing);
    if (herr & kErrOverlap) fail(ctx, DVL_E_OVERLAP, "duplicate or overlapping cells");
    ranges_from(d, h_ing);
    alloc_update_state(ctx, d);
  } catch (Fail& f) {
    cleanup();
    free_dataset(ctx, d);
    return f.s;
  }
  cleanup();
  return commit_dataset(ctx, d, false, 0, (uint64_t)d.n, d.Lmax);
}

namespace {

// the in-process stand-in for a communicator handle (dvl_local_group_create)
struct GroupHandle {
  LocalGroup* g;
};

void attach_comm(dvl_ctx* ctx, Comm* c) {
  dfree(ctx, ctx->d_totals);
  ctx->d_totals = dalloc<unsigned long long>(ctx, (size_t)c->nranks);
  ctx->comm = c;
  ctx->comm_ranks = c->nranks;
  ctx->comm_rank = c->rank;
}

// a collective helper: small u64 vectors through device memory
struct Small {
  dvl_ctx* ctx;
  unsigned long long* d = nullptr;
  size_t cap = 0;
  Small(dvl_ctx* c, size_t words) : ctx(c), cap(words) { d = dalloc<unsigned long long>(ctx, words); }
  ~Small() { dfree(ctx, d); }
  void put(const std::vector<uint64_t>& v) {
    CK(cudaMemcpyAsync(d, v.data(), 8 * v.size(), cudaMemcpyHostToDevice, ctx->stream));
  }
  std::vector<uint64_t> get(size_t words) {
    std::vector<uint64_t> v(words);
    CK(cudaMemcpyAsync(v.data(), d, 8 * words, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return v;
  }
};

void comm_ck(dvl_ctx* ctx, const char* e, const char* what) {
  if (e) fail(ctx, DVL_E_NCCL, std::string(what) + ": " + e);
}

// error agreement: every rank learns the largest local status, so all ranks fail together
// (a rank must never leave the others waiting in a collective)
dvl_status agree(dvl_ctx* ctx, dvl_status local, const std::string& msg) {
  Small sm(ctx, 1);
  sm.put({(uint64_t)local});
  comm_ck(ctx, ctx->comm->allreduce(sm.d, 1, kU64, kMax, ctx->stream), "status all_reduce");
  const dvl_status g = (dvl_status)sm.get(1)[0];
  if (g != DVL_OK) fail(ctx, g, local != DVL_OK ? msg : "another rank failed: " + std::string(dvl_status_string(g)));
  return g;
}

// SURVEY 8(e) "Build": the Hilbert-key sample sort across the communicator's ranks.  Each
// rank passes its slice of the cells (any slice, possibly empty); each ends with one
// contiguous range of the global curve order, built and described as a shard.
dvl_status dist_build(dvl_ctx* ctx, uint64_t n, const uint32_t* lower_xyz, const uint8_t* level,
                      uint32_t members, const float* const* scalars, dvl_mem where) {
  Comm& C = *ctx->comm;
  const int G = C.nranks, r = C.rank;
  Dataset d;
  Tmp tmp;
  auto cleanup = [&]() {
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    for (void* p : tmp) dfree(ctx, p);
  };
  uint64_t cell_offset = 0, n_global = 0;
  int lmax_global = 0;
  try {
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    const int64_t nl = (int64_t)n;
    const int M = (int)members;
    // local argument errors join the first agreement
    dvl_status argst = DVL_OK;
    std::string argmsg;
    if (n >= (1ull << 30)) { argst = DVL_E_RANGE; argmsg = "n must be < 2^30 per device"; }
    if (members < 1 || members > (uint32_t)kMaxM) { argst = DVL_E_INVAL; argmsg = "members must be in [1, 64]"; }
    if (n > 0 && (!lower_xyz || !level || !scalars)) { argst = DVL_E_INVAL; argmsg = "NULL input pointer"; }
    if (where != DVL_MEM_HOST && where != DVL_MEM_DEVICE) { argst = DVL_E_INVAL; argmsg = "bad dvl_mem"; }
    if (argst == DVL_OK && n > 0)
      for (uint32_t m = 0; m < members; ++m)
        if (!scalars[m]) { argst = DVL_E_INVAL; argmsg = "NULL scalar pointer"; }
    agree(ctx, argst, argmsg);

    // ---- 0. ingest of the local slice; global extent, Lmax, n, M (all ranks must agree)
    tic(ctx, PH_INGEST);
    Inputs in = stage_inputs(ctx, nl, lower_xyz, level, M, scalars, where, tmp);
    IngestOut* d_ing = new_ingest(ctx, tmp);
    if (nl > 0) {
      launch_ingest_geom(in.lower, in.level, nl, d_ing, ctx->num_sms, st);
      CKLAUNCH();
    }
    toc(ctx, PH_INGEST);
    IngestOut h_ing;
    read_ingest(ctx, d_ing, &h_ing);
    {
      Small mx(ctx, 4), sm(ctx, 2);
      mx.put({h_ing.extent, h_ing.lmax, h_ing.err, (uint64_t)M});
      sm.put({(uint64_t)nl, (uint64_t)M});
      comm_ck(ctx, C.allreduce(mx.d, 4, kU64, kMax, st), "all_reduce MAX");
      comm_ck(ctx, C.allreduce(sm.d, 2, kU64, kSum, st), "all_reduce SUM");
      const std::vector<uint64_t> a = mx.get(4), b = sm.get(2);
      if (a[2] & kErrInval) fail(ctx, DVL_E_INVAL, "a cell has L > 20 or a lower corner not a multiple of 2^L");
      if (b[1] != (uint64_t)G * (uint64_t)M || a[3] != (uint64_t)M)
        fail(ctx, DVL_E_INVAL, "the ranks pass different member counts");
      if (b[0] == 0) fail(ctx, DVL_E_INVAL, "no cells on any rank");
      if (a[0] > (1ull << 21)) fail(ctx, DVL_E_RANGE, "logical extent E > 2^21");
      if (ceil_lmax_p(lscale(ctx) * (int)a[1], ctx->P) > 100)
        fail(ctx, DVL_E_RANGE, "ceil(Lmax * P) > 100 (fp32 weight overflow)");
      n_global = b[0];
      lmax_global = (int)a[1];
      d.b = std::max(1, ceil_log2_u64(a[0]));
      if (ctx->global_bits > 0) d.b = std::max(d.b, ctx->global_bits);
    }
    d.M = M;
    d.E = (uint32_t)h_ing.extent;
    const int kb = 3 * d.b <= 32 ? 4 : 8;
    // input offsets of the slices (global input ids = offset + local id)
    std::vector<uint64_t> nin(G);
    {
      Small one(ctx, 1), all(ctx, G);
      one.put({(uint64_t)nl});
      comm_ck(ctx, C.allgather(one.d, all.d, 8, st), "all_gather n");
      nin = all.get(G);
    }
    uint64_t in_offset = 0;
    for (int p = 0; p < r; ++p) in_offset += nin[p];

    // ---- 1. local encode + sort, gather into curve-ordered SoA (+ global ids)
    CK(cudaMemsetAsync(ctx->d_err, 0, 4, st));
    const int64_t nl8 = (nl + 7) & ~7ll;
    void* keys_l = dmalloc(ctx, (size_t)kb * std::max<int64_t>(nl, 1));
    tmp.push_back(keys_l);
    unsigned long long* ids_l = dalloc<unsigned long long>(ctx, std::max<int64_t>(nl, 1));
    uint8_t* lev_l = dalloc<uint8_t>(ctx, std::max<int64_t>(nl8, 8));
    float* sc_l = dalloc<float>(ctx, (size_t)M * std::max<int64_t>(nl8, 8));
    tmp.push_back(ids_l);
    tmp.push_back(lev_l);
    tmp.push_back(sc_l);
    Sorted loc;
    if (nl > 0) {
      loc = sort_codes(ctx, in.lower, in.level, keys_l, nl, d.b, kb, tmp);
      if (loc.keys != keys_l) tmp.push_back(loc.keys);
      tmp.push_back(loc.perm);
      Dataset t;
      t.n = nl;
      t.n_pad = nl8;
      t.M = M;
      t.key_bytes = kb;
      t.keys = loc.keys;
      t.perm = loc.perm;
      t.level_s = lev_l;
      t.scal_s = sc_l;
      launch_gather_validate4(t.keys, kb, t.perm, in.level, in.d_ptrs, nl, M, nl8, lev_l, sc_l,
                              ctx->d_err, d_ing, ctx->num_sms, st);
      CKLAUNCH();
      launch_offset_ids(loc.perm, nl, in_offset, ids_l, ctx->num_sms, st);
      CKLAUNCH();
    }
    const void* skeys = nl > 0 ? loc.keys : keys_l;

    // ---- 2. samples -> splitters (identical on every rank)
    constexpr int S = 1024;
    std::vector<uint64_t> spl(std::max(G - 1, 1));
    {
      Small samp(ctx, S), all(ctx, (size_t)G * S);
      launch_sample_keys(skeys, kb, nl, S, samp.d, st);
      CKLAUNCH();
      comm_ck(ctx, C.allgather(samp.d, all.d, 8 * S, st), "all_gather samples");
      const std::vector<uint64_t> hs = all.get((size_t)G * S);
      if (G > 1 && !select_splitters(hs.data(), nin.data(), G, S, spl.data()))
        fail(ctx, DVL_E_INVAL, "fewer distinct cells than ranks: no valid splitters");
    }
    // ---- 3. send ranges (lower_bound of each splitter), the G x G count matrix
    std::vector<uint64_t> bnd(G + 1, 0);
    bnd[G] = (uint64_t)nl;
    if (G > 1 && nl > 0) {
      Small ds(ctx, G - 1), db(ctx, G - 1);
      ds.put(std::vector<uint64_t>(spl.begin(), spl.begin() + (G - 1)));
      launch_lower_bounds(skeys, kb, nl, ds.d, G - 1, db.d, st);
      CKLAUNCH();
      const std::vector<uint64_t> lb = db.get(G - 1);
      for (int p = 1; p < G; ++p) bnd[p] = lb[p - 1];
    } else if (G > 1) {
      for (int p = 1; p < G; ++p) bnd[p] = 0;
    }
    const uint32_t lerr = read_err(ctx);   // overlap inside the local run
    std::vector<uint64_t> mat((size_t)G * (G + 1));
    {
      std::vector<uint64_t> row(G + 1);
      for (int p = 0; p < G; ++p) row[p] = bnd[p + 1] - bnd[p];
      row[G] = lerr;
      Small one(ctx, G + 1), all(ctx, (size_t)G * (G + 1));
      one.put(row);
      comm_ck(ctx, C.allgather(one.d, all.d, 8 * (G + 1), st), "all_gather counts");
      mat = all.get((size_t)G * (G + 1));
    }
    std::vector<uint64_t> nrecv(G, 0);   // cells each rank receives
    for (int src = 0; src < G; ++src) {
      if (mat[(size_t)src * (G + 1) + G] & kErrOverlap) fail(ctx, DVL_E_OVERLAP, "duplicate or overlapping cells");
      for (int dst = 0; dst < G; ++dst) nrecv[dst] += mat[(size_t)src * (G + 1) + dst];
    }
    for (int p = 0; p < G; ++p)
      if (nrecv[p] == 0) fail(ctx, DVL_E_INVAL, "a rank would hold no cells (fewer distinct cells than ranks)");
    for (int p = 0; p < r; ++p) cell_offset += nrecv[p];
    const int64_t nr = (int64_t)nrecv[r];
    if (nr >= (1ll << 30)) fail(ctx, DVL_E_RANGE, "a rank would hold >= 2^30 cells");

    // ---- 4. exchange (codes, global ids, levels, member rows), each in curve order
    const int64_t nr8 = (nr + 7) & ~7ll;
    void* keys_r = dmalloc(ctx, (size_t)kb * nr);
    unsigned long long* ids_r = dalloc<unsigned long long>(ctx, nr);
    uint8_t* lev_r = dalloc<uint8_t>(ctx, nr8);
    float* sc_r = dalloc<float>(ctx, (size_t)M * nr8);
    tmp.push_back(keys_r);
    tmp.push_back(ids_r);
    tmp.push_back(lev_r);
    tmp.push_back(sc_r);
    std::vector<uint64_t> roff(G + 1, 0);   // received segment offsets (source rank order)
    for (int p = 0; p < G; ++p) roff[p + 1] = roff[p] + mat[(size_t)p * (G + 1) + r];
    auto exchange = [&](const void* sbase, void* rbase, size_t esize, const char* what) {
      std::vector<const void*> sp(G);
      std::vector<void*> rp(G);
      std::vector<size_t> sb(G), rb(G);
      for (int p = 0; p < G; ++p) {
        sp[p] = static_cast<const char*>(sbase) + bnd[p] * esize;
        sb[p] = (bnd[p + 1] - bnd[p]) * esize;
        rp[p] = static_cast<char*>(rbase) + roff[p] * esize;
        rb[p] = (roff[p + 1] - roff[p]) * esize;
      }
      comm_ck(ctx, C.alltoallv(sp.data(), sb.data(), rp.data(), rb.data(), st), what);
    };
    exchange(skeys, keys_r, kb, "exchange codes");
    exchange(ids_l, ids_r, 8, "exchange ids");
    exchange(lev_l, lev_r, 1, "exchange levels");
    for (int m = 0; m < M; ++m)
      exchange(sc_l + (size_t)m * nl8, sc_r + (size_t)m * nr8, 4, "exchange scalars");

    // ---- 5. combine the G sorted runs: the codes are distinct, so the bucket placement
    //         (slots, offsets, bitmap rank) gives the order without re-encoding
    CK(cudaMemsetAsync(ctx->d_err, 0, 4, st));
    d.n = nr;
    d.Lmax = lmax_global;
    set_geometry(ctx, d);
    Sorted fin = sort_codes(ctx, nullptr, nullptr, keys_r, nr, d.b, kb, tmp);
    if (fin.keys == keys_r) tmp.erase(std::find(tmp.begin(), tmp.end(), keys_r));
    d.keys = fin.keys;
    d.perm = fin.perm;   // index into the received arrays (replaced by gids for get_sorted)
    std::vector<const float*> rows(M);
    for (int m = 0; m < M; ++m) rows[m] = sc_r + (size_t)m * nr8;
    const float** d_rows = (const float**)dmalloc(ctx, sizeof(float*) * M);
    tmp.push_back((void*)d_rows);
    CK(cudaMemcpyAsync(d_rows, rows.data(), sizeof(float*) * M, cudaMemcpyHostToDevice, st));
    IngestOut* d_rng = new_ingest(ctx, tmp);
    gather_sorted(ctx, d, lev_r, d_rows, d_rng);
    d.gids = dalloc<unsigned long long>(ctx, nr);
    launch_gather_u64(ids_r, fin.perm, nr, d.gids, ctx->num_sms, st);
    CKLAUNCH();

    // ---- 6. overlap inside the range and across the rank boundaries; global ranges
    const uint32_t ferr = read_err(ctx);
    std::vector<uint64_t> ends(5, 0);
    {
      uint64_t k0 = 0, k1 = 0;
      uint8_t l0 = 0, l1 = 0;
      CK(cudaMemcpyAsync(&k0, d.keys, kb, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(&k1, static_cast<char*>(d.keys) + (size_t)(nr - 1) * kb, kb,
                         cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(&l0, d.level_s, 1, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(&l1, d.level_s + nr - 1, 1, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      ends = {ferr, k0, l0, k1, l1};
    }
    std::vector<uint64_t> allends;
    {
      Small one(ctx, 5), all(ctx, (size_t)G * 5);
      one.put(ends);
      comm_ck(ctx, C.allgather(one.d, all.d, 40, st), "all_gather run ends");
      allends = all.get((size_t)G * 5);
    }
    for (int p = 0; p < G; ++p)
      if (allends[5 * p] & kErrOverlap) fail(ctx, DVL_E_OVERLAP, "duplicate or overlapping cells");
    for (int p = 0; p + 1 < G; ++p) {
      const uint64_t a = allends[5 * p + 3], La = allends[5 * p + 4];
      const uint64_t b = allends[5 * (p + 1) + 1], Lb = allends[5 * (p + 1) + 2];
      const uint64_t lena = 1ull << (3 * La), lenb = 1ull << (3 * Lb);
      if (a >= b || (a & ~(lena - 1)) + lena > (b & ~(lenb - 1)))
        fail(ctx, DVL_E_OVERLAP, "duplicate or overlapping cells across ranks");
    }
    {
      IngestOut h;
      read_ingest(ctx, d_rng, &h);
      Small rng(ctx, 3 * (size_t)M);
      std::vector<uint64_t> v(3 * (size_t)M);
      for (int m = 0; m < M; ++m) {
        v[m] = h.any[m] ? h.vmin[m] : 0xffffffffull;
        v[M + m] = h.any[m] ? h.vmax[m] : 0ull;
        v[2 * M + m] = h.any[m];
      }
      rng.put(v);
      comm_ck(ctx, C.allreduce(rng.d, M, kU64, kMin, st), "all_reduce MIN ranges");
      comm_ck(ctx, C.allreduce(rng.d + M, 2 * (size_t)M, kU64, kMax, st), "all_reduce MAX ranges");
      v = rng.get(3 * (size_t)M);
      for (int m = 0; m < M; ++m) {
        h.vmin[m] = (uint32_t)v[m];
        h.vmax[m] = (uint32_t)v[M + m];
        h.any[m] = (uint32_t)v[2 * M + m];
      }
      ranges_from(d, h);
    }
    alloc_update_state(ctx, d);
  } catch (Fail& f) {
    cleanup();
    free_dataset(ctx, d);
    return f.s;
  }
  cleanup();
  return commit_dataset(ctx, d, true, cell_offset, n_global, lmax_global);
}

}  // namespace

dvl_status dvl_set_params(dvl_ctx* ctx, float P, float eps, dvl_maxv_mode mode) {
  if (!ctx) return DVL_E_INVAL;
  if (!(P >= 0.0f && P <= 16.0f)) {
    set_err(ctx, "P must be in [0, 16]");
    return DVL_E_INVAL;
  }
  if (!(eps >= 0.0f && eps <= 1.0f)) {
    set_err(ctx, "eps must be in [0, 1]");
    return DVL_E_INVAL;
  }
  if (mode != DVL_MAXV_CONSERVATIVE && mode != DVL_MAXV_PER_ENTRY && mode != DVL_MAXV_EXACT) {
    set_err(ctx, "bad maxV mode");
    return DVL_E_INVAL;
  }
  if (ctx->built && ceil_lmax_p(lscale(ctx) * lmax_eff(ctx), P) > 100) {
    set_err(ctx, "ceil(Lmax * P) > 100 (fp32 weight overflow)");
    return DVL_E_RANGE;
  }
  ctx->P = P;
  ctx->eps = eps;
  ctx->mode = mode;
  if (ctx->built) {
    try {
      CK(cudaSetDevice(ctx->device));
      run_weights(ctx, false, nullptr);
    } catch (Fail& f) {
      return f.s;
    }
  }
  return DVL_OK;
}

dvl_status dvl_set_level_scale(dvl_ctx* ctx, dvl_level_scale scale) {
  if (!ctx) return DVL_E_INVAL;
  if (scale != DVL_SCALE_WIDTH && scale != DVL_SCALE_VOLUME) {
    set_err(ctx, "bad level scale");
    return DVL_E_INVAL;
  }
  const int c = scale == DVL_SCALE_VOLUME ? 3 : 1;
  if (ctx->built && ceil_lmax_p(c * lmax_eff(ctx), ctx->P) > 100) {
    set_err(ctx, "ceil(c Lmax P) > 100 (fp32 weight overflow)");
    return DVL_E_RANGE;
  }
  ctx->volume = scale == DVL_SCALE_VOLUME;
  if (ctx->built) {
    try {
      CK(cudaSetDevice(ctx->device));
      run_weights(ctx, false, nullptr);
    } catch (Fail& f) {
      return f.s;
    }
  }
  return DVL_OK;
}

dvl_status dvl_set_domain(dvl_ctx* ctx, uint32_t member, float lo, float hi) {
  if (!ctx) return DVL_E_INVAL;
  if (!ctx->built) {
    set_err(ctx, "dvl_set_domain before dvl_build");
    return DVL_E_STATE;
  }
  if (member >= (uint32_t)ctx->ds.M || !std::isfinite(lo) || !std::isfinite(hi) || hi < lo) {
    set_err(ctx, "bad member or domain");
    return DVL_E_INVAL;
  }
  try {
    CK(cudaSetDevice(ctx->device));
    ctx->lo_h[member] = lo;
    ctx->hi_h[member] = hi;
    ctx->inv_h[member] = hi > lo ? 1.0f / (hi - lo) : 0.0f;
    CK(cudaStreamSynchronize(ctx->stream));   // host vectors are the copy source
    upload_domains(ctx);
    run_weights(ctx, false, nullptr);
  } catch (Fail& f) {
    return f.s;
  }
  return DVL_OK;
}

static dvl_status check_tf(dvl_ctx* ctx, const float* rgba, uint32_t N) {
  if (!rgba || N < 2 || N > (uint32_t)kMaxN) {
    set_err(ctx, "TF size N must be in [2, 4096]");
    return DVL_E_INVAL;
  }
  for (uint32_t i = 0; i < 4 * N; ++i)
    if (!(rgba[i] >= 0.0f && rgba[i] <= 1.0f)) {
      set_err(ctx, "TF channels must be in [0, 1]");
      return DVL_E_INVAL;
    }
  return DVL_OK;
}

dvl_status dvl_update_tf(dvl_ctx* ctx, uint32_t member, const float* rgba, uint32_t N) {
  if (!ctx) return DVL_E_INVAL;

  if (!ctx->built) {
    set_err(ctx, "dvl_update_tf before dvl_build");
    return DVL_E_STATE;
  }
  if (member >= (uint32_t)ctx->ds.M) {
    set_err(ctx, "member out of range");
    return DVL_E_INVAL;
  }
  dvl_status s = check_tf(ctx, rgba, N);
  if (s != DVL_OK) return s;
  if ((int)N != ctx->N) {
    set_err(ctx, "all members share one TF size; use dvl_reset_tfs to change it");
    return DVL_E_INVAL;
  }
  try {
    CK(cudaSetDevice(ctx->device));
    stage_tf(ctx, rgba, (int)N);
    run_weights(ctx, false, nullptr, (int)member);
  } catch (Fail& f) {
    return f.s;
  }
  return DVL_OK;
}

dvl_status dvl_reset_tfs(dvl_ctx* ctx, uint32_t N) {
  if (!ctx) return DVL_E_INVAL;
  if (!ctx->built) {
    set_err(ctx, "dvl_reset_tfs before dvl_build");
    return DVL_E_STATE;
  }
  if (N < 2 || N > (uint32_t)kMaxN) {
    set_err(ctx, "TF size N must be in [2, 4096]");
    return DVL_E_INVAL;
  }
  try {
    CK(cudaSetDevice(ctx->device));
    ctx->N = (int)N;
    std::vector<float> tf;
    identity_tf_host(tf, (int)N);
    set_all_tfs(ctx, tf, (int)N);
    run_weights(ctx, false, nullptr);
  } catch (Fail& f) {
    return f.s;
  }
  return DVL_OK;
}

dvl_status dvl_shard_reduce(dvl_ctx* ctx, uint32_t W, const uint64_t* totals_dev, int nshards,
                            int shard, int64_t* export_dev);
dvl_status dvl_shard_finish(dvl_ctx* ctx, uint32_t W, const int64_t* merged_dev, dvl_vertex* out,
                            dvl_mem where);

// dvl_get_polylines of a context with its own communicator: the sharded edit of SURVEY 8(e)
// as one call -- all_gather of the Q totals, pass 2 with the global offset, the export, one
// grouped MAX + SUM all_reduce of it, the merged epilogue -- all on the context stream.
static dvl_status sharded_polylines(dvl_ctx* ctx, uint32_t W, dvl_vertex* out, dvl_mem where) {
  try {
    CK(cudaSetDevice(ctx->device));
    const uint64_t words = dvl_shard_export_words(ctx, W);
    if (words > ctx->export_cap) {
      dfree(ctx, ctx->d_export);
      ctx->d_export = dalloc<int64_t>(ctx, (size_t)words);
      ctx->export_cap = words;
    }
    if (const char* e = ctx->comm->allgather(ctx->d_qtot, ctx->d_totals, 8, ctx->stream))
      fail(ctx, DVL_E_NCCL, std::string("all_gather of the totals: ") + e);
  } catch (Fail& f) {
    return f.s;
  }
  dvl_status s = dvl_shard_reduce(ctx, W, (const uint64_t*)ctx->d_totals, ctx->comm_ranks,
                                  ctx->comm_rank, ctx->d_export);
  if (s != DVL_OK) return s;
  const uint64_t MW = (uint64_t)ctx->ds.M * W;
  if (const char* e = ctx->comm->merge_export(ctx->d_export, 2 * (W + MW), 3 * MW, ctx->stream)) {
    set_err(ctx, std::string("merge of the exports: ") + e);
    return DVL_E_NCCL;
  }
  return dvl_shard_finish(ctx, W, ctx->d_export, out, where);
}

dvl_status dvl_get_polylines(dvl_ctx* ctx, uint32_t W, dvl_vertex* out, dvl_mem where) {
  if (!ctx) return DVL_E_INVAL;

  if (!ctx->built) {
    set_err(ctx, "dvl_get_polylines before dvl_build");
    return DVL_E_STATE;
  }
  if (W < 2 || W > kMaxW || !out || (where != DVL_MEM_HOST && where != DVL_MEM_DEVICE)) {
    set_err(ctx, "W must be in [2, 65536] and out non-NULL");
    return DVL_E_INVAL;
  }
  if (ctx->comm && ctx->sharded) return sharded_polylines(ctx, W, out, where);
  try {
    CK(cudaSetDevice(ctx->device));
    ensure_acc(ctx, W);
    Dataset& d = ctx->ds;
    UpdParams p = upd_params(ctx);
    // the member planes are indexed m * W + x for this call (capacity >= W); the epilogue
    // restores the identity of every entry it reads, so all entries stay identity
    Acc a = cur_acc(ctx);
    tic(ctx, PH_BREDUCE);
    if (d.tma)   // (1-3 kernels; CKLAUNCH counts one)
      ctx->launches += launch_agg_reduce(p, pass2_plan(d), d.chunk_prefix, ctx->d_qtot, W, a,
                                         ctx->cell_offset, ctx->d_err, d.tile_meta, d.meta2, d.agg,
                                         d.blist, d.bctr, ctx->num_sms, ctx->stream) - 1;
    else
      launch_bin_reduce(d.items, smem_tab_ok(ctx), p, d.tile_prefix, ctx->d_qtot, W, a,
                        ctx->cell_offset, ctx->d_err, d.tiles, ctx->stream);
    CKLAUNCH();
    toc(ctx, PH_BREDUCE);
    // a page-locked host destination is written by the epilogue itself (zero copy through
    // its device alias); pageable host memory goes through the context's device buffer
    dvl_vertex* dst = where == DVL_MEM_DEVICE ? out : ctx->d_out;
    bool direct = false;
    if (where == DVL_MEM_HOST) {
      cudaPointerAttributes at{};
      if (cudaPointerGetAttributes(&at, out) == cudaSuccess && at.type == cudaMemoryTypeHost &&
          at.devicePointer != nullptr && (reinterpret_cast<uintptr_t>(at.devicePointer) & 15) == 0) {
        dst = static_cast<dvl_vertex*>(at.devicePointer);
        direct = true;
      }
      (void)cudaGetLastError();
    }
    // the error word lands in the context's mapped staging (written by the epilogue)
    const bool check = where == DVL_MEM_HOST || maybe_degenerate(ctx);
    uint32_t* herr_p = reinterpret_cast<uint32_t*>(ctx->h_stage + 2 * 4 * kMaxN);
    uint32_t* herr_dev = reinterpret_cast<uint32_t*>(ctx->d_hstage + 2 * 4 * kMaxN);
    tic(ctx, PH_EPI);
    launch_epilogue(a, W, d.M, ctx->N, d.d_rgba, dst, ctx->d_bin_lo, ctx->d_bin_hi, ctx->d_err,
                    check ? herr_dev : nullptr, ctx->stream);
    CKLAUNCH();
    // the epilogue restored the other copy over [0, W); if an earlier, wider call left
    // pixels beyond W in it, restore those too, so the next call (which uses it) starts
    // from the identity whatever its width
    {
      const int other = ctx->acc_par ^ 1;
      if (ctx->acc_dirty[other] > W) {
        const size_t tail = (size_t)(ctx->acc_dirty[other] - W) * sizeof(unsigned long long);
        CK(cudaMemsetAsync(a.lo2 + W, 0xff, tail, ctx->stream));
        CK(cudaMemsetAsync(a.hi2 + W, 0x00, tail, ctx->stream));
      }
      ctx->acc_dirty[other] = 0;
      ctx->acc_dirty[ctx->acc_par] = W;
    }
    ctx->acc_par ^= 1;   // this call's copy is restored by the next call's epilogue
    toc(ctx, PH_EPI);
    ctx->last_W = W;
    if (where == DVL_MEM_HOST && !direct) {
      // pageable destination: the driver's staged copy
      CK(cudaMemcpyAsync(out, ctx->d_out, sizeof(dvl_vertex) * (size_t)W * d.M,
                         cudaMemcpyDeviceToHost, ctx->stream));
    }
    if (check) {
      CK(cudaStreamSynchronize(ctx->stream));
      const uint32_t herr = *(volatile uint32_t*)herr_p;
      if (herr & kErrDegenerate) {
        CK(cudaMemsetAsync(ctx->d_err, 0, 4, ctx->stream));
        ctx->last_W = 0;
        fail(ctx, DVL_E_DEGENERATE, "all weights are 0 (Qtot = 0)");
      }
    }
  } catch (Fail& f) {
    return f.s;
  }
  return DVL_OK;
}

dvl_status dvl_set_global_bits(dvl_ctx* ctx, int bits) {
  if (!ctx) return DVL_E_INVAL;
  if (bits < 0 || bits > 21) {
    set_err(ctx, "global bits must be in [0, 21]");
    return DVL_E_INVAL;
  }
  ctx->global_bits = bits;
  return DVL_OK;
}

dvl_status dvl_set_shard(dvl_ctx* ctx, const dvl_shard_info* info) {
  if (!ctx || !info) return DVL_E_INVAL;
  if (!ctx->built) {
    set_err(ctx, "dvl_set_shard before dvl_build");
    return DVL_E_STATE;
  }
  const Dataset& d = ctx->ds;
  if (info->cell_offset + (uint64_t)d.n > info->n_global || info->n_global >= (1ull << 40) ||
      info->lmax_global < d.Lmax || info->lmax_global > 20) {
    set_err(ctx, "inconsistent shard description");
    return DVL_E_INVAL;
  }
  if (ceil_lmax_p(lscale(ctx) * (int)info->lmax_global, ctx->P) > 100) {
    set_err(ctx, "ceil(Lmax * P) > 100 (fp32 weight overflow)");
    return DVL_E_RANGE;
  }
  try {
    CK(cudaSetDevice(ctx->device));
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->sharded = true;
    ctx->cell_offset = info->cell_offset;
    ctx->n_global = info->n_global;
    ctx->lmax_global = info->lmax_global;
    Dataset& dd = ctx->ds;
    if (info->vmin && info->vmax) {
      for (int m = 0; m < dd.M; ++m) {
        dd.vmin[m] = info->vmin[m];
        dd.vmax[m] = info->vmax[m];
      }
      CK(cudaMemcpyAsync(dd.d_vmin, dd.vmin.data(), 4 * dd.M, cudaMemcpyHostToDevice, ctx->stream));
      CK(cudaMemcpyAsync(dd.d_vmax, dd.vmax.data(), 4 * dd.M, cudaMemcpyHostToDevice, ctx->stream));
    }
    ctx->lo_h = dd.vmin;
    ctx->hi_h = dd.vmax;
    for (int m = 0; m < dd.M; ++m)
      ctx->inv_h[m] = ctx->hi_h[m] > ctx->lo_h[m] ? 1.0f / (ctx->hi_h[m] - ctx->lo_h[m]) : 0.0f;
    upload_domains(ctx);
    run_weights(ctx, false, nullptr);
  } catch (Fail& f) {
    return f.s;
  }
  return DVL_OK;
}

dvl_status dvl_shard_total(dvl_ctx* ctx, uint64_t* total_dev) {
  if (!ctx || !total_dev) return DVL_E_INVAL;
  if (!ctx->built) {
    set_err(ctx, "no dataset");
    return DVL_E_STATE;
  }
  try {
    CK(cudaSetDevice(ctx->device));
    CK(cudaMemcpyAsync(total_dev, ctx->d_qtot, 8, cudaMemcpyDeviceToDevice, ctx->stream));
  } catch (Fail& f) {
    return f.s;
  }
  return DVL_OK;
}

dvl_status dvl_nccl_unique_id(void* id128) {
  if (!id128) return DVL_E_INVAL;
  return nccl_unique_id(id128) ? DVL_E_NCCL : DVL_OK;
}

dvl_status dvl_local_group_create(int nranks, void** group) {
  if (!group || nranks < 1) return DVL_E_INVAL;
  *group = new GroupHandle{local_group_create(nranks)};
  return DVL_OK;
}

void dvl_local_group_destroy(void* group) {
  if (!group) return;
  GroupHandle* h = static_cast<GroupHandle*>(group);
  local_group_release(h->g);
  delete h;
}

dvl_status dvl_set_local_comm(dvl_ctx* ctx, void* group, int rank) {
  if (!ctx) return DVL_E_INVAL;
  GroupHandle* h = static_cast<GroupHandle*>(group);
  if (!h || rank < 0 || rank >= local_group_size(h->g)) {
    set_err(ctx, "bad local group or rank");
    return DVL_E_INVAL;
  }
  try {
    CK(cudaSetDevice(ctx->device));
    if (ctx->comm) {
      CK(cudaStreamSynchronize(ctx->stream));
      delete ctx->comm;
      ctx->comm = nullptr;
    }
    attach_comm(ctx, make_local_comm(h->g, rank));
  } catch (Fail& f) {
    return f.s;
  }
  return DVL_OK;
}

dvl_status dvl_get_shard(dvl_ctx* ctx, dvl_shard_info* out) {
  if (!ctx || !out) return DVL_E_INVAL;
  if (!ctx->built) {
    set_err(ctx, "no dataset");
    return DVL_E_STATE;
  }
  memset(out, 0, sizeof *out);
  out->cell_offset = ctx->cell_offset;
  out->n_global = ctx->sharded ? ctx->n_global : (uint64_t)ctx->ds.n;
  out->lmax_global = ctx->sharded ? ctx->lmax_global : ctx->ds.Lmax;
  return DVL_OK;
}

dvl_status dvl_select_splitters(const uint64_t* samples, const uint64_t* counts, int nranks,
                                int per_rank, uint64_t* splitters) {
  if (!samples || !counts || !splitters || nranks < 2 || per_rank < 1) return DVL_E_INVAL;
  return select_splitters(samples, counts, nranks, per_rank, splitters) ? DVL_OK : DVL_E_INVAL;
}

dvl_status dvl_set_comm(dvl_ctx* ctx, int nranks, int rank, const void* id128) {
  if (!ctx) return DVL_E_INVAL;
  if (nranks < 1 || rank < 0 || rank >= nranks || !id128) {
    set_err(ctx, "bad communicator arguments");
    return DVL_E_INVAL;
  }
  try {
    CK(cudaSetDevice(ctx->device));
    if (ctx->comm) {
      CK(cudaStreamSynchronize(ctx->stream));
      delete ctx->comm;
      ctx->comm = nullptr;
    }
    const char* e = nullptr;
    Comm* c = make_nccl_comm(nranks, rank, id128, &e);
    if (!c) fail(ctx, DVL_E_NCCL, std::string("ncclCommInitRank: ") + (e ? e : "?"));
    attach_comm(ctx, c);
  } catch (Fail& f) {
    return f.s;
  }
  return DVL_OK;
}

uint64_t dvl_shard_export_words(dvl_ctx* ctx, uint32_t W) {
  if (!ctx || !ctx->built) return 0;
  const uint64_t MW = (uint64_t)ctx->ds.M * W;
  return 2 * (W + MW) + 3 * MW;
}

dvl_status dvl_shard_reduce(dvl_ctx* ctx, uint32_t W, const uint64_t* totals_dev, int nshards,
                            int shard, int64_t* export_dev) {
  if (!ctx) return DVL_E_INVAL;
  if (!ctx->built) {
    set_err(ctx, "dvl_shard_reduce before dvl_build");
    return DVL_E_STATE;
  }
  if (W < 2 || W > kMaxW || !totals_dev || !export_dev || nshards < 1 || shard < 0 ||
      shard >= nshards) {
    set_err(ctx, "bad shard reduce arguments");
    return DVL_E_INVAL;
  }
  try {
    CK(cudaSetDevice(ctx->device));
    ensure_acc(ctx, W);
    Dataset& d = ctx->ds;
    UpdParams p = upd_params(ctx);
    if (d.tma) {   // pass 2 sums the offset and Qtot from the totals itself
      p.shard_totals = (const unsigned long long*)totals_dev;
      p.nshards = nshards;
      p.shard = shard;
    } else {
      launch_shard_offsets((const unsigned long long*)totals_dev, nshards, shard, ctx->d_offset,
                           ctx->d_qtot_glob, ctx->stream);
      CKLAUNCH();
      p.offset_dev = ctx->d_offset;
    }
    Acc a = cur_acc(ctx);
    tic(ctx, PH_BREDUCE);
    if (d.tma)   // (1-3 kernels; CKLAUNCH counts one)
      ctx->launches += launch_agg_reduce(p, pass2_plan(d), d.chunk_prefix, ctx->d_qtot_glob, W, a,
                                         ctx->cell_offset, ctx->d_err, d.tile_meta, d.meta2, d.agg,
                                         d.blist, d.bctr, ctx->num_sms, ctx->stream) - 1;
    else
      launch_bin_reduce(d.items, smem_tab_ok(ctx), p, d.tile_prefix, ctx->d_qtot_glob, W, a,
                        ctx->cell_offset, ctx->d_err, d.tiles, ctx->stream);
    CKLAUNCH();
    toc(ctx, PH_BREDUCE);
    launch_acc_export(a, W, d.M, (long long*)export_dev, ctx->stream);
    CKLAUNCH();
  } catch (Fail& f) {
    return f.s;
  }
  return DVL_OK;
}

dvl_status dvl_shard_finish(dvl_ctx* ctx, uint32_t W, const int64_t* merged_dev, dvl_vertex* out,
                            dvl_mem where) {
  if (!ctx) return DVL_E_INVAL;
  if (!ctx->built) {
    set_err(ctx, "dvl_shard_finish before dvl_build");
    return DVL_E_STATE;
  }
  if (W < 2 || W > kMaxW || !merged_dev || !out || (where != DVL_MEM_HOST && where != DVL_MEM_DEVICE)) {
    set_err(ctx, "bad shard finish arguments");
    return DVL_E_INVAL;
  }
  try {
    CK(cudaSetDevice(ctx->device));
    ensure_acc(ctx, W);
    Dataset& d = ctx->ds;
    dvl_vertex* dst = where == DVL_MEM_DEVICE ? out : ctx->d_out;
    tic(ctx, PH_EPI);
    launch_epilogue_merged((const long long*)merged_dev, W, d.M, ctx->N, d.d_rgba, dst,
                           ctx->d_bin_lo, ctx->d_bin_hi, ctx->stream);
    CKLAUNCH();
    toc(ctx, PH_EPI);
    ctx->last_W = W;
    if (where == DVL_MEM_HOST) {
      CK(cudaMemcpyAsync(out, ctx->d_out, sizeof(dvl_vertex) * (size_t)W * d.M,
                         cudaMemcpyDeviceToHost, ctx->stream));
      uint32_t herr = 0;
      CK(cudaMemcpyAsync(&herr, ctx->d_err, 4, cudaMemcpyDeviceToHost, ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));
      if (herr & kErrDegenerate) {
        CK(cudaMemsetAsync(ctx->d_err, 0, 4, ctx->stream));
        ctx->last_W = 0;
        fail(ctx, DVL_E_DEGENERATE, "all weights are 0 (Qtot = 0)");
      }
    }
  } catch (Fail& f) {
    return f.s;
  }
  return DVL_OK;
}

dvl_status dvl_info(dvl_ctx* ctx, dvl_info_t* info) {
  if (!ctx || !info) return DVL_E_INVAL;
  memset(info, 0, sizeof *info);
  try {
    CK(cudaSetDevice(ctx->device));
    CK(cudaStreamSynchronize(ctx->stream));
    info->P = ctx->P;
    info->eps = ctx->eps;
    info->maxv_mode = ctx->mode;
    info->device_bytes = ctx->bytes;
    info->tf_size = ctx->N;
    if (ctx->built) {
      const Dataset& d = ctx->ds;
      info->n = (uint64_t)d.n;
      info->members = (uint32_t)d.M;
      info->extent = d.E;
      info->bits = d.b;
      info->Lmax = d.Lmax;
      info->key_bytes = d.key_bytes;
      info->shift = ctx->shift;
      info->cells_per_tile = kBlock * d.items;
      CK(cudaMemcpy(&info->maxV, ctx->d_maxv, 4, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(&info->Qtot, ctx->d_qtot, 8, cudaMemcpyDeviceToHost));
    }
  } catch (Fail& f) {
    return f.s;
  }
  return DVL_OK;
}

static cudaMemcpyKind out_kind(dvl_mem where) {
  return where == DVL_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
}

dvl_status dvl_get_sorted(dvl_ctx* ctx, uint64_t* codes, uint64_t* ids, dvl_mem where) {
  if (!ctx) return DVL_E_INVAL;
  if (!ctx->built) {
    set_err(ctx, "no dataset");
    return DVL_E_STATE;
  }
  std::vector<void*> tmp;
  try {
    CK(cudaSetDevice(ctx->device));
    const int64_t n = ctx->ds.n;
    uint64_t* dc = nullptr;
    uint64_t* di = nullptr;
    if (codes) {
      dc = where == DVL_MEM_DEVICE ? codes : dalloc<uint64_t>(ctx, n);
      if (where != DVL_MEM_DEVICE) tmp.push_back(dc);
    }
    if (ids) {
      di = where == DVL_MEM_DEVICE ? ids : dalloc<uint64_t>(ctx, n);
      if (where != DVL_MEM_DEVICE) tmp.push_back(di);
    }
    launch_widen(ctx->ds.keys, ctx->ds.key_bytes, ctx->ds.perm, n, dc, ctx->ds.gids ? nullptr : di,
                 ctx->stream);
    CKLAUNCH();
    if (ctx->ds.gids && di)   // distributed build: the global input ids
      CK(cudaMemcpyAsync(di, ctx->ds.gids, 8 * n, cudaMemcpyDeviceToDevice, ctx->stream));
    if (where == DVL_MEM_HOST) {
      if (codes) CK(cudaMemcpyAsync(codes, dc, 8 * n, cudaMemcpyDeviceToHost, ctx->stream));
      if (ids) CK(cudaMemcpyAsync(ids, di, 8 * n, cudaMemcpyDeviceToHost, ctx->stream));
    }
    CK(cudaStreamSynchronize(ctx->stream));
  } catch (Fail& f) {
    for (void* p : tmp) dfree(ctx, p);
    return f.s;
  }
  for (void* p : tmp) dfree(ctx, p);
  return DVL_OK;
}

dvl_status dvl_get_sorted_data(dvl_ctx* ctx, uint8_t* level_sorted, float* scalars_sorted,
                               dvl_mem where) {
  if (!ctx) return DVL_E_INVAL;
  if (!ctx->built) {
    set_err(ctx, "no dataset");
    return DVL_E_STATE;
  }
  try {
    CK(cudaSetDevice(ctx->device));
    const Dataset& d = ctx->ds;
    if (level_sorted)
      CK(cudaMemcpyAsync(level_sorted, d.level_s, d.n, out_kind(where), ctx->stream));
    if (scalars_sorted)
      CK(cudaMemcpy2DAsync(scalars_sorted, 4 * d.n, d.scal_s, 4 * d.n_pad, 4 * d.n, d.M,
                           out_kind(where), ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  } catch (Fail& f) {
    return f.s;
  }
  return DVL_OK;
}

dvl_status dvl_get_prefix(dvl_ctx* ctx, uint64_t* Q, dvl_mem where) {
  if (!ctx || !Q) return DVL_E_INVAL;
  if (!ctx->built) {
    set_err(ctx, "no dataset");
    return DVL_E_STATE;
  }
  void* tmp = nullptr;
  try {
    CK(cudaSetDevice(ctx->device));
    const int64_t n = ctx->ds.n;
    unsigned long long* dq =
        where == DVL_MEM_DEVICE ? (unsigned long long*)Q : dalloc<unsigned long long>(ctx, n);
    if (where != DVL_MEM_DEVICE) tmp = dq;
    run_weights(ctx, true, dq);
    if (where == DVL_MEM_HOST) CK(cudaMemcpyAsync(Q, dq, 8 * n, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  } catch (Fail& f) {
    dfree(ctx, tmp);
    return f.s;
  }
  dfree(ctx, tmp);
  return DVL_OK;
}

namespace {
// point location, or (roi != nullptr: [lo code, hi code] on the host) the ROI test
dvl_status locate_points(dvl_ctx* ctx, uint64_t npts, const uint32_t* xyz, int64_t* cell,
                         dvl_mem where, const uint64_t* roi) {
  if (!ctx) return DVL_E_INVAL;
  if (!ctx->built) {
    set_err(ctx, "dvl_locate before dvl_build");
    return DVL_E_STATE;
  }
  if ((npts && (!xyz || !cell)) || (where != DVL_MEM_HOST && where != DVL_MEM_DEVICE)) {
    set_err(ctx, "dvl_locate: null buffer or bad memory space");
    return DVL_E_INVAL;
  }
  if (npts == 0) return DVL_OK;
  uint32_t* dx = nullptr;
  int64_t* dc = nullptr;
  unsigned long long* dr = nullptr;
  try {
    CK(cudaSetDevice(ctx->device));
    const Dataset& d = ctx->ds;
    const uint32_t* px = xyz;
    int64_t* pc = cell;
    if (where == DVL_MEM_HOST) {
      dx = dalloc<uint32_t>(ctx, 3 * (size_t)npts);
      dc = dalloc<int64_t>(ctx, (size_t)npts);
      CK(cudaMemcpyAsync(dx, xyz, 12 * (size_t)npts, cudaMemcpyHostToDevice, ctx->stream));
      px = dx;
      pc = dc;
    }
    if (roi) {
      dr = dalloc<unsigned long long>(ctx, 2);
      CK(cudaMemcpyAsync(dr, roi, 16, cudaMemcpyHostToDevice, ctx->stream));
    }
    launch_locate(px, (int64_t)npts, d.b, ctx->d_t1, ctx->d_t2, ctx->nstates, d.keys, d.key_bytes,
                  d.level_s, d.n, ctx->cell_offset, pc, ctx->stream, dr);
    CKLAUNCH();
    if (where == DVL_MEM_HOST) {
      CK(cudaMemcpyAsync(cell, dc, 8 * (size_t)npts, cudaMemcpyDeviceToHost, ctx->stream));
    }
    CK(cudaStreamSynchronize(ctx->stream));
  } catch (Fail& f) {
    dfree(ctx, dx);
    dfree(ctx, dc);
    dfree(ctx, dr);
    return f.s;
  }
  dfree(ctx, dx);
  dfree(ctx, dc);
  dfree(ctx, dr);
  return DVL_OK;
}
}  // namespace

dvl_status dvl_locate(dvl_ctx* ctx, uint64_t npts, const uint32_t* xyz, int64_t* cell,
                      dvl_mem where) {
  return locate_points(ctx, npts, xyz, cell, where, nullptr);
}

dvl_status dvl_roi_contains(dvl_ctx* ctx, uint64_t npts, const uint32_t* xyz, uint64_t code_lo,
                            uint64_t code_hi, int64_t* flag, dvl_mem where) {
  const uint64_t roi[2] = {code_lo, code_hi};
  return locate_points(ctx, npts, xyz, flag, where, roi);
}

dvl_status dvl_brush(dvl_ctx* ctx, uint32_t W, uint32_t x0, uint32_t x1, uint64_t* out4) {
  if (!ctx || !out4) return DVL_E_INVAL;
  if (!ctx->built || ctx->last_W != W || W == 0) {
    set_err(ctx, "no polylines of this width yet");
    return DVL_E_STATE;
  }
  if (x0 > x1 || x1 >= W) {
    set_err(ctx, "brush: need x0 <= x1 < W");
    return DVL_E_INVAL;
  }
  try {
    CK(cudaSetDevice(ctx->device));
    const Dataset& d = ctx->ds;
    unsigned long long r[4] = {0, 0, ~0ull, ~0ull};
    CK(cudaMemcpyAsync(&r[0], ctx->d_bin_lo + x0, 8, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(&r[1], ctx->d_bin_hi + x1, 8, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    // the codes of the first and the last brushed cell, from the shard that holds each
    for (int e = 0; e < 2; ++e) {
      const uint64_t c = r[e];
      if (c >= ctx->cell_offset && c < ctx->cell_offset + (uint64_t)d.n) {
        uint64_t k = 0;
        CK(cudaMemcpyAsync(&k, static_cast<const char*>(d.keys) + (c - ctx->cell_offset) * d.key_bytes,
                           d.key_bytes, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        r[2 + e] = k;
      }
    }
    if (ctx->comm && ctx->sharded) {   // collective: every shard learns both codes
      Small sm(ctx, 2);
      sm.put({r[2], r[3]});
      comm_ck(ctx, ctx->comm->allreduce(sm.d, 2, kU64, kMin, ctx->stream), "all_reduce MIN brush codes");
      const std::vector<uint64_t> v = sm.get(2);
      r[2] = v[0];
      r[3] = v[1];
    }
    for (int i = 0; i < 4; ++i) out4[i] = r[i];
  } catch (Fail& f) {
    return f.s;
  }
  return DVL_OK;
}

dvl_status dvl_get_bin_ranges(dvl_ctx* ctx, uint32_t W, uint64_t* lo, uint64_t* hi,
                              dvl_mem where) {
  if (!ctx) return DVL_E_INVAL;
  if (!ctx->built || ctx->last_W != W || W == 0) {
    set_err(ctx, "no polylines of this width yet");
    return DVL_E_STATE;
  }
  try {
    CK(cudaSetDevice(ctx->device));
    if (lo) CK(cudaMemcpyAsync(lo, ctx->d_bin_lo, 8 * (size_t)W, out_kind(where), ctx->stream));
    if (hi) CK(cudaMemcpyAsync(hi, ctx->d_bin_hi, 8 * (size_t)W, out_kind(where), ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  } catch (Fail& f) {
    return f.s;
  }
  return DVL_OK;
}

dvl_status dvl_set_timing(dvl_ctx* ctx, int enable) {
  if (!ctx) return DVL_E_INVAL;
  if (enable)
    ctx->flags |= DVL_FLAG_TIMING;
  else
    ctx->flags &= ~DVL_FLAG_TIMING;
  return DVL_OK;
}

dvl_status dvl_get_timings(dvl_ctx* ctx, dvl_timings* t) {
  if (!ctx || !t) return DVL_E_INVAL;
  memset(t, 0, sizeof *t);
  try {
    CK(cudaSetDevice(ctx->device));
    CK(cudaStreamSynchronize(ctx->stream));
    float* dst[PH_N] = {&t->ingest_ms, &t->encode_ms, &t->sort_ms, &t->gather_ms,
                        &t->maxv_ms, &t->weights_scan_ms, &t->bin_reduce_ms, &t->epilogue_ms,
                        &t->bin_boundary_ms};
    for (int i = 0; i < PH_N; ++i)
      if (ctx->ev_used[i]) CK(cudaEventElapsedTime(dst[i], ctx->ev[i][0], ctx->ev[i][1]));
    t->sort_passes = ctx->sort_passes;
    t->launches = ctx->launches;
    ctx->launches = 0;
  } catch (Fail& f) {
    return f.s;
  }
  return DVL_OK;
}

}  // extern "C"

#ifdef DVL_PROF
// timing experiments of the profiling build: pass-2 phase clock sums (see update_tma.cu);
// not part of dvl.h
extern "C" __attribute__((visibility("default"))) int dvl_debug_stats(unsigned long long* out) {
  return dvl::debug_stats(out, true) == cudaSuccess ? 0 : 1;
}
extern "C" __attribute__((visibility("default"))) int dvl_debug_bt(unsigned long long* out) {
  return dvl::debug_bt(out) == cudaSuccess ? 0 : 1;
}
extern "C" __attribute__((visibility("default"))) int dvl_debug_tl2(unsigned long long* out) {
  return dvl::debug_tl2(out) == cudaSuccess ? 0 : 1;
}
extern "C" __attribute__((visibility("default"))) int dvl_debug_aw(unsigned long long* out) {
  return dvl::debug_aw(out) == cudaSuccess ? 0 : 1;
}
extern "C" __attribute__((visibility("default"))) int dvl_debug_nored(int v) {
  return dvl::debug_nored(v) == cudaSuccess ? 0 : 1;
}
extern "C" __attribute__((visibility("default"))) int dvl_debug_p1(unsigned long long* out) {
  return dvl::debug_p1(out) == cudaSuccess ? 0 : 1;
}
#endif
