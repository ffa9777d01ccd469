// update.cu -- the TF-update path (U0-U5), every step a kernel on the context stream.
//
//   tf_prepare    canonical RGBA table + alpha slope table of one member
//   maxv_*        max(V_h) normaliser: R2 / R1 from TFs and data ranges on one
//                 block, or the exact max over cells
//   weights_scan  pass 1 (U1+U2): per cell, every member's TF alpha of its normalised
//                 scalar, V_h = max - min (Eq. 1), f = (max(V/maxV, eps) 2^L)^P (Eq. 3),
//                 q = trunc(f 2^s) in u64; per-tile sums chained by a decoupled look-back
//                 into exclusive tile prefixes and Qtot (Eq. 4 in exact fixed point)
//   bin_reduce    pass 2 (U3+U4): recompute q from the same scalars (design D2: q never
//                 goes to HBM), rebuild the exact Q(h) in registers from the tile prefix,
//                 bin each cell with integer thresholds T(x) = ceil(x Qtot / W) (P:226-229,
//                 reading O13) and reduce each pixel's contiguous cell range per member
//                 (P:229-233): min/max of t as ordered u32, sums as 2^-48 fixed point;
//                 tile/warp pre-reduction, integer atomics only per segment
//   epilogue      U5: count = hi - lo + 1, mean = sum / count, y = alpha(mean), rgb
//                 (P:250-256); resets the accumulators for the next call
#include <algorithm>
#include <cstring>

#include "dvl_common.cuh"
#include "dvl_internal.h"

namespace dvl {

// ------------------------------------------------------------------------- TF prepare
__global__ void tf_prepare_kernel(const float* __restrict__ in, int N, float4* __restrict__ rgba,
                                  float2* __restrict__ tab) {
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    // x + 0 turns -0 into +0 (canonical table)
    float4 e = make_float4(__fadd_rn(in[4 * i], 0.0f), __fadd_rn(in[4 * i + 1], 0.0f),
                           __fadd_rn(in[4 * i + 2], 0.0f), __fadd_rn(in[4 * i + 3], 0.0f));
    rgba[i] = e;
    float d = 0.0f;
    if (i + 1 < N) d = __fsub_rn(__fadd_rn(in[4 * i + 7], 0.0f), e.w);
    tab[i] = make_float2(e.w, d);
  }
}

void launch_tf_prepare(const float* rgba_in, int N, float4* rgba_out, float2* tab_out,
                       cudaStream_t st) {
  tf_prepare_kernel<<<1, 256, 0, st>>>(rgba_in, N, rgba_out, tab_out);
}

// --------------------------------------------------------------- maxV approximations
__global__ void maxv_approx_kernel(int mode, int M, int N, const float2* __restrict__ tab,
                                   const float* __restrict__ vmin, const float* __restrict__ vmax,
                                   const float* __restrict__ lo, const float* __restrict__ inv,
                                   float* maxv) {
  __shared__ int s_i, s_j;
  __shared__ uint32_t s_hi, s_lo, s_best;
  const int tid = threadIdx.x;
  if (tid == 0) {
    s_i = N - 1;
    s_j = 0;
    s_hi = 0;
    s_lo = 0xffffffffu;
    s_best = 0;
  }
  __syncthreads();
  const float nm1 = (float)(N - 1);
  for (int m = tid; m < M; m += blockDim.x) {
    float tl = norm_t(vmin[m], lo[m], inv[m]);
    float th = norm_t(vmax[m], lo[m], inv[m]);
    int i = (int)floorf(__fmul_rn(tl, nm1));
    int j = (int)ceilf(__fmul_rn(th, nm1));
    j = min(j, N - 1);
    atomicMin(&s_i, i);
    atomicMax(&s_j, j);
  }
  __syncthreads();
  const int i = s_i, j = s_j, w = j - i + 1;
  if (mode == 0) {
    uint32_t hi = 0, lo_ = 0xffffffffu;
    for (int k = tid; k < M * w; k += blockDim.x) {
      int m = k / w, a = i + k % w;
      uint32_t b = __float_as_uint(tab[m * N + a].x);   // alpha >= +0: bits order as values
      hi = max(hi, b);
      lo_ = min(lo_, b);
    }
    atomicMax(&s_hi, hi);
    atomicMin(&s_lo, lo_);
    __syncthreads();
    if (tid == 0) *maxv = __fsub_rn(__uint_as_float(s_hi), __uint_as_float(s_lo));
  } else {
    uint32_t best = 0;
    for (int a = i + tid; a <= j; a += blockDim.x) {
      float mx = tab[a].x, mn = mx;
      for (int m = 1; m < M; ++m) {
        float v = tab[m * N + a].x;
        mx = v > mx ? v : mx;
        mn = v < mn ? v : mn;
      }
      best = max(best, __float_as_uint(__fsub_rn(mx, mn)));
    }
    atomicMax(&s_best, best);
    __syncthreads();
    if (tid == 0) *maxv = __uint_as_float(s_best);
  }
}

void launch_maxv_approx(int mode, int M, int N, const float2* tab, const float* vmin,
                        const float* vmax, const float* lo, const float* inv, float* maxv,
                        cudaStream_t st) {
  maxv_approx_kernel<<<1, 256, 0, st>>>(mode, M, N, tab, vmin, vmax, lo, inv, maxv);
}

// Fused U0 prologue of one TF edit, one block: (member >= 0) install that member's TF
// straight from the caller-filled pinned staging buffer (mapped host memory: the 16 N
// bytes cross PCIe inside this kernel, no separate copy), zero the pass-1 look-back state,
// then (mode 0/1) max(V_h) as maxv_approx_kernel.
#ifdef DVL_PROF
// timeline of the prologue and epilogue (globaltimer ns, read by dvl_debug_tl2): slots
// 2k = ~(first start), 2k+1 = last end; k = 0 prologue, 1 epilogue, 2 epilogue after wait
__device__ unsigned long long g_tl2[8 + 1 + 64 * 4];   // + step counter, per step (64 ring):
// prologue start, prologue end, epilogue after wait (block 0), epilogue end
__device__ __forceinline__ unsigned long long gtime2() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TL2_START(k) \
  if (threadIdx.x == 0) atomicMax(&g_tl2[2 * (k)], ~gtime2());
#define TL2_END(k) \
  if (threadIdx.x == 0) atomicMax(&g_tl2[2 * (k) + 1], gtime2());
cudaError_t debug_tl2(unsigned long long* out) {
  cudaError_t e = cudaMemcpyFromSymbol(out, g_tl2, sizeof(g_tl2));
  static unsigned long long z[8 + 1 + 64 * 4];
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_tl2, z, sizeof(z));
  return e;
}
#else
#define TL2_START(k)
#define TL2_END(k)
cudaError_t debug_tl2(unsigned long long*) { return cudaErrorNotSupported; }
#endif

constexpr int kProloguAlpha = 12 * 1024;   // alphas the prologue stages in shared memory (48 KB)

__global__ void __launch_bounds__(1024)
tf_prologue_kernel(const float* __restrict__ stage, int member, int mode, int M, int N,
                   float4* __restrict__ rgba_all, float2* __restrict__ tab_all,
                   const float* __restrict__ vmin, const float* __restrict__ vmax,
                   const float* __restrict__ lo, const float* __restrict__ inv, float* maxv,
                   unsigned long long* zero, int zero_words) {
  // let pass 1 be scheduled now: its producer streams the scalars meanwhile, its consumers
  // wait for this kernel (griddepcontrol.wait)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  TL2_START(0)
#ifdef DVL_PROF
  unsigned step = 0;
  if (threadIdx.x == 0) {
    step = (unsigned)atomicAdd(&g_tl2[8], 1ull) & 63u;
    g_tl2[9 + 4 * step] = gtime2();
  }
#define TL2_STEP_END if (threadIdx.x == 0) g_tl2[9 + 4 * step + 1] = gtime2();
#else
#define TL2_STEP_END
#endif
  const int tid = threadIdx.x;
  // Every input is requested up front, so that the PCIe read of the staged TF, the domain
  // loads and (maxV from shared memory, s_alpha) the other members' alpha columns overlap.
  extern __shared__ float s_alpha[];   // M x N alphas when s_alpha_ok (the launch sized it)
  const bool s_alpha_ok = mode >= 0 && M * N <= kProloguAlpha;
  __shared__ int s_i, s_j;
  __shared__ uint32_t s_hi, s_lo;
  if (tid == 0) {
    s_i = N - 1;
    s_j = 0;
    s_hi = 0;
    s_lo = 0xffffffffu;
  }
  if (s_alpha_ok)
    for (int k = tid; k < M * N; k += blockDim.x)
      if (k / N != member) s_alpha[k] = tab_all[k].x;
  float tl = 0.0f, th = 0.0f;
  if (mode >= 0 && tid < M) {
    tl = norm_t(vmin[tid], lo[tid], inv[tid]);
    th = norm_t(vmax[tid], lo[tid], inv[tid]);
  }
  if (member >= 0) {
    float4* rgba = rgba_all + (int64_t)member * N;
    float2* tab = tab_all + (int64_t)member * N;
    for (int i = tid; i < N; i += blockDim.x) {
      const float4 r = reinterpret_cast<const float4*>(stage)[i];   // one 16-byte PCIe read
      const float4 e = make_float4(__fadd_rn(r.x, 0.0f), __fadd_rn(r.y, 0.0f),
                                   __fadd_rn(r.z, 0.0f), __fadd_rn(r.w, 0.0f));
      rgba[i] = e;
      float d = 0.0f;
      if (i + 1 < N) d = __fsub_rn(__fadd_rn(stage[4 * i + 7], 0.0f), e.w);
      tab[i] = make_float2(e.w, d);
      if (s_alpha_ok) s_alpha[member * N + i] = e.w;
    }
  }
  for (int k = tid; k < zero_words; k += blockDim.x) zero[k] = 0ull;
  if (mode < 0) {
    TL2_END(0)
    TL2_STEP_END
    return;
  }
  __syncthreads();   // the new table and the alphas are visible to the whole block
  const float nm1 = (float)(N - 1);
  if (tid < M) {
    int i = (int)floorf(__fmul_rn(tl, nm1));
    int j = (int)ceilf(__fmul_rn(th, nm1));
    j = min(j, N - 1);
    atomicMin(&s_i, i);
    atomicMax(&s_j, j);
  }
  __syncthreads();
  const int i = s_i, j = s_j, w = j - i + 1;
  auto alpha = [&](int m, int a) { return s_alpha_ok ? s_alpha[m * N + a] : tab_all[m * N + a].x; };
  uint32_t hi = 0, lo_ = 0xffffffffu;
  if (mode == 0) {
    for (int k = tid; k < M * w; k += blockDim.x) {
      int m = k / w, a = i + k % w;
      uint32_t b = __float_as_uint(alpha(m, a));   // alpha >= +0: bits order as values
      hi = max(hi, b);
      lo_ = min(lo_, b);
    }
  } else {
    for (int a = i + tid; a <= j; a += blockDim.x) {
      float mx = alpha(0, a), mn = mx;
      for (int m = 1; m < M; ++m) {
        float v = alpha(m, a);
        mx = v > mx ? v : mx;
        mn = v < mn ? v : mn;
      }
      hi = max(hi, __float_as_uint(__fsub_rn(mx, mn)));
    }
  }
  hi = __reduce_max_sync(0xffffffffu, hi);
  lo_ = __reduce_min_sync(0xffffffffu, lo_);
  if ((tid & 31) == 0) {
    atomicMax(&s_hi, hi);
    atomicMin(&s_lo, lo_);
  }
  __syncthreads();
  if (tid == 0)
    *maxv = mode == 0 ? __fsub_rn(__uint_as_float(s_hi), __uint_as_float(s_lo))
                      : __uint_as_float(s_hi);
  TL2_END(0)
  TL2_STEP_END
}

void launch_tf_prologue(const float* stage, int member, int mode, int M, int N, float4* rgba_all,
                        float2* tab_all, const float* vmin, const float* vmax, const float* lo,
                        const float* inv, float* maxv, unsigned long long* zero, int zero_words,
                        cudaStream_t st) {
  const size_t sm = mode >= 0 && M * N <= kProloguAlpha ? sizeof(float) * (size_t)M * N : 0;
  tf_prologue_kernel<<<1, 1024, sm, st>>>(stage, member, mode, M, N, rgba_all, tab_all, vmin, vmax,
                                          lo, inv, maxv, zero, zero_words);
}

// ------------------------------------------------------------ per-cell weights (U1)
// Alpha min/max over the members of ITEMS consecutive cells starting at c0, then q.
// With STAGE, the normalised t of every (member, cell) goes to shared memory s_t laid out
// [(m * ITEMS + i) * kBlock + tid] (conflict-free) for the reduction of pass 2.
template <int ITEMS, bool STAGE>
__device__ __forceinline__ void cell_alpha_range(const UpdParams& p, const float2* tab, int64_t c0,
                                                 float (&amax)[ITEMS], float (&amin)[ITEMS],
                                                 float* s_t, int tid) {
  const float nm1 = (float)(p.N - 1);
  for (int m = 0; m < p.M; ++m) {
    float v[ITEMS];
    load_f<ITEMS>(p.scal + (int64_t)m * p.n_pad + c0, v);
    const float lo = __ldg(p.lo + m), inv = __ldg(p.inv + m);
    const float2* tb = tab + m * p.N;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      float t = norm_t(v[i], lo, inv);
      if (STAGE) s_t[(m * ITEMS + i) * kBlock + tid] = t;
      float a = sample_tab(tb, nm1, t);
      if (m == 0) {
        amax[i] = a;
        amin[i] = a;
      } else {
        amax[i] = a > amax[i] ? a : amax[i];
        amin[i] = a < amin[i] ? a : amin[i];
      }
    }
  }
}

template <int ITEMS, bool STAGE>
__device__ __forceinline__ void cell_weights(const UpdParams& p, const float2* tab, int64_t c0,
                                             float maxv, unsigned long long (&q)[ITEMS],
                                             float* s_t, int tid) {
  float amax[ITEMS], amin[ITEMS];
  cell_alpha_range<ITEMS, STAGE>(p, tab, c0, amax, amin, s_t, tid);
  int L[ITEMS];
  load_u8<ITEMS>(p.level + c0, L);
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    float V = __fsub_rn(amax[i], amin[i]);
    float f = importance(V, maxv, L[i] * p.lscale, p.eps, p.pw);
    q[i] = (c0 + i < p.n) ? __float2ull_rz(__fmul_rn(f, p.scale)) : 0ull;
  }
}

__device__ __forceinline__ const float2* stage_tab(const UpdParams& p, float2* s_tab, bool smem) {
  if (!smem) return p.tab;
  const int total = p.M * p.N;
  for (int k = threadIdx.x; k < total; k += kBlock) s_tab[k] = p.tab[k];
  return s_tab;
}

// exact max(V_h) over all cells (mode EXACT); *maxv must be 0 before the launch
template <int ITEMS>
__global__ void __launch_bounds__(kBlock) maxv_exact_kernel(UpdParams p, float* maxv) {
  const int64_t c0 = ((int64_t)blockIdx.x * kBlock + threadIdx.x) * ITEMS;
  if (c0 >= p.n_pad) return;
  float amax[ITEMS], amin[ITEMS];
  cell_alpha_range<ITEMS, false>(p, p.tab, c0, amax, amin, nullptr, threadIdx.x);
  uint32_t best = 0;
#pragma unroll
  for (int i = 0; i < ITEMS; ++i)
    if (c0 + i < p.n) best = max(best, __float_as_uint(__fsub_rn(amax[i], amin[i])));
  best = __reduce_max_sync(0xffffffffu, best);
  if ((threadIdx.x & 31) == 0 && best) atomicMax(reinterpret_cast<uint32_t*>(maxv), best);
}

void launch_maxv_exact(const UpdParams& p, float* maxv, int grid, cudaStream_t st) {
  cudaMemsetAsync(maxv, 0, sizeof(float), st);
  int64_t per = p.n_pad / ((int64_t)grid * kBlock);
  switch (per) {
    case 16: maxv_exact_kernel<16><<<grid, kBlock, 0, st>>>(p, maxv); break;
    case 8: maxv_exact_kernel<8><<<grid, kBlock, 0, st>>>(p, maxv); break;
    case 4: maxv_exact_kernel<4><<<grid, kBlock, 0, st>>>(p, maxv); break;
    case 2: maxv_exact_kernel<2><<<grid, kBlock, 0, st>>>(p, maxv); break;
    default: maxv_exact_kernel<1><<<grid, kBlock, 0, st>>>(p, maxv); break;
  }
}

// --------------------------------------------------------------- pass 1: weights + scan
template <int ITEMS, bool SMEM_TAB, bool EXPORT_Q>
__global__ void __launch_bounds__(kBlock)
weights_scan_kernel(UpdParams p, unsigned long long* status, uint32_t* ctr,
                    unsigned long long* tile_prefix, unsigned long long* qtot,
                    unsigned long long* q_out) {
  extern __shared__ __align__(16) unsigned char smem[];
  float2* s_tab = reinterpret_cast<float2*>(smem);
  __shared__ unsigned long long s_warp[kBlock / 32];
  __shared__ unsigned long long s_excl;
  __shared__ int64_t s_tile;
  constexpr int T = kBlock * ITEMS;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(ctr, 1u);
  const float2* tab = stage_tab(p, s_tab, SMEM_TAB);
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t c0 = tile * T + (int64_t)tid * ITEMS;
  const float maxv = *p.maxv;

  unsigned long long q[ITEMS];
  cell_weights<ITEMS, false>(p, tab, c0, maxv, q, nullptr, tid);
  unsigned long long tsum = 0;
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) tsum += q[i];
  unsigned long long wincl = warp_incl_scan_u64(tsum, lane);
  if (lane == 31) s_warp[warp] = wincl;
  __syncthreads();
  if (warp == 0) {
    unsigned long long total = warp_sum_u64(lane < kBlock / 32 ? s_warp[lane] : 0ull);
    if (lane == 0)
      atomicExch(status + tile, (tile == 0 ? kScanInc : kScanAgg) | total);
    unsigned long long excl = 0;
    if (tile > 0) {
      int64_t base = tile - 1;
      while (true) {
        int64_t j = base - lane;
        unsigned long long s = kScanInc;
        if (j >= 0) {
          volatile unsigned long long* sp = status + j;
          do {
            s = *sp;
          } while ((s >> 62) == 0);
        }
        uint32_t incm = __ballot_sync(0xffffffffu, (s >> 62) == 2);
        int first = incm ? __ffs(incm) - 1 : 32;
        excl += warp_sum_u64(lane <= first ? (s & kScanMask) : 0ull);
        if (incm) break;
        base -= 32;
      }
      if (lane == 0) atomicExch(status + tile, kScanInc | (excl + total));
    }
    if (lane == 0) {
      tile_prefix[tile] = excl;
      if ((tile + 1) * T >= p.n) *qtot = excl + total;
      s_excl = excl;
    }
  }
  if (EXPORT_Q) {
    __syncthreads();
    unsigned long long wpre = 0;
    for (int w = 0; w < warp; ++w) wpre += s_warp[w];
    unsigned long long run = p.offset + s_excl + wpre + wincl - tsum;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      run += q[i];
      if (c0 + i < p.n) q_out[c0 + i] = run;
    }
  }
}

// ---------------------------------------------------------- pass 2: bins + reduction
__device__ __forceinline__ void flush_member(const Acc& acc, uint32_t W, int m, int x, uint32_t mn,
                                             uint32_t mx, float sum) {
  const int64_t k = (int64_t)m * W + x;
  atomicMin(acc.tmin + k, mn);
  atomicMax(acc.tmax + k, mx);
  red_add_sum(acc.slo + k, acc.shi + k, __float2ull_rn(__fmul_rn(sum, kSumScale)));
}

__device__ __forceinline__ void flush_range(const Acc& acc, int x, unsigned long long first,
                                            unsigned long long last) {
  atomicMin(acc.lo + x, first);
  atomicMax(acc.hi + x, last);
}

template <int ITEMS, bool SMEM_TAB>
__global__ void __launch_bounds__(kBlock)
bin_reduce_kernel(UpdParams p, const unsigned long long* __restrict__ tile_prefix,
                  const unsigned long long* __restrict__ qtot_p, uint32_t W, Acc acc,
                  uint64_t cell_offset, uint32_t* err) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int T = kBlock * ITEMS;
  float2* s_tab = reinterpret_cast<float2*>(smem);
  float* s_t = reinterpret_cast<float*>(smem + (SMEM_TAB ? sizeof(float2) * p.M * p.N : 0));
  __shared__ unsigned long long s_warp[kBlock / 32];
  __shared__ uint32_t s_rmin[kBlock / 32][kMaxM];
  __shared__ uint32_t s_rmax[kBlock / 32][kMaxM];
  __shared__ unsigned long long s_rsum[kBlock / 32][kMaxM];
  __shared__ int s_b1first;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t tile = blockIdx.x;
  const int64_t c0 = tile * T + (int64_t)tid * ITEMS;
  const float2* tab = stage_tab(p, s_tab, SMEM_TAB);
  __syncthreads();
  const unsigned long long Qtot = *qtot_p;
  if (Qtot == 0) {
    if (tid == 0 && tile == 0) atomicOr(err, kErrDegenerate);
    return;
  }
  const float maxv = *p.maxv;
  unsigned long long q[ITEMS];
  cell_weights<ITEMS, true>(p, tab, c0, maxv, q, s_t, tid);

  // exact inclusive prefix Q(h) of this thread's cells
  unsigned long long tsum = 0;
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) tsum += q[i];
  unsigned long long wincl = warp_incl_scan_u64(tsum, lane);
  if (lane == 31) s_warp[warp] = wincl;
  __syncthreads();
  unsigned long long wpre = 0;
  for (int w = 0; w < warp; ++w) wpre += s_warp[w];
  const unsigned long long base =
      p.offset + (p.offset_dev ? *p.offset_dev : 0ull) + tile_prefix[tile] + wpre + wincl - tsum;

  // bins: b1 = min(W-1, max{x : ceil(x Qtot/W) <= E}), b2 = min(W-1, max(b1, max{x <= W-1 :
  // floor(x Qtot/W) < Q})).  T(x) = x a + ceil(x r / W), T'(x) = x a + floor(x r / W).
  const unsigned long long qa = Qtot / W, qr = Qtot % W;
  auto Tc = [&](int x) -> unsigned long long {
    unsigned long long xr = (unsigned long long)x * qr;
    return (unsigned long long)x * qa + (xr + W - 1) / W;
  };
  auto Tf = [&](int x) -> unsigned long long {
    unsigned long long xr = (unsigned long long)x * qr;
    return (unsigned long long)x * qa + xr / W;
  };
  int b1[ITEMS], b2[ITEMS];
  {
    const unsigned long long E0 = base, Q0 = base + q[0];
    double inv = (double)W / (double)Qtot;
    int x1 = (int)fmin((double)W, floor((double)E0 * inv));
    x1 = max(x1, 0);
    while (x1 > 0 && Tc(x1) > E0) --x1;
    while (x1 < (int)W && Tc(x1 + 1) <= E0) ++x1;
    int x2 = (int)fmin((double)W - 1.0, ceil((double)Q0 * inv) - 1.0);
    x2 = max(x2, -1);
    while (x2 >= 0 && Tf(x2) >= Q0) --x2;
    while (x2 < (int)W - 1 && Tf(x2 + 1) < Q0) ++x2;
    unsigned long long n1 = x1 < (int)W ? Tc(x1 + 1) : ~0ull;
    unsigned long long n2 = x2 < (int)W - 1 ? Tf(x2 + 1) : ~0ull;
    unsigned long long E = E0;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      unsigned long long Q = E + q[i];
      while (E >= n1) {
        ++x1;
        n1 = x1 < (int)W ? Tc(x1 + 1) : ~0ull;
      }
      while (Q > n2) {
        ++x2;
        n2 = x2 < (int)W - 1 ? Tf(x2 + 1) : ~0ull;
      }
      b1[i] = min(x1, (int)W - 1);
      b2[i] = max(b1[i], x2);
      E = Q;
    }
  }
  bool valid[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) valid[i] = c0 + i < p.n;

  // tile-uniform fast path: every cell of the tile falls into one bin
  if (tid == 0) s_b1first = b1[0];
  __syncthreads();
  const int xt = s_b1first;
  bool mine = true;
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) mine = mine && (!valid[i] || (b1[i] == xt && b2[i] == xt));
  const bool tile_uniform = __syncthreads_and(mine);
  const unsigned long long g0 = cell_offset + (unsigned long long)c0;  // global index of cell 0

  if (tile_uniform) {
    for (int m = 0; m < p.M; ++m) {
      uint32_t mn = 0xffffffffu, mx = 0u;
      float s = 0.0f;
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) {
        if (valid[i]) {
          float t = s_t[(m * ITEMS + i) * kBlock + tid];
          uint32_t bits = __float_as_uint(t);
          mn = min(mn, bits);
          mx = max(mx, bits);
          s = __fadd_rn(s, t);
        }
      }
      unsigned long long fx = __float2ull_rn(__fmul_rn(s, kSumScale));
      mn = __reduce_min_sync(0xffffffffu, mn);
      mx = __reduce_max_sync(0xffffffffu, mx);
      fx = warp_sum_u64(fx);
      if (lane == 0) {
        s_rmin[warp][m] = mn;
        s_rmax[warp][m] = mx;
        s_rsum[warp][m] = fx;
      }
    }
    __syncthreads();
    for (int m = tid; m < p.M; m += kBlock) {
      uint32_t mn = 0xffffffffu, mx = 0u;
      unsigned long long fx = 0;
      for (int w = 0; w < kBlock / 32; ++w) {
        mn = min(mn, s_rmin[w][m]);
        mx = max(mx, s_rmax[w][m]);
        fx += s_rsum[w][m];
      }
      const int64_t k = (int64_t)m * W + xt;
      atomicMin(acc.tmin + k, mn);
      atomicMax(acc.tmax + k, mx);
      red_add_sum(acc.slo + k, acc.shi + k, fx);
    }
    if (tid == 0) {
      const unsigned long long first = cell_offset + (unsigned long long)(tile * T);
      const unsigned long long last =
          cell_offset + (unsigned long long)(min((int64_t)(tile + 1) * T, p.n) - 1);
      flush_range(acc, xt, first, last);
    }
    return;
  }

  // general path.  Warp-uniform sub-case first.
  const int xw = __shfl_sync(0xffffffffu, b1[0], 0);
  bool wmine = true;
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) wmine = wmine && (!valid[i] || (b1[i] == xw && b2[i] == xw));
  const bool any_valid = valid[0];
  if (__all_sync(0xffffffffu, wmine)) {
    for (int m = 0; m < p.M; ++m) {
      uint32_t mn = 0xffffffffu, mx = 0u;
      float s = 0.0f;
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) {
        if (valid[i]) {
          float t = s_t[(m * ITEMS + i) * kBlock + tid];
          uint32_t bits = __float_as_uint(t);
          mn = min(mn, bits);
          mx = max(mx, bits);
          s = __fadd_rn(s, t);
        }
      }
      unsigned long long fx = __float2ull_rn(__fmul_rn(s, kSumScale));
      mn = __reduce_min_sync(0xffffffffu, mn);
      mx = __reduce_max_sync(0xffffffffu, mx);
      fx = warp_sum_u64(fx);
      if (lane == 0 && mx != 0u | mn != 0xffffffffu) {
        const int64_t k = (int64_t)m * W + xw;
        atomicMin(acc.tmin + k, mn);
        atomicMax(acc.tmax + k, mx);
        red_add_sum(acc.slo + k, acc.shi + k, fx);
      }
    }
    // cell range of the warp: first valid cell of lane 0, last valid cell of the warp
    unsigned long long lastc = 0;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i)
      if (valid[i]) lastc = g0 + i;
    unsigned long long wl = lastc;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      unsigned long long u = __shfl_xor_sync(0xffffffffu, wl, o);
      wl = u > wl ? u : wl;
    }
    if (lane == 0 && any_valid) flush_range(acc, xw, g0, wl);
    return;
  }

  // per-thread runs of equal b1 (head segments) + spanned interior/tail bins
  {
    int run_x = -1;
    unsigned long long run_first = 0, run_last = 0;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      if (!valid[i]) continue;
      if (b1[i] != run_x) {
        if (run_x >= 0) flush_range(acc, run_x, run_first, run_last);
        run_x = b1[i];
        run_first = g0 + i;
      }
      run_last = g0 + i;
      for (int x = b1[i] + 1; x <= b2[i]; ++x) flush_range(acc, x, g0 + i, g0 + i);
    }
    if (run_x >= 0) flush_range(acc, run_x, run_first, run_last);
  }
  for (int m = 0; m < p.M; ++m) {
    int run_x = -1;
    uint32_t mn = 0xffffffffu, mx = 0u;
    float s = 0.0f;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      if (!valid[i]) continue;
      float t = s_t[(m * ITEMS + i) * kBlock + tid];
      uint32_t bits = __float_as_uint(t);
      if (b1[i] != run_x) {
        if (run_x >= 0) flush_member(acc, W, m, run_x, mn, mx, s);
        run_x = b1[i];
        mn = 0xffffffffu;
        mx = 0u;
        s = 0.0f;
      }
      mn = min(mn, bits);
      mx = max(mx, bits);
      s = __fadd_rn(s, t);
      for (int x = b1[i] + 1; x <= b2[i]; ++x) flush_member(acc, W, m, x, bits, bits, t);
    }
    if (run_x >= 0) flush_member(acc, W, m, run_x, mn, mx, s);
  }
}

// ------------------------------------------------------------------------- epilogue
// One thread per (member m, pixel x), x fastest (coalesced): reads the pixel's cell range
// (current copy), m = 0 writes the bin ranges and restores the identity of the other copy;
// every thread restores the identity of its member partials.
__global__ void __launch_bounds__(256)
epilogue_kernel(Acc acc, WDiv wd, int M, int N, const float4* __restrict__ rgba,
                dvl_vertex* __restrict__ out, unsigned long long* bin_lo,
                unsigned long long* bin_hi, bool stage_tf, const uint32_t* err,
                volatile uint32_t* err_host) {
  const uint32_t W = wd.d;   // M W <= 2^20: 32-bit entry indices, divisions by W via WDiv
  extern __shared__ float4 s_tf[];
  TL2_START(1)
  // the TF rows of the block's members into shared memory before the wait (pass 2 lets this
  // kernel start only once pass 1 -- and so the prologue that wrote them -- is complete)
  const uint32_t k0 = blockIdx.x * blockDim.x;
  const int m0 = (int)wd.div(k0);
  if (stage_tf) {
    const int m1 = min(M - 1, (int)wd.div(k0 + blockDim.x - 1));
    const int cnt = (m1 - m0 + 1) * N;
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) s_tf[i] = rgba[(int64_t)m0 * N + i];
    __syncthreads();
  }
  const uint32_t k = k0 + threadIdx.x;
  const int m = min((int)wd.div(k), M - 1);
  const uint32_t x = k - (uint32_t)m * W;
  const float4* tf = stage_tf ? s_tf + (m - m0) * N : rgba + (int64_t)m * N;
  // The vertex code runs twice: first on a dummy entry before the wait, so that its
  // instructions are in the SM's instruction cache when the real entry comes (this kernel
  // is short and runs once per edit: cold instruction fetches were most of its time).
  dvl_vertex vtx;
  uint32_t cnt = 1, mn = 0, mx = 0;
  unsigned long long sl = 0, sh = 0;
#pragma unroll 1
  for (int pass = 0; pass < 2; ++pass) {
    if (pass == 1) {
      asm volatile("griddepcontrol.wait;" ::: "memory");   // launched dependent on pass 2
      TL2_START(2)
      TL2_END(2)
      // the error word of this edit to the host's mapped staging (no separate copy)
      if (err_host && k == 0) *err_host = *(volatile const uint32_t*)err;
      if (k >= (uint32_t)M * W) return;
      const unsigned long long lo = acc.lo[x], hi = acc.hi[x];
      if (m == 0) {
        bin_lo[x] = lo;
        bin_hi[x] = hi;
        acc.lo2[x] = ~0ull;
        acc.hi2[x] = 0ull;
      }
      cnt = lo <= hi ? (uint32_t)(hi - lo + 1) : 0u;
      mn = acc.tmin[k];
      mx = acc.tmax[k];
      sum_words(acc.slo[k], acc.shi[k], sh, sl);
      acc.tmin[k] = 0xffffffffu;
      acc.tmax[k] = 0u;
      acc.slo[k] = 0ull;
      acc.shi[k] = 0ull;
    }
    vtx = make_vertex(cnt, mn, mx, sh, sl, tf, N);
  }
#ifdef DVL_PROF
  const unsigned step = (unsigned)(*(volatile unsigned long long*)&g_tl2[8] - 1) & 63u;
#endif
  // two 16-byte stores (the output may be mapped host memory: whole lines over PCIe)
  float4* o = reinterpret_cast<float4*>(out + k);
  o[0] = make_float4(vtx.t_min, vtx.t_max, vtx.t_mean, vtx.y);
  o[1] = make_float4(vtx.r, vtx.g, vtx.b, __uint_as_float(vtx.count));
  TL2_END(1)
#ifdef DVL_PROF
  if (threadIdx.x == 0) atomicMax(&g_tl2[9 + 4 * step + 3], gtime2());
#endif
}

__global__ void acc_init_kernel(Acc acc, uint32_t W, int M) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < (int64_t)W * M;
       k += (int64_t)gridDim.x * blockDim.x) {
    if (k < W) {
      acc.lo[k] = ~0ull;
      acc.hi[k] = 0ull;
      acc.lo2[k] = ~0ull;
      acc.hi2[k] = 0ull;
    }
    acc.tmin[k] = 0xffffffffu;
    acc.tmax[k] = 0u;
    acc.slo[k] = 0ull;
    acc.shi[k] = 0ull;
  }
}

void launch_epilogue(const Acc& acc, uint32_t W, int M, int N, const float4* rgba,
                     dvl_vertex* out, unsigned long long* bin_lo, unsigned long long* bin_hi,
                     const uint32_t* err, uint32_t* err_host, cudaStream_t st) {
  const int grid = (int)(((int64_t)M * W + 255) / 256);
  // members a block of 256 entries spans, and their TF rows in shared memory if they fit
  const int64_t rows = std::min<int64_t>(M, (255 + W - 1) / W + 1);
  const size_t tf_bytes = (size_t)rows * N * sizeof(float4);
  const bool stage_tf = tf_bytes <= 32 * 1024;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = stage_tf ? tf_bytes : 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  (void)cudaLaunchKernelEx(&cfg, epilogue_kernel, acc, WDiv::make(W), M, N, rgba, out, bin_lo, bin_hi,
                           stage_tf, err, (volatile uint32_t*)err_host);
}

void launch_acc_init(const Acc& acc, uint32_t W, int M, cudaStream_t st) {
  int64_t tot = (int64_t)W * M;
  int grid = (int)std::min<int64_t>((tot + 255) / 256, 4096);
  acc_init_kernel<<<grid, 256, 0, st>>>(acc, W, M);
}

// --------------------------------------------------------------------- dispatch
size_t bin_reduce_smem(int items, int M, int N, bool smem_tab) {
  return (smem_tab ? sizeof(float2) * (size_t)M * N : 0) + sizeof(float) * (size_t)M * kBlock * items;
}

template <int ITEMS>
static cudaError_t prep_items() {
  cudaError_t e;
  const int big = 200 * 1024;
  if ((e = cudaFuncSetAttribute(weights_scan_kernel<ITEMS, true, false>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, big)) != cudaSuccess)
    return e;
  if ((e = cudaFuncSetAttribute(weights_scan_kernel<ITEMS, true, true>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, big)) != cudaSuccess)
    return e;
  if ((e = cudaFuncSetAttribute(bin_reduce_kernel<ITEMS, true>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, big)) != cudaSuccess)
    return e;
  return cudaFuncSetAttribute(bin_reduce_kernel<ITEMS, false>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize, big);
}

cudaError_t prepare_update_kernels() {
  cudaError_t e;
  if ((e = prep_items<16>()) != cudaSuccess) return e;
  if ((e = prep_items<8>()) != cudaSuccess) return e;
  if ((e = prep_items<4>()) != cudaSuccess) return e;
  if ((e = prep_items<2>()) != cudaSuccess) return e;
  return prep_items<1>();
}

template <int ITEMS>
static void ws_dispatch(bool smem_tab, bool export_q, const UpdParams& p,
                        unsigned long long* status, uint32_t* ctr, unsigned long long* tp,
                        unsigned long long* qtot, unsigned long long* q_out, int tiles,
                        cudaStream_t st) {
  size_t sm = smem_tab ? sizeof(float2) * (size_t)p.M * p.N : 0;
  if (smem_tab) {
    if (export_q)
      weights_scan_kernel<ITEMS, true, true><<<tiles, kBlock, sm, st>>>(p, status, ctr, tp, qtot, q_out);
    else
      weights_scan_kernel<ITEMS, true, false><<<tiles, kBlock, sm, st>>>(p, status, ctr, tp, qtot, q_out);
  } else {
    if (export_q)
      weights_scan_kernel<ITEMS, false, true><<<tiles, kBlock, 0, st>>>(p, status, ctr, tp, qtot, q_out);
    else
      weights_scan_kernel<ITEMS, false, false><<<tiles, kBlock, 0, st>>>(p, status, ctr, tp, qtot, q_out);
  }
}

void launch_weights_scan(int items, bool smem_tab, bool export_q, const UpdParams& p,
                         unsigned long long* status, uint32_t* ctr,
                         unsigned long long* tile_prefix, unsigned long long* qtot,
                         unsigned long long* q_out, int tiles, cudaStream_t st) {
  switch (items) {
    case 16: ws_dispatch<16>(smem_tab, export_q, p, status, ctr, tile_prefix, qtot, q_out, tiles, st); break;
    case 8: ws_dispatch<8>(smem_tab, export_q, p, status, ctr, tile_prefix, qtot, q_out, tiles, st); break;
    case 4: ws_dispatch<4>(smem_tab, export_q, p, status, ctr, tile_prefix, qtot, q_out, tiles, st); break;
    case 2: ws_dispatch<2>(smem_tab, export_q, p, status, ctr, tile_prefix, qtot, q_out, tiles, st); break;
    default: ws_dispatch<1>(smem_tab, export_q, p, status, ctr, tile_prefix, qtot, q_out, tiles, st); break;
  }
}

template <int ITEMS>
static void br_dispatch(bool smem_tab, const UpdParams& p, const unsigned long long* tp,
                        const unsigned long long* qtot, uint32_t W, const Acc& acc,
                        uint64_t cell_offset, uint32_t* err, int tiles, cudaStream_t st) {
  size_t sm = bin_reduce_smem(ITEMS, p.M, p.N, smem_tab);
  if (smem_tab)
    bin_reduce_kernel<ITEMS, true><<<tiles, kBlock, sm, st>>>(p, tp, qtot, W, acc, cell_offset, err);
  else
    bin_reduce_kernel<ITEMS, false><<<tiles, kBlock, sm, st>>>(p, tp, qtot, W, acc, cell_offset, err);
}

void launch_bin_reduce(int items, bool smem_tab, const UpdParams& p,
                       const unsigned long long* tile_prefix, const unsigned long long* qtot,
                       uint32_t W, const Acc& acc, uint64_t cell_offset, uint32_t* err, int tiles,
                       cudaStream_t st) {
  switch (items) {
    case 16: br_dispatch<16>(smem_tab, p, tile_prefix, qtot, W, acc, cell_offset, err, tiles, st); break;
    case 8: br_dispatch<8>(smem_tab, p, tile_prefix, qtot, W, acc, cell_offset, err, tiles, st); break;
    case 4: br_dispatch<4>(smem_tab, p, tile_prefix, qtot, W, acc, cell_offset, err, tiles, st); break;
    case 2: br_dispatch<2>(smem_tab, p, tile_prefix, qtot, W, acc, cell_offset, err, tiles, st); break;
    default: br_dispatch<1>(smem_tab, p, tile_prefix, qtot, W, acc, cell_offset, err, tiles, st); break;
  }
}

}  // namespace dvl
