// dvl_common.cuh -- shared definitions of the sm_100a DVL library (product side).
//
// Nothing in this directory is shared with oracle/: the fp32 recipes below are written
// from DESIGN.md section 3 (readings O6-O11), with explicit round-to-nearest intrinsics
// so that no contraction or fast-math can change a bit (the library is also compiled
// with -fmad=false -ftz=false -prec-div=true).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "dvl.h"

namespace dvl {

constexpr int kBlock = 256;            // threads of every streaming kernel
constexpr int kSortItems = 16;         // keys per thread in the onesweep passes
constexpr int kSortTile = kBlock * kSortItems;
constexpr int kMaxN = 4096;            // largest TF
constexpr int kMaxM = 64;              // largest ensemble
constexpr uint32_t kMaxW = 65536;      // largest plot width

// status words of the weight scan's decoupled look-back (u64: 2 flag bits + 62 value bits)
constexpr uint64_t kScanAgg = 1ull << 62;
constexpr uint64_t kScanInc = 2ull << 62;
constexpr uint64_t kScanMask = (1ull << 62) - 1;
// status words of the onesweep digit look-back (u32: 2 flag bits + 30 count bits)
constexpr uint32_t kSortAgg = 1u << 30;
constexpr uint32_t kSortInc = 2u << 30;
constexpr uint32_t kSortMask = (1u << 30) - 1;

// fixed point of per-thread partial t sums: round(sum * 2^40) as u64 (a thread's running
// total over <= 2^22 cells stays < 2^63; global totals are 128-bit)
constexpr float kSumScale = 1099511627776.0f;     // 2^40
constexpr double kSumUnscale = 1.0 / 1099511627776.0;

// error bits written by kernels
constexpr uint32_t kErrInval = 1u;      // L > 20 or lower not a multiple of 2^L
constexpr uint32_t kErrOverlap = 2u;    // codes not strictly increasing / dyadic overlap
constexpr uint32_t kErrDegenerate = 4u; // Qtot == 0

// exponent classes of Eq. 3's ^P (reading O10)
enum PowKind : int { kPow0 = 0, kPow1 = 1, kPowInt = 2, kPowDet = 3 };

struct PowParams {
  int kind;
  int k;       // integer exponent for kPowInt
  float P;     // exponent for kPowDet
};

// Inputs of the two update passes.
struct UpdParams {
  int64_t n;               // cells on this device
  int64_t n_pad;           // member stride of scal (multiple of the tile)
  int M, N;
  const uint8_t* level;    // n_pad, curve order
  const float* scal;       // M x n_pad, curve order
  const float* lo;         // M domain lower bounds
  const float* inv;        // M inverse domain widths
  const float2* tab;       // M x N (alpha[i], alpha[i+1]-alpha[i])
  const float* maxv;       // device scalar
  float eps;
  PowParams pw;
  float scale;             // 2^s
  int shift;               // s
  int lscale;              // 1: f scales by the cell width 2^L (Eq. 3); 3: by its volume 2^3L
  uint64_t offset;         // global prefix before this device's cells (sharding, host part)
  const unsigned long long* offset_dev;   // ... and its device part (nullptr: 0)
  // sharded pass 2 (TMA path): the gathered Q totals of all shards; the scan offset of this
  // shard and the global Qtot are summed from them inside the kernel (nullptr: not sharded)
  const unsigned long long* shard_totals;
  int nshards, shard;
  uint32_t prod_sleep;     // producer's suspend-time hint (ns) while waiting for a free stage
  int pass2_mode;          // 0 auto, 1 boundary tiles inline, 2 listed, 3 jobs (DVL_FLAG_PASS2_*)
  int dbg;                 // DVL_PROF builds only (DVL_DBG): 4 = kernel timeline / phase probes
  // edit cache (repeated TF edits of one member): per cell the min / max of the alpha bits
  // of the members other than cmember (identity 0xffffffff / 0 when there are none)
  uint32_t* cmin;
  uint32_t* cmax;
  int cmember;
};

// Work split of the TMA-pipelined update kernels (host-computed).
struct TmaPlan {
  // pass 2: tiles of 1024 cells (8 warps x 128), 3 / 2 / 1 CTAs per SM for M <= 4 / 8 / 16
  int tiles;              // tiles of pass 2
  int tpc;                // pass 2: tiles per chunk (one chunk per CTA)
  int stages;             // pass 2: shared-memory ring depth
  uint32_t stage_bytes;   // pass 2: M * T * 4 + T + its 8 warp sums, rounded up to 128
  // pass 1: one CTA per SM, tiles of CW * 128 cells
  int tiles1;
  int tpc1;
  int stages1;
  uint32_t stage_bytes1;  // M * T1 * 4 + T1, rounded up to 128
  uint32_t tab_bytes;     // pass 1: alpha table in shared memory (0: read through L1)
};

// Division by the pixel count W of one get_polylines call (2 <= W <= 2^16) with a
// multiply-high and shifts (Granlund and Montgomery, "Division by invariant integers using
// multiplication", PLDI 1994, Fig. 4.1): exact for every 32-bit numerator.  Built on the host.
struct WDiv {
  uint32_t d, m, s;   // divisor, magic, l - 1 with l = ceil(log2 d) >= 1
  static WDiv make(uint32_t d) {
    uint32_t l = 0;
    while ((1ull << l) < d) ++l;
    WDiv w;
    w.d = d;
    w.s = l - 1;
    w.m = (uint32_t)(((1ull << 32) * ((1ull << l) - d)) / d + 1);
    return w;
  }
  __host__ __device__ __forceinline__ uint32_t div(uint32_t n) const {
#ifdef __CUDA_ARCH__
    const uint32_t t = __umulhi(m, n);
#else
    const uint32_t t = (uint32_t)(((unsigned long long)m * n) >> 32);
#endif
    return (t + ((n - t) >> 1)) >> s;
  }
};

// Per-bin accumulators of U4 (integer-exact, combined with atomics in any order).
struct Acc {
  unsigned long long* lo;    // W: first cell (min)
  unsigned long long* hi;    // W: last cell (max)
  uint32_t* tmin;            // M x W: min of t bits (t >= 0, so bits order like values)
  uint32_t* tmax;            // M x W
  unsigned long long* slo;   // M x W: sum of the low 32-bit halves of the 2^-40 fixed-point adds
  unsigned long long* shi;   // M x W: sum of the high halves (sum = slo + shi * 2^32, red_add_sum)
  // the other copy of lo / hi: get_polylines alternates between the two, and its epilogue
  // restores the identity of the copy the previous call used (the current copy is read by
  // the M threads of each pixel, so it cannot be reset in the same kernel)
  unsigned long long* lo2;
  unsigned long long* hi2;
};

// ------------------------------------------------------------------ fp32 recipes
// 2^k as fp32, exact for -149 <= k <= 127.
__host__ __device__ inline float pow2f(int k) {
  uint32_t u = k >= -126 ? (uint32_t)(k + 127) << 23 : 1u << (k + 149);
  float f;
#ifdef __CUDA_ARCH__
  f = __uint_as_float(u);
#else
  __builtin_memcpy(&f, &u, 4);
#endif
  return f;
}

// O7: t = clamp((v - lo) * inv, 0, 1), NaN -> 0.
__device__ __forceinline__ float norm_t(float v, float lo, float inv) {
  float x = __fmul_rn(__fsub_rn(v, lo), inv);
  return x > 0.0f ? (x < 1.0f ? x : 1.0f) : 0.0f;
}

// O7 in two instructions: mul.rn.sat rounds the product, then clamps it to [0, 1] with
// NaN -> +0 (the same value as norm_t; -0 -> +0 is checked by the parity tests).
__device__ __forceinline__ float norm_sat(float v, float lo, float inv) {
  float d = __fsub_rn(v, lo), t;
  asm("mul.rn.sat.f32 %0, %1, %2;" : "=f"(t) : "f"(d), "f"(inv));
  return t;
}

// O8 on a shared-memory slope table: `base` is the shared address of tab[0] minus
// 8 * 0x4B000000 (mod 2^32), so the address of tab[floor(pos)] is base + 8 * bits(pos +
// 2^23 rounded toward zero).
__device__ __forceinline__ float sample_smem(uint32_t base, float nm1, float t) {
  float pos = __fmul_rn(t, nm1);
  float f = __fadd_rz(pos, 8388608.0f);
  uint32_t addr = base + (__float_as_uint(f) << 3);
  float a0, d;
  asm("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(a0), "=f"(d) : "r"(addr));
  float fr = __fsub_rn(pos, __fsub_rn(f, 8388608.0f));
  return __fmaf_rn(fr, d, a0);
}

// O8: piecewise-linear lookup on t * (N - 1) with the slope table tab[i] =
// (A[i], A[i+1] - A[i]) and tab[N-1] = (A[N-1], 0): at pos = N-1 the result is A[N-1].
// floor(pos) for 0 <= pos < 2^23 without a conversion instruction: pos + 2^23 rounded
// toward zero is 2^23 + floor(pos) exactly; its low mantissa bits are the integer.
__device__ __forceinline__ float sample_tab(const float2* tab, float nm1, float t) {
  float pos = __fmul_rn(t, nm1);
  float f = __fadd_rz(pos, 8388608.0f);
  int i0 = __float_as_int(f) - 0x4B000000;
  float fr = __fsub_rn(pos, __fsub_rn(f, 8388608.0f));   // pos - (float)i0, exact
  float2 e = tab[i0];
  return __fmaf_rn(fr, e.y, e.x);
}

// O8 on an RGBA table (one channel c), identical op order.
__device__ __forceinline__ float sample_rgba(const float4* tf, int N, float t, int c) {
  float nm1 = (float)(N - 1);
  float pos = __fmul_rn(t, nm1);
  if (pos >= nm1) {
    float4 e = tf[N - 1];
    return c == 0 ? e.x : c == 1 ? e.y : c == 2 ? e.z : e.w;
  }
  int i0 = (int)pos;
  float fr = __fsub_rn(pos, (float)i0);
  float4 a = tf[i0], b = tf[i0 + 1];
  float a0 = c == 0 ? a.x : c == 1 ? a.y : c == 2 ? a.z : a.w;
  float a1 = c == 0 ? b.x : c == 1 ? b.y : c == 2 ? b.z : b.w;
  return __fmaf_rn(fr, __fsub_rn(a1, a0), a0);
}

// O10 detpow for non-integer P: log2 by atanh series, exp2 by Taylor polynomial.
__device__ __forceinline__ float det_log2(float g) {
  int e;
  float m = frexpf(g, &e);
  if (m < 0x1.6a09e6p-1f) {
    m = __fmul_rn(m, 2.0f);
    e = e - 1;
  }
  float u = __fdiv_rn(__fsub_rn(m, 1.0f), __fadd_rn(m, 1.0f));
  float z = __fmul_rn(u, u);
  float p = 0x1.c71c72p-4f;
  p = __fmaf_rn(p, z, 0x1.24924ap-3f);
  p = __fmaf_rn(p, z, 0x1.99999ap-3f);
  p = __fmaf_rn(p, z, 0x1.555556p-2f);
  p = __fmaf_rn(p, z, 1.0f);
  float t1 = __fmul_rn(u, p);
  float t2 = __fmul_rn(t1, 0x1.715476p+1f);
  return __fadd_rn((float)e, t2);
}

__device__ __forceinline__ float det_exp2(float y) {
  float k = floorf(y);
  float fr = __fsub_rn(y, k);
  float w = __fmul_rn(fr, 0x1.62e430p-1f);
  float p = 0x1.a01a02p-16f;
  p = __fmaf_rn(p, w, 0x1.a01a02p-13f);
  p = __fmaf_rn(p, w, 0x1.6c16c2p-10f);
  p = __fmaf_rn(p, w, 0x1.111112p-7f);
  p = __fmaf_rn(p, w, 0x1.555556p-5f);
  p = __fmaf_rn(p, w, 0x1.555556p-3f);
  p = __fmaf_rn(p, w, 0.5f);
  p = __fmaf_rn(p, w, 1.0f);
  p = __fmaf_rn(p, w, 1.0f);
  if (k < -149.0f) return 0.0f;
  if (k > 127.0f) return __int_as_float(0x7f800000);
  return __fmul_rn(p, pow2f((int)k));
}

__device__ __forceinline__ float pow_p(float g, const PowParams& pw) {
  if (pw.kind == kPow0) return 1.0f;
  if (pw.kind == kPow1) return g;
  if (pw.kind == kPowInt) {
    float f = g;
    for (int k = 1; k < pw.k; ++k) f = __fmul_rn(f, g);
    return f;
  }
  if (g == 0.0f) return 0.0f;
  return det_exp2(__fmul_rn(pw.P, det_log2(g)));
}

// Eq. 3 with the minimum importance clamped on the ratio (reading A9-A11).
__device__ __forceinline__ float importance(float V, float maxv, int L, float eps,
                                            const PowParams& pw) {
  float r = maxv > 0.0f ? __fdiv_rn(V, maxv) : 0.0f;
  r = r > eps ? r : eps;
  r = r < 1.0f ? r : 1.0f;
  float g = __fmul_rn(r, pow2f(L));
  return pow_p(g, pw);
}

// ------------------------------------------------------------------ small helpers
template <int ITEMS>
__device__ __forceinline__ void load_f(const float* __restrict__ p, float (&v)[ITEMS]) {
  if constexpr (ITEMS % 4 == 0) {
#pragma unroll
    for (int j = 0; j < ITEMS / 4; ++j) {
      float4 q = __ldg(reinterpret_cast<const float4*>(p) + j);
      v[4 * j] = q.x; v[4 * j + 1] = q.y; v[4 * j + 2] = q.z; v[4 * j + 3] = q.w;
    }
  } else if constexpr (ITEMS == 2) {
    float2 q = __ldg(reinterpret_cast<const float2*>(p));
    v[0] = q.x; v[1] = q.y;
  } else {
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) v[j] = __ldg(p + j);
  }
}

template <int ITEMS>
__device__ __forceinline__ void load_u8(const uint8_t* __restrict__ p, int (&v)[ITEMS]) {
  if constexpr (ITEMS == 16) {
    uint4 q = __ldg(reinterpret_cast<const uint4*>(p));
    uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = (w[j >> 2] >> (8 * (j & 3))) & 0xff;
  } else if constexpr (ITEMS == 8) {
    uint2 q = __ldg(reinterpret_cast<const uint2*>(p));
    uint32_t w[2] = {q.x, q.y};
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = (w[j >> 2] >> (8 * (j & 3))) & 0xff;
  } else if constexpr (ITEMS == 4) {
    uint32_t w = __ldg(reinterpret_cast<const uint32_t*>(p));
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = (w >> (8 * j)) & 0xff;
  } else {
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) v[j] = __ldg(p + j);
  }
}

// O14-O15: the vertex of one (member, pixel) from its count, min / max bits of t and the
// 128-bit 2^-40 fixed-point sum of t (hi:lo words): mean = sum / count in double, rounded
// to float, then the TF's RGBA at the mean.
__device__ __forceinline__ dvl_vertex make_vertex(uint32_t cnt, uint32_t mn, uint32_t mx,
                                                  unsigned long long shi, unsigned long long slo,
                                                  const float4* tf, int N) {
  dvl_vertex v;
  v.count = cnt;
  if (cnt) {
    const double sum = ((double)shi * 18446744073709551616.0 + (double)slo) * kSumUnscale;
    const float mean = (float)(sum / (double)cnt);
    v.t_min = __uint_as_float(mn);
    v.t_max = __uint_as_float(mx);
    v.t_mean = mean;
    v.r = sample_rgba(tf, N, mean, 0);
    v.g = sample_rgba(tf, N, mean, 1);
    v.b = sample_rgba(tf, N, mean, 2);
    v.y = sample_rgba(tf, N, mean, 3);
  } else {
    v.t_min = v.t_max = v.t_mean = v.y = v.r = v.g = v.b = 0.0f;
  }
  return v;
}

// The same sum (mod 2^64) from three 32-bit warp reductions of 22-bit chunks (each chunk
// sum < 2^27: no overflow), every lane gets it.
__device__ __forceinline__ unsigned long long warp_sum_u64_redux(unsigned long long v) {
  const uint32_t c0 = __reduce_add_sync(0xffffffffu, (uint32_t)v & 0x3fffffu);
  const uint32_t c1 = __reduce_add_sync(0xffffffffu, (uint32_t)(v >> 22) & 0x3fffffu);
  const uint32_t c2 = __reduce_add_sync(0xffffffffu, (uint32_t)(v >> 44));
  return (unsigned long long)c0 + ((unsigned long long)c1 << 22) + ((unsigned long long)c2 << 44);
}

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ unsigned long long warp_incl_scan_u64(unsigned long long v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    unsigned long long u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += u;
  }
  return v;
}

// 128-bit atomic add of a u64 into (lo, hi) words: exact in any order.
// The fixed-point sums are kept as two 64-bit counters, of the low and of the high 32-bit
// halves of the added values (sum = slo + shi * 2^32): no carry to propagate, so both adds
// are fire-and-forget reductions (no round trip to L2 for a returned value).  Exact while a
// counter takes < 2^32 adds (one per flush of a warp or group: n < 2^38 cells).
__device__ __forceinline__ void red_add_sum(unsigned long long* slo, unsigned long long* shi,
                                            unsigned long long v) {
  if (v == 0) return;
  atomicAdd(slo, v & 0xffffffffull);
  if (v >> 32) atomicAdd(shi, v >> 32);
}
// the 128-bit sum (hi:lo words) of the two counters
__device__ __forceinline__ void sum_words(unsigned long long slo, unsigned long long shi,
                                          unsigned long long& hw, unsigned long long& lw) {
  lw = slo + (shi << 32);
  hw = (shi >> 32) + (lw < slo ? 1ull : 0ull);
}

}  // namespace dvl
