// build.cu -- B0 (ingest + validate) and B3 (permute into curve order + overlap check).
//   B0 (reading O1/A22): E = max(lower + 2^L), Lmax, L <= 20 and lower multiple
//      of 2^L; the member min/max over finite values are folded into B3.
//   B3 (readings O4/O5): level_s[k] = level[perm[k]], scal_s[m][k] =
//      scal[m][perm[k]]; codes strictly increasing and consecutive dyadic code blocks
//      [code & ~(8^L - 1), +8^L) disjoint (a laminar family is disjoint iff consecutive
//      members are), which detects every duplicate or overlapping cell.
#include <algorithm>
#include <cstring>

#include "dvl_common.cuh"
#include "dvl_internal.h"

namespace dvl {

__device__ __forceinline__ uint32_t float_to_ordered(float f) {
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

float ordered_to_float(uint32_t u) {
  uint32_t b = (u & 0x80000000u) ? (u & 0x7fffffffu) : ~u;
  float f;
  memcpy(&f, &b, 4);
  return f;
}

// B0 over the geometry only (13 B per cell; the member ranges are folded into B3, which
// reads every scalar anyway): four cells per thread, 16-byte loads of the AoS corners.
template <bool VEC>
__global__ void __launch_bounds__(kBlock)
ingest_geom_kernel(const uint32_t* __restrict__ lower, const uint8_t* __restrict__ level,
                   int64_t n, IngestOut* out) {
  unsigned long long ext = 0;
  uint32_t lmax = 0, err = 0;
  const int64_t groups = (n + 3) >> 2;
  for (int64_t g = (int64_t)blockIdx.x * kBlock + threadIdx.x; g < groups;
       g += (int64_t)gridDim.x * kBlock) {
    const int64_t h0 = 4 * g;
    const int cnt = (int)(n - h0 < 4 ? n - h0 : 4);
    uint32_t c[12], L[4];
    if (VEC && cnt == 4) {
      const uint4* l4 = reinterpret_cast<const uint4*>(lower) + 3 * g;
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const uint4 v = l4[q];
        c[4 * q] = v.x;
        c[4 * q + 1] = v.y;
        c[4 * q + 2] = v.z;
        c[4 * q + 3] = v.w;
      }
      const uint32_t L4 = reinterpret_cast<const uint32_t*>(level)[g];
#pragma unroll
      for (int i = 0; i < 4; ++i) L[i] = (L4 >> (8 * i)) & 255u;
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const bool ok = i < cnt;
        L[i] = ok ? level[h0 + i] : 0u;
        c[3 * i] = ok ? lower[3 * (h0 + i)] : 0u;
        c[3 * i + 1] = ok ? lower[3 * (h0 + i) + 1] : 0u;
        c[3 * i + 2] = ok ? lower[3 * (h0 + i) + 2] : 0u;
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (i >= cnt) continue;
      if (L[i] > 20) {
        err |= kErrInval;
        continue;
      }
      const uint32_t w = 1u << L[i];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        if (c[3 * i + k] & (w - 1)) err |= kErrInval;
        const unsigned long long e = (unsigned long long)c[3 * i + k] + w;
        ext = e > ext ? e : ext;
      }
      lmax = L[i] > lmax ? L[i] : lmax;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long e2 = __shfl_xor_sync(0xffffffffu, ext, o);
    ext = e2 > ext ? e2 : ext;
    lmax = max(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
    err |= __shfl_xor_sync(0xffffffffu, err, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(&out->extent, ext);
    atomicMax(&out->lmax, lmax);
    if (err) atomicOr(&out->err, err);
  }
}

void launch_ingest_geom(const uint32_t* lower, const uint8_t* level, int64_t n, IngestOut* out,
                        int num_sms, cudaStream_t st) {
  const int64_t groups = (n + 3) / 4;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((groups + kBlock - 1) / kBlock,
                                                                (int64_t)num_sms * 8));
  const bool vec = (reinterpret_cast<uintptr_t>(lower) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(level) & 3) == 0;
  if (vec)
    ingest_geom_kernel<true><<<grid, kBlock, 0, st>>>(lower, level, n, out);
  else
    ingest_geom_kernel<false><<<grid, kBlock, 0, st>>>(lower, level, n, out);
}

// B3 with eight consecutive curve positions per thread: the permutation and the keys by
// 16-byte loads, all gathered loads of the eight cells issued before their stores (level,
// then each member), level_s as 4-byte stores and each member row as 16-byte stores; the
// overlap check takes the next cell's key and level from the neighbour lane; the member
// ranges (finite min / max, for the default domains) are folded in here.
constexpr int kGI = 8;   // cells per thread

template <typename K>
__global__ void __launch_bounds__(kBlock)
gather_validate8_kernel(const K* __restrict__ keys, const uint32_t* __restrict__ perm,
                        const uint8_t* __restrict__ level_in, const float* const* __restrict__ scal_in,
                        int64_t n, int M, int64_t n_pad, uint8_t* __restrict__ level_s,
                        float* __restrict__ scal_s, uint32_t* err, IngestOut* ranges) {
  __shared__ uint32_t s_mn[64], s_mx[64];
  for (int m = threadIdx.x; m < M; m += kBlock) {
    s_mn[m] = 0xffffffffu;
    s_mx[m] = 0u;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t groups = (n + kGI - 1) / kGI;
  const int64_t wstride = (int64_t)gridDim.x * kBlock;
  uint32_t bad = 0;
  for (int64_t g0 = (int64_t)blockIdx.x * kBlock + (threadIdx.x & ~31); g0 < groups; g0 += wstride) {
    const int64_t g = g0 + lane;
    const int64_t k0 = (int64_t)kGI * g;
    const int cnt = g < groups ? (int)(n - k0 < kGI ? n - k0 : kGI) : 0;
    uint32_t p[kGI];
    K key[kGI];
    if (cnt == kGI) {
#pragma unroll
      for (int q = 0; q < kGI / 4; ++q) {
        const uint4 v = reinterpret_cast<const uint4*>(perm)[2 * g + q];
        p[4 * q] = v.x; p[4 * q + 1] = v.y; p[4 * q + 2] = v.z; p[4 * q + 3] = v.w;
      }
      if (sizeof(K) == 4) {
#pragma unroll
        for (int q = 0; q < kGI / 4; ++q) {
          const uint4 v = reinterpret_cast<const uint4*>(keys)[2 * g + q];
          key[4 * q] = v.x; key[4 * q + 1] = v.y; key[4 * q + 2] = v.z; key[4 * q + 3] = v.w;
        }
      } else {
#pragma unroll
        for (int q = 0; q < kGI / 2; ++q) {
          const ulonglong2 v = reinterpret_cast<const ulonglong2*>(keys)[4 * g + q];
          key[2 * q] = (K)v.x; key[2 * q + 1] = (K)v.y;
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < kGI; ++i) {
        p[i] = i < cnt ? perm[k0 + i] : 0u;
        key[i] = i < cnt ? keys[k0 + i] : (K)0;
      }
    }
    // a source index out of range can only come from duplicate codes (the sort's slots
    // of a duplicate are not all written): the cell is skipped and the build fails OVERLAP
#pragma unroll
    for (int i = 0; i < kGI; ++i) {
      if (i < cnt && p[i] >= (uint64_t)n) {
        bad = 1;
        p[i] = 0;
      }
    }
    uint32_t L[kGI];
#pragma unroll
    for (int i = 0; i < kGI; ++i) L[i] = i < cnt ? (uint32_t)level_in[p[i]] : 0u;
    // the cell after this thread's last one: the next lane's first, or loaded by lane 31
    K knext = __shfl_down_sync(0xffffffffu, key[0], 1);
    uint32_t Lnext = __shfl_down_sync(0xffffffffu, L[0], 1);
    if (lane == 31 && cnt == kGI && k0 + kGI < n) {
      knext = keys[k0 + kGI];
      const uint32_t pn = perm[k0 + kGI];
      Lnext = pn < (uint64_t)n ? level_in[pn] : 0u;
    }
#pragma unroll
    for (int i = 0; i < kGI; ++i) {
      if (i >= cnt || k0 + i + 1 >= n) continue;
      const unsigned long long a = key[i];
      const unsigned long long b = i + 1 < kGI ? (unsigned long long)key[i + 1] : (unsigned long long)knext;
      const uint32_t Lb = i + 1 < kGI ? L[i + 1] : Lnext;
      const unsigned long long lena = 1ull << (3 * L[i]), lenb = 1ull << (3 * Lb);
      const unsigned long long sa = a & ~(lena - 1), sb = b & ~(lenb - 1);
      if (a >= b || sa + lena > sb) bad = 1;
    }
    if (cnt == kGI) {
#pragma unroll
      for (int q = 0; q < kGI / 4; ++q)
        reinterpret_cast<uint32_t*>(level_s)[2 * g + q] =
            L[4 * q] | (L[4 * q + 1] << 8) | (L[4 * q + 2] << 16) | (L[4 * q + 3] << 24);
    } else {
      for (int i = 0; i < cnt; ++i) level_s[k0 + i] = (uint8_t)L[i];
    }
    for (int m = 0; m < M; ++m) {
      const float* __restrict__ src = scal_in[m];
      float v[kGI];
#pragma unroll
      for (int i = 0; i < kGI; ++i) v[i] = i < cnt ? __ldg(src + p[i]) : 0.0f;
      float* dst = scal_s + (int64_t)m * n_pad;
      if (cnt == kGI) {
#pragma unroll
        for (int q = 0; q < kGI / 4; ++q)
          reinterpret_cast<float4*>(dst)[2 * g + q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
      } else {
        for (int i = 0; i < cnt; ++i) dst[k0 + i] = v[i];
      }
      uint32_t mn = 0xffffffffu, mx = 0u;
#pragma unroll
      for (int i = 0; i < kGI; ++i) {
        if (i < cnt && isfinite(v[i])) {
          const uint32_t o = float_to_ordered(v[i]);
          mn = min(mn, o);
          mx = max(mx, o);
        }
      }
      mn = __reduce_min_sync(0xffffffffu, mn);
      mx = __reduce_max_sync(0xffffffffu, mx);
      if (lane == 0 && mn != 0xffffffffu) {   // the warp saw a finite value
        atomicMin(&s_mn[m], mn);
        atomicMax(&s_mx[m], mx);
      }
    }
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(err, kErrOverlap);
  __syncthreads();
  for (int m = threadIdx.x; m < M; m += kBlock) {
    if (s_mn[m] != 0xffffffffu) {
      atomicMin(&ranges->vmin[m], s_mn[m]);
      atomicMax(&ranges->vmax[m], s_mx[m]);
      atomicOr(&ranges->any[m], 1u);
    }
  }
}

void launch_gather_validate4(const void* keys, int key_bytes, const uint32_t* perm,
                             const uint8_t* level_in, const float* const* scal_in, int64_t n,
                             int M, int64_t n_pad, uint8_t* level_s, float* scal_s, uint32_t* err,
                             IngestOut* ranges, int num_sms, cudaStream_t st) {
  const int64_t groups = (n + kGI - 1) / kGI;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((groups + kBlock - 1) / kBlock,
                                                                (int64_t)num_sms * 8));
  if (key_bytes == 4)
    gather_validate8_kernel<uint32_t><<<grid, kBlock, 0, st>>>(
        (const uint32_t*)keys, perm, level_in, scal_in, n, M, n_pad, level_s, scal_s, err, ranges);
  else
    gather_validate8_kernel<unsigned long long><<<grid, kBlock, 0, st>>>(
        (const unsigned long long*)keys, perm, level_in, scal_in, n, M, n_pad, level_s, scal_s, err,
        ranges);
}

template <typename K>
__global__ void widen_kernel(const K* __restrict__ keys, const uint32_t* __restrict__ perm,
                             int64_t n, uint64_t* codes, uint64_t* ids) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    if (codes) codes[k] = keys[k];
    if (ids) ids[k] = perm[k];
  }
}

void launch_widen(const void* keys, int key_bytes, const uint32_t* perm, int64_t n,
                  uint64_t* codes_out, uint64_t* ids_out, cudaStream_t st) {
  int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
  if (grid < 1) grid = 1;
  if (key_bytes == 4)
    widen_kernel<uint32_t><<<grid, 256, 0, st>>>((const uint32_t*)keys, perm, n, codes_out, ids_out);
  else
    widen_kernel<unsigned long long><<<grid, 256, 0, st>>>((const unsigned long long*)keys, perm,
                                                           n, codes_out, ids_out);
}

}  // namespace dvl
