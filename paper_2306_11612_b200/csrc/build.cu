// build.cu -- B0 (ingest + validate) and B3 (permute into curve order + overlap check).
//   B0 (reading O1/A22): E = max(lower + 2^L), Lmax, L <= 20 and lower multiple
//      of 2^L, member min/max over finite values.
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

__global__ void __launch_bounds__(kBlock)
ingest_geom_kernel(const uint32_t* __restrict__ lower, const uint8_t* __restrict__ level,
                   int64_t n, IngestOut* out) {
  unsigned long long ext = 0;
  uint32_t lmax = 0, err = 0;
  for (int64_t h = (int64_t)blockIdx.x * kBlock + threadIdx.x; h < n;
       h += (int64_t)gridDim.x * kBlock) {
    uint32_t L = level[h];
    if (L > 20) {
      err |= kErrInval;
      continue;
    }
    uint32_t w = 1u << L;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      uint32_t c = lower[3 * h + k];
      if (c & (w - 1)) err |= kErrInval;
      unsigned long long e = (unsigned long long)c + w;
      ext = e > ext ? e : ext;
    }
    lmax = L > lmax ? L : lmax;
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

__global__ void __launch_bounds__(kBlock)
ingest_member_kernel(const float* const* __restrict__ scal, int64_t n, IngestOut* out) {
  const int m = blockIdx.y;
  const float* __restrict__ v = scal[m];
  uint32_t mn = 0xffffffffu, mx = 0u, any = 0u;
  for (int64_t h = (int64_t)blockIdx.x * kBlock + threadIdx.x; h < n;
       h += (int64_t)gridDim.x * kBlock) {
    float f = v[h];
    if (isfinite(f)) {
      uint32_t o = float_to_ordered(f);
      mn = min(mn, o);
      mx = max(mx, o);
      any = 1u;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    any |= __shfl_xor_sync(0xffffffffu, any, o);
  }
  if ((threadIdx.x & 31) == 0 && any) {
    atomicMin(&out->vmin[m], mn);
    atomicMax(&out->vmax[m], mx);
    atomicOr(&out->any[m], 1u);
  }
}

void launch_ingest(const uint32_t* lower, const uint8_t* level, const float* const* scal,
                   int64_t n, int M, IngestOut* out, int grid, cudaStream_t st) {
  ingest_geom_kernel<<<grid, kBlock, 0, st>>>(lower, level, n, out);
  dim3 g2((unsigned)((grid + M - 1) / M > 0 ? (grid + M - 1) / M : 1), (unsigned)M);
  ingest_member_kernel<<<g2, kBlock, 0, st>>>(scal, n, out);
}

template <typename K>
__global__ void __launch_bounds__(kBlock)
gather_validate_kernel(const K* __restrict__ keys, const uint32_t* __restrict__ perm,
                       const uint8_t* __restrict__ level_in, const float* const* __restrict__ scal_in,
                       int64_t n, int M, int64_t n_pad, uint8_t* __restrict__ level_s,
                       float* __restrict__ scal_s, uint32_t* err) {
  uint32_t bad = 0;
  for (int64_t k = (int64_t)blockIdx.x * kBlock + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * kBlock) {
    uint32_t p = perm[k];
    uint32_t L = level_in[p];
    level_s[k] = (uint8_t)L;
    for (int m = 0; m < M; ++m) scal_s[(int64_t)m * n_pad + k] = __ldg(scal_in[m] + p);
    if (k + 1 < n) {
      unsigned long long a = keys[k], b = keys[k + 1];
      uint32_t Lb = level_in[perm[k + 1]];
      unsigned long long lena = 1ull << (3 * L), lenb = 1ull << (3 * Lb);
      unsigned long long sa = a & ~(lena - 1), sb = b & ~(lenb - 1);
      if (a >= b || sa + lena > sb) bad = 1;
    }
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(err, kErrOverlap);
}

void launch_gather_validate(const void* keys, int key_bytes, const uint32_t* perm,
                            const uint8_t* level_in, const float* const* scal_in, int64_t n,
                            int M, int64_t n_pad, uint8_t* level_s, float* scal_s,
                            uint32_t* err, int grid, cudaStream_t st) {
  if (key_bytes == 4)
    gather_validate_kernel<uint32_t><<<grid, kBlock, 0, st>>>(
        (const uint32_t*)keys, perm, level_in, scal_in, n, M, n_pad, level_s, scal_s, err);
  else
    gather_validate_kernel<unsigned long long><<<grid, kBlock, 0, st>>>(
        (const unsigned long long*)keys, perm, level_in, scal_in, n, M, n_pad, level_s, scal_s,
        err);
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
