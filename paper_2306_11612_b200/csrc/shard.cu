// shard.cu -- per-shard pieces of the sharded TF update.  A shard holds one
// contiguous range of the global curve order; only two global quantities cross shards:
//   * the scan offset: the sum of the earlier shards' fixed-point weights (and Qtot), from
//     the gathered shard totals (shard_offsets_kernel);
//   * the per-pixel accumulators, exported as int64 planes that two collectives combine:
//     one MAX over the first two planes (the minima are exported negated: min x =
//     -max(-x)) and one SUM over the third (acc_export_kernel); turned into vertices after
//     the merge (epilogue_merged_kernel).
// Everything is integer, so the merged result is bit-identical to the unsharded one.
//
// Export layout (int64, W pixels, M members):
//   -MIN plane [W + M W]: -lo (first cell; none -> -INT64_MAX), -tmin bits (none -> -(2^32-1))
//   MAX plane  [W + M W]: hi (last cell; none -> 0),       tmax bits (none -> 0)
//   SUM plane  [3 M W]:   the 128-bit sum as three 32-bit limbs, limb-major
#include <algorithm>

#include "dvl_common.cuh"
#include "dvl_internal.h"

namespace dvl {

__global__ void shard_offsets_kernel(const unsigned long long* __restrict__ totals, int nshards,
                                     int shard, unsigned long long* offset,
                                     unsigned long long* qtot) {
  if (threadIdx.x != 0) return;
  unsigned long long o = 0, t = 0;
  for (int r = 0; r < nshards; ++r) {
    t += totals[r];
    if (r < shard) o += totals[r];
  }
  *offset = o;
  *qtot = t;
}

void launch_shard_offsets(const unsigned long long* totals, int nshards, int shard,
                          unsigned long long* offset, unsigned long long* qtot, cudaStream_t st) {
  shard_offsets_kernel<<<1, 32, 0, st>>>(totals, nshards, shard, offset, qtot);
}

__global__ void acc_export_kernel(Acc acc, uint32_t W, int M, long long* __restrict__ out) {
  const int64_t MW = (int64_t)M * W;
  long long* mn = out;
  long long* mx = out + W + MW;
  long long* sm = out + 2 * (W + MW);
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < MW;
       k += (int64_t)gridDim.x * blockDim.x) {
    if (k < W) {
      const unsigned long long lo = acc.lo[k], hi = acc.hi[k];
      mn[k] = -(lo == ~0ull ? 0x7fffffffffffffffll : (long long)lo);
      mx[k] = (long long)hi;
      acc.lo[k] = ~0ull;
      acc.hi[k] = 0ull;
    }
    mn[W + k] = -(long long)acc.tmin[k];
    mx[W + k] = (long long)acc.tmax[k];
    // limbs of 2^0, 2^32, 2^64 (sum = slo + shi * 2^32; each limb < 2^33)
    const unsigned long long sl = acc.slo[k], sh = acc.shi[k];
    sm[k] = (long long)(sl & 0xffffffffull);
    sm[MW + k] = (long long)((sl >> 32) + (sh & 0xffffffffull));
    sm[2 * MW + k] = (long long)(sh >> 32);
    acc.tmin[k] = 0xffffffffu;
    acc.tmax[k] = 0u;
    acc.slo[k] = 0ull;
    acc.shi[k] = 0ull;
  }
}

void launch_acc_export(const Acc& acc, uint32_t W, int M, long long* out, cudaStream_t st) {
  const int64_t MW = (int64_t)M * W;
  const int grid = (int)std::min<int64_t>((MW + 255) / 256, 4096);
  acc_export_kernel<<<grid, 256, 0, st>>>(acc, W, M, out);
}

// as epilogue_kernel (one thread per (member, pixel), pixel fastest), from the merged planes
__global__ void __launch_bounds__(256)
epilogue_merged_kernel(const long long* __restrict__ merged, uint32_t W, int M, int N,
                       const float4* __restrict__ rgba, dvl_vertex* __restrict__ out,
                       unsigned long long* bin_lo, unsigned long long* bin_hi) {
  const int64_t MW = (int64_t)M * W;
  const long long* mn = merged;
  const long long* mx = merged + W + MW;
  const long long* sm = merged + 2 * (W + MW);
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= MW) return;
  const int m = (int)(k / W);
  const uint32_t x = (uint32_t)(k - (int64_t)m * W);
  const long long lo_s = -mn[x];   // the plane holds -min
  const unsigned long long lo = lo_s == 0x7fffffffffffffffll ? ~0ull : (unsigned long long)lo_s;
  const unsigned long long hi = (unsigned long long)mx[x];
  if (m == 0) {
    bin_lo[x] = lo;
    bin_hi[x] = hi;
  }
  const uint32_t cnt = lo <= hi ? (uint32_t)(hi - lo + 1) : 0u;
  // 128-bit sum from the three limbs (each < 2^49 after summing <= 2^16 shards)
  const unsigned long long l0 = (unsigned long long)sm[k], l1 = (unsigned long long)sm[MW + k],
                           l2 = (unsigned long long)sm[2 * MW + k];
  const unsigned long long a = l0 + (l1 << 32);
  const unsigned long long carry = (a < l0 ? 1ull : 0ull) + (l1 >> 32);
  const unsigned long long hiw = l2 + carry;
  out[k] = make_vertex(cnt, (uint32_t)(-mn[W + k]), (uint32_t)mx[W + k], hiw, a,
                       rgba + (int64_t)m * N, N);
}

void launch_epilogue_merged(const long long* merged, uint32_t W, int M, int N, const float4* rgba,
                            dvl_vertex* out, unsigned long long* bin_lo, unsigned long long* bin_hi,
                            cudaStream_t st) {
  const int grid = (int)(((int64_t)M * W + 255) / 256);
  epilogue_merged_kernel<<<grid, 256, 0, st>>>(merged, W, M, N, rgba, out, bin_lo, bin_hi);
}

}  // namespace dvl
