// sort.cu -- B2: onesweep LSD radix sort of (Hilbert code, cell id) pairs (P:309-311:
// the order is established once).  8-bit digits, one kernel per digit pass:
//   * tiles of 256 threads x 16 keys, tile ids from an atomic counter (forward progress
//     of the look-back does not depend on block scheduling order);
//   * warp-level digit ranking with __match_any_sync and per-warp running counts in
//     shared memory (stable: items are ranked in input order);
//   * per-digit decoupled look-back over the tiles' digit counts (u32 status words,
//     2 flag bits + 30 count bits) on top of the pass's global digit histogram, which the
//     Hilbert encoder produced for all passes in one read of the keys;
//   * keys/ids staged in shared memory in tile-sorted order, so the global scatter writes
//     runs of equal digits contiguously.
#include "dvl_common.cuh"
#include "dvl_internal.h"
#include "dvl_tma.cuh"

namespace dvl {

// exclusive scan of each pass's 256-bucket histogram (one block per pass)
__global__ void hist_scan_kernel(const uint32_t* __restrict__ hist, uint32_t* __restrict__ base) {
  __shared__ uint32_t s[256];
  int p = blockIdx.x, d = threadIdx.x;
  s[d] = hist[p * 256 + d];
  __syncthreads();
  if (d == 0) {
    uint32_t run = 0;
    for (int i = 0; i < 256; ++i) {
      uint32_t c = s[i];
      s[i] = run;
      run += c;
    }
  }
  __syncthreads();
  base[p * 256 + d] = s[d];
}

template <typename K, bool IOTA>
__global__ void __launch_bounds__(kBlock, 2)
onesweep_kernel(const K* __restrict__ kin, const uint32_t* __restrict__ vin,
                K* __restrict__ kout, uint32_t* __restrict__ vout, int64_t n, int shift,
                const uint32_t* __restrict__ digit_base, uint32_t* status, uint32_t* tile_ctr) {
  extern __shared__ __align__(16) unsigned char smem[];
  K* s_keys = reinterpret_cast<K*>(smem);
  uint32_t* s_vals = reinterpret_cast<uint32_t*>(smem + sizeof(K) * kSortTile);
  __shared__ uint32_t s_warp[kBlock / 32][256];
  __shared__ uint32_t s_start[256];
  __shared__ int64_t s_scatter[256];
  __shared__ uint32_t s_wsum[kBlock / 32];
  __shared__ uint32_t s_tile;
  __shared__ uint64_t s_bar;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    s_tile = atomicAdd(tile_ctr, 1u);
    mbar_init(&s_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = tid; i < (kBlock / 32) * 256; i += kBlock) (&s_warp[0][0])[i] = 0;
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t tile_base = tile * kSortTile;
  const int64_t wbase = tile_base + warp * (32 * kSortItems);

  K key[kSortItems];
  uint32_t val[kSortItems];
  uint32_t rank[kSortItems];
  if (tile_base + kSortTile <= n) {
    // a full tile: one bulk copy of its keys (and ids) into shared memory (the staging area
    // of the scatter below, free until then), so that the ranking reads them at shared
    // memory latency instead of waiting on each global load
    if (tid == 0) {
      const uint64_t pol = policy_evict_first();
      mbar_arrive_expect_tx(&s_bar, kSortTile * (uint32_t)(sizeof(K) + (IOTA ? 0 : 4)));
      tma_load_1d(s_keys, kin + tile_base, kSortTile * (uint32_t)sizeof(K), &s_bar, pol);
      if (!IOTA) tma_load_1d(s_vals, vin + tile_base, kSortTile * 4u, &s_bar, pol);
    }
    mbar_wait(&s_bar, 0);
#pragma unroll
    for (int i = 0; i < kSortItems; ++i) {
      const int l = warp * (32 * kSortItems) + i * 32 + lane;
      key[i] = s_keys[l];
      val[i] = IOTA ? (uint32_t)(tile_base + l) : s_vals[l];   // first pass: ids are implicit
    }
  } else {
#pragma unroll
    for (int i = 0; i < kSortItems; ++i) {
      int64_t idx = wbase + i * 32 + lane;
      bool ok = idx < n;
      key[i] = ok ? kin[idx] : (K)0;
      val[i] = ok ? (IOTA ? (uint32_t)idx : vin[idx]) : 0u;
    }
  }
  const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    int64_t idx = wbase + i * 32 + lane;
    bool ok = idx < n;
    uint32_t d = ok ? (uint32_t)((key[i] >> shift) & 255) : 256u;
    uint32_t peers = __match_any_sync(0xffffffffu, d);
    int leader = __ffs(peers) - 1;
    uint32_t base = 0;
    if (ok && lane == leader) base = s_warp[warp][d];
    base = __shfl_sync(0xffffffffu, base, leader);
    rank[i] = base + __popc(peers & lt);
    if (ok && lane == leader) s_warp[warp][d] = base + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // per digit: exclusive scan over warps -> warp offsets; tile count
  const int d = tid;
  uint32_t cnt = 0;
#pragma unroll
  for (int w = 0; w < kBlock / 32; ++w) {
    uint32_t c = s_warp[w][d];
    s_warp[w][d] = cnt;
    cnt += c;
  }
  // publish this tile's aggregate count of digit d
  if (tile == 0)
    atomicExch(status + d, kSortInc | cnt);
  else
    atomicExch(status + tile * 256 + d, kSortAgg | cnt);
  // tile-local exclusive scan of the digit counts (block scan over 256 digits)
  uint32_t incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u;
  }
  if (lane == 31) s_wsum[warp] = incl;
  __syncthreads();
  uint32_t wpre = 0;
  for (int w = 0; w < warp; ++w) wpre += s_wsum[w];
  const uint32_t start = wpre + incl - cnt;
  s_start[d] = start;
  __syncthreads();
  // stage keys in tile-sorted order
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    int64_t idx = wbase + i * 32 + lane;
    if (idx < n) {
      uint32_t dd = (uint32_t)((key[i] >> shift) & 255);
      uint32_t pos = s_start[dd] + s_warp[warp][dd] + rank[i];
      s_keys[pos] = key[i];
      s_vals[pos] = val[i];
    }
  }
  // decoupled look-back of digit d over the preceding tiles
  if (tile > 0) {
    // four predecessors per round trip; tile 0 always publishes an inclusive count
    uint32_t excl = 0;
    int64_t j = tile - 1;
    bool done = false;
    while (!done) {
      uint32_t sv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        sv[u] = j - u >= 0 ? *(volatile uint32_t*)(status + (j - u) * 256 + d) : (2u << 30);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (!done) {
          while ((sv[u] >> 30) == 0) sv[u] = *(volatile uint32_t*)(status + (j - u) * 256 + d);
          excl += sv[u] & kSortMask;
          done = (sv[u] >> 30) == 2;
        }
      }
      j -= 4;
    }
    atomicExch(status + tile * 256 + d, kSortInc | (excl + cnt));
    s_scatter[d] = (int64_t)digit_base[d] + excl - start;
  } else {
    s_scatter[d] = (int64_t)digit_base[d] - start;
  }
  __syncthreads();
  const int64_t valid = min((int64_t)kSortTile, n - tile_base);
  for (int j = tid; j < valid; j += kBlock) {
    K k = s_keys[j];
    int64_t dest = s_scatter[(uint32_t)((k >> shift) & 255)] + j;
    kout[dest] = k;
    vout[dest] = s_vals[j];
  }
}

// the digit histograms of all passes over codes already computed (the LSD sort of the
// distributed build's received runs; B1 builds them while it encodes)
template <typename K>
__global__ void __launch_bounds__(kBlock)
key_hist_kernel(const K* __restrict__ keys, int64_t n, int passes, uint32_t* __restrict__ hist) {
  __shared__ uint32_t s_hist[8][256];
  for (int i = threadIdx.x; i < passes * 256; i += kBlock) (&s_hist[0][0])[i] = 0;
  __syncthreads();
  for (int64_t h = (int64_t)blockIdx.x * kBlock + threadIdx.x; h < n; h += (int64_t)gridDim.x * kBlock) {
    const uint64_t code = keys[h];
    for (int p = 0; p < passes; ++p) atomicAdd(&s_hist[p][(code >> (8 * p)) & 255], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * 256; i += kBlock) {
    const uint32_t c = (&s_hist[0][0])[i];
    if (c) atomicAdd(hist + i, c);
  }
}

void launch_key_hist(const void* keys, int key_bytes, int64_t n, int passes, uint32_t* hist,
                     int num_sms, cudaStream_t st) {
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + kBlock - 1) / kBlock, (int64_t)num_sms * 8));
  if (key_bytes == 4)
    key_hist_kernel<uint32_t><<<grid, kBlock, 0, st>>>((const uint32_t*)keys, n, passes, hist);
  else
    key_hist_kernel<unsigned long long><<<grid, kBlock, 0, st>>>((const unsigned long long*)keys, n, passes, hist);
}

void launch_hist_scan(const uint32_t* hist, uint32_t* base, int passes, cudaStream_t st) {
  hist_scan_kernel<<<passes, 256, 0, st>>>(hist, base);
}

cudaError_t prepare_onesweep() {
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(onesweep_kernel<uint32_t, false>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kSortTile * 8))))
    return e;
  if ((e = cudaFuncSetAttribute(onesweep_kernel<uint32_t, true>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kSortTile * 8))))
    return e;
  if ((e = cudaFuncSetAttribute(onesweep_kernel<unsigned long long, false>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kSortTile * 12))))
    return e;
  return cudaFuncSetAttribute(onesweep_kernel<unsigned long long, true>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kSortTile * 12));
}

void launch_onesweep(const void* kin, const uint32_t* vin, void* kout, uint32_t* vout, int64_t n,
                     int key_bytes, int shift, const uint32_t* digit_base, uint32_t* status,
                     uint32_t* tile_ctr, cudaStream_t st) {
  int tiles = (int)((n + kSortTile - 1) / kSortTile);
  const bool iota = vin == nullptr;
  if (key_bytes == 4) {
    if (iota)
      onesweep_kernel<uint32_t, true><<<tiles, kBlock, kSortTile * 8, st>>>(
          (const uint32_t*)kin, vin, (uint32_t*)kout, vout, n, shift, digit_base, status, tile_ctr);
    else
      onesweep_kernel<uint32_t, false><<<tiles, kBlock, kSortTile * 8, st>>>(
          (const uint32_t*)kin, vin, (uint32_t*)kout, vout, n, shift, digit_base, status, tile_ctr);
  } else {
    if (iota)
      onesweep_kernel<unsigned long long, true><<<tiles, kBlock, kSortTile * 12, st>>>(
          (const unsigned long long*)kin, vin, (unsigned long long*)kout, vout, n, shift,
          digit_base, status, tile_ctr);
    else
      onesweep_kernel<unsigned long long, false><<<tiles, kBlock, kSortTile * 12, st>>>(
          (const unsigned long long*)kin, vin, (unsigned long long*)kout, vout, n, shift,
          digit_base, status, tile_ctr);
  }
}

}  // namespace dvl
