// bsort.cu -- B2 for 3b <= 36 (every BASELINE config): a two-pass bucket sort of the
// (Hilbert code, cell id) pairs that uses what the method guarantees about its keys.
//
// The order is established once and valid cells have pairwise distinct codes
// (reading A4: a duplicate means overlapping cells, DVL_E_OVERLAP).  So:
//   * bucket = code >> lb, an aligned run of 2^lb codes (lb = 12: one 16^3 dyadic block);
//     B1 counts the cells per bucket with returning atomics and keeps each cell's slot in
//     its bucket (hilbert.cu: encode_bucket_kernel);
//   * scan: exclusive prefix of the bucket counts -> each bucket's first output slot;
//   * scatter (pass A): every cell to start[bucket] + slot, writing (code, id);
//   * rank (pass B): a warp per bucket; the codes of a bucket differ in their low lb bits
//     only and are distinct, so a code's rank inside its bucket is the number of set bits
//     below it in a 2^lb-bit occupancy bitmap (shared memory): set the bits, a warp prefix
//     of the word popcounts, then rank = prefix[word] + popc(word & below).  A bit found
//     already set is a duplicate code: the error word gets kErrOverlap.
// Two passes over (code, id) instead of ceil(3b / 8) LSD passes, and the second one reads
// and writes each bucket's contiguous range.  The result does not depend on the order in
// which the scatter's atomics land (every bucket is fully ranked), so it is deterministic
// and equal to the LSD sort's.  For 3b > 36 the bucket count 2^(3b-12) is too large and
// the library uses the onesweep LSD sort (sort.cu).
#include <algorithm>

#include "bsort.cuh"
#include "dvl_common.cuh"
#include "dvl_internal.h"

namespace dvl {

constexpr int kScanItems = 16;                       // counts per thread
constexpr int kScanTile = kBlock * kScanItems;       // 4096 counts per block

// ---------------------------------------------------------------- bucket offsets (scan)
__global__ void __launch_bounds__(kBlock)
scan_reduce_kernel(const uint32_t* __restrict__ cnt, int64_t nb, uint32_t* __restrict__ bsum) {
  const int64_t base = (int64_t)blockIdx.x * kScanTile;
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const int64_t k = base + (int64_t)i * kBlock + threadIdx.x;
    if (k < nb) s += cnt[k];
  }
  __shared__ uint32_t ws[kBlock / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < kBlock / 32; ++w) t += ws[w];
    bsum[blockIdx.x] = t;
  }
}

// exclusive scan of the block sums in place (one block; nblk <= 2^24 / 4096)
__global__ void __launch_bounds__(1024) scan_top_kernel(uint32_t* bsum, int nblk) {
  __shared__ uint32_t ws[32];
  __shared__ uint32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int base = 0; base < nblk; base += 1024) {
    const int k = base + threadIdx.x;
    const uint32_t v = k < nblk ? bsum[k] : 0u;
    uint32_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += u;
    }
    if (lane == 31) ws[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      uint32_t w = ws[lane];
      uint32_t wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += u;
      }
      ws[lane] = wi - w;
    }
    __syncthreads();
    const uint32_t c0 = carry;
    if (k < nblk) bsum[k] = c0 + ws[warp] + inc - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry = c0 + ws[warp] + inc;
    __syncthreads();
  }
}

// each block rescans its 4096 counts from its block offset: start[k] (exclusive);
// start[nb] = n.  A bucket holding more cells than it has codes (2^lb) has duplicates.
__global__ void __launch_bounds__(kBlock)
scan_down_kernel(const uint32_t* __restrict__ cnt, int64_t nb, const uint32_t* __restrict__ bsum,
                 uint32_t* __restrict__ start, uint32_t total, uint32_t cap, uint32_t* err) {
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  uint32_t v[kScanItems];
  uint32_t s = 0;
  bool over = false;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    v[i] = base + i < nb ? cnt[base + i] : 0u;
    s += v[i];
    over |= v[i] > cap;   // more cells than codes in the bucket: duplicates
  }
  if (over) atomicOr(err, kErrOverlap);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t inc = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += u;
  }
  __shared__ uint32_t ws[kBlock / 32];
  if (lane == 31) ws[warp] = inc;
  __syncthreads();
  uint32_t wpre = 0;
  for (int w = 0; w < warp; ++w) wpre += ws[w];
  uint32_t run = bsum[blockIdx.x] + wpre + inc - s;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    if (base + i < nb) start[base + i] = run;
    run += v[i];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) start[nb] = total;
}

// ---------------------------------------------------- slots of codes already computed
// (the distributed build's received runs): the B1 counting step without the encode
template <typename K, bool VEC>
__global__ void __launch_bounds__(kBlock)
bucket_slot_kernel(const K* __restrict__ keys, int64_t n, int lb, uint16_t* __restrict__ slot,
                   uint32_t* __restrict__ count) {
  const int lane = threadIdx.x & 31;
  const int64_t groups = (n + 3) >> 2;
  const int64_t wstride = (int64_t)gridDim.x * kBlock;
  for (int64_t g0 = (int64_t)blockIdx.x * kBlock + (threadIdx.x & ~31); g0 < groups; g0 += wstride) {
    const int64_t g = g0 + lane;
    const int64_t h0 = g * 4;
    const int cnt = g < groups ? (int)(n - h0 < 4 ? n - h0 : 4) : 0;
    K code[4] = {0, 0, 0, 0};
    if (VEC && cnt == 4) {
      if (sizeof(K) == 4) {
        const uint4 q = reinterpret_cast<const uint4*>(keys)[g];
        code[0] = q.x; code[1] = q.y; code[2] = q.z; code[3] = q.w;
      } else {
        const ulonglong2* k2 = reinterpret_cast<const ulonglong2*>(keys) + 2 * g;
        const ulonglong2 a = k2[0], c = k2[1];
        code[0] = (K)a.x; code[1] = (K)a.y; code[2] = (K)c.x; code[3] = (K)c.y;
      }
    } else {
      for (int i = 0; i < cnt; ++i) code[i] = keys[h0 + i];
    }
    uint32_t sl[4];
    bucket_slots<K>(code, cnt, lb, count, sl);
    if (cnt) store_slots(slot, g, h0, cnt, sl);
  }
}

void launch_bucket_slot(const void* keys, int key_bytes, int64_t n, int lb, uint16_t* slot,
                        uint32_t* count, int num_sms, cudaStream_t st) {
  const int64_t groups = (n + 3) / 4;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((groups + kBlock - 1) / kBlock,
                                                                (int64_t)num_sms * 8));
  const bool vec = (reinterpret_cast<uintptr_t>(keys) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(slot) & 7) == 0;
  if (key_bytes == 4) {
    if (vec) bucket_slot_kernel<uint32_t, true><<<grid, kBlock, 0, st>>>((const uint32_t*)keys, n, lb, slot, count);
    else bucket_slot_kernel<uint32_t, false><<<grid, kBlock, 0, st>>>((const uint32_t*)keys, n, lb, slot, count);
  } else {
    using U = unsigned long long;
    if (vec) bucket_slot_kernel<U, true><<<grid, kBlock, 0, st>>>((const U*)keys, n, lb, slot, count);
    else bucket_slot_kernel<U, false><<<grid, kBlock, 0, st>>>((const U*)keys, n, lb, slot, count);
  }
}

// ------------------------------------------------------------------- pass A: scatter
// every cell to start[bucket] + its slot from B1: a streaming pass with no atomics (a slot
// past the bucket's end -- only possible with more than 65536 duplicate codes -- is an
// overlap and is dropped)
constexpr int kScatGP = 2;   // groups of 4 cells per lane and iteration (8 cells)

template <typename K, bool VEC>
__global__ void __launch_bounds__(kBlock)
bucket_scatter_kernel(const K* __restrict__ keys, const uint16_t* __restrict__ slot, int64_t n,
                      int lb, const uint32_t* __restrict__ start, K* __restrict__ kout,
                      uint32_t* __restrict__ vout, uint32_t* err) {
  // each lane takes kScatGP groups of 4 cells per iteration (all their loads issued before
  // the bucket-start lookups, all those before the stores); the warp's destinations are
  // staged in shared memory and stored transposed (lane l writes cells l, l + 32, ...):
  // consecutive cells mostly go to consecutive slots, so each store instruction writes a
  // few whole sectors instead of 32 scattered pieces
  constexpr int WC = 128 * kScatGP;   // cells per warp and iteration
  __shared__ K s_k[kBlock / 32][WC];
  __shared__ uint32_t s_p[kBlock / 32][WC];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t groups = (n + 3) >> 2;
  bool bad = false;
  for (int64_t g0 = ((int64_t)blockIdx.x * (kBlock / 32) + warp) * (32 * kScatGP); g0 < groups;
       g0 += (int64_t)gridDim.x * (kBlock / 32) * (32 * kScatGP)) {
    K code[kScatGP][4];
    uint32_t sl[kScatGP][4];
    int cnt[kScatGP];
#pragma unroll
    for (int j = 0; j < kScatGP; ++j) {
      const int64_t g = g0 + 32 * j + lane;
      const int64_t h0 = g * 4;
      cnt[j] = g < groups ? (int)(n - h0 < 4 ? n - h0 : 4) : 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        code[j][i] = 0;
        sl[j][i] = 0;
      }
      if (VEC && cnt[j] == 4) {
        if (sizeof(K) == 4) {
          const uint4 q = reinterpret_cast<const uint4*>(keys)[g];
          code[j][0] = q.x; code[j][1] = q.y; code[j][2] = q.z; code[j][3] = q.w;
        } else {
          const ulonglong2* k2 = reinterpret_cast<const ulonglong2*>(keys) + 2 * g;
          const ulonglong2 a = k2[0], c = k2[1];
          code[j][0] = (K)a.x; code[j][1] = (K)a.y; code[j][2] = (K)c.x; code[j][3] = (K)c.y;
        }
        const uint2 s2 = reinterpret_cast<const uint2*>(slot)[g];
        sl[j][0] = s2.x & 0xffffu; sl[j][1] = s2.x >> 16; sl[j][2] = s2.y & 0xffffu; sl[j][3] = s2.y >> 16;
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (i < cnt[j]) {
            code[j][i] = keys[h0 + i];
            sl[j][i] = slot[h0 + i];
          }
        }
      }
    }
    uint32_t pos[kScatGP][4], lim[kScatGP][4];
#pragma unroll
    for (int j = 0; j < kScatGP; ++j)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t bkt = (uint32_t)(code[j][i] >> lb);
        pos[j][i] = i < cnt[j] ? start[bkt] + sl[j][i] : 0u;
        lim[j][i] = i < cnt[j] ? start[bkt + 1] : 0u;
      }
#pragma unroll
    for (int j = 0; j < kScatGP; ++j)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const bool ok = i < cnt[j] && pos[j][i] < lim[j][i];
        bad |= i < cnt[j] && !ok;
        s_k[warp][128 * j + 4 * lane + i] = code[j][i];
        s_p[warp][128 * j + 4 * lane + i] = ok ? pos[j][i] : 0xffffffffu;
      }
    __syncwarp();
    const int64_t c0 = 4 * g0;   // the warp's first cell
#pragma unroll
    for (int i = 0; i < 4 * kScatGP; ++i) {
      const int c = 32 * i + lane;
      const uint32_t ps = s_p[warp][c];
      if (ps != 0xffffffffu) {
        kout[ps] = s_k[warp][c];
        vout[ps] = (uint32_t)(c0 + c);
      }
    }
    __syncwarp();
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(err, kErrOverlap);
}

// ---------------------------------------------------------------------- pass B: rank
constexpr int kRankWarps = 8;
constexpr int kRankR = 8;            // codes per lane held in registers (256 per warp batch)
constexpr int kRankChunkMax = 4096;  // cells per work grab (at most)

template <typename K>
__global__ void __launch_bounds__(kRankWarps * 32)
bucket_rank_kernel(const K* __restrict__ kin, const uint32_t* __restrict__ vin,
                   const uint32_t* __restrict__ start, int64_t nb, int lb, uint32_t chunk_cells,
                   K* __restrict__ kout, uint32_t* __restrict__ vout, uint32_t* work, uint32_t* err) {
  __shared__ uint32_t s_bm[kRankWarps][128];
  __shared__ uint32_t s_pre[kRankWarps][128];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t* bm = s_bm[warp];
  uint32_t* pre = s_pre[warp];
#pragma unroll
  for (int i = 0; i < 4; ++i) bm[4 * lane + i] = 0u;
  __syncwarp();
  const uint32_t lowmask = (uint32_t)((1ull << lb) - 1ull);
  bool dup = false;
  const uint32_t ntot = start[nb];
  const uint32_t nchunks = (ntot + chunk_cells - 1) / chunk_cells;
  int64_t blo = 0, bhi = 0, bk0 = 0;
  for (;;) {
    if (bk0 >= bhi) {
      // the next chunk of about chunk_cells cells: the buckets whose first slot lies in
      // [c chunk_cells, (c + 1) chunk_cells), found by binary searches over the bucket
      // starts (lane 0: the first bucket, lane 1: the end), so every grab is about equal work
      uint32_t c = 0;
      if (lane == 0) c = atomicAdd(work, 1u);
      c = __shfl_sync(0xffffffffu, c, 0);
      if (c >= nchunks) break;
      int64_t r = 0;
      if (lane < 2) {
        const uint32_t key = (c + (uint32_t)lane) * chunk_cells;
        int64_t lo = 0, hi = nb;   // first bucket with start >= key
        if (lane == 1 && c + 1 >= nchunks) {
          lo = nb;
        } else {
          while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (start[mid] < key) lo = mid + 1; else hi = mid;
          }
        }
        r = lo;
      }
      blo = __shfl_sync(0xffffffffu, r, 0);
      bhi = __shfl_sync(0xffffffffu, r, 1);
      bk0 = blo;
      if (blo >= bhi) continue;
    }
    const int64_t bk = bk0 + lane;
    bk0 += 32;
    uint32_t s = 0, e = 0;
    if (bk < bhi) {
      s = start[bk];
      e = start[bk + 1];
    }
    // single-cell buckets (most of them when coarse cells stay unrefined): copied by their
    // own lane, all at once
    if (e - s == 1) {
      kout[s] = kin[s];
      vout[s] = vin[s];
    }
    uint32_t todo = __ballot_sync(0xffffffffu, e > s + 1);
    while (todo) {
      const int j = __ffs(todo) - 1;
      todo &= todo - 1;
      const uint32_t S = __shfl_sync(0xffffffffu, s, j);
      const uint32_t C = __shfl_sync(0xffffffffu, e - s, j);
      if (C <= 32) {
        // rank by comparison with the other codes of the bucket (one per lane)
        const bool ok = (uint32_t)lane < C;
        const K k = ok ? kin[S + lane] : (K)0;
        const uint32_t v = ok ? vin[S + lane] : 0u;
        uint32_t r = 0;
        for (uint32_t q = 0; q < C; ++q) {
          const K kq = __shfl_sync(0xffffffffu, k, (int)q);
          r += kq < k ? 1u : 0u;
          dup |= ok && kq == k && q != (uint32_t)lane;
        }
        if (ok) {
          kout[S + r] = k;
          vout[S + r] = v;
        }
      } else {
        // occupancy bitmap of the low lb bits in batches of 256 codes (8 independent loads
        // per lane in flight), then a warp prefix of the word popcounts
        K kr[kRankR];
        uint32_t vr[kRankR];
        for (uint32_t b0 = 0; b0 < C; b0 += 32 * kRankR) {
#pragma unroll
          for (int r = 0; r < kRankR; ++r) {
            const uint32_t i = b0 + r * 32 + lane;
            kr[r] = i < C ? kin[S + i] : (K)0;
          }
#pragma unroll
          for (int r = 0; r < kRankR; ++r) {
            const uint32_t i = b0 + r * 32 + lane;
            if (i < C) {
              const uint32_t lo = (uint32_t)kr[r] & lowmask;
              const uint32_t bit = 1u << (lo & 31);
              const uint32_t old = atomicOr(&bm[lo >> 5], bit);
              dup |= (old & bit) != 0;
            }
          }
        }
        __syncwarp();
        uint32_t c[4], t = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          c[i] = __popc(bm[4 * lane + i]);
          t += c[i];
        }
        uint32_t inc = t;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
          if (lane >= o) inc += u;
        }
        uint32_t run = inc - t;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          pre[4 * lane + i] = run;
          run += c[i];
        }
        __syncwarp();
        for (uint32_t b0 = 0; b0 < C; b0 += 32 * kRankR) {
          if (C > 32 * kRankR) {   // the batch's codes are no longer in registers
#pragma unroll
            for (int r = 0; r < kRankR; ++r) {
              const uint32_t i = b0 + r * 32 + lane;
              kr[r] = i < C ? kin[S + i] : (K)0;
            }
          }
#pragma unroll
          for (int r = 0; r < kRankR; ++r) {
            const uint32_t i = b0 + r * 32 + lane;
            vr[r] = i < C ? vin[S + i] : 0u;
          }
#pragma unroll
          for (int r = 0; r < kRankR; ++r) {
            const uint32_t i = b0 + r * 32 + lane;
            if (i < C) {
              const uint32_t lo = (uint32_t)kr[r] & lowmask;
              const uint32_t w = lo >> 5;
              const uint32_t rk = pre[w] + __popc(bm[w] & ((1u << (lo & 31)) - 1u));
              kout[S + rk] = kr[r];
              vout[S + rk] = vr[r];
            }
          }
        }
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 4; ++i) bm[4 * lane + i] = 0u;
        __syncwarp();
      }
    }
  }
  if (__any_sync(0xffffffffu, dup) && lane == 0) atomicOr(err, kErrOverlap);
}

// ---------------------------------------------------------------------------- host
int64_t bucket_count(int b, int* lb) {
  const int bits = 3 * b;
  *lb = std::min(12, bits);
  return 1ll << (bits - *lb);
}

void launch_bucket_scan(const uint32_t* cnt, int64_t nb, int lb, uint32_t* bsum, uint32_t* start,
                        uint32_t total, uint32_t* err, cudaStream_t st) {
  const int nblk = (int)((nb + kScanTile - 1) / kScanTile);
  scan_reduce_kernel<<<nblk, kBlock, 0, st>>>(cnt, nb, bsum);
  scan_top_kernel<<<1, 1024, 0, st>>>(bsum, nblk);
  scan_down_kernel<<<nblk, kBlock, 0, st>>>(cnt, nb, bsum, start, total, 1u << lb, err);
}

void launch_bucket_sort(const void* keys, const uint16_t* slot, int key_bytes, int64_t n, int lb,
                        int64_t nb, const uint32_t* start, void* kA, uint32_t* vA, void* kB,
                        uint32_t* vB, uint32_t* work, uint32_t* err, int num_sms, cudaStream_t st) {
  const int64_t groups = (n + 3) / 4;
  const int gA = (int)std::max<int64_t>(1, std::min<int64_t>((groups + kBlock * kScatGP - 1) / (kBlock * kScatGP),
                                                             (int64_t)num_sms * 8));
  const bool vec = (reinterpret_cast<uintptr_t>(keys) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(slot) & 7) == 0;
  const int gB = num_sms * (2048 / (kRankWarps * 32));
  // about four grabs per warp, 256 .. 4096 cells each
  const uint32_t chunk = (uint32_t)std::max<int64_t>(
      256, std::min<int64_t>(kRankChunkMax, n / ((int64_t)gB * kRankWarps * 4)));

  if (key_bytes == 4) {
    if (vec)
      bucket_scatter_kernel<uint32_t, true><<<gA, kBlock, 0, st>>>(
          (const uint32_t*)keys, slot, n, lb, start, (uint32_t*)kA, vA, err);
    else
      bucket_scatter_kernel<uint32_t, false><<<gA, kBlock, 0, st>>>(
          (const uint32_t*)keys, slot, n, lb, start, (uint32_t*)kA, vA, err);
    bucket_rank_kernel<uint32_t><<<gB, kRankWarps * 32, 0, st>>>(
        (const uint32_t*)kA, vA, start, nb, lb, chunk, (uint32_t*)kB, vB, work, err);
  } else {
    using U = unsigned long long;
    if (vec)
      bucket_scatter_kernel<U, true><<<gA, kBlock, 0, st>>>((const U*)keys, slot, n, lb, start, (U*)kA, vA, err);
    else
      bucket_scatter_kernel<U, false><<<gA, kBlock, 0, st>>>((const U*)keys, slot, n, lb, start, (U*)kA, vA, err);
    bucket_rank_kernel<U><<<gB, kRankWarps * 32, 0, st>>>((const U*)kA, vA, start, nb, lb, chunk,
                                                          (U*)kB, vB, work, err);
  }
}

}  // namespace dvl
