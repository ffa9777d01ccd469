// bsort.cuh -- the bucket-slot step shared by the Hilbert encoder (hilbert.cu) and the
// slot kernel over existing codes (bsort.cu): four cells per lane; every cell gets the
// bucket count before it (a slot inside its bucket) from one returning atomic per bucket
// per warp (lanes grouped with __match_any_sync).
#pragma once

#include <stdint.h>

namespace dvl {

template <typename K>
__device__ __forceinline__ void bucket_slots(const K (&code)[4], int cnt, int lb, uint32_t* count,
                                             uint32_t (&sl)[4]) {
  const uint32_t lt = (1u << (threadIdx.x & 31)) - 1u;
  const uint32_t b0 = cnt ? (uint32_t)(code[0] >> lb) : 0xffffffffu;
  const bool same = cnt == 4 && (uint32_t)(code[1] >> lb) == b0 && (uint32_t)(code[2] >> lb) == b0 &&
                    (uint32_t)(code[3] >> lb) == b0;
  if (__all_sync(0xffffffffu, same || cnt == 0)) {   // every lane's four cells share a bucket
    const uint32_t peers = __match_any_sync(0xffffffffu, b0);
    uint32_t base = 0;
    if (b0 != 0xffffffffu && (peers & lt) == 0) base = atomicAdd(count + b0, 4u * __popc(peers));
    base = __shfl_sync(0xffffffffu, base, __ffs(peers) - 1) + 4u * __popc(peers & lt);
#pragma unroll
    for (int i = 0; i < 4; ++i) sl[i] = base + i;
  } else {
    uint32_t bkt[4], peers[4], base[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      bkt[i] = i < cnt ? (uint32_t)(code[i] >> lb) : 0xffffffffu;
      peers[i] = __match_any_sync(0xffffffffu, bkt[i]);
      base[i] = 0;
      if (bkt[i] != 0xffffffffu && (peers[i] & lt) == 0)
        base[i] = atomicAdd(count + bkt[i], (uint32_t)__popc(peers[i]));
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
      sl[i] = __shfl_sync(0xffffffffu, base[i], __ffs(peers[i]) - 1) + __popc(peers[i] & lt);
  }
}

// the four slots as 16-bit values (a bucket holds at most 2^12 distinct codes)
__device__ __forceinline__ void store_slots(uint16_t* slot, int64_t g, int64_t h0, int cnt,
                                            const uint32_t (&sl)[4]) {
  if (cnt == 4) {
    reinterpret_cast<uint2*>(slot)[g] = make_uint2((sl[0] & 0xffffu) | (sl[1] << 16),
                                                   (sl[2] & 0xffffu) | (sl[3] << 16));
  } else {
    for (int i = 0; i < cnt; ++i) slot[h0 + i] = (uint16_t)sl[i];
  }
}

}  // namespace dvl
