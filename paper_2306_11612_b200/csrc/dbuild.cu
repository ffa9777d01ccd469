// dbuild.cu -- the device steps and the host splitter rule of the distributed build
// ("Build": a Hilbert-key sample sort; orchestrated by dvl_build in api.cu when
// the context has a communicator):
//   * regular samples of the rank's locally sorted codes;
//   * splitters: the G-1 global quantiles of the weighted union of all ranks' samples
//     (host, identical on every rank);
//   * the send ranges: lower_bound of every splitter in the local sorted run;
//   * global input ids of the local cells (input offset of the rank + local id);
//   * the final gather of the received ids through the combined order.
#include <algorithm>
#include <vector>

#include "dvl_common.cuh"
#include "dvl_internal.h"

namespace dvl {

template <typename K>
__global__ void sample_keys_kernel(const K* __restrict__ keys, int64_t n, int S,
                                   unsigned long long* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= S) return;
  const int64_t s = n < S ? n : S;   // samples taken (all cells when n < S)
  out[i] = i < s ? (unsigned long long)keys[((int64_t)i * n) / s] : ~0ull;
}

template <typename K>
__global__ void lower_bounds_kernel(const K* __restrict__ keys, int64_t n,
                                    const unsigned long long* __restrict__ spl, int k,
                                    unsigned long long* __restrict__ out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= k) return;
  const unsigned long long v = spl[j];
  int64_t lo = 0, hi = n;   // first position with key >= v
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((unsigned long long)keys[mid] < v) lo = mid + 1; else hi = mid;
  }
  out[j] = (unsigned long long)lo;
}

__global__ void offset_ids_kernel(const uint32_t* __restrict__ perm, int64_t n, uint64_t off,
                                  unsigned long long* __restrict__ out) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    out[k] = off + perm[k];
}

__global__ void gather_u64_kernel(const unsigned long long* __restrict__ src,
                                  const uint32_t* __restrict__ idx, int64_t n,
                                  unsigned long long* __restrict__ out) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t i = idx[k];
    out[k] = i < n ? src[i] : 0ull;   // out of range only with duplicate codes (OVERLAP)
  }
}

static int grid_for(int64_t n, int num_sms) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)num_sms * 8));
}

void launch_sample_keys(const void* keys, int key_bytes, int64_t n, int S, unsigned long long* out,
                        cudaStream_t st) {
  const int g = (S + 255) / 256;
  if (key_bytes == 4)
    sample_keys_kernel<uint32_t><<<g, 256, 0, st>>>((const uint32_t*)keys, n, S, out);
  else
    sample_keys_kernel<unsigned long long><<<g, 256, 0, st>>>((const unsigned long long*)keys, n, S, out);
}

void launch_lower_bounds(const void* keys, int key_bytes, int64_t n, const unsigned long long* spl,
                         int k, unsigned long long* out, cudaStream_t st) {
  const int g = std::max(1, (k + 127) / 128);
  if (key_bytes == 4)
    lower_bounds_kernel<uint32_t><<<g, 128, 0, st>>>((const uint32_t*)keys, n, spl, k, out);
  else
    lower_bounds_kernel<unsigned long long><<<g, 128, 0, st>>>((const unsigned long long*)keys, n, spl, k, out);
}

void launch_offset_ids(const uint32_t* perm, int64_t n, uint64_t off, unsigned long long* out,
                       int num_sms, cudaStream_t st) {
  offset_ids_kernel<<<grid_for(n, num_sms), 256, 0, st>>>(perm, n, off, out);
}

void launch_gather_u64(const unsigned long long* src, const uint32_t* idx, int64_t n,
                       unsigned long long* out, int num_sms, cudaStream_t st) {
  gather_u64_kernel<<<grid_for(n, num_sms), 256, 0, st>>>(src, idx, n, out);
}

// Splitters of the sample sort (host; every rank computes the same from the same input).
// Rank p took s_p = min(S, n_p) regularly spaced samples of its sorted run (sample j at
// position floor(j n_p / s_p)), so sample j stands for the floor((j+1) n_p / s_p) -
// floor(j n_p / s_p) cells that follow it.  Sorting all samples by code and accumulating
// these weights approximates the global rank of every sample; splitter k (k = 1..G-1) is
// the first sample whose preceding weight reaches k n / G.  Ranks holding no cells
// contribute no samples (their padding is ~0), so an uneven input cannot produce empty
// splitters.  Returns false if the splitters cannot be strictly increasing (fewer distinct
// samples than ranks).
bool select_splitters(const uint64_t* samples, const uint64_t* counts, int G, int S,
                      uint64_t* out) {
  std::vector<std::pair<uint64_t, uint64_t>> items;   // (code, weight)
  uint64_t n = 0;
  for (int p = 0; p < G; ++p) {
    const uint64_t np = counts[p];
    n += np;
    const uint64_t s = std::min<uint64_t>((uint64_t)S, np);
    for (uint64_t j = 0; j < s; ++j)
      items.emplace_back(samples[(size_t)p * S + j], ((j + 1) * np) / s - (j * np) / s);
  }
  std::sort(items.begin(), items.end());
  uint64_t before = 0;
  size_t i = 0;
  for (int k = 1; k < G; ++k) {
    const unsigned __int128 target = (unsigned __int128)k * n / G;
    while (i < items.size() && before < target) before += items[i++].second;
    if (i >= items.size()) return false;
    out[k - 1] = items[i].first;
    if (k > 1 && out[k - 1] <= out[k - 2]) return false;
  }
  return true;
}

}  // namespace dvl
