// hilbert.cu -- B1: centroid quantisation + 3D Hilbert code (
// readings O2/O3/A1-A3) as a table-driven state machine, fused with the digit histograms
// of the radix sort (B2).
//
// The curve is Skilling's (2004) transpose construction with x-major interleave (reading
// A1).  Instead of running Skilling's per-bit loop (~45 ALU ops per level per cell), the
// library derives a finite-state machine from the construction once on the host:
//   * processing the levels top-down, everything the higher levels do to the lower bits
//     is a signed permutation S of the three axes (the "invert X[0]" and "exchange X[0],
//     X[i]" steps), and the final Gray-code correction is the parity p of the x^y^z bits
//     seen above;
//   * one level maps (S, p, octant) -> (3-bit digit, S', p').
// The reachable (S, p) states are enumerated by BFS; two levels are composed into one
// 64-entry row per state, so a b-bit code costs ceil(b/2) shared-memory lookups.
#include <algorithm>
#include <cstring>
#include <map>
#include <vector>

#include "bsort.cuh"
#include "dvl_common.cuh"
#include "dvl_internal.h"

namespace dvl {

namespace {

// a 3-bit vector: axis 0 (x) in bit 2, axis 1 (y) in bit 1, axis 2 (z) in bit 0
inline int bit_of(int v, int axis) { return (v >> (2 - axis)) & 1; }

inline int swap_axes(int v, int a, int b) {
  int ba = bit_of(v, a), bb = bit_of(v, b);
  v &= ~((1 << (2 - a)) | (1 << (2 - b)));
  return v | (bb << (2 - a)) | (ba << (2 - b));
}

struct State {
  uint8_t map[8];   // y = S(x)
  uint8_t parity;
  bool operator<(const State& o) const {
    int c = memcmp(map, o.map, 8);
    return c != 0 ? c < 0 : parity < o.parity;
  }
};

// One level of the construction applied to state s and input octant x.
void step(const State& s, int x, int* digit, State* next) {
  int y = s.map[x];
  int y0 = bit_of(y, 0), y1 = bit_of(y, 1), y2 = bit_of(y, 2);
  int yi[3] = {y0, y1, y2};
  // the operations of this level on every lower level, in Skilling's order i = 0, 1, 2
  for (int v = 0; v < 8; ++v) {
    int w = s.map[v];
    for (int i = 0; i < 3; ++i) w = yi[i] ? (w ^ 4) : swap_axes(w, 0, i);
    next->map[v] = (uint8_t)w;
  }
  int g0 = y0, g1 = y1 ^ y0, g2 = y2 ^ y1 ^ y0;
  int d = (g0 << 2) | (g1 << 1) | g2;
  if (s.parity) d ^= 7;
  *digit = d;
  next->parity = (uint8_t)(s.parity ^ g2);
}

struct Tables {
  int nstates = 0;
  std::vector<uint16_t> t1;   // nstates x 8:  (next << 3) | digit
  std::vector<uint16_t> t2;   // nstates x 64: (next << 6) | two digits
};

Tables build_tables() {
  Tables T;
  std::map<State, int> id;
  std::vector<State> states;
  State s0;
  for (int v = 0; v < 8; ++v) s0.map[v] = (uint8_t)v;
  s0.parity = 0;
  id[s0] = 0;
  states.push_back(s0);
  std::vector<std::pair<int, int>> edges;  // (next, digit) per (state, octant)
  for (size_t k = 0; k < states.size(); ++k) {
    for (int x = 0; x < 8; ++x) {
      int d;
      State nx;
      step(states[k], x, &d, &nx);
      auto it = id.find(nx);
      int j;
      if (it == id.end()) {
        j = (int)states.size();
        id[nx] = j;
        states.push_back(nx);
      } else {
        j = it->second;
      }
      edges.push_back({j, d});
    }
  }
  T.nstates = (int)states.size();
  T.t1.resize(T.nstates * 8);
  for (int k = 0; k < T.nstates; ++k)
    for (int x = 0; x < 8; ++x) {
      auto e = edges[k * 8 + x];
      T.t1[k * 8 + x] = (uint16_t)((e.first << 3) | e.second);
    }
  T.t2.resize(T.nstates * 64);
  for (int k = 0; k < T.nstates; ++k)
    for (int xh = 0; xh < 8; ++xh)
      for (int xl = 0; xl < 8; ++xl) {
        auto a = edges[k * 8 + xh];
        auto b = edges[a.first * 8 + xl];
        T.t2[k * 64 + xh * 8 + xl] = (uint16_t)((b.first << 6) | (a.second << 3) | b.second);
      }
  return T;
}

const Tables& tables() {
  static Tables T = build_tables();
  return T;
}

}  // namespace

int hilbert_num_states() { return tables().nstates; }

uint64_t hilbert_encode_host(uint32_t x, uint32_t y, uint32_t z, int b) {
  const Tables& T = tables();
  int s = 0;
  uint64_t h = 0;
  int j = b - 1;
  if (b & 1) {
    int oct = (((x >> j) & 1) << 2) | (((y >> j) & 1) << 1) | ((z >> j) & 1);
    uint16_t e = T.t1[s * 8 + oct];
    h = e & 7;
    s = e >> 3;
    --j;
  }
  for (; j >= 1; j -= 2) {
    int oh = (((x >> j) & 1) << 2) | (((y >> j) & 1) << 1) | ((z >> j) & 1);
    int ol = (((x >> (j - 1)) & 1) << 2) | (((y >> (j - 1)) & 1) << 1) | ((z >> (j - 1)) & 1);
    uint16_t e = T.t2[s * 64 + oh * 8 + ol];
    h = (h << 6) | (e & 63);
    s = e >> 6;
  }
  return h;
}

// ----------------------------------------------------------------------- device side
// spread the 2 bits (j, j-1) of x, y, z into the 6-bit index oh*8 + ol
__device__ __forceinline__ int two_levels(uint32_t x, uint32_t y, uint32_t z, int j) {
  uint32_t xb = (x >> (j - 1)) & 3, yb = (y >> (j - 1)) & 3, zb = (z >> (j - 1)) & 3;
  // oh = (x_j, y_j, z_j), ol = (x_{j-1}, y_{j-1}, z_{j-1})
  return (int)(((xb >> 1) << 5) | ((yb >> 1) << 4) | ((zb >> 1) << 3) | ((xb & 1) << 2) |
               ((yb & 1) << 1) | (zb & 1));
}

// the code with the two-level table stored in coordinate-major index order
// (x_j x_{j-1} y_j y_{j-1} z_j z_{j-1}): each step takes 2 bits of x, y and z directly,
// with no bit interleaving; the code accumulates in K (32-bit for 3b <= 32)
template <typename K>
__device__ __forceinline__ K hilbert_code_cm(uint32_t x, uint32_t y, uint32_t z, int b,
                                             const uint16_t* s_t1, const uint16_t* s_t2p) {
  uint32_t s = 0;
  K code = 0;
  int j = b - 1;
  if (b & 1) {
    const uint32_t oct = (((x >> j) & 1u) << 2) | (((y >> j) & 1u) << 1) | ((z >> j) & 1u);
    const uint32_t e = s_t1[oct];
    code = (K)(e & 7u);
    s = e >> 3;
    --j;
  }
  for (; j >= 1; j -= 2) {
    const uint32_t idx = (((x >> (j - 1)) & 3u) << 4) | (((y >> (j - 1)) & 3u) << 2) | ((z >> (j - 1)) & 3u);
    const uint32_t e = s_t2p[s * 64 + idx];
    code = (code << 6) | (K)(e & 63u);
    s = e >> 6;
  }
  return code;
}

// B1 for the bucket sort (3b <= 36, see bsort.cu): four cells per thread with 16-byte
// loads of the AoS corners (3 x uint4 = 4 cells) and one 4-byte load of their levels, the
// four codes stored with one (u32) or two (u64) 16-byte stores, and the bucket counts
// (bucket = code >> lb, an aligned run of 2^lb codes) taken with one returning global
// atomic per bucket per warp (lanes grouped by __match_any_sync: consecutive input cells
// mostly share a bucket).  The value an atomic returns gives each cell a slot inside its
// bucket (any order: the rank pass orders the bucket), stored as a u16 next to the code,
// so the scatter pass needs no atomics.
template <typename K, bool VEC>
__global__ void __launch_bounds__(kBlock)
encode_bucket_kernel(const uint32_t* __restrict__ lower, const uint8_t* __restrict__ level,
                     int64_t n, int b, int lb, const uint16_t* __restrict__ t1g,
                     const uint16_t* __restrict__ t2g, int nstates, K* __restrict__ keys,
                     uint16_t* __restrict__ slot, uint32_t* __restrict__ count) {
  extern __shared__ uint16_t s_tab[];
  uint16_t* s_t1 = s_tab;
  uint16_t* s_t2p = s_tab + nstates * 8;
  for (int i = threadIdx.x; i < nstates * 8; i += kBlock) s_t1[i] = t1g[i];
  for (int i = threadIdx.x; i < nstates * 64; i += kBlock) {
    // coordinate-major index p = x_j x_{j-1} y_j y_{j-1} z_j z_{j-1} <- octant-major o
    const int p = i & 63;
    const int o = (((p >> 5) & 1) << 5) | (((p >> 3) & 1) << 4) | (((p >> 1) & 1) << 3) |
                  (((p >> 4) & 1) << 2) | (((p >> 2) & 1) << 1) | (p & 1);
    s_t2p[i] = t2g[(i & ~63) + o];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t groups = (n + 3) >> 2;
  const int64_t wstride = (int64_t)gridDim.x * (kBlock / 32) * 32;
  for (int64_t g0 = ((int64_t)blockIdx.x * (kBlock / 32) + (threadIdx.x >> 5)) * 32; g0 < groups;
       g0 += wstride) {
    const int64_t g = g0 + lane;
    const int64_t h0 = g * 4;
    uint32_t xs[4] = {0, 0, 0, 0}, ys[4] = {0, 0, 0, 0}, zs[4] = {0, 0, 0, 0}, lv[4] = {0, 0, 0, 0};
    int cnt = 0;
    if (g < groups) {
      cnt = (int)(n - h0 < 4 ? n - h0 : 4);
      if (VEC && cnt == 4) {
        const uint4* l4 = reinterpret_cast<const uint4*>(lower) + 3 * g;
        const uint4 a = l4[0], bq = l4[1], c = l4[2];
        const uint32_t L4 = reinterpret_cast<const uint32_t*>(level)[g];
        xs[0] = a.x; ys[0] = a.y; zs[0] = a.z;
        xs[1] = a.w; ys[1] = bq.x; zs[1] = bq.y;
        xs[2] = bq.z; ys[2] = bq.w; zs[2] = c.x;
        xs[3] = c.y; ys[3] = c.z; zs[3] = c.w;
#pragma unroll
        for (int i = 0; i < 4; ++i) lv[i] = (L4 >> (8 * i)) & 255u;
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const bool ok = i < cnt;
          xs[i] = ok ? lower[3 * (h0 + i)] : 0u;
          ys[i] = ok ? lower[3 * (h0 + i) + 1] : 0u;
          zs[i] = ok ? lower[3 * (h0 + i) + 2] : 0u;
          lv[i] = ok ? level[h0 + i] : 0u;
        }
      }
    }
    K code[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t half = (1u << lv[i]) >> 1;
      code[i] = hilbert_code_cm<K>(xs[i] + half, ys[i] + half, zs[i] + half, b, s_t1, s_t2p);
    }
    if (cnt == 4) {
      if (sizeof(K) == 4) {
        reinterpret_cast<uint4*>(keys)[g] =
            make_uint4((uint32_t)code[0], (uint32_t)code[1], (uint32_t)code[2], (uint32_t)code[3]);
      } else {
        ulonglong2* k2 = reinterpret_cast<ulonglong2*>(keys) + 2 * g;
        k2[0] = make_ulonglong2(code[0], code[1]);
        k2[1] = make_ulonglong2(code[2], code[3]);
      }
    } else {
      for (int i = 0; i < cnt; ++i) keys[h0 + i] = code[i];
    }
    uint32_t sl[4];
    bucket_slots<K>(code, cnt, lb, count, sl);
    store_slots(slot, g, h0, cnt, sl);
  }
}

void launch_encode_bucket(const uint32_t* lower, const uint8_t* level, int64_t n, int b, int lb,
                          int key_bytes, const uint16_t* d_t1, const uint16_t* d_t2, int nstates,
                          void* keys, uint16_t* slot, uint32_t* count, int num_sms, cudaStream_t st) {
  const size_t smem = (size_t)nstates * (8 + 64) * sizeof(uint16_t);
  const bool vec = (reinterpret_cast<uintptr_t>(lower) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(level) & 3) == 0;
  const int64_t warps = ((n + 3) / 4 + 31) / 32;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((warps + 7) / 8, (int64_t)num_sms * 8));
#define EB(K, V)                                                                               \
  encode_bucket_kernel<K, V><<<grid, kBlock, smem, st>>>(lower, level, n, b, lb, d_t1, d_t2,   \
                                                         nstates, (K*)keys, slot, count)
  if (key_bytes == 4) {
    if (vec) EB(uint32_t, true); else EB(uint32_t, false);
  } else {
    if (vec) EB(unsigned long long, true); else EB(unsigned long long, false);
  }
#undef EB
}

template <typename K>
__global__ void __launch_bounds__(kBlock)
encode_hist_kernel(const uint32_t* __restrict__ lower, const uint8_t* __restrict__ level,
                   int64_t n, int b, int passes, const uint16_t* __restrict__ t1g,
                   const uint16_t* __restrict__ t2g, int nstates, K* __restrict__ keys,
                   uint32_t* __restrict__ ids, uint32_t* __restrict__ hist) {
  extern __shared__ uint16_t s_tab[];   // t1 (nstates*8) then t2 (nstates*64)
  __shared__ uint32_t s_hist[8][256];
  uint16_t* s_t1 = s_tab;
  uint16_t* s_t2 = s_tab + nstates * 8;
  for (int i = threadIdx.x; i < nstates * 8; i += kBlock) s_t1[i] = t1g[i];
  for (int i = threadIdx.x; i < nstates * 64; i += kBlock) s_t2[i] = t2g[i];
  for (int i = threadIdx.x; i < passes * 256; i += kBlock) (&s_hist[0][0])[i] = 0;
  __syncthreads();
  for (int64_t h = (int64_t)blockIdx.x * kBlock + threadIdx.x; h < n;
       h += (int64_t)gridDim.x * kBlock) {
    uint32_t half = (1u << level[h]) >> 1;
    uint32_t x = lower[3 * h] + half, y = lower[3 * h + 1] + half, z = lower[3 * h + 2] + half;
    int s = 0;
    uint64_t code = 0;
    int j = b - 1;
    if (b & 1) {
      int oct = (((x >> j) & 1) << 2) | (((y >> j) & 1) << 1) | ((z >> j) & 1);
      uint16_t e = s_t1[s * 8 + oct];
      code = e & 7;
      s = e >> 3;
      --j;
    }
    for (; j >= 1; j -= 2) {
      uint16_t e = s_t2[s * 64 + two_levels(x, y, z, j)];
      code = (code << 6) | (e & 63);
      s = e >> 6;
    }
    keys[h] = (K)code;   // the ids (0..n-1) are implicit in the first sort pass
    for (int p = 0; p < passes; ++p) atomicAdd(&s_hist[p][(code >> (8 * p)) & 255], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * 256; i += kBlock) {
    uint32_t c = (&s_hist[0][0])[i];
    if (c) atomicAdd(hist + i, c);
  }
}

void launch_encode_hist(const uint32_t* lower, const uint8_t* level, int64_t n, int b,
                        int key_bytes, int passes, const uint16_t* d_t1, const uint16_t* d_t2,
                        int nstates, void* keys, uint32_t* ids, uint32_t* hist, int grid,
                        cudaStream_t st) {
  size_t smem = (size_t)nstates * (8 + 64) * sizeof(uint16_t);
  if (key_bytes == 4)
    encode_hist_kernel<uint32_t><<<grid, kBlock, smem, st>>>(
        lower, level, n, b, passes, d_t1, d_t2, nstates, (uint32_t*)keys, ids, hist);
  else
    encode_hist_kernel<unsigned long long><<<grid, kBlock, smem, st>>>(
        lower, level, n, b, passes, d_t1, d_t2, nstates, (unsigned long long*)keys, ids, hist);
}

// Point location (brushing / linking): the cell containing each integer point
// of the logical grid, as its global index in curve order (-1: no cell contains it).  A
// cell of level L covers the aligned 2^L cube, whose points the curve visits as one aligned
// run of 8^L codes, so the point's code h lies in the run of the last cell with key <= h or
// of the next one (whose centroid may come after h in its run): a binary search over the
// sorted keys and two range checks.
template <typename K>
__global__ void __launch_bounds__(kBlock)
locate_kernel(const uint32_t* __restrict__ xyz, int64_t npts, int b,
              const uint16_t* __restrict__ t1g, const uint16_t* __restrict__ t2g, int nstates,
              const K* __restrict__ keys, const uint8_t* __restrict__ level, int64_t n,
              uint64_t cell_offset, int64_t* __restrict__ out, const unsigned long long* roi) {
  extern __shared__ uint16_t s_tab[];
  uint16_t* s_t1 = s_tab;
  uint16_t* s_t2 = s_tab + nstates * 8;
  for (int i = threadIdx.x; i < nstates * 8; i += kBlock) s_t1[i] = t1g[i];
  for (int i = threadIdx.x; i < nstates * 64; i += kBlock) s_t2[i] = t2g[i];
  __syncthreads();
  for (int64_t h = (int64_t)blockIdx.x * kBlock + threadIdx.x; h < npts;
       h += (int64_t)gridDim.x * kBlock) {
    const uint32_t x = xyz[3 * h], y = xyz[3 * h + 1], z = xyz[3 * h + 2];
    int64_t res = -1;
    if (n > 0 && ((x | y | z) >> b) == 0) {
      int s = 0;
      uint64_t code = 0;
      int j = b - 1;
      if (b & 1) {
        int oct = (((x >> j) & 1) << 2) | (((y >> j) & 1) << 1) | ((z >> j) & 1);
        uint16_t e = s_t1[s * 8 + oct];
        code = e & 7;
        s = e >> 3;
        --j;
      }
      for (; j >= 1; j -= 2) {
        uint16_t e = s_t2[s * 64 + two_levels(x, y, z, j)];
        code = (code << 6) | (e & 63);
        s = e >> 6;
      }
      // i = the number of keys <= code, minus 1
      int64_t lo = 0, hi = n;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if ((uint64_t)keys[mid] <= code) lo = mid + 1; else hi = mid;
      }
      for (int64_t c = lo - 1; c <= lo; ++c) {
        if (c < 0 || c >= n) continue;
        const uint64_t len = 1ull << (3 * level[c]);
        const uint64_t start = (uint64_t)keys[c] & ~(len - 1);
        if (code >= start && code - start < len) {
          res = (int64_t)(cell_offset + (uint64_t)c);
          break;
        }
      }
    }
    // roi (brushing): 1 if the containing cell's code lies in [roi[0], roi[1]]
    if (roi) {
      const int64_t c = res - (int64_t)cell_offset;
      res = res >= 0 && (uint64_t)keys[c] >= roi[0] && (uint64_t)keys[c] <= roi[1] ? 1 : 0;
    }
    out[h] = res;
  }
}

void launch_locate(const uint32_t* xyz, int64_t npts, int b, const uint16_t* d_t1,
                   const uint16_t* d_t2, int nstates, const void* keys, int key_bytes,
                   const uint8_t* level, int64_t n, uint64_t cell_offset, int64_t* out,
                   cudaStream_t st, const unsigned long long* roi) {
  const size_t smem = (size_t)nstates * (8 + 64) * sizeof(uint16_t);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((npts + kBlock - 1) / kBlock, 4096));
  if (key_bytes == 4)
    locate_kernel<uint32_t><<<grid, kBlock, smem, st>>>(xyz, npts, b, d_t1, d_t2, nstates,
                                                        (const uint32_t*)keys, level, n,
                                                        cell_offset, out, roi);
  else
    locate_kernel<unsigned long long><<<grid, kBlock, smem, st>>>(
        xyz, npts, b, d_t1, d_t2, nstates, (const unsigned long long*)keys, level, n, cell_offset,
        out, roi);
}

__global__ void iota_kernel(uint32_t* v, int64_t n) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    v[k] = (uint32_t)k;
}

void launch_iota(uint32_t* v, int64_t n, cudaStream_t st) {
  iota_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 4096), 256, 0, st>>>(v, n);
}

void hilbert_tables_host(std::vector<uint16_t>* t1, std::vector<uint16_t>* t2, int* nstates) {
  const Tables& T = tables();
  *t1 = T.t1;
  *t2 = T.t2;
  *nstates = T.nstates;
}

}  // namespace dvl
