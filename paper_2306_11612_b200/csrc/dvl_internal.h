// dvl_internal.h -- host-side declarations shared by the library's translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "dvl.h"

namespace dvl {

struct UpdParams;
struct Acc;

// hilbert.cu
int hilbert_num_states();
uint64_t hilbert_encode_host(uint32_t x, uint32_t y, uint32_t z, int b);
void hilbert_tables_host(std::vector<uint16_t>* t1, std::vector<uint16_t>* t2, int* nstates);
void launch_iota(uint32_t* v, int64_t n, cudaStream_t st);
void launch_encode_hist(const uint32_t* lower, const uint8_t* level, int64_t n, int b,
                        int key_bytes, int passes, const uint16_t* d_t1, const uint16_t* d_t2,
                        int nstates, void* keys, uint32_t* ids, uint32_t* hist, int grid,
                        cudaStream_t st);

void launch_encode_bucket(const uint32_t* lower, const uint8_t* level, int64_t n, int b, int lb,
                          int key_bytes, const uint16_t* d_t1, const uint16_t* d_t2, int nstates,
                          void* keys, uint16_t* slot, uint32_t* count, int num_sms, cudaStream_t st);

// bsort.cu (3b <= 36)
int64_t bucket_count(int b, int* lb);
void launch_bucket_scan(const uint32_t* cnt, int64_t nb, int lb, uint32_t* bsum, uint32_t* start,
                        uint32_t total, uint32_t* err, cudaStream_t st);
void launch_bucket_sort(const void* keys, const uint16_t* slot, int key_bytes, int64_t n, int lb,
                        int64_t nb, const uint32_t* start, void* kA, uint32_t* vA, void* kB,
                        uint32_t* vB, uint32_t* work, uint32_t* err, int num_sms, cudaStream_t st);

void launch_bucket_slot(const void* keys, int key_bytes, int64_t n, int lb, uint16_t* slot,
                        uint32_t* count, int num_sms, cudaStream_t st);

// sort.cu
cudaError_t prepare_onesweep();
void launch_key_hist(const void* keys, int key_bytes, int64_t n, int passes, uint32_t* hist,
                     int num_sms, cudaStream_t st);
void launch_hist_scan(const uint32_t* hist, uint32_t* base, int passes, cudaStream_t st);
void launch_onesweep(const void* kin, const uint32_t* vin, void* kout, uint32_t* vout, int64_t n,
                     int key_bytes, int shift, const uint32_t* digit_base, uint32_t* status,
                     uint32_t* tile_ctr, cudaStream_t st);

// build.cu
struct IngestOut {                 // device-side results of the ingest reduction
  unsigned long long extent;      // max(lower + 2^L)
  uint32_t lmax;
  uint32_t err;
  uint32_t vmin[64];              // ordered-int encoded floats (finite values only)
  uint32_t vmax[64];
  uint32_t any[64];               // 1 if the member has a finite value
};
void launch_ingest_geom(const uint32_t* lower, const uint8_t* level, int64_t n, IngestOut* out,
                        int num_sms, cudaStream_t st);
void launch_gather_validate4(const void* keys, int key_bytes, const uint32_t* perm,
                             const uint8_t* level_in, const float* const* scal_in, int64_t n,
                             int M, int64_t n_pad, uint8_t* level_s, float* scal_s, uint32_t* err,
                             IngestOut* ranges, int num_sms, cudaStream_t st);
void launch_widen(const void* keys, int key_bytes, const uint32_t* perm, int64_t n,
                  uint64_t* codes_out, uint64_t* ids_out, cudaStream_t st);
float ordered_to_float(uint32_t u);

// update.cu
void launch_tf_prepare(const float* rgba_in, int N, float4* rgba_out, float2* tab_out,
                       cudaStream_t st);
void launch_tf_prologue(const float* stage, int member, int mode, int M, int N, float4* rgba_all,
                        float2* tab_all, const float* vmin, const float* vmax, const float* lo,
                        const float* inv, float* maxv, unsigned long long* zero, int zero_words,
                        cudaStream_t st);
void launch_maxv_approx(int mode, int M, int N, const float2* tab, const float* vmin,
                        const float* vmax, const float* lo, const float* inv, float* maxv,
                        cudaStream_t st);
void launch_maxv_exact(const UpdParams& p, float* maxv, int grid, cudaStream_t st);
void launch_weights_scan(int items, bool smem_tab, bool export_q, const UpdParams& p,
                         unsigned long long* status, uint32_t* ctr,
                         unsigned long long* tile_prefix, unsigned long long* qtot,
                         unsigned long long* q_out, int tiles, cudaStream_t st);
void launch_bin_reduce(int items, bool smem_tab, const UpdParams& p,
                       const unsigned long long* tile_prefix, const unsigned long long* qtot,
                       uint32_t W, const Acc& acc, uint64_t cell_offset, uint32_t* err, int tiles,
                       cudaStream_t st);

// shard.cu
void launch_shard_offsets(const unsigned long long* totals, int nshards, int shard,
                          unsigned long long* offset, unsigned long long* qtot, cudaStream_t st);
void launch_acc_export(const Acc& acc, uint32_t W, int M, long long* out, cudaStream_t st);
void launch_epilogue_merged(const long long* merged, uint32_t W, int M, int N, const float4* rgba,
                            dvl_vertex* out, unsigned long long* bin_lo, unsigned long long* bin_hi,
                            cudaStream_t st);
// err_host (device alias of mapped host memory, or nullptr): receives the error word
void launch_epilogue(const Acc& acc, uint32_t W, int M, int N, const float4* rgba,
                     dvl_vertex* out, unsigned long long* bin_lo, unsigned long long* bin_hi,
                     const uint32_t* err, uint32_t* err_host, cudaStream_t st);
void launch_acc_init(const Acc& acc, uint32_t W, int M, cudaStream_t st);
cudaError_t prepare_update_kernels();

// update_tma.cu
struct TmaPlan;
cudaError_t prepare_tma_kernels();
int tma_items_for(int M);
size_t tma_smem(const TmaPlan& plan);
cudaError_t debug_stats(unsigned long long* out8, bool reset);
cudaError_t debug_p1(unsigned long long* out);
int tma_blocks_per_sm(int M, bool smem_tab, const TmaPlan& plan, int pass);
int tma_blocks_per_sm_cache(int M, const TmaPlan& plan);
int tma_tile2_cells(int M);
int tma_pass2_ctas_per_sm(int M);
int tma_warp_tile_cells();
// cmode: 0 every member, 1 edited member + edit cache, 2 every member + write the cache
void launch_weights_reduce_tma(bool smem_tab, const UpdParams& p, const TmaPlan& plan, int grid,
                               unsigned long long* chunk_status, uint32_t* ctr,
                               unsigned long long* chunk_prefix, unsigned long long* qtot,
                               unsigned long long* meta, unsigned long long* meta2, int cmode,
                               cudaStream_t st);
void launch_locate(const uint32_t* xyz, int64_t npts, int b, const uint16_t* d_t1,
                   const uint16_t* d_t2, int nstates, const void* keys, int key_bytes,
                   const uint8_t* level, int64_t n, uint64_t cell_offset, int64_t* out,
                   cudaStream_t st, const unsigned long long* roi = nullptr);
// dbuild.cu: the distributed build's device steps and splitter rule
void launch_sample_keys(const void* keys, int key_bytes, int64_t n, int S, unsigned long long* out,
                        cudaStream_t st);
void launch_lower_bounds(const void* keys, int key_bytes, int64_t n, const unsigned long long* spl,
                         int k, unsigned long long* out, cudaStream_t st);
void launch_offset_ids(const uint32_t* perm, int64_t n, uint64_t off, unsigned long long* out,
                       int num_sms, cudaStream_t st);
void launch_gather_u64(const unsigned long long* src, const uint32_t* idx, int64_t n,
                       unsigned long long* out, int num_sms, cudaStream_t st);
bool select_splitters(const uint64_t* samples, const uint64_t* counts, int G, int S, uint64_t* out);

// comm.cu: the collectives of sharded contexts (NCCL resolved at run time, or an
// in-process group of contexts driven by host threads); each returns nullptr or an error text
enum RedType { kU32 = 0, kU64 = 1, kI64 = 2 };
enum RedOp { kSum = 0, kMin = 1, kMax = 2 };
struct Comm {
  int rank = 0, nranks = 1;
  virtual ~Comm() {}
  // recv = nranks blocks of `bytes`, rank order
  virtual const char* allgather(const void* send, void* recv, size_t bytes, cudaStream_t st) = 0;
  // in place, element-wise over the ranks
  virtual const char* allreduce(void* buf, size_t count, RedType t, RedOp op, cudaStream_t st) = 0;
  // in place: int64 MAX over [0, max_words), SUM over the next sum_words
  virtual const char* merge_export(int64_t* buf, size_t max_words, size_t sum_words,
                                   cudaStream_t st) = 0;
  // send[p] (sbytes[p] bytes) to rank p, recv[p] (rbytes[p] bytes) from rank p
  virtual const char* alltoallv(const void* const* send, const size_t* sbytes, void* const* recv,
                                const size_t* rbytes, cudaStream_t st) = 0;
};
struct LocalGroup;
const char* nccl_unique_id(void* id128);
Comm* make_nccl_comm(int nranks, int rank, const void* id128, const char** err);
LocalGroup* local_group_create(int n);
void local_group_release(LocalGroup* g);
int local_group_size(const LocalGroup* g);
Comm* make_local_comm(LocalGroup* g, int rank);
size_t agg_bytes(int M, int64_t nwt);
cudaError_t debug_tl2(unsigned long long* out);
cudaError_t debug_bt(unsigned long long* out);     // DVL_PROF builds
cudaError_t debug_nored(int v);                    // DVL_PROF builds
cudaError_t debug_aw(unsigned long long* out);     // DVL_PROF builds
void launch_agg_build(const UpdParams& p, void* agg, int64_t nwt, int num_sms, cudaStream_t st);
// blist / bctr (2 x n_pad / 128 + n_pad / 4096 + 2 u64, 4 u32 zeroed once): the boundary-tile
// list, used when the pixels outnumber agg_reduce's warps (then a bin_boundary launch
// follows), then the straddling-job list of the many-jobs form (agg_jobs + agg_reduce).
// Returns the number of kernels it launched (1-3).
int launch_agg_reduce(const UpdParams& p, const TmaPlan& plan, const unsigned long long* chunk_prefix,
                       const unsigned long long* qtot, uint32_t W, const Acc& acc,
                       uint64_t cell_offset, uint32_t* err, const unsigned long long* meta,
                       const unsigned long long* meta2, const void* agg, unsigned long long* blist,
                       uint32_t* bctr, int num_sms, cudaStream_t st);
void launch_q_export_tma(bool smem_tab, const UpdParams& p, const TmaPlan& plan, int grid,
                         const unsigned long long* chunk_prefix, const unsigned long long* qtot,
                         uint32_t* err, unsigned long long* q_out, const unsigned long long* meta,
                         cudaStream_t st);
size_t bin_reduce_smem(int items, int M, int N, bool smem_tab);

}  // namespace dvl
