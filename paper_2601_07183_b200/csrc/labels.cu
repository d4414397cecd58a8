// labels.cu -- caller-supplied vector ids ("labels": the
// optional `ids` of rairs_build_index / rairs_add).
//
// Inside the index every row keeps its internal global id (local row * G +
// shard): the candidate keys (s, id) of the selection use it (reading R5 ties).
// A label is a payload: the refine writes (delta, label) keys, so results,
// their tie order and the shard merge use labels.  Labels are unique,
// in [0, 2^32 - 2] (the keys hold 32-bit ids, like the internal ids).  A
// sorted (label, row) table serves deletes by label.
#include <cub/cub.cuh>

#include "index.cuh"

namespace rairs {

constexpr uint32_t kMaxLabel = 0xFFFFFFFEu;

static inline unsigned lgrid(int64_t n) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16));
}

// flags[0] += ids out of range; keys = (u32) ids
__global__ void label_range_kernel(const int64_t* __restrict__ ids, int64_t m,
                                   uint32_t* __restrict__ keys, unsigned* __restrict__ bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = ids[i];
    if (v < 0 || v > (int64_t)kMaxLabel) atomicAdd(bad, 1u);
    keys[i] = (uint32_t)(v < 0 ? 0 : (v > (int64_t)kMaxLabel ? kMaxLabel : v));
  }
}

// bad[1] += adjacent duplicates of a sorted array
__global__ void label_dup_kernel(const uint32_t* __restrict__ sorted, int64_t m,
                                 unsigned* __restrict__ bad) {
  for (int64_t i = 1 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    if (sorted[i] == sorted[i - 1]) atomicAdd(bad, 1u);
}

__device__ __forceinline__ int64_t label_find(const uint32_t* sorted, int64_t m, uint32_t v) {
  int64_t lo = 0, hi = m;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (sorted[mid] < v) lo = mid + 1; else hi = mid;
  }
  return (lo < m && sorted[lo] == v) ? lo : -1;
}

// the (label, row) table keeps the labels of deleted rows (rows are never
// reused): the row holding label v is the first LIVE one among its entries
// (at most one is live -- a label is unique among live rows), or -1
__device__ __forceinline__ int64_t label_find_live(const uint32_t* sorted, const uint32_t* rows,
                                                   const uint32_t* live_bits, int64_t m, uint32_t v) {
  int64_t p = label_find(sorted, m, v);
  if (p < 0) return -1;
  for (; p < m && sorted[p] == v; ++p) {
    const uint32_t r = rows[p];
    if (live_bits == nullptr || ((live_bits[r >> 5] >> (r & 31)) & 1u)) return p;
  }
  return -1;
}

// bad[2] += new labels already held by a live row of the index (a label whose
// row was deleted may be added again)
__global__ void label_clash_kernel(const uint32_t* __restrict__ keys, int64_t m,
                                   const uint32_t* __restrict__ sorted,
                                   const uint32_t* __restrict__ rows,
                                   const uint32_t* __restrict__ live_bits, int64_t ns,
                                   unsigned* __restrict__ bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    if (label_find_live(sorted, rows, live_bits, ns, keys[i]) >= 0) atomicAdd(bad, 1u);
}

__global__ void iota_u32_kernel(uint32_t* __restrict__ a, int64_t m) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    a[i] = (uint32_t)i;
}

rairs_status labels_validate(const rairs_index_s* idx, const int64_t* ids, int64_t m,
                             cudaStream_t s) {
  if (m <= 0) return RAIRS_OK;
  uint32_t *keys = nullptr, *sorted = nullptr;
  unsigned* bad = nullptr;
  void* tmp = nullptr;
  size_t tb = 0;
  auto done = [&](rairs_status st) {
    cudaFreeAsync(keys, s); cudaFreeAsync(sorted, s); cudaFreeAsync(bad, s); cudaFreeAsync(tmp, s);
    return st;
  };
#define LB_TRY(x) do { cudaError_t _e = (x); if (_e != cudaSuccess) { set_error(std::string(#x) + ": " + cudaGetErrorString(_e)); return done(_e == cudaErrorMemoryAllocation ? RAIRS_E_OOM : RAIRS_E_CUDA); } } while (0)
  LB_TRY(ws_malloc(&keys, (size_t)m * 4, s));
  LB_TRY(ws_malloc(&sorted, (size_t)m * 4, s));
  LB_TRY(ws_malloc(&bad, 3 * sizeof(unsigned), s));
  LB_TRY(cudaMemsetAsync(bad, 0, 3 * sizeof(unsigned), s));
  label_range_kernel<<<lgrid(m), 256, 0, s>>>(ids, m, keys, bad);
  LB_TRY(cudaGetLastError());
  LB_TRY(cub::DeviceRadixSort::SortKeys(nullptr, tb, keys, sorted, m, 0, 32, s));
  LB_TRY(ws_malloc(&tmp, std::max<size_t>(tb, 16), s));
  LB_TRY(cub::DeviceRadixSort::SortKeys(tmp, tb, keys, sorted, m, 0, 32, s));
  label_dup_kernel<<<lgrid(m), 256, 0, s>>>(sorted, m, bad + 1);
  LB_TRY(cudaGetLastError());
  if (idx && idx->lab_sorted && idx->n > 0) {
    label_clash_kernel<<<lgrid(m), 256, 0, s>>>(keys, m, idx->lab_sorted, idx->lab_rows,
                                                idx->live_bits, idx->n, bad + 2);
    LB_TRY(cudaGetLastError());
  }
  unsigned h[3] = {0, 0, 0};
  LB_TRY(cudaMemcpyAsync(h, bad, sizeof(h), cudaMemcpyDeviceToHost, s));
  LB_TRY(cudaStreamSynchronize(s));
#undef LB_TRY
  if (h[0]) {
    set_error("ids must be in [0, 2^32 - 2]");
    return done(RAIRS_E_INVALID);
  }
  if (h[1]) {
    set_error("duplicate ids");
    return done(RAIRS_E_INVALID);
  }
  if (h[2]) {
    set_error("ids already in the index");
    return done(RAIRS_E_INVALID);
  }
  return done(RAIRS_OK);
}

__global__ void label_store_kernel(const int64_t* __restrict__ ids, int64_t m,
                                   uint32_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (uint32_t)ids[i];
}

rairs_status labels_store(rairs_index_s* idx, const int64_t* ids, int64_t row0, int64_t m,
                          cudaStream_t s) {
  if (!idx->labels) return RAIRS_OK;
  if (m > 0) {
    label_store_kernel<<<lgrid(m), 256, 0, s>>>(ids, m, idx->labels + row0);
    RAIRS_CHECK_LAUNCH();
  }
  // rebuild the sorted (label, row) table over every row
  const int64_t n = row0 + m;
  cudaFree(idx->lab_sorted);
  cudaFree(idx->lab_rows);
  idx->lab_sorted = idx->lab_rows = nullptr;
  uint32_t* rows_in = nullptr;
  void* tmp = nullptr;
  size_t tb = 0;
  RAIRS_CUDA_TRY(cudaMalloc(&idx->lab_sorted, (size_t)std::max<int64_t>(n, 1) * 4));
  RAIRS_CUDA_TRY(cudaMalloc(&idx->lab_rows, (size_t)std::max<int64_t>(n, 1) * 4));
  RAIRS_CUDA_TRY(ws_malloc(&rows_in, (size_t)std::max<int64_t>(n, 1) * 4, s));
  iota_u32_kernel<<<lgrid(n), 256, 0, s>>>(rows_in, n);
  RAIRS_CHECK_LAUNCH();
  RAIRS_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tb, idx->labels, idx->lab_sorted, rows_in,
                                                 idx->lab_rows, n, 0, 32, s));
  RAIRS_CUDA_TRY(ws_malloc(&tmp, std::max<size_t>(tb, 16), s));
  RAIRS_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp, tb, idx->labels, idx->lab_sorted, rows_in,
                                                 idx->lab_rows, n, 0, 32, s));
  cudaFreeAsync(tmp, s);
  cudaFreeAsync(rows_in, s);
  RAIRS_CUDA_TRY(cudaStreamSynchronize(s));
  return RAIRS_OK;
}

// labels -> internal global ids row * G + shard (-1 when the index does not
// hold the label)
__global__ void label_rows_kernel(const int64_t* __restrict__ ids, int64_t m,
                                  const uint32_t* __restrict__ sorted,
                                  const uint32_t* __restrict__ rows,
                                  const uint32_t* __restrict__ live_bits, int64_t n, int G, int shard,
                                  int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = ids[i];
    int64_t r = -1;
    if (v >= 0 && v <= (int64_t)kMaxLabel) {
      const int64_t p = label_find_live(sorted, rows, live_bits, n, (uint32_t)v);
      if (p >= 0) r = (int64_t)rows[p] * G + shard;
    }
    out[i] = r;
  }
}

rairs_status labels_to_gids(const rairs_index_s* idx, const int64_t* ids, int64_t m,
                            int64_t* gids_out, cudaStream_t s) {
  if (m <= 0) return RAIRS_OK;
  label_rows_kernel<<<lgrid(m), 256, 0, s>>>(ids, m, idx->lab_sorted, idx->lab_rows, idx->live_bits,
                                             idx->n, idx->nshards, idx->shard_id, gids_out);
  RAIRS_CHECK_LAUNCH();
  return RAIRS_OK;
}

}  // namespace rairs
