// seil_paper.cu -- the paper-literal SEIL list layout (NEXT-2), built from the
// cell-major layout on demand (rairs_set_seil_layout(idx, 1)).
//
// SeilInsert (Alg. 4; structure P:1371-1419): the items of
// cell (i, j) (i <= j) are cut into floor(n/32) 32-item blocks, stored ONCE in
// list i ("shared blocks", referenced from list j by an (i, nblocks, bptr)
// entry), and n % 32 remainder items appended to the miscellaneous area of
// list i AND of list j, each copy carrying the other list's id (
// reading R12: a single-assigned cell (l, l) embeds l itself).  Per list l the
// region here is [shared blocks of the cells (l, j >= l), ascending j][misc:
// remainders of the cells (l, j >= l), then copies of the remainders of the
// cells (i < l, l), ascending i], starting on a 32-slot boundary, so every
// shared block is a 32-aligned block of the 8-item nibble-group code layout
// the query-major scan reads (`codes_g`, fastscan_kernels.cu).
//
// SeilSearch (Alg. 5) over this layout is the query-major scan
// with `a.paper`: per probed list its shared blocks, its misc area (an item is
// dropped after its score is computed when its embedded other list was
// visited, RemoveVectorIfVisited), and each reference whose owner was not
// visited.  Visiting the probe set in ascending list order -- the order under
// which Alg. 5 reaches exactly U(q) (reading R9, tests/seil_paper_sim.py) --
// "visited" = probed with a smaller id, and a reference's owner is always
// smaller than its list.  The scanned item count is the paper's
// DCO_paperSEIL (oracle O12); the candidates equal the cell-major ones.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "index.cuh"

namespace rairs {

constexpr uint32_t kNoOther = 0xFFFFFFFFu;
// hybrid layout: cells below one 8-item group are copied (RAIRS_SEIL_TINY
// overrides it, for measurement)
static uint32_t seil_tiny() {
  const char* e = getenv("RAIRS_SEIL_TINY");
  return e ? (uint32_t)std::max(0, atoi(e)) : 8u;
}

static inline unsigned sp_grid(int64_t n) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), 148 * 32));
}

// thread per (destination group of 8 slots, m4): gathers the 8 items' nibbles
// of subquantizers 4 m4 .. 4 m4 + 3 from the cell-major group layout
__global__ void seil_paper_gather_kernel(const uint8_t* __restrict__ src_g, const uint32_t* __restrict__ map,
                                         const uint32_t* __restrict__ slot_rows, int64_t n_groups, int M4,
                                         uint64_t blk_bytes, uint8_t* __restrict__ dst_g,
                                         uint32_t* __restrict__ dst_rows) {
  const int64_t total = n_groups * M4;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t gi = e / M4;
    const int m4 = (int)(e - gi * M4);
    uint32_t wd[4] = {0u, 0u, 0u, 0u};
    for (int v = 0; v < 8; ++v) {
      const uint32_t s = map[gi * 8 + v];
      if (m4 == 0) dst_rows[gi * 8 + v] = s == kNoOther ? kSlotPad : slot_rows[s];
      if (s == kNoOther) continue;
      const uint32_t sg = s >> 3, sv = s & 7u;
      const uint4 w = *reinterpret_cast<const uint4*>(src_g + (uint64_t)(sg >> 2) * blk_bytes +
                                                      (uint64_t)m4 * 64 + (sg & 3u) * 16);
      wd[0] |= ((w.x >> (4 * sv)) & 0xFu) << (4 * v);
      wd[1] |= ((w.y >> (4 * sv)) & 0xFu) << (4 * v);
      wd[2] |= ((w.z >> (4 * sv)) & 0xFu) << (4 * v);
      wd[3] |= ((w.w >> (4 * sv)) & 0xFu) << (4 * v);
    }
    *reinterpret_cast<uint4*>(dst_g + (uint64_t)(gi >> 2) * blk_bytes + (uint64_t)m4 * 64 + (gi & 3) * 16) =
        make_uint4(wd[0], wd[1], wd[2], wd[3]);
  }
}

void seil_paper_free(rairs_index_s* idx) {
  cudaFree(idx->p_codes_g); cudaFree(idx->p_slot_rows); cudaFree(idx->p_other);
  cudaFree(idx->p_off); cudaFree(idx->p_shared); cudaFree(idx->p_misc);
  cudaFree(idx->p_ref_start); cudaFree(idx->p_ref_cnt);
  idx->p_codes_g = nullptr; idx->p_slot_rows = nullptr; idx->p_other = nullptr;
  idx->p_off = idx->p_shared = idx->p_misc = nullptr;
  idx->p_ref_start = idx->p_ref_cnt = nullptr;
  idx->device_bytes -= idx->p_bytes;
  idx->p_bytes = 0;
  idx->p_slots = 0;
  idx->p_kind = 0;
}

rairs_status seil_paper_prepare(rairs_index_s* idx, cudaStream_t s) {
  seil_paper_free(idx);
  if (!idx->codes_g) {
    set_error("paper SEIL layout: the group code layout is missing");
    return RAIRS_E_INTERNAL;
  }
  const int nlist = idx->nlist;
  const int64_t n_slots = idx->n_slots, nr = idx->n_refs;
  std::vector<uint32_t> own_off(nlist), own_cnt(nlist), slot_rows((size_t)std::max<int64_t>(n_slots, 1));
  std::vector<int32_t> l2((size_t)std::max<int64_t>(idx->n, 1));
  std::vector<uint32_t> ref_ptr(nlist + 1), ref_start((size_t)std::max<int64_t>(nr, 1));
  RAIRS_CUDA_TRY(cudaMemcpyAsync(own_off.data(), idx->own_off, nlist * 4, cudaMemcpyDeviceToHost, s));
  RAIRS_CUDA_TRY(cudaMemcpyAsync(own_cnt.data(), idx->own_cnt, nlist * 4, cudaMemcpyDeviceToHost, s));
  if (n_slots > 0)
    RAIRS_CUDA_TRY(cudaMemcpyAsync(slot_rows.data(), idx->slot_rows, n_slots * 4, cudaMemcpyDeviceToHost, s));
  if (idx->n > 0) RAIRS_CUDA_TRY(cudaMemcpyAsync(l2.data(), idx->l2, idx->n * 4, cudaMemcpyDeviceToHost, s));
  RAIRS_CUDA_TRY(cudaMemcpyAsync(ref_ptr.data(), idx->ref_ptr, (nlist + 1) * 4, cudaMemcpyDeviceToHost, s));
  if (nr > 0) RAIRS_CUDA_TRY(cudaMemcpyAsync(ref_start.data(), idx->ref_start, nr * 4, cudaMemcpyDeviceToHost, s));
  RAIRS_CUDA_TRY(cudaStreamSynchronize(s));

  // cells in cell-major order: owner l ascending, other j ascending (Alg. 4 line 8)
  struct Cell { uint32_t l, j, start, n; };
  std::vector<Cell> cells;
  std::vector<int64_t> shared(nlist, 0), misc_own(nlist, 0), misc_copy(nlist, 0);
  for (int l = 0; l < nlist; ++l) {
    const uint32_t b = own_off[l], e = b + own_cnt[l];
    uint32_t p = b;
    while (p < e) {
      const uint32_t j = (uint32_t)l2[slot_rows[p]];
      uint32_t q = p + 1;
      while (q < e && (uint32_t)l2[slot_rows[q]] == j) ++q;
      const uint32_t n = q - p;
      cells.push_back({(uint32_t)l, j, p, n});
      shared[l] += 32 * (n / 32);                    // lines 12-13
      misc_own[l] += n % 32;
      if (j != (uint32_t)l) misc_copy[j] += n % 32;  // lines 14-15
      p = q;
    }
  }
  const bool hybrid = idx->seil_layout == 3;
  const uint32_t kTiny = seil_tiny();
  std::vector<uint32_t> p_off(nlist), p_shared(nlist), p_misc(nlist);
  std::vector<uint32_t> map, other;
  std::vector<uint32_t> p_ref_start((size_t)std::max<int64_t>(nr, 1), 0), p_ref_cnt((size_t)std::max<int64_t>(nr, 1), 0);
  int64_t p_slots = 0;
  if (hybrid) {
    // hybrid: per list l, [its cell-major owned range, unchanged][misc: copies
    // of the cross cells (i < l, l) with n < kTiny items, ascending i].  A
    // copy is dropped when its owner i was probed (fs_paper_drop: i < l
    // always), so U(q) is the cell-major one; the larger cells stay references.
    std::vector<int64_t> copies(nlist, 0);
    for (const Cell& x : cells)
      if (x.j != x.l && x.n < kTiny) copies[x.j] += x.n;
    int64_t off = 0;
    for (int l = 0; l < nlist; ++l) {
      p_off[l] = (uint32_t)off;
      p_shared[l] = own_cnt[l];
      p_misc[l] = (uint32_t)copies[l];
      off += round_up((int64_t)own_cnt[l] + copies[l], 32);
    }
    if (off >= (int64_t)0xFFFFFFFFll) {
      set_error("hybrid SEIL layout: slot count exceeds 2^32");
      return RAIRS_E_UNSUPPORTED;
    }
    p_slots = std::max<int64_t>(off, 32);
    map.assign((size_t)p_slots, kNoOther);
    other.assign((size_t)p_slots, kNoOther);
    std::vector<uint32_t> mc(nlist);
    for (int l = 0; l < nlist; ++l) {
      mc[l] = p_off[l] + own_cnt[l];
      for (uint32_t t = 0; t < own_cnt[l]; ++t) map[p_off[l] + t] = own_off[l] + t;
    }
    std::vector<uint32_t> cell_start((size_t)cells.size()), cell_pos((size_t)cells.size()),
        cell_n((size_t)cells.size());
    for (size_t c = 0; c < cells.size(); ++c) {
      const Cell& x = cells[c];
      cell_start[c] = x.start;
      cell_pos[c] = p_off[x.l] + (x.start - own_off[x.l]);
      cell_n[c] = x.n;
      if (x.j != x.l && x.n < kTiny)
        for (uint32_t p = 0; p < x.n; ++p) {
          map[mc[x.j]] = x.start + p;
          other[mc[x.j]++] = x.l;
        }
    }
    for (int64_t e = 0; e < nr; ++e) {
      const auto it = std::lower_bound(cell_start.begin(), cell_start.end(), ref_start[e]);
      if (it == cell_start.end() || *it != ref_start[e]) {
        set_error("hybrid SEIL layout: reference without its cell");
        return RAIRS_E_INTERNAL;
      }
      const size_t c = (size_t)(it - cell_start.begin());
      p_ref_start[e] = cell_pos[c];
      p_ref_cnt[e] = cell_n[c] < kTiny ? 0u : cell_n[c];
    }
  } else {
    // regions (line 16): 32-aligned, [shared][misc own][misc copies]
    int64_t off = 0;
    for (int l = 0; l < nlist; ++l) {
      p_off[l] = (uint32_t)off;
      p_shared[l] = (uint32_t)shared[l];
      p_misc[l] = (uint32_t)(misc_own[l] + misc_copy[l]);
      off += round_up(shared[l] + misc_own[l] + misc_copy[l], 32);
    }
    if (off >= (int64_t)0xFFFFFFFFll) {
      set_error("paper SEIL layout: slot count exceeds 2^32");
      return RAIRS_E_UNSUPPORTED;
    }
    p_slots = std::max<int64_t>(off, 32);
    map.assign((size_t)p_slots, kNoOther);
    other.assign((size_t)p_slots, kNoOther);
    std::vector<uint32_t> sh(nlist), mo(nlist), mc(nlist);
    for (int l = 0; l < nlist; ++l) {
      sh[l] = p_off[l];
      mo[l] = p_off[l] + p_shared[l];
      mc[l] = (uint32_t)(p_off[l] + p_shared[l] + misc_own[l]);
    }
    // shared-block start of every cell (the references' bptr), by cell-major start
    std::vector<uint32_t> cell_start((size_t)cells.size()), cell_bptr((size_t)cells.size()),
        cell_full((size_t)cells.size());
    for (size_t c = 0; c < cells.size(); ++c) {  // lines 17-32
      const Cell& x = cells[c];
      const uint32_t full = 32 * (x.n / 32);
      cell_start[c] = x.start;
      cell_bptr[c] = sh[x.l];
      cell_full[c] = full;
      for (uint32_t p = 0; p < full; ++p) map[sh[x.l]++] = x.start + p;  // shared blocks
      for (uint32_t p = full; p < x.n; ++p) {                            // misc, both lists
        map[mo[x.l]] = x.start + p;
        other[mo[x.l]++] = x.j;
        if (x.j != x.l) {
          map[mc[x.j]] = x.start + p;
          other[mc[x.j]++] = x.l;
        }
      }
    }
    // the references of list j (cell-major order = ascending owner): the shared
    // blocks of cell (owner, j) in the owner's region
    for (int64_t e = 0; e < nr; ++e) {
      const auto it = std::lower_bound(cell_start.begin(), cell_start.end(), ref_start[e]);
      if (it == cell_start.end() || *it != ref_start[e]) {
        set_error("paper SEIL layout: reference without its cell");
        return RAIRS_E_INTERNAL;
      }
      const size_t c = (size_t)(it - cell_start.begin());
      p_ref_start[e] = cell_bptr[c];
      p_ref_cnt[e] = cell_full[c];
    }
  }

  const int M4 = idx->M_pad / 4;
  const uint64_t blk_bytes = 16ull * (uint64_t)idx->M_pad;
  const size_t gbytes = (size_t)(p_slots / 32) * blk_bytes;
  uint32_t* d_map = nullptr;
  auto fail = [&](cudaError_t e) {
    cudaFree(d_map);
    seil_paper_free(idx);
    set_error(std::string("paper SEIL layout: ") + cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? RAIRS_E_OOM : RAIRS_E_CUDA;
  };
#define SP_TRY(x) do { cudaError_t _e = (x); if (_e != cudaSuccess) return fail(_e); } while (0)
  SP_TRY(cudaMalloc(&idx->p_codes_g, gbytes));
  SP_TRY(cudaMalloc(&idx->p_slot_rows, (size_t)p_slots * 4));
  SP_TRY(cudaMalloc(&idx->p_other, (size_t)p_slots * 4));
  SP_TRY(cudaMalloc(&idx->p_off, nlist * 4));
  SP_TRY(cudaMalloc(&idx->p_shared, nlist * 4));
  SP_TRY(cudaMalloc(&idx->p_misc, nlist * 4));
  SP_TRY(cudaMalloc(&idx->p_ref_start, (size_t)std::max<int64_t>(nr, 1) * 4));
  SP_TRY(cudaMalloc(&idx->p_ref_cnt, (size_t)std::max<int64_t>(nr, 1) * 4));
  SP_TRY(cudaMalloc(&d_map, (size_t)p_slots * 4));
  idx->p_bytes = (int64_t)gbytes + p_slots * 8 + nlist * 12 + std::max<int64_t>(nr, 1) * 8;
  idx->device_bytes += idx->p_bytes;
  idx->p_slots = p_slots;
  SP_TRY(cudaMemcpyAsync(d_map, map.data(), (size_t)p_slots * 4, cudaMemcpyHostToDevice, s));
  SP_TRY(cudaMemcpyAsync(idx->p_other, other.data(), (size_t)p_slots * 4, cudaMemcpyHostToDevice, s));
  SP_TRY(cudaMemcpyAsync(idx->p_off, p_off.data(), nlist * 4, cudaMemcpyHostToDevice, s));
  SP_TRY(cudaMemcpyAsync(idx->p_shared, p_shared.data(), nlist * 4, cudaMemcpyHostToDevice, s));
  SP_TRY(cudaMemcpyAsync(idx->p_misc, p_misc.data(), nlist * 4, cudaMemcpyHostToDevice, s));
  SP_TRY(cudaMemcpyAsync(idx->p_ref_start, p_ref_start.data(), (size_t)std::max<int64_t>(nr, 1) * 4,
                         cudaMemcpyHostToDevice, s));
  SP_TRY(cudaMemcpyAsync(idx->p_ref_cnt, p_ref_cnt.data(), (size_t)std::max<int64_t>(nr, 1) * 4,
                         cudaMemcpyHostToDevice, s));
  const int64_t n_groups = p_slots / 8;
  seil_paper_gather_kernel<<<sp_grid(n_groups * M4), 256, 0, s>>>(idx->codes_g, d_map, idx->slot_rows,
                                                                   n_groups, M4, blk_bytes, idx->p_codes_g,
                                                                   idx->p_slot_rows);
  SP_TRY(cudaGetLastError());
  SP_TRY(cudaStreamSynchronize(s));
  cudaFree(d_map);
  idx->p_kind = hybrid ? 3 : 1;
#undef SP_TRY
  return RAIRS_OK;
}

}  // namespace rairs
