// tls_graph.cuh — decomposition on the device: the symmetrised sparsity graph,
// the overlap rings of every subdomain and the subdomain colouring, bit-exact with the
// reference's symmetrized_graph (src/sparsemat.py:180-195), extend_overlap
// (src/partition.py:278-301) and color_subdomains (src/partition.py:304-334).
//
//  * graph: edge {i, j}, i != j, iff |a_ij| > 0 or |a_ji| > 0.  Symmetric matrices (flag verified
//    by SparseMat): the nonzero off-diagonal entries of each row, compacted in place order (a
//    count / scan / fill pass).  General: both orientations of every such entry as 64-bit
//    (row, col) keys, radix-sorted and de-duplicated.
//  * overlap: layer k of subdomain s = the sorted unique graph neighbours of layer k-1 (layer 0 =
//    the interior) that are neither interior to s nor in an earlier layer of s.  All subdomains
//    at once: candidate (s, u) pairs written by a count / scan / fill pass over the frontier
//    (owner lookups and binary searches in the sorted earlier layers filter them), one CUB
//    segmented sort per layer (segments = subdomains), then a flag / scan / compact pass keeps
//    the first of each run -- ascending global index, exactly np.unique's order.
//  * colouring: (node, subdomain) incidence keys radix-sorted by node; every node's run of
//    subdomains emits all ordered pairs; sorted unique pairs = the intersection graph; the greedy
//    largest-degree-first colouring (ties by index, smallest free colour) runs on the host over
//    those adjacency lists (a few thousand subdomains).
#pragma once
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>
#include <cub/device/device_select.cuh>

#include <algorithm>
#include <string>
#include <vector>

namespace tls {
namespace graph {

constexpr int GT = 256;

inline int gblocks(long long work) {
  long long g = (work + GT - 1) / GT;
  return (int)std::max<long long>(1, std::min<long long>(g, 148LL * 16));
}

// ---- symmetrised graph ----------------------------------------------------------------------
__global__ void k_offdiag_count(int n, const int* __restrict__ rowptr, const int* __restrict__ col,
                                const double* __restrict__ val, long long* __restrict__ cnt) {
  for (int i = blockIdx.x * GT + threadIdx.x; i < n; i += gridDim.x * GT) {
    int c = 0;
    for (int k = rowptr[i]; k < rowptr[i + 1]; ++k) c += (col[k] != i && val[k] != 0.0);
    cnt[i] = c;
  }
}

__global__ void k_offdiag_fill(int n, const int* __restrict__ rowptr, const int* __restrict__ col,
                               const double* __restrict__ val, const long long* __restrict__ ptr,
                               int* __restrict__ adj) {
  for (int i = blockIdx.x * GT + threadIdx.x; i < n; i += gridDim.x * GT) {
    long long p = ptr[i];
    for (int k = rowptr[i]; k < rowptr[i + 1]; ++k)
      if (col[k] != i && val[k] != 0.0) adj[p++] = col[k];
  }
}

__global__ void k_offdiag_pairs(int n, const int* __restrict__ rowptr, const int* __restrict__ col,
                                const double* __restrict__ val, const long long* __restrict__ ptr,
                                unsigned long long* __restrict__ keys) {
  for (int i = blockIdx.x * GT + threadIdx.x; i < n; i += gridDim.x * GT) {
    long long p = ptr[i];
    for (int k = rowptr[i]; k < rowptr[i + 1]; ++k)
      if (col[k] != i && val[k] != 0.0) {
        keys[2 * p] = ((unsigned long long)i << 32) | (unsigned)col[k];
        keys[2 * p + 1] = ((unsigned long long)col[k] << 32) | (unsigned)i;
        ++p;
      }
  }
}

__global__ void k_keys_split(long long m, const unsigned long long* __restrict__ keys, int* __restrict__ adj,
                             long long* __restrict__ rowcnt) {
  for (long long p = blockIdx.x * (long long)GT + threadIdx.x; p < m; p += (long long)gridDim.x * GT) {
    const unsigned long long k = keys[p];
    adj[p] = (int)(k & 0xffffffffULL);
    atomicAdd((unsigned long long*)&rowcnt[k >> 32], 1ULL);
  }
}

// ---- overlap ----------------------------------------------------------------------------------
// seen(s, u): u interior to s, or in one of the first `nl` layers of s (sorted: binary search)
__device__ __forceinline__ bool seen_in(int s, int u, const int* __restrict__ owner, int nl,
                                        int* const* __restrict__ lnode, long long* const* __restrict__ loff) {
  if (owner[u] == s) return true;
  for (int l = 0; l < nl; ++l) {
    long long lo = loff[l][s], hi = loff[l][s + 1];
    const int* a = lnode[l];
    while (lo < hi) {
      const long long mid = (lo + hi) >> 1;
      if (a[mid] < u) lo = mid + 1; else hi = mid;
    }
    if (lo < loff[l][s + 1] && a[lo] == u) return true;
  }
  return false;
}

struct LayerPtrs {
  int* node[8];
  long long* off[8];
};

__global__ void k_cand_count(long long F, const int* __restrict__ fnode, const int* __restrict__ fsub,
                             const long long* __restrict__ gptr, const int* __restrict__ adj,
                             const int* __restrict__ owner, int nl, LayerPtrs L, long long* __restrict__ cnt) {
  for (long long e = blockIdx.x * (long long)GT + threadIdx.x; e < F; e += (long long)gridDim.x * GT) {
    const int v = fnode[e], s = fsub[e];
    long long c = 0;
    for (long long k = gptr[v]; k < gptr[v + 1]; ++k) c += !seen_in(s, adj[k], owner, nl, L.node, L.off);
    cnt[e] = c;
  }
}

__global__ void k_cand_fill(long long F, const int* __restrict__ fnode, const int* __restrict__ fsub,
                            const long long* __restrict__ gptr, const int* __restrict__ adj,
                            const int* __restrict__ owner, int nl, LayerPtrs L, const long long* __restrict__ pos,
                            int* __restrict__ cand) {
  for (long long e = blockIdx.x * (long long)GT + threadIdx.x; e < F; e += (long long)gridDim.x * GT) {
    const int v = fnode[e], s = fsub[e];
    long long p = pos[e];
    for (long long k = gptr[v]; k < gptr[v + 1]; ++k) {
      const int u = adj[k];
      if (!seen_in(s, u, owner, nl, L.node, L.off)) cand[p++] = u;
    }
  }
}

// seg[s] = pos[fo[s]] (candidate segment of subdomain s)
__global__ void k_gather_ll(int m, const long long* __restrict__ idx, const long long* __restrict__ src,
                            long long* __restrict__ dst) {
  for (int i = blockIdx.x * GT + threadIdx.x; i < m; i += gridDim.x * GT) dst[i] = src[idx[i]];
}

// keep the first of every run of equal candidates inside a segment
__global__ void k_run_first(int nsub, const long long* __restrict__ seg, const int* __restrict__ cand,
                            long long* __restrict__ flag) {
  for (int s = blockIdx.x; s < nsub; s += gridDim.x)
    for (long long p = seg[s] + threadIdx.x; p < seg[s + 1]; p += GT)
      flag[p] = (p == seg[s] || cand[p] != cand[p - 1]) ? 1 : 0;
}

__global__ void k_compact_sub(int nsub, const long long* __restrict__ seg, const int* __restrict__ cand,
                              const long long* __restrict__ flag, const long long* __restrict__ npos,
                              int* __restrict__ out, int* __restrict__ osub) {
  for (int s = blockIdx.x; s < nsub; s += gridDim.x)
    for (long long p = seg[s] + threadIdx.x; p < seg[s + 1]; p += GT)
      if (flag[p]) {
        out[npos[p]] = cand[p];
        osub[npos[p]] = s;
      }
}

// interior: start of every owner id in the owner-sorted node list
__global__ void k_owner_starts(int n, int nsub, const int* __restrict__ sowner, long long* __restrict__ st) {
  for (int i = blockIdx.x * GT + threadIdx.x; i <= n; i += gridDim.x * GT) {
    const int cur = i < n ? sowner[i] : nsub;
    const int prev = i > 0 ? sowner[i - 1] : -1;
    for (int s = prev + 1; s <= cur; ++s) st[s] = i;
  }
}

__global__ void k_iota(int n, int* __restrict__ a) {
  for (int i = blockIdx.x * GT + threadIdx.x; i < n; i += gridDim.x * GT) a[i] = i;
}

// ---- colouring --------------------------------------------------------------------------------
__global__ void k_incidence(long long m, const int* __restrict__ node, const int* __restrict__ sub,
                            unsigned long long* __restrict__ keys) {
  for (long long p = blockIdx.x * (long long)GT + threadIdx.x; p < m; p += (long long)gridDim.x * GT)
    keys[p] = ((unsigned long long)(unsigned)node[p] << 32) | (unsigned)sub[p];
}

// run r of equal nodes = keys[rs[r], rs[r+1]); rs from the run starts
__global__ void k_run_starts(long long m, const unsigned long long* __restrict__ keys, long long* __restrict__ flag) {
  for (long long p = blockIdx.x * (long long)GT + threadIdx.x; p < m; p += (long long)gridDim.x * GT)
    flag[p] = (p == 0 || (keys[p] >> 32) != (keys[p - 1] >> 32)) ? 1 : 0;
}

__global__ void k_run_index(long long m, const long long* __restrict__ flag, const long long* __restrict__ rid,
                            long long* __restrict__ rs) {
  for (long long p = blockIdx.x * (long long)GT + threadIdx.x; p < m; p += (long long)gridDim.x * GT)
    if (flag[p]) rs[rid[p]] = p;
}

__global__ void k_pair_count(long long R, const long long* __restrict__ rs, long long* __restrict__ cnt) {
  for (long long r = blockIdx.x * (long long)GT + threadIdx.x; r < R; r += (long long)gridDim.x * GT) {
    const long long k = rs[r + 1] - rs[r];
    cnt[r] = k * (k - 1);
  }
}

__global__ void k_pair_fill(long long R, const long long* __restrict__ rs, const unsigned long long* __restrict__ keys,
                            const long long* __restrict__ pos, unsigned long long* __restrict__ pairs) {
  for (long long r = blockIdx.x * (long long)GT + threadIdx.x; r < R; r += (long long)gridDim.x * GT) {
    long long p = pos[r];
    for (long long a = rs[r]; a < rs[r + 1]; ++a)
      for (long long b = rs[r]; b < rs[r + 1]; ++b)
        if (a != b)
          pairs[p++] = ((keys[a] & 0xffffffffULL) << 32) | (keys[b] & 0xffffffffULL);
  }
}

// ---- host drivers ---------------------------------------------------------------------------
// A small RAII arena: every temporary goes back when the driver returns.
struct Arena {
  std::vector<void*> ptrs;
  cudaError_t err = cudaSuccess;
  template <class T>
  T* alloc(long long count) {
    void* p = nullptr;
    if (err != cudaSuccess) return nullptr;
    err = cudaMalloc(&p, (size_t)std::max<long long>(1, count) * sizeof(T));
    if (err != cudaSuccess) return nullptr;
    ptrs.push_back(p);
    return (T*)p;
  }
  void release(void* p) {
    for (auto& q : ptrs)
      if (q == p) {
        cudaFree(q);
        q = nullptr;
      }
  }
  ~Arena() {
    for (void* p : ptrs)
      if (p) cudaFree(p);
  }
};

template <class T>
inline cudaError_t exclusive_sum(Arena& ar, const T* in, T* out, long long n, cudaStream_t s) {
  size_t tb = 0;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, n, s);
  if (e != cudaSuccess) return e;
  void* tmp = ar.alloc<char>((long long)tb);
  if (ar.err != cudaSuccess) return ar.err;
  e = cub::DeviceScan::ExclusiveSum(tmp, tb, in, out, n, s);
  ar.release(tmp);
  return e;
}

inline cudaError_t sort_keys64(Arena& ar, unsigned long long*& keys, long long m, int end_bit, cudaStream_t s) {
  unsigned long long* alt = ar.alloc<unsigned long long>(m);
  if (ar.err != cudaSuccess) return ar.err;
  cub::DoubleBuffer<unsigned long long> db(keys, alt);
  size_t tb = 0;
  cudaError_t e = cub::DeviceRadixSort::SortKeys(nullptr, tb, db, m, 0, end_bit, s);
  if (e != cudaSuccess) return e;
  void* tmp = ar.alloc<char>((long long)tb);
  if (ar.err != cudaSuccess) return ar.err;
  e = cub::DeviceRadixSort::SortKeys(tmp, tb, db, m, 0, end_bit, s);
  ar.release(tmp);
  keys = db.Current();
  return e;
}

inline cudaError_t unique_keys64(Arena& ar, const unsigned long long* in, long long m, unsigned long long* out,
                                 long long& m_out, cudaStream_t s) {
  long long* d_n = ar.alloc<long long>(1);
  size_t tb = 0;
  cudaError_t e = cub::DeviceSelect::Unique(nullptr, tb, in, out, d_n, m, s);
  if (e != cudaSuccess) return e;
  void* tmp = ar.alloc<char>((long long)tb);
  if (ar.err != cudaSuccess) return ar.err;
  if ((e = cub::DeviceSelect::Unique(tmp, tb, in, out, d_n, m, s)) != cudaSuccess) return e;
  if ((e = cudaMemcpyAsync(&m_out, d_n, sizeof(long long), cudaMemcpyDeviceToHost, s)) != cudaSuccess) return e;
  return cudaStreamSynchronize(s);
}

// Symmetrised graph of a device CSR (int32 rowptr/col, fp64 values); gptr (n+1, int64) and adj
// (int32) are cudaMalloc'ed here and owned by the caller.
inline cudaError_t build_graph(int n, const int* rowptr, const int* col, const double* val, bool sym,
                               long long*& gptr, int*& adj, long long& m, cudaStream_t s, std::string& err) {
  Arena ar;
  long long* cnt = ar.alloc<long long>(n + 1);
  if (ar.err != cudaSuccess) return ar.err;
  cudaError_t e;
  if ((e = cudaMemsetAsync(cnt, 0, sizeof(long long) * (n + 1), s)) != cudaSuccess) return e;
  k_offdiag_count<<<gblocks(n), GT, 0, s>>>(n, rowptr, col, val, cnt);
  long long* ptr0 = ar.alloc<long long>(n + 1);
  if (ar.err != cudaSuccess) return ar.err;
  if ((e = exclusive_sum(ar, cnt, ptr0, (long long)n + 1, s)) != cudaSuccess) return e;
  long long m0 = 0;
  if ((e = cudaMemcpyAsync(&m0, ptr0 + n, sizeof(long long), cudaMemcpyDeviceToHost, s)) != cudaSuccess) return e;
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
  if (sym) {
    if ((e = cudaMalloc(&gptr, sizeof(long long) * (n + 1))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&adj, sizeof(int) * std::max<long long>(1, m0))) != cudaSuccess) return e;
    if ((e = cudaMemcpyAsync(gptr, ptr0, sizeof(long long) * (n + 1), cudaMemcpyDeviceToDevice, s)) != cudaSuccess)
      return e;
    k_offdiag_fill<<<gblocks(n), GT, 0, s>>>(n, rowptr, col, val, ptr0, adj);
    m = m0;
    return cudaGetLastError();
  }
  unsigned long long* keys = ar.alloc<unsigned long long>(2 * m0);
  if (ar.err != cudaSuccess) return ar.err;
  k_offdiag_pairs<<<gblocks(n), GT, 0, s>>>(n, rowptr, col, val, ptr0, keys);
  if ((e = sort_keys64(ar, keys, 2 * m0, 64, s)) != cudaSuccess) return e;
  unsigned long long* uk = ar.alloc<unsigned long long>(2 * m0);
  if (ar.err != cudaSuccess) return ar.err;
  if ((e = unique_keys64(ar, keys, 2 * m0, uk, m, s)) != cudaSuccess) return e;
  if ((e = cudaMalloc(&gptr, sizeof(long long) * (n + 1))) != cudaSuccess) return e;
  if ((e = cudaMalloc(&adj, sizeof(int) * std::max<long long>(1, m))) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(cnt, 0, sizeof(long long) * (n + 1), s)) != cudaSuccess) return e;
  k_keys_split<<<gblocks(m), GT, 0, s>>>(m, uk, adj, cnt);
  if ((e = exclusive_sum(ar, cnt, gptr, (long long)n + 1, s)) != cudaSuccess) return e;
  (void)err;
  return cudaStreamSynchronize(s);
}

// Overlap rings + colouring.  owner: device int32 (n).  Outputs (host): per subdomain
// offsets (nsub+1), layer sizes (nsub x delta), the concatenated index lists (interior, layer
// 1..delta; int64), colours, k_c.
inline cudaError_t overlap_and_colour(int n, const long long* gptr, const int* adj, const int* owner, int nsub,
                                      int delta, std::vector<long long>& offsets, std::vector<long long>& lsizes,
                                      std::vector<long long>& indices, std::vector<long long>& colors, int& k_c,
                                      cudaStream_t s, std::string& err) {
  if (delta < 1 || delta > 8) {
    err = "overlap must be between 1 and 8 on the device path";
    return cudaErrorInvalidValue;
  }
  Arena ar;
  cudaError_t e;
  // interior lists: nodes sorted by owner (stable radix sort: ascending ids inside each owner)
  int* iota = ar.alloc<int>(n);
  int* order = ar.alloc<int>(n);
  int* sowner = ar.alloc<int>(n);
  long long* ist = ar.alloc<long long>(nsub + 1);
  if (ar.err != cudaSuccess) return ar.err;
  k_iota<<<gblocks(n), GT, 0, s>>>(n, iota);
  {
    size_t tb = 0;
    int end_bit = 1;
    while ((1LL << end_bit) <= nsub) ++end_bit;
    if ((e = cub::DeviceRadixSort::SortPairs(nullptr, tb, owner, sowner, iota, order, n, 0, end_bit, s)) != cudaSuccess)
      return e;
    void* tmp = ar.alloc<char>((long long)tb);
    if (ar.err != cudaSuccess) return ar.err;
    if ((e = cub::DeviceRadixSort::SortPairs(tmp, tb, owner, sowner, iota, order, n, 0, end_bit, s)) != cudaSuccess)
      return e;
    ar.release(tmp);
  }
  k_owner_starts<<<gblocks((long long)n + 1), GT, 0, s>>>(n, nsub, sowner, ist);
  std::vector<long long> h_ist(nsub + 1);
  if ((e = cudaMemcpyAsync(h_ist.data(), ist, sizeof(long long) * (nsub + 1), cudaMemcpyDeviceToHost, s)) != cudaSuccess)
    return e;
  // layers
  LayerPtrs L{};
  std::vector<int*> lsubs(delta, nullptr);
  std::vector<std::vector<long long>> h_loff(delta);
  std::vector<std::vector<int>> h_layer(delta);
  const int* fnode = order;
  const int* fsub = sowner;
  long long F = n;
  const long long* fo = ist;
  for (int k = 0; k < delta; ++k) {
    long long* cnt = ar.alloc<long long>(F + 1);
    long long* pos = ar.alloc<long long>(F + 1);
    long long* seg = ar.alloc<long long>(nsub + 1);
    if (ar.err != cudaSuccess) return ar.err;
    if ((e = cudaMemsetAsync(cnt, 0, sizeof(long long) * (F + 1), s)) != cudaSuccess) return e;
    k_cand_count<<<gblocks(F), GT, 0, s>>>(F, fnode, fsub, gptr, adj, owner, k, L, cnt);
    if ((e = exclusive_sum(ar, cnt, pos, F + 1, s)) != cudaSuccess) return e;
    k_gather_ll<<<gblocks(nsub + 1), GT, 0, s>>>(nsub + 1, fo, pos, seg);
    long long tot = 0;
    if ((e = cudaMemcpyAsync(&tot, pos + F, sizeof(long long), cudaMemcpyDeviceToHost, s)) != cudaSuccess) return e;
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
    int* cand = ar.alloc<int>(tot);
    int* cand2 = ar.alloc<int>(tot);
    if (ar.err != cudaSuccess) return ar.err;
    k_cand_fill<<<gblocks(F), GT, 0, s>>>(F, fnode, fsub, gptr, adj, owner, k, L, pos, cand);
    {
      size_t tb = 0;
      if ((e = cub::DeviceSegmentedSort::SortKeys(nullptr, tb, cand, cand2, tot, nsub, seg, seg + 1, s)) != cudaSuccess)
        return e;
      void* tmp = ar.alloc<char>((long long)tb);
      if (ar.err != cudaSuccess) return ar.err;
      if ((e = cub::DeviceSegmentedSort::SortKeys(tmp, tb, cand, cand2, tot, nsub, seg, seg + 1, s)) != cudaSuccess)
        return e;
      ar.release(tmp);
    }
    long long* flag = ar.alloc<long long>(tot + 1);
    long long* npos = ar.alloc<long long>(tot + 1);
    if (ar.err != cudaSuccess) return ar.err;
    if ((e = cudaMemsetAsync(flag, 0, sizeof(long long) * (tot + 1), s)) != cudaSuccess) return e;
    k_run_first<<<std::min(nsub, 148 * 8), GT, 0, s>>>(nsub, seg, cand2, flag);
    if ((e = exclusive_sum(ar, flag, npos, tot + 1, s)) != cudaSuccess) return e;
    long long m = 0;
    if ((e = cudaMemcpyAsync(&m, npos + tot, sizeof(long long), cudaMemcpyDeviceToHost, s)) != cudaSuccess) return e;
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
    int* lnode = ar.alloc<int>(m);
    int* lsub = ar.alloc<int>(m);
    long long* loff = ar.alloc<long long>(nsub + 1);
    if (ar.err != cudaSuccess) return ar.err;
    k_compact_sub<<<std::min(nsub, 148 * 8), GT, 0, s>>>(nsub, seg, cand2, flag, npos, lnode, lsub);
    k_gather_ll<<<gblocks(nsub + 1), GT, 0, s>>>(nsub + 1, seg, npos, loff);
    L.node[k] = lnode;
    L.off[k] = loff;
    lsubs[k] = lsub;
    h_loff[k].resize(nsub + 1);
    h_layer[k].resize(m);
    if ((e = cudaMemcpyAsync(h_loff[k].data(), loff, sizeof(long long) * (nsub + 1), cudaMemcpyDeviceToHost, s)) !=
        cudaSuccess)
      return e;
    if (m && (e = cudaMemcpyAsync(h_layer[k].data(), lnode, sizeof(int) * m, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
      return e;
    ar.release(cand);
    ar.release(cand2);
    ar.release(flag);
    ar.release(npos);
    ar.release(cnt);
    ar.release(pos);
    fnode = lnode;
    fsub = lsub;
    F = m;
    fo = loff;
  }
  // colouring: (node, subdomain) incidence over interiors and all layers
  long long tot_inc = n;
  for (int k = 0; k < delta; ++k) tot_inc += h_loff[k][nsub];
  unsigned long long* inc = ar.alloc<unsigned long long>(tot_inc);
  if (ar.err != cudaSuccess) return ar.err;
  {
    k_incidence<<<gblocks(n), GT, 0, s>>>(n, order, sowner, inc);
    long long o = n;
    for (int k = 0; k < delta; ++k) {  // layer entries with their subdomain (the compaction's lsub)
      const long long m = h_loff[k][nsub];
      if (m) k_incidence<<<gblocks(m), GT, 0, s>>>(m, L.node[k], lsubs[k], inc + o);
      o += m;
    }
  }
  if ((e = sort_keys64(ar, inc, tot_inc, 64, s)) != cudaSuccess) return e;
  long long* rflag = ar.alloc<long long>(tot_inc + 1);
  long long* rid = ar.alloc<long long>(tot_inc + 1);
  if (ar.err != cudaSuccess) return ar.err;
  if ((e = cudaMemsetAsync(rflag, 0, sizeof(long long) * (tot_inc + 1), s)) != cudaSuccess) return e;
  k_run_starts<<<gblocks(tot_inc), GT, 0, s>>>(tot_inc, inc, rflag);
  if ((e = exclusive_sum(ar, rflag, rid, tot_inc + 1, s)) != cudaSuccess) return e;
  long long R = 0;
  if ((e = cudaMemcpyAsync(&R, rid + tot_inc, sizeof(long long), cudaMemcpyDeviceToHost, s)) != cudaSuccess) return e;
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
  long long* rs = ar.alloc<long long>(R + 1);
  long long* pc = ar.alloc<long long>(R + 1);
  long long* pp = ar.alloc<long long>(R + 1);
  if (ar.err != cudaSuccess) return ar.err;
  k_run_index<<<gblocks(tot_inc), GT, 0, s>>>(tot_inc, rflag, rid, rs);
  if ((e = cudaMemcpyAsync(rs + R, &tot_inc, sizeof(long long), cudaMemcpyHostToDevice, s)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(pc, 0, sizeof(long long) * (R + 1), s)) != cudaSuccess) return e;
  k_pair_count<<<gblocks(R), GT, 0, s>>>(R, rs, pc);
  if ((e = exclusive_sum(ar, pc, pp, R + 1, s)) != cudaSuccess) return e;
  long long P = 0;
  if ((e = cudaMemcpyAsync(&P, pp + R, sizeof(long long), cudaMemcpyDeviceToHost, s)) != cudaSuccess) return e;
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
  std::vector<unsigned long long> hp;
  if (P > 0) {
    unsigned long long* pairs = ar.alloc<unsigned long long>(P);
    if (ar.err != cudaSuccess) return ar.err;
    k_pair_fill<<<gblocks(R), GT, 0, s>>>(R, rs, inc, pp, pairs);
    if ((e = sort_keys64(ar, pairs, P, 64, s)) != cudaSuccess) return e;
    unsigned long long* up = ar.alloc<unsigned long long>(P);
    long long U = 0;
    if ((e = unique_keys64(ar, pairs, P, up, U, s)) != cudaSuccess) return e;
    hp.resize(U);
    if ((e = cudaMemcpy(hp.data(), up, sizeof(unsigned long long) * U, cudaMemcpyDeviceToHost)) != cudaSuccess) return e;
  }
  // greedy colouring (src/partition.py:323-334): largest degree first, ties by index, smallest
  // colour not used by an already-coloured neighbour
  std::vector<long long> aptr(nsub + 1, 0);
  for (unsigned long long k : hp) aptr[(k >> 32) + 1]++;
  for (int q = 0; q < nsub; ++q) aptr[q + 1] += aptr[q];
  std::vector<int> ord(nsub);
  for (int q = 0; q < nsub; ++q) ord[q] = q;
  std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) {
    return (aptr[a + 1] - aptr[a]) > (aptr[b + 1] - aptr[b]);
  });
  colors.assign(nsub, -1);
  std::vector<int> mark;
  for (int q : ord) {
    mark.assign(aptr[q + 1] - aptr[q] + 2, 0);
    for (long long p = aptr[q]; p < aptr[q + 1]; ++p) {
      const long long c = colors[hp[p] & 0xffffffffULL];
      if (c >= 0 && c < (long long)mark.size()) mark[c] = 1;
    }
    int c = 0;
    while (mark[c]) ++c;
    colors[q] = c;
  }
  k_c = 0;
  for (long long c : colors) k_c = std::max<int>(k_c, (int)c + 1);
  // host assembly: interior then layers 1..delta per subdomain
  std::vector<int> h_order(n);
  if ((e = cudaMemcpy(h_order.data(), order, sizeof(int) * n, cudaMemcpyDeviceToHost)) != cudaSuccess) return e;
  offsets.assign(nsub + 1, 0);
  lsizes.assign((size_t)nsub * delta, 0);
  for (int q = 0; q < nsub; ++q) {
    long long t = h_ist[q + 1] - h_ist[q];
    for (int k = 0; k < delta; ++k) {
      lsizes[(size_t)q * delta + k] = h_loff[k][q + 1] - h_loff[k][q];
      t += lsizes[(size_t)q * delta + k];
    }
    offsets[q + 1] = offsets[q] + t;
  }
  indices.resize(offsets[nsub]);
  for (int q = 0; q < nsub; ++q) {
    long long o = offsets[q];
    for (long long p = h_ist[q]; p < h_ist[q + 1]; ++p) indices[o++] = h_order[p];
    for (int k = 0; k < delta; ++k)
      for (long long p = h_loff[k][q]; p < h_loff[k][q + 1]; ++p) indices[o++] = h_layer[k][p];
  }
  return cudaSuccess;
}

}  // namespace graph
}  // namespace tls
