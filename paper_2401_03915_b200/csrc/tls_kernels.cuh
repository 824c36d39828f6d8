// tls_kernels.cuh — sm_100a device kernels of the two-level Schwarz Krylov hot path.
//
// Every per-iteration operator of the reference is one of the
// kernels below; all are HBM-bound fp64 (single right-hand side), so the design rules are
// coalesced 128-bit loads, enough bytes in flight per SM, and fixed-shape (deterministic)
// reductions.  File:line citations are into /root/reference/pkg/src/tlschwarz (src/...).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace tls {

// Programmatic dependent launch (sm_90+): every kernel waits for its predecessors' completion
// before touching memory; with the launch attribute set (tls_b200.cu launch_k) its launch is
// processed while the predecessor still runs (implicit trigger at the predecessor's end).  An
// explicit early trigger (TLS_PDL_EARLY_TRIGGER) let dependents occupy SM slots during
// multi-wave predecessors: measured -16% on GMRES configurations.  Without the attribute the
// wait is a no-op.
#ifndef TLS_PDL_EARLY_TRIGGER
#define PDL_ENTRY() asm volatile("griddepcontrol.wait;" ::: "memory")
#else
#define PDL_ENTRY()                                                          \
  do {                                                                       \
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");          \
    asm volatile("griddepcontrol.wait;" ::: "memory");                       \
  } while (0)
#endif

constexpr int TT = 64;          // tile edge (64x64 fp64 = 32 KiB, column-major inside)
constexpr int UR = 8;           // tile-rows per work unit
constexpr int UW = 8;           // tile-cols per work unit
constexpr int SLOTS_PER_UNIT = UR + UW;
constexpr int NTHR = 256;
constexpr unsigned FULL = 0xffffffffu;

struct BlkDesc {                // one dense local operator (a subdomain or the coarse A0^{-1})
  const double* tiles;          // tile (I,J) at tiles + tile_index(I,J)*TT*TT
  long long xoff;               // offset of its local vector in xloc / yloc (multiple of TT)
  int n, nt, sym, pad_;
};
struct Unit { int blk, i0, j0, slot; short ni, nj, pad0, pad1; };  // tile-rows [i0, i0+ni) x cols [j0, j0+nj)
struct OutTile { int blk, J, beg, end; };   // reduce slots red[beg:end] into y tile J of blk

struct PcgState {
  double bnorm, tol, rz, alpha, beta, pap, rnorm, pad0;
  int it, maxit, done, converged, status, bad_it, pad1, pad2;
  double bad_val;
};

struct GmState {
  double bnorm, tol, rn, tolc, scale, hn;
  int m_cycle, k, total, maxit, restart, cycle_stop, done, converged, restarted, pad_;
};

__device__ __forceinline__ long long tile_index(int I, int J, int nt, int sym) {
  return sym ? (long long)I * (I + 1) / 2 + J : (long long)I * nt + J;
}

__device__ __forceinline__ double2 ldg_stream2(const double* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
               : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

// Deterministic block sum (fixed xor-butterfly then fixed warp order); result in all threads
// of warp 0.  Must be called by all threads of the block.
__device__ __forceinline__ double block_sum(double v, double* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  __syncthreads();
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < nw ? sh[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  }
  return v;
}

// Sum of np partials, fixed assignment; valid in thread 0.
__device__ __forceinline__ double sum_partials(const double* __restrict__ p, int np, double* sh) {
  double v = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) v += p[i];
  return block_sum(v, sh);
}

// ---------------------------------------------------------------------------------------
// K1  CSR SpMV  (replaces scipy csr_matvec behind SparseMat.matvec, src/sparsemat.py:125-129)
//   MODE 0: y = A x          MODE 1: y = b - A x       (src/krylov.py:88-89 replacement)
//   DOT  0: none   1: partial sum x.y   2: partial sum y.y
// LPR lanes per row (1 = thread per row), grid-stride over row groups with a fixed grid ->
// deterministic partials.
// ---------------------------------------------------------------------------------------
template <int LPR, int MODE, int DOT>
__global__ void __launch_bounds__(NTHR) k_spmv(int r0, int n, const int* __restrict__ rowptr,
                                               const int* __restrict__ col,
                                               const double* __restrict__ val,
                                               const double* __restrict__ x, double* __restrict__ y,
                                               const double* __restrict__ b,
                                               double* __restrict__ part, const int* done) {
  PDL_ENTRY();
  // rows [r0, n): the whole matrix, or this rank's owned row range on the sharded path
  if (done && *done) return;
  __shared__ double sh[32];
  const int g = threadIdx.x / LPR, gl = threadIdx.x % LPR;
  const int rows_per_block = NTHR / LPR;
  double dacc = 0.0;
  for (int row0 = r0 + blockIdx.x * rows_per_block; row0 < n; row0 += gridDim.x * rows_per_block) {
    const int row = row0 + g;
    double s = 0.0;
    if (row < n) {
      const int beg = __ldg(rowptr + row), end = __ldg(rowptr + row + 1);
      for (int e = beg + gl; e < end; e += LPR) s += __ldg(val + e) * __ldg(x + __ldg(col + e));
    }
#pragma unroll
    for (int o = LPR / 2; o > 0; o >>= 1) s += __shfl_xor_sync(FULL, s, o, LPR);
    if (row < n && gl == 0) {
      const double out = MODE == 1 ? __ldg(b + row) - s : s;
      y[row] = out;
      if (DOT == 1) dacc += x[row] * out;
      if (DOT == 2) dacc += out * out;
    }
  }
  if (DOT) {
    const double t = block_sum(dacc, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = t;
  }
}

// ---------------------------------------------------------------------------------------
// K2  overlap restriction r_i = R_i r for every subdomain at once (src/precond.py:118,
//     SubdomainMap.restrict src/partition.py:83-84).  gidx[p] = global row of padded local
//     position p, -1 on padding.
// ---------------------------------------------------------------------------------------
__global__ void __launch_bounds__(NTHR) k_gather(long long m, const int* __restrict__ gidx,
                                                 const double* __restrict__ r,
                                                 double* __restrict__ xloc, const int* done) {
  PDL_ENTRY();
  if (done && *done) return;
  for (long long p = blockIdx.x * (long long)NTHR + threadIdx.x; p < m;
       p += (long long)gridDim.x * NTHR) {
    const int gi = __ldg(gidx + p);
    xloc[p] = gi >= 0 ? __ldg(r + gi) : 0.0;
  }
}

// Block-tridiagonal coarse solve (tls_coarse_chain): z[r] -= sum_e val[e] * y[idx[e]] for the rows
// r in [r0, r1) of one sparse off-diagonal block row of A0 = Z^T A Z (src/coarse.py:158-183).
// One warp per row, lanes stride the row's entries, fixed xor-butterfly -> deterministic.
__global__ void __launch_bounds__(NTHR) k_chain_spmv(int r0, int r1, const int* __restrict__ ptr,
                                                     const int* __restrict__ idx,
                                                     const double* __restrict__ val,
                                                     const double* __restrict__ y, double* z,
                                                     const int* done) {
  PDL_ENTRY();
  if (done && *done) return;
  const int lane = threadIdx.x & 31;
  const int row = r0 + (int)((blockIdx.x * (unsigned)blockDim.x + threadIdx.x) >> 5);
  if (row >= r1) return;
  const int e0 = __ldg(ptr + row), e1 = __ldg(ptr + row + 1);
  double a0 = 0.0, a1 = 0.0;
  int e = e0 + lane;
  for (; e + 32 < e1; e += 64) {
    a0 += __ldg(val + e) * y[__ldg(idx + e)];
    a1 += __ldg(val + e + 32) * y[__ldg(idx + e + 32)];
  }
  if (e < e1) a0 += __ldg(val + e) * y[__ldg(idx + e)];
  double v = a0 + a1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  if (lane == 0 && e1 > e0) z[row] -= v;
}


// ---------------------------------------------------------------------------------------
// K5  coarse restriction c = Z^T r (CoarseSpace.restrict, src/coarse.py:40-41).  Z is
//     block-diagonal by subdomain with interior support (src/coarse.py:1-7): one CTA per
//     subdomain, Z_s stored column by column (k x n_int, each column contiguous) so every
//     load instruction is coalesced.  c lands in the coarse segment of xloc.
// ---------------------------------------------------------------------------------------
// one warp per coarse column (blockDim = 32 * max k, up to 1024): r_int is gathered once per
// subdomain into shared memory and every column is streamed by its own warp
__global__ void __launch_bounds__(1024) k_restrict(const long long* __restrict__ sub_idxoff,
                                                   const int* __restrict__ idx,
                                                   const int* __restrict__ nint,
                                                   const long long* __restrict__ zoff,
                                                   const int* __restrict__ kcnt,
                                                   const int* __restrict__ cstart,
                                                   const double* __restrict__ Z,
                                                   const double* __restrict__ r,
                                                   double* __restrict__ c, const int* done) {
  PDL_ENTRY();
  if (done && *done) return;
  extern __shared__ __align__(16) double rs[];  // r on this subdomain's interior
  // grid (subdomains, column groups): CTA (s, g) handles columns g*nw .. g*nw+nw-1 of Z_s
  const int s = blockIdx.x;
  const int ks = kcnt[s], ni = nint[s];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if ((int)blockIdx.y * nw >= ks) return;
  const int* id = idx + sub_idxoff[s];
  for (int p = threadIdx.x; p < ni; p += blockDim.x) rs[p] = __ldg(r + __ldg(id + p));
  __syncthreads();
  const long long zo = zoff[s];
  const double* zs = Z + zo;
  // even n_int and an even offset: every column starts 16-byte aligned -> 128-bit streaming loads,
  // 8 in flight per lane (4 KB per warp); otherwise 64-bit loads, 4 in flight
  const bool vec = ((ni | (int)(zo & 1)) & 1) == 0;
  for (int col = blockIdx.y * nw + warp; col < ks; col += nw * gridDim.y) {
    const double* zc = zs + (long long)col * ni;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    if (vec) {
      const int n2 = ni >> 1;
      const double2* rs2 = reinterpret_cast<const double2*>(rs);
      int p = lane;
      for (; p + 224 < n2; p += 256) {
        double2 z[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) z[u] = ldg_stream2(zc + 2 * (p + 32 * u));
#pragma unroll
        for (int u = 0; u < 8; u += 4) {
          const double2 r0 = rs2[p + 32 * u], r1 = rs2[p + 32 * (u + 1)];
          const double2 r2 = rs2[p + 32 * (u + 2)], r3 = rs2[p + 32 * (u + 3)];
          a0 += z[u].x * r0.x + z[u].y * r0.y;
          a1 += z[u + 1].x * r1.x + z[u + 1].y * r1.y;
          a2 += z[u + 2].x * r2.x + z[u + 2].y * r2.y;
          a3 += z[u + 3].x * r3.x + z[u + 3].y * r3.y;
        }
      }
      for (; p < n2; p += 32) {
        const double2 z = ldg_stream2(zc + 2 * p), r0 = rs2[p];
        a0 += z.x * r0.x + z.y * r0.y;
      }
    } else {
      int p = lane;
      for (; p + 96 < ni; p += 128) {  // 4 independent coalesced loads in flight per lane
        a0 += __ldg(zc + p) * rs[p];
        a1 += __ldg(zc + p + 32) * rs[p + 32];
        a2 += __ldg(zc + p + 64) * rs[p + 64];
        a3 += __ldg(zc + p + 96) * rs[p + 96];
      }
      for (; p < ni; p += 32) a0 += __ldg(zc + p) * rs[p];
    }
    double v = (a0 + a1) + (a2 + a3);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    if (lane == 0) c[cstart[s] + col] = v;
  }
}

// 8-value transpose-reduction across a warp: returns, in every lane, the full 32-lane sum
// of v[colsel(lane)], colsel = 4*bit4 + 2*bit3 + bit2 (9 shuffles instead of 40).
__device__ __forceinline__ double warp_reduce8(const double (&v)[8], int lane) {
  double w[4];
  const bool h16 = lane & 16;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const double keep = h16 ? v[i + 4] : v[i], send = h16 ? v[i] : v[i + 4];
    w[i] = keep + __shfl_xor_sync(FULL, send, 16);
  }
  const bool h8 = lane & 8;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const double keep = h8 ? w[i + 2] : w[i], send = h8 ? w[i] : w[i + 2];
    w[i] = keep + __shfl_xor_sync(FULL, send, 8);
  }
  const bool h4 = lane & 4;
  const double keep = h4 ? w[1] : w[0], send = h4 ? w[0] : w[1];
  double t = keep + __shfl_xor_sync(FULL, send, 4);
  t += __shfl_xor_sync(FULL, t, 2);
  t += __shfl_xor_sync(FULL, t, 1);
  return t;
}

// ---------------------------------------------------------------------------------------
// K3/K6  batched local solves y_i = A_ii^{-1} r_i and the coarse solve y = A0^{-1} c
//   (the factor_dense solve closures src/subdomain.py:80-89 called at src/precond.py:117-118,
//    CoarseSpace.solve_coarse src/coarse.py:46-49).
// Each operator is stored as 64x64 fp64 tiles (column-major inside a tile); symmetric
// operators keep only the lower triangle of tiles, so every stored byte is read ONCE per
// apply and used twice: row partial (y_I += S_IJ x_J) and column partial (y_J += S_IJ^T x_I).
// CTA = 8 warps; warp w owns tile columns [8w, 8w+8), lane l owns rows {2l, 2l+1}: each
// 128-bit load instruction of a warp covers 512 contiguous bytes.  Row partials stay in
// registers across the unit's tile-columns (one smem cross-warp sum per tile-row); column
// partials are completed inside the warp with warp_reduce8.  Partials go to fixed slots that
// k_reduce_tiles sums in a fixed order -> bit-reproducible.
// ---------------------------------------------------------------------------------------
__global__ void __launch_bounds__(NTHR, 2) k_symv_tiles(const BlkDesc* __restrict__ blks,
                                                        const Unit* __restrict__ units,
                                                        const double* __restrict__ x,
                                                        double* __restrict__ slots,
                                                        const int* done) {
  PDL_ENTRY();
  if (done && *done) return;
  __shared__ __align__(16) double xr[UR * TT];
  __shared__ __align__(16) double xc[UW * TT];
  __shared__ __align__(16) double red[NTHR / 32][TT];
  const Unit un = units[blockIdx.x];
  const BlkDesc b = blks[un.blk];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int I0 = un.i0, J0 = un.j0;
  const int nI = un.ni, nJ = un.nj;
  for (int t = threadIdx.x; t < UR * TT; t += NTHR) {
    xr[t] = t < nI * TT ? x[b.xoff + (long long)I0 * TT + t] : 0.0;
    xc[t] = t < nJ * TT ? x[b.xoff + (long long)J0 * TT + t] : 0.0;
  }
  __syncthreads();
  const int c0 = warp * 8;
  double cacc[UW];
#pragma unroll
  for (int j = 0; j < UW; ++j) cacc[j] = 0.0;
  for (int i = 0; i < nI; ++i) {
    const int I = I0 + i;
    const double xi0 = xr[i * TT + 2 * lane], xi1 = xr[i * TT + 2 * lane + 1];
    const int jmax = b.sym ? min(nJ, I - J0 + 1) : nJ;
    double ra0 = 0.0, ra1 = 0.0;
#pragma unroll
    for (int j = 0; j < UW; ++j) {
      if (j < jmax) {
        const int J = J0 + j;
        const double* tp = b.tiles + tile_index(I, J, b.nt, b.sym) * (TT * TT) + c0 * TT + 2 * lane;
        double2 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = ldg_stream2(tp + k * TT);
        const double2* xj2 = reinterpret_cast<const double2*>(xc + j * TT + c0);
        double xj[8];
#pragma unroll
        for (int k = 0; k < 4; ++k) { const double2 t2 = xj2[k]; xj[2 * k] = t2.x; xj[2 * k + 1] = t2.y; }
#pragma unroll
        for (int k = 0; k < 8; ++k) { ra0 += v[k].x * xj[k]; ra1 += v[k].y * xj[k]; }
        if (b.sym && J < I) {
          double cp[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) cp[k] = v[k].x * xi0 + v[k].y * xi1;
          cacc[j] += warp_reduce8(cp, lane);
        }
      }
    }
    // cross-warp sum of the row partial of tile-row I
    red[warp][2 * lane] = ra0;
    red[warp][2 * lane + 1] = ra1;
    __syncthreads();
    if (threadIdx.x < TT) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < NTHR / 32; ++w) s += red[w][threadIdx.x];
      slots[(long long)(un.slot + i) * TT + threadIdx.x] = s;
    }
    __syncthreads();
  }
  if (b.sym) {
    const int colsel = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
    if ((lane & 3) == 0) {
#pragma unroll
      for (int j = 0; j < UW; ++j)
        if (j < nJ) slots[(long long)(un.slot + UR + j) * TT + c0 + colsel] = cacc[j];
    }
  }
}

// Sum the slot partials of each output tile in list order (one warp per tile).
__global__ void __launch_bounds__(NTHR) k_reduce_tiles(const BlkDesc* __restrict__ blks,
                                                       const OutTile* __restrict__ outs, int nout,
                                                       const int* __restrict__ red,
                                                       const double* __restrict__ slots,
                                                       double* __restrict__ y, const int* done) {
  PDL_ENTRY();
  if (done && *done) return;
  const int o = blockIdx.x * (NTHR / 32) + (threadIdx.x >> 5);
  if (o >= nout) return;
  const int lane = threadIdx.x & 31;
  const OutTile ot = outs[o];
  double a0 = 0.0, a1 = 0.0;
  for (int q = ot.beg; q < ot.end; ++q) {
    const double2 v = *reinterpret_cast<const double2*>(slots + (long long)__ldg(red + q) * TT + 2 * lane);
    a0 += v.x;
    a1 += v.y;
  }
  double2* yp = reinterpret_cast<double2*>(y + blks[ot.blk].xoff + (long long)ot.J * TT + 2 * lane);
  *yp = make_double2(a0, a1);
}

// ---------------------------------------------------------------------------------------
// K4/K7  prolongation.  One-level part: z[g] = sum over the subdomains containing g (RAS:
// only the owner, the Boolean PoU src/precond.py:119-120) of y_s at g, added in ascending
// subdomain order exactly like np.add.at (src/precond.py:121) -> conflict-free pull, no
// atomics.  Coarse part: (Z yc)[g] = Z_owner[p, :] . yc[cols] (CoarseSpace.prolong,
// src/coarse.py:43-44).
//   MODE 0: z = one-level          1: z = one-level + coarse  (additive, src/precond.py:132)
//   MODE 2: z = coarse             3: z = (q + w) - coarse    (deflated, src/precond.py:134-136)
//   MODE 4: z = one-level + qv     (additive with the coarse part Z yc precomputed into qv by a
//           MODE 2 launch on the side branch that overlaps the local solves)
//   DOT: partial sum rdot[g] * z[g]
// ---------------------------------------------------------------------------------------
template <int MODE, int DOT>
__global__ void __launch_bounds__(NTHR, 8) k_prolong(int n, const int* __restrict__ pull_ptr,
                                                  const int* __restrict__ pull_pos,
                                                  const double* __restrict__ yloc,
                                                  const long long* __restrict__ zrow,
                                                  const int* __restrict__ zst,
                                                  const int* __restrict__ zk,
                                                  const int* __restrict__ zc,
                                                  const double* __restrict__ Z,
                                                  const double* __restrict__ yc,
                                                  const double* __restrict__ qv,
                                                  const double* __restrict__ wv,
                                                  const double* __restrict__ rdot,
                                                  double* __restrict__ z, double* __restrict__ part,
                                                  const int* done) {
  PDL_ENTRY();
  if (done && *done) return;
  __shared__ double sh[32];
  double dacc = 0.0;
  for (int g = blockIdx.x * NTHR + threadIdx.x; g < n; g += gridDim.x * NTHR) {
    double one = 0.0, cz = 0.0;
    if (MODE == 0 || MODE == 1 || MODE == 4) {
      const int beg = __ldg(pull_ptr + g), end = __ldg(pull_ptr + g + 1);
      for (int q = beg; q < end; ++q) one += __ldg(yloc + __ldg(pull_pos + q));
    }
    if (MODE >= 1 && MODE <= 3) {
      const long long zo = __ldg(zrow + g);
      if (zo >= 0) {
        const int k = __ldg(zk + g), c0 = __ldg(zc + g), st = __ldg(zst + g);
#pragma unroll 4
        for (int t = 0; t < k; ++t) cz += __ldg(Z + zo + (long long)t * st) * __ldg(yc + c0 + t);
      }
    }
    double out;
    if (MODE == 0) out = one;
    else if (MODE == 1) out = one + cz;
    else if (MODE == 2) out = cz;
    else if (MODE == 3) out = (qv[g] + wv[g]) - cz;
    else out = one + qv[g];
    z[g] = out;
    if (DOT) dacc += rdot[g] * out;
  }
  if (DOT) {
    const double t = block_sum(dacc, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = t;
  }
}

// ---------------------------------------------------------------------------------------
// Sharded path: the system is renumbered so every rank owns a contiguous row
// range; vectors enter/leave in the caller's numbering, and the halo / reverse-halo exchanges
// move only the rows a rank's SpMV, gathers and ASM prolongation touch.
// ---------------------------------------------------------------------------------------
// dst[nofo[g]] = src[g]  (caller numbering -> internal numbering, all rows)
__global__ void __launch_bounds__(NTHR) k_perm_in(int n, const int* __restrict__ nofo,
                                                  const double* __restrict__ src, double* __restrict__ dst) {
  PDL_ENTRY();
  for (int g = blockIdx.x * NTHR + threadIdx.x; g < n; g += gridDim.x * NTHR) dst[__ldg(nofo + g)] = src[g];
}
// dst[g] = src[nofo[g]] for owned rows, 0 elsewhere (completed by a sum all-reduce)
__global__ void __launch_bounds__(NTHR) k_perm_out(int n, const int* __restrict__ nofo, int r0, int r1,
                                                   const double* __restrict__ src, double* __restrict__ dst) {
  PDL_ENTRY();
  for (int g = blockIdx.x * NTHR + threadIdx.x; g < n; g += gridDim.x * NTHR) {
    const int i = __ldg(nofo + g);
    dst[g] = (i >= r0 && i < r1) ? src[i] : 0.0;
  }
}
// ---------------------------------------------------------------------------------------
// K11 helper: batched symmetric eigensolver for the small Rayleigh-Ritz matrices of the setup's
// subspace iteration (p x p, p <= 64; src/spectral.py:69-85 solves the full pencil with LAPACK
// instead).  One CTA per matrix, matrix + eigenvectors in shared memory; parallel cyclic Jacobi
// (round-robin pairing: p/2 disjoint rotations per round, p-1 rounds per sweep, the symmetric
// 2x2 Schur rotation of Golub & Van Loan 8.5.1), until the off-diagonal Frobenius norm is below
// 1e-15 of the whole; eigenvalues returned in descending order with their eigenvectors as
// columns of V (row-major p x p).  Replaces a host round trip per Ritz step.
// ---------------------------------------------------------------------------------------
constexpr int EJ_MAX = 64;
constexpr int EJ_LD = EJ_MAX + 1;

__global__ void __launch_bounds__(256) k_syevj_batched(const double* __restrict__ T, int p,
                                                       double* __restrict__ w, double* __restrict__ V,
                                                       int max_sweeps) {
  PDL_ENTRY();
  extern __shared__ __align__(16) double ej_smem[];
  double* A = ej_smem;                       // p x EJ_LD
  double* Q = ej_smem + EJ_MAX * EJ_LD;      // p x EJ_LD
  __shared__ double cs[EJ_MAX / 2], sn[EJ_MAX / 2], red[256];
  __shared__ int pi_[EJ_MAX / 2], qi_[EJ_MAX / 2];
  __shared__ int stop;
  const int b = blockIdx.x, tid = threadIdx.x;
  const double* Tb = T + (long long)b * p * p;
  for (int e = tid; e < p * p; e += 256) {
    const int i = e / p, j = e % p;
    A[i * EJ_LD + j] = 0.5 * (Tb[i * p + j] + Tb[j * p + i]);
    Q[i * EJ_LD + j] = i == j ? 1.0 : 0.0;
  }
  const int P = (p + 1) & ~1, np_ = P / 2;
  __syncthreads();
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    // convergence: off-diagonal vs total Frobenius norm
    double off = 0.0, tot = 0.0;
    for (int e = tid; e < p * p; e += 256) {
      const int i = e / p, j = e % p;
      const double a = A[i * EJ_LD + j];
      tot += a * a;
      if (i != j) off += a * a;
    }
    red[tid] = off;
    __syncthreads();
    for (int h = 128; h > 0; h >>= 1) {
      if (tid < h) red[tid] += red[tid + h];
      __syncthreads();
    }
    const double offs = red[0];
    __syncthreads();
    red[tid] = tot;
    __syncthreads();
    for (int h = 128; h > 0; h >>= 1) {
      if (tid < h) red[tid] += red[tid + h];
      __syncthreads();
    }
    if (tid == 0) stop = !(offs > 1e-30 * red[0]) ? 1 : 0;
    __syncthreads();
    if (stop) break;
    for (int r = 0; r < P - 1; ++r) {
      if (tid < np_) {  // round-robin pair tid of round r (player 0 fixed, the others rotate)
        const int m = tid;
        const int pa = m == 0 ? 0 : ((m - 1 + r) % (P - 1)) + 1;
        const int pb = ((P - 1 - m - 1 + r) % (P - 1)) + 1;
        int i = min(pa, pb), j = max(pa, pb);
        double c = 1.0, s = 0.0;
        if (j < p) {
          const double apq = A[i * EJ_LD + j];
          if (apq != 0.0) {
            const double tau = (A[j * EJ_LD + j] - A[i * EJ_LD + i]) / (2.0 * apq);
            const double t = tau >= 0.0 ? 1.0 / (tau + sqrt(1.0 + tau * tau)) : -1.0 / (-tau + sqrt(1.0 + tau * tau));
            c = 1.0 / sqrt(1.0 + t * t);
            s = t * c;
          }
        } else {
          j = i;  // dummy partner (odd p): identity
        }
        pi_[m] = i;
        qi_[m] = j;
        cs[m] = c;
        sn[m] = s;
      }
      __syncthreads();
      // A <- A J and Q <- Q J (columns i, j of every pair)
      for (int t = tid; t < p * np_; t += 256) {
        const int k = t / np_, m = t % np_;
        const int i = pi_[m], j = qi_[m];
        if (i == j) continue;
        const double c = cs[m], s = sn[m];
        const double aki = A[k * EJ_LD + i], akj = A[k * EJ_LD + j];
        A[k * EJ_LD + i] = c * aki - s * akj;
        A[k * EJ_LD + j] = s * aki + c * akj;
        const double qki = Q[k * EJ_LD + i], qkj = Q[k * EJ_LD + j];
        Q[k * EJ_LD + i] = c * qki - s * qkj;
        Q[k * EJ_LD + j] = s * qki + c * qkj;
      }
      __syncthreads();
      // A <- J^T A (rows i, j of every pair)
      for (int t = tid; t < p * np_; t += 256) {
        const int k = t / np_, m = t % np_;
        const int i = pi_[m], j = qi_[m];
        if (i == j) continue;
        const double c = cs[m], s = sn[m];
        const double aik = A[i * EJ_LD + k], ajk = A[j * EJ_LD + k];
        A[i * EJ_LD + k] = c * aik - s * ajk;
        A[j * EJ_LD + k] = s * aik + c * ajk;
      }
      __syncthreads();
    }
  }
  // descending order: rank of each eigenvalue (ties by index)
  for (int j = tid; j < p; j += 256) {
    const double d = A[j * EJ_LD + j];
    int rk = 0;
    for (int i = 0; i < p; ++i) {
      const double e = A[i * EJ_LD + i];
      rk += (e > d) || (e == d && i < j);
    }
    w[(long long)b * p + rk] = d;
    for (int k = 0; k < p; ++k) V[(long long)b * p * p + (long long)k * p + rk] = Q[k * EJ_LD + j];
  }
}

// ---------------------------------------------------------------------------------------
// K13: batched one-sided Jacobi SVD (Hestenes) for the SVD coarse modes (src/spectral.py:135-154
// takes LAPACK's thin SVD of the harmonic extension; here E = Q R first, then this kernel on the
// small R).  One CTA per matrix X (m x n, column-major, leading dimension m, in global memory --
// L1/L2 resident: 268^2 doubles on configuration 3), rotated in place: X <- X V with mutually
// orthogonal columns, so column j ends as sigma_j u_j and the left singular vectors need no
// accumulation.  Round-robin pairing: n/2 disjoint column pairs per round, one warp per pair
// (coalesced column reads, three dot products by warp shuffles, the rotation written back),
// n-1 rounds per sweep, sweeps until no pair has |x_i . x_j| > tol |x_i| |x_j|.  (Keeping the larger
// column of a rotated pair at the lower index -- de Rijk's device for the row-cyclic order -- was
// measured to DOUBLE the sweep count under the round-robin order: 30 vs 18 on a harmonic
// extension; the columns are ranked by norm after convergence instead.)
// sig[b*n + j] = |column j|; info[b] = sweeps used, or -1 if max_sweeps did not converge.
// ---------------------------------------------------------------------------------------
constexpr int SVJ_THREADS = 1024;
__global__ void __launch_bounds__(SVJ_THREADS) k_svdj_batched(double* __restrict__ Xall, int m, int n,
                                                              double* __restrict__ sig,
                                                              int* __restrict__ info, double tol,
                                                              int max_sweeps) {
  PDL_ENTRY();
  double* X = Xall + (long long)blockIdx.x * m * n;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = SVJ_THREADS / 32;
  const int P = (n + 1) & ~1, np_ = P / 2;
  int sweeps = -1;
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    int rotated = 0;
    for (int r = 0; r < P - 1; ++r) {
      int mine = 0;
      for (int q = warp; q < np_; q += NW) {
        const int pa = q == 0 ? 0 : ((q - 1 + r) % (P - 1)) + 1;
        const int pb = ((P - 2 - q + r) % (P - 1)) + 1;
        const int i = min(pa, pb), j = max(pa, pb);
        if (j >= n) continue;  // dummy partner (odd n)
        double* xi = X + (long long)i * m;
        double* xj = X + (long long)j * m;
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int k = lane; k < m; k += 32) {
          const double a = xi[k], b = xj[k];
          al += a * a;
          be += b * b;
          ga += a * b;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          al += __shfl_xor_sync(FULL, al, o);
          be += __shfl_xor_sync(FULL, be, o);
          ga += __shfl_xor_sync(FULL, ga, o);
        }
        if (!(fabs(ga) > tol * sqrt(al) * sqrt(be))) continue;  // also when a column is zero
        const double zeta = (be - al) / (2.0 * ga);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
        mine = 1;
        for (int k = lane; k < m; k += 32) {
          const double a = xi[k], b = xj[k];
          xi[k] = c * a - s * b;
          xj[k] = s * a + c * b;
        }
      }
      rotated += __syncthreads_count(mine);
    }
    if (rotated == 0) {
      sweeps = sweep + 1;
      break;
    }
  }
  for (int j = warp; j < n; j += NW) {
    const double* xj = X + (long long)j * m;
    double al = 0.0;
    for (int k = lane; k < m; k += 32) al += xj[k] * xj[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) al += __shfl_xor_sync(FULL, al, o);
    if (lane == 0) sig[(long long)blockIdx.x * n + j] = sqrt(al);
  }
  if (threadIdx.x == 0) info[blockIdx.x] = sweeps;
}

// sharded dot products: part[0] = fixed-order sum of part[0..np), part[1..np) = 0 (one CTA)
__global__ void __launch_bounds__(NTHR) k_fold_partials(double* __restrict__ part, int np) {
  PDL_ENTRY();
  __shared__ double red[NTHR];
  double s = 0.0;
  for (int i = threadIdx.x; i < np; i += NTHR) s += part[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = NTHR / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  for (int i = threadIdx.x; i < np; i += NTHR) part[i] = i == 0 ? red[0] : 0.0;
}

// sharded coarse restriction: c[ccol[q] + i] = recv[q * cmax + i] for i < ccol[q+1] - ccol[q]
__global__ void __launch_bounds__(NTHR) k_coarse_unpack(long long tot, long long cmax,
                                                        const long long* __restrict__ ccol,
                                                        const double* __restrict__ recv,
                                                        double* __restrict__ c, const int* done) {
  PDL_ENTRY();
  if (done && *done) return;
  for (long long j = blockIdx.x * (long long)NTHR + threadIdx.x; j < tot; j += (long long)gridDim.x * NTHR) {
    const long long q = j / cmax, i = j - q * cmax;
    if (i < ccol[q + 1] - ccol[q]) c[ccol[q] + i] = recv[j];
  }
}

// out = a + beta * b (b may be null: a copy); coarse-segment arithmetic of the refinement step
__global__ void __launch_bounds__(NTHR) k_lincomb(int n, const double* __restrict__ a,
                                                  const double* __restrict__ b, double beta,
                                                  double* __restrict__ out, const int* done) {
  PDL_ENTRY();
  if (done && *done) return;
  for (int i = blockIdx.x * NTHR + threadIdx.x; i < n; i += gridDim.x * NTHR)
    out[i] = b ? a[i] + beta * b[i] : a[i];
}
__global__ void __launch_bounds__(NTHR) k_xpack(long long m, const int* __restrict__ idx,
                                                const double* __restrict__ src, double* __restrict__ buf,
                                                const int* done) {
  PDL_ENTRY();
  if (done && *done) return;
  for (long long p = blockIdx.x * (long long)NTHR + threadIdx.x; p < m; p += (long long)gridDim.x * NTHR)
    buf[p] = src[__ldg(idx + p)];
}
__global__ void __launch_bounds__(NTHR) k_xunpack(long long m, const int* __restrict__ idx,
                                                  const double* __restrict__ buf, double* __restrict__ dst,
                                                  const int* done) {
  PDL_ENTRY();
  if (done && *done) return;
  for (long long p = blockIdx.x * (long long)NTHR + threadIdx.x; p < m; p += (long long)gridDim.x * NTHR)
    dst[__ldg(idx + p)] = buf[p];
}


// ---------------------------------------------------------------------------------------
// K8  Krylov vector kernels and scalar steps (src/krylov.py:58-107)
// ---------------------------------------------------------------------------------------
template <int DOT>  // z = r (precond None, src/krylov.py:52-55); DOT: partial r.z
__global__ void __launch_bounds__(NTHR) k_copy_dot(int n, const double* __restrict__ r,
                                                   double* __restrict__ z, double* __restrict__ part,
                                                   const int* done) {
  PDL_ENTRY();
  if (done && *done) return;
  __shared__ double sh[32];
  double acc = 0.0;
  for (int i = blockIdx.x * NTHR + threadIdx.x; i < n; i += gridDim.x * NTHR) {
    const double v = r[i];
    z[i] = v;
    if (DOT) acc += v * v;
  }
  if (DOT) {
    const double t = block_sum(acc, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(NTHR) k_dot(int n, const double* __restrict__ a,
                                              const double* __restrict__ b,
                                              double* __restrict__ part, const int* done) {
  PDL_ENTRY();
  if (done && *done) return;
  __shared__ double sh[32];
  double acc = 0.0;
  for (int i = blockIdx.x * NTHR + threadIdx.x; i < n; i += gridDim.x * NTHR) acc += a[i] * b[i];
  const double t = block_sum(acc, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = t;
}

// PCG scalars ------------------------------------------------------------------------------
__global__ void k_pcg_init(PcgState* st, const double* part, int np) {
  PDL_ENTRY();
  __shared__ double sh[32];
  const double s = sum_partials(part, np, sh);
  if (threadIdx.x == 0) {
    st->bnorm = sqrt(s);
    st->it = 0;
    st->done = st->bnorm == 0.0 ? 1 : 0;
    st->converged = st->done;
    st->status = 0;
  }
}
__global__ void k_pcg_rz0(PcgState* st, const double* part, int np) {
  PDL_ENTRY();
  __shared__ double sh[32];
  const double s = sum_partials(part, np, sh);
  if (threadIdx.x == 0) st->rz = s;
}
// curvature p.Ap -> alpha; BreakdownError when <= 0 (src/krylov.py:81-85)
__global__ void k_pcg_alpha(PcgState* st, const double* part, int np, double* ab) {
  PDL_ENTRY();
  if (st->done) return;
  __shared__ double sh[32];
  const double s = sum_partials(part, np, sh);
  if (threadIdx.x == 0) {
    st->it += 1;
    st->pap = s;
    if (!(s > 0.0)) {
      st->status = 2;
      st->bad_it = st->it;
      st->bad_val = s;
      st->done = 1;
    } else {
      st->alpha = st->rz / s;
      ab[2 * (st->it - 1)] = st->alpha;
    }
  }
}
// x += alpha p; r -= alpha Ap; partial r.r (src/krylov.py:86-87)
__global__ void __launch_bounds__(NTHR) k_pcg_update(int n, const PcgState* st, double* __restrict__ x,
                                                     double* __restrict__ r,
                                                     const double* __restrict__ p,
                                                     const double* __restrict__ ap,
                                                     double* __restrict__ part, int update_r) {
  PDL_ENTRY();
  if (st->done) return;
  __shared__ double sh[32];
  const double alpha = st->alpha;
  double acc = 0.0;
  for (int i = blockIdx.x * NTHR + threadIdx.x; i < n; i += gridDim.x * NTHR) {
    x[i] += alpha * p[i];
    if (update_r) {
      const double rv = r[i] - alpha * ap[i];
      r[i] = rv;
      acc += rv * rv;
    }
  }
  if (update_r) {
    const double t = block_sum(acc, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = t;
  }
}
// history entry and stopping test (src/krylov.py:90-96)
__global__ void k_pcg_hist(PcgState* st, const double* part, int np, double* hist) {
  PDL_ENTRY();
  if (st->done) return;
  __shared__ double sh[32];
  const double s = sum_partials(part, np, sh);
  if (threadIdx.x == 0) {
    st->rnorm = sqrt(s);
    const double h = st->rnorm / st->bnorm;
    hist[st->it] = h;
    if (h <= st->tol) {
      st->converged = 1;
      st->done = 1;
    } else if (st->it >= st->maxit) {
      st->done = 1;
    }
  }
}
__global__ void k_pcg_beta(PcgState* st, const double* part, int np, double* ab) {
  PDL_ENTRY();
  if (st->done) return;
  __shared__ double sh[32];
  const double s = sum_partials(part, np, sh);
  if (threadIdx.x == 0) {
    st->beta = s / st->rz;
    ab[2 * (st->it - 1) + 1] = st->beta;
    st->rz = s;
  }
}
// p = z + beta p (src/krylov.py:101)
__global__ void __launch_bounds__(NTHR) k_pcg_pupdate(int n, const PcgState* st, double* __restrict__ p,
                                                      const double* __restrict__ z) {
  PDL_ENTRY();
  if (st->done) return;
  const double beta = st->beta;
  for (int i = blockIdx.x * NTHR + threadIdx.x; i < n; i += gridDim.x * NTHR) p[i] = z[i] + beta * p[i];
}

// ---------------------------------------------------------------------------------------
// GMRES (src/krylov.py:127-195): Arnoldi with classical Gram-Schmidt twice (CGS2 — the
// reference's MGS + correction pass, src/krylov.py:157-165, to the same accuracy), Givens
// rotations, both stopping rules, x += M^{-1} V y at the end of each cycle.
// ---------------------------------------------------------------------------------------
constexpr int GCH = 8;  // columns per gemv_t pass
// part[i*G + block] = partial V[:, i] . w for i < ncols
__global__ void __launch_bounds__(NTHR, 8) k_gm_gemvt(int n, const double* __restrict__ V, long long ldv,
                                                   int ncols, const double* __restrict__ w,
                                                   double* __restrict__ part, const int* stop) {
  PDL_ENTRY();
  if (*stop) return;
  __shared__ double sh[NTHR / 32][GCH];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int c0 = 0; c0 < ncols; c0 += GCH) {
    double acc[GCH];
#pragma unroll
    for (int k = 0; k < GCH; ++k) acc[k] = 0.0;
    for (int i = blockIdx.x * NTHR + threadIdx.x; i < n; i += gridDim.x * NTHR) {
      const double wv = w[i];
#pragma unroll
      for (int k = 0; k < GCH; ++k)
        if (c0 + k < ncols) acc[k] += V[(long long)(c0 + k) * ldv + i] * wv;
    }
#pragma unroll
    for (int k = 0; k < GCH; ++k) {
      double v = acc[k];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
      if (lane == 0) sh[warp][k] = v;
    }
    __syncthreads();
    if (threadIdx.x < GCH && c0 + threadIdx.x < ncols) {
      double v = 0.0;
#pragma unroll
      for (int q = 0; q < NTHR / 32; ++q) v += sh[q][threadIdx.x];
      part[(long long)(c0 + threadIdx.x) * gridDim.x + blockIdx.x] = v;
    }
    __syncthreads();
  }
}
// CGS2 middle step, one read of V instead of two: w -= V[:, :ncols] h (pass-1 update) and the
// pass-2 projections part[i*G + block] = partial V[:, i] . w_new.  Rows go through shared memory
// in tiles of NTHR: the tile of V (ncols x NTHR, coalesced column loads) is used for the update
// of its rows and, after a barrier, for the dot products (warp c reduces columns c, c+8, ...),
// accumulated per CTA in a fixed tile order -> deterministic.  Dynamic smem: (ncols+1)*NTHR + ncols doubles.
__global__ void __launch_bounds__(NTHR) k_gm_update_gemvt(int n, const double* __restrict__ V, long long ldv,
                                                          int ncols, const double* __restrict__ h,
                                                          double* __restrict__ w, double* __restrict__ part,
                                                          const int* stop) {
  PDL_ENTRY();
  if (*stop) return;
  extern __shared__ __align__(16) double smv[];
  double* vt = smv;                       // ncols x NTHR
  double* wt = smv + (long long)ncols * NTHR;
  double* acc = wt + NTHR;                // ncols
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int c = threadIdx.x; c < ncols; c += NTHR) acc[c] = 0.0;
  for (long long row0 = (long long)blockIdx.x * NTHR; row0 < n; row0 += (long long)gridDim.x * NTHR) {
    const long long i = row0 + threadIdx.x;
    double s = 0.0;
    if (i < n) {
      for (int c = 0; c < ncols; ++c) {
        const double v = V[(long long)c * ldv + i];
        vt[c * NTHR + threadIdx.x] = v;
        s += v * __ldg(h + c);
      }
      const double out = w[i] - s;
      w[i] = out;
      wt[threadIdx.x] = out;
    } else {
      for (int c = 0; c < ncols; ++c) vt[c * NTHR + threadIdx.x] = 0.0;
      wt[threadIdx.x] = 0.0;
    }
    __syncthreads();
    for (int c = warp; c < ncols; c += NTHR / 32) {
      double d = 0.0;
#pragma unroll
      for (int r = lane; r < NTHR; r += 32) d += vt[c * NTHR + r] * wt[r];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(FULL, d, o);
      if (lane == 0) acc[c] += d;
    }
    __syncthreads();
  }
  for (int c = threadIdx.x; c < ncols; c += NTHR) part[(long long)c * gridDim.x + blockIdx.x] = acc[c];
}

// h[i] = sum_b part[i*G + b]; one block per column
__global__ void k_gm_hreduce(const double* __restrict__ part, int G, double* __restrict__ h,
                             const int* stop) {
  PDL_ENTRY();
  if (*stop) return;
  __shared__ double sh[32];
  const double s = sum_partials(part + (long long)blockIdx.x * G, G, sh);
  if (threadIdx.x == 0) h[blockIdx.x] = s;
}
// w -= V[:, :ncols] h  (ncols < 0: read the count from st->k); optional partial w.w
template <int NORM>
__global__ void __launch_bounds__(NTHR, 8) k_gm_gemvn(int n, const double* __restrict__ V, long long ldv,
                                                   int ncols, const GmState* st,
                                                   const double* __restrict__ h,
                                                   double* __restrict__ w, double* __restrict__ part,
                                                   int subtract, const int* stop) {
  PDL_ENTRY();
  if (stop && *stop) return;
  __shared__ double sh[32];
  const int nc = ncols >= 0 ? ncols : st->k;
  double acc2 = 0.0;
  for (int i = blockIdx.x * NTHR + threadIdx.x; i < n; i += gridDim.x * NTHR) {
    double s = 0.0;
    for (int c = 0; c < nc; ++c) s += V[(long long)c * ldv + i] * __ldg(h + c);
    const double out = subtract ? w[i] - s : s;
    w[i] = out;
    if (NORM) acc2 += out * out;
  }
  if (NORM) {
    const double t = block_sum(acc2, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = t;
  }
}
// Hessenberg column j, rotations, residual estimate, both stopping tests (src/krylov.py:166-189)
__global__ void k_gm_givens(GmState* st, int j, int ldh, double* __restrict__ H,
                            const double* __restrict__ h1, const double* __restrict__ h2,
                            const double* __restrict__ part, int np, double* __restrict__ cs,
                            double* __restrict__ sn, double* __restrict__ g, double* __restrict__ hist) {
  PDL_ENTRY();
  if (st->cycle_stop) return;
  __shared__ double sh[32];
  const double s = sum_partials(part, np, sh);
  if (threadIdx.x != 0) return;
  double* hc = H + (long long)j * ldh;
  for (int i = 0; i <= j; ++i) hc[i] = h1[i] + h2[i];
  const double hn = sqrt(s);
  st->hn = hn;
  hc[j + 1] = hn;
  for (int i = 0; i < j; ++i) {
    const double t = cs[i] * hc[i] + sn[i] * hc[i + 1];
    hc[i + 1] = -sn[i] * hc[i] + cs[i] * hc[i + 1];
    hc[i] = t;
  }
  const double den = hypot(hc[j], hc[j + 1]);
  cs[j] = den != 0.0 ? hc[j] / den : 1.0;
  sn[j] = den != 0.0 ? hc[j + 1] / den : 0.0;
  hc[j] = den;
  hc[j + 1] = 0.0;
  g[j + 1] = -sn[j] * g[j];
  g[j] = cs[j] * g[j];
  st->k = j + 1;
  const double rel = fabs(g[j + 1]) / st->rn;
  hist[st->total + j + 1] = st->restarted ? rel * st->scale : rel;
  if (rel <= st->tolc) {
    st->converged = 1;
    st->cycle_stop = 1;
  } else if (hn <= 1e-14 * st->rn) {
    st->converged = 1;  // happy breakdown (src/krylov.py:187-189)
    st->cycle_stop = 1;
  } else if (j + 1 >= st->m_cycle) {
    st->cycle_stop = 1;
  }
}
// Givens step + v_{j+1} = w / hn in ONE launch of G CTAs: every CTA sums the same norm partials in
// the same fixed order (bit-identical hn everywhere), CTA 0 thread 0 updates the Hessenberg column,
// the rotations and the stopping tests exactly as k_gm_givens, and all CTAs scale their rows.  When
// this step ends the cycle the scaled column is simply never read (a CTA that already sees
// cycle_stop = 1 from CTA 0 may skip its rows).
__global__ void __launch_bounds__(NTHR) k_gm_givens_scale(GmState* st, int j, int ldh, double* __restrict__ H,
                                                          const double* __restrict__ h1,
                                                          const double* __restrict__ h2,
                                                          const double* __restrict__ part, int np,
                                                          double* __restrict__ cs, double* __restrict__ sn,
                                                          double* __restrict__ g, double* __restrict__ hist,
                                                          int n, const double* __restrict__ w,
                                                          double* __restrict__ v) {
  PDL_ENTRY();
  if (*(volatile int*)&st->cycle_stop) return;
  __shared__ double sh[32];
  __shared__ double hn_s;
  const double s = sum_partials(part, np, sh);
  if (threadIdx.x == 0) hn_s = sqrt(s);
  __syncthreads();
  const double hn = hn_s;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double* hc = H + (long long)j * ldh;
    for (int i = 0; i <= j; ++i) hc[i] = h1[i] + h2[i];
    st->hn = hn;
    hc[j + 1] = hn;
    for (int i = 0; i < j; ++i) {
      const double t = cs[i] * hc[i] + sn[i] * hc[i + 1];
      hc[i + 1] = -sn[i] * hc[i] + cs[i] * hc[i + 1];
      hc[i] = t;
    }
    const double den = hypot(hc[j], hc[j + 1]);
    cs[j] = den != 0.0 ? hc[j] / den : 1.0;
    sn[j] = den != 0.0 ? hc[j + 1] / den : 0.0;
    hc[j] = den;
    hc[j + 1] = 0.0;
    g[j + 1] = -sn[j] * g[j];
    g[j] = cs[j] * g[j];
    st->k = j + 1;
    const double rel = fabs(g[j + 1]) / st->rn;
    hist[st->total + j + 1] = st->restarted ? rel * st->scale : rel;
    if (rel <= st->tolc) {
      st->converged = 1;
      st->cycle_stop = 1;
    } else if (hn <= 1e-14 * st->rn) {
      st->converged = 1;  // happy breakdown (src/krylov.py:187-189)
      st->cycle_stop = 1;
    } else if (j + 1 >= st->m_cycle) {
      st->cycle_stop = 1;
    }
  }
  if (hn == 0.0) return;
  for (int i = blockIdx.x * NTHR + threadIdx.x; i < n; i += gridDim.x * NTHR) v[i] = w[i] / hn;
}
// v_{j+1} = w / hn
__global__ void __launch_bounds__(NTHR) k_gm_scale(int n, const GmState* st, const double* __restrict__ w,
                                                   double* __restrict__ v, int use_rn) {
  PDL_ENTRY();
  if (!use_rn && st->cycle_stop) return;
  const double d = use_rn ? st->rn : st->hn;
  for (int i = blockIdx.x * NTHR + threadIdx.x; i < n; i += gridDim.x * NTHR) v[i] = w[i] / d;
}
// y = H[:k,:k]^{-1} g[:k] (solve_triangular, src/krylov.py:191)
__global__ void k_gm_trisolve(const GmState* st, int ldh, const double* __restrict__ H,
                              const double* __restrict__ g, double* __restrict__ y) {
  PDL_ENTRY();
  if (threadIdx.x != 0) return;
  const int k = st->k;
  for (int i = k - 1; i >= 0; --i) {
    double s = g[i];
    for (int l = i + 1; l < k; ++l) s -= H[(long long)l * ldh + i] * y[l];
    y[i] = s / H[(long long)i * ldh + i];
  }
}
__global__ void __launch_bounds__(NTHR) k_axpy1(int n, double* __restrict__ x, const double* __restrict__ t,
                                                const int* done) {
  PDL_ENTRY();
  if (done && *done) return;
  for (int i = blockIdx.x * NTHR + threadIdx.x; i < n; i += gridDim.x * NTHR) x[i] += t[i];
}
// end of a cycle: account iterations, decide whether to restart
__global__ void k_gm_cycle_end(GmState* st) {
  PDL_ENTRY();
  if (threadIdx.x != 0) return;
  st->total += st->k;
  if (st->converged || st->total >= st->maxit || !st->restarted) st->done = 1;
}
// new cycle on r = b - A x: rn, tolerance rescale, V_0 = r / rn, g = rn e1
__global__ void k_gm_cycle_begin(GmState* st, const double* part, int np, double* g, int mcols) {
  PDL_ENTRY();
  if (st->done) return;
  __shared__ double sh[32];
  const double s = sum_partials(part, np, sh);
  if (threadIdx.x != 0) return;
  st->rn = sqrt(s);
  if (st->rn == 0.0) {
    st->done = 1;
    st->converged = 1;
    return;
  }
  st->tolc = st->restarted ? st->tol * st->bnorm / st->rn : st->tol;
  st->scale = st->rn / st->bnorm;
  int m = st->maxit - st->total;
  if (st->restarted && st->restart < m) m = st->restart;
  if (m > mcols) m = mcols;
  st->m_cycle = m;
  st->k = 0;
  st->cycle_stop = 0;
  for (int i = 0; i <= mcols; ++i) g[i] = 0.0;
  g[0] = st->rn;
}

// ---------------------------------------------------------------------------------------
// Setup kernels (src/subdomain.py:53-69 extraction; tile packing of local inverses)
// ---------------------------------------------------------------------------------------
// local-index lookup for the extraction: the batch's global index lists are sorted per
// subdomain (keys) together with their local positions (vals); a CSR column is then found by a
// binary search in its subdomain's sorted list -- no n-sized map per subdomain.
__global__ void k_seg_prep(int count, const long long* __restrict__ sub_idxoff, const int* __restrict__ sub_n,
                           int first, int* __restrict__ beg, int* __restrict__ end, int* __restrict__ pos) {
  PDL_ENTRY();
  const int b = blockIdx.y;
  const int s = first + b;
  const long long base = sub_idxoff[first];
  const int o = (int)(sub_idxoff[s] - base), ns = sub_n[s];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    beg[b] = o;
    end[b] = o + ns;
  }
  for (int l = blockIdx.x * NTHR + threadIdx.x; l < ns; l += gridDim.x * NTHR) pos[o + l] = l;
}
__device__ __forceinline__ int seg_find(const int* __restrict__ keys, int n, int c) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (keys[mid] < c) lo = mid + 1;
    else hi = mid;
  }
  return (lo < n && keys[lo] == c) ? lo : -1;
}
__global__ void k_extract(int count, const long long* __restrict__ sub_idxoff,
                          const int* __restrict__ sub_n, const int* __restrict__ idx, int first,
                          const int* __restrict__ skey, const int* __restrict__ sval,
                          const int* __restrict__ rowptr, const int* __restrict__ col,
                          const double* __restrict__ val, double* __restrict__ out, long long ld) {
  PDL_ENTRY();
  const int b = blockIdx.y;
  const int s = first + b;
  const int ns = sub_n[s];
  const int* id = idx + sub_idxoff[s];
  const int o = (int)(sub_idxoff[s] - sub_idxoff[first]);
  const int* kb = skey + o;
  const int* vb = sval + o;
  double* ob = out + (long long)b * ld * ld;
  const int warp = (blockIdx.x * NTHR + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int nwarps = gridDim.x * (NTHR / 32);
  for (int l = warp; l < (int)ld; l += nwarps) {
    if (l >= ns) {
      if (lane == 0) ob[(long long)l * ld + l] = 1.0;
      continue;
    }
    const int g = id[l];
    for (int e = rowptr[g] + lane; e < rowptr[g + 1]; e += 32) {
      const int q = seg_find(kb, ns, col[e]);
      if (q >= 0) ob[(long long)l * ld + vb[q]] = val[e];
    }
  }
}
// tile (I,J) of subdomain s <- inv[b] (row-major ld x ld), zero outside n_s.  One CTA per tile:
// coalesced row reads into shared memory, column-major (tile layout) coalesced writes.
__global__ void k_pack_tiles(const BlkDesc* __restrict__ blks, int first_blk, const double* __restrict__ inv,
                             long long ld, long long batch_stride) {
  PDL_ENTRY();
  __shared__ double tile[TT][TT + 1];
  const int b = blockIdx.y;
  const BlkDesc bd = blks[first_blk + b];
  const long long ntiles = bd.sym ? (long long)bd.nt * (bd.nt + 1) / 2 : (long long)bd.nt * bd.nt;
  const double* src = inv + b * batch_stride;
  for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
    int I, J;
    if (bd.sym) {
      I = (int)floor((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
      while ((long long)(I + 1) * (I + 2) / 2 <= t) ++I;
      while ((long long)I * (I + 1) / 2 > t) --I;
      J = (int)(t - (long long)I * (I + 1) / 2);
    } else {
      I = (int)(t / bd.nt);
      J = (int)(t % bd.nt);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < TT * TT; e += NTHR) {
      const int r = e / TT, c = e % TT;  // row-major walk: consecutive threads, consecutive columns
      const int gi = I * TT + r, gj = J * TT + c;
      tile[r][c] = (gi < bd.n && gj < bd.n) ? src[(long long)gi * ld + gj] : 0.0;
    }
    __syncthreads();
    double* dst = const_cast<double*>(bd.tiles) + t * (TT * TT);
    for (int e = threadIdx.x; e < TT * TT; e += NTHR) {
      const int c = e / TT, r = e % TT;  // column-major tile layout
      dst[e] = tile[r][c];
    }
  }
}

// ---------------------------------------------------------------------------------------
// K3b  banded Cholesky local solves y_i = A_ii^{-1} r_i = L^{-T} L^{-1} r_i for SPD blocks
// (the cho_solve closure of src/subdomain.py:80-82, same factorisation, other row order).
// The local rows are ordered lexicographically by global index (a plane sweep for grid
// operators), so the Cholesky factor lives in a band of ~one grid plane.  Per 64-row block I
// the factor is stored as one contiguous "step": K_I panel tiles L[I, I-K_I .. I-1] and the
// inverse of the diagonal tile (64x64 fp64, column-major).  One CTA per subdomain keeps the
// whole local vector in shared memory and sweeps: forward u_I = D_I^{-1}(v_I - panel.u) with
// row partials (lane-local, cross-warp smem sum), backward y_J = D_J^{-T} v_J and
// v_{J-k} -= L_{J,J-k}^T y_J with column partials completed inside the warp (warp_reduce8).
// Both sweeps stream every stored byte once; the loads do not depend on the solve, only the
// FMAs do, and 4 CTAs per SM overlap one CTA's barriers with the others' loads.
// ---------------------------------------------------------------------------------------
struct BandDesc {
  const double* data;          // L steps of this subdomain (forward order)
  const long long* step_off;   // nb offsets (doubles) into data
  const int* kcnt;             // nb codes: K_I | (first nonzero 8-column panel strip << 16)
  long long xoff;              // offset of the local vector in xloc / yloc
  int n, nb, pad0, pad1;
  // LU only (nonsymmetric blocks): U steps stored in backward-sweep order (block nb-1 first)
  const double* udata;         // null for Cholesky (backward sweep uses L^T)
  const long long* ustep_off;  // nb offsets, indexed by block row I
  const int* ucnt;             // nb codes: R_I | (number of all-zero trailing strips << 16)
};

// bulk L2 prefetch (TMA engine, no registers): pull the next step's factor block into L2
__device__ __forceinline__ void prefetch_l2(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// inverted diagonal tile, lower triangular: warp w's 8-column strip is stored from row 8w on
constexpr int DIAG_PACK = 2304;  // = sum_w 8 * (64 - 8w)
__device__ __forceinline__ int diag_strip_off(int w) { return 512 * w - 32 * w * (w - 1); }
// L2 prefetch of item j of step I of an L stream in forward order (item j < K_I: panel tile j
// without its leading zero strips, j == K_I: the packed diagonal), spilling into later steps.
__device__ __forceinline__ void prefetch_fwd_item(const BandDesc& b, int I, int j) {
  while (I < b.nb) {
    const int code = b.kcnt[I], K = code & 0xffff, fz = code >> 16;
    if (j <= K) {
      const double* base = b.data + b.step_off[I];
      if (j == K) {
        prefetch_l2(base + (long long)K * TT * TT, 8u * DIAG_PACK);
      } else {
        const int z = j == 0 ? min(fz, 8) : 0;
        if (z < 8) prefetch_l2(base + (long long)j * TT * TT + z * 8 * TT, 8u * (unsigned)((8 - z) * 8 * TT));
      }
      return;
    }
    j -= K + 1;
    ++I;
  }
}
// backward (Cholesky L^T) order per step J: diagonal first, then panel tiles 0..K-1; steps descend
__device__ __forceinline__ void prefetch_bwd_item(const BandDesc& b, int J, int j) {
  while (J >= 0) {
    const int code = b.kcnt[J], K = code & 0xffff, fz = code >> 16;
    if (j <= K) {
      const double* base = b.data + b.step_off[J];
      if (j == 0) {
        prefetch_l2(base + (long long)K * TT * TT, 8u * DIAG_PACK);
      } else {
        const int t = j - 1, z = t == 0 ? min(fz, 8) : 0;
        if (z < 8) prefetch_l2(base + (long long)t * TT * TT + z * 8 * TT, 8u * (unsigned)((8 - z) * 8 * TT));
      }
      return;
    }
    j -= K + 1;
    --J;
  }
}
// backward (LU, U stream) order per step I: panel tiles 0..R-1 (trailing zero strips dropped),
// then the packed diagonal; steps descend
__device__ __forceinline__ void prefetch_u_item(const BandDesc& b, int I, int j) {
  while (I >= 0) {
    const int code = b.ucnt[I], R = code & 0xffff, tz = code >> 16;
    if (j <= R) {
      const double* base = b.udata + b.ustep_off[I];
      if (j == R) {
        prefetch_l2(base + (long long)R * TT * TT, 8u * DIAG_PACK);
      } else {
        const int keep = j == R - 1 ? 8 - min(tz, 8) : 8;
        if (keep > 0) prefetch_l2(base + (long long)j * TT * TT, 8u * (unsigned)(keep * 8 * TT));
      }
      return;
    }
    j -= R + 1;
    --I;
  }
}

// inverted diagonal tile, upper triangular: warp w's strip keeps rows 0 .. 8w+7
__device__ __forceinline__ int udiag_strip_off(int w) { return 32 * w * w + 32 * w; }

// pf: L2 prefetch distance in items (2 measured best; TLS_BAND_PF overrides for sweeps)
// gidx != nullptr: the restriction R_i r is fused into the load (v[p] = r[gidx[xoff + p]],
// K2 without its own launch and without the xloc round trip); otherwise v = x[xoff ...]
// UNR = tiles loaded per round (1: 64 registers, 4 CTAs/SM -- many subdomains per GPU; 2: two
// tiles in flight per warp, 2 CTAs/SM -- few subdomain CTAs per SM, where one CTA's sweep is the
// critical path).  Both accumulate in the same order (bit-identical results).
template <int UNR>
__global__ void __launch_bounds__(NTHR, UNR == 1 ? 4 : 2) k_band_solve(const BandDesc* __restrict__ bands,
                                                        const double* __restrict__ x,
                                                        double* __restrict__ y, const int* done,
                                                        int pf, const int* __restrict__ gidx,
                                                        const double* __restrict__ r) {
  PDL_ENTRY();
  if (done && *done) return;
  extern __shared__ __align__(16) double sm[];
  const BandDesc b = bands[blockIdx.x];
  const int npad = b.nb * TT;
  double* v = sm;                  // npad
  double* red = sm + npad;         // 8 x 64
  double* t = red + 8 * TT;        // 64
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, c0 = warp * 8;
  const int dlen = TT - 8 * warp;                    // rows stored in this warp's diagonal strip
  const bool drow = lane >= 4 * warp;                // rows 2l, 2l+1 inside the strip
  const int doff = diag_strip_off(warp) + (2 * lane - 8 * warp);
  if (threadIdx.x == 0)
    for (int j = 2; j < pf; ++j) prefetch_fwd_item(b, 0, j);  // items >= 2 of the stream head
  if (gidx) {
    for (int i = threadIdx.x; i < npad; i += NTHR) {
      const int g = __ldg(gidx + b.xoff + i);
      v[i] = g >= 0 ? __ldg(r + g) : 0.0;
    }
  } else {
    for (int i = threadIdx.x; i < npad; i += NTHR) v[i] = x[b.xoff + i];
  }
  __syncthreads();
  // forward sweep: L u = x  (the factor is one contiguous stream in this order)
  for (int I = 0; I < b.nb; ++I) {
    const double* blk = b.data + b.step_off[I];
    const int code = b.kcnt[I], K = code & 0xffff, fz = code >> 16;
    double ra0 = 0.0, ra1 = 0.0;
    for (int k = 0; k < K; k += UNR) {
      if (threadIdx.x == 0) {                        // pf items ahead, into L2
        prefetch_fwd_item(b, I, k + pf);
        if (UNR == 2 && k + 1 < K) prefetch_fwd_item(b, I, k + 1 + pf);
      }
      double2 w[UNR][8];
      bool act[UNR];
#pragma unroll
      for (int q = 0; q < UNR; ++q) {
        act[q] = k + q < K && !((k + q) * 8 + warp < fz);  // strips left of the profile: zeros
        if (act[q]) {
          const double* tp = blk + (long long)(k + q) * TT * TT + c0 * TT + 2 * lane;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) w[q][kk] = ldg_stream2(tp + kk * TT);
        }
      }
#pragma unroll
      for (int q = 0; q < UNR; ++q) {
        if (!act[q]) continue;
        const double* uj = v + (I - K + k + q) * TT + c0;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) { ra0 += w[q][kk].x * uj[kk]; ra1 += w[q][kk].y * uj[kk]; }
      }
    }
    if (threadIdx.x == 0) prefetch_fwd_item(b, I, K + pf);
    red[warp * TT + 2 * lane] = ra0;
    red[warp * TT + 2 * lane + 1] = ra1;
    __syncthreads();
    if (threadIdx.x < TT) {
      double sacc = v[I * TT + threadIdx.x];
#pragma unroll
      for (int w = 0; w < 8; ++w) sacc -= red[w * TT + threadIdx.x];
      t[threadIdx.x] = sacc;
    }
    __syncthreads();
    {
      double d0 = 0.0, d1 = 0.0;
      if (drow) {
        const double* dp = blk + (long long)K * TT * TT + doff;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const double2 w = ldg_stream2(dp + kk * dlen);
          d0 += w.x * t[c0 + kk];
          d1 += w.y * t[c0 + kk];
        }
      }
      red[warp * TT + 2 * lane] = d0;
      red[warp * TT + 2 * lane + 1] = d1;
    }
    __syncthreads();
    if (threadIdx.x < TT) {
      double sacc = 0.0;
#pragma unroll
      for (int w = 0; w < 8; ++w) sacc += red[w * TT + threadIdx.x];
      v[I * TT + threadIdx.x] = sacc;
    }
    __syncthreads();
  }
  if (b.udata) {
    // backward sweep with U (LU): y_I = U_II^{-1} (u_I - sum_k U[I, I+1+k] y_{I+1+k}), row partials
    const int ulen = 8 * warp + 8;                   // rows stored in this warp's upper strip
    const bool urow = lane <= 4 * warp + 3;
    const int uoff = udiag_strip_off(warp) + 2 * lane;
    for (int I = b.nb - 1; I >= 0; --I) {
      const double* blk = b.udata + b.ustep_off[I];
      const int code = b.ucnt[I], R = code & 0xffff, tz = code >> 16;
      double ra0 = 0.0, ra1 = 0.0;
      for (int k = 0; k < R; k += UNR) {
        if (threadIdx.x == 0) {
          prefetch_u_item(b, I, k + pf);
          if (UNR == 2 && k + 1 < R) prefetch_u_item(b, I, k + 1 + pf);
        }
        double2 w[UNR][8];
        bool act[UNR];
#pragma unroll
        for (int q = 0; q < UNR; ++q) {
          act[q] = k + q < R && !((k + q) * 8 + warp >= 8 * R - tz);  // right of the profile
          if (act[q]) {
            const double* tp = blk + (long long)(k + q) * TT * TT + c0 * TT + 2 * lane;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) w[q][kk] = ldg_stream2(tp + kk * TT);
          }
        }
#pragma unroll
        for (int q = 0; q < UNR; ++q) {
          if (!act[q]) continue;
          const double* yj = v + (I + 1 + k + q) * TT + c0;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) { ra0 += w[q][kk].x * yj[kk]; ra1 += w[q][kk].y * yj[kk]; }
        }
      }
      if (threadIdx.x == 0) prefetch_u_item(b, I, R + pf);
      red[warp * TT + 2 * lane] = ra0;
      red[warp * TT + 2 * lane + 1] = ra1;
      __syncthreads();
      if (threadIdx.x < TT) {
        double sacc = v[I * TT + threadIdx.x];
#pragma unroll
        for (int w = 0; w < 8; ++w) sacc -= red[w * TT + threadIdx.x];
        t[threadIdx.x] = sacc;
      }
      __syncthreads();
      {
        double d0 = 0.0, d1 = 0.0;
        if (urow) {
          const double* dp = blk + (long long)R * TT * TT + uoff;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const double2 w = ldg_stream2(dp + kk * ulen);
            d0 += w.x * t[c0 + kk];
            d1 += w.y * t[c0 + kk];
          }
        }
        red[warp * TT + 2 * lane] = d0;
        red[warp * TT + 2 * lane + 1] = d1;
      }
      __syncthreads();
      if (threadIdx.x < TT) {
        double sacc = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) sacc += red[w * TT + threadIdx.x];
        v[I * TT + threadIdx.x] = sacc;
      }
      __syncthreads();
    }
    for (int i = threadIdx.x; i < npad; i += NTHR) y[b.xoff + i] = v[i];
    return;
  }
  // backward sweep: L^T y = u
  const int colsel = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
  for (int J = b.nb - 1; J >= 0; --J) {
    const double* blk = b.data + b.step_off[J];
    const int code = b.kcnt[J], K = code & 0xffff, fz = code >> 16;
    if (threadIdx.x == 0) prefetch_bwd_item(b, J, pf);
    {
      const double u0 = v[J * TT + 2 * lane], u1 = v[J * TT + 2 * lane + 1];
      double cp[8];
      if (drow) {
        const double* dp = blk + (long long)K * TT * TT + doff;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const double2 w = ldg_stream2(dp + kk * dlen);
          cp[kk] = w.x * u0 + w.y * u1;
        }
      } else {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) cp[kk] = 0.0;
      }
      const double yv = warp_reduce8(cp, lane);
      __syncthreads();  // every warp has read v_J
      if ((lane & 3) == 0) v[J * TT + c0 + colsel] = yv;
      __syncthreads();
    }
    const double y0 = v[J * TT + 2 * lane], y1 = v[J * TT + 2 * lane + 1];
    for (int k = 0; k < K; k += UNR) {
      if (threadIdx.x == 0) {
        prefetch_bwd_item(b, J, k + 1 + pf);
        if (UNR == 2 && k + 1 < K) prefetch_bwd_item(b, J, k + 2 + pf);
      }
      double2 w[UNR][8];
      bool act[UNR];
#pragma unroll
      for (int q = 0; q < UNR; ++q) {
        act[q] = k + q < K && !((k + q) * 8 + warp < fz);
        if (act[q]) {
          const double* tp = blk + (long long)(k + q) * TT * TT + c0 * TT + 2 * lane;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) w[q][kk] = ldg_stream2(tp + kk * TT);
        }
      }
#pragma unroll
      for (int q = 0; q < UNR; ++q) {
        if (!act[q]) continue;
        double cp[8];
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) cp[kk] = w[q][kk].x * y0 + w[q][kk].y * y1;
        const double val = warp_reduce8(cp, lane);
        if ((lane & 3) == 0) v[(J - K + k + q) * TT + c0 + colsel] -= val;
      }
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < npad; i += NTHR) y[b.xoff + i] = v[i];
}

// ---------------------------------------------------------------------------------------
// K9 prologue: the dense block in its factor order, lower triangle only, and its row profile, in
// ONE pass: AP[b, i, j] = A[b, P[b,i], P[b,j]] for j <= i (0 above the diagonal: the factor
// kernels never read it and the band packing expects zeros there), first[b, i] = the smallest j
// with a nonzero.  Replaces two torch gathers, a != 0 mask, an argmax and a masked fill over the
// (count, ld, ld) batch (51 -> ~6 ms per batch of 54 on configuration 5).  One CTA per row.
// ---------------------------------------------------------------------------------------
__global__ void __launch_bounds__(NTHR) k_perm_lower(const double* __restrict__ A,
                                                     const long long* __restrict__ P,
                                                     double* __restrict__ AP, int* __restrict__ first,
                                                     int ld) {
  PDL_ENTRY();
  __shared__ int red[NTHR / 32];
  const int b = blockIdx.y, i = blockIdx.x;
  const long long* Pb = P + (long long)b * ld;
  const double* arow = A + ((long long)b * ld + Pb[i]) * ld;
  double* orow = AP + ((long long)b * ld + i) * ld;
  int fm = ld;
  for (int j = threadIdx.x; j < ld; j += NTHR) {
    const double v = j <= i ? arow[Pb[j]] : 0.0;
    orow[j] = v;
    if (v != 0.0 && j < fm) fm = j;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) fm = min(fm, __shfl_xor_sync(FULL, fm, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = fm;
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int w = 1; w < NTHR / 32; ++w) fm = min(fm, red[w]);
    first[(long long)b * ld + i] = fm == ld ? 0 : fm;
  }
}

// ---------------------------------------------------------------------------------------
// K9  Banded Cholesky of a batch of SPD blocks (setup; src/subdomain.py:80-82 in the factor
//     order), one CTA per block, the whole right-looking blocked factorisation in ONE launch:
//     per 64-column panel J, the 64 x 64 diagonal block is factored and inverted in shared
//     memory, the panel below it (rows up to reach[J], the band's lowest reach) becomes
//     P L_JJ^{-T}, and the trailing band square is updated T -= P P^T -- the two tile products
//     on the FP64 tensor cores (DMMA, mma.sync.m8n8k4.f64).  Rows/columns outside the envelope
//     stay zero (no fill outside the profile).  Writes the factor in place (lower; the strict
//     upper part of the diagonal blocks is cleared), the inverted diagonal
//     blocks to dinv (nbk x 64 x 64 row-major per block) and info = 1-based row of the first
//     non-positive pivot (0: SPD).  Dynamic smem: 5 padded 64 x 65 tiles.
// ---------------------------------------------------------------------------------------
constexpr int CP = 65;  // padded smem tile row
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
// acc(64 x 64) = X (64 x 64, smem, padded) * Y^T (Y 64 x 64, smem, padded); warp w owns output
// rows 8w..8w+7 (8 blocks of 8 x 8, 16 doubles per lane)
__device__ __forceinline__ void tile_xyt(const double* X, const double* Y, double (&acc)[8][2]) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, gr = lane >> 2, gc = lane & 3;
#pragma unroll
  for (int bj = 0; bj < 8; ++bj) acc[bj][0] = acc[bj][1] = 0.0;
#pragma unroll 4
  for (int k0 = 0; k0 < 64; k0 += 4) {
    const double a = X[(8 * w + gr) * CP + k0 + gc];
#pragma unroll
    for (int bj = 0; bj < 8; ++bj) dmma_8x8x4(acc[bj][0], acc[bj][1], a, Y[(8 * bj + gr) * CP + k0 + gc]);
  }
}
__device__ __forceinline__ void load_tile(double* T, const double* G, long long ld) {
  for (int e = threadIdx.x; e < 64 * 64; e += blockDim.x) T[(e >> 6) * CP + (e & 63)] = G[(long long)(e >> 6) * ld + (e & 63)];
}

// CL > 1: a thread-block cluster of CL CTAs per subdomain (blockIdx.x / CL).  Rank 0 factors and
// inverts the 64 x 64 diagonal block and publishes L_JJ / L_JJ^{-1} through global memory (L2);
// the panel tiles and the trailing-band tile products -- the bulk of the work, ~mt^2/2 tile
// products per panel -- are dealt round-robin to the CL CTAs; three cluster barriers per panel
// (barrier.cluster arrive.release / wait.acquire order the global writes at cluster scope).
// CL = 1 is the single-CTA kernel.
template <int CL>
__device__ __forceinline__ void k9_sync() {
  if (CL > 1) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  } else {
    __syncthreads();
  }
}

template <int CL>
__global__ void __launch_bounds__(256, 1) k_band_chol(double* __restrict__ AP, long long ld, const int* __restrict__ reach,
                                                      int nbk, double* __restrict__ dinv, int* __restrict__ info) {
  PDL_ENTRY();
  extern __shared__ __align__(16) double cs[];
  double* Ds = cs;                 // diagonal block -> L_JJ (lower)
  double* Ls = Ds + 64 * CP;       // L_JJ^{-1}
  double* Ta = Ls + 64 * CP;
  double* Tb = Ta + 64 * CP;
  __shared__ int bad;
  const int sub = blockIdx.x / CL, crank = blockIdx.x % CL;
  double* A = AP + (long long)sub * ld * ld;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, gr = lane >> 2, gc = lane & 3;
  if (tid == 0) bad = 0;
  for (int J = 0; J < nbk; ++J) {
    const long long j0 = 64LL * J;
    double* dv = dinv + ((long long)sub * nbk + J) * 4096;
    if (crank == 0) {
      load_tile(Ds, A + j0 * ld + j0, ld);
      __syncthreads();
      // 64 x 64 Cholesky in shared memory, blocked by 8 columns (right-looking, lower triangle):
      // the 8 x 8 diagonal block by warp 0 (lane = row, warp-synchronous), the 8-column panel
      // below it by one thread per row, the trailing triangle by all threads
      for (int c0 = 0; c0 < 64; c0 += 8) {
        if (w == 0) {
          for (int k = 0; k < 8; ++k) {
            const int kk = c0 + k;
            if (lane == 0) {
              double d = Ds[kk * CP + kk];
              if (!(d > 0.0)) {
                if (bad == 0) bad = (int)(j0 + kk + 1);
                d = 1.0;  // keep going without NaNs; the caller raises on info
              }
              Ds[kk * CP + kk] = sqrt(d);
            }
            __syncwarp();
            const double piv = Ds[kk * CP + kk];
            if (lane > k && lane < 8) Ds[(c0 + lane) * CP + kk] /= piv;
            __syncwarp();
            if (lane > k && lane < 8) {
              const double lik = Ds[(c0 + lane) * CP + kk];
              for (int j = k + 1; j <= lane; ++j) Ds[(c0 + lane) * CP + c0 + j] -= lik * Ds[(c0 + j) * CP + kk];
            }
            __syncwarp();
          }
        }
        __syncthreads();
        for (int r = c0 + 8 + tid; r < 64; r += blockDim.x) {
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            double v = Ds[r * CP + c0 + k];
            for (int q = 0; q < k; ++q) v -= Ds[r * CP + c0 + q] * Ds[(c0 + k) * CP + c0 + q];
            Ds[r * CP + c0 + k] = v / Ds[(c0 + k) * CP + c0 + k];
          }
        }
        __syncthreads();
        const int m = 56 - c0;
        for (int e = tid; e < m * m; e += blockDim.x) {
          const int i = c0 + 8 + e / m, j = c0 + 8 + e % m;
          if (j <= i) {
            double acc = 0.0;
#pragma unroll
            for (int q = 0; q < 8; ++q) acc += Ds[i * CP + c0 + q] * Ds[j * CP + c0 + q];
            Ds[i * CP + j] -= acc;
          }
        }
        __syncthreads();
      }
      // L_JJ^{-1}: column j by the 4 lanes 4j..4j+3 (forward substitution, each row's dot product
      // split 4 ways and completed by two xor-shuffles)
      {
        const int j = tid >> 2, sl = tid & 3;
        for (int i = 0; i < 64; ++i) {
          double part = 0.0;
          if (i > j)
            for (int q = j + sl; q < i; q += 4) part += Ds[i * CP + q] * Ls[q * CP + j];
          part += __shfl_xor_sync(FULL, part, 1);
          part += __shfl_xor_sync(FULL, part, 2);
          if (sl == 0) Ls[i * CP + j] = i < j ? 0.0 : (i == j ? 1.0 / Ds[j * CP + j] : -part / Ds[i * CP + i]);
          __syncwarp();
        }
      }
      __syncthreads();
      for (int e = tid; e < 64 * 64; e += blockDim.x) {
        const int r = e >> 6, c = e & 63;
        A[(j0 + r) * ld + j0 + c] = c <= r ? Ds[r * CP + c] : 0.0;  // strict upper part cleared
        dv[e] = Ls[r * CP + c];
      }
    }
    k9_sync<CL>();  // L_JJ and L_JJ^{-1} published
    if (crank != 0) {
      for (int e = tid; e < 64 * 64; e += blockDim.x) Ls[(e >> 6) * CP + (e & 63)] = dv[e];
      __syncthreads();
    }
    const int mt = (int)((reach[J] - j0 - 64) / 64);
    // panel: P_t <- P_t L_JJ^{-T}, tiles dealt round-robin over the cluster
    for (int t = crank; t < mt; t += CL) {
      double* G = A + (j0 + 64 + 64LL * t) * ld + j0;
      __syncthreads();
      load_tile(Ta, G, ld);
      __syncthreads();
      double acc[8][2];
      tile_xyt(Ta, Ls, acc);
#pragma unroll
      for (int bj = 0; bj < 8; ++bj) {
        G[(long long)(8 * w + gr) * ld + 8 * bj + 2 * gc] = acc[bj][0];
        G[(long long)(8 * w + gr) * ld + 8 * bj + 2 * gc + 1] = acc[bj][1];
      }
    }
    k9_sync<CL>();  // the whole panel is final
    // trailing band square: T(ti, tj) -= P_ti P_tj^T, tj <= ti, tile products round-robin
    int q = 0, loaded = -1;
    for (int ti = 0; ti < mt; ++ti) {
      for (int tj = 0; tj <= ti; ++tj, ++q) {
        if (q % CL != crank) continue;
        if (loaded != ti) {
          __syncthreads();
          load_tile(Ta, A + (j0 + 64 + 64LL * ti) * ld + j0, ld);
          loaded = ti;
        }
        double* G = A + (j0 + 64 + 64LL * ti) * ld + j0 + 64 + 64LL * tj;
        load_tile(Tb, A + (j0 + 64 + 64LL * tj) * ld + j0, ld);
        __syncthreads();
        double acc[8][2];
        tile_xyt(Ta, Tb, acc);
#pragma unroll
        for (int bj = 0; bj < 8; ++bj) {
          G[(long long)(8 * w + gr) * ld + 8 * bj + 2 * gc] -= acc[bj][0];
          G[(long long)(8 * w + gr) * ld + 8 * bj + 2 * gc + 1] -= acc[bj][1];
        }
        __syncthreads();
      }
    }
    k9_sync<CL>();  // the trailing update is complete before the next diagonal block is read
  }
  if (tid == 0 && crank == 0) info[sub] = bad;
}

// ---------------------------------------------------------------------------------------
// K3d  k_band_solve_ring<S>: the same sweeps as k_band_solve, but every warp streams ITS slice of
//      the panel tiles (8 columns x 64 rows = 4 KB) through a private S-deep shared-memory ring
//      with cp.async (16 B per lane, one commit group per tile): S tiles are always in flight per
//      warp, across step boundaries (the tiles do not depend on the solve), so a sweep never
//      waits on DRAM latency when one CTA holds an SM -- the regime of few subdomains per GPU
//      (ncu on k_band_solve there: long-scoreboard + barrier stalls, 37% L2 hits).  One CTA per
//      SM (ring + local vector); same arithmetic order as k_band_solve (bit-identical results).
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// producer cursor over one stream of panel tiles (forward: L by ascending steps; bwd: L by
// descending steps; U: U by descending steps); issues this warp's slice of the next tile
struct RingProducer {
  int I, k, slot;
  __device__ __forceinline__ void issue(const BandDesc& b, int mode, double* ring, int warp, int lane, int S) {
    const int c0 = warp * 8;
    // advance to the next existing tile
    while (I >= 0 && I < b.nb) {
      const int code = mode == 2 ? b.ucnt[I] : b.kcnt[I];
      const int K = code & 0xffff;
      if (k < K) break;
      I += mode == 0 ? 1 : -1;
      k = 0;
    }
    if (I >= 0 && I < b.nb) {
      const int code = mode == 2 ? b.ucnt[I] : b.kcnt[I];
      const int K = code & 0xffff, z = code >> 16;
      const bool zero = mode == 2 ? (k * 8 + warp >= 8 * K - z) : (k * 8 + warp < z);
      if (!zero) {
        const double* base = mode == 2 ? b.udata + b.ustep_off[I] : b.data + b.step_off[I];
        const double* tp = base + (long long)k * TT * TT + c0 * TT + 2 * lane;
        double* dst = ring + (long long)slot * 512 + 2 * lane;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) cp_async16(dst + kk * 64, tp + kk * TT);
      }
      ++k;
    }
    cp_async_commit();  // (possibly empty) group: one per consumed position
    slot = slot + 1 == S ? 0 : slot + 1;
  }
};

template <int S>
__global__ void __launch_bounds__(NTHR, S <= 2 ? 2 : 1) k_band_solve_ring(const BandDesc* __restrict__ bands,
                                                             const double* __restrict__ x,
                                                             double* __restrict__ y, const int* done,
                                                             const int* __restrict__ gidx,
                                                             const double* __restrict__ r) {
  PDL_ENTRY();
  if (done && *done) return;
  extern __shared__ __align__(16) double sm[];
  const BandDesc b = bands[blockIdx.x];
  const int npad = b.nb * TT;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, c0 = warp * 8;
  double* ringw = sm + (long long)warp * S * 512;  // this warp's ring (S x 512 doubles)
  double* v = sm + 8 * S * 512;
  double* red = v + npad;
  double* t = red + 8 * TT;
  const int dlen = TT - 8 * warp;
  const bool drow = lane >= 4 * warp;
  const int doff = diag_strip_off(warp) + (2 * lane - 8 * warp);
  RingProducer prod{0, 0, 0};
#pragma unroll
  for (int q = 0; q < S; ++q) prod.issue(b, 0, ringw, warp, lane, S);
  if (gidx) {
    for (int i = threadIdx.x; i < npad; i += NTHR) {
      const int g = __ldg(gidx + b.xoff + i);
      v[i] = g >= 0 ? __ldg(r + g) : 0.0;
    }
  } else {
    for (int i = threadIdx.x; i < npad; i += NTHR) v[i] = x[b.xoff + i];
  }
  __syncthreads();
  int cs = 0;
  // forward sweep
  for (int I = 0; I < b.nb; ++I) {
    const double* blk = b.data + b.step_off[I];
    const int code = b.kcnt[I], K = code & 0xffff, fz = code >> 16;
    double ra0 = 0.0, ra1 = 0.0;
    for (int k = 0; k < K; ++k) {
      cp_async_wait<S - 1>();
      if (!(k * 8 + warp < fz)) {
        const double* rs = ringw + (long long)cs * 512 + 2 * lane;
        const double* uj = v + (I - K + k) * TT + c0;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const double2 w = *reinterpret_cast<const double2*>(rs + kk * 64);
          ra0 += w.x * uj[kk];
          ra1 += w.y * uj[kk];
        }
      }
      cs = cs + 1 == S ? 0 : cs + 1;
      prod.issue(b, 0, ringw, warp, lane, S);
    }
    red[warp * TT + 2 * lane] = ra0;
    red[warp * TT + 2 * lane + 1] = ra1;
    __syncthreads();
    if (threadIdx.x < TT) {
      double sacc = v[I * TT + threadIdx.x];
#pragma unroll
      for (int w = 0; w < 8; ++w) sacc -= red[w * TT + threadIdx.x];
      t[threadIdx.x] = sacc;
    }
    __syncthreads();
    {
      double d0 = 0.0, d1 = 0.0;
      if (drow) {
        const double* dp = blk + (long long)K * TT * TT + doff;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const double2 w = ldg_stream2(dp + kk * dlen);
          d0 += w.x * t[c0 + kk];
          d1 += w.y * t[c0 + kk];
        }
      }
      red[warp * TT + 2 * lane] = d0;
      red[warp * TT + 2 * lane + 1] = d1;
    }
    __syncthreads();
    if (threadIdx.x < TT) {
      double sacc = 0.0;
#pragma unroll
      for (int w = 0; w < 8; ++w) sacc += red[w * TT + threadIdx.x];
      v[I * TT + threadIdx.x] = sacc;
    }
    __syncthreads();
  }
  cp_async_wait<0>();  // drain the (empty) tail groups before the ring is reused
  if (b.udata) {
    const int ulen = 8 * warp + 8;
    const bool urow = lane <= 4 * warp + 3;
    const int uoff = udiag_strip_off(warp) + 2 * lane;
    RingProducer up{b.nb - 1, 0, 0};
#pragma unroll
    for (int q = 0; q < S; ++q) up.issue(b, 2, ringw, warp, lane, S);
    cs = 0;
    for (int I = b.nb - 1; I >= 0; --I) {
      const double* blk = b.udata + b.ustep_off[I];
      const int code = b.ucnt[I], R = code & 0xffff, tz = code >> 16;
      double ra0 = 0.0, ra1 = 0.0;
      for (int k = 0; k < R; ++k) {
        cp_async_wait<S - 1>();
        if (!(k * 8 + warp >= 8 * R - tz)) {
          const double* rs = ringw + (long long)cs * 512 + 2 * lane;
          const double* yj = v + (I + 1 + k) * TT + c0;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const double2 w = *reinterpret_cast<const double2*>(rs + kk * 64);
            ra0 += w.x * yj[kk];
            ra1 += w.y * yj[kk];
          }
        }
        cs = cs + 1 == S ? 0 : cs + 1;
        up.issue(b, 2, ringw, warp, lane, S);
      }
      red[warp * TT + 2 * lane] = ra0;
      red[warp * TT + 2 * lane + 1] = ra1;
      __syncthreads();
      if (threadIdx.x < TT) {
        double sacc = v[I * TT + threadIdx.x];
#pragma unroll
        for (int w = 0; w < 8; ++w) sacc -= red[w * TT + threadIdx.x];
        t[threadIdx.x] = sacc;
      }
      __syncthreads();
      {
        double d0 = 0.0, d1 = 0.0;
        if (urow) {
          const double* dp = blk + (long long)R * TT * TT + uoff;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const double2 w = ldg_stream2(dp + kk * ulen);
            d0 += w.x * t[c0 + kk];
            d1 += w.y * t[c0 + kk];
          }
        }
        red[warp * TT + 2 * lane] = d0;
        red[warp * TT + 2 * lane + 1] = d1;
      }
      __syncthreads();
      if (threadIdx.x < TT) {
        double sacc = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) sacc += red[w * TT + threadIdx.x];
        v[I * TT + threadIdx.x] = sacc;
      }
      __syncthreads();
    }
    cp_async_wait<0>();
    for (int i = threadIdx.x; i < npad; i += NTHR) y[b.xoff + i] = v[i];
    return;
  }
  // Cholesky backward: L^T y = u
  const int colsel = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
  RingProducer bp{b.nb - 1, 0, 0};
#pragma unroll
  for (int q = 0; q < S; ++q) bp.issue(b, 1, ringw, warp, lane, S);
  cs = 0;
  for (int J = b.nb - 1; J >= 0; --J) {
    const double* blk = b.data + b.step_off[J];
    const int code = b.kcnt[J], K = code & 0xffff, fz = code >> 16;
    {
      const double u0 = v[J * TT + 2 * lane], u1 = v[J * TT + 2 * lane + 1];
      double cp[8];
      if (drow) {
        const double* dp = blk + (long long)K * TT * TT + doff;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const double2 w = ldg_stream2(dp + kk * dlen);
          cp[kk] = w.x * u0 + w.y * u1;
        }
      } else {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) cp[kk] = 0.0;
      }
      const double yv = warp_reduce8(cp, lane);
      __syncthreads();  // every warp has read v_J
      if ((lane & 3) == 0) v[J * TT + c0 + colsel] = yv;
      __syncthreads();
    }
    const double y0 = v[J * TT + 2 * lane], y1 = v[J * TT + 2 * lane + 1];
    for (int k = 0; k < K; ++k) {
      cp_async_wait<S - 1>();
      if (!(k * 8 + warp < fz)) {
        const double* rs = ringw + (long long)cs * 512 + 2 * lane;
        double cp[8];
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const double2 w = *reinterpret_cast<const double2*>(rs + kk * 64);
          cp[kk] = w.x * y0 + w.y * y1;
        }
        const double val = warp_reduce8(cp, lane);
        if ((lane & 3) == 0) v[(J - K + k) * TT + c0 + colsel] -= val;
      }
      cs = cs + 1 == S ? 0 : cs + 1;
      bp.issue(b, 1, ringw, warp, lane, S);
    }
    __syncthreads();
  }
  cp_async_wait<0>();
  for (int i = threadIdx.x; i < npad; i += NTHR) y[b.xoff + i] = v[i];
}

// ---------------------------------------------------------------------------------------
// K3e  k_band_solve_tma<S>: the per-warp rings of k_band_solve_ring fed by the TMA engine.  A
//      warp's slice of a panel tile is 8 columns x 64 rows = 4 KB CONTIGUOUS in the packed factor,
//      so one elected lane issues ONE bulk copy per tile (cp.async.bulk.shared.global with
//      mbarrier::complete_tx, SASS UBLKCP) instead of 8 x 32 16-byte cp.async (LDGSTS); each ring
//      slot has its own mbarrier (arrival count 1: the producer's expect_tx; tiles skipped as
//      zero strips arrive without bytes), consumers spin on try_wait.parity.  The slot is refilled
//      by the same warp after its lanes have consumed it (program order inside the warp), so no
//      "empty" barrier is needed.  Same sweeps and arithmetic order as k_band_solve / _ring.
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  unsigned ok;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// producer cursor over one stream of panel tiles (modes as RingProducer); one bulk copy per tile
struct TmaProducer {
  int I, k, slot;
  __device__ __forceinline__ void issue(const BandDesc& b, int mode, double* ring, unsigned long long* bars, int warp,
                                        int lane, int S) {
    const int c0 = warp * 8;
    while (I >= 0 && I < b.nb) {
      const int code = mode == 2 ? b.ucnt[I] : b.kcnt[I];
      const int K = code & 0xffff;
      if (k < K) break;
      I += mode == 0 ? 1 : -1;
      k = 0;
    }
    bool copy = false;
    const double* tp = nullptr;
    if (I >= 0 && I < b.nb) {
      const int code = mode == 2 ? b.ucnt[I] : b.kcnt[I];
      const int K = code & 0xffff, z = code >> 16;
      const bool zero = mode == 2 ? (k * 8 + warp >= 8 * K - z) : (k * 8 + warp < z);
      if (!zero) {
        const double* base = mode == 2 ? b.udata + b.ustep_off[I] : b.data + b.step_off[I];
        tp = base + (long long)k * TT * TT + c0 * TT;
        copy = true;
      }
      ++k;
    }
    __syncwarp();  // every lane has consumed the slot's previous tile
    if (lane == 0) {
      if (copy) {
        mbar_expect_tx(bars + slot, 4096u);
        bulk_g2s(ring + (long long)slot * 512, tp, 4096u, bars + slot);
      } else {
        mbar_arrive(bars + slot);  // (skipped or past-the-end item: the phase completes without bytes)
      }
    }
    slot = slot + 1 == S ? 0 : slot + 1;
  }
};

template <int S>
__global__ void __launch_bounds__(NTHR, 1) k_band_solve_tma(const BandDesc* __restrict__ bands,
                                                             const double* __restrict__ x,
                                                             double* __restrict__ y, const int* done,
                                                             const int* __restrict__ gidx,
                                                             const double* __restrict__ r) {
  PDL_ENTRY();
  if (done && *done) return;
  extern __shared__ __align__(16) double sm[];
  const BandDesc b = bands[blockIdx.x];
  const int npad = b.nb * TT;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, c0 = warp * 8;
  double* ringw = sm + (long long)warp * S * 512;  // this warp's ring (S x 512 doubles)
  double* v = sm + 8 * S * 512;
  double* red = v + npad;
  double* t = red + 8 * TT;
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(t + TT) + warp * S;  // this warp's S mbarriers
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < S; ++q) mbar_init(bars + q, 1);
  }
  mbar_fence_init();
  __syncthreads();
  unsigned cons = 0;  // tiles consumed so far (slot = cons % S, phase = (cons / S) & 1)
  const int dlen = TT - 8 * warp;
  const bool drow = lane >= 4 * warp;
  const int doff = diag_strip_off(warp) + (2 * lane - 8 * warp);
  TmaProducer prod{0, 0, 0};
#pragma unroll
  for (int q = 0; q < S; ++q) prod.issue(b, 0, ringw, bars, warp, lane, S);
  if (gidx) {
    for (int i = threadIdx.x; i < npad; i += NTHR) {
      const int g = __ldg(gidx + b.xoff + i);
      v[i] = g >= 0 ? __ldg(r + g) : 0.0;
    }
  } else {
    for (int i = threadIdx.x; i < npad; i += NTHR) v[i] = x[b.xoff + i];
  }
  __syncthreads();
  int cs = 0;
  // forward sweep
  for (int I = 0; I < b.nb; ++I) {
    const double* blk = b.data + b.step_off[I];
    const int code = b.kcnt[I], K = code & 0xffff, fz = code >> 16;
    double ra0 = 0.0, ra1 = 0.0;
    for (int k = 0; k < K; ++k) {
      mbar_wait(bars + cs, (cons / S) & 1);
      ++cons;
      if (!(k * 8 + warp < fz)) {
        const double* rs = ringw + (long long)cs * 512 + 2 * lane;
        const double* uj = v + (I - K + k) * TT + c0;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const double2 w = *reinterpret_cast<const double2*>(rs + kk * 64);
          ra0 += w.x * uj[kk];
          ra1 += w.y * uj[kk];
        }
      }
      cs = cs + 1 == S ? 0 : cs + 1;
      prod.issue(b, 0, ringw, bars, warp, lane, S);
    }
    red[warp * TT + 2 * lane] = ra0;
    red[warp * TT + 2 * lane + 1] = ra1;
    __syncthreads();
    if (threadIdx.x < TT) {
      double sacc = v[I * TT + threadIdx.x];
#pragma unroll
      for (int w = 0; w < 8; ++w) sacc -= red[w * TT + threadIdx.x];
      t[threadIdx.x] = sacc;
    }
    __syncthreads();
    {
      double d0 = 0.0, d1 = 0.0;
      if (drow) {
        const double* dp = blk + (long long)K * TT * TT + doff;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const double2 w = ldg_stream2(dp + kk * dlen);
          d0 += w.x * t[c0 + kk];
          d1 += w.y * t[c0 + kk];
        }
      }
      red[warp * TT + 2 * lane] = d0;
      red[warp * TT + 2 * lane + 1] = d1;
    }
    __syncthreads();
    if (threadIdx.x < TT) {
      double sacc = 0.0;
#pragma unroll
      for (int w = 0; w < 8; ++w) sacc += red[w * TT + threadIdx.x];
      v[I * TT + threadIdx.x] = sacc;
    }
    __syncthreads();
  }
  for (int q = 0; q < S; ++q) {  // the S (empty) items issued past the end of the sweep
    mbar_wait(bars + cs, (cons / S) & 1);
    ++cons;
    cs = cs + 1 == S ? 0 : cs + 1;
  }
  __syncwarp();
  if (b.udata) {
    const int ulen = 8 * warp + 8;
    const bool urow = lane <= 4 * warp + 3;
    const int uoff = udiag_strip_off(warp) + 2 * lane;
    TmaProducer up{b.nb - 1, 0, cs};
#pragma unroll
    for (int q = 0; q < S; ++q) up.issue(b, 2, ringw, bars, warp, lane, S);
    for (int I = b.nb - 1; I >= 0; --I) {
      const double* blk = b.udata + b.ustep_off[I];
      const int code = b.ucnt[I], R = code & 0xffff, tz = code >> 16;
      double ra0 = 0.0, ra1 = 0.0;
      for (int k = 0; k < R; ++k) {
        mbar_wait(bars + cs, (cons / S) & 1);
      ++cons;
        if (!(k * 8 + warp >= 8 * R - tz)) {
          const double* rs = ringw + (long long)cs * 512 + 2 * lane;
          const double* yj = v + (I + 1 + k) * TT + c0;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const double2 w = *reinterpret_cast<const double2*>(rs + kk * 64);
            ra0 += w.x * yj[kk];
            ra1 += w.y * yj[kk];
          }
        }
        cs = cs + 1 == S ? 0 : cs + 1;
        up.issue(b, 2, ringw, bars, warp, lane, S);
      }
      red[warp * TT + 2 * lane] = ra0;
      red[warp * TT + 2 * lane + 1] = ra1;
      __syncthreads();
      if (threadIdx.x < TT) {
        double sacc = v[I * TT + threadIdx.x];
#pragma unroll
        for (int w = 0; w < 8; ++w) sacc -= red[w * TT + threadIdx.x];
        t[threadIdx.x] = sacc;
      }
      __syncthreads();
      {
        double d0 = 0.0, d1 = 0.0;
        if (urow) {
          const double* dp = blk + (long long)R * TT * TT + uoff;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const double2 w = ldg_stream2(dp + kk * ulen);
            d0 += w.x * t[c0 + kk];
            d1 += w.y * t[c0 + kk];
          }
        }
        red[warp * TT + 2 * lane] = d0;
        red[warp * TT + 2 * lane + 1] = d1;
      }
      __syncthreads();
      if (threadIdx.x < TT) {
        double sacc = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) sacc += red[w * TT + threadIdx.x];
        v[I * TT + threadIdx.x] = sacc;
      }
      __syncthreads();
    }
    for (int i = threadIdx.x; i < npad; i += NTHR) y[b.xoff + i] = v[i];
    return;
  }
  // Cholesky backward: L^T y = u
  const int colsel = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
  TmaProducer bp{b.nb - 1, 0, cs};
#pragma unroll
  for (int q = 0; q < S; ++q) bp.issue(b, 1, ringw, bars, warp, lane, S);
  for (int J = b.nb - 1; J >= 0; --J) {
    const double* blk = b.data + b.step_off[J];
    const int code = b.kcnt[J], K = code & 0xffff, fz = code >> 16;
    {
      const double u0 = v[J * TT + 2 * lane], u1 = v[J * TT + 2 * lane + 1];
      double cp[8];
      if (drow) {
        const double* dp = blk + (long long)K * TT * TT + doff;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const double2 w = ldg_stream2(dp + kk * dlen);
          cp[kk] = w.x * u0 + w.y * u1;
        }
      } else {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) cp[kk] = 0.0;
      }
      const double yv = warp_reduce8(cp, lane);
      __syncthreads();  // every warp has read v_J
      if ((lane & 3) == 0) v[J * TT + c0 + colsel] = yv;
      __syncthreads();
    }
    const double y0 = v[J * TT + 2 * lane], y1 = v[J * TT + 2 * lane + 1];
    for (int k = 0; k < K; ++k) {
      mbar_wait(bars + cs, (cons / S) & 1);
      ++cons;
      if (!(k * 8 + warp < fz)) {
        const double* rs = ringw + (long long)cs * 512 + 2 * lane;
        double cp[8];
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const double2 w = *reinterpret_cast<const double2*>(rs + kk * 64);
          cp[kk] = w.x * y0 + w.y * y1;
        }
        const double val = warp_reduce8(cp, lane);
        if ((lane & 3) == 0) v[(J - K + k) * TT + c0 + colsel] -= val;
      }
      cs = cs + 1 == S ? 0 : cs + 1;
      bp.issue(b, 1, ringw, bars, warp, lane, S);
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < npad; i += NTHR) y[b.xoff + i] = v[i];
}

// pack band steps of one subdomain batch: L (row-major ld x ld, factor order, identity
// padding) and the inverted diagonal tiles dinv (nbmax x 64 x 64 row-major per subdomain)
__global__ void k_pack_band(const BandDesc* __restrict__ bands, int first_band, const double* __restrict__ L,
                            long long ld, const double* __restrict__ dinv, int nbmax) {
  PDL_ENTRY();
  const int bi = blockIdx.y;
  const BandDesc bd = bands[first_band + bi];
  const double* Lb = L + (long long)bi * ld * ld;
  const double* Db = dinv + (long long)bi * nbmax * TT * TT;
  for (int I = blockIdx.x; I < bd.nb; I += gridDim.x) {
    const int K = bd.kcnt[I] & 0xffff;
    double* dst = const_cast<double*>(bd.data) + bd.step_off[I];
    for (int k = 0; k < K; ++k) {
      const int J = I - K + k;
      for (int e = threadIdx.x; e < TT * TT; e += NTHR) {
        const int c = e / TT, r = e % TT;
        const long long gi = (long long)I * TT + r, gj = (long long)J * TT + c;
        dst[(long long)k * TT * TT + e] = (gi < ld && gj < ld) ? Lb[gi * ld + gj] : 0.0;
      }
    }
    double* dd = dst + (long long)K * TT * TT;
    for (int w = 0; w < 8; ++w) {
      const int len = TT - 8 * w, off = diag_strip_off(w);
      for (int e = threadIdx.x; e < 8 * len; e += NTHR) {
        const int kk = e / len, r = 8 * w + e % len;
        dd[off + e] = Db[(long long)I * TT * TT + r * TT + (8 * w + kk)];
      }
    }
  }
}

// pack the U steps of one LU batch: U (row-major ld x ld, upper part of the packed LU) and
// the inverted upper diagonal tiles udinv (nbmax x 64 x 64 row-major per subdomain)
__global__ void k_pack_band_u(const BandDesc* __restrict__ bands, int first_band, const double* __restrict__ LU,
                              long long ld, const double* __restrict__ udinv, int nbmax) {
  PDL_ENTRY();
  const int bi = blockIdx.y;
  const BandDesc bd = bands[first_band + bi];
  const double* Ub = LU + (long long)bi * ld * ld;
  const double* Db = udinv + (long long)bi * nbmax * TT * TT;
  for (int I = blockIdx.x; I < bd.nb; I += gridDim.x) {
    const int R = bd.ucnt[I] & 0xffff;
    double* dst = const_cast<double*>(bd.udata) + bd.ustep_off[I];
    for (int k = 0; k < R; ++k) {
      const int J = I + 1 + k;
      for (int e = threadIdx.x; e < TT * TT; e += NTHR) {
        const int c = e / TT, r = e % TT;
        const long long gi = (long long)I * TT + r, gj = (long long)J * TT + c;
        dst[(long long)k * TT * TT + e] = (gi < ld && gj < ld) ? Ub[gi * ld + gj] : 0.0;
      }
    }
    double* dd = dst + (long long)R * TT * TT;
    for (int w = 0; w < 8; ++w) {
      const int len = 8 * w + 8, off = udiag_strip_off(w);
      for (int e = threadIdx.x; e < 8 * len; e += NTHR) {
        const int kk = e / len, r = e % len;
        dd[off + e] = Db[(long long)I * TT * TT + r * TT + (8 * w + kk)];
      }
    }
  }
}

// ---------------------------------------------------------------------------------------
// K10  Banded triangular solves with many right-hand sides (setup: the harmonic extension,
//      src/subdomain.py:108-120, as B[:, ring] = A_ii^{-1} E_ring on the band factor):
//      X = (L L^T)^{-1} X for a batch of banded Cholesky factors (factor order, lower, 64-row
//      blocks; kc[b][I] panel tiles left of the diagonal in block row I; dinv = inverted diagonal
//      tiles, row-major).  Grid (RHS chunks of 64 columns, subdomains): every CTA sweeps its own
//      64 columns forward (X_I = D_I^{-1} (X_I - sum_J L_IJ X_J)) and backward
//      (X_I = D_I^{-T} X_I; X_J -= L_IJ^T X_I), every 64 x 64 x 64 tile product on the FP64
//      tensor cores (mma.sync.m8n8k4.f64, tile_xyt: warp w owns output rows 8w..8w+7).
//      Dynamic smem: 2 padded 64 x 65 tiles.
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ void tile_xyt_acc(const double* X, const double* Y, double (&acc)[8][2]) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, gr = lane >> 2, gc = lane & 3;
#pragma unroll 4
  for (int k0 = 0; k0 < 64; k0 += 4) {
    const double a = X[(8 * w + gr) * CP + k0 + gc];
#pragma unroll
    for (int bj = 0; bj < 8; ++bj) dmma_8x8x4(acc[bj][0], acc[bj][1], a, Y[(8 * bj + gr) * CP + k0 + gc]);
  }
}

// T[n][k] = G[k][n] for the valid columns n < nv (64 x 64 block of a row-major matrix, ld)
__device__ __forceinline__ void load_tile_t(double* T, const double* G, long long ld, int nv) {
  for (int e = threadIdx.x; e < 64 * 64; e += blockDim.x) {
    const int k = e >> 6, n = e & 63;
    T[n * CP + k] = n < nv ? G[(long long)k * ld + n] : 0.0;
  }
}

__global__ void __launch_bounds__(256) k_band_trsm_multi(const double* __restrict__ L, long long ld,
                                                         const double* __restrict__ dinv, const int* __restrict__ kc,
                                                         int nb, double* __restrict__ Xall, long long nrhs) {
  PDL_ENTRY();
  extern __shared__ __align__(16) double ts[];
  double* Xs = ts;             // X operand (rows m, cols k)
  double* Ys = ts + 64 * CP;   // Y operand (rows n, cols k)
  const int b = blockIdx.y;
  const long long c0 = 64LL * blockIdx.x;
  const int nv = (int)min(64LL, nrhs - c0);
  const double* Lb = L + (long long)b * ld * ld;
  const double* Db = dinv + (long long)b * nb * 64 * 64;
  const int* kb = kc + (long long)b * nb;
  double* X = Xall + (long long)b * ld * nrhs + c0;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, gr = lane >> 2, gc = lane & 3;
  const int row = 8 * w + gr;
  double acc[8][2];
  // forward: X_I = D_I^{-1} (X_I - sum_J L_IJ X_J)
  for (int I = 0; I < nb; ++I) {
    const long long r0 = 64LL * I;
    const int K = kb[I];
#pragma unroll
    for (int bj = 0; bj < 8; ++bj) acc[bj][0] = acc[bj][1] = 0.0;
    for (int t = 0; t < K; ++t) {
      const long long j0 = r0 - 64LL * (K - t);
      load_tile(Xs, Lb + r0 * ld + j0, ld);
      load_tile_t(Ys, X + j0 * nrhs, nrhs, nv);
      __syncthreads();
      tile_xyt_acc(Xs, Ys, acc);
      __syncthreads();
    }
    // Ys[n][m] = X_I[m][n] - acc[m][n]
#pragma unroll
    for (int bj = 0; bj < 8; ++bj)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int n = 8 * bj + 2 * gc + e;
        Ys[n * CP + row] = n < nv ? X[(r0 + row) * nrhs + n] - acc[bj][e] : 0.0;
      }
    load_tile(Xs, Db + (long long)I * 64 * 64, 64);
    __syncthreads();
#pragma unroll
    for (int bj = 0; bj < 8; ++bj) acc[bj][0] = acc[bj][1] = 0.0;
    tile_xyt_acc(Xs, Ys, acc);
#pragma unroll
    for (int bj = 0; bj < 8; ++bj)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int n = 8 * bj + 2 * gc + e;
        if (n < nv) X[(r0 + row) * nrhs + n] = acc[bj][e];
      }
    __syncthreads();
  }
  // backward: X_I = D_I^{-T} X_I; X_J -= L_IJ^T X_I
  for (int I = nb - 1; I >= 0; --I) {
    const long long r0 = 64LL * I;
    const int K = kb[I];
    for (int e = threadIdx.x; e < 64 * 64; e += blockDim.x) {  // Xs[m][k] = D_I[k][m]
      const int k = e >> 6, m = e & 63;
      Xs[m * CP + k] = Db[(long long)I * 64 * 64 + e];
    }
    load_tile_t(Ys, X + r0 * nrhs, nrhs, nv);
    __syncthreads();
#pragma unroll
    for (int bj = 0; bj < 8; ++bj) acc[bj][0] = acc[bj][1] = 0.0;
    tile_xyt_acc(Xs, Ys, acc);
    __syncthreads();
#pragma unroll
    for (int bj = 0; bj < 8; ++bj)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int n = 8 * bj + 2 * gc + e;
        Ys[n * CP + row] = n < nv ? acc[bj][e] : 0.0;
        if (n < nv) X[(r0 + row) * nrhs + n] = acc[bj][e];
      }
    for (int t = 0; t < K; ++t) {
      const long long j0 = r0 - 64LL * (K - t);
      __syncthreads();
      for (int e = threadIdx.x; e < 64 * 64; e += blockDim.x) {  // Xs[m][k] = L[r0 + k][j0 + m]
        const int k = e >> 6, m = e & 63;
        Xs[m * CP + k] = Lb[(r0 + k) * ld + j0 + m];
      }
      __syncthreads();
#pragma unroll
      for (int bj = 0; bj < 8; ++bj) acc[bj][0] = acc[bj][1] = 0.0;
      tile_xyt_acc(Xs, Ys, acc);
#pragma unroll
      for (int bj = 0; bj < 8; ++bj)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int n = 8 * bj + 2 * gc + e;
          if (n < nv) X[(j0 + row) * nrhs + n] -= acc[bj][e];
        }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------------------
// K12a  Rank filter pivots (setup; src/coarse.py:119-155 runs LAPACK geqp3 per subdomain block):
//       column-pivoted Householder QR of each subdomain's coarse block W (n x k, column-major,
//       overwritten), one CTA per subdomain.  Step j recomputes the remaining columns' norms over
//       rows j.. (no downdating), takes the first largest as pivot, swaps it to j, and applies the
//       Householder reflector that zeroes W[j+1:, j] to the columns right of it.  Outputs |R_jj|
//       (rdiag, k per block) and the pivot order (perm: original column at position j).
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ double block_sum256(double v, double* red) {
  red[threadIdx.x] = v;
  __syncthreads();
  for (int h = 128; h > 0; h >>= 1) {
    if (threadIdx.x < h) red[threadIdx.x] += red[threadIdx.x + h];
    __syncthreads();
  }
  const double r = red[0];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(256) k_pivoted_qr(double* __restrict__ Wall, const long long* __restrict__ woff,
                                                    const int* __restrict__ nrows, const int* __restrict__ ncols,
                                                    const long long* __restrict__ roff, double* __restrict__ rdiag,
                                                    int* __restrict__ perm) {
  PDL_ENTRY();
  __shared__ double red[256];
  __shared__ double nrm[64];
  __shared__ int pv[64];
  const int s = blockIdx.x;
  const int n = nrows[s], k = ncols[s];
  double* W = Wall + woff[s];
  double* rd = rdiag + roff[s];
  int* pm = perm + roff[s];
  if (threadIdx.x < k) pv[threadIdx.x] = threadIdx.x;
  __syncthreads();
  for (int j = 0; j < k && j < n; ++j) {
    for (int c = j; c < k; ++c) {
      double a = 0.0;
      for (int i = j + threadIdx.x; i < n; i += 256) {
        const double x = W[(long long)c * n + i];
        a += x * x;
      }
      const double t = block_sum256(a, red);
      if (threadIdx.x == 0) nrm[c] = t;
    }
    __syncthreads();
    int p = j;
    for (int c = j + 1; c < k; ++c)
      if (nrm[c] > nrm[p]) p = c;
    if (p != j) {  // swap columns j and p
      for (int i = threadIdx.x; i < n; i += 256) {
        const double t = W[(long long)j * n + i];
        W[(long long)j * n + i] = W[(long long)p * n + i];
        W[(long long)p * n + i] = t;
      }
      if (threadIdx.x == 0) {
        const int t = pv[j];
        pv[j] = pv[p];
        pv[p] = t;
      }
    }
    __syncthreads();
    // Householder: v = x - alpha e_1, alpha = -sign(x_0) ||x||; R_jj = alpha
    const double xn = sqrt(nrm[p]);
    const double x0 = W[(long long)j * n + j];
    const double alpha = x0 >= 0.0 ? -xn : xn;
    if (threadIdx.x == 0) rd[j] = fabs(alpha);
    const double v0 = x0 - alpha;
    const double vtv = xn * xn - x0 * x0 + v0 * v0;
    __syncthreads();
    if (vtv > 0.0) {
      for (int c = j + 1; c < k; ++c) {
        double a = threadIdx.x == 0 ? v0 * W[(long long)c * n + j] : 0.0;
        for (int i = j + 1 + threadIdx.x; i < n; i += 256) a += W[(long long)j * n + i] * W[(long long)c * n + i];
        const double f = 2.0 * block_sum256(a, red) / vtv;
        if (threadIdx.x == 0) W[(long long)c * n + j] -= f * v0;
        for (int i = j + 1 + threadIdx.x; i < n; i += 256) W[(long long)c * n + i] -= f * W[(long long)j * n + i];
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) W[(long long)j * n + j] = alpha;
    __syncthreads();
  }
  for (int j = threadIdx.x; j < k; j += 256) {
    pm[j] = pv[j];
    if (j >= n) rd[j] = 0.0;
  }
}

// ---------------------------------------------------------------------------------------
// K9b  Banded LU with partial pivoting of a batch of general blocks (setup; the getrf of
//      src/subdomain.py:83-89 on the block in its factor order), one CTA per block, in place in
//      LAPACK's format (unit-lower L and U packed, piv 1-based, rows interchanged across the whole
//      width).  Per 64-column panel J: an unblocked panel factorisation over rows [j0, lreach[J])
//      (pivot = first largest |a|, as idamax), then U_J = L_JJ^{-1} A[J, right] and the trailing
//      band update A[below, right] -= L_below U_J with the tile products on the FP64 tensor cores.
//      lreach[J] / ureach[J] bound the rows / columns the band can touch (partial pivoting keeps
//      L within the lower bandwidth and U within lower + upper).  info = first zero pivot (1-based).
//      Dynamic smem: 3 padded 64 x 65 tiles.
// ---------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256, 1) k_band_lu(double* __restrict__ AP, long long ld,
                                                    const int* __restrict__ lreach, const int* __restrict__ ureach,
                                                    int nbk, int* __restrict__ pivots, int* __restrict__ info) {
  PDL_ENTRY();
  extern __shared__ __align__(16) double ls[];
  double* Ls = ls;                 // L_JJ^{-1} (unit lower)
  double* Ta = Ls + 64 * CP;
  double* Tb = Ta + 64 * CP;
  __shared__ double rv[8];
  __shared__ int ri[8];
  __shared__ int prow, bad;
  double* A = AP + (long long)blockIdx.x * ld * ld;
  int* piv = pivots + (long long)blockIdx.x * ld;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, gr = lane >> 2, gc = lane & 3;
  if (tid == 0) bad = 0;
  for (int J = 0; J < nbk; ++J) {
    const long long j0 = 64LL * J;
    const long long r1 = lreach[J], c1 = ureach[J];
    // ---- unblocked panel factorisation with partial pivoting
    for (int k = 0; k < 64; ++k) {
      const long long jc = j0 + k;
      double best = -1.0;
      int bi = (int)jc;
      for (long long i = jc + tid; i < r1; i += 256) {
        const double v = fabs(A[i * ld + jc]);
        if (v > best) { best = v; bi = (int)i; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_down_sync(FULL, best, o);
        const int oi = __shfl_down_sync(FULL, bi, o);
        if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
      }
      if (lane == 0) { rv[w] = best; ri[w] = bi; }
      __syncthreads();
      if (tid == 0) {
        double b = rv[0];
        int q = ri[0];
        for (int ww = 1; ww < 8; ++ww)
          if (rv[ww] > b || (rv[ww] == b && ri[ww] < q)) { b = rv[ww]; q = ri[ww]; }
        prow = q;
        piv[jc] = q + 1;
        if (b == 0.0 && bad == 0) bad = (int)jc + 1;
      }
      __syncthreads();
      const long long p = prow;
      if (p != jc)
        for (long long c = tid; c < c1; c += 256) {
          const double t = A[jc * ld + c];
          A[jc * ld + c] = A[p * ld + c];
          A[p * ld + c] = t;
        }
      __syncthreads();
      const double d = A[jc * ld + jc];
      if (d != 0.0)
        for (long long i = jc + 1 + tid; i < r1; i += 256) A[i * ld + jc] /= d;
      __syncthreads();
      const int nc = 63 - k;
      const long long nr = r1 - jc - 1;
      for (long long e = tid; e < nr * nc; e += 256) {
        const long long i = jc + 1 + e / nc, c = jc + 1 + e % nc;
        A[i * ld + c] -= A[i * ld + jc] * A[jc * ld + c];
      }
      __syncthreads();
    }
    if (c1 <= j0 + 64) continue;
    // ---- L_JJ^{-1} (unit lower), one column per thread
    if (tid < 64) {
      const int j = tid;
      for (int i = 0; i < 64; ++i) Ls[i * CP + j] = i == j ? 1.0 : 0.0;
      for (int i = j + 1; i < 64; ++i) {
        double acc = 0.0;
        for (int q = j; q < i; ++q) acc += A[(j0 + i) * ld + j0 + q] * Ls[q * CP + j];
        Ls[i * CP + j] = -acc;
      }
    }
    __syncthreads();
    // ---- U row block: U_J,t = L_JJ^{-1} A[J, t] for the column tiles right of the diagonal
    const int nt = (int)((c1 - j0 - 64 + 63) / 64);
    for (int t = 0; t < nt; ++t) {
      double* G = A + j0 * ld + j0 + 64 + 64LL * t;
      for (int e = tid; e < 64 * 64; e += 256) {   // Ta[n][k] = G[k][n]
        const int kk = e >> 6, n = e & 63;
        Ta[n * CP + kk] = G[(long long)kk * ld + n];
      }
      __syncthreads();
      double acc[8][2];
      tile_xyt(Ls, Ta, acc);
      __syncthreads();
#pragma unroll
      for (int bj = 0; bj < 8; ++bj) {
        G[(long long)(8 * w + gr) * ld + 8 * bj + 2 * gc] = acc[bj][0];
        G[(long long)(8 * w + gr) * ld + 8 * bj + 2 * gc + 1] = acc[bj][1];
      }
      __syncthreads();
    }
    // ---- trailing band update: A[ti, tj] -= L[ti, J] U[J, tj]
    const int mt = (int)((r1 - j0 - 64 + 63) / 64);
    for (int ti = 0; ti < mt; ++ti) {
      load_tile(Ta, A + (j0 + 64 + 64LL * ti) * ld + j0, ld);   // L tile (rows m, cols k)
      for (int tj = 0; tj < nt; ++tj) {
        const double* U = A + j0 * ld + j0 + 64 + 64LL * tj;
        for (int e = tid; e < 64 * 64; e += 256) {               // Tb[n][k] = U[k][n]
          const int kk = e >> 6, n = e & 63;
          Tb[n * CP + kk] = U[(long long)kk * ld + n];
        }
        __syncthreads();
        double acc[8][2];
        tile_xyt(Ta, Tb, acc);
        double* G = A + (j0 + 64 + 64LL * ti) * ld + j0 + 64 + 64LL * tj;
#pragma unroll
        for (int bj = 0; bj < 8; ++bj) {
          G[(long long)(8 * w + gr) * ld + 8 * bj + 2 * gc] -= acc[bj][0];
          G[(long long)(8 * w + gr) * ld + 8 * bj + 2 * gc + 1] -= acc[bj][1];
        }
        __syncthreads();
      }
    }
    __syncthreads();
  }
  if (tid == 0) info[blockIdx.x] = bad;
}

// ---------------------------------------------------------------------------------------
// K12b  Galerkin assembly A0 = Z^T (A Z) (setup; src/coarse.py:158-168 forms it as a sparse
//       triple product).  Column block s of A Z is W_s = A_ii[:, :n_int] Z_s on the local rows of
//       subdomain s; its rows owned by subdomain j contract with Z_j.  One CTA per (s, j) pair of
//       the plan (rows[o0:o1] = interior positions in j, grp[o0:o1] = local rows of s), 32-row
//       chunks staged in shared memory, thread (a, b) accumulates A0[cstart_j + a, cstart_s + b]
//       in a fixed order (deterministic); every block of A0 has exactly one writer.
// ---------------------------------------------------------------------------------------
struct GalPlan { int s, j; long long o0, o1; };

__global__ void __launch_bounds__(256) k_galerkin_blocks(const GalPlan* __restrict__ plan,
                                                         const long long* __restrict__ zptr,
                                                         const long long* __restrict__ wptr,
                                                         const int* __restrict__ kcnt,
                                                         const long long* __restrict__ cstart,
                                                         const long long* __restrict__ rows,
                                                         const long long* __restrict__ grp,
                                                         double* __restrict__ A0, long long nC) {
  PDL_ENTRY();
  __shared__ double zs[32][64];
  __shared__ double ws[32][64];
  const GalPlan pl = plan[blockIdx.x];
  const int kj = kcnt[pl.j], ks = kcnt[pl.s];
  const double* Z = reinterpret_cast<const double*>(zptr[pl.j]);
  const double* W = reinterpret_cast<const double*>(wptr[pl.s]);
  const int tid = threadIdx.x;
  double acc[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) acc[q] = 0.0;
  for (long long r0 = pl.o0; r0 < pl.o1; r0 += 32) {
    const int nr = (int)min(32LL, pl.o1 - r0);
    for (int e = tid; e < 32 * 64; e += 256) {
      const int r = e >> 6, c = e & 63;
      zs[r][c] = (r < nr && c < kj) ? Z[rows[r0 + r] * kj + c] : 0.0;
      ws[r][c] = (r < nr && c < ks) ? W[grp[r0 + r] * ks + c] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int o = tid + 256 * q;
      const int a = o >> 6, b = o & 63;
      if (a < kj && b < ks) {
        double t = acc[q];
        for (int r = 0; r < nr; ++r) t += zs[r][a] * ws[r][b];
        acc[q] = t;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const int o = tid + 256 * q;
    const int a = o >> 6, b = o & 63;
    if (a < kj && b < ks) A0[(cstart[pl.j] + a) * nC + cstart[pl.s] + b] = acc[q];
  }
}

}  // namespace tls
