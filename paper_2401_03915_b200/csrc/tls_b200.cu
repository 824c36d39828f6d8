// tls_b200.cu — host side of libtls_b200.so: handle, apply schedule, CUDA-graph Krylov drivers.
//
// C ABI declared in include/tls_b200.h.  All per-iteration work is enqueued on the caller's
// stream; the PCG iteration (25 iterations = one residual-replacement period,
// src/krylov.py:88-89) and the GMRES cycle are captured once into CUDA graphs and replayed,
// with a device-side `done` flag turning the remaining kernels into no-ops after convergence,
// so one host sync happens per 25 PCG iterations / per GMRES cycle instead of per kernel.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <cub/device/device_segmented_sort.cuh>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "tls_b200.h"
#include "tls_comm.h"
#include "tls_kernels.cuh"
#include "tls_graph.cuh"

using namespace tls;

namespace {

constexpr int PCG_GRAPH_ITERS = 25;  // replacement period of src/krylov.py:88
constexpr int MAX_GRID = 148 * 8;    // 148 SMs x 8 resident 256-thread CTAs
constexpr int GM_FUSED_MAXCOLS = 96; // fused CGS2 step while (nc + 1) x 256 doubles fit in smem
// shared memory of the per-warp rings of k_band_solve_ring<S> (8 warps x S tiles x 4 KB)
constexpr size_t ring_bytes(int S) { return sizeof(double) * 8 * (size_t)S * 512; }
constexpr size_t TMA_BAR_BYTES = 8 * 8 * 8;  // k_band_solve_tma: up to 8 mbarriers per warp
// shared memory of k_band_solve for subdomains of up to nb 64-row blocks (local vector + scratch)
constexpr size_t band_smem_bytes(int nb) { return sizeof(double) * ((size_t)nb * 64 + 8 * 64 + 64); }
// largest subdomain (rows) whose local vector fits `optin` bytes of shared memory
static int band_max_rows(size_t optin) { return (int)((optin / sizeof(double) - 8 * 64 - 64) / 64) * 64; }

// NVTX range over a C entry point (visible to Nsight tools; a no-op without an injected tool)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
#define TLS_RANGE(name) NvtxRange nvtx_range_(name)

template <class T>
void dfree(T*& p) {
  if (p) cudaFree((void*)p);
  p = nullptr;
}

}  // namespace

struct tls_ctx {
  int device = 0;
  std::string err;
  int64_t dev_bytes = 0;
  cudaStream_t cap = nullptr;
  cudaStream_t aux = nullptr;                          // side branch (coarse chain overlap)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // ---- matrix (CSR, int32 indices)
  int n = 0;
  int64_t nnz = 0;
  int sym = 0;
  int lpr = 8;
  int *rowptr = nullptr, *col = nullptr;
  double* val = nullptr;
  // ---- subdomains
  int nsub = 0, max_n = 0;
  std::vector<int64_t> h_off;
  std::vector<int> h_idx, h_n, h_nint;
  long long* d_sub_idxoff = nullptr;
  int *d_sub_n = nullptr, *d_idx = nullptr, *d_nint = nullptr;
  // ---- local operators
  std::vector<BlkDesc> h_blk;  // nsub local blocks (+1 coarse after finalize)
  BlkDesc* d_blk = nullptr;
  double* tiles = nullptr;
  int64_t tile_doubles = 0;
  std::vector<int> stored;  // which subdomains have their inverse stored
  // ---- coarse
  int ncoarse = 0;
  int kmax = 1;
  std::vector<int> h_k, h_cstart;
  std::vector<long long> h_zoff;
  double *d_Z = nullptr, *ctiles = nullptr;
  // one step of iterative refinement of the coarse solve, y = X c; y += X (c - A0 y) (X = the
  // stored A0^{-1}): blocks nsub+1 (A0 tiles) and nsub+2 (X again) behind the coarse block
  bool cref = false;
  double* a0tiles = nullptr;
  long long cpad = 0;                 // padded coarse length (nt * TT)
  int nu_ref1 = 0, no_ref1 = 0, nu_ref2 = 0, no_ref2 = 0;
  // block-tridiagonal coarse solve (tls_coarse_chain): A0 is banded in subdomain order, so the
  // coarse solve runs as a block forward / backward substitution with the inverted Schur blocks
  // S_i^{-1} (tile blocks nsub+3 .. nsub+3+nb-1) and the sparse off-diagonal blocks of A0 (two
  // CSR matrices: strictly block-lower part and its transpose) instead of a dense n_C^2 inverse
  int chain_nb = 0, chain_bs = 0;
  double* chain_tiles = nullptr;
  int *d_lo_ptr = nullptr, *d_lo_idx = nullptr, *d_up_ptr = nullptr, *d_up_idx = nullptr;
  double *d_lo_val = nullptr, *d_up_val = nullptr;
  long long chain_nnz = 0;
  std::vector<int> chain_u0, chain_nu, chain_o0, chain_no;
  // sharded coarse restriction: every rank's columns [ccol[q], ccol[q+1]) travel by one
  // all-gather of cmax doubles per rank (instead of an all-reduce of the whole n_C vector)
  std::vector<long long> ccol;
  long long cmax = 0;
  long long* d_ccol = nullptr;
  double *cg_send = nullptr, *cg_recv = nullptr;
  long long* d_zoff = nullptr;
  int *d_kcnt = nullptr, *d_cstart = nullptr;
  // ---- schedule
  bool finalized = false;
  int one_level = 0, combine = 0;
  long long X = 0, Xloc = 0, coarse_xoff = 0;
  Unit* d_units = nullptr;  // [local | coarse]
  int nu_local = 0, nu_coarse = 0;
  OutTile* d_outs = nullptr;  // [local | coarse]
  int no_local = 0, no_coarse = 0;
  int* d_red = nullptr;
  int* d_gidx = nullptr;
  int *d_pull_ptr = nullptr, *d_pull_pos = nullptr;
  long long* d_zrow = nullptr;
  int *d_zk = nullptr, *d_zc = nullptr, *d_zst = nullptr;
  double *xloc = nullptr, *yloc = nullptr, *slots = nullptr;
  int64_t nslots = 0;
  double algo_local = 0.0, algo_coarse = 0.0;
  // ---- work vectors
  double *t1 = nullptr, *t2 = nullptr, *t3 = nullptr, *t4 = nullptr, *t5 = nullptr, *t6 = nullptr,
         *t7 = nullptr, *vb = nullptr, *vx = nullptr, *vr = nullptr, *vp = nullptr, *vap = nullptr,
         *vz = nullptr, *hist = nullptr, *ab = nullptr, *h_x = nullptr,
         *cz = nullptr;  // coarse prolongation Z yc of the additive band schedule
  int hist_cap = 0;
  double* part = nullptr;
  int64_t part_cap = 0;
  int G = 1, Gs = 1;
  PcgState* pcg = nullptr;
  GmState* gm = nullptr;
  int* h_flag = nullptr;  // pinned
  // ---- gmres workspace
  double *V = nullptr, *H = nullptr, *cs = nullptr, *sn = nullptr, *gv = nullptr, *yv = nullptr,
         *h1 = nullptr, *h2 = nullptr;
  int gm_cols = 0;
  bool gm_fused = true;               // CGS2 middle step as one kernel (TLS_GM_FUSED=0: two)
  bool gm_givens_fused = true;        // Givens + v_{j+1} = w / hn in one launch (TLS_GM_GIVENS_FUSED=0: two)
  // ---- graphs
  cudaGraphExec_t pcg_exec[2] = {nullptr, nullptr};
  int pcg_exec_launches[2] = {0, 0};
  cudaGraphExec_t gm_exec[2] = {nullptr, nullptr};
  int gm_exec_cols[2] = {0, 0};
  int gm_exec_launches[2] = {0, 0};
  int launches = 0;  // kernels enqueued since the counter was reset
  int pdl = 1;       // programmatic dependent launch on every kernel (TLS_PDL=0: off)
  // ---- in-graph timing of the local-solve kernel (bench roofline over real solves)
  bool ktime = false, capturing = false;
  std::vector<cudaEvent_t> kt_a, kt_b;  // one pair per band-solve node of the captured graph
  int kt_n = 0;                         // pairs recorded by the current capture
  int kt_n_graph[2][2] = {{0, 0}, {0, 0}};  // [pcg|gmres][prec]: pairs in that graph
  double kt_sum_ms = 0.0;
  long long kt_count = 0;
  // ---- kernel trace (tls_set_kernel_trace): an event pair around EVERY launch of the host-driven
  // loops (warm caches, the kernels' real inputs, no graph / PDL overlap): per-kernel durations
  mutable bool ktrace = false;
  mutable std::vector<std::pair<const void*, std::pair<cudaEvent_t, cudaEvent_t>>> kt_trace;
  // ---- banded Cholesky local operators (local_kind == 1)
  int local_kind = 0;                 // 0: packed inverse tiles, 1: band factors
  size_t restrict_smem = 0;
  int restrict_cw = 32;               // coarse columns (warps) per k_restrict CTA (measured:
                                      // 8 per CTA loses 7% on configuration 3, tools/ab_env.sh)
  std::vector<BandDesc> h_band;
  BandDesc* d_band = nullptr;
  std::vector<void*> band_allocs;
  std::vector<int> h_perm;            // per owned subdomain: perm[p] = local index at output position p
  std::vector<int> h_perm_in;         // LU: local index gathered into input position p (row pivots)
  double band_bytes = 0.0;            // stored factor bytes (read twice per apply)
  size_t band_smem = 0;
  int band_pf = 2;                    // L2 prefetch distance of k_band_solve (items)
  int band_unr = 1;                   // tiles per load round (k_band_solve<UNR>)
  int band_ring = 0;                  // k_band_solve_ring (per-warp cp.async rings)
  int band_tma = 0;                   // k_band_solve_tma<S> (rings fed by bulk TMA copies + mbarriers), S = 4 or 5
  // ---- sharding: this handle owns global subdomains [own_lo, own_hi) and the
  // rows [r0, r1) of the internal numbering (rows renumbered rank by rank: nofo[g] = internal id
  // of caller row g; identity and [0, n) on one GPU)
  int own_lo = 0, own_hi = -1, nsub_global = 0;
  Comm* comm = nullptr;
  int r0 = 0, r1 = -1;
  std::vector<int> h_nofo;            // empty: identity numbering
  std::vector<int> row_starts;        // per rank [row_starts[q], row_starts[q+1])
  int* d_nofo = nullptr;
  XPlan halo;                         // ghost rows (SpMV columns + overlap rows) from their owners
  XPlan rev;                          // ASM overlap contributions to rows owned by other ranks
  std::vector<int> rc_peer, rc_cnt, rc_sub, rc_row;  // remote contributions received (in order)
  long long Xrecv = 0;                // tail of yloc holding the received contributions
  double *pin = nullptr, *pout = nullptr;  // caller-numbering staging vectors
  // ---- decomposition on the device (tls_graph_build / tls_overlap_build)
  long long* g_ptr = nullptr;
  int* g_adj = nullptr;
  long long g_m = -1;
  std::vector<long long> ov_off, ov_ls, ov_idx, ov_col;
  int ov_nsub = 0, ov_delta = 0, ov_kc = 0;
};

template <typename... KArgs, typename... Args>
static void launch_k(const tls_ctx* ctx, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                     cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  const bool trace = ctx && ctx->ktrace && !ctx->capturing;
  if (ctx && ctx->pdl && !trace) {
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
  }
  if (trace) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, s);
    cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
    cudaEventRecord(b, s);
    ctx->kt_trace.push_back({(const void*)kernel, {a, b}});
    return;
  }
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

struct tls_group {
  GroupShared shared;
  explicit tls_group(int n) : shared(n) {}
};

#define CK(call)                                                                             \
  do {                                                                                       \
    cudaError_t e_ = (call);                                                                 \
    if (e_ != cudaSuccess) {                                                                 \
      ctx->err = std::string(#call) + ": " + cudaGetErrorString(e_);                         \
      return e_ == cudaErrorMemoryAllocation ? TLS_ERR_OOM : TLS_ERR_CUDA;                   \
    }                                                                                        \
  } while (0)

#define CKL()                                                                                \
  do {                                                                                       \
    cudaError_t e_ = cudaGetLastError();                                                     \
    if (e_ != cudaSuccess) {                                                                 \
      ctx->err = std::string("kernel launch: ") + cudaGetErrorString(e_);                    \
      return TLS_ERR_CUDA;                                                                   \
    }                                                                                        \
    ctx->launches++;                                                                         \
  } while (0)

#define TRY(...)               \
  do {                         \
    int rc_ = (__VA_ARGS__);   \
    if (rc_ != TLS_OK) return rc_; \
  } while (0)

static int fail(tls_ctx* ctx, int code, const std::string& msg) {
  ctx->err = msg;
  return code;
}

template <class T>
static int dalloc(tls_ctx* ctx, T*& p, int64_t count) {
  dfree(p);
  if (count <= 0) count = 1;
  cudaError_t e = cudaMalloc((void**)&p, sizeof(T) * (size_t)count);
  if (e != cudaSuccess) {
    p = nullptr;
    ctx->err = "cudaMalloc(" + std::to_string(sizeof(T) * (size_t)count) + " B): " + cudaGetErrorString(e);
    return TLS_ERR_OOM;
  }
  ctx->dev_bytes += (int64_t)sizeof(T) * count;
  return TLS_OK;
}

template <class T>
static int upload(tls_ctx* ctx, T*& d, const T* h, int64_t count) {
  TRY(dalloc(ctx, d, count));
  if (count > 0) CK(cudaMemcpy(d, h, sizeof(T) * (size_t)count, cudaMemcpyHostToDevice));
  return TLS_OK;
}

// Host worker threads for the large host-side passes (CSR validation, staging copies)
static int host_threads() {
  const unsigned hc = std::thread::hardware_concurrency();
  return (int)std::max(1u, std::min(8u, hc ? hc : 1u));
}

template <class F>
static void parallel_chunks(int64_t count, int nthreads, F f) {  // f(thread, begin, end)
  if (nthreads <= 1 || count < (1 << 20)) {
    f(0, (int64_t)0, count);
    return;
  }
  std::vector<std::thread> th;
  const int64_t per = (count + nthreads - 1) / nthreads;
  for (int t = 0; t < nthreads; ++t) {
    const int64_t b = std::min<int64_t>(count, t * per), e = std::min<int64_t>(count, b + per);
    th.emplace_back([=] { f(t, b, e); });
  }
  for (auto& x : th) x.join();
}

// Large host arrays (the CSR of configuration 5: 5.4 GB) go to the device through a ring of
// pinned staging buffers filled by several host threads while the previous chunk is in flight
// (pageable cudaMemcpy ran at ~5 GB/s: 1.0 s of that setup); small ones by a plain copy.
template <class T>
static int upload_staged(tls_ctx* ctx, T*& d, const T* h, int64_t count) {
  const size_t bytes = sizeof(T) * (size_t)std::max<int64_t>(count, 0);
  size_t CH = (size_t)32 << 20, min_bytes = (size_t)256 << 20;
  if (const char* e = getenv("TLS_STAGED_CHUNK_BYTES")) CH = std::max<size_t>(4096, (size_t)atoll(e));  // tests
  if (const char* e = getenv("TLS_STAGED_MIN_BYTES")) min_bytes = (size_t)atoll(e);
  constexpr int NBUF = 3;
  if (bytes < min_bytes || bytes == 0) return upload(ctx, d, h, count);
  TRY(dalloc(ctx, d, count));
  void* pin[NBUF] = {nullptr, nullptr, nullptr};
  cudaEvent_t ev[NBUF];
  cudaStream_t st = nullptr;
  bool ok = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) == cudaSuccess;
  int nev = 0;
  for (int i = 0; ok && i < NBUF; ++i) {
    ok = cudaHostAlloc(&pin[i], CH, cudaHostAllocDefault) == cudaSuccess &&
         cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming) == cudaSuccess;
    if (ok) ++nev;
  }
  cudaError_t err = cudaSuccess;
  if (ok) {
    const int nt = host_threads();
    const char* src = reinterpret_cast<const char*>(h);
    char* dst = reinterpret_cast<char*>(d);
    int c = 0;
    for (size_t off = 0; off < bytes && err == cudaSuccess; off += CH, ++c) {
      const int b = c % NBUF;
      const size_t nb = std::min(CH, bytes - off);
      if (c >= NBUF) err = cudaEventSynchronize(ev[b]);
      if (err != cudaSuccess) break;
      char* p = static_cast<char*>(pin[b]);
      parallel_chunks((int64_t)nb, nt, [&](int, int64_t b0, int64_t e0) { memcpy(p + b0, src + off + b0, (size_t)(e0 - b0)); });
      err = cudaMemcpyAsync(dst + off, p, nb, cudaMemcpyHostToDevice, st);
      if (err == cudaSuccess) err = cudaEventRecord(ev[b], st);
    }
    if (err == cudaSuccess) err = cudaStreamSynchronize(st);
  } else {
    cudaGetLastError();
  }
  for (int i = 0; i < NBUF; ++i) {
    if (i < nev) cudaEventDestroy(ev[i]);
    if (pin[i]) cudaFreeHost(pin[i]);
  }
  if (st) cudaStreamDestroy(st);
  if (!ok) {  // no pinned memory: plain copy
    CK(cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice));
    return TLS_OK;
  }
  CK(err);
  return TLS_OK;
}

// The dynamic shared-memory limit is a per-(function, device) attribute: cudaFuncSetAttribute
// applies to the CURRENT device only, so the raised value is remembered per device and only ever
// raised, under a lock (several handles may be set up concurrently from host threads, possibly on
// different GPUs).  The caller must have made `device` current.
static cudaError_t raise_smem(int device, const void* fn, size_t bytes) {
  static std::mutex m;
  static std::map<std::pair<const void*, int>, size_t> current;
  std::lock_guard<std::mutex> lk(m);
  size_t& cur = current[{fn, device}];
  if (cur == 0) cur = 48 * 1024;  // the default limit every kernel starts with
  if (bytes <= cur) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) cur = bytes;
  return e;
}

// opt-in shared memory per block of `device` (227 KB on B200)
static size_t smem_optin(int device) {
  int v = 0;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, device) != cudaSuccess || v <= 0)
    v = 227 * 1024;
  return (size_t)v;
}

// every kernel launch of the library: cudaLaunchKernelEx with programmatic stream serialization
// (PDL) when ctx->pdl; errors surface through cudaGetLastError (CKL / the callers' checks)
template <typename... KArgs, typename... Args>
static void launch_k(const tls_ctx* ctx, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                     cudaStream_t s, Args&&... args);

static int grid_for(int64_t work, int per_block) {
  int64_t g = (work + per_block - 1) / per_block;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, MAX_GRID));
}

// after a replay of a timed graph: add the band-solve node durations; nodes whose kernel
// returned at once (the solve had converged) take a few us and are not launches of the solve
static void harvest_ktime(tls_ctx* ctx, int npairs) {
  if (!ctx->ktime) return;
  std::vector<float> ms(npairs, 0.f);
  float mx = 0.f;
  for (int i = 0; i < npairs; ++i) {
    if (cudaEventElapsedTime(&ms[i], ctx->kt_a[i], ctx->kt_b[i]) != cudaSuccess) ms[i] = 0.f;
    mx = std::max(mx, ms[i]);
  }
  for (int i = 0; i < npairs; ++i)
    if (ms[i] > 0.25f * mx && ms[i] > 0.004f) {
      ctx->kt_sum_ms += ms[i];
      ctx->kt_count++;
    }
}

static void destroy_graphs(tls_ctx* ctx) {
  for (int i = 0; i < 2; ++i) {
    if (ctx->pcg_exec[i]) cudaGraphExecDestroy(ctx->pcg_exec[i]);
    if (ctx->gm_exec[i]) cudaGraphExecDestroy(ctx->gm_exec[i]);
    ctx->pcg_exec[i] = ctx->gm_exec[i] = nullptr;
    ctx->gm_exec_cols[i] = 0;
  }
}

// ---------------------------------------------------------------------------------------------
// enqueue helpers
// ---------------------------------------------------------------------------------------------
// rows [r0, r1): all rows on one GPU, the owned range on the sharded path
template <int MODE, int DOT>
static int spmv_lpr(tls_ctx* ctx, cudaStream_t s, const double* x, double* y, const double* b,
                    double* part, const int* done) {
  const int grid = ctx->Gs;
#define SPMV_CASE(L)                                                                                 \
  case L:                                                                                            \
    launch_k(ctx, k_spmv<L, MODE, DOT>, grid, NTHR, 0, s, ctx->r0, ctx->r1, ctx->rowptr, ctx->col, ctx->val, x, y, \
                                               b, part, done);                                       \
    break;
  switch (ctx->lpr) {
    SPMV_CASE(1)
    SPMV_CASE(2)
    SPMV_CASE(4)
    SPMV_CASE(8)
    SPMV_CASE(16)
    SPMV_CASE(32)
    default: return fail(ctx, TLS_ERR_ARG, "bad lanes-per-row");
  }
#undef SPMV_CASE
  CKL();
  return TLS_OK;
}

// which unit/out lists a solve stage uses
enum { L_LOCAL = 0, L_COARSE = 1, L_ALL = 2 };

// y0 = X c is in yloc's coarse segment, c in xloc's: one refinement step
// rho = c - A0 y0 (block nsub+1), y0 += X rho (block nsub+2) -- restores a backward-stable coarse
// solve (the reference factors A0, src/coarse.py:178-182) when cond(A0) makes X c alone lose digits
static int enq_coarse_refine(tls_ctx* ctx, cudaStream_t s, const int* done) {
  const long long c0 = ctx->coarse_xoff, P = ctx->cpad;
  const int nc = ctx->ncoarse, g = grid_for(nc, NTHR);
  const int u1 = ctx->nu_local + ctx->nu_coarse, o1 = ctx->no_local + ctx->no_coarse;
  const int u2 = u1 + ctx->nu_ref1, o2 = o1 + ctx->no_ref1;
  launch_k(ctx, k_lincomb, g, NTHR, 0, s, nc, (const double*)(ctx->yloc + c0), (const double*)nullptr, 0.0,
           ctx->xloc + c0 + P, done);
  CKL();
  launch_k(ctx, k_symv_tiles, ctx->nu_ref1, NTHR, 0, s, ctx->d_blk, ctx->d_units + u1, ctx->xloc, ctx->slots, done);
  CKL();
  launch_k(ctx, k_reduce_tiles, (ctx->no_ref1 + 7) / 8, NTHR, 0, s, ctx->d_blk, ctx->d_outs + o1, ctx->no_ref1,
           ctx->d_red, ctx->slots, ctx->yloc, done);
  CKL();
  launch_k(ctx, k_lincomb, g, NTHR, 0, s, nc, (const double*)(ctx->xloc + c0), (const double*)(ctx->yloc + c0 + P),
           -1.0, ctx->xloc + c0 + 2 * P, done);
  CKL();
  launch_k(ctx, k_symv_tiles, ctx->nu_ref2, NTHR, 0, s, ctx->d_blk, ctx->d_units + u2, ctx->xloc, ctx->slots, done);
  CKL();
  launch_k(ctx, k_reduce_tiles, (ctx->no_ref2 + 7) / 8, NTHR, 0, s, ctx->d_blk, ctx->d_outs + o2, ctx->no_ref2,
           ctx->d_red, ctx->slots, ctx->yloc, done);
  CKL();
  launch_k(ctx, k_lincomb, g, NTHR, 0, s, nc, (const double*)(ctx->yloc + c0), (const double*)(ctx->yloc + c0 + 2 * P),
           1.0, ctx->yloc + c0, done);
  CKL();
  return TLS_OK;
}

// r_src (band local operators only): gather R_i r inside the band kernel instead of from xloc
// Coarse solve A0 yc = c by block forward / backward substitution on the block-tridiagonal A0
// (blocks of chain_bs columns; S_0 = A_00, S_i = A_ii - A_{i,i-1} S_{i-1}^{-1} A_{i-1,i}):
//   forward   z_i = c_i - A_{i,i-1} y_{i-1},  y_i = S_i^{-1} z_i
//   backward  x_i = S_i^{-1} (z_i - A_{i,i+1} x_{i+1})          (x_{nb-1} = y_{nb-1})
// in place on the coarse segments: z overwrites c in xloc, y and then x live in yloc.  The
// products with S_i^{-1} are tile blocks of k_symv_tiles, the off-diagonal ones sparse row sweeps.
// Replaces the solve_coarse closure of src/coarse.py:178-182 (a Cholesky solve with A0).
static int enq_coarse_chain(tls_ctx* ctx, cudaStream_t s, const int* done) {
  const int nb = ctx->chain_nb, bs = ctx->chain_bs, nc = ctx->ncoarse;
  double* z = ctx->xloc + ctx->coarse_xoff;
  double* y = ctx->yloc + ctx->coarse_xoff;
  auto block = [&](int i) -> int {
    launch_k(ctx, k_symv_tiles, ctx->chain_nu[i], NTHR, 0, s, ctx->d_blk, ctx->d_units + ctx->chain_u0[i],
             ctx->xloc, ctx->slots, done);
    CKL();
    launch_k(ctx, k_reduce_tiles, (ctx->chain_no[i] + 7) / 8, NTHR, 0, s, ctx->d_blk,
             ctx->d_outs + ctx->chain_o0[i], ctx->chain_no[i], ctx->d_red, ctx->slots, ctx->yloc, done);
    CKL();
    return TLS_OK;
  };
  auto offdiag = [&](int i, const int* ptr, const int* idx, const double* val) -> int {
    const int r0 = i * bs, r1 = std::min(nc, r0 + bs);
    launch_k(ctx, k_chain_spmv, grid_for((long long)(r1 - r0) * 32, NTHR), NTHR, 0, s, r0, r1, ptr, idx, val,
             (const double*)y, z, done);
    CKL();
    return TLS_OK;
  };
  for (int i = 0; i < nb; ++i) {
    if (i > 0) TRY(offdiag(i, ctx->d_lo_ptr, ctx->d_lo_idx, ctx->d_lo_val));
    TRY(block(i));
  }
  for (int i = nb - 2; i >= 0; --i) {
    TRY(offdiag(i, ctx->d_up_ptr, ctx->d_up_idx, ctx->d_up_val));
    TRY(block(i));
  }
  return TLS_OK;
}

static int enq_solve(tls_ctx* ctx, cudaStream_t s, int which, const int* done,
                     const double* r_src = nullptr) {
  if (ctx->local_kind >= 1 && which != L_COARSE) {
    const bool timed = ctx->ktime && ctx->capturing;
    if (timed) {
      while ((int)ctx->kt_a.size() <= ctx->kt_n) {
        cudaEvent_t a, b;
        CK(cudaEventCreate(&a));
        CK(cudaEventCreate(&b));
        ctx->kt_a.push_back(a);
        ctx->kt_b.push_back(b);
      }
      CK(cudaEventRecordWithFlags(ctx->kt_a[ctx->kt_n], s, cudaEventRecordExternal));
    }
    if (ctx->band_tma == 5)
      launch_k(ctx, k_band_solve_tma<5>, ctx->nsub, NTHR, ctx->band_smem + ring_bytes(5) + TMA_BAR_BYTES, s,
               ctx->d_band, ctx->xloc, ctx->yloc, done, r_src ? ctx->d_gidx : nullptr, r_src);
    else if (ctx->band_tma == 4)
      launch_k(ctx, k_band_solve_tma<4>, ctx->nsub, NTHR, ctx->band_smem + ring_bytes(4) + TMA_BAR_BYTES, s,
               ctx->d_band, ctx->xloc, ctx->yloc, done, r_src ? ctx->d_gidx : nullptr, r_src);
    else if (ctx->band_ring == 4)
      launch_k(ctx, k_band_solve_ring<4>, ctx->nsub, NTHR, ctx->band_smem + ring_bytes(4), s, 
          ctx->d_band, ctx->xloc, ctx->yloc, done, r_src ? ctx->d_gidx : nullptr, r_src);
    else if (ctx->band_ring == 2)
      launch_k(ctx, k_band_solve_ring<2>, ctx->nsub, NTHR, ctx->band_smem + ring_bytes(2), s, 
          ctx->d_band, ctx->xloc, ctx->yloc, done, r_src ? ctx->d_gidx : nullptr, r_src);
    else if (ctx->band_unr == 2)
      launch_k(ctx, k_band_solve<2>, ctx->nsub, NTHR, ctx->band_smem, s, ctx->d_band, ctx->xloc, ctx->yloc, done, ctx->band_pf,
                                                              r_src ? ctx->d_gidx : nullptr, r_src);
    else
      launch_k(ctx, k_band_solve<1>, ctx->nsub, NTHR, ctx->band_smem, s, ctx->d_band, ctx->xloc, ctx->yloc, done, ctx->band_pf,
                                                              r_src ? ctx->d_gidx : nullptr, r_src);
    CKL();
    if (timed) CK(cudaEventRecordWithFlags(ctx->kt_b[ctx->kt_n++], s, cudaEventRecordExternal));
    if (which == L_LOCAL) return TLS_OK;
    which = L_COARSE;
  }
  if (ctx->chain_nb > 0 && which != L_LOCAL) {
    if (which == L_ALL) TRY(enq_solve(ctx, s, L_LOCAL, done));
    return enq_coarse_chain(ctx, s, done);
  }
  int u0 = 0, nu = 0, o0 = 0, no = 0;
  if (which == L_LOCAL) { nu = ctx->nu_local; no = ctx->no_local; }
  if (which == L_COARSE) { u0 = ctx->nu_local; nu = ctx->nu_coarse; o0 = ctx->no_local; no = ctx->no_coarse; }
  if (which == L_ALL) { nu = ctx->nu_local + ctx->nu_coarse; no = ctx->no_local + ctx->no_coarse; }
  if (nu > 0) {
    launch_k(ctx, k_symv_tiles, nu, NTHR, 0, s, ctx->d_blk, ctx->d_units + u0, ctx->xloc, ctx->slots, done);
    CKL();
  }
  if (no > 0) {
    launch_k(ctx, k_reduce_tiles, (no + 7) / 8, NTHR, 0, s, ctx->d_blk, ctx->d_outs + o0, no, ctx->d_red,
                                                 ctx->slots, ctx->yloc, done);
    CKL();
  }
  if (ctx->cref && which != L_LOCAL) TRY(enq_coarse_refine(ctx, s, done));
  return TLS_OK;
}

static int enq_gather(tls_ctx* ctx, cudaStream_t s, const double* r, const int* done) {
  launch_k(ctx, k_gather, grid_for(ctx->Xloc, NTHR), NTHR, 0, s, ctx->Xloc, ctx->d_gidx, r, ctx->xloc, done);
  CKL();
  return TLS_OK;
}

static int enq_restrict(tls_ctx* ctx, cudaStream_t s, const double* r, const int* done) {
  // one warp per coarse column; all columns of a subdomain in one CTA (r_int gathered once)
  const int cw = ctx->restrict_cw;
  const dim3 grid(ctx->nsub, (ctx->kmax + cw - 1) / cw);
  launch_k(ctx, k_restrict, grid, 32 * std::min(ctx->kmax, cw), ctx->restrict_smem, s, 
      ctx->d_sub_idxoff, ctx->d_idx, ctx->d_nint, ctx->d_zoff,
                                        ctx->d_kcnt, ctx->d_cstart, ctx->d_Z, r,
                                        ctx->xloc + ctx->coarse_xoff, done);
  CKL();
  return TLS_OK;
}

// rows [r0, r1) only (all rows on one GPU); row-indexed arrays are offset, yloc / yc are not
template <int MODE, int DOT>
static int enq_prolong(tls_ctx* ctx, cudaStream_t s, const double* qv, const double* wv,
                       const double* rdot, double* z, const int* done) {
  const int r0 = ctx->r0;
  launch_k(ctx, k_prolong<MODE, DOT>, ctx->G, NTHR, 0, s, 
      ctx->r1 - r0, ctx->d_pull_ptr + r0, ctx->d_pull_pos, ctx->yloc, ctx->d_zrow + r0, ctx->d_zst + r0,
      ctx->d_zk + r0, ctx->d_zc + r0, ctx->d_Z, ctx->yloc + ctx->coarse_xoff, qv ? qv + r0 : nullptr,
      wv ? wv + r0 : nullptr, rdot ? rdot + r0 : nullptr, z + r0, ctx->part, done);
  CKL();
  return TLS_OK;
}

static bool has_coarse(const tls_ctx* ctx) { return ctx->ncoarse > 0 && ctx->combine != TLS_NONE; }

// a communicator of one rank (Shard(single=True): the NCCL transport exercised on a 1-GPU box) runs
// the sharded schedule as well; the plain single-GPU path never creates a communicator
static bool sharded(const tls_ctx* ctx) { return ctx->comm != nullptr; }

static int nown(const tls_ctx* ctx) { return ctx->r1 - ctx->r0; }

// in-place sum over the ranks (NCCL or in-process group); no-op on one GPU
static int enq_allreduce(tls_ctx* ctx, cudaStream_t s, double* buf, long long count) {
  if (!sharded(ctx)) return TLS_OK;
  std::string err;
  cudaError_t e = ctx->comm->allreduce_sum(buf, count, s, err);
  if (e != cudaSuccess) return fail(ctx, TLS_ERR_CUDA, err.empty() ? cudaGetErrorString(e) : err);
  return TLS_OK;
}

// the np (fixed, equal on every rank) partial sums of a dot product: folded to ONE scalar on each
// rank (fixed-order sum into part[0], the rest zeroed, so the consumers' partial sums are
// unchanged), then that scalar is summed over the ranks -- an 8-byte all-reduce, not 8 np bytes
static int enq_allreduce_part(tls_ctx* ctx, cudaStream_t s, int np) {
  if (!sharded(ctx)) return TLS_OK;
  launch_k(ctx, k_fold_partials, 1, NTHR, 0, s, ctx->part, np);
  CKL();
  return enq_allreduce(ctx, s, ctx->part, 1);
}

// point-to-point exchange: pack src rows, send/recv, unpack into dst.  Every rank calls every
// exchange of the schedule (possibly with an empty plan) so the collective order matches.
static int enq_exchange(tls_ctx* ctx, cudaStream_t s, XPlan& x, const double* src, double* dst,
                        const int* done) {
  if (!sharded(ctx)) return TLS_OK;
  if (x.stot > 0) {
    launch_k(ctx, k_xpack, grid_for(x.stot, NTHR), NTHR, 0, s, x.stot, x.d_sidx, src, x.sbuf, done);
    CKL();
  }
  std::string err;
  cudaError_t e = ctx->comm->exchange(x, s, err);
  if (e != cudaSuccess) return fail(ctx, TLS_ERR_CUDA, err.empty() ? cudaGetErrorString(e) : err);
  if (x.rtot > 0) {
    launch_k(ctx, k_xunpack, grid_for(x.rtot, NTHR), NTHR, 0, s, x.rtot, x.d_ridx, x.rbuf, dst, done);
    CKL();
  }
  return TLS_OK;
}

// ghost rows of v (rows other ranks own that this rank's SpMV rows / subdomains read)
static int enq_halo(tls_ctx* ctx, cudaStream_t s, double* v, const int* done) {
  return enq_exchange(ctx, s, ctx->halo, v, v, done);
}

// ASM: local-solve outputs on rows owned by other ranks travel to the owners, who add them in
// ascending subdomain order (their pull maps point into the received tail of yloc)
static int enq_rev(tls_ctx* ctx, cudaStream_t s, const int* done) {
  if (ctx->one_level != TLS_ASM) return TLS_OK;
  return enq_exchange(ctx, s, ctx->rev, ctx->yloc, ctx->yloc, done);
}

// coarse coefficients c = Z^T r: this rank's columns, then every rank's columns everywhere (an
// all-gather of the per-rank column segments when the layout is known, else a sum all-reduce of
// the zero-padded vector)
static int enq_restrict_all(tls_ctx* ctx, cudaStream_t s, const double* r, const int* done) {
  double* c = ctx->xloc + ctx->coarse_xoff;
  const bool gather = sharded(ctx) && ctx->d_ccol && ctx->cmax > 0;
  if (sharded(ctx) && !gather) CK(cudaMemsetAsync(c, 0, sizeof(double) * ctx->ncoarse, s));
  TRY(enq_restrict(ctx, s, r, done));
  if (!gather) return enq_allreduce(ctx, s, c, ctx->ncoarse);
  const int q = ctx->comm->rank;
  const long long c0 = ctx->ccol[q], cnt = ctx->ccol[q + 1] - c0;
  if (cnt > 0) CK(cudaMemcpyAsync(ctx->cg_send, c + c0, sizeof(double) * cnt, cudaMemcpyDeviceToDevice, s));
  std::string err;
  cudaError_t e = ctx->comm->allgather(ctx->cg_send, ctx->cmax, ctx->cg_recv, s, err);
  if (e != cudaSuccess) return fail(ctx, TLS_ERR_CUDA, err.empty() ? cudaGetErrorString(e) : err);
  const long long tot = (long long)ctx->comm->nranks * ctx->cmax;
  launch_k(ctx, k_coarse_unpack, grid_for(tot, NTHR), NTHR, 0, s, tot, ctx->cmax, (const long long*)ctx->d_ccol,
           (const double*)ctx->cg_recv, c, done);
  CKL();
  return TLS_OK;
}

static int enq_dot(tls_ctx* ctx, cudaStream_t s, const double* a, const double* b, const int* done) {
  launch_k(ctx, k_dot, ctx->G, NTHR, 0, s, nown(ctx), a + ctx->r0, b + ctx->r0, ctx->part, done);
  CKL();
  return enq_allreduce_part(ctx, s, ctx->G);
}

// one-level local solves of r: gather + tiles, or the band kernel gathering r itself
static int enq_local(tls_ctx* ctx, cudaStream_t s, const double* r, const int* done) {
  if (ctx->local_kind >= 1) return enq_solve(ctx, s, L_LOCAL, done, r);
  TRY(enq_gather(ctx, s, r, done));
  return enq_solve(ctx, s, L_LOCAL, done);
}

// z = M^{-1} r (src/precond.py:128-136) on the owned rows.  r must be valid on the owned rows;
// r_full: its ghost rows are valid too (no halo needed).  dot: r.z partials (summed over the
// ranks) in ctx->part (G of them).
static int enq_apply(tls_ctx* ctx, cudaStream_t s, double* r, double* z, bool dot, const int* done,
                     bool r_full = false) {
  if (!has_coarse(ctx)) {
    if (!r_full) TRY(enq_halo(ctx, s, r, done));
    TRY(enq_local(ctx, s, r, done));
    TRY(enq_rev(ctx, s, done));
    TRY(dot ? enq_prolong<0, 1>(ctx, s, nullptr, nullptr, r, z, done)
            : enq_prolong<0, 0>(ctx, s, nullptr, nullptr, r, z, done));
  } else if (ctx->combine == TLS_ADDITIVE && ctx->local_kind >= 1) {
    if (!r_full) TRY(enq_halo(ctx, s, r, done));
    // the coarse chain (restrict -> [sum over ranks] -> A0^{-1} tiles -> reduce) reads r and
    // writes only the coarse segments, the band solve reads/writes only the local segments: run
    // them side by side (a fork/join that CUDA-graph capture turns into parallel branches)
    // (the coarse prolongation Z yc is computed on that branch too, into cz; the prolongation
    // after the join only adds the local-solve contributions to it)
    CK(cudaEventRecord(ctx->ev_fork, s));
    CK(cudaStreamWaitEvent(ctx->aux, ctx->ev_fork, 0));
    TRY(enq_restrict_all(ctx, ctx->aux, r, done));
    TRY(enq_solve(ctx, ctx->aux, L_COARSE, done));
    TRY((enq_prolong<2, 0>(ctx, ctx->aux, nullptr, nullptr, nullptr, ctx->cz, done)));
    CK(cudaEventRecord(ctx->ev_join, ctx->aux));
    TRY(enq_local(ctx, s, r, done));
    CK(cudaStreamWaitEvent(s, ctx->ev_join, 0));
    TRY(enq_rev(ctx, s, done));
    TRY(dot ? enq_prolong<4, 1>(ctx, s, ctx->cz, nullptr, r, z, done)
            : enq_prolong<4, 0>(ctx, s, ctx->cz, nullptr, r, z, done));
  } else if (ctx->combine == TLS_ADDITIVE) {
    if (!r_full) TRY(enq_halo(ctx, s, r, done));
    TRY(enq_gather(ctx, s, r, done));
    TRY(enq_restrict_all(ctx, s, r, done));
    TRY(enq_solve(ctx, s, L_ALL, done));
    TRY(enq_rev(ctx, s, done));
    TRY(dot ? enq_prolong<1, 1>(ctx, s, nullptr, nullptr, r, z, done)
            : enq_prolong<1, 0>(ctx, s, nullptr, nullptr, r, z, done));
  } else {
    // deflated: q = Q r; w = M1 (r - A q); z = q + w - Q A w  (only the owned rows of r are read
    // directly; q and w get their ghost rows by halo before each SpMV / gather)
    TRY(enq_restrict_all(ctx, s, r, done));
    TRY(enq_solve(ctx, s, L_COARSE, done));
    TRY((enq_prolong<2, 0>(ctx, s, nullptr, nullptr, nullptr, ctx->t1, done)));
    TRY(enq_halo(ctx, s, ctx->t1, done));
    TRY((spmv_lpr<1, 0>(ctx, s, ctx->t1, ctx->t2, r, nullptr, done)));
    TRY(enq_halo(ctx, s, ctx->t2, done));
    TRY(enq_local(ctx, s, ctx->t2, done));
    TRY(enq_rev(ctx, s, done));
    TRY((enq_prolong<0, 0>(ctx, s, nullptr, nullptr, nullptr, ctx->t3, done)));
    TRY(enq_halo(ctx, s, ctx->t3, done));
    TRY((spmv_lpr<0, 0>(ctx, s, ctx->t3, ctx->t4, nullptr, nullptr, done)));
    TRY(enq_restrict_all(ctx, s, ctx->t4, done));
    TRY(enq_solve(ctx, s, L_COARSE, done));
    TRY(dot ? enq_prolong<3, 1>(ctx, s, ctx->t1, ctx->t3, r, z, done)
            : enq_prolong<3, 0>(ctx, s, ctx->t1, ctx->t3, r, z, done));
  }
  return dot ? enq_allreduce_part(ctx, s, ctx->G) : TLS_OK;
}

static int enq_identity(tls_ctx* ctx, cudaStream_t s, const double* r, double* z, bool dot,
                        const int* done) {
  const int r0 = ctx->r0;
  if (dot)
    launch_k(ctx, k_copy_dot<1>, ctx->G, NTHR, 0, s, nown(ctx), r + r0, z + r0, ctx->part, done);
  else
    launch_k(ctx, k_copy_dot<0>, ctx->G, NTHR, 0, s, nown(ctx), r + r0, z + r0, ctx->part, done);
  CKL();
  return dot ? enq_allreduce_part(ctx, s, ctx->G) : TLS_OK;
}

// Caller-numbering vectors at the C ABI.  One GPU: used in place.  Sharded: v_in is permuted
// into the internal numbering (all rows, so no halo is needed), the operator writes its owned
// rows of ctx->pout, and out = the sum over ranks of the owned rows scattered back.
static int api_in(tls_ctx* ctx, cudaStream_t s, const double* v_in, double** v_int) {
  if (ctx->h_nofo.empty()) {
    *v_int = const_cast<double*>(v_in);
    return TLS_OK;
  }
  launch_k(ctx, k_perm_in, grid_for(ctx->n, NTHR), NTHR, 0, s, ctx->n, ctx->d_nofo, v_in, ctx->pin);
  CKL();
  *v_int = ctx->pin;
  return TLS_OK;
}
static double* api_out_buf(tls_ctx* ctx, double* out) { return ctx->h_nofo.empty() ? out : ctx->pout; }
static int api_out(tls_ctx* ctx, cudaStream_t s, const double* v_int, double* out) {
  if (ctx->h_nofo.empty()) {
    if (v_int != out) CK(cudaMemcpyAsync(out, v_int, sizeof(double) * ctx->n, cudaMemcpyDeviceToDevice, s));
    return TLS_OK;
  }
  launch_k(ctx, k_perm_out, grid_for(ctx->n, NTHR), NTHR, 0, s, ctx->n, ctx->d_nofo, ctx->r0, ctx->r1, v_int, out);
  CKL();
  return enq_allreduce(ctx, s, out, ctx->n);
}

// ---------------------------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------------------------
extern "C" {

int32_t tls_abi_version(void) { return TLS_ABI_VERSION; }

int32_t tls_ctx_create(int32_t device, tls_ctx** out) {
  if (!out) return TLS_ERR_ARG;
  *out = nullptr;
  tls_ctx* ctx = new tls_ctx();
  ctx->device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->cap, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->aux, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaMallocHost((void**)&ctx->h_flag, sizeof(int) * 4);
  if (e != cudaSuccess) {
    delete ctx;
    return TLS_ERR_CUDA;
  }
  if (cudaMalloc((void**)&ctx->pcg, sizeof(PcgState)) != cudaSuccess ||
      cudaMalloc((void**)&ctx->gm, sizeof(GmState)) != cudaSuccess) {
    delete ctx;
    return TLS_ERR_OOM;
  }
  if (const char* e = getenv("TLS_PDL")) ctx->pdl = atoi(e) != 0;
  *out = ctx;
  return TLS_OK;
}

void tls_ctx_destroy(tls_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaDeviceSynchronize();
  destroy_graphs(ctx);
  dfree(ctx->rowptr); dfree(ctx->col); dfree(ctx->val);
  dfree(ctx->d_sub_idxoff); dfree(ctx->d_sub_n); dfree(ctx->d_idx); dfree(ctx->d_nint);
  dfree(ctx->d_blk); dfree(ctx->tiles); dfree(ctx->d_Z); dfree(ctx->ctiles); dfree(ctx->a0tiles); dfree(ctx->d_zoff);
  dfree(ctx->chain_tiles); dfree(ctx->d_lo_ptr); dfree(ctx->d_lo_idx); dfree(ctx->d_lo_val);
  dfree(ctx->d_up_ptr); dfree(ctx->d_up_idx); dfree(ctx->d_up_val);
  dfree(ctx->d_kcnt); dfree(ctx->d_cstart); dfree(ctx->d_units); dfree(ctx->d_outs); dfree(ctx->d_red);
  dfree(ctx->d_gidx); dfree(ctx->d_pull_ptr); dfree(ctx->d_pull_pos); dfree(ctx->d_zrow);
  dfree(ctx->d_zk); dfree(ctx->d_zc); dfree(ctx->d_zst); dfree(ctx->xloc); dfree(ctx->yloc); dfree(ctx->slots);
  double** vecs[] = {&ctx->t1, &ctx->t2, &ctx->t3, &ctx->t4, &ctx->t5, &ctx->t6, &ctx->t7, &ctx->vb,
                     &ctx->vx, &ctx->vr, &ctx->vp, &ctx->vap, &ctx->vz, &ctx->hist, &ctx->part,
                     &ctx->V, &ctx->H, &ctx->cs, &ctx->sn, &ctx->gv, &ctx->yv, &ctx->h1, &ctx->h2,
                     &ctx->pin, &ctx->pout, &ctx->cz, &ctx->halo.sbuf, &ctx->halo.rbuf, &ctx->rev.sbuf,
                     &ctx->rev.rbuf};
  for (double** v : vecs) dfree(*v);
  dfree(ctx->d_nofo); dfree(ctx->halo.d_sidx); dfree(ctx->halo.d_ridx); dfree(ctx->rev.d_sidx);
  dfree(ctx->rev.d_ridx);
  dfree(ctx->pcg); dfree(ctx->gm);
  dfree(ctx->d_ccol); dfree(ctx->cg_send); dfree(ctx->cg_recv);
  dfree(ctx->g_ptr); dfree(ctx->g_adj);
  for (auto e : ctx->kt_a) cudaEventDestroy(e);
  for (auto e : ctx->kt_b) cudaEventDestroy(e);
  for (void* pb : ctx->band_allocs) cudaFree(pb);
  dfree(ctx->d_band);
  if (ctx->h_flag) cudaFreeHost(ctx->h_flag);
  if (ctx->h_x) cudaFreeHost(ctx->h_x);
  dfree(ctx->ab);
  if (ctx->cap) cudaStreamDestroy(ctx->cap);
  if (ctx->aux) cudaStreamDestroy(ctx->aux);
  if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
  if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
  delete ctx->comm;
  delete ctx;
}

const char* tls_ctx_last_error(const tls_ctx* ctx) { return ctx ? ctx->err.c_str() : "null handle"; }

int64_t tls_ctx_device_bytes(const tls_ctx* ctx) { return ctx ? ctx->dev_bytes : 0; }

int32_t tls_matrix_upload(tls_ctx* ctx, int64_t nrows, int64_t nnz, const int64_t* indptr,
                          const int32_t* indices, const double* data, int32_t symmetric) {
  TLS_RANGE("tls_matrix_upload");
  if (!ctx || nrows <= 0 || nrows > INT32_MAX || nnz < 0 || nnz >= INT32_MAX)
    return ctx ? fail(ctx, TLS_ERR_ARG, "matrix size out of the supported int32 range") : TLS_ERR_ARG;
  // host-side bounds check of the CSR structure: every device kernel indexes through indptr and
  // indices without checks, so a malformed matrix is refused here, before anything is uploaded
  if (!indptr || (nnz > 0 && (!indices || !data)))
    return fail(ctx, TLS_ERR_ARG, "null CSR array");
  if (indptr[0] != 0 || indptr[nrows] != nnz)
    return fail(ctx, TLS_ERR_DIM, "indptr must start at 0 and end at nnz");
  for (int64_t i = 0; i < nrows; ++i)
    if (indptr[i + 1] < indptr[i])
      return fail(ctx, TLS_ERR_DIM, "indptr decreases at row " + std::to_string(i));
  {  // the first out-of-range column, found by all host threads
    const int nt = host_threads();
    std::vector<int64_t> bad(nt, -1);
    parallel_chunks(nnz, nt, [&](int t, int64_t b, int64_t e) {
      for (int64_t k = b; k < e; ++k)
        if ((uint32_t)indices[k] >= (uint32_t)nrows) {
          bad[t] = k;
          return;
        }
    });
    for (int t = 0; t < nt; ++t)
      if (bad[t] >= 0)
        return fail(ctx, TLS_ERR_DIM, "column index out of range at entry " + std::to_string(bad[t]));
  }
  CK(cudaSetDevice(ctx->device));
  const bool renum = !ctx->h_nofo.empty();
  if (renum && (int64_t)ctx->h_nofo.size() != nrows)
    return fail(ctx, TLS_ERR_DIM, "row partition and matrix sizes differ");
  ctx->n = (int)nrows;
  ctx->nnz = nnz;
  ctx->sym = symmetric ? 1 : 0;
  std::vector<int> rp(nrows + 1);
  if (!renum) {
    for (int64_t i = 0; i <= nrows; ++i) rp[i] = (int)indptr[i];
    TRY(upload(ctx, ctx->rowptr, rp.data(), nrows + 1));
    TRY(upload_staged(ctx, ctx->col, indices, nnz));
    TRY(upload_staged(ctx, ctx->val, data, nnz));
    ctx->r0 = 0;
    ctx->r1 = (int)nrows;
  } else {
    // P A P^T in the internal numbering; each row keeps its entries in the caller's order, so
    // every row sum (SpMV) is bit-identical to the unpermuted one
    std::vector<int> oldof(nrows);
    for (int64_t g = 0; g < nrows; ++g) oldof[ctx->h_nofo[g]] = (int)g;
    rp[0] = 0;
    for (int64_t i = 0; i < nrows; ++i) rp[i + 1] = rp[i] + (int)(indptr[oldof[i] + 1] - indptr[oldof[i]]);
    std::vector<int> pc(nnz);
    std::vector<double> pv(nnz);
    for (int64_t i = 0; i < nrows; ++i) {
      const int64_t b = indptr[oldof[i]], e = indptr[oldof[i] + 1];
      for (int64_t k = b; k < e; ++k) {
        pc[rp[i] + (k - b)] = ctx->h_nofo[indices[k]];
        pv[rp[i] + (k - b)] = data[k];
      }
    }
    TRY(upload(ctx, ctx->rowptr, rp.data(), nrows + 1));
    TRY(upload(ctx, ctx->col, pc.data(), nnz));
    TRY(upload(ctx, ctx->val, pv.data(), nnz));
  }
  const double avg = nrows ? (double)nnz / (double)nrows : 1.0;
  // lanes per row ~ nnz/row / 7 (measured on B200: 7-point rows run best one thread per row,
  // 27-point rows with 4 lanes; tools/bench_spmv.py)
  int l = 1;
  while (l < 32 && 7 * l < avg) l *= 2;
  if (const char* e = getenv("TLS_SPMV_LPR")) {  // tuning override (1, 2, 4, 8, 16, 32)
    const int v = atoi(e);
    if (v == 1 || v == 2 || v == 4 || v == 8 || v == 16 || v == 32) l = v;
  }
  ctx->lpr = l;
  ctx->G = grid_for(nrows, NTHR);
  ctx->Gs = grid_for(nrows, NTHR / l);
  if (renum) ctx->G = ctx->Gs = MAX_GRID;  // equal partial counts on every rank (summed elementwise)
  const int64_t need = std::max<int64_t>(ctx->G, ctx->Gs);
  if (need > ctx->part_cap) {
    TRY(dalloc(ctx, ctx->part, need));
    ctx->part_cap = need;
  }
  double** vecs[] = {&ctx->t1, &ctx->t2, &ctx->t3, &ctx->t4, &ctx->t5, &ctx->t6, &ctx->t7,
                     &ctx->vb, &ctx->vx, &ctx->vr, &ctx->vp, &ctx->vap, &ctx->vz, &ctx->pin, &ctx->pout,
                     &ctx->cz};
  for (double** v : vecs) {
    TRY(dalloc(ctx, *v, nrows));
    CK(cudaMemset(*v, 0, sizeof(double) * nrows));  // ghost rows are read (x 0) before any halo
  }
  if (ctx->h_x) cudaFreeHost(ctx->h_x);
  CK(cudaMallocHost((void**)&ctx->h_x, sizeof(double) * nrows));
  destroy_graphs(ctx);
  ctx->finalized = false;
  return TLS_OK;
}

int32_t tls_spmv(tls_ctx* ctx, const double* x, double* y, void* stream) {
  TLS_RANGE("tls_spmv");
  if (!ctx || !ctx->rowptr) return ctx ? fail(ctx, TLS_ERR_STATE, "no matrix uploaded") : TLS_ERR_ARG;
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = (cudaStream_t)stream;
  double* xi;
  TRY(api_in(ctx, s, x, &xi));
  double* yi = api_out_buf(ctx, y);
  TRY((spmv_lpr<0, 0>(ctx, s, xi, yi, nullptr, nullptr, nullptr)));
  return api_out(ctx, s, yi, y);
}

int32_t tls_subdomains_upload(tls_ctx* ctx, int32_t n_sub_global, const int64_t* offsets_g,
                              const int64_t* indices_g, const int32_t* n_interior_g) {
  TLS_RANGE("tls_subdomains_upload");
  if (!ctx || n_sub_global <= 0) return ctx ? fail(ctx, TLS_ERR_ARG, "n_sub must be positive") : TLS_ERR_ARG;
  if (!ctx->rowptr) return fail(ctx, TLS_ERR_STATE, "upload the matrix first");
  CK(cudaSetDevice(ctx->device));
  // this handle keeps only its owned slab [own_lo, own_hi) of the global subdomain list
  const int lo = ctx->own_lo, hi = ctx->own_hi < 0 ? n_sub_global : ctx->own_hi;
  if (lo < 0 || hi > n_sub_global || lo >= hi) return fail(ctx, TLS_ERR_ARG, "owned subdomain range out of bounds");
  ctx->nsub_global = n_sub_global;
  ctx->own_hi = hi;
  const int n_sub = hi - lo;
  const int64_t base = offsets_g[lo];
  ctx->nsub = n_sub;
  ctx->h_off.resize(n_sub + 1);
  for (int s = 0; s <= n_sub; ++s) ctx->h_off[s] = offsets_g[lo + s] - base;
  const int64_t* offsets = ctx->h_off.data();
  const int64_t tot = offsets[n_sub];
  ctx->h_idx.resize(tot);
  for (int64_t i = 0; i < tot; ++i) {
    const int64_t g = indices_g[base + i];
    if (g < 0 || g >= ctx->n) return fail(ctx, TLS_ERR_DIM, "subdomain index out of range");
    ctx->h_idx[i] = ctx->h_nofo.empty() ? (int)g : ctx->h_nofo[g];  // internal numbering
  }
  ctx->h_n.resize(n_sub);
  ctx->h_nint.assign(n_interior_g + lo, n_interior_g + hi);
  ctx->max_n = 0;
  std::vector<long long> idxoff(n_sub);
  for (int s = 0; s < n_sub; ++s) {
    ctx->h_n[s] = (int)(offsets[s + 1] - offsets[s]);
    idxoff[s] = offsets[s];
    ctx->max_n = std::max(ctx->max_n, ctx->h_n[s]);
  }
  TRY(upload(ctx, ctx->d_sub_idxoff, idxoff.data(), n_sub));
  TRY(upload(ctx, ctx->d_idx, ctx->h_idx.data(), tot));
  TRY(upload(ctx, ctx->d_sub_n, ctx->h_n.data(), n_sub));
  TRY(upload(ctx, ctx->d_nint, ctx->h_nint.data(), n_sub));
  // tile storage for the local inverses: packed lower triangle (symmetric) or full
  ctx->h_blk.assign(n_sub + 3, BlkDesc{});  // + coarse block, + the two refinement blocks
  int64_t tiles = 0;
  long long xo = 0;
  std::vector<int64_t> tbase(n_sub);
  for (int s = 0; s < n_sub; ++s) {
    const int nt = (ctx->h_n[s] + TT - 1) / TT;
    tbase[s] = tiles;
    tiles += ctx->sym ? (int64_t)nt * (nt + 1) / 2 : (int64_t)nt * nt;
    ctx->h_blk[s].n = ctx->h_n[s];
    ctx->h_blk[s].nt = nt;
    ctx->h_blk[s].sym = ctx->sym;
    ctx->h_blk[s].xoff = xo;
    xo += (long long)nt * TT;
  }
  ctx->Xloc = xo;
  {
    int mi = 1;
    for (int s = 0; s < n_sub; ++s) mi = std::max(mi, ctx->h_nint[s]);
    ctx->restrict_smem = sizeof(double) * (size_t)mi;
    if (const char* e = getenv("TLS_RESTRICT_CW")) {  // tuning override (1..32)
      const int v = atoi(e);
      if (v >= 1 && v <= 32) ctx->restrict_cw = v;
    }
    if (ctx->restrict_smem > smem_optin(ctx->device))
      return fail(ctx, TLS_ERR_ARG, "subdomain interior of " + std::to_string(mi) +
                                        " rows exceeds the shared memory of the coarse restriction");
    CK(raise_smem(ctx->device, (const void*)k_restrict, ctx->restrict_smem));
  }
  ctx->tile_doubles = ctx->local_kind >= 1 ? 0 : tiles * TT * TT;
  dfree(ctx->tiles);
  TRY(dalloc(ctx, ctx->tiles, ctx->tile_doubles));
  if (ctx->local_kind >= 1) {
    ctx->h_band.assign(n_sub, BandDesc{});
    int maxnb = 0;
    for (int s = 0; s < n_sub; ++s) {
      ctx->h_band[s].n = ctx->h_n[s];
      ctx->h_band[s].nb = ctx->h_blk[s].nt;
      ctx->h_band[s].xoff = ctx->h_blk[s].xoff;
      maxnb = std::max(maxnb, ctx->h_blk[s].nt);
    }
    TRY(upload(ctx, ctx->d_band, ctx->h_band.data(), n_sub));
    ctx->band_smem = band_smem_bytes(maxnb);
    // the whole local vector lives in shared memory: refuse (clear error; setup then keeps the
    // inverse tiles) when even the plain kernel cannot hold the largest subdomain, and raise the
    // limit of a cp.async ring variant only when its rings fit too
    const size_t optin = smem_optin(ctx->device);
    if (ctx->band_smem > optin)
      return fail(ctx, TLS_ERR_ARG, "band local operators: a subdomain of " + std::to_string(ctx->max_n) +
                                        " rows exceeds the shared memory of k_band_solve (max " +
                                        std::to_string(band_max_rows(optin)) + " rows); use local='inverse'");
    CK(raise_smem(ctx->device, (const void*)k_band_solve<1>, ctx->band_smem));
    CK(raise_smem(ctx->device, (const void*)k_band_solve<2>, ctx->band_smem));
    // per-warp cp.async rings, 4 deep at 1 CTA/SM, when the subdomains fit one wave (<= 148;
    // an 8-rank configuration-2 slab: 0.79 -> 0.57 ms per iteration); otherwise the 4-CTA/SM
    // kernel (the 2-deep ring at 2 CTAs/SM for <= 296 subdomains measured cfg3 -4.5%, cfg4 +4.9%,
    // 2-rank slab +2%: selectable with TLS_BAND_RING=2; profiles/ab_band_ring_r01.txt)
    ctx->band_ring = n_sub <= 148 ? 4 : 0;
    if (const char* e = getenv("TLS_BAND_RING")) {
      const int v = atoi(e);
      if (v == 0 || v == 2 || v == 4) ctx->band_ring = v;
    }
    while (ctx->band_ring > 0 && ctx->band_smem + ring_bytes(ctx->band_ring) > optin) ctx->band_ring /= 2;
    if (ctx->band_ring == 1) ctx->band_ring = 0;
    if (ctx->band_ring == 4)
      CK(raise_smem(ctx->device, (const void*)k_band_solve_ring<4>, ctx->band_smem + ring_bytes(4)));
    // the same rings fed by the TMA engine (one 4 KB bulk copy + mbarrier per warp and tile instead
    // of 256 16-byte cp.async): TLS_BAND_TMA=4|5 (ring depth) where the ring kernel would run
    ctx->band_tma = 0;
    if (const char* e = getenv("TLS_BAND_TMA")) {
      const int v = atoi(e);
      if ((v == 4 || v == 5) && ctx->band_ring == 4) ctx->band_tma = v;
    }
    if (ctx->band_tma == 5 && ctx->band_smem + ring_bytes(5) + TMA_BAR_BYTES > optin) ctx->band_tma = 4;
    if (ctx->band_tma == 4 && ctx->band_smem + ring_bytes(4) + TMA_BAR_BYTES > optin) ctx->band_tma = 0;
    if (ctx->band_tma == 5)
      CK(raise_smem(ctx->device, (const void*)k_band_solve_tma<5>, ctx->band_smem + ring_bytes(5) + TMA_BAR_BYTES));
    if (ctx->band_tma == 4)
      CK(raise_smem(ctx->device, (const void*)k_band_solve_tma<4>, ctx->band_smem + ring_bytes(4) + TMA_BAR_BYTES));
    if (ctx->band_ring == 2)
      CK(raise_smem(ctx->device, (const void*)k_band_solve_ring<2>, ctx->band_smem + ring_bytes(2)));
    // one tile per load round: two (UNR = 2, 128 registers, 2 CTAs/SM) measured slower on
    // configuration 3 (1,249 vs 1,300 it/s) and mixed on 8-rank configuration 2 slabs
    // (profiles/ab_band_unr_r01.txt); kept selectable for the few-subdomains-per-GPU regime
    ctx->band_unr = 1;
    if (const char* e = getenv("TLS_BAND_UNR")) {
      const int v = atoi(e);
      if (v == 1 || v == 2) ctx->band_unr = v;
    }
    // prefetch distance 2 items (measured: 4 and 6 lose 1-15% on configurations 2 and 3 --
    // tools/sweep_pf.sh, profiles/pf_sweep_r01.txt)
    ctx->band_pf = 2;
    if (const char* e = getenv("TLS_BAND_PF")) {
      const int v = atoi(e);
      if (v >= 1 && v <= 16) ctx->band_pf = v;
    }
    ctx->h_perm.assign(tot, -1);
    ctx->h_perm_in.assign(ctx->local_kind == 2 ? tot : 0, -1);
    ctx->band_bytes = 0.0;
  }
  for (int s = 0; s < n_sub; ++s) ctx->h_blk[s].tiles = ctx->tiles + tbase[s] * TT * TT;
  TRY(upload(ctx, ctx->d_blk, ctx->h_blk.data(), n_sub + 3));
  ctx->stored.assign(n_sub, 0);
  ctx->ncoarse = 0;
  ctx->cref = false;
  ctx->finalized = false;
  destroy_graphs(ctx);
  return TLS_OK;
}

int32_t tls_subdomain_max_size(const tls_ctx* ctx) { return ctx ? ctx->max_n : 0; }

int32_t tls_extract_blocks(tls_ctx* ctx, int32_t first_g, int32_t count, double* out, int64_t ld,
                           void* stream) {
  TLS_RANGE("tls_extract_blocks");
  if (!ctx) return TLS_ERR_ARG;
  const int first = first_g - ctx->own_lo;
  if (first < 0 || count <= 0 || first + count > ctx->nsub)
    return fail(ctx, TLS_ERR_ARG, "subdomain range not owned by this handle");
  for (int s = first; s < first + count; ++s)
    if (ctx->h_n[s] > ld) return fail(ctx, TLS_ERR_ARG, "ld smaller than a local block");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = (cudaStream_t)stream;
  const long long base = ctx->h_off[first];
  const int items = (int)(ctx->h_off[first + count] - base);
  int *beg = nullptr, *pos = nullptr, *skey = nullptr, *sval = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  CK(cub::DeviceSegmentedSort::SortPairs(nullptr, tmp_bytes, ctx->d_idx + base, skey, pos, sval, items,
                                         count, beg, beg + count, s));
  CK(cudaMallocAsync((void**)&beg, sizeof(int) * 2 * (size_t)count, s));
  CK(cudaMallocAsync((void**)&pos, sizeof(int) * 3 * (size_t)items, s));
  CK(cudaMallocAsync(&tmp, tmp_bytes + 16, s));
  skey = pos + items;
  sval = pos + 2 * (size_t)items;
  CK(cudaMemsetAsync(out, 0, sizeof(double) * (size_t)count * ld * ld, s));
  dim3 g1(grid_for(ctx->max_n, NTHR) / 4 + 1, count);
  launch_k(ctx, k_seg_prep, g1, NTHR, 0, s, count, ctx->d_sub_idxoff, ctx->d_sub_n, first, beg, beg + count, pos);
  CKL();
  CK(cub::DeviceSegmentedSort::SortPairs(tmp, tmp_bytes, ctx->d_idx + base, skey, pos, sval, items, count, beg,
                                         beg + count, s));
  dim3 g2(std::max<int>(1, (int)std::min<int64_t>((ld + 7) / 8, 4096)), count);
  launch_k(ctx, k_extract, g2, NTHR, 0, s, count, ctx->d_sub_idxoff, ctx->d_sub_n, ctx->d_idx, first, skey, sval,
                                ctx->rowptr, ctx->col, ctx->val, out, ld);
  CKL();
  CK(cudaFreeAsync(tmp, s));
  CK(cudaFreeAsync(pos, s));
  CK(cudaFreeAsync(beg, s));
  return TLS_OK;
}

int32_t tls_store_local_inverse(tls_ctx* ctx, int32_t first_g, int32_t count, const double* inv,
                                int64_t ld, void* stream) {
  TLS_RANGE("tls_store_local_inverse");
  if (!ctx) return TLS_ERR_ARG;
  const int first = first_g - ctx->own_lo;
  if (first < 0 || count <= 0 || first + count > ctx->nsub)
    return fail(ctx, TLS_ERR_ARG, "subdomain range not owned by this handle");
  if (ctx->local_kind != 0) return fail(ctx, TLS_ERR_STATE, "handle stores band factors, not inverses");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = (cudaStream_t)stream;
  dim3 g(512, count);
  launch_k(ctx, k_pack_tiles, g, NTHR, 0, s, ctx->d_blk, first, inv, ld, ld * ld);
  CKL();
  for (int i = first; i < first + count; ++i) ctx->stored[i] = 1;
  ctx->finalized = false;
  return TLS_OK;
}

int32_t tls_coarse_upload(tls_ctx* ctx, int32_t n_coarse, const int32_t* k, const double* basis,
                          const double* a0inv, void* stream) {
  TLS_RANGE("tls_coarse_upload");
  if (!ctx || !ctx->nsub) return ctx ? fail(ctx, TLS_ERR_STATE, "upload subdomains first") : TLS_ERR_ARG;
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = (cudaStream_t)stream;
  ctx->finalized = false;
  destroy_graphs(ctx);
  ctx->cref = false;
  ctx->chain_nb = 0;
  dfree(ctx->chain_tiles);
  if (n_coarse <= 0 || !k) {
    ctx->ncoarse = 0;
    return TLS_OK;
  }
  // k[] covers all global subdomains (column numbering); the basis holds the owned ones
  ctx->h_k.assign(k + ctx->own_lo, k + ctx->own_hi);
  ctx->h_cstart.resize(ctx->nsub);
  ctx->h_zoff.resize(ctx->nsub);
  int c = 0;
  for (int g = 0; g < ctx->own_lo; ++g) c += k[g];
  long long zo = 0;
  for (int i = 0; i < ctx->nsub; ++i) {
    ctx->h_cstart[i] = c;
    ctx->h_zoff[i] = zo;
    c += ctx->h_k[i];
    zo += (long long)ctx->h_nint[i] * ctx->h_k[i];
  }
  for (int g = ctx->own_hi; g < ctx->nsub_global; ++g) c += k[g];
  if (c != n_coarse) return fail(ctx, TLS_ERR_ARG, "sum of k differs from n_coarse");
  ctx->kmax = 1;
  for (int i = 0; i < ctx->nsub; ++i) ctx->kmax = std::max(ctx->kmax, ctx->h_k[i]);
  ctx->ncoarse = n_coarse;
  TRY(dalloc(ctx, ctx->d_Z, zo));
  if (zo) CK(cudaMemcpyAsync(ctx->d_Z, basis, sizeof(double) * zo, cudaMemcpyDeviceToDevice, s));
  TRY(upload(ctx, ctx->d_zoff, ctx->h_zoff.data(), ctx->nsub));
  TRY(upload(ctx, ctx->d_kcnt, ctx->h_k.data(), ctx->nsub));
  TRY(upload(ctx, ctx->d_cstart, ctx->h_cstart.data(), ctx->nsub));
  // coarse operator tiles (block index nsub)
  BlkDesc cb{};
  cb.n = n_coarse;
  cb.nt = (n_coarse + TT - 1) / TT;
  cb.sym = ctx->sym;
  cb.xoff = ctx->Xloc;
  const int64_t ntiles = cb.sym ? (int64_t)cb.nt * (cb.nt + 1) / 2 : (int64_t)cb.nt * cb.nt;
  ctx->cpad = (long long)cb.nt * TT;
  ctx->h_blk.resize(ctx->nsub + 3);
  if (!a0inv) {  // no dense inverse: the operator follows as a block-tridiagonal chain
    dfree(ctx->ctiles);
    cb.tiles = nullptr;
    ctx->h_blk[ctx->nsub] = cb;
    return TLS_OK;
  }
  TRY(dalloc(ctx, ctx->ctiles, ntiles * TT * TT));
  cb.tiles = ctx->ctiles;
  ctx->h_blk[ctx->nsub] = cb;
  TRY(upload(ctx, ctx->d_blk, ctx->h_blk.data(), ctx->nsub + 3));
  dim3 g((unsigned)std::min<int64_t>(ntiles, 8192), 1);
  launch_k(ctx, k_pack_tiles, g, NTHR, 0, s, ctx->d_blk, ctx->nsub, a0inv, n_coarse, 0);
  CKL();
  return TLS_OK;
}

int32_t tls_coarse_chain(tls_ctx* ctx, int32_t n_blocks, int32_t block_size, const uint64_t* sinv,
                         const int32_t* lo_indptr, const int32_t* lo_indices, const double* lo_values,
                         const int32_t* up_indptr, const int32_t* up_indices, const double* up_values,
                         int64_t nnz, void* stream) {
  TLS_RANGE("tls_coarse_chain");
  if (!ctx || ctx->ncoarse <= 0) return ctx ? fail(ctx, TLS_ERR_STATE, "upload the coarse basis first") : TLS_ERR_ARG;
  if (!ctx->sym) return fail(ctx, TLS_ERR_ARG, "the block-tridiagonal coarse solve needs a symmetric operator");
  if (ctx->cref) return fail(ctx, TLS_ERR_STATE, "coarse refinement and the block-tridiagonal solve exclude each other");
  const int nc = ctx->ncoarse;
  if (n_blocks < 2 || block_size <= 0 || block_size % TT != 0 ||
      (long long)(n_blocks - 1) * block_size >= nc || (long long)n_blocks * block_size < nc)
    return fail(ctx, TLS_ERR_ARG, "block size must be a multiple of 64 and n_blocks = ceil(n_coarse / block_size) >= 2");
  if (!sinv || !lo_indptr || !up_indptr || nnz < 0 || (nnz > 0 && (!lo_indices || !lo_values || !up_indices || !up_values)))
    return fail(ctx, TLS_ERR_ARG, "null chain array");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = (cudaStream_t)stream;
  ctx->finalized = false;
  destroy_graphs(ctx);
  dfree(ctx->ctiles);
  ctx->h_blk.resize(ctx->nsub + 3);
  ctx->h_blk[ctx->nsub].tiles = nullptr;
  int64_t tiles = 0;
  std::vector<int64_t> tb(n_blocks);
  for (int i = 0; i < n_blocks; ++i) {
    const int ni = std::min(block_size, nc - i * block_size), nt = (ni + TT - 1) / TT;
    tb[i] = tiles;
    tiles += (int64_t)nt * (nt + 1) / 2;
  }
  TRY(dalloc(ctx, ctx->chain_tiles, tiles * TT * TT));
  for (int i = 0; i < n_blocks; ++i) {
    BlkDesc b{};
    b.n = std::min(block_size, nc - i * block_size);
    b.nt = (b.n + TT - 1) / TT;
    b.sym = 1;
    b.xoff = ctx->Xloc + (long long)i * block_size;
    b.tiles = ctx->chain_tiles + tb[i] * TT * TT;
    ctx->h_blk.push_back(b);
  }
  TRY(upload(ctx, ctx->d_blk, ctx->h_blk.data(), (int64_t)ctx->h_blk.size()));
  for (int i = 0; i < n_blocks; ++i) {
    const BlkDesc& b = ctx->h_blk[ctx->nsub + 3 + i];
    if (!sinv[i]) return fail(ctx, TLS_ERR_ARG, "null S_i^{-1} block");
    const int64_t nt = (int64_t)b.nt * (b.nt + 1) / 2;
    dim3 g((unsigned)std::min<int64_t>(nt, 8192), 1);
    launch_k(ctx, k_pack_tiles, g, NTHR, 0, s, ctx->d_blk, ctx->nsub + 3 + i,
             reinterpret_cast<const double*>(sinv[i]), (long long)b.n, 0LL);
    CKL();
  }
  TRY(dalloc(ctx, ctx->d_lo_ptr, (int64_t)nc + 1));
  TRY(dalloc(ctx, ctx->d_up_ptr, (int64_t)nc + 1));
  TRY(dalloc(ctx, ctx->d_lo_idx, nnz));
  TRY(dalloc(ctx, ctx->d_up_idx, nnz));
  TRY(dalloc(ctx, ctx->d_lo_val, nnz));
  TRY(dalloc(ctx, ctx->d_up_val, nnz));
  CK(cudaMemcpyAsync(ctx->d_lo_ptr, lo_indptr, sizeof(int) * ((size_t)nc + 1), cudaMemcpyDeviceToDevice, s));
  CK(cudaMemcpyAsync(ctx->d_up_ptr, up_indptr, sizeof(int) * ((size_t)nc + 1), cudaMemcpyDeviceToDevice, s));
  if (nnz > 0) {
    CK(cudaMemcpyAsync(ctx->d_lo_idx, lo_indices, sizeof(int) * (size_t)nnz, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(ctx->d_up_idx, up_indices, sizeof(int) * (size_t)nnz, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(ctx->d_lo_val, lo_values, sizeof(double) * (size_t)nnz, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(ctx->d_up_val, up_values, sizeof(double) * (size_t)nnz, cudaMemcpyDeviceToDevice, s));
  }
  // the structure the substitution relies on: row r of the lower part only reads columns of the
  // block before r's, row r of the upper part only columns of the block after it
  std::vector<int> hp((size_t)nc + 1), hi((size_t)std::max<int64_t>(nnz, 1));
  for (int pass = 0; pass < 2; ++pass) {
    CK(cudaMemcpyAsync(hp.data(), pass ? ctx->d_up_ptr : ctx->d_lo_ptr, sizeof(int) * ((size_t)nc + 1), cudaMemcpyDeviceToHost, s));
    if (nnz > 0)
      CK(cudaMemcpyAsync(hi.data(), pass ? ctx->d_up_idx : ctx->d_lo_idx, sizeof(int) * (size_t)nnz, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (hp[0] != 0 || hp[nc] != nnz) return fail(ctx, TLS_ERR_ARG, "chain CSR: indptr[0] != 0 or indptr[n] != nnz");
    for (int r = 0; r < nc; ++r) {
      if (hp[r + 1] < hp[r]) return fail(ctx, TLS_ERR_ARG, "chain CSR: indptr decreases at row " + std::to_string(r));
      const int b = r / block_size + (pass ? 1 : -1);
      const long long c0 = (long long)b * block_size, c1 = std::min<long long>(c0 + block_size, nc);
      for (int e = hp[r]; e < hp[r + 1]; ++e)
        if (b < 0 || b >= n_blocks || hi[e] < c0 || hi[e] >= c1)
          return fail(ctx, TLS_ERR_ARG, "chain CSR: entry (" + std::to_string(r) + ", " + std::to_string(hi[e]) +
                                            ") outside the neighbouring block");
    }
  }
  ctx->chain_nb = n_blocks;
  ctx->chain_bs = block_size;
  ctx->chain_nnz = nnz;
  return TLS_OK;
}

// Units and reduction lists for one block (see k_symv_tiles): units of ur tile-rows x UW
// tile-cols (ur <= UR); symmetric blocks only plan units touching the lower triangle.
static void plan_block(int blk, int nt, int sym, int ur, int& slot, std::vector<Unit>& units,
                       std::vector<OutTile>& outs, std::vector<int>& red) {
  const int np = (nt + ur - 1) / ur, nq = (nt + UW - 1) / UW;
  std::vector<int> uslot((size_t)np * nq, -1);
  for (int p = 0; p < np; ++p) {
    const int i0 = p * ur, ni = std::min(ur, nt - i0);
    for (int q = 0; q < nq; ++q) {
      const int j0 = q * UW, nj = std::min(UW, nt - j0);
      if (sym && j0 > i0 + ni - 1) break;  // entirely above the diagonal
      uslot[(size_t)p * nq + q] = slot;
      units.push_back(Unit{blk, i0, j0, slot, (short)ni, (short)nj, 0, 0});
      slot += SLOTS_PER_UNIT;
    }
  }
  for (int J = 0; J < nt; ++J) {
    OutTile ot{blk, J, (int)red.size(), 0};
    const int p = J / ur;
    for (int q = 0; q < nq; ++q)  // row partials of tile-row J
      if (uslot[(size_t)p * nq + q] >= 0) red.push_back(uslot[(size_t)p * nq + q] + (J - p * ur));
    if (sym) {  // column partials of tile-col J from units strictly below it
      const int q = J / UW;
      for (int pp = 0; pp < np; ++pp) {
        if (uslot[(size_t)pp * nq + q] < 0) continue;
        const int imax = std::min((pp + 1) * ur, nt) - 1;
        if (imax > J) red.push_back(uslot[(size_t)pp * nq + q] + UR + (J - q * UW));
      }
    }
    ot.end = (int)red.size();
    outs.push_back(ot);
  }
}

int32_t tls_precond_finalize(tls_ctx* ctx, int32_t one_level, int32_t combine) {
  TLS_RANGE("tls_precond_finalize");
  if (!ctx || !ctx->nsub) return ctx ? fail(ctx, TLS_ERR_STATE, "upload subdomains first") : TLS_ERR_ARG;
  if (one_level != TLS_ASM && one_level != TLS_RAS) return fail(ctx, TLS_ERR_ARG, "unknown one-level kind");
  if (combine < TLS_NONE || combine > TLS_DEFLATED) return fail(ctx, TLS_ERR_ARG, "unknown combination");
  for (int s = 0; s < ctx->nsub; ++s)
    if (!ctx->stored[s])
      return fail(ctx, TLS_ERR_STATE, "local operator of subdomain " + std::to_string(s + ctx->own_lo) + " missing");
  CK(cudaSetDevice(ctx->device));
  ctx->one_level = one_level;
  ctx->combine = ctx->ncoarse > 0 ? combine : TLS_NONE;
  const int nsub = ctx->nsub, n = ctx->n;
  // padded local layout
  // local position of local index l (band mode stores the local vector in its factor order)
  std::vector<int> posl(ctx->h_idx.size());
  for (int s = 0; s < nsub; ++s)
    for (int l = 0; l < ctx->h_n[s]; ++l)
      posl[ctx->h_off[s] + l] = ctx->local_kind >= 1 ? -1 : l;
  if (ctx->local_kind >= 1)
    for (int s = 0; s < nsub; ++s)
      for (int p = 0; p < ctx->h_n[s]; ++p) posl[ctx->h_off[s] + ctx->h_perm[ctx->h_off[s] + p]] = p;
  std::vector<int> gidx(ctx->Xloc, -1);
  for (int s = 0; s < nsub; ++s)
    for (int l = 0; l < ctx->h_n[s]; ++l)
      gidx[ctx->h_blk[s].xoff + posl[ctx->h_off[s] + l]] = ctx->h_idx[ctx->h_off[s] + l];
  if (ctx->local_kind == 2)  // LU input order: the pivoted rows (P^T r), output order stays perm
    for (int s = 0; s < nsub; ++s)
      for (int p = 0; p < ctx->h_n[s]; ++p)
        gidx[ctx->h_blk[s].xoff + p] = ctx->h_idx[ctx->h_off[s] + ctx->h_perm_in[ctx->h_off[s] + p]];
  TRY(upload(ctx, ctx->d_gidx, gidx.data(), ctx->Xloc));
  ctx->coarse_xoff = ctx->Xloc;
  ctx->X = ctx->Xloc + (ctx->ncoarse > 0 ? ctx->cpad : 0) + (ctx->cref ? 2 * ctx->cpad : 0);
  const bool part = !ctx->h_nofo.empty();
  const bool asm_ = one_level == TLS_ASM;
  ctx->Xrecv = 0;
  if (part && asm_)
    for (int c : ctx->rc_cnt) ctx->Xrecv += c;
  TRY(dalloc(ctx, ctx->xloc, ctx->X));
  TRY(dalloc(ctx, ctx->yloc, ctx->X + ctx->Xrecv));
  CK(cudaMemset(ctx->xloc, 0, sizeof(double) * ctx->X));
  CK(cudaMemset(ctx->yloc, 0, sizeof(double) * (ctx->X + ctx->Xrecv)));
  // work units + reduction lists
  std::vector<Unit> units;
  std::vector<OutTile> outs;
  std::vector<int> red;
  int slot = 0;
  ctx->algo_local = 0.0;
  for (int s = 0; s < nsub && ctx->local_kind == 0; ++s) {
    plan_block(s, ctx->h_blk[s].nt, ctx->sym, UR, slot, units, outs, red);
    const double ns = ctx->h_n[s];
    ctx->algo_local += ctx->sym ? 8.0 * ns * (ns + 1) / 2 + 8.0 * ns : 8.0 * ns * ns + 8.0 * ns;
  }
  if (ctx->local_kind >= 1) {  // sweeps over the stored factors (band_bytes counts the reads) + x, y
    ctx->algo_local = ctx->band_bytes;
    for (int s = 0; s < nsub; ++s) ctx->algo_local += 16.0 * ctx->h_n[s];
  }
  ctx->nu_local = (int)units.size();
  ctx->no_local = (int)outs.size();
  ctx->nu_coarse = ctx->no_coarse = 0;
  ctx->algo_coarse = 0.0;
  ctx->chain_u0.clear(); ctx->chain_nu.clear(); ctx->chain_o0.clear(); ctx->chain_no.clear();
  if (ctx->ncoarse > 0 && ctx->chain_nb == 0 && !ctx->h_blk[nsub].tiles)
    return fail(ctx, TLS_ERR_STATE, "coarse basis uploaded without a coarse operator (tls_coarse_chain missing)");
  if (ctx->ncoarse > 0 && ctx->chain_nb > 0) {
    // block-tridiagonal coarse solve: one tile plan per inverted Schur block, launched one after
    // the other (every rank runs the whole substitution: it does not partition by rows)
    double bytes = 0.0;
    int chain_ur = 2;  // tile-rows per work unit (TLS_CHAIN_UR: tuning override, 1..8)
    if (const char* e = getenv("TLS_CHAIN_UR")) chain_ur = std::max(1, std::min(UR, atoi(e)));
    for (int i = 0; i < ctx->chain_nb; ++i) {
      const BlkDesc& b = ctx->h_blk[nsub + 3 + i];
      ctx->chain_u0.push_back((int)units.size());
      ctx->chain_o0.push_back((int)outs.size());
      plan_block(nsub + 3 + i, b.nt, 1, chain_ur, slot, units, outs, red);
      ctx->chain_nu.push_back((int)units.size() - ctx->chain_u0.back());
      ctx->chain_no.push_back((int)outs.size() - ctx->chain_o0.back());
      const double ni = b.n;
      bytes += (i + 1 < ctx->chain_nb ? 2.0 : 1.0) * (8.0 * ni * (ni + 1) / 2 + 16.0 * ni);
    }
    ctx->algo_coarse = bytes + 2.0 * (12.0 * (double)ctx->chain_nnz + 4.0 * ctx->ncoarse);
    ctx->nu_coarse = (int)units.size() - ctx->nu_local;
    ctx->no_coarse = (int)outs.size() - ctx->no_local;
    ctx->nu_ref1 = ctx->no_ref1 = ctx->nu_ref2 = ctx->no_ref2 = 0;
  } else if (ctx->ncoarse > 0) {
    // the coarse operator is ONE block: thinner units (2 tile-rows) to fill the machine
    plan_block(nsub, ctx->h_blk[nsub].nt, ctx->sym, 2, slot, units, outs, red);
    const double nc = ctx->ncoarse;
    ctx->algo_coarse = ctx->sym ? 8.0 * nc * (nc + 1) / 2 + 8.0 * nc : 8.0 * nc * nc + 8.0 * nc;
    if (part) {
      // sharded: only the output tiles of this rank's coarse rows (its subdomains' columns, the
      // only entries of A0^{-1} c its prolongation reads) and the units that feed them; each
      // kept tile reduces the same slots in the same order as on one GPU
      const long long c0 = ctx->h_cstart[0], c1 = ctx->h_cstart[nsub - 1] + ctx->h_k[nsub - 1];
      std::vector<OutTile> kept_outs;
      std::vector<int> kept_red;
      std::vector<char> used((size_t)slot / SLOTS_PER_UNIT + 1, 0);
      for (size_t o = ctx->no_local; o < outs.size(); ++o) {
        const OutTile& ot = outs[o];
        if (c1 <= c0 || (long long)ot.J * TT >= c1 || (long long)(ot.J + 1) * TT <= c0) continue;
        OutTile nt{ot.blk, ot.J, (int)(red.size() + kept_red.size()), 0};
        for (int e = ot.beg; e < ot.end; ++e) {
          kept_red.push_back(red[e]);
          used[red[e] / SLOTS_PER_UNIT] = 1;
        }
        nt.end = (int)(red.size() + kept_red.size());
        kept_outs.push_back(nt);
      }
      // the kept reduction lists go behind all existing ones (their beg/end already say so)
      outs.resize(ctx->no_local);
      outs.insert(outs.end(), kept_outs.begin(), kept_outs.end());
      red.insert(red.end(), kept_red.begin(), kept_red.end());
      std::vector<Unit> ku(units.begin(), units.begin() + ctx->nu_local);
      double tiles_read = 0.0;
      for (size_t u = ctx->nu_local; u < units.size(); ++u) {
        const Unit& un = units[u];
        if (!used[un.slot / SLOTS_PER_UNIT]) continue;
        ku.push_back(un);
        for (int I = un.i0; I < un.i0 + un.ni; ++I)
          for (int J = un.j0; J < un.j0 + un.nj; ++J)
            if (!ctx->sym || J <= I) tiles_read += 1.0;
      }
      units.swap(ku);
      ctx->algo_coarse = tiles_read * TT * TT * 8.0 + 16.0 * (double)(c1 - c0);
    }
    ctx->nu_coarse = (int)units.size() - ctx->nu_local;
    ctx->no_coarse = (int)outs.size() - ctx->no_local;
    ctx->nu_ref1 = ctx->no_ref1 = ctx->nu_ref2 = ctx->no_ref2 = 0;
    if (ctx->cref) {  // A0 (general tiles) then X again, each with its own units / slots
      const int nt = ctx->h_blk[nsub].nt;
      size_t u0 = units.size(), o0 = outs.size();
      plan_block(nsub + 1, nt, 0, 2, slot, units, outs, red);
      ctx->nu_ref1 = (int)(units.size() - u0);
      ctx->no_ref1 = (int)(outs.size() - o0);
      u0 = units.size(), o0 = outs.size();
      plan_block(nsub + 2, nt, ctx->sym, 2, slot, units, outs, red);
      ctx->nu_ref2 = (int)(units.size() - u0);
      ctx->no_ref2 = (int)(outs.size() - o0);
      const double nc = ctx->ncoarse;
      ctx->algo_coarse = 2.0 * ctx->algo_coarse + 8.0 * nc * nc;  // X twice + the A0 tiles
    }
  }
  TRY(upload(ctx, ctx->d_units, units.data(), (int64_t)units.size()));
  TRY(upload(ctx, ctx->d_outs, outs.data(), (int64_t)outs.size()));
  TRY(upload(ctx, ctx->d_red, red.data(), (int64_t)red.size()));
  ctx->nslots = slot;
  TRY(dalloc(ctx, ctx->slots, (int64_t)slot * TT));
  // prolongation pull map: contributions to node g in ascending subdomain order (np.add.at)
  std::vector<int> cnt(n + 1, 0);
  std::vector<int> pos;
  if (!part) {
    for (int s = 0; s < nsub; ++s) {
      const int lim = one_level == TLS_RAS ? ctx->h_nint[s] : ctx->h_n[s];
      for (int l = 0; l < lim; ++l) cnt[ctx->h_idx[ctx->h_off[s] + l] + 1]++;
    }
    for (int g = 0; g < n; ++g) cnt[g + 1] += cnt[g];
    pos.resize(cnt[n]);
    std::vector<int> fill(cnt.begin(), cnt.end() - 1);
    for (int s = 0; s < nsub; ++s) {
      const int lim = one_level == TLS_RAS ? ctx->h_nint[s] : ctx->h_n[s];
      for (int l = 0; l < lim; ++l) {
        const int g = ctx->h_idx[ctx->h_off[s] + l];
        pos[fill[g]++] = (int)(ctx->h_blk[s].xoff + posl[ctx->h_off[s] + l]);
      }
    }
  } else {
    // owned rows only; contributions of other ranks' subdomains arrive in the yloc tail (the
    // reverse halo) and are merged in ascending subdomain order; contributions of this rank's
    // subdomains to other ranks' rows are sent to their owners in (subdomain, local index) order
    struct Ent { int row, sub; long long pos; };
    std::vector<Ent> ent;
    const int nr = (int)ctx->row_starts.size() - 1;
    std::vector<std::vector<int>> sendpos(nr);
    for (int s = 0; s < nsub; ++s) {
      const int lim = asm_ ? ctx->h_n[s] : ctx->h_nint[s];
      for (int l = 0; l < lim; ++l) {
        const int g = ctx->h_idx[ctx->h_off[s] + l];
        const long long p = ctx->h_blk[s].xoff + posl[ctx->h_off[s] + l];
        if (g >= ctx->r0 && g < ctx->r1) {
          ent.push_back(Ent{g, ctx->own_lo + s, p});
        } else {
          const int q = (int)(std::upper_bound(ctx->row_starts.begin(), ctx->row_starts.end(), g) -
                              ctx->row_starts.begin()) - 1;
          sendpos[q].push_back((int)p);
        }
      }
    }
    if (asm_) {
      long long k = 0;
      for (size_t b = 0; b < ctx->rc_peer.size(); ++b)
        for (int e = 0; e < ctx->rc_cnt[b]; ++e, ++k) {
          const int g = ctx->rc_row[k];
          if (g < ctx->r0 || g >= ctx->r1) return fail(ctx, TLS_ERR_ARG, "remote contribution to a row not owned");
          ent.push_back(Ent{g, ctx->rc_sub[k], ctx->X + k});
        }
    }
    std::stable_sort(ent.begin(), ent.end(),
                     [](const Ent& a, const Ent& b) { return a.row != b.row ? a.row < b.row : a.sub < b.sub; });
    for (const Ent& e : ent) cnt[e.row + 1]++;
    for (int g = 0; g < n; ++g) cnt[g + 1] += cnt[g];
    pos.resize(ent.size());
    for (size_t i = 0; i < ent.size(); ++i) pos[i] = (int)ent[i].pos;
    // reverse-halo plan
    XPlan& x = ctx->rev;
    x.peers.clear(); x.scnt.clear(); x.rcnt.clear(); x.soff.clear(); x.roff.clear();
    std::vector<int> sidx, ridx;
    for (int q = 0; q < nr; ++q) {
      long long rc = 0;
      for (size_t b = 0; b < ctx->rc_peer.size(); ++b)
        if (asm_ && ctx->rc_peer[b] == q) rc = ctx->rc_cnt[b];
      if (sendpos[q].empty() && rc == 0) continue;
      x.peers.push_back(q);
      x.soff.push_back((long long)sidx.size());
      x.scnt.push_back((int)sendpos[q].size());
      sidx.insert(sidx.end(), sendpos[q].begin(), sendpos[q].end());
      x.roff.push_back((long long)ridx.size());
      x.rcnt.push_back((int)rc);
      long long k0 = 0;
      for (size_t b = 0; b < ctx->rc_peer.size() && ctx->rc_peer[b] != q; ++b) k0 += ctx->rc_cnt[b];
      for (long long e = 0; e < rc; ++e) ridx.push_back((int)(ctx->X + k0 + e));
    }
    if (!asm_ && !sidx.empty()) return fail(ctx, TLS_ERR_STATE, "RAS interior row owned by another rank");
    x.stot = (long long)sidx.size();
    x.rtot = (long long)ridx.size();
    TRY(upload(ctx, x.d_sidx, sidx.data(), x.stot));
    TRY(upload(ctx, x.d_ridx, ridx.data(), x.rtot));
    TRY(dalloc(ctx, x.sbuf, x.stot));
    TRY(dalloc(ctx, x.rbuf, x.rtot));
  }
  TRY(upload(ctx, ctx->d_pull_ptr, cnt.data(), n + 1));
  TRY(upload(ctx, ctx->d_pull_pos, pos.data(), (int64_t)pos.size()));
  // coarse prolongation rows: node g in the interior of s at position p -> Z_s[p, :]
  std::vector<long long> zrow(n, -1);
  std::vector<int> zk(n, 0), zc(n, 0), zst(n, 0);
  if (ctx->ncoarse > 0) {
    for (int s = 0; s < nsub; ++s) {
      if (ctx->h_k[s] == 0) continue;
      for (int p = 0; p < ctx->h_nint[s]; ++p) {
        const int g = ctx->h_idx[ctx->h_off[s] + p];
        zrow[g] = ctx->h_zoff[s] + p;  // column-major block: element (p, t) at + t * n_int
        zst[g] = ctx->h_nint[s];
        zk[g] = ctx->h_k[s];
        zc[g] = ctx->h_cstart[s];
      }
    }
  } else {
    TRY(dalloc(ctx, ctx->d_Z, 1));
  }
  TRY(upload(ctx, ctx->d_zrow, zrow.data(), n));
  TRY(upload(ctx, ctx->d_zk, zk.data(), n));
  TRY(upload(ctx, ctx->d_zst, zst.data(), n));
  TRY(upload(ctx, ctx->d_zc, zc.data(), n));
  if (ctx->ncoarse == 0) {
    std::vector<int> zero(nsub, 0);
    std::vector<long long> zero64(nsub, 0);
    TRY(upload(ctx, ctx->d_kcnt, zero.data(), nsub));
    TRY(upload(ctx, ctx->d_cstart, zero.data(), nsub));
    TRY(upload(ctx, ctx->d_zoff, zero64.data(), nsub));
  }
  destroy_graphs(ctx);
  CK(cudaDeviceSynchronize());
  ctx->finalized = true;
  return TLS_OK;
}

static int need_final(tls_ctx* ctx) {
  if (!ctx) return TLS_ERR_ARG;
  if (!ctx->finalized) return fail(ctx, TLS_ERR_STATE, "preconditioner not finalized");
  return TLS_OK;
}

int32_t tls_precond_apply(tls_ctx* ctx, const double* r, double* z, void* stream) {
  TLS_RANGE("tls_precond_apply");
  TRY(need_final(ctx));
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = (cudaStream_t)stream;
  double* ri;
  TRY(api_in(ctx, s, r, &ri));
  double* zi = api_out_buf(ctx, z);
  TRY(enq_apply(ctx, s, ri, zi, false, nullptr, true));
  return api_out(ctx, s, zi, z);
}

int32_t tls_apply_one_level(tls_ctx* ctx, const double* r, double* z, void* stream) {
  TLS_RANGE("tls_apply_one_level");
  TRY(need_final(ctx));
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = (cudaStream_t)stream;
  double* ri;
  TRY(api_in(ctx, s, r, &ri));
  double* zi = api_out_buf(ctx, z);
  TRY(enq_local(ctx, s, ri, nullptr));
  TRY(enq_rev(ctx, s, nullptr));
  TRY((enq_prolong<0, 0>(ctx, s, nullptr, nullptr, nullptr, zi, nullptr)));
  return api_out(ctx, s, zi, z);
}

int32_t tls_coarse_apply(tls_ctx* ctx, const double* r, double* z, void* stream) {
  TLS_RANGE("tls_coarse_apply");
  TRY(need_final(ctx));
  if (ctx->ncoarse == 0) return fail(ctx, TLS_ERR_STATE, "no coarse space");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = (cudaStream_t)stream;
  double* ri;
  TRY(api_in(ctx, s, r, &ri));
  double* zi = api_out_buf(ctx, z);
  TRY(enq_restrict_all(ctx, s, ri, nullptr));
  TRY(enq_solve(ctx, s, L_COARSE, nullptr));
  TRY((enq_prolong<2, 0>(ctx, s, nullptr, nullptr, nullptr, zi, nullptr)));
  return api_out(ctx, s, zi, z);
}

// y_i = A_ii^{-1} R_i r for the listed (owned, global ids) subdomains, each in the reference's
// local order (interior, then the layers; src/partition.py:295-298), concatenated into out --
// the local_solves closures of src/precond.py:117-118 / src/subdomain.py:72-95, run by the same
// kernels as the apply (band sweeps or inverse tiles) and read back from yloc
int32_t tls_local_solve(tls_ctx* ctx, const double* r, int32_t count, const int32_t* subdomains, double* out,
                        void* stream) {
  TRY(need_final(ctx));
  if (count <= 0 || !subdomains || !out) return fail(ctx, TLS_ERR_ARG, "empty subdomain list");
  std::vector<int> pos;
  for (int i = 0; i < count; ++i) {
    const int sl = subdomains[i] - ctx->own_lo;
    if (sl < 0 || sl >= ctx->nsub) return fail(ctx, TLS_ERR_ARG, "subdomain " + std::to_string(subdomains[i]) + " not owned by this handle");
    const int ns = ctx->h_n[sl];
    std::vector<int> posl(ns);
    for (int l = 0; l < ns; ++l) posl[l] = l;
    if (ctx->local_kind >= 1)
      for (int p = 0; p < ns; ++p) posl[ctx->h_perm[ctx->h_off[sl] + p]] = p;
    for (int l = 0; l < ns; ++l) pos.push_back((int)(ctx->h_blk[sl].xoff + posl[l]));
  }
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = (cudaStream_t)stream;
  int* d_pos = nullptr;
  CK(cudaMallocAsync((void**)&d_pos, sizeof(int) * pos.size(), s));
  CK(cudaMemcpyAsync(d_pos, pos.data(), sizeof(int) * pos.size(), cudaMemcpyHostToDevice, s));
  double* ri;
  TRY(api_in(ctx, s, r, &ri));
  TRY(enq_local(ctx, s, ri, nullptr));
  launch_k(ctx, k_xpack, grid_for((long long)pos.size(), NTHR), NTHR, 0, s, (long long)pos.size(), (const int*)d_pos,
           (const double*)ctx->yloc, out, (const int*)nullptr);
  CKL();
  CK(cudaFreeAsync(d_pos, s));
  CK(cudaStreamSynchronize(s));  // pos (host) must outlive the async copy
  return TLS_OK;
}

// CoarseSpace.restrict / solve_coarse / prolong (src/coarse.py:40-49) on the device, with the
// kernels of the apply: c = Z^T r (n_C, summed over the ranks), y = A0^{-1} c (one GPU), z = Z y
int32_t tls_coarse_restrict(tls_ctx* ctx, const double* r, double* c, void* stream) {
  TRY(need_final(ctx));
  if (ctx->ncoarse == 0) return fail(ctx, TLS_ERR_STATE, "no coarse space");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = (cudaStream_t)stream;
  double* ri;
  TRY(api_in(ctx, s, r, &ri));
  TRY(enq_restrict_all(ctx, s, ri, nullptr));
  CK(cudaMemcpyAsync(c, ctx->xloc + ctx->coarse_xoff, sizeof(double) * ctx->ncoarse, cudaMemcpyDeviceToDevice, s));
  return TLS_OK;
}

int32_t tls_coarse_solve(tls_ctx* ctx, const double* c, double* y, void* stream) {
  TRY(need_final(ctx));
  if (ctx->ncoarse == 0) return fail(ctx, TLS_ERR_STATE, "no coarse space");
  if (sharded(ctx)) return fail(ctx, TLS_ERR_STATE, "tls_coarse_solve: a sharded handle holds only its rows of A0^{-1}");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = (cudaStream_t)stream;
  CK(cudaMemcpyAsync(ctx->xloc + ctx->coarse_xoff, c, sizeof(double) * ctx->ncoarse, cudaMemcpyDeviceToDevice, s));
  TRY(enq_solve(ctx, s, L_COARSE, nullptr));
  CK(cudaMemcpyAsync(y, ctx->yloc + ctx->coarse_xoff, sizeof(double) * ctx->ncoarse, cudaMemcpyDeviceToDevice, s));
  return TLS_OK;
}

// the basis blocks as uploaded (per owned subdomain k_s x n_interior[s] row-major, subdomain
// order) copied to HOST memory: behind CoarseSpace.basis (src/coarse.py:23-38), read on demand
int32_t tls_coarse_basis_fetch(tls_ctx* ctx, double* out, int64_t count) {
  if (!ctx || !out) return ctx ? fail(ctx, TLS_ERR_ARG, "null output") : TLS_ERR_ARG;
  if (ctx->ncoarse == 0 || !ctx->d_Z) return fail(ctx, TLS_ERR_STATE, "no coarse space");
  long long total = 0;
  for (int i = 0; i < ctx->nsub; ++i) total += (long long)ctx->h_nint[i] * ctx->h_k[i];
  if (count != total) return fail(ctx, TLS_ERR_ARG, "basis size mismatch: the handle holds " + std::to_string(total) + " doubles");
  CK(cudaSetDevice(ctx->device));
  CK(cudaDeviceSynchronize());
  if (total) CK(cudaMemcpy(out, ctx->d_Z, sizeof(double) * (size_t)total, cudaMemcpyDeviceToHost));
  return TLS_OK;
}

int32_t tls_coarse_prolong(tls_ctx* ctx, const double* y, double* z, void* stream) {
  TRY(need_final(ctx));
  if (ctx->ncoarse == 0) return fail(ctx, TLS_ERR_STATE, "no coarse space");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = (cudaStream_t)stream;
  CK(cudaMemcpyAsync(ctx->yloc + ctx->coarse_xoff, y, sizeof(double) * ctx->ncoarse, cudaMemcpyDeviceToDevice, s));
  double* zi = api_out_buf(ctx, z);
  TRY((enq_prolong<2, 0>(ctx, s, nullptr, nullptr, nullptr, zi, nullptr)));
  return api_out(ctx, s, zi, z);
}

// sharded: global coarse column ranges of every rank (nranks + 1 starts; rank q's subdomains own
// columns [col_starts[q], col_starts[q+1]) -- contiguous because slabs are contiguous)
int32_t tls_set_coarse_layout(tls_ctx* ctx, int32_t nranks, const int64_t* col_starts) {
  if (!ctx || nranks <= 0 || !col_starts) return ctx ? fail(ctx, TLS_ERR_ARG, "bad coarse layout") : TLS_ERR_ARG;
  if (!ctx->comm || ctx->comm->nranks != nranks) return fail(ctx, TLS_ERR_STATE, "initialise the communicator first");
  if (col_starts[0] != 0 || col_starts[nranks] != ctx->ncoarse)
    return fail(ctx, TLS_ERR_ARG, "coarse layout does not cover the n_coarse columns");
  CK(cudaSetDevice(ctx->device));
  ctx->ccol.assign(col_starts, col_starts + nranks + 1);
  ctx->cmax = 0;
  for (int q = 0; q < nranks; ++q) {
    if (ctx->ccol[q + 1] < ctx->ccol[q]) return fail(ctx, TLS_ERR_ARG, "coarse layout not ascending");
    ctx->cmax = std::max(ctx->cmax, ctx->ccol[q + 1] - ctx->ccol[q]);
  }
  if (ctx->nsub > 0 && ctx->ncoarse > 0 &&
      (ctx->h_cstart[0] != ctx->ccol[ctx->comm->rank] ||
       ctx->h_cstart[ctx->nsub - 1] + ctx->h_k[ctx->nsub - 1] != ctx->ccol[ctx->comm->rank + 1]))
    return fail(ctx, TLS_ERR_ARG, "coarse layout disagrees with this rank's subdomain columns");
  TRY(upload(ctx, ctx->d_ccol, (const long long*)ctx->ccol.data(), nranks + 1));
  TRY(dalloc(ctx, ctx->cg_send, std::max<long long>(1, ctx->cmax)));
  TRY(dalloc(ctx, ctx->cg_recv, std::max<long long>(1, ctx->cmax * nranks)));
  destroy_graphs(ctx);
  return TLS_OK;
}

// K12b: Galerkin blocks of A0 = Z^T (A Z) from the per-subdomain Z_j and W_s = A_ii[:, :n_int] Z_s
int32_t tls_galerkin_assemble(const int32_t* plan_sj, const int64_t* plan_off, int64_t nplan, const int64_t* zptr,
                              const int64_t* wptr, const int32_t* kcnt, const int64_t* cstart, int32_t nsub,
                              const int64_t* rows, const int64_t* grp, int64_t nrows, double* A0, int64_t nC,
                              void* stream) {
  TLS_RANGE("tls_galerkin_assemble");
  if (!plan_sj || !plan_off || nplan <= 0 || !zptr || !wptr || !kcnt || !cstart || !rows || !grp || !A0)
    return TLS_ERR_ARG;
  for (int s = 0; s < nsub; ++s)
    if (kcnt[s] < 0 || kcnt[s] > 64) return TLS_ERR_ARG;
  std::vector<GalPlan> plan(nplan);
  for (int64_t p = 0; p < nplan; ++p) {
    plan[p] = GalPlan{plan_sj[2 * p], plan_sj[2 * p + 1], plan_off[p], plan_off[p + 1]};
    if (plan[p].s < 0 || plan[p].s >= nsub || plan[p].j < 0 || plan[p].j >= nsub || plan[p].o0 < 0 ||
        plan[p].o1 > nrows || plan[p].o1 < plan[p].o0)
      return TLS_ERR_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  GalPlan* d_plan = nullptr;
  long long *d_z = nullptr, *d_w = nullptr, *d_c = nullptr, *d_rows = nullptr, *d_grp = nullptr;
  int* d_k = nullptr;
  if (cudaMallocAsync((void**)&d_plan, sizeof(GalPlan) * nplan, s) != cudaSuccess ||
      cudaMallocAsync((void**)&d_z, sizeof(long long) * nsub, s) != cudaSuccess ||
      cudaMallocAsync((void**)&d_w, sizeof(long long) * nsub, s) != cudaSuccess ||
      cudaMallocAsync((void**)&d_c, sizeof(long long) * (nsub + 1), s) != cudaSuccess ||
      cudaMallocAsync((void**)&d_k, sizeof(int) * nsub, s) != cudaSuccess ||
      cudaMallocAsync((void**)&d_rows, sizeof(long long) * std::max<int64_t>(1, nrows), s) != cudaSuccess ||
      cudaMallocAsync((void**)&d_grp, sizeof(long long) * std::max<int64_t>(1, nrows), s) != cudaSuccess)
    return TLS_ERR_OOM;
  cudaMemcpyAsync(d_plan, plan.data(), sizeof(GalPlan) * nplan, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(d_z, zptr, sizeof(long long) * nsub, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(d_w, wptr, sizeof(long long) * nsub, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(d_c, cstart, sizeof(long long) * (nsub + 1), cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(d_k, kcnt, sizeof(int) * nsub, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(d_rows, rows, sizeof(long long) * nrows, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(d_grp, grp, sizeof(long long) * nrows, cudaMemcpyHostToDevice, s);
  for (int64_t p0 = 0; p0 < nplan; p0 += 1 << 30) {
    const int np = (int)std::min<int64_t>(nplan - p0, 1 << 30);
    launch_k(nullptr, k_galerkin_blocks, np, 256, 0, s, (const GalPlan*)(d_plan + p0), (const long long*)d_z,
             (const long long*)d_w, (const int*)d_k, (const long long*)d_c, (const long long*)d_rows,
             (const long long*)d_grp, A0, (long long)nC);
  }
  if (cudaGetLastError() != cudaSuccess) return TLS_ERR_CUDA;
  cudaFreeAsync(d_plan, s); cudaFreeAsync(d_z, s); cudaFreeAsync(d_w, s); cudaFreeAsync(d_c, s);
  cudaFreeAsync(d_k, s); cudaFreeAsync(d_rows, s); cudaFreeAsync(d_grp, s);
  return cudaStreamSynchronize(s) == cudaSuccess ? TLS_OK : TLS_ERR_CUDA;  // host arrays
}

// K9b: banded LU with partial pivoting of a batch, in place, LAPACK format
int32_t tls_band_lu(double* ap, int64_t ld, int32_t count, const int32_t* lreach, const int32_t* ureach, int32_t nbk,
                    int32_t* piv, int32_t* info, void* stream) {
  TLS_RANGE("tls_band_lu");
  if (!ap || !lreach || !ureach || !piv || !info || count <= 0 || nbk <= 0 || ld != 64LL * nbk) return TLS_ERR_ARG;
  for (int J = 0; J < nbk; ++J)
    if (lreach[J] < 64 * (J + 1) || lreach[J] > ld || ureach[J] < 64 * (J + 1) || ureach[J] > ld ||
        lreach[J] % 64 || ureach[J] % 64)
      return TLS_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const size_t smem = sizeof(double) * 3 * 64 * CP;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return TLS_ERR_CUDA;
  if (raise_smem(dev, (const void*)k_band_lu, smem) != cudaSuccess) return TLS_ERR_CUDA;
  int* d_r = nullptr;
  if (cudaMallocAsync((void**)&d_r, sizeof(int) * 2 * nbk, s) != cudaSuccess) return TLS_ERR_OOM;
  if (cudaMemcpyAsync(d_r, lreach, sizeof(int) * nbk, cudaMemcpyHostToDevice, s) != cudaSuccess ||
      cudaMemcpyAsync(d_r + nbk, ureach, sizeof(int) * nbk, cudaMemcpyHostToDevice, s) != cudaSuccess)
    return TLS_ERR_CUDA;
  launch_k(nullptr, k_band_lu, count, 256, smem, s, ap, (long long)ld, (const int*)d_r, (const int*)(d_r + nbk),
           (int)nbk, piv, info);
  if (cudaGetLastError() != cudaSuccess) return TLS_ERR_CUDA;
  cudaFreeAsync(d_r, s);
  return cudaStreamSynchronize(s) == cudaSuccess ? TLS_OK : TLS_ERR_CUDA;  // host reach arrays
}

// K10: X <- (L L^T)^{-1} X for a batch of band Cholesky factors, many right-hand sides (DMMA)
int32_t tls_band_solve_multi(const double* L, int64_t ld, int32_t count, const double* dinv, const int32_t* kc,
                             int32_t nb, double* X, int64_t nrhs, void* stream) {
  TLS_RANGE("tls_band_solve_multi");
  if (!L || !dinv || !kc || !X || count <= 0 || nb <= 0 || ld != 64LL * nb || nrhs <= 0) return TLS_ERR_ARG;
  for (int64_t i = 0; i < (int64_t)count * nb; ++i)
    if (kc[i] < 0 || kc[i] > i % nb) return TLS_ERR_ARG;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return TLS_ERR_CUDA;
  cudaStream_t s = (cudaStream_t)stream;
  const size_t smem = sizeof(double) * 2 * 64 * CP;
  if (raise_smem(dev, (const void*)k_band_trsm_multi, smem) != cudaSuccess) return TLS_ERR_CUDA;
  int* d_kc = nullptr;
  if (cudaMallocAsync((void**)&d_kc, sizeof(int) * (size_t)count * nb, s) != cudaSuccess) return TLS_ERR_OOM;
  if (cudaMemcpyAsync(d_kc, kc, sizeof(int) * (size_t)count * nb, cudaMemcpyHostToDevice, s) != cudaSuccess)
    return TLS_ERR_CUDA;
  dim3 grid((unsigned)((nrhs + 63) / 64), (unsigned)count);
  launch_k(nullptr, k_band_trsm_multi, grid, 256, smem, s, L, (long long)ld, dinv, (const int*)d_kc, (int)nb, X,
           (long long)nrhs);
  if (cudaGetLastError() != cudaSuccess) return TLS_ERR_CUDA;
  cudaFreeAsync(d_kc, s);
  return cudaStreamSynchronize(s) == cudaSuccess ? TLS_OK : TLS_ERR_CUDA;  // kc (host) lifetime
}

// K12a: pivoted-QR pivot magnitudes of every subdomain's coarse block (rank filter)
int32_t tls_rank_filter_pivots(double* W, const int64_t* woff, const int32_t* nrows, const int32_t* ncols,
                               int32_t count, double* rdiag, int32_t* perm, void* stream) {
  TLS_RANGE("tls_rank_filter_pivots");
  if (!W || !woff || !nrows || !ncols || !rdiag || !perm || count <= 0) return TLS_ERR_ARG;
  std::vector<long long> roff(count + 1, 0);
  for (int s = 0; s < count; ++s) {
    if (ncols[s] < 0 || ncols[s] > 64 || nrows[s] < 0) return TLS_ERR_ARG;
    roff[s + 1] = roff[s] + ncols[s];
  }
  cudaStream_t st = (cudaStream_t)stream;
  long long* d_woff = nullptr;
  long long* d_roff = nullptr;
  int *d_n = nullptr, *d_k = nullptr;
  if (cudaMallocAsync((void**)&d_woff, sizeof(long long) * count, st) != cudaSuccess ||
      cudaMallocAsync((void**)&d_roff, sizeof(long long) * (count + 1), st) != cudaSuccess ||
      cudaMallocAsync((void**)&d_n, sizeof(int) * count, st) != cudaSuccess ||
      cudaMallocAsync((void**)&d_k, sizeof(int) * count, st) != cudaSuccess)
    return TLS_ERR_OOM;
  cudaMemcpyAsync(d_woff, woff, sizeof(long long) * count, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(d_roff, roff.data(), sizeof(long long) * (count + 1), cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(d_n, nrows, sizeof(int) * count, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(d_k, ncols, sizeof(int) * count, cudaMemcpyHostToDevice, st);
  double* d_rd = nullptr;
  int* d_pm = nullptr;
  if (cudaMallocAsync((void**)&d_rd, sizeof(double) * std::max<long long>(1, roff[count]), st) != cudaSuccess ||
      cudaMallocAsync((void**)&d_pm, sizeof(int) * std::max<long long>(1, roff[count]), st) != cudaSuccess)
    return TLS_ERR_OOM;
  launch_k(nullptr, k_pivoted_qr, count, 256, 0, st, W, (const long long*)d_woff, (const int*)d_n, (const int*)d_k,
           (const long long*)d_roff, d_rd, d_pm);
  if (cudaGetLastError() != cudaSuccess) return TLS_ERR_CUDA;
  cudaMemcpyAsync(rdiag, d_rd, sizeof(double) * roff[count], cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(perm, d_pm, sizeof(int) * roff[count], cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(d_woff, st);
  cudaFreeAsync(d_roff, st);
  cudaFreeAsync(d_n, st);
  cudaFreeAsync(d_k, st);
  cudaFreeAsync(d_rd, st);
  cudaFreeAsync(d_pm, st);
  return cudaStreamSynchronize(st) == cudaSuccess ? TLS_OK : TLS_ERR_CUDA;
}

// batched symmetric eigensolver (k_syevj_batched) for the setup's Rayleigh-Ritz matrices
int32_t tls_syevj_batched(const double* T, int64_t batch, int32_t p, double* w, double* V, void* stream) {
  TLS_RANGE("tls_syevj_batched");
  if (!T || !w || !V || batch <= 0 || p <= 0 || p > EJ_MAX) return TLS_ERR_ARG;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return TLS_ERR_CUDA;
  const size_t smem = sizeof(double) * 2 * EJ_MAX * EJ_LD;
  if (raise_smem(dev, (const void*)k_syevj_batched, smem) != cudaSuccess) return TLS_ERR_CUDA;
  for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
    const int nb = (int)std::min<int64_t>(65535, batch - b0);
    launch_k(nullptr, k_syevj_batched, nb, 256, smem, (cudaStream_t)stream, T + b0 * p * p, (int)p, w + b0 * p,
             V + b0 * p * p, 30);
  }
  return cudaGetLastError() == cudaSuccess ? TLS_OK : TLS_ERR_CUDA;
}

// batched one-sided Jacobi SVD (k_svdj_batched) for the SVD coarse modes (src/spectral.py:135-154)
int32_t tls_svdj_batched(double* X, int64_t batch, int32_t m, int32_t n, double* sig, int32_t* info, void* stream) {
  TLS_RANGE("tls_svdj_batched");
  if (!X || !sig || !info || batch <= 0 || m <= 0 || n <= 0) return TLS_ERR_ARG;
  // |cos(x_i, x_j)| <= tol ends a pair: above the rounding noise of an m-term dot product
  const double tol = std::max(1.0e-14, 2.220446049250313e-16 * sqrt((double)m));
  for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
    const int nb = (int)std::min<int64_t>(65535, batch - b0);
    launch_k(nullptr, k_svdj_batched, nb, SVJ_THREADS, 0, (cudaStream_t)stream, X + b0 * m * n, (int)m, (int)n,
             sig + b0 * n, info + b0, tol, 60);
  }
  return cudaGetLastError() == cudaSuccess ? TLS_OK : TLS_ERR_CUDA;
}

// ---- decomposition on the device (tls_graph.cuh; src/sparsemat.py:180-195, src/partition.py:278-334)
int32_t tls_graph_build(tls_ctx* ctx, int64_t* nedges) {
  TLS_RANGE("tls_graph_build");
  if (!ctx || !ctx->rowptr) return ctx ? fail(ctx, TLS_ERR_STATE, "upload the matrix first") : TLS_ERR_ARG;
  if (!ctx->h_nofo.empty()) return fail(ctx, TLS_ERR_STATE, "tls_graph_build needs the caller's row numbering");
  CK(cudaSetDevice(ctx->device));
  dfree(ctx->g_ptr);
  dfree(ctx->g_adj);
  long long m = 0;
  std::string err;
  cudaError_t e = graph::build_graph(ctx->n, ctx->rowptr, ctx->col, ctx->val, ctx->sym != 0, ctx->g_ptr, ctx->g_adj, m,
                                     ctx->cap, err);
  if (e != cudaSuccess)
    return fail(ctx, e == cudaErrorMemoryAllocation ? TLS_ERR_OOM : TLS_ERR_CUDA,
                "symmetrised graph: " + (err.empty() ? std::string(cudaGetErrorString(e)) : err));
  CK(cudaStreamSynchronize(ctx->cap));
  ctx->g_m = m;
  if (nedges) *nedges = m;
  return TLS_OK;
}

int32_t tls_graph_fetch(tls_ctx* ctx, int64_t* gptr, int32_t* gadj) {
  if (!ctx || ctx->g_m < 0) return ctx ? fail(ctx, TLS_ERR_STATE, "build the graph first") : TLS_ERR_ARG;
  CK(cudaSetDevice(ctx->device));
  if (gptr) CK(cudaMemcpy(gptr, ctx->g_ptr, sizeof(long long) * (ctx->n + 1), cudaMemcpyDeviceToHost));
  if (gadj && ctx->g_m > 0) CK(cudaMemcpy(gadj, ctx->g_adj, sizeof(int) * ctx->g_m, cudaMemcpyDeviceToHost));
  return TLS_OK;
}

int32_t tls_overlap_build(tls_ctx* ctx, int32_t n_sub, const int64_t* owner, int32_t overlap, int64_t* total,
                          int32_t* k_c) {
  TLS_RANGE("tls_overlap_build");
  if (!ctx || ctx->g_m < 0) return ctx ? fail(ctx, TLS_ERR_STATE, "build the graph first") : TLS_ERR_ARG;
  if (n_sub <= 0 || !owner) return fail(ctx, TLS_ERR_ARG, "bad subdomain count or owner vector");
  if (overlap < 1) return fail(ctx, TLS_ERR_ARG, "overlap must be at least 1");
  std::vector<int> own(ctx->n);
  for (int i = 0; i < ctx->n; ++i) {
    if (owner[i] < 0 || owner[i] >= n_sub) return fail(ctx, TLS_ERR_ARG, "owner ids out of range");
    own[i] = (int)owner[i];
  }
  CK(cudaSetDevice(ctx->device));
  int* d_owner = nullptr;
  TRY(upload(ctx, d_owner, own.data(), ctx->n));
  std::string err;
  cudaError_t e = graph::overlap_and_colour(ctx->n, ctx->g_ptr, ctx->g_adj, d_owner, n_sub, overlap, ctx->ov_off,
                                            ctx->ov_ls, ctx->ov_idx, ctx->ov_col, ctx->ov_kc, ctx->cap, err);
  ctx->dev_bytes -= (int64_t)sizeof(int) * ctx->n;
  dfree(d_owner);
  if (e != cudaSuccess)
    return fail(ctx, e == cudaErrorMemoryAllocation ? TLS_ERR_OOM : (e == cudaErrorInvalidValue ? TLS_ERR_ARG : TLS_ERR_CUDA),
                "overlap: " + (err.empty() ? std::string(cudaGetErrorString(e)) : err));
  ctx->ov_nsub = n_sub;
  ctx->ov_delta = overlap;
  if (total) *total = ctx->ov_idx.size();
  if (k_c) *k_c = ctx->ov_kc;
  return TLS_OK;
}

int32_t tls_overlap_fetch(tls_ctx* ctx, int64_t* offsets, int64_t* layer_sizes, int64_t* indices, int64_t* colors) {
  if (!ctx || ctx->ov_nsub == 0) return ctx ? fail(ctx, TLS_ERR_STATE, "run tls_overlap_build first") : TLS_ERR_ARG;
  if (offsets) std::copy(ctx->ov_off.begin(), ctx->ov_off.end(), offsets);
  if (layer_sizes) std::copy(ctx->ov_ls.begin(), ctx->ov_ls.end(), layer_sizes);
  if (indices) std::copy(ctx->ov_idx.begin(), ctx->ov_idx.end(), indices);
  if (colors) std::copy(ctx->ov_col.begin(), ctx->ov_col.end(), colors);
  return TLS_OK;
}

int32_t tls_graph_release(tls_ctx* ctx) {
  if (!ctx) return TLS_ERR_ARG;
  CK(cudaSetDevice(ctx->device));
  dfree(ctx->g_ptr);
  dfree(ctx->g_adj);
  ctx->g_m = -1;
  std::vector<long long>().swap(ctx->ov_idx);
  std::vector<long long>().swap(ctx->ov_off);
  std::vector<long long>().swap(ctx->ov_ls);
  std::vector<long long>().swap(ctx->ov_col);
  ctx->ov_nsub = 0;
  return TLS_OK;
}

// store A0 (row-major n_C x n_C, device) and turn on one refinement step of every coarse solve
int32_t tls_coarse_refine(tls_ctx* ctx, const double* a0, void* stream) {
  TLS_RANGE("tls_coarse_refine");
  if (!ctx || !ctx->nsub) return ctx ? fail(ctx, TLS_ERR_STATE, "upload subdomains first") : TLS_ERR_ARG;
  if (ctx->ncoarse == 0) return fail(ctx, TLS_ERR_STATE, "upload the coarse space first");
  if (!ctx->h_nofo.empty()) return fail(ctx, TLS_ERR_STATE, "coarse refinement needs the whole A0^{-1} (one GPU)");
  if (!a0) return fail(ctx, TLS_ERR_ARG, "null A0");
  if (ctx->chain_nb > 0 || !ctx->h_blk[ctx->nsub].tiles)
    return fail(ctx, TLS_ERR_STATE, "coarse refinement needs the stored A0^{-1} (not the block-tridiagonal solve)");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = (cudaStream_t)stream;
  const int nsub = ctx->nsub;
  BlkDesc a = ctx->h_blk[nsub];
  a.sym = 0;
  a.xoff = ctx->Xloc + ctx->cpad;
  TRY(dalloc(ctx, ctx->a0tiles, (int64_t)a.nt * a.nt * TT * TT));
  a.tiles = ctx->a0tiles;
  BlkDesc x2 = ctx->h_blk[nsub];
  x2.xoff = ctx->Xloc + 2 * ctx->cpad;
  ctx->h_blk[nsub + 1] = a;
  ctx->h_blk[nsub + 2] = x2;
  CK(cudaMemcpy(ctx->d_blk, ctx->h_blk.data(), sizeof(BlkDesc) * (nsub + 3), cudaMemcpyHostToDevice));
  dim3 g((unsigned)std::min<int64_t>((int64_t)a.nt * a.nt, 8192), 1);
  launch_k(ctx, k_pack_tiles, g, NTHR, 0, s, ctx->d_blk, nsub + 1, a0, (long long)ctx->ncoarse, 0LL);
  CKL();
  ctx->cref = true;
  ctx->finalized = false;
  destroy_graphs(ctx);
  return TLS_OK;
}

// ---------------------------------------------------------------------------------------------
// PCG (src/krylov.py:58-107)
// ---------------------------------------------------------------------------------------------
static int enq_pcg_iter(tls_ctx* ctx, cudaStream_t s, bool replace, bool prec) {
  PcgState* st = ctx->pcg;
  const int* done = &st->done;
  const int r0 = ctx->r0, no = nown(ctx);
  TRY(enq_halo(ctx, s, ctx->vp, done));
  TRY((spmv_lpr<0, 1>(ctx, s, ctx->vp, ctx->vap, nullptr, ctx->part, done)));
  TRY(enq_allreduce_part(ctx, s, ctx->Gs));
  launch_k(ctx, k_pcg_alpha, 1, NTHR, 0, s, st, ctx->part, ctx->Gs, ctx->ab);
  CKL();
  if (!replace) {
    launch_k(ctx, k_pcg_update, ctx->G, NTHR, 0, s, no, st, ctx->vx + r0, ctx->vr + r0, ctx->vp + r0, ctx->vap + r0,
                                         ctx->part, 1);
    CKL();
    TRY(enq_allreduce_part(ctx, s, ctx->G));
    launch_k(ctx, k_pcg_hist, 1, NTHR, 0, s, st, ctx->part, ctx->G, ctx->hist);
    CKL();
  } else {
    launch_k(ctx, k_pcg_update, ctx->G, NTHR, 0, s, no, st, ctx->vx + r0, ctx->vr + r0, ctx->vp + r0, ctx->vap + r0,
                                         ctx->part, 0);
    CKL();
    TRY(enq_halo(ctx, s, ctx->vx, done));
    TRY((spmv_lpr<1, 2>(ctx, s, ctx->vx, ctx->vr, ctx->vb, ctx->part, done)));
    TRY(enq_allreduce_part(ctx, s, ctx->Gs));
    launch_k(ctx, k_pcg_hist, 1, NTHR, 0, s, st, ctx->part, ctx->Gs, ctx->hist);
    CKL();
  }
  if (prec)
    TRY(enq_apply(ctx, s, ctx->vr, ctx->vz, true, done));
  else
    TRY(enq_identity(ctx, s, ctx->vr, ctx->vz, true, done));
  launch_k(ctx, k_pcg_beta, 1, NTHR, 0, s, st, ctx->part, ctx->G, ctx->ab);
  CKL();
  launch_k(ctx, k_pcg_pupdate, ctx->G, NTHR, 0, s, no, st, ctx->vp + r0, ctx->vz + r0);
  CKL();
  return TLS_OK;
}

static int ensure_hist(tls_ctx* ctx, int maxit) {
  if (maxit + 2 > ctx->hist_cap) {
    TRY(dalloc(ctx, ctx->hist, maxit + 2));
    TRY(dalloc(ctx, ctx->ab, 2 * (int64_t)maxit + 4));
    destroy_graphs(ctx);
    ctx->hist_cap = maxit + 2;
  }
  return TLS_OK;
}

int32_t tls_pcg(tls_ctx* ctx, const double* b, double* x, double tol, int32_t maxit,
                int32_t use_precond, double* history, double* coeffs, tls_status* st_out,
                tls_iter_cb cb, void* user, void* stream) {
  TLS_RANGE("tls_pcg");
  if (!ctx || !ctx->rowptr) return ctx ? fail(ctx, TLS_ERR_STATE, "no matrix uploaded") : TLS_ERR_ARG;
  if (use_precond) TRY(need_final(ctx));
  if (maxit < 0) return fail(ctx, TLS_ERR_ARG, "maxit must be non-negative");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = (cudaStream_t)stream;
  const bool prec = use_precond != 0;
  const int n = ctx->n;
  TRY(ensure_hist(ctx, maxit));
  const int launches0 = ctx->launches;
  tls_status stt{};
  // init: x = 0, r = b (all rows, internal numbering), ||b||
  if (ctx->h_nofo.empty()) {
    CK(cudaMemcpyAsync(ctx->vb, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  } else {
    launch_k(ctx, k_perm_in, grid_for(n, NTHR), NTHR, 0, s, n, ctx->d_nofo, b, ctx->vb);
    CKL();
  }
  CK(cudaMemcpyAsync(ctx->vr, ctx->vb, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  CK(cudaMemsetAsync(ctx->vx, 0, sizeof(double) * n, s));
  PcgState h{};
  h.tol = tol;
  h.maxit = maxit;
  CK(cudaMemcpyAsync(ctx->pcg, &h, sizeof(PcgState), cudaMemcpyHostToDevice, s));
  TRY(enq_dot(ctx, s, ctx->vb, ctx->vb, nullptr));
  launch_k(ctx, k_pcg_init, 1, NTHR, 0, s, ctx->pcg, ctx->part, ctx->G);
  CKL();
  CK(cudaMemcpyAsync(&h, ctx->pcg, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (h.bnorm == 0.0) {  // src/krylov.py:69-70
    CK(cudaMemsetAsync(x, 0, sizeof(double) * n, s));
    CK(cudaStreamSynchronize(s));
    history[0] = 0.0;
    stt.iterations = 0;
    stt.converged = 1;
    stt.gpu_launches = ctx->launches - launches0;
    if (st_out) *st_out = stt;
    return TLS_OK;
  }
  const double one = 1.0;
  CK(cudaMemcpyAsync(ctx->hist, &one, sizeof(double), cudaMemcpyHostToDevice, s));
  if (prec)
    TRY(enq_apply(ctx, s, ctx->vr, ctx->vz, true, nullptr, true));
  else
    TRY(enq_identity(ctx, s, ctx->vr, ctx->vz, true, nullptr));
  launch_k(ctx, k_pcg_rz0, 1, NTHR, 0, s, ctx->pcg, ctx->part, ctx->G);
  CKL();
  CK(cudaMemcpyAsync(ctx->vp, ctx->vz, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  const bool host_loop = cb || (sharded(ctx) && !ctx->comm->capturable());
  if (maxit > 0) {
    if (host_loop) {
      // per-iteration host loop (callback(it, x.copy()), src/krylov.py:92-93)
      for (int it = 1; it <= maxit; ++it) {
        TRY(enq_pcg_iter(ctx, s, it % PCG_GRAPH_ITERS == 0, prec));
        CK(cudaMemcpyAsync(&h, ctx->pcg, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (h.status == 2) break;
        if (cb) {
          TRY(api_out(ctx, s, ctx->vx, ctx->pout));
          CK(cudaStreamSynchronize(s));
          CK(cudaMemcpy(ctx->h_x, ctx->pout, sizeof(double) * n, cudaMemcpyDeviceToHost));
          if (cb(user, h.it, ctx->h_x) != 0)
            return fail(ctx, TLS_ERR_CALLBACK, "callback stopped the solve at iteration " + std::to_string(h.it));
        }
        if (h.done) break;
      }
    } else {
      const int gi = prec ? 1 : 0;
      if (!ctx->pcg_exec[gi]) {
        const int before = ctx->launches;
        cudaGraph_t graph;
        CK(cudaStreamBeginCapture(ctx->cap, cudaStreamCaptureModeThreadLocal));
        ctx->capturing = true;
        ctx->kt_n = 0;
        int rc = TLS_OK;
        for (int i = 1; i <= PCG_GRAPH_ITERS && rc == TLS_OK; ++i)
          rc = enq_pcg_iter(ctx, ctx->cap, i == PCG_GRAPH_ITERS, prec);
        ctx->capturing = false;
        ctx->kt_n_graph[0][gi] = ctx->kt_n;
        cudaError_t ec = cudaStreamEndCapture(ctx->cap, &graph);
        if (rc != TLS_OK) return rc;
        if (ec != cudaSuccess) return fail(ctx, TLS_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(ec));
        CK(cudaGraphInstantiate(&ctx->pcg_exec[gi], graph, 0));
        cudaGraphDestroy(graph);
        ctx->pcg_exec_launches[gi] = ctx->launches - before;
        ctx->launches = before;
      }
      const int max_launch = (maxit + PCG_GRAPH_ITERS - 1) / PCG_GRAPH_ITERS;
      for (int L = 0; L < max_launch; ++L) {
        CK(cudaGraphLaunch(ctx->pcg_exec[gi], s));
        ctx->launches += ctx->pcg_exec_launches[gi];
        CK(cudaMemcpyAsync(ctx->h_flag, &ctx->pcg->done, sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        harvest_ktime(ctx, ctx->kt_n_graph[0][gi]);
        if (ctx->h_flag[0]) break;
      }
    }
  }
  CK(cudaMemcpyAsync(&h, ctx->pcg, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
  TRY(api_out(ctx, s, ctx->vx, x));
  CK(cudaStreamSynchronize(s));
  const int its = h.it;
  CK(cudaMemcpy(history, ctx->hist, sizeof(double) * (its + 1), cudaMemcpyDeviceToHost));
  if (coeffs && its > 0) CK(cudaMemcpy(coeffs, ctx->ab, sizeof(double) * 2 * its, cudaMemcpyDeviceToHost));
  stt.iterations = its;
  stt.converged = h.converged;
  stt.gpu_launches = ctx->launches - launches0;
  if (h.status == 2) {
    stt.code = TLS_ERR_BREAKDOWN;
    stt.iteration = h.bad_it;
    stt.value = h.bad_val;
    if (st_out) *st_out = stt;
    char buf[128];
    snprintf(buf, sizeof buf, "non-positive curvature %.3e at iteration %d; matrix is not SPD", h.bad_val, h.bad_it);
    return fail(ctx, TLS_ERR_BREAKDOWN, buf);
  }
  if (st_out) *st_out = stt;
  return TLS_OK;
}

// ---------------------------------------------------------------------------------------------
// GMRES (src/krylov.py:127-195) + GMRES(m) restarts
// ---------------------------------------------------------------------------------------------
static int enq_gm_step(tls_ctx* ctx, cudaStream_t s, int j, bool prec) {
  GmState* st = ctx->gm;
  const int* stop = &st->cycle_stop;
  const long long ldv = ctx->n;
  const int r0 = ctx->r0, no = nown(ctx);
  double* vj = ctx->V + (long long)j * ldv;
  double* w = ctx->t6;
  if (prec) {
    TRY(enq_apply(ctx, s, vj, ctx->t5, false, stop));
    TRY(enq_halo(ctx, s, ctx->t5, stop));
    TRY((spmv_lpr<0, 0>(ctx, s, ctx->t5, w, nullptr, nullptr, stop)));
  } else {
    TRY(enq_halo(ctx, s, vj, stop));
    TRY((spmv_lpr<0, 0>(ctx, s, vj, w, nullptr, nullptr, stop)));
  }
  const int nc = j + 1;
  // CGS2 (src/krylov.py:157-165 to the same accuracy): h1 = V^T w; w -= V h1 fused with
  // h2 = V^T w (one read of V); w -= V h2 with the norm partials -> 3 reads of V, not 4
  launch_k(ctx, k_gm_gemvt, ctx->G, NTHR, 0, s, no, ctx->V + r0, ldv, nc, w + r0, ctx->part, stop);
  CKL();
  launch_k(ctx, k_gm_hreduce, nc, NTHR, 0, s, ctx->part, ctx->G, ctx->h1, stop);
  CKL();
  TRY(enq_allreduce(ctx, s, ctx->h1, nc));
  if (ctx->gm_fused && nc <= GM_FUSED_MAXCOLS) {
    launch_k(ctx, k_gm_update_gemvt, ctx->G, NTHR, sizeof(double) * ((size_t)(nc + 1) * NTHR + nc), s, 
        no, ctx->V + r0, ldv, nc, ctx->h1, w + r0, ctx->part, stop);
    CKL();
  } else {
    launch_k(ctx, k_gm_gemvn<0>, ctx->G, NTHR, 0, s, no, ctx->V + r0, ldv, nc, st, ctx->h1, w + r0, ctx->part, 1, stop);
    CKL();
    launch_k(ctx, k_gm_gemvt, ctx->G, NTHR, 0, s, no, ctx->V + r0, ldv, nc, w + r0, ctx->part, stop);
    CKL();
  }
  launch_k(ctx, k_gm_hreduce, nc, NTHR, 0, s, ctx->part, ctx->G, ctx->h2, stop);
  CKL();
  TRY(enq_allreduce(ctx, s, ctx->h2, nc));
  launch_k(ctx, k_gm_gemvn<1>, ctx->G, NTHR, 0, s, no, ctx->V + r0, ldv, nc, st, ctx->h2, w + r0, ctx->part, 1, stop);
  CKL();
  TRY(enq_allreduce_part(ctx, s, ctx->G));
  if (ctx->gm_givens_fused) {
    launch_k(ctx, k_gm_givens_scale, ctx->G, NTHR, 0, s, st, j, ctx->gm_cols + 1, ctx->H, ctx->h1, ctx->h2, ctx->part,
             ctx->G, ctx->cs, ctx->sn, ctx->gv, ctx->hist, no, (const double*)(w + r0),
             ctx->V + (long long)(j + 1) * ldv + r0);
    CKL();
    return TLS_OK;
  }
  launch_k(ctx, k_gm_givens, 1, NTHR, 0, s, st, j, ctx->gm_cols + 1, ctx->H, ctx->h1, ctx->h2, ctx->part, ctx->G,
                                 ctx->cs, ctx->sn, ctx->gv, ctx->hist);
  CKL();
  launch_k(ctx, k_gm_scale, ctx->G, NTHR, 0, s, no, st, w + r0, ctx->V + (long long)(j + 1) * ldv + r0, 0);
  CKL();
  return TLS_OK;
}

static int enq_gm_cycle_end(tls_ctx* ctx, cudaStream_t s, bool prec) {
  GmState* st = ctx->gm;
  const int r0 = ctx->r0, no = nown(ctx);
  launch_k(ctx, k_gm_trisolve, 1, 32, 0, s, st, ctx->gm_cols + 1, ctx->H, ctx->gv, ctx->yv);
  CKL();
  launch_k(ctx, k_gm_gemvn<0>, ctx->G, NTHR, 0, s, no, ctx->V + r0, ctx->n, -1, st, ctx->yv, ctx->t7 + r0, nullptr, 0,
                                        nullptr);
  CKL();
  if (prec) {
    TRY(enq_apply(ctx, s, ctx->t7, ctx->t5, false, nullptr));
    launch_k(ctx, k_axpy1, ctx->G, NTHR, 0, s, no, ctx->vx + r0, ctx->t5 + r0, nullptr);
  } else {
    launch_k(ctx, k_axpy1, ctx->G, NTHR, 0, s, no, ctx->vx + r0, ctx->t7 + r0, nullptr);
  }
  CKL();
  launch_k(ctx, k_gm_cycle_end, 1, 32, 0, s, st);
  CKL();
  TRY(enq_halo(ctx, s, ctx->vx, &st->done));
  TRY((spmv_lpr<1, 2>(ctx, s, ctx->vx, ctx->vr, ctx->vb, ctx->part, &st->done)));
  TRY(enq_allreduce_part(ctx, s, ctx->Gs));
  launch_k(ctx, k_gm_cycle_begin, 1, NTHR, 0, s, st, ctx->part, ctx->Gs, ctx->gv, ctx->gm_cols);
  CKL();
  launch_k(ctx, k_gm_scale, ctx->G, NTHR, 0, s, no, st, ctx->vr + r0, ctx->V + r0, 1);
  CKL();
  return TLS_OK;
}

static int ensure_gm(tls_ctx* ctx, int mcols) {
  if (mcols == ctx->gm_cols && ctx->V) return TLS_OK;
  const int64_t n = ctx->n;
  TRY(dalloc(ctx, ctx->V, n * (mcols + 1)));
  CK(cudaMemset(ctx->V, 0, sizeof(double) * n * (mcols + 1)));
  TRY(dalloc(ctx, ctx->H, (int64_t)(mcols + 1) * (mcols + 1)));
  TRY(dalloc(ctx, ctx->cs, mcols + 1));
  TRY(dalloc(ctx, ctx->sn, mcols + 1));
  TRY(dalloc(ctx, ctx->gv, mcols + 2));
  TRY(dalloc(ctx, ctx->yv, mcols + 1));
  TRY(dalloc(ctx, ctx->h1, mcols + 1));
  TRY(dalloc(ctx, ctx->h2, mcols + 1));
  const int64_t need = std::max<int64_t>((int64_t)(mcols + 1) * ctx->G, ctx->Gs);
  if (need > ctx->part_cap) {
    TRY(dalloc(ctx, ctx->part, need));
    ctx->part_cap = need;
    destroy_graphs(ctx);
  }
  ctx->gm_cols = mcols;
  if (const char* e = getenv("TLS_GM_FUSED")) ctx->gm_fused = atoi(e) != 0;
  if (const char* e = getenv("TLS_GM_GIVENS_FUSED")) ctx->gm_givens_fused = atoi(e) != 0;
  if (ctx->gm_fused) {  // (nc + 1) x NTHR + nc doubles of shared memory for the widest fused step

    const int mc = std::min(mcols + 1, GM_FUSED_MAXCOLS);
    CK(raise_smem(ctx->device, (const void*)k_gm_update_gemvt, sizeof(double) * ((size_t)(mc + 1) * NTHR + mc)));
  }
  for (int i = 0; i < 2; ++i) {
    if (ctx->gm_exec[i]) cudaGraphExecDestroy(ctx->gm_exec[i]);
    ctx->gm_exec[i] = nullptr;
  }
  return TLS_OK;
}

int32_t tls_gmres(tls_ctx* ctx, const double* b, double* x, double tol, int32_t maxit,
                  int32_t restart, int32_t use_precond, double* history, tls_status* st_out,
                  tls_iter_cb cb, void* user, void* stream) {
  TLS_RANGE("tls_gmres");
  if (!ctx || !ctx->rowptr) return ctx ? fail(ctx, TLS_ERR_STATE, "no matrix uploaded") : TLS_ERR_ARG;
  if (use_precond) TRY(need_final(ctx));
  const bool restarted = restart > 0 && restart < maxit;
  if (!restarted && maxit > 1000) {
    char buf[96];
    snprintf(buf, sizeof buf, "maxit %d exceeds the hard cap 1000", maxit);
    return fail(ctx, TLS_ERR_CAP, buf);
  }
  if (restarted && restart > 1000) return fail(ctx, TLS_ERR_CAP, "restart exceeds the hard cap 1000");
  if (maxit < 0) return fail(ctx, TLS_ERR_ARG, "maxit must be non-negative");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = (cudaStream_t)stream;
  const bool prec = use_precond != 0;
  const int n = ctx->n;
  const int mcols = std::max(1, std::min(restarted ? restart : maxit, n));
  TRY(ensure_gm(ctx, mcols));
  TRY(ensure_hist(ctx, maxit));
  const int launches0 = ctx->launches;
  tls_status stt{};
  GmState h{};
  h.tol = tol;
  h.maxit = maxit;
  h.restart = restarted ? restart : 0;
  h.restarted = restarted ? 1 : 0;
  CK(cudaMemcpyAsync(ctx->gm, &h, sizeof(GmState), cudaMemcpyHostToDevice, s));
  if (ctx->h_nofo.empty()) {
    CK(cudaMemcpyAsync(ctx->vb, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  } else {
    launch_k(ctx, k_perm_in, grid_for(n, NTHR), NTHR, 0, s, n, ctx->d_nofo, b, ctx->vb);
    CKL();
  }
  CK(cudaMemcpyAsync(ctx->vr, ctx->vb, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  CK(cudaMemsetAsync(ctx->vx, 0, sizeof(double) * n, s));
  CK(cudaMemsetAsync(ctx->H, 0, sizeof(double) * (size_t)(mcols + 1) * (mcols + 1), s));
  TRY(enq_dot(ctx, s, ctx->vb, ctx->vb, nullptr));
  // reuse pcg init to get ||b|| then seed the first cycle
  launch_k(ctx, k_pcg_init, 1, NTHR, 0, s, ctx->pcg, ctx->part, ctx->G);
  CKL();
  PcgState hp{};
  CK(cudaMemcpyAsync(&hp, ctx->pcg, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (hp.bnorm == 0.0 || maxit == 0) {  // src/krylov.py:140-141
    CK(cudaMemsetAsync(x, 0, sizeof(double) * n, s));
    CK(cudaStreamSynchronize(s));
    history[0] = hp.bnorm == 0.0 ? 0.0 : 1.0;
    stt.converged = hp.bnorm == 0.0;
    stt.gpu_launches = ctx->launches - launches0;
    if (st_out) *st_out = stt;
    return TLS_OK;
  }
  h.bnorm = hp.bnorm;
  CK(cudaMemcpyAsync(ctx->gm, &h, sizeof(GmState), cudaMemcpyHostToDevice, s));
  launch_k(ctx, k_gm_cycle_begin, 1, NTHR, 0, s, ctx->gm, ctx->part, ctx->G, ctx->gv, mcols);
  CKL();
  launch_k(ctx, k_gm_scale, ctx->G, NTHR, 0, s, nown(ctx), ctx->gm, ctx->vr + ctx->r0, ctx->V + ctx->r0, 1);
  CKL();
  const double one = 1.0;
  CK(cudaMemcpyAsync(ctx->hist, &one, sizeof(double), cudaMemcpyHostToDevice, s));
  GmState hs{};
  if (cb || (sharded(ctx) && !ctx->comm->capturable())) {
    for (int guard = 0; guard <= maxit; ++guard) {
      for (int j = 0; j < mcols; ++j) {
        TRY(enq_gm_step(ctx, s, j, prec));
        CK(cudaMemcpyAsync(&hs, ctx->gm, sizeof(GmState), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (cb && cb(user, hs.total + hs.k, nullptr) != 0)
          return fail(ctx, TLS_ERR_CALLBACK,
                      "callback stopped the solve at iteration " + std::to_string(hs.total + hs.k));
        if (hs.cycle_stop) break;
      }
      TRY(enq_gm_cycle_end(ctx, s, prec));
      CK(cudaMemcpyAsync(&hs, ctx->gm, sizeof(GmState), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      if (hs.done) break;
    }
  } else {
    const int gi = prec ? 1 : 0;
    if (!ctx->gm_exec[gi] || ctx->gm_exec_cols[gi] != mcols) {
      if (ctx->gm_exec[gi]) cudaGraphExecDestroy(ctx->gm_exec[gi]);
      ctx->gm_exec[gi] = nullptr;
      const int before = ctx->launches;
      cudaGraph_t graph;
      CK(cudaStreamBeginCapture(ctx->cap, cudaStreamCaptureModeThreadLocal));
      ctx->capturing = true;
      ctx->kt_n = 0;
      int rc = TLS_OK;
      for (int j = 0; j < mcols && rc == TLS_OK; ++j) rc = enq_gm_step(ctx, ctx->cap, j, prec);
      if (rc == TLS_OK) rc = enq_gm_cycle_end(ctx, ctx->cap, prec);
      ctx->capturing = false;
      ctx->kt_n_graph[1][gi] = ctx->kt_n;
      cudaError_t ec = cudaStreamEndCapture(ctx->cap, &graph);
      if (rc != TLS_OK) return rc;
      if (ec != cudaSuccess) return fail(ctx, TLS_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(ec));
      CK(cudaGraphInstantiate(&ctx->gm_exec[gi], graph, 0));
      cudaGraphDestroy(graph);
      ctx->gm_exec_cols[gi] = mcols;
      ctx->gm_exec_launches[gi] = ctx->launches - before;
      ctx->launches = before;
    }
    for (int guard = 0; guard <= maxit; ++guard) {
      CK(cudaGraphLaunch(ctx->gm_exec[gi], s));
      ctx->launches += ctx->gm_exec_launches[gi];
      CK(cudaMemcpyAsync(ctx->h_flag, &ctx->gm->done, sizeof(int), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      harvest_ktime(ctx, ctx->kt_n_graph[1][gi]);
      if (ctx->h_flag[0]) break;
    }
  }
  CK(cudaMemcpyAsync(&hs, ctx->gm, sizeof(GmState), cudaMemcpyDeviceToHost, s));
  TRY(api_out(ctx, s, ctx->vx, x));
  CK(cudaStreamSynchronize(s));
  CK(cudaMemcpy(history, ctx->hist, sizeof(double) * (hs.total + 1), cudaMemcpyDeviceToHost));
  stt.iterations = hs.total;
  stt.converged = hs.converged;
  stt.gpu_launches = ctx->launches - launches0;
  if (st_out) *st_out = stt;
  return TLS_OK;
}

int32_t tls_report(const tls_ctx* ctx, int64_t* n, int32_t* n_sub, int32_t* n_coarse, int64_t* tile_bytes) {
  if (!ctx) return TLS_ERR_ARG;
  if (n) *n = ctx->n;
  if (n_sub) *n_sub = ctx->nsub;
  if (n_coarse) *n_coarse = ctx->ncoarse;
  if (tile_bytes) *tile_bytes = ctx->tile_doubles * 8;
  return TLS_OK;
}

int32_t tls_profile_local_solve(tls_ctx* ctx, int32_t reps, double* avg_ms, double* algorithmic_bytes,
                                void* stream) {
  TRY(need_final(ctx));
  if (reps <= 0) return fail(ctx, TLS_ERR_ARG, "reps must be positive");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = (cudaStream_t)stream;
  const int which = ctx->combine == TLS_ADDITIVE ? L_ALL : L_LOCAL;
  const int u0 = 0;
  const int nu = which == L_ALL && ctx->chain_nb == 0 ? ctx->nu_local + ctx->nu_coarse : ctx->nu_local;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const bool band = ctx->local_kind >= 1;
  for (int i = 0; i <= reps; ++i) {
    if (i == 1) CK(cudaEventRecord(e0, s));
    if (band)
      if (ctx->band_tma == 5)
        launch_k(ctx, k_band_solve_tma<5>, ctx->nsub, NTHR, ctx->band_smem + ring_bytes(5) + TMA_BAR_BYTES, s,
                 ctx->d_band, ctx->xloc, ctx->yloc, nullptr, nullptr, nullptr);
      else if (ctx->band_tma == 4)
        launch_k(ctx, k_band_solve_tma<4>, ctx->nsub, NTHR, ctx->band_smem + ring_bytes(4) + TMA_BAR_BYTES, s,
                 ctx->d_band, ctx->xloc, ctx->yloc, nullptr, nullptr, nullptr);
      else if (ctx->band_ring == 4)
        launch_k(ctx, k_band_solve_ring<4>, ctx->nsub, NTHR, ctx->band_smem + ring_bytes(4), s, 
            ctx->d_band, ctx->xloc, ctx->yloc, nullptr, nullptr, nullptr);
      else if (ctx->band_ring == 2)
        launch_k(ctx, k_band_solve_ring<2>, ctx->nsub, NTHR, ctx->band_smem + ring_bytes(2), s, 
            ctx->d_band, ctx->xloc, ctx->yloc, nullptr, nullptr, nullptr);
      else if (ctx->band_unr == 2)
        launch_k(ctx, k_band_solve<2>, ctx->nsub, NTHR, ctx->band_smem, s, ctx->d_band, ctx->xloc, ctx->yloc, nullptr,
                                                                ctx->band_pf, nullptr, nullptr);
      else
        launch_k(ctx, k_band_solve<1>, ctx->nsub, NTHR, ctx->band_smem, s, ctx->d_band, ctx->xloc, ctx->yloc, nullptr,
                                                                ctx->band_pf, nullptr, nullptr);
    else
      launch_k(ctx, k_symv_tiles, nu, NTHR, 0, s, ctx->d_blk, ctx->d_units + u0, ctx->xloc, ctx->slots, nullptr);
    CKL();
  }
  CK(cudaEventRecord(e1, s));
  CK(cudaEventSynchronize(e1));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (avg_ms) *avg_ms = ms / reps;
  if (algorithmic_bytes)
    *algorithmic_bytes = ctx->algo_local + (which == L_ALL && !band && ctx->chain_nb == 0 ? ctx->algo_coarse : 0.0);
  return TLS_OK;
}

// in-graph timing of the local-solve kernel: on = 1 re-captures the solve graphs with CUDA event
// nodes around every band-solve node and resets the accumulators; *avg_ms = mean duration of
// the launches that did work (early exits after convergence are not counted), *count = their number
int32_t tls_set_kernel_timing(tls_ctx* ctx, int32_t on) {
  if (!ctx) return TLS_ERR_ARG;
  CK(cudaSetDevice(ctx->device));
  if ((on != 0) != ctx->ktime) destroy_graphs(ctx);
  ctx->ktime = on != 0;
  ctx->kt_sum_ms = 0.0;
  ctx->kt_count = 0;
  return TLS_OK;
}

// Kernel trace: while on, every launch made OUTSIDE graph capture (the host-driven PCG / GMRES loops a
// callback selects, and the apply entry points) is bracketed by an event pair.  tls_kernel_trace_dump
// synchronises, writes "name count total_ms" lines (descending total) into buf and clears the trace.
int32_t tls_set_kernel_trace(tls_ctx* ctx, int32_t on) {
  if (!ctx) return TLS_ERR_ARG;
  ctx->ktrace = on != 0;
  return TLS_OK;
}

int64_t tls_kernel_trace_dump(tls_ctx* ctx, char* buf, int64_t cap) {
  if (!ctx) return -1;
  cudaSetDevice(ctx->device);
  cudaDeviceSynchronize();
  std::map<std::string, std::pair<long long, double>> acc;
  for (auto& e : ctx->kt_trace) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e.second.first, e.second.second);
    const char* nm = nullptr;
    if (cudaFuncGetName(&nm, e.first) != cudaSuccess || !nm) nm = "?";
    auto& a = acc[nm];
    a.first++;
    a.second += ms;
    cudaEventDestroy(e.second.first);
    cudaEventDestroy(e.second.second);
  }
  ctx->kt_trace.clear();
  std::vector<std::pair<std::string, std::pair<long long, double>>> v(acc.begin(), acc.end());
  std::sort(v.begin(), v.end(), [](const auto& x, const auto& y) { return x.second.second > y.second.second; });
  std::string out;
  for (auto& e : v) {
    char line[512];
    snprintf(line, sizeof line, "%s %lld %.6f\n", e.first.c_str(), e.second.first, e.second.second);
    out += line;
  }
  if (buf && cap > 0) {
    const size_t k = std::min<size_t>(out.size(), (size_t)cap - 1);
    memcpy(buf, out.data(), k);
    buf[k] = 0;
  }
  return (int64_t)out.size();
}

int32_t tls_kernel_timing(const tls_ctx* ctx, double* avg_ms, int64_t* count) {
  if (!ctx) return TLS_ERR_ARG;
  if (avg_ms) *avg_ms = ctx->kt_count ? ctx->kt_sum_ms / (double)ctx->kt_count : 0.0;
  if (count) *count = ctx->kt_count;
  return TLS_OK;
}

// ---- banded local factors ---------------------------------------------------------------------
int32_t tls_set_local_kind(tls_ctx* ctx, int32_t kind) {
  if (!ctx || kind < 0 || kind > 2)
    return ctx ? fail(ctx, TLS_ERR_ARG, "local kind is 0 (inverse tiles), 1 (band Cholesky) or 2 (band LU)") : TLS_ERR_ARG;
  if (ctx->nsub) return fail(ctx, TLS_ERR_STATE, "set the local kind before tls_subdomains_upload");
  ctx->local_kind = kind;
  return TLS_OK;
}

int32_t tls_store_local_band(tls_ctx* ctx, int32_t first_g, int32_t count, const double* L,
                             int64_t ld, const double* dinv, int32_t nbmax, const int32_t* perm,
                             const int32_t* kcnt, void* stream) {
  TLS_RANGE("tls_store_local_band");
  if (!ctx) return TLS_ERR_ARG;
  if (ctx->local_kind != 1) return fail(ctx, TLS_ERR_STATE, "handle is not in band-Cholesky mode");
  if (!ctx->sym) return fail(ctx, TLS_ERR_ARG, "band factors need a symmetric matrix (Cholesky)");
  const int first = first_g - ctx->own_lo;
  if (first < 0 || count <= 0 || first + count > ctx->nsub)
    return fail(ctx, TLS_ERR_ARG, "subdomain range not owned by this handle");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = (cudaStream_t)stream;
  // step offsets of the batch: one allocation for data, one for offsets, one for counts
  std::vector<long long> offs;
  std::vector<int> ks;
  std::vector<long long> dstart(count), ostart(count);
  long long tot = 0;
  double need = 0.0;  // doubles the solve actually reads (zero strips skipped)
  int kp = 0;
  for (int b = 0; b < count; ++b) {
    const int sl = first + b, nb = ctx->h_band[sl].nb;
    if (nb > nbmax) return fail(ctx, TLS_ERR_ARG, "nbmax smaller than a subdomain's block count");
    if (ctx->h_n[sl] > ld) return fail(ctx, TLS_ERR_ARG, "ld smaller than a local block");
    dstart[b] = tot;
    ostart[b] = (long long)offs.size();
    for (int I = 0; I < nb; ++I) {
      const int code = kcnt[kp + I], K = code & 0xffff, fz = code >> 16;
      if (K < 0 || K > I || fz < 0 || fz > 8 * K) return fail(ctx, TLS_ERR_ARG, "band panel code out of range");
      offs.push_back(tot - dstart[b]);
      ks.push_back(code);
      tot += (long long)K * TT * TT + DIAG_PACK;
      need += (double)((long long)K * TT * TT - (long long)fz * 8 * TT + DIAG_PACK);
    }
    kp += nb;
  }
  double* data = nullptr;
  long long* d_off = nullptr;
  int* d_k = nullptr;
  if (cudaMalloc((void**)&data, sizeof(double) * tot) != cudaSuccess ||
      cudaMalloc((void**)&d_off, sizeof(long long) * offs.size()) != cudaSuccess ||
      cudaMalloc((void**)&d_k, sizeof(int) * ks.size()) != cudaSuccess)
    return fail(ctx, TLS_ERR_OOM, "band storage allocation failed");
  ctx->band_allocs.push_back(data);
  ctx->band_allocs.push_back(d_off);
  ctx->band_allocs.push_back(d_k);
  ctx->dev_bytes += (int64_t)(sizeof(double) * tot + sizeof(long long) * offs.size() + sizeof(int) * ks.size());
  CK(cudaMemcpy(d_off, offs.data(), sizeof(long long) * offs.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_k, ks.data(), sizeof(int) * ks.size(), cudaMemcpyHostToDevice));
  long long pp = 0;
  for (int b = 0; b < count; ++b) {
    const int sl = first + b;
    BandDesc& bd = ctx->h_band[sl];
    bd.data = data + dstart[b];
    bd.step_off = d_off + ostart[b];
    bd.kcnt = d_k + ostart[b];
    const int n = ctx->h_n[sl];
    for (int p = 0; p < n; ++p) {
      const int l = perm[pp + p];
      if (l < 0 || l >= n) return fail(ctx, TLS_ERR_ARG, "band permutation out of range");
      ctx->h_perm[ctx->h_off[sl] + p] = l;
    }
    pp += n;
  }
  ctx->band_bytes += 2.0 * 8.0 * need;  // forward with L, backward with L^T
  CK(cudaMemcpy(ctx->d_band + first, ctx->h_band.data() + first, sizeof(BandDesc) * count, cudaMemcpyHostToDevice));
  dim3 g(std::min(nbmax, 256), count);
  launch_k(ctx, k_pack_band, g, NTHR, 0, s, ctx->d_band, first, L, ld, dinv, nbmax);
  CKL();
  for (int i = first; i < first + count; ++i) ctx->stored[i] = 1;
  ctx->finalized = false;
  return TLS_OK;
}

// one step stream (K/R tiles + packed diagonal strips per block) for a batch: returns offsets
static int band_layout(tls_ctx* ctx, int first, int count, const int32_t* codes, bool upper,
                       std::vector<long long>& dstart, std::vector<long long>& offs,
                       std::vector<int>& ks, long long& tot, double& need) {
  dstart.assign(count, 0);
  offs.clear();
  ks.clear();
  tot = 0;
  need = 0.0;
  int kp = 0;
  for (int b = 0; b < count; ++b) {
    const int sl = first + b, nb = ctx->h_band[sl].nb;
    dstart[b] = tot;
    std::vector<long long> local(nb);
    // upper (U) steps are stored in backward-sweep order: block nb-1 first
    for (int q = 0; q < nb; ++q) {
      const int I = upper ? nb - 1 - q : q;
      const int code = codes[kp + I], K = code & 0xffff, z = code >> 16;
      const int lim = upper ? nb - 1 - I : I;
      if (K < 0 || K > lim || z < 0 || z > 8 * K) return fail(ctx, TLS_ERR_ARG, "band panel code out of range");
      local[I] = tot - dstart[b];
      tot += (long long)K * TT * TT + DIAG_PACK;
      need += (double)((long long)K * TT * TT - (long long)z * 8 * TT + DIAG_PACK);
    }
    for (int I = 0; I < nb; ++I) {
      offs.push_back(local[I]);
      ks.push_back(codes[kp + I]);
    }
    kp += nb;
  }
  return TLS_OK;
}

static int band_alloc(tls_ctx* ctx, long long tot, const std::vector<long long>& offs,
                      const std::vector<int>& ks, double** data, long long** d_off, int** d_k) {
  if (cudaMalloc((void**)data, sizeof(double) * tot) != cudaSuccess ||
      cudaMalloc((void**)d_off, sizeof(long long) * offs.size()) != cudaSuccess ||
      cudaMalloc((void**)d_k, sizeof(int) * ks.size()) != cudaSuccess)
    return fail(ctx, TLS_ERR_OOM, "band storage allocation failed");
  ctx->band_allocs.push_back(*data);
  ctx->band_allocs.push_back(*d_off);
  ctx->band_allocs.push_back(*d_k);
  ctx->dev_bytes += (int64_t)(sizeof(double) * tot + sizeof(long long) * offs.size() + sizeof(int) * ks.size());
  CK(cudaMemcpy(*d_off, offs.data(), sizeof(long long) * offs.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(*d_k, ks.data(), sizeof(int) * ks.size(), cudaMemcpyHostToDevice));
  return TLS_OK;
}

int32_t tls_store_local_band_lu(tls_ctx* ctx, int32_t first_g, int32_t count, const double* LU,
                                int64_t ld, const double* ldinv, const double* udinv, int32_t nbmax,
                                const int32_t* perm_in, const int32_t* perm_out, const int32_t* lcode,
                                const int32_t* ucode, void* stream) {
  TLS_RANGE("tls_store_local_band_lu");
  if (!ctx) return TLS_ERR_ARG;
  if (ctx->local_kind != 2) return fail(ctx, TLS_ERR_STATE, "handle is not in band-LU mode");
  const int first = first_g - ctx->own_lo;
  if (first < 0 || count <= 0 || first + count > ctx->nsub)
    return fail(ctx, TLS_ERR_ARG, "subdomain range not owned by this handle");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = (cudaStream_t)stream;
  for (int b = 0; b < count; ++b) {
    const int sl = first + b;
    if (ctx->h_band[sl].nb > nbmax || ctx->h_n[sl] > ld) return fail(ctx, TLS_ERR_ARG, "batch dimensions too small");
  }
  std::vector<long long> dsL, offL, dsU, offU;
  std::vector<int> kL, kU;
  long long totL, totU;
  double needL, needU;
  TRY(band_layout(ctx, first, count, lcode, false, dsL, offL, kL, totL, needL));
  TRY(band_layout(ctx, first, count, ucode, true, dsU, offU, kU, totU, needU));
  double *dL, *dU;
  long long *oL, *oU;
  int *cL, *cU;
  TRY(band_alloc(ctx, totL, offL, kL, &dL, &oL, &cL));
  TRY(band_alloc(ctx, totU, offU, kU, &dU, &oU, &cU));
  long long pp = 0, op = 0;
  for (int b = 0; b < count; ++b) {
    const int sl = first + b, n = ctx->h_n[sl];
    BandDesc& bd = ctx->h_band[sl];
    bd.data = dL + dsL[b];
    bd.step_off = oL + op;
    bd.kcnt = cL + op;
    bd.udata = dU + dsU[b];
    bd.ustep_off = oU + op;
    bd.ucnt = cU + op;
    op += bd.nb;
    for (int p = 0; p < n; ++p) {
      const int lo = perm_out[pp + p], li = perm_in[pp + p];
      if (lo < 0 || lo >= n || li < 0 || li >= n) return fail(ctx, TLS_ERR_ARG, "band permutation out of range");
      ctx->h_perm[ctx->h_off[sl] + p] = lo;
      ctx->h_perm_in[ctx->h_off[sl] + p] = li;
    }
    pp += n;
  }
  ctx->band_bytes += 8.0 * (needL + needU);  // forward with L, backward with U
  CK(cudaMemcpy(ctx->d_band + first, ctx->h_band.data() + first, sizeof(BandDesc) * count, cudaMemcpyHostToDevice));
  dim3 g(std::min(nbmax, 256), count);
  launch_k(ctx, k_pack_band, g, NTHR, 0, s, ctx->d_band, first, LU, ld, ldinv, nbmax);
  CKL();
  launch_k(ctx, k_pack_band_u, g, NTHR, 0, s, ctx->d_band, first, LU, ld, udinv, nbmax);
  CKL();
  for (int i = first; i < first + count; ++i) ctx->stored[i] = 1;
  ctx->finalized = false;
  return TLS_OK;
}

// ---- setup: banded Cholesky of a batch (K9, DMMA) ----------------------------------------------
// factor-order lower triangle + row profile of a batch of dense blocks (k_perm_lower)
int32_t tls_perm_lower(const double* a, const int64_t* perm, double* ap, int32_t* first, int32_t count, int64_t ld,
                       void* stream) {
  TLS_RANGE("tls_perm_lower");
  if (!a || !perm || !ap || !first || count <= 0 || ld <= 0 || ld > 65535 * 64) return TLS_ERR_ARG;
  launch_k(nullptr, k_perm_lower, dim3((unsigned)ld, (unsigned)count), NTHR, 0, (cudaStream_t)stream, a,
           (const long long*)perm, ap, (int*)first, (int)ld);
  return cudaGetLastError() == cudaSuccess ? TLS_OK : TLS_ERR_CUDA;
}

int32_t tls_band_cholesky(double* ap, int64_t ld, int32_t count, const int32_t* reach, int32_t nbk,
                          double* dinv, int32_t* info, void* stream) {
  TLS_RANGE("tls_band_cholesky");
  if (!ap || !dinv || !info || !reach || count <= 0 || nbk <= 0 || ld != 64LL * nbk) return TLS_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  for (int J = 0; J < nbk; ++J)
    if (reach[J] < 64 * (J + 1) || reach[J] > ld || reach[J] % 64) return TLS_ERR_ARG;
  const size_t smem = sizeof(double) * 4 * 64 * CP;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return TLS_ERR_CUDA;
  // cluster of CL CTAs per subdomain (one CTA per SM: 133 KB of tiles) -- the trailing-band tile
  // products of a panel run on CL SMs instead of one.  CL = the largest of 4, 2, 1 that keeps the
  // whole batch in ONE wave (count * CL <= SMs): 59 subdomains x 4 CTAs ran as two waves of 9.9 ms,
  // x 2 CTAs as one wave (TLS_K9_CLUSTER overrides).
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int cl = count * 4 <= sms ? 4 : (count * 2 <= sms ? 2 : 1);
  if (const char* e = getenv("TLS_K9_CLUSTER")) {
    const int v = atoi(e);
    if (v == 1 || v == 2 || v == 4) cl = v;
  }
  int* d_reach = nullptr;
  if (cudaMallocAsync((void**)&d_reach, sizeof(int) * nbk, s) != cudaSuccess) return TLS_ERR_OOM;
  if (cudaMemcpyAsync(d_reach, reach, sizeof(int) * nbk, cudaMemcpyHostToDevice, s) != cudaSuccess) return TLS_ERR_CUDA;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(count * cl));
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cl;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e;
  if (cl == 4) {
    if (raise_smem(dev, (const void*)k_band_chol<4>, smem) != cudaSuccess) return TLS_ERR_CUDA;
    e = cudaLaunchKernelEx(&cfg, k_band_chol<4>, ap, (long long)ld, (const int*)d_reach, (int)nbk, dinv, info);
  } else if (cl == 2) {
    if (raise_smem(dev, (const void*)k_band_chol<2>, smem) != cudaSuccess) return TLS_ERR_CUDA;
    e = cudaLaunchKernelEx(&cfg, k_band_chol<2>, ap, (long long)ld, (const int*)d_reach, (int)nbk, dinv, info);
  } else {
    if (raise_smem(dev, (const void*)k_band_chol<1>, smem) != cudaSuccess) return TLS_ERR_CUDA;
    cfg.numAttrs = 0;
    e = cudaLaunchKernelEx(&cfg, k_band_chol<1>, ap, (long long)ld, (const int*)d_reach, (int)nbk, dinv, info);
  }
  if (e != cudaSuccess || cudaGetLastError() != cudaSuccess) return TLS_ERR_CUDA;
  cudaFreeAsync(d_reach, s);
  // the host array must outlive the async copy
  return cudaStreamSynchronize(s) == cudaSuccess ? TLS_OK : TLS_ERR_CUDA;
}

// ---- sharding -------------------------------------------------------------------------------
int32_t tls_set_row_partition(tls_ctx* ctx, int64_t n, const int32_t* new_of_old, int32_t nranks,
                              const int32_t* row_starts, int32_t rank) {
  if (!ctx) return TLS_ERR_ARG;
  if (ctx->rowptr) return fail(ctx, TLS_ERR_STATE, "set the row partition before tls_matrix_upload");
  if (n <= 0 || n > INT32_MAX || !new_of_old || nranks < 1 || !row_starts || rank < 0 || rank >= nranks)
    return fail(ctx, TLS_ERR_ARG, "bad row partition");
  if (row_starts[0] != 0 || row_starts[nranks] != n) return fail(ctx, TLS_ERR_ARG, "row ranges must cover [0, n)");
  for (int q = 0; q < nranks; ++q)
    if (row_starts[q + 1] < row_starts[q]) return fail(ctx, TLS_ERR_ARG, "row ranges must be ascending");
  std::vector<char> seen(n, 0);
  for (int64_t g = 0; g < n; ++g) {
    const int v = new_of_old[g];
    if (v < 0 || v >= n || seen[v]) return fail(ctx, TLS_ERR_ARG, "new_of_old is not a permutation");
    seen[v] = 1;
  }
  CK(cudaSetDevice(ctx->device));
  ctx->h_nofo.assign(new_of_old, new_of_old + n);
  ctx->row_starts.assign(row_starts, row_starts + nranks + 1);
  ctx->r0 = row_starts[rank];
  ctx->r1 = row_starts[rank + 1];
  TRY(upload(ctx, ctx->d_nofo, ctx->h_nofo.data(), n));
  return TLS_OK;
}

// halo plan: per peer (ascending), the owned rows this rank sends and the ghost rows it receives
// (internal numbering, both sides in ascending row order)
int32_t tls_set_halo(tls_ctx* ctx, int32_t npeers, const int32_t* peers, const int32_t* send_counts,
                     const int32_t* send_rows, const int32_t* recv_counts, const int32_t* recv_rows) {
  if (!ctx) return TLS_ERR_ARG;
  if (ctx->h_nofo.empty()) return fail(ctx, TLS_ERR_STATE, "no row partition");
  if (npeers < 0) return fail(ctx, TLS_ERR_ARG, "bad peer count");
  CK(cudaSetDevice(ctx->device));
  XPlan& x = ctx->halo;
  x.peers.assign(peers, peers + npeers);
  x.scnt.assign(send_counts, send_counts + npeers);
  x.rcnt.assign(recv_counts, recv_counts + npeers);
  x.soff.assign(npeers, 0);
  x.roff.assign(npeers, 0);
  long long so = 0, ro = 0;
  for (int k = 0; k < npeers; ++k) {
    if (x.scnt[k] < 0 || x.rcnt[k] < 0) return fail(ctx, TLS_ERR_ARG, "negative halo count");
    x.soff[k] = so;
    x.roff[k] = ro;
    so += x.scnt[k];
    ro += x.rcnt[k];
  }
  for (long long i = 0; i < so; ++i)
    if (send_rows[i] < ctx->r0 || send_rows[i] >= ctx->r1) return fail(ctx, TLS_ERR_ARG, "halo sends a row not owned");
  for (long long i = 0; i < ro; ++i)
    if (recv_rows[i] < 0 || recv_rows[i] >= ctx->n || (recv_rows[i] >= ctx->r0 && recv_rows[i] < ctx->r1))
      return fail(ctx, TLS_ERR_ARG, "halo receives an owned or out-of-range row");
  x.stot = so;
  x.rtot = ro;
  TRY(upload(ctx, x.d_sidx, send_rows, so));
  TRY(upload(ctx, x.d_ridx, recv_rows, ro));
  TRY(dalloc(ctx, x.sbuf, so));
  TRY(dalloc(ctx, x.rbuf, ro));
  destroy_graphs(ctx);
  return TLS_OK;
}

// ASM overlap contributions this rank receives: per peer (ascending), `counts` entries of
// (global subdomain, internal row) in the sender's (subdomain, local index) order
int32_t tls_set_remote_contrib(tls_ctx* ctx, int32_t npeers, const int32_t* peers, const int32_t* counts,
                               const int32_t* subs, const int32_t* rows) {
  if (!ctx) return TLS_ERR_ARG;
  if (ctx->h_nofo.empty()) return fail(ctx, TLS_ERR_STATE, "no row partition");
  if (npeers < 0) return fail(ctx, TLS_ERR_ARG, "bad peer count");
  ctx->rc_peer.assign(peers, peers + npeers);
  ctx->rc_cnt.assign(counts, counts + npeers);
  long long tot = 0;
  for (int k = 0; k < npeers; ++k) tot += counts[k];
  ctx->rc_sub.assign(subs, subs + tot);
  ctx->rc_row.assign(rows, rows + tot);
  ctx->finalized = false;
  return TLS_OK;
}

int32_t tls_set_owned_range(tls_ctx* ctx, int32_t s_lo, int32_t s_hi) {
  if (!ctx || s_lo < 0 || s_hi <= s_lo) return ctx ? fail(ctx, TLS_ERR_ARG, "bad owned range") : TLS_ERR_ARG;
  ctx->own_lo = s_lo;
  ctx->own_hi = s_hi;
  return TLS_OK;
}

int32_t tls_nccl_unique_id(void* out, int32_t bytes) {
  std::string err;
  if (!out || bytes < (int32_t)sizeof(ncclUniqueId)) return TLS_ERR_ARG;
  if (!nccl_api().load(err)) return TLS_ERR_STATE;
  ncclUniqueId id;
  if (nccl_api().get_id(&id) != ncclSuccess) return TLS_ERR_CUDA;
  memcpy(out, &id, sizeof(id));
  return TLS_OK;
}

int32_t tls_comm_init_nccl(tls_ctx* ctx, const void* unique_id, int32_t nranks, int32_t rank) {
  if (!ctx || !unique_id || nranks < 1 || rank < 0 || rank >= nranks)
    return ctx ? fail(ctx, TLS_ERR_ARG, "bad communicator arguments") : TLS_ERR_ARG;
  std::string err;
  if (!nccl_api().load(err)) return fail(ctx, TLS_ERR_STATE, err);
  CK(cudaSetDevice(ctx->device));
  auto* c = new NcclComm();
  ncclUniqueId id;
  memcpy(&id, unique_id, sizeof(id));
  ncclResult_t r = nccl_api().init_rank(&c->comm, nranks, id, rank);
  if (r != ncclSuccess) {
    delete c;
    return fail(ctx, TLS_ERR_CUDA, std::string("ncclCommInitRank: ") + nccl_api().errstr(r));
  }
  c->rank = rank;
  c->nranks = nranks;
  delete ctx->comm;
  ctx->comm = c;
  destroy_graphs(ctx);
  return TLS_OK;
}

// test transport: capturable, moves nothing, logs the collective sequence (RecordComm)
int32_t tls_comm_init_record(tls_ctx* ctx, int32_t nranks, int32_t rank) {
  if (!ctx || nranks < 2 || rank < 0 || rank >= nranks) return ctx ? fail(ctx, TLS_ERR_ARG, "bad record comm") : TLS_ERR_ARG;
  auto* c = new RecordComm();
  c->rank = rank;
  c->nranks = nranks;
  delete ctx->comm;
  ctx->comm = c;
  destroy_graphs(ctx);
  return TLS_OK;
}

// transport of the handle: 0 none (plain single-GPU path), 1 NCCL, 2 in-process group,
// 3 recording; out3 (optional) = all-reduce / exchange / all-gather calls issued so far through
// the NCCL API (captured calls count once per capture, not per replay)
int32_t tls_comm_info(const tls_ctx* ctx, int64_t* out3) {
  if (!ctx) return -1;
  if (!ctx->comm) return 0;
  if (out3)
    for (int i = 0; i < 3; ++i) out3[i] = ctx->comm->calls[i];
  return ctx->comm->kind();
}

// how the coarse solve runs (after tls_precond_finalize): returns 0 = no coarse level, 1 = stored
// dense inverse tiles, 2 = block-tridiagonal substitution; out4 (optional) = {n_coarse, blocks,
// block size, algorithmic bytes one coarse solve on this rank streams}
int32_t tls_coarse_info(const tls_ctx* ctx, double* out4) {
  if (!ctx) return -1;
  if (out4) {
    out4[0] = ctx->ncoarse;
    out4[1] = ctx->chain_nb;
    out4[2] = ctx->chain_bs;
    out4[3] = ctx->algo_coarse;
  }
  return ctx->ncoarse <= 0 ? 0 : ctx->chain_nb > 0 ? 2 : 1;
}

int64_t tls_comm_record_log(const tls_ctx* ctx, int64_t* out, int64_t cap) {
  auto* rc = ctx ? dynamic_cast<RecordComm*>(ctx->comm) : nullptr;
  if (!rc) return -1;
  const int64_t n = (int64_t)rc->log.size();
  for (int64_t i = 0; i < std::min(n, cap); ++i) out[i] = rc->log[i];
  return n;
}

int32_t tls_group_create(int32_t nmembers, tls_group** out) {
  if (!out || nmembers < 1 || nmembers > MAX_GROUP) return TLS_ERR_ARG;
  auto* g = new tls_group(nmembers);
  for (int r = 0; r < nmembers; ++r) {
    if (cudaEventCreateWithFlags(&g->shared.ev_in[r], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&g->shared.ev_out[r], cudaEventDisableTiming) != cudaSuccess) {
      delete g;
      return TLS_ERR_CUDA;
    }
  }
  *out = g;
  return TLS_OK;
}

void tls_group_destroy(tls_group* g) {
  if (!g) return;
  for (auto e : g->shared.ev_in) if (e) cudaEventDestroy(e);
  for (auto e : g->shared.ev_out) if (e) cudaEventDestroy(e);
  delete g;
}

int32_t tls_comm_init_group(tls_ctx* ctx, tls_group* g, int32_t rank) {
  if (!ctx || !g || rank < 0 || rank >= g->shared.n) return ctx ? fail(ctx, TLS_ERR_ARG, "bad group rank") : TLS_ERR_ARG;
  auto* c = new GroupComm();
  c->g = &g->shared;
  c->rank = rank;
  c->nranks = g->shared.n;
  delete ctx->comm;
  ctx->comm = c;
  destroy_graphs(ctx);
  return TLS_OK;
}

}  // extern "C"
