/*
 * tls_b200.h — C ABI of the B200-native two-level Schwarz Krylov hot path.
 *
 * Drop-in boundary for the reference package ``tlschwarz`` (pure Python over
 * numpy/scipy, /root/reference/pkg/src/tlschwarz).  Each entry point names
 * the reference interface it replaces (file:line, prefix src/ =
 * pkg/src/tlschwarz/).  The Python mirror of the reference API
 * (paper_2401_03915_b200/{sparsemat,precond,krylov}.py) binds these through
 * ctypes; INTEGRATION.md shows the binding a tlschwarz maintainer would add.
 *
 * Conventions
 *  - plain pointers and sizes only; ``stream`` is a cudaStream_t passed as
 *    void* (NULL = legacy default stream);
 *  - vectors (r, z, x, b) are DEVICE pointers of length n (fp64) unless a
 *    parameter says "host";
 *  - every call returns a tls_code; on failure tls_ctx_last_error() holds a
 *    message and tls_status (for solves) the reference exception payload;
 *  - the handle owns the CSR, subdomain maps, local inverse tiles and the
 *    coarse data; all are immutable after tls_precond_finalize (mirrors the
 *    read-only SparseMat buffers, src/sparsemat.py:51-52).  Calls on one
 *    handle must be serialised by the caller.
 */
#ifndef TLS_B200_H
#define TLS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TLS_ABI_VERSION 2
#define TLS_TILE 64           /* edge of the dense tiles of local operators */

typedef enum {
  TLS_OK = 0,
  TLS_ERR_DIM = 1,        /* ValueError "dimension mismatch"  (src/sparsemat.py:127-128) */
  TLS_ERR_BREAKDOWN = 2,  /* BreakdownError(iteration, curvature) (src/krylov.py:22-29)   */
  TLS_ERR_SUBDOMAIN = 3,  /* SubdomainSetupError(subdomain)       (src/subdomain.py:22-27) */
  TLS_ERR_COARSE = 4,     /* RuntimeError coarse not SPD/singular (src/coarse.py:175-181)  */
  TLS_ERR_CAP = 5,        /* ValueError maxit above hard cap 1000 (src/krylov.py:136-137)  */
  TLS_ERR_ARG = 6,        /* invalid argument / unsupported option                         */
  TLS_ERR_STATE = 7,      /* call order violated (e.g. apply before finalize)              */
  TLS_ERR_CUDA = 8,       /* CUDA runtime failure                                          */
  TLS_ERR_OOM = 9,        /* device allocation failed                                      */
  TLS_ERR_FORMAT = 10,    /* MatrixMarketError(lineno, message)  (src/sparsemat.py:20-25)  */
  TLS_ERR_IO = 11,        /* file could not be opened / written (OSError)                  */
  TLS_ERR_CALLBACK = 12   /* the per-iteration callback asked to stop (it raised: the binding
                             re-raises that exception, as src/krylov.py:92-93 lets it propagate) */
} tls_code;

typedef enum { TLS_ASM = 0, TLS_RAS = 1 } tls_one_level;                       /* src/precond.py:34 */
typedef enum { TLS_NONE = 0, TLS_ADDITIVE = 1, TLS_DEFLATED = 2 } tls_combine; /* src/precond.py:35 */

/* Solve outcome; mirrors SolveReport (src/krylov.py:32-49) + the exception payloads. */
typedef struct tls_status {
  int32_t code;          /* tls_code */
  int32_t iterations;    /* SolveReport.iterations */
  int32_t converged;     /* SolveReport.converged */
  int32_t iteration;     /* BreakdownError.iteration (code == TLS_ERR_BREAKDOWN) */
  double value;          /* BreakdownError curvature */
  int32_t gpu_launches;  /* kernels enqueued by this call (bench evidence) */
  int32_t pad_;
} tls_status;

typedef struct tls_ctx tls_ctx;

/* per-iteration hook: (user, iteration, HOST copy of the current iterate, or NULL for GMRES).
 * Non-NULL forces one host sync per iteration (src/krylov.py:92-93, 182-183).  Returns 0 to go
 * on; any other value stops the solve at once with TLS_ERR_CALLBACK (a binding whose callback
 * raised returns 1 and re-raises after the call). */
typedef int32_t (*tls_iter_cb)(void* user, int32_t iteration, const double* x_host);

/* ---- lifecycle --------------------------------------------------------- */
int32_t tls_abi_version(void);
int32_t tls_ctx_create(int32_t device, tls_ctx** out);
void tls_ctx_destroy(tls_ctx* ctx);
const char* tls_ctx_last_error(const tls_ctx* ctx);
/* device bytes owned by the handle (tiles, maps, workspaces) */
int64_t tls_ctx_device_bytes(const tls_ctx* ctx);

/* ---- SparseMat: replaces SparseMat(csr) canonical storage (src/sparsemat.py:36-52)
 * indptr/indices/data are HOST arrays of a canonical CSR (sorted, unique columns).
 * The structure is bounds-checked on the host (indptr[0] = 0, non-decreasing, indptr[n] = nnz,
 * 0 <= indices < n): TLS_ERR_DIM with the offending row / entry in tls_ctx_last_error. */
int32_t tls_matrix_upload(tls_ctx* ctx, int64_t nrows, int64_t nnz, const int64_t* indptr,
                          const int32_t* indices, const double* data, int32_t symmetric);
/* y = A x : replaces SparseMat.matvec (src/sparsemat.py:125-129) */
int32_t tls_spmv(tls_ctx* ctx, const double* x, double* y, void* stream);

/* ---- SubdomainMap list: replaces extend_overlap output (src/partition.py:201-231, 278-301)
 * offsets[n_sub+1], indices[offsets[n_sub]] (local order: interior ascending, then each
 * layer ascending), n_interior[n_sub]; all HOST arrays. */
int32_t tls_subdomains_upload(tls_ctx* ctx, int32_t n_sub, const int64_t* offsets,
                              const int64_t* indices, const int32_t* n_interior);
/* largest local size (for the setup batch workspace) */
int32_t tls_subdomain_max_size(const tls_ctx* ctx);

/* ---- setup helpers on the device --------------------------------------
 * Dense local blocks A_ii = A[idx][:, idx] (src/subdomain.py:53-69) for subdomains
 * [first, first+count), written row-major into out (count x ld x ld, device), padded
 * with the identity beyond n_i. */
int32_t tls_extract_blocks(tls_ctx* ctx, int32_t first, int32_t count, double* out,
                           int64_t ld, void* stream);
/* Store A_ii^{-1} (row-major, count x ld x ld, device) as 64x64 tiles: packed lower
 * triangle if the matrix is symmetric, all tiles otherwise.  Replaces the
 * factor_dense solve closures (src/subdomain.py:72-95) used at src/precond.py:117-118. */
int32_t tls_store_local_inverse(tls_ctx* ctx, int32_t first, int32_t count, const double* inv,
                                int64_t ld, void* stream);
/* Banded Cholesky local operators (SPD matrices; alternative to the inverse tiles).
 * tls_set_local_kind(ctx, 1) before tls_subdomains_upload.  For a batch of owned subdomains:
 * L = Cholesky factor of the block in factor order (row-major count x ld x ld, identity
 * padded), dinv = inverses of its 64x64 diagonal tiles (count x nbmax x 64 x 64 row-major),
 * perm (HOST, concatenated) = local index stored at each factor position, kcnt (HOST,
 * concatenated) = per 64-row block K_I | (z_I << 16): the band is L[I, I-K_I .. I] and its first
 * z_I 8-column strips are identically zero (skipped by the solve). */
int32_t tls_set_local_kind(tls_ctx* ctx, int32_t kind);  /* 0 inverse tiles, 1 band Cholesky, 2 band LU */
int32_t tls_store_local_band(tls_ctx* ctx, int32_t first, int32_t count, const double* L,
                             int64_t ld, const double* dinv, int32_t nbmax, const int32_t* perm,
                             const int32_t* kcnt, void* stream);
/* Banded LU local operators (general matrices, kind 2; the lu_solve closure of
 * src/subdomain.py:83-89).  LU = packed getrf factors of the block in factor order (row-major
 * count x ld x ld; strictly-lower part = L, upper part = U), ldinv / udinv = inverses of the
 * unit-lower / upper 64x64 diagonal tiles, perm_in = local index gathered into each input
 * position (factor order composed with the row pivots), perm_out = local index of each output
 * position, lcode = K_I | (leading zero strips << 16) of L, ucode = R_I | (trailing zero strips
 * << 16) of U (panel U[I, I+1 .. I+R_I]); all codes/permutations HOST, concatenated. */
int32_t tls_store_local_band_lu(tls_ctx* ctx, int32_t first, int32_t count, const double* LU,
                                int64_t ld, const double* ldinv, const double* udinv, int32_t nbmax,
                                const int32_t* perm_in, const int32_t* perm_out, const int32_t* lcode,
                                const int32_t* ucode, void* stream);
/* Coarse space (src/coarse.py:23-49): per subdomain a dense block Z_s of shape
 * n_interior[s] x k[s] stored column by column (k[s] x n_interior[s] row-major, device,
 * concatenated in subdomain order), columns
 * [col_start[s], col_start[s]+k[s]) of the global basis; a0inv = (Z^T A Z)^{-1}
 * (row-major n_coarse^2, device; NULL when tls_coarse_chain supplies the operator).  k == NULL or
 * n_coarse == 0 disables the coarse level. */
int32_t tls_coarse_upload(tls_ctx* ctx, int32_t n_coarse, const int32_t* k, const double* basis,
                          const double* a0inv, void* stream);
/* Block-tridiagonal coarse solve instead of a stored dense inverse (call tls_coarse_upload with
 * a0inv == NULL first).  A0 = Z^T A Z (src/coarse.py:158-170) couples neighbouring subdomains
 * only, so in subdomain order it is block tridiagonal for blocks of block_size >= half bandwidth
 * + 1 columns (a multiple of 64; n_blocks = ceil(n_coarse / block_size) >= 2).  sinv[i] (host
 * array of n_blocks DEVICE addresses): the inverse of the Schur block S_i (S_0 = A_00,
 * S_i = A_ii - A_{i,i-1} S_{i-1}^{-1} A_{i-1,i}), row-major n_i x n_i, symmetric.  lo_* / up_*:
 * the strictly block-lower part of A0 and its transpose as CSR over all n_coarse rows with
 * global column indices (device, int32 / fp64, nnz entries each).  The coarse solve of
 * src/coarse.py:178-182 (a Cholesky solve with A0) then runs as a block forward / backward
 * substitution: 2 n_blocks - 1 products with the S_i^{-1} tiles and 2 (n_blocks - 1) sparse block
 * rows -- ~2 n_C * block_size doubles per solve instead of n_C^2 / 2.  Symmetric operators only;
 * excludes tls_coarse_refine.  Call before tls_precond_finalize. */
int32_t tls_coarse_chain(tls_ctx* ctx, int32_t n_blocks, int32_t block_size, const uint64_t* sinv,
                         const int32_t* lo_indptr, const int32_t* lo_indices, const double* lo_values,
                         const int32_t* up_indptr, const int32_t* up_indices, const double* up_values,
                         int64_t nnz, void* stream);
/* One step of iterative refinement on every coarse solve: y = X c; y += X (c - A0 y), X the
 * stored A0^{-1}.  a0 = Z^T A Z (row-major n_coarse^2, device).  The reference solves with an LU /
 * Cholesky factor of A0 (src/coarse.py:172-182, backward stable); the explicit inverse alone
 * leaves a residual ~cond(A0)*eps, so setup turns this on when cond_1(A0) > 1e8 (one GPU only).
 * Call after tls_coarse_upload, before tls_precond_finalize. */
int32_t tls_coarse_refine(tls_ctx* ctx, const double* a0, void* stream);
/* Build the apply schedule (work units, reduction lists, prolongation pull map). */
int32_t tls_precond_finalize(tls_ctx* ctx, int32_t one_level, int32_t combine);

/* ---- apply: replaces Preconditioner.apply / apply_one_level / coarse_apply
 * (src/precond.py:114-136) */
int32_t tls_precond_apply(tls_ctx* ctx, const double* r, double* z, void* stream);
int32_t tls_apply_one_level(tls_ctx* ctx, const double* r, double* z, void* stream);
int32_t tls_coarse_apply(tls_ctx* ctx, const double* r, double* z, void* stream);
/* The pieces of the apply, for the reference's attribute API and for parity checks:
 * tls_local_solve: y_i = A_ii^{-1} R_i r for `count` listed subdomains (global ids, owned by this
 *   handle), each in the reference's local order, concatenated into out (device, sum of n_i) --
 *   Preconditioner.local_solves[i] (src/subdomain.py:72-95, called at src/precond.py:117-118);
 * tls_coarse_restrict: c = Z^T r (n_coarse)      -- CoarseSpace.restrict     (src/coarse.py:40-41);
 * tls_coarse_solve:    y = A0^{-1} c (one GPU)   -- CoarseSpace.solve_coarse (src/coarse.py:46-49);
 * tls_coarse_prolong:  z = Z y (n)               -- CoarseSpace.prolong      (src/coarse.py:43-44). */
int32_t tls_local_solve(tls_ctx* ctx, const double* r, int32_t count, const int32_t* subdomains,
                        double* out, void* stream);
int32_t tls_coarse_restrict(tls_ctx* ctx, const double* r, double* c, void* stream);
int32_t tls_coarse_solve(tls_ctx* ctx, const double* c, double* y, void* stream);
int32_t tls_coarse_prolong(tls_ctx* ctx, const double* y, double* z, void* stream);

/* ---- Krylov: replaces pcg (src/krylov.py:58-107) and gmres (src/krylov.py:127-195).
 * b, x device; history HOST buffer of maxit+1 doubles (SolveReport.residuals);
 * coeffs (pcg, may be NULL) HOST buffer of 2*maxit doubles receiving (alpha_k, beta_k) for
 * the tridiagonal condition estimate (src/krylov.py:110-124);
 * use_precond = 0 reproduces precond=None (src/krylov.py:52-55).
 * gmres: restart <= 0 is the reference's unrestarted GMRES (maxit <= 1000);
 * restart > 0 runs GMRES(restart) cycles on the true residual (build extension). */
int32_t tls_pcg(tls_ctx* ctx, const double* b, double* x, double tol, int32_t maxit,
                int32_t use_precond, double* history, double* coeffs, tls_status* st,
                tls_iter_cb cb, void* user, void* stream);
int32_t tls_gmres(tls_ctx* ctx, const double* b, double* x, double tol, int32_t maxit,
                  int32_t restart, int32_t use_precond, double* history, tls_status* st,
                  tls_iter_cb cb, void* user, void* stream);

/* ---- decomposition on the device, bit-exact with symmetrized_graph
 * (src/sparsemat.py:180-195), extend_overlap (src/partition.py:278-301) and color_subdomains
 * (src/partition.py:304-334).  Works on the uploaded matrix in the caller's numbering (not on a
 * sharded handle).
 * tls_graph_build: edges {i,j}, i != j, with |a_ij| > 0 or |a_ji| > 0 -> *nedges (directed count);
 * tls_graph_fetch: host copies, gptr (n+1), gadj (nedges), rows in ascending column order;
 * tls_overlap_build: overlap rings of every subdomain (owner: host, n entries in [0, n_sub)) and
 *   the greedy colouring -> *total = sum of the index-set sizes, *k_c = colours used;
 * tls_overlap_fetch: offsets (n_sub+1), layer_sizes (n_sub x overlap), indices (total: interior
 *   ascending, then each layer ascending), colors (n_sub); host buffers;
 * tls_graph_release: frees the device graph and the host results. */
int32_t tls_graph_build(tls_ctx* ctx, int64_t* nedges);
int32_t tls_graph_fetch(tls_ctx* ctx, int64_t* gptr, int32_t* gadj);
int32_t tls_overlap_build(tls_ctx* ctx, int32_t n_sub, const int64_t* owner, int32_t overlap, int64_t* total,
                          int32_t* k_c);
int32_t tls_overlap_fetch(tls_ctx* ctx, int64_t* offsets, int64_t* layer_sizes, int64_t* indices, int64_t* colors);
int32_t tls_graph_release(tls_ctx* ctx);

/* ---- setup kernel K12b: Galerkin assembly (src/coarse.py:158-168): for each plan entry p =
 * (s, j) = plan_sj[2p..2p+1] and rows [plan_off[p], plan_off[p+1]) of rows / grp (HOST arrays):
 * A0[cstart[j] + a, cstart[s] + b] = sum_r Z_j[rows[r], a] W_s[grp[r], b], with Z_j / W_s device
 * row-major (n x kcnt) blocks at zptr[j] / wptr[s] (HOST pointer tables); A0 device n_C x n_C. */
int32_t tls_galerkin_assemble(const int32_t* plan_sj, const int64_t* plan_off, int64_t nplan, const int64_t* zptr,
                              const int64_t* wptr, const int32_t* kcnt, const int64_t* cstart, int32_t nsub,
                              const int64_t* rows, const int64_t* grp, int64_t nrows, double* A0, int64_t nC,
                              void* stream);

/* ---- setup kernel K9b: banded LU with partial pivoting (src/subdomain.py:83-89) of `count` blocks
 * (ap: count x ld x ld row-major, device, in place; ld = 64 nbk) in LAPACK's getrf format: packed
 * unit-lower L and U, piv (device, count x ld, 1-based, interchanges applied across the whole row
 * width), info (device, count: first zero pivot, 1-based, or 0).  lreach[J] / ureach[J] (HOST,
 * multiples of 64): rows / columns the band can touch in panel J. */
int32_t tls_band_lu(double* ap, int64_t ld, int32_t count, const int32_t* lreach, const int32_t* ureach, int32_t nbk,
                    int32_t* piv, int32_t* info, void* stream);

/* ---- setup kernel K10: X <- (L L^T)^{-1} X for `count` banded Cholesky factors (L: count x ld x ld
 * row-major, lower, factor order, ld = 64 nb; dinv: count x nb x 64 x 64 inverted diagonal tiles;
 * kc: HOST count x nb panel-tile counts; X: count x ld x nrhs row-major, in place) on the FP64
 * tensor cores -- the harmonic extension's multi-RHS solve (src/subdomain.py:108-120). */
int32_t tls_band_solve_multi(const double* L, int64_t ld, int32_t count, const double* dinv, const int32_t* kc,
                             int32_t nb, double* X, int64_t nrhs, void* stream);

/* ---- setup kernel K12a: rank-filter pivots (src/coarse.py:119-155): column-pivoted Householder
 * QR of `count` coarse blocks (block s: nrows[s] x ncols[s] column-major at W + woff[s], device,
 * overwritten; ncols <= 64) -> HOST rdiag / perm (concatenated, sum(ncols) entries): |R_jj| and
 * the original column at pivot position j. */
int32_t tls_rank_filter_pivots(double* W, const int64_t* woff, const int32_t* nrows, const int32_t* ncols,
                               int32_t count, double* rdiag, int32_t* perm, void* stream);

/* ---- setup helper: batched symmetric eigensolver (parallel cyclic Jacobi, one CTA per matrix)
 * for the p x p Rayleigh-Ritz matrices of the setup's subspace iteration (p <= 64): T (batch x p x
 * p, device, symmetrised on load) -> w (batch x p, descending), V (batch x p x p, row-major, the
 * eigenvectors as columns).  Stream-ordered; replaces the LAPACK eigh of src/spectral.py:80 on the
 * projected problem. */
int32_t tls_syevj_batched(const double* T, int64_t batch, int32_t p, double* w, double* V, void* stream);

/* ---- setup helper: batched one-sided Jacobi SVD (one CTA per matrix) for the SVD coarse modes
 * (src/spectral.py:135-154 calls LAPACK's thin SVD of the harmonic extension E; the setup takes
 * E = Q R and passes the small R here).  X (batch x [m x n column-major, leading dimension m],
 * device) is rotated in place to X V with mutually orthogonal columns: column j = sigma_j u_j
 * (unsorted); sig (batch x n) receives the column norms, info (batch) the sweeps used or -1 when
 * 60 sweeps did not converge.  Stream-ordered. */
int32_t tls_svdj_batched(double* X, int64_t batch, int32_t m, int32_t n, double* sig, int32_t* info, void* stream);

/* ---- SetupReport getters (src/precond.py:39-83) */
int32_t tls_report(const tls_ctx* ctx, int64_t* n, int32_t* n_sub, int32_t* n_coarse,
                   int64_t* tile_bytes);

/* ---- sharding across GPUs (build extension, the reference is single-process).
 * Each rank owns a contiguous slab [s_lo, s_hi) of the global subdomain list and the rows
 * those subdomains own.  tls_set_row_partition (before tls_matrix_upload) renumbers the rows
 * rank by rank (new_of_old[g] = internal row of caller row g; rank q owns internal rows
 * [row_starts[q], row_starts[q+1])); the library then stores P A P^T and maps every subdomain
 * index through new_of_old.  Vectors at the ABI stay in the caller's numbering (inputs full,
 * outputs completed on every rank).  Inside a solve each rank computes only its owned rows:
 * SpMV, local solves of its subdomains, its rows of A0^{-1} c, prolongation, vector updates.
 * Exchanges: a halo of ghost rows (tls_set_halo: rows each peer sends / this rank receives, in
 * ascending internal order), the ASM overlap contributions to rows of other ranks
 * (tls_set_remote_contrib: what this rank receives, (global subdomain, internal row) in the
 * sender's (subdomain, local index) order -- the sender side is derived by the library), sum
 * all-reduces of the dot-product partials and of c = Z^T r.  tls_set_owned_range before
 * tls_subdomains_upload (which still receives the global maps; extract/store/coarse-upload then
 * take global subdomain ids of owned subdomains, coarse k[] for all subdomains and the basis of
 * the owned ones).  NCCL communicators are CUDA-graph capturable; an in-process group (several
 * handles on one GPU driven from host threads) runs the identical schedule for validation. */
typedef struct tls_group tls_group;
int32_t tls_set_owned_range(tls_ctx* ctx, int32_t s_lo, int32_t s_hi);
int32_t tls_set_row_partition(tls_ctx* ctx, int64_t n, const int32_t* new_of_old, int32_t nranks,
                              const int32_t* row_starts, int32_t rank);
int32_t tls_set_halo(tls_ctx* ctx, int32_t npeers, const int32_t* peers, const int32_t* send_counts,
                     const int32_t* send_rows, const int32_t* recv_counts, const int32_t* recv_rows);
int32_t tls_set_remote_contrib(tls_ctx* ctx, int32_t npeers, const int32_t* peers,
                               const int32_t* counts, const int32_t* subs, const int32_t* rows);
int32_t tls_nccl_unique_id(void* out, int32_t bytes);
int32_t tls_comm_init_nccl(tls_ctx* ctx, const void* unique_id, int32_t nranks, int32_t rank);
int32_t tls_group_create(int32_t nmembers, tls_group** out);
void tls_group_destroy(tls_group* g);
int32_t tls_comm_init_group(tls_ctx* ctx, tls_group* g, int32_t rank);
/* test transport: capturable, moves no data, logs (kind, count, peers) of every collective the
 * sharded schedule issues -- validates CUDA-graph capture of the NCCL schedule on one GPU */
int32_t tls_comm_init_record(tls_ctx* ctx, int32_t nranks, int32_t rank);
/* Sharded coarse restriction by all-gather: rank q's subdomains own the global coarse columns
 * [col_starts[q], col_starts[q+1]) (nranks + 1 entries; after tls_coarse_upload and the
 * communicator).  Without it c = Z^T r is summed by an all-reduce of the whole n_C vector. */
int32_t tls_set_coarse_layout(tls_ctx* ctx, int32_t nranks, const int64_t* col_starts);
int64_t tls_comm_record_log(const tls_ctx* ctx, int64_t* out, int64_t cap);
/* Transport of the handle: 0 none (plain single-GPU path), 1 NCCL, 2 in-process group,
 * 3 recording.  out3 (may be NULL): all-reduce / exchange / all-gather calls issued through the
 * NCCL API so far (a captured call counts once per capture, not per graph replay). */
int32_t tls_comm_info(const tls_ctx* ctx, int64_t* out3);
/* The uploaded basis blocks (per owned subdomain k[s] x n_interior[s] row-major, subdomain order,
 * count = sum n_interior[s] * k[s] doubles) copied to HOST memory: the data behind
 * CoarseSpace.basis (src/coarse.py:23-38), read on demand instead of during setup. */
int32_t tls_coarse_basis_fetch(tls_ctx* ctx, double* out, int64_t count);
/* How the coarse solve of src/coarse.py:178-182 runs (after tls_precond_finalize): 0 no coarse
 * level, 1 stored dense A0^{-1} tiles, 2 block-tridiagonal substitution (tls_coarse_chain).
 * out4 (may be NULL): {n_coarse, blocks, block size, algorithmic bytes one coarse solve streams
 * on this rank}. */
int32_t tls_coarse_info(const tls_ctx* ctx, double* out4);

/* ---- measurement: average device time (ms) of the dominant kernel (batched local
 * solve) over the last solve, timed with CUDA events on the launching stream, and
 * the algorithmic bytes one launch of it must move. */
int32_t tls_profile_local_solve(tls_ctx* ctx, int32_t reps, double* avg_ms,
                                double* algorithmic_bytes, void* stream);
/* in-graph timing of the band local-solve kernel inside real PCG / GMRES solves: on = 1
 * re-captures the solve graphs with CUDA event nodes around each band-solve node (and resets);
 * tls_kernel_timing returns the mean duration of the launches that did work. */
int32_t tls_set_kernel_timing(tls_ctx* ctx, int32_t on);
int32_t tls_kernel_timing(const tls_ctx* ctx, double* avg_ms, int64_t* count);

/* kernel trace (profiling aid): while on, every launch made outside graph capture -- the host-driven
 * PCG / GMRES loops (selected by a callback) and the apply entry points -- is bracketed by CUDA
 * events; tls_kernel_trace_dump synchronises, writes "kernel count total_ms" lines (descending
 * total) into buf (NUL-terminated, truncated to cap) and returns the untruncated length. */
int32_t tls_set_kernel_trace(tls_ctx* ctx, int32_t on);
int64_t tls_kernel_trace_dump(tls_ctx* ctx, char* buf, int64_t cap);

/* ---- setup: a batch of dense blocks a (count x ld x ld, row-major, device) in factor order, lower
 * triangle only: ap[b, i, j] = a[b, perm[b,i], perm[b,j]] for j <= i, 0 above the diagonal, and the
 * row profile first[b, i] = smallest j with a nonzero (count x ld int32) -- the input of
 * tls_band_cholesky (src/subdomain.py:80-82 factors the block in its local order instead). */
int32_t tls_perm_lower(const double* a, const int64_t* perm, double* ap, int32_t* first, int32_t count, int64_t ld,
                       void* stream);

/* ---- setup: banded Cholesky of a batch of SPD blocks (factor order, dense ld x ld row-major,
 * ld = 64 nbk) in place on the device, one CTA per block, DMMA tile products; reach[J] (host,
 * multiple of 64) = end row of the band below panel J; dinv receives the inverted 64 x 64
 * diagonal blocks (count x nbk x 64 x 64), info the 1-based first non-positive pivot row. */
int32_t tls_band_cholesky(double* ap, int64_t ld, int32_t count, const int32_t* reach, int32_t nbk,
                          double* dinv, int32_t* info, void* stream);

/* ---- Matrix Market ingest / output (src/sparsemat.py:201-372).
 * Host-side, multithreaded.  tls_mm_parse / tls_mm_load parse text / a file (nthreads <= 0: all
 * host threads) with the reference's dialect, validation order and error texts; on
 * TLS_ERR_FORMAT the handle carries (line, message) of MatrixMarketError.  On success
 * tls_mm_info gives the sizes and tls_mm_export copies the canonical CSR (sorted columns,
 * duplicates summed, explicit zeros of coordinate files kept, symmetric lower storage expanded;
 * array zeros dropped) into caller buffers of nrows+1 / nnz / nnz elements, ready for
 * tls_matrix_upload.  Always release the handle with tls_mm_free (also after an error).
 * tls_mm_write writes general coordinate format with %.17g values (write_matrix_market). */
typedef struct tls_mm tls_mm;
int32_t tls_mm_parse(const char* text, int64_t len, int32_t nthreads, tls_mm** out);
int32_t tls_mm_load(const char* path, int32_t nthreads, tls_mm** out);
int32_t tls_mm_info(const tls_mm* mm, int64_t* nrows, int64_t* ncols, int64_t* nnz, int32_t* symmetric,
                    int64_t* err_line, const char** err_msg);
int32_t tls_mm_export(const tls_mm* mm, int64_t* indptr, int32_t* indices, double* data);
void tls_mm_free(tls_mm* mm);
int32_t tls_mm_write(const char* path, int64_t nrows, int64_t ncols, const int64_t* indptr,
                     const int32_t* indices, const double* data, int32_t nthreads);

#ifdef __cplusplus
}
#endif
#endif /* TLS_B200_H */
