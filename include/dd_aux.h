/*
 * dd_aux.h -- C ABI of the B200-native auxiliary-matrix solver (arXiv:2002.05019).
 *
 * The operation (§II APPROACH): the auxiliary (interface / dual-DoF)
 * matrix A of the direct domain-decomposition method is "symmetric ... block-wise
 * sparse (sparse collection of dense blocks)"; it "is LDL^T factorized via a very
 * fast symbolic factorization step [on the] attributed clique graph of the
 * block-wise sparse matrix, followed by a custom block LDL^T with restricted
 * Bunch-Kaufman pivoting [BUNCH1977]"; the factored auxiliary problem is then solved
 * for many excitations ("forward/backward substitution ... for
 * 200 excitations").  The three calls follow the north_star (BASELINE.json):
 *   dd_aux_analyze  block pattern + interface sizes -> clique-graph symbolic
 *                   factorization, elimination tree, block storage layout (host only)
 *   dd_aux_factor   block values -> P A P^T = L D L^T on the GPU
 *   dd_aux_solve    nrhs right-hand sides -> X = A^{-1} B on the GPU
 * Readings of the paper (restricted pivoting domain, CABS1, tie rule, explicit L,
 * refinement, norms) are listed in DESIGN.md "Readings" (L1-L16).
 *
 * Scalars: DD_REAL64 = IEEE binary64; DD_COMPLEX128 = (re, im) binary64 pairs,
 * complex SYMMETRIC (A^T = A, never conjugated anywhere).
 *
 * Memory ownership: the handle owns host symbolic data only.  Every device buffer
 * (values, factor, workspace, right-hand sides) is allocated and owned by the
 * caller (PyTorch in this repo); the library never calls cudaMalloc/cudaFree.
 * Pointers named d_* are DEVICE pointers, all others HOST pointers.  Streams are
 * passed as an opaque `void*` holding a cudaStream_t (NULL = legacy default stream).
 *
 * Errors: 0 = DD_OK.  -k = argument k invalid (LAPACK style, 1-based position).
 * DD_ZERO_PIVOT (+1): factorization completed but D is singular; a later solve
 * returns DD_ERR_SINGULAR.  Negative DD_ERR_* codes below.  dd_aux_last_error()
 * returns a thread-local message for the last failing call.  Handles are not
 * thread-safe; separate handles are independent.
 */
#ifndef DD_AUX_H
#define DD_AUX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dd_aux_handle_s* dd_aux_handle_t;

enum { DD_REAL64 = 0, DD_COMPLEX128 = 1 };

/* Block elimination orders.  AUTO = the lower-flop of ND and MINDEG (reading L8). */
enum { DD_ORDER_AUTO = 0, DD_ORDER_ND = 1, DD_ORDER_MINDEG = 2, DD_ORDER_NATURAL = 3, DD_ORDER_USER = 4 };

enum {
  DD_OK = 0,
  DD_ZERO_PIVOT = 1,           /* D is singular (reading L4): first_zero_pivot names the DoF     */
  DD_NONFINITE = 2,            /* a pivot column held NaN/Inf (reading L4b); first_zero_pivot names
                                  the first such (or zero) pivot in elimination order             */
  DD_ERR_CUDA = -100,          /* message carries the cudaError_t string                 */
  DD_ERR_WORKSPACE = -101,     /* a buffer size argument is smaller than required        */
  DD_ERR_NOT_FACTORED = -102,  /* dd_aux_solve before a successful dd_aux_factor         */
  DD_ERR_SINGULAR = -103,      /* solve with a factor that reported DD_ZERO_PIVOT        */
  DD_ERR_PATTERN = -104,       /* invalid block pattern (message says which rule)        */
  DD_ERR_INTERNAL = -105
};

typedef struct {
  int32_t order;              /* DD_ORDER_*                                               */
  const int32_t* user_order;  /* [nblk] block elimination order for DD_ORDER_USER (copied) */
  int32_t refine_steps;       /* iterative-refinement steps in dd_aux_solve (default 1, L7) */
  int32_t use_graphs;         /* 1: dd_aux_factor's level loop and the whole dd_aux_solve are captured
                                 once into CUDA graphs (per buffer-pointer set) and replayed; default 0.
                                 Ignored while tracing is enabled (the trace brackets every launch). */
  double refine_tol;          /* a refinement step is skipped (on the device, no host sync) when
                                 every column already has berr <= refine_tol; 0 = always refine */
  int32_t complex_3m;         /* complex Schur update with 3 real products (Gauss/3M, default 1) or
                                 4 (0); flop counts stay in the standard 8-flop convention */
  int32_t perturb;            /* reading L4 (opt-in, "perturbation fallback ... flagged"):
                                 1 = an EXACTLY zero pivot column (max(|a_kk|, colmax) == 0) gets the 1x1
                                 pivot d = perturb_tau * ||A||_inf instead of reporting DD_ZERO_PIVOT;
                                 counted in dd_aux_factor_info.nperturbed.  Default 0 (LAPACK semantics). */
  double perturb_tau;         /* > 0 when perturb = 1 (e.g. 1e-12)                                */
} dd_aux_options;

typedef struct {
  int64_t n, nblk, nnzb_in, nnzb_filled, n_levels, max_front; /* max_front = max_k s_k + r_k */
  int64_t max_level_width;                                    /* max nodes in one level       */
  double flops_factor;          /* algorithmic: mu*sum_k(s^3/3 + r s^2 + r^2 s), mu=4 complex */
  double flops_solve_per_rhs;   /* mu*2*sum_k(s^2 + 2 r s)                                     */
  double factor_value_bytes;    /* sum_k (s^2 + r s) * scalar bytes           */
  size_t factor_bytes;          /* size of d_factor                                            */
  size_t work_bytes;            /* size of d_work for dd_aux_factor                            */
  int32_t dtype, order_used;
  int64_t n_schur, n_groups;    /* Schur mode (dd_aux_analyze_partial): kept blocks, groups; else 0 */
  int64_t n_aux_dof;            /* Schur mode: DoFs of the auxiliary numbering (rows of G / X_b)   */
} dd_aux_info;

typedef struct {
  int64_t npos, nneg, nzero;    /* inertia from D (real only; complex: all zero)  (a6)        */
  int64_t n2x2, nswaps;         /* 2x2 pivots, symmetric interchanges                          */
  int64_t first_zero_pivot;     /* 0, or 1 + ORIGINAL global DoF index of the first zero or
                                   non-finite pivot in ELIMINATION order (block order, then the
                                   pivoted column order inside the block: LAPACK INFO order)   */
  float ms_load, ms_factor;     /* device time of the load and factor phases (CUDA events)     */
  int64_t nperturbed;           /* zero pivots replaced by the static perturbation (opt-in)    */
  int64_t nonfinite;            /* pivot columns with NaN/Inf decision values (reading L4b)    */
  double max_abs_L;             /* max |L_ij| over the unit-lower factor (>= 1; modulus for
                                   complex): the element-growth diagnostic of the restricted BK */
} dd_aux_factor_info;

/* Default options: AUTO order, 1 refinement step, 3M complex products. */
void dd_aux_default_options(dd_aux_options* opt);

/* Host-only symbolic phase ("very fast symbolic factorization step").
 *  nblk        number of interfaces (blocks), > 0
 *  blk_size    [nblk] interface sizes 0 < s_I <= 3328 (real) / 1664 (complex): the in-block
 *              Bunch-Kaufman kernel keeps a panel copy of L_II in shared memory
 *  colptr      [nblk+1] block-CSC column pointers of the LOWER block pattern
 *  rowidx      [colptr[nblk]] row block ids: sorted ascending per column, >= column,
 *              diagonal block present (first), no duplicates
 *  dtype       DD_REAL64 or DD_COMPLEX128
 *  opt         options (NULL = defaults); user_order is copied
 *  out         receives the new handle
 * All arrays are read during the call only.  Returns DD_ERR_PATTERN on an invalid
 * pattern (dd_aux_last_error names the rule). */
int dd_aux_analyze(int64_t nblk, const int64_t* blk_size, const int64_t* colptr, const int32_t* rowidx,
                   int32_t dtype, const dd_aux_options* opt, dd_aux_handle_t* out);

int dd_aux_get_info(dd_aux_handle_t h, dd_aux_info* info);

/* order[t] = original block id eliminated at position t (host out, [nblk]). */
int dd_aux_get_order(dd_aux_handle_t h, int32_t* order);

/* Elimination tree by ORIGINAL block id: parent[k] (-1 = root) and level[k] (height, leaves 0);
 * either pointer may be NULL.  nnz_struct (if non-NULL) receives sum_k |struct(k)|. */
int dd_aux_get_etree(dd_aux_handle_t h, int32_t* parent, int32_t* level, int64_t* nnz_struct);

/* struct(k) of every block k: the blocks adjacent to k when it is eliminated
 * (after fill), as ORIGINAL block ids in elimination order.  Host out: st_ptr [nblk+1] (by block
 * id), st_blk [nnz_struct]; either may be NULL (st_ptr alone gives the sizes). */
int dd_aux_get_struct(dd_aux_handle_t h, int64_t* st_ptr, int32_t* st_blk);

/* Bytes of d_work needed by dd_aux_solve for nrhs right-hand sides. */
int dd_aux_solve_work_bytes(dd_aux_handle_t h, int64_t nrhs, size_t* bytes);

/* Numeric factorization on the GPU.
 *  d_vals      device; all input blocks concatenated; block p (CSC position) is column-major
 *              s_row x s_col with leading dimension s_row at element offset val_offset[p];
 *              complex values interleaved (re, im) like torch.complex128.  Diagonal blocks are
 *              passed full, only their lower triangle is read.  Never written.  Must stay alive
 *              and unchanged while dd_aux_solve may refine (it re-reads A for the residual).
 *  val_offset  host [nnzb_in] element (not byte) offsets; copied into the handle
 *  d_factor    device, info.factor_bytes, 256-byte aligned; holds L, D, pivots and the
 *              device descriptor tables; must not be modified between factor and solve
 *  d_work      device, info.work_bytes, 256-byte aligned; scratch, free after return
 *  stream      cudaStream_t (as void*); the call enqueues all work on it and synchronizes it
 *              once at exit to return finfo
 *  finfo       host out (may be NULL)
 * Returns DD_OK, DD_ZERO_PIVOT (D singular), DD_NONFINITE (NaN/Inf met in a pivot column; the
 * factor is unusable), or an error.  With options.perturb an exactly zero pivot is perturbed
 * instead (DD_OK, finfo.nperturbed > 0).  After DD_ZERO_PIVOT / DD_NONFINITE a solve returns
 * DD_ERR_SINGULAR.
 * Reproducibility: the factor (and the solve) are bitwise reproducible run to run and between
 * direct launches and CUDA-graph replays: every Schur-update tile sums its contributors in a fixed
 * order and is subtracted from its target by exactly ONE L2 reduction per element and launch
 * (no accumulation order to depend on, K3). */
int dd_aux_factor(dd_aux_handle_t h, const void* d_vals, const int64_t* val_offset, void* d_factor,
                  void* d_work, void* stream, dd_aux_factor_info* finfo);

/* Multi-RHS solve X = A^{-1} B (forward L, D^{-1}, backward L^T) plus refine_steps steps of
 * iterative refinement r = b - A x, x += solve(r) against the ORIGINAL blocks d_vals.
 *  d_vals      the same buffer passed to dd_aux_factor (may be NULL iff refine_steps == 0)
 *  nrhs        >= 0 (0 is a no-op)
 *  d_B         device, n x nrhs column-major, leading dimension ldb >= n, ORIGINAL DoF order
 *              (DoF = sum_{I'<I} s_I' + local); overwritten by X (like LAPACK ?sytrs)
 *  d_work      device, dd_aux_solve_work_bytes(nrhs) bytes
 *  stream      enqueued asynchronously on this stream (no host synchronization) */
int dd_aux_solve(dd_aux_handle_t h, const void* d_factor, const void* d_vals, int64_t nrhs, void* d_B,
                 int64_t ldb, void* d_work, void* stream);

/* Diagnostics (synchronizes): per-position pivots of the factored diagonal blocks, host out.
 *  ipiv  [n] LAPACK convention, 1-based LOCAL to each block: ipiv = kp+1 (1x1) or -(kp+1) twice (2x2)
 *  perm  [n] composite in-block permutation, local 0-based: (P_k A_kk P_k^T)[a,b] = A_kk[perm[a], perm[b]]
 *  d, e  [n] diagonal and 2x2 sub-diagonal of D (scalar type of the handle; e = 0 off 2x2 firsts)
 * Entries are grouped by elimination position (block order[0] first).  Any pointer may be NULL. */
int dd_aux_get_pivots(dd_aux_handle_t h, const void* d_factor, int32_t* ipiv, int32_t* perm, void* d, void* e);

/* f1: on-device assembly of the auxiliary matrix from its cliques.
 * PAPER.md:27 (§II): eliminating a subdomain's primal unknowns leaves a dense contribution
 * over the dual DoFs of the interfaces it touches; the auxiliary matrix is the
 * resulting "sparse collection of dense blocks" (one dense clique per subdomain).  This call
 * writes every lower block of the handle's pattern:
 *     A_IJ = sum over cliques p containing I and J (ascending p) of  S_p[I rows, J cols]
 * or, with symmetrize != 0, of (S_p + S_p^T)/2 restricted to those rows/cols (reading L12;
 * complex: plain transpose, never conjugated).  Blocks no clique covers are written as zero.
 *  nclq        number of cliques (>= 0)
 *  clq_ptr     host [nclq+1]: clique p's members are clq_blk[clq_ptr[p] .. clq_ptr[p+1])
 *  clq_blk     host: interface (block) ids, strictly ascending within a clique; every pair of
 *              members must be in the handle's block pattern (else DD_ERR_PATTERN)
 *  d_S         device: clique p's dense m_p x m_p matrix (m_p = sum of its members' sizes,
 *              DoFs = members concatenated in the listed order), column-major, ld = m_p, at
 *              element offset S_offset[p]; complex interleaved (re, im).  Read only.
 *  S_offset    host [nclq] element offsets
 *  val_offset  host [nnzb_in] element offsets of the output blocks in d_vals (the layout
 *              dd_aux_factor reads: block at CSC position q is s_row x s_col, ld = s_row)
 *  d_vals      device out; every element of every block is written
 *  d_work      device, dd_aux_assemble_work_bytes() bytes, 256-byte aligned (descriptor tables)
 *  stream      enqueued asynchronously; the host tables are copied before the call returns
 * The sum is evaluated in a fixed order with correctly rounded additions, so it is bitwise
 * reproducible and equals the plain loop of oracle/assemble.py exactly. */
int dd_aux_assemble_work_bytes(dd_aux_handle_t h, int64_t nclq, const int64_t* clq_ptr, const int32_t* clq_blk,
                               size_t* bytes);
int dd_aux_assemble(dd_aux_handle_t h, int64_t nclq, const int64_t* clq_ptr, const int32_t* clq_blk,
                    const void* d_S, const int64_t* S_offset, int32_t symmetrize, const int64_t* val_offset,
                    void* d_vals, void* d_work, void* stream);
/* Same, accumulating: d_vals += the clique sum for every block some clique covers; blocks no
 * clique covers keep their values (f4: the top separators' own blocks plus the Schur contributions
 * of the subtrees factored on other GPUs).  symmetrize must be 0 (the cliques must be symmetric). */
int dd_aux_assemble_acc(dd_aux_handle_t h, int64_t nclq, const int64_t* clq_ptr, const int32_t* clq_blk,
                        const void* d_S, const int64_t* S_offset, int32_t symmetrize, const int64_t* val_offset,
                        void* d_vals, void* d_work, void* stream);
/* Algorithmic (unique) HBM bytes of the last dd_aux_assemble: every output element written once,
 * every contributing S_p element read once (the mirrored S_p[J, I] too for the symmetric part of
 * an off-diagonal block). */
double dd_aux_last_assemble_bytes(dd_aux_handle_t h);

/* Change the refinement policy of an analyzed handle (same meaning as the options fields). */
int dd_aux_set_refine(dd_aux_handle_t h, int32_t refine_steps, double refine_tol);

/* Enable / disable CUDA-graph replay (options.use_graphs) on an analyzed handle. */
int dd_aux_set_graphs(dd_aux_handle_t h, int32_t enable);

/* Tracing (SURVEY.md §5 "CUDA events per phase").  Launch counts and algorithmic flops per
 * kernel class are always accumulated; with tracing enabled every kernel launch is also
 * bracketed by a CUDA-event pair recorded on the launching stream, so ms[] is device time.
 * dd_aux_get_trace synchronizes the recorded events, returns the sums since the last reset
 * and resets them when reset != 0. */
enum {
  DD_PH_LOAD = 0, DD_PH_K1, DD_PH_ROWPERM, DD_PH_K2, DD_PH_K3, DD_PH_STATS,
  DD_PH_PERM, DD_PH_FDIAG, DD_PH_FUPD, DD_PH_DSOLVE, DD_PH_BUPD, DD_PH_BDIAG, DD_PH_SPMV,
  DD_PH_LINV, DD_PH_ASSEMBLE, DD_PH_SCHUR, DD_NPHASE
};
typedef struct {
  double ms[16];        /* device milliseconds per kernel class (tracing enabled only) */
  int64_t launches[16]; /* kernel launches per class                                     */
  double flops[16];     /* algorithmic flops per class (SURVEY.md §8(d) formulas)          */
} dd_aux_trace;
int dd_aux_set_trace(dd_aux_handle_t h, int32_t enable);
int dd_aux_get_trace(dd_aux_handle_t h, dd_aux_trace* out, int32_t reset);
/* Per-level factor trace since the last reset, row-major [n_levels][16] (DD_PH_* columns):
 * device ms (tracing enabled) and algorithmic flops.  Call after dd_aux_get_trace(reset=0). */
int dd_aux_get_level_trace(dd_aux_handle_t h, double* ms, double* flops);

/* ---------------------------------------------------------------------------------------------
 * f3 / f2: partial factorization ("Schur mode"), subdomain elimination and
 * primal recovery.  PAPER.md:27 (§II): the arrowhead system [K C; C^T A_bb] "is then reduced in
 * size by eliminating via many independent sparse direct factorizations the primal DoFs";
 * "the solution of all or a subset of primal unknowns are recovered in an
 * embarrassingly parallel manner via many smaller size sparse forward backward substitutions".
 *
 * The caller lays out every subdomain's arrowhead rows as ONE block-sparse symmetric matrix (same
 * input format as dd_aux_analyze): the primal DoFs of each subdomain grouped into blocks (a
 * supernode partition, e.g. a nested dissection -- the ordering input), followed by the KEPT
 * blocks: the last n_schur block ids, one per (subdomain, interface) pair, holding that
 * subdomain's copy of the interface's dual DoFs with A_bb,p on the diagonal block and C_p^T
 * against the primal blocks.  Subdomains share no block, so their eliminations are independent
 * and the level scheduler runs them side by side ("many independent ... factorizations").
 * dd_aux_factor then eliminates every non-kept block (restricted BK, as for the auxiliary matrix)
 * and leaves in the kept blocks of subdomain p its dense Schur contribution
 *     S_p = A_bb,p - C_p^T K_p^{-1} C_p.
 *  schur_target [n_schur] auxiliary block id I of kept block (nblk - n_schur + k); sizes must match
 *  schur_group  [n_schur] subdomain (clique) id of kept block k; one target per group at most
 *  n_aux, aux_blk_size [n_aux]  sizes of the auxiliary blocks (the auxiliary DoF numbering
 *               sum_{I'<I} s_I' + local is the row order of G and X_b below)
 *  opt->order   applies to the eliminated blocks (DD_ORDER_USER: a permutation of
 *               [0, nblk - n_schur)); the kept blocks follow in ascending id
 * dd_aux_factor on such a handle returns the inertia / pivot statistics of the eliminated part;
 * dd_aux_solve returns an error (use dd_aux_condense / dd_aux_recover).                        */
int dd_aux_analyze_partial(int64_t nblk, const int64_t* blk_size, const int64_t* colptr, const int32_t* rowidx,
                           int32_t dtype, const dd_aux_options* opt, int64_t n_schur, const int32_t* schur_target,
                           const int32_t* schur_group, int64_t n_aux, const int64_t* aux_blk_size,
                           dd_aux_handle_t* out);

/* Cliques of the exported Schur complements: groups g = distinct schur_group values ascending;
 * clq_blk[clq_ptr[g] .. clq_ptr[g+1]) = the targets of g's kept blocks, ascending (the clique
 * format of dd_aux_assemble).  Host out: ngroups, clq_ptr [ngroups+1], clq_blk [n_schur]; any
 * pointer may be NULL. */
int dd_aux_schur_cliques(dd_aux_handle_t h, int64_t* ngroups, int64_t* clq_ptr, int32_t* clq_blk);

/* f3 output: write every group's dense S_g (m_g x m_g, both triangles, column-major, ld = m_g,
 * DoFs = its kept blocks concatenated in clique order) at element offset S_offset[g] of d_S
 * (complex interleaved).  These are exactly the per-subdomain cliques dd_aux_assemble sums into
 * the auxiliary matrix.  Asynchronous on `stream`; HBM-bound gather from the factor arena. */
int dd_aux_schur_export(dd_aux_handle_t h, const void* d_factor, void* d_S, const int64_t* S_offset, void* stream);

/* Condensation of the right-hand side onto the auxiliary DoFs (forward sweep of the partial
 * factorization):  G <- G - sum_p R_p^T C_p^T K_p^{-1} f_p,  R_p = the auxiliary rows of p's
 * kept blocks.  d_F: n x nrhs (ld ldf, the handle's DoF numbering; kept rows are ignored);
 * d_G: n_aux_dof x nrhs (ld ldg), accumulated in a fixed order (pass G = b_b to obtain the
 * auxiliary right-hand side).  d_work: dd_aux_solve_work_bytes(h, nrhs).  Asynchronous. */
int dd_aux_condense(dd_aux_handle_t h, const void* d_factor, int64_t nrhs, const void* d_F, int64_t ldf, void* d_G,
                    int64_t ldg, void* d_work, void* stream);

/* f2 primal recovery (forward + backward sweep of the partial factorization with the kept rows
 * set to the auxiliary solution):  x_p = K_p^{-1} (f_p - C_p R_p x_b)  for every subdomain.
 * d_F as above; d_Xb: n_aux_dof x nrhs (ld ldxb); d_X: n x nrhs out (ld ldx; primal rows = x_p,
 * kept rows = the copies of x_b; d_X may equal d_F).  Asynchronous. */
int dd_aux_recover(dd_aux_handle_t h, const void* d_factor, int64_t nrhs, const void* d_F, int64_t ldf,
                   const void* d_Xb, int64_t ldxb, void* d_X, int64_t ldx, void* d_work, void* stream);

/* Residual R = B - A X over the handle's ORIGINAL blocks d_vals (both triangles; the kernel of
 * a8's refinement, K6), all n x nrhs column-major in the ORIGINAL DoF order.  Needs a factored
 * d_factor (its row maps); d_work: dd_aux_solve_work_bytes(h, nrhs).  Works on Schur-mode handles
 * (f4 refines across a partial handle per GPU plus the top handle).  Asynchronous. */
int dd_aux_residual(dd_aux_handle_t h, const void* d_factor, const void* d_vals, int64_t nrhs, const void* d_B,
                    int64_t ldb, const void* d_X, int64_t ldx, void* d_R, int64_t ldr, void* d_work, void* stream);

/* Convergence report: per-column backward error ||b_j - A x_j||_inf /
 * (||A||_inf ||x_j||_inf) (reading L6) of any X against the ORIGINAL blocks, computed on the device
 * and copied to berr [nrhs] (host); synchronizes `stream`.  nrhs <= 32768. */
int dd_aux_backward_error(dd_aux_handle_t h, const void* d_factor, const void* d_vals, int64_t nrhs, const void* d_B,
                          int64_t ldb, const void* d_X, int64_t ldx, void* d_work, double* berr, void* stream);

/* Debug check (host only): every access the kernels derive from the handle's descriptor tables
 * (panels, inverse tiles, W / K1 workspace, Schur-update targets and contributors, solve tiles,
 * Schur-mode export / scatter items) lies inside its buffer and the arena regions are disjoint.
 * DD_OK or DD_ERR_INTERNAL with the failed rule in dd_aux_last_error(). */
int dd_aux_validate(dd_aux_handle_t h);

int dd_aux_destroy(dd_aux_handle_t h);

const char* dd_aux_last_error(void);

/* Library version string. */
const char* dd_aux_version(void);

#ifdef __cplusplus
}
#endif
#endif /* DD_AUX_H */
