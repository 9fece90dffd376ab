// Kernel argument blocks and launchers (host <-> device boundary inside the library).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "layout.hpp"

namespace ddk {
using namespace ddaux;

struct LoadBlock {     // K0: one caller block -> arena
  int64_t voff;        // element offset in d_vals
  int64_t dst;         // element offset of the destination (row 0, col 0) in the arena
  int64_t ld;          // destination leading dimension
  int32_t rows, cols;  // stored block shape s_I x s_J
  int32_t trans, diag; // write transposed; diagonal block (lower only)
};

struct K1Args {
  const int* nodes;
  const NodeDev* nd;
  double* arena;
  int64_t aim;
  double* work;
  int64_t wim;
  int* perm;
  int* ipiv;
  int* gperm;
  int* ginv;
  int64_t d_off, e_off;
  int64_t* stats;
  int nb;  // K1 panel width override (0 = automatic; env DD_AUX_K1NB, A/B only)
  int fullw;  // 1: whole-block W cache when it fits with a >= 32-column panel (env DD_AUX_K1FULLW=0 off)
  // reading L4 (opt-in): an exactly-zero pivot column gets d = perturb_tau * ||A||_inf, with
  // ||A||_inf read from *normA (bits of a double, computed on the device before K1); 0 = off
  double perturb_tau;
  const unsigned long long* normA;
  unsigned long long* maxL;  // atomicMax of max |L_ij| (bits of a non-negative double)
};

struct RowpermArgs {
  const RowPerm* list;
  const NodeDev* nd;
  double* arena;
  int64_t aim;
  const int* perm;
};

struct K2Args {
  unsigned long long* maxL;  // atomicMax of max |L_ik| (bits of a non-negative double)
  const Tile* items;      // GEMM tiles (node, row strip, column tile)
  const Strip* strips;    // row strips for L = W D^{-1}
  const NodeDev* nd;
  double* arena;
  int64_t aim;
  double* work;
  int64_t wim;
  const int* perm;
  const int* ipiv;
  int64_t d_off, e_off;
};

struct K3Args {
  const UpdTarget* targets;   // this launch's targets (cost-sorted)
  const int64_t* tprefix;     // tprefix[t] = level-relative index of target t's first tile
  int ntargets;
  int64_t tile0;              // level-relative index of this launch's first tile
  const UpdContrib* contribs;
  const NodeDev* nd;
  double* arena;
  int64_t aim;
  const double* work;
  int64_t wim;
  int64_t ntiles;             // persistent variant: tiles of this launch
  unsigned long long* counter;  // persistent variant: dynamic tile counter (zeroed before the launch)
};

struct LinvArgs {      // full inverse of each unit-lower L_tt from its TB x TB tile inverses
  const DTile* items;  // (node, column tile of width TB)
  const NodeDev* nd;
  double* arena;
  int64_t aim;
};

struct SolveArgs {
  const NodeDev* nd;
  const double* arena;  // factor values
  int64_t aim;
  double* y;            // position-ordered padded RHS block, planar
  int64_t yim, ldy;
  int nrhs;
  const int* nodes;             // level nodes (diag kernels)
  const SolveTarget* ftargets;  // forward update tiles
  const SolveContrib* fcontribs;
  const int2* btiles;           // backward update tiles (t, tm)
  const int* st_pos;            // struct arrays
  const int* st_row;
  const int* ipiv;
  int64_t d_off, e_off;
  int64_t nrows;                // padded n
  const int* flag;              // refinement sweep: run only if *flag != 0 (nullptr = always)
  const DTile* dtiles;          // diagonal-solve tiles of the level (node, 64-row tile, T offset)
  double* T;                    // level buffer for the diagonal solves (planar), ld ldT
  int64_t Tim, ldT;
  int* cnt;                     // backward split-K arrival counters (zero between launches), or null
};

struct PermArgs {
  const int* gperm;   // padded position row -> original DoF (-1 pad)
  int64_t nrows;      // padded n
  int64_t rowlim;     // perm_in: rows >= rowlim are zeroed instead of gathered (0 = no limit)
  int nrhs;
  const double* src;  // interleaved (complex) or real, column-major, leading dim lds
  int64_t lds;
  double* dst;
  int64_t ldd;
  double* y;
  int64_t yim, ldy;
  int accumulate;
  const int* flag;    // accumulate only if *flag != 0 (nullptr = always)
};

struct SpmvArgs {
  const SpRow* rows;
  const SpSeg* segs;
  const int64_t* blk_size;   // original sizes
  const int64_t* odof;       // original DoF offsets per block
  const double* vals;        // caller's original blocks (interleaved complex)
  const double* X;           // current solution (caller's B buffer), ld ldx
  int64_t ldx;
  const double* Bsave;       // original right-hand sides, ld n
  int64_t ldb;
  const int* ginv;           // original DoF -> padded position row
  double* y;                 // residual out (position order, planar)
  int64_t yim, ldy;
  int nrhs;
};

struct AsmItem {       // f1: one 32-column chunk of one output block (lower pattern, caller layout)
  int64_t dst;         // element offset of the block in d_vals (column-major rows x cols, ld = rows)
  int32_t rows, cols;  // s_I, s_J
  int32_t c0;          // first column of the chunk
  int32_t k0, k1;      // contributor range (ascending clique index)
  int32_t pad;         // 1 = diagonal block (byte accounting only)
};

struct AsmContrib {    // clique p's sub-block: S_p[ra + r, cb + c], S_p column-major with ld = m_p
  int64_t soff;        // element offset of S_p in d_S
  int64_t ld;
  int32_t ra, cb;
};

struct AsmArgs {
  const AsmItem* items;
  const AsmContrib* con;
  const double* S;     // interleaved complex or real
  double* vals;
  int accumulate;      // 1: vals += sum (symmetrize off), uncovered blocks untouched
};

void launch_assemble(bool cplx, bool sym, const AsmArgs& a, int nitems, cudaStream_t st);

// ---- f3/f2: partial (Schur-mode) factorization helpers (kernels_schur.cu)
struct SxItem {        // one (member a, member b) sub-block of group g's dense Schur complement S_g
  int64_t src;         // element offset (re plane) in the arena of the stored block's element (0, 0)
  int64_t dst;         // element offset of S_g[ra, cb] inside S_g (ra + cb * m)
  int32_t ld;          // leading dimension of the stored block (panel ld)
  int32_t mode;        // 0: S = stored; 1: S = stored^T; 2: diagonal block (lower stored, mirrored); 3: zero
  int32_t rows, cols;  // s_a, s_b
  int32_t group, m;    // group index; m_g (leading dimension of S_g)
};
struct SxTile {        // 32 x 32 output tile of an item
  int32_t item, r0, c0, pad;
};
struct SchurExportArgs {
  const SxItem* items;
  const SxTile* tiles;
  const double* arena;
  int64_t aim;
  double* S;            // caller's output (interleaved complex or real)
  const int64_t* soff;  // [ngroups] element offsets of S_g in S (uploaded per call)
};
struct SgItem {        // aux block I of the condensed right-hand side: its kept copies
  int64_t aux_row;     // first row of I in the auxiliary DoF numbering
  int32_t s;           // s_I
  int32_t c0, c1;      // range in the contributor list (kept positions, ascending)
  int32_t pad;
};
struct SchurVecArgs {
  const NodeDev* nd;
  const SgItem* items;   // gather: per aux block; scatter: per kept node (c0 = its position)
  const int* contrib;    // kept positions
  double* y;             // solve vector (position order, planar)
  int64_t yim, ldy;
  double* G;             // gather: caller's aux-ordered block (interleaved), += ; scatter: source
  int64_t ldg;
  int nrhs;
};
void launch_schur_export(bool cplx, const SchurExportArgs& a, int ntiles, cudaStream_t st);
void launch_schur_gather(bool cplx, const SchurVecArgs& a, int nitems, cudaStream_t st);
void launch_schur_scatter(bool cplx, const SchurVecArgs& a, int nitems, cudaStream_t st);
int asm_chunk();

void launch_load(bool cplx, const double* vals, const LoadBlock* lb, int nblocks, int64_t max_elems, double* arena,
                 int64_t aim, cudaStream_t st);
size_t k1_smem(bool cplx, int max_s, int nb_req);
void launch_k1(bool cplx, const K1Args& a, int nnodes, int max_s, cudaStream_t st);
// largest interface (diagonal block) size K1 supports: its panel copy of L (s x 8 columns at the
// narrowest panel) + the W window must fit the 210 KB shared-memory budget
constexpr int K1_MAX_BLOCK_REAL = 3328, K1_MAX_BLOCK_CPLX = 1664;
constexpr int K1_MAX_BLOCK = K1_MAX_BLOCK_REAL;
void launch_rowperm(bool cplx, const RowpermArgs& a, int nlist, int max_s, cudaStream_t st);
void launch_k2(bool cplx, int cfg, const K2Args& a, int nitems, int nstrips, int max_s, cudaStream_t st);
int k3_bm(bool cplx, int cfg);
int k3_bn(bool cplx, int cfg);
void launch_k3(bool cplx, int cfg, const K3Args& a, int ntiles, cudaStream_t st, bool persistent = false);
// totals: [npos, nneg, nzero, n2x2, nswaps, first zero/non-finite pivot (1 + original DoF, in
// elimination order; 0 = none), nperturbed, nonfinite]
void launch_k4(const int64_t* node_stats, int nnodes, const int* gperm, int64_t* out, cudaStream_t st);

int solve_bm(bool cplx);   // row tile of the forward/backward update kernels
void launch_perm_in(bool cplx, const PermArgs& a, cudaStream_t st);
void launch_perm_out(bool cplx, const PermArgs& a, cudaStream_t st);
void launch_copy(bool cplx, const double* src, int64_t lds, double* dst, int64_t ldd, int64_t n, int nrhs,
                 cudaStream_t st);
void launch_linv(bool cplx, const LinvArgs& a, int nitems, cudaStream_t st);
// m3: complex products in the 3M (Gauss) form
void launch_diag_gemm(bool cplx, bool m3, bool backward, const SolveArgs& a, int ntiles, cudaStream_t st);
void launch_fupd(bool cplx, bool m3, const SolveArgs& a, int ntiles, cudaStream_t st);
void launch_dsolve(bool cplx, const SolveArgs& a, cudaStream_t st);
// max_rp: largest padded struct-row count of the level's nodes (bounds the split-K factor)
void launch_bupd(bool cplx, bool m3, const SolveArgs& a, int ntiles, int max_rp, double* part, cudaStream_t st);
size_t bupd_part_bytes(bool cplx, int nrhs);
size_t bupd_cnt_bytes(bool cplx, int nrhs);
int spmv_bm();
// ||A||_inf of the caller's original blocks (max row sum of moduli) -> *out (bits of a double)
void launch_norm_a(bool cplx, const SpmvArgs& a, int nrow_tiles, unsigned long long* out, cudaStream_t st);
// per-column backward error of the residual held in y against X; sets *flag if any > tol
void launch_berr(bool cplx, const double* y, int64_t yim, int64_t ldy, int64_t nrows, const double* X, int64_t ldx,
                 int64_t n, int nrhs, const unsigned long long* normA, double tol, double* berr, int* flag,
                 cudaStream_t st);
void launch_spmv(bool cplx, const SpmvArgs& a, int nrows_tiles, cudaStream_t st);

}  // namespace ddk
