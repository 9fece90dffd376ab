// Device data layout and descriptor tables (host- and device-visible PODs).
//
// HBM layout of the factor: supernodal panel storage
// in elimination-position order.  Panel t is one dense column-major
// (ld_t x s_t) matrix whose rows are [diagonal block t | struct(t) members in
// position order]; every row segment starts at an even row (16-byte aligned
// cp.async chunks) and ld_t is a multiple of 8 elements.  Complex values are
// planar: the imaginary plane of every buffer lives at a fixed element offset.
#pragma once
#include <cstdint>

namespace ddaux {

constexpr int TB = 32;     // diagonal-tile size of the precomputed L_kk^{-1} tiles (TRSM via GEMM)
constexpr int K1NB = 32;      // panel width of the blocked in-block Bunch-Kaufman (dlasyf-style)
constexpr int K1NB_MAX = 64;  // widest K1 panel (real blocks small enough for a 64-column smem panel)

inline int64_t pad2(int64_t x) { return (x + 1) & ~int64_t(1); }
inline int64_t pad8(int64_t x) { return (x + 7) & ~int64_t(7); }

struct NodeDev {     // one per elimination position t (64-byte aligned record)
  int64_t panel;     // element offset of panel t in the arena (re plane)
  int64_t linv;      // element offset of its TB x TB inverse diagonal tiles
  int64_t w;         // element offset of W_t = A_struct,t L_tt^{-T} in the level workspace
  int64_t k1w;       // element offset of the K1 (dlasyf) scratch in the level workspace
  int64_t ydof;      // row offset in position order (padded): y vectors and per-DoF arrays
  int64_t odof;      // original DoF offset of the block
  int32_t s, sp;     // size and pad2(size)
  int32_t rp, ld;    // padded struct rows; panel leading dimension
  int32_t ldw, nst;  // W leading dimension; |struct(t)|
  int32_t st0, blk;  // first index into the struct arrays; original block id
  int64_t inv;       // element offset of the full inverse L_tt^{-1} (s x s, lower, ld = ldi)
  int32_t ldi, pad;
};

struct DTile {       // diagonal-solve / inverse work item: node t, tile index, level buffer offset
  int32_t t, tm;
  int64_t toff;      // row offset of node t in the level buffer T
};

struct UpdTarget {   // Schur-update target block (i, j), i at/after j, stored in panel j
  int32_t j, ro;     // panel node; row offset of block i in panel j (0 for the diagonal)
  int32_t M, N;      // s_i, s_j
  int32_t c0, c1;    // contributor range
  int32_t diag, pad;
};

struct UpdContrib {  // contributor k of a target: A = W_k rows arow.., B = panel_k rows brow..
  int32_t k, arow, brow, pad;
};

struct Tile {        // one output tile of a target (tm, tn in tile units)
  int32_t target, tm, tn, pad;
};

struct Strip {       // K2 row strip of panel t's struct rows [row0, row0 + nrows)
  int32_t t, row0, nrows, pad;
};

struct RowPerm {     // row block of node t inside an earlier panel k (rows ro..ro+s_t)
  int32_t t, k, ro, pad;
};

struct SolveTarget {  // forward solve: y_i -= sum_k L_ik z_k (contributors k of one level)
  int32_t i, tm, c0, c1;
};

struct SolveContrib {  // contributor: L_ik = panel_k rows ro..
  int32_t k, ro;
};

struct SpSeg {       // K6 residual: block row I of the full symmetric A, one stored block
  int64_t voff;      // element offset into d_vals (caller's layout)
  int32_t J, mode;   // column block; 0 = stored (I,J), 1 = stored (J,I) used transposed, 2 = diagonal
};

struct SpRow {       // K6: block row I, row tile tm, segment range
  int32_t I, tm, c0, c1;
};

}  // namespace ddaux
