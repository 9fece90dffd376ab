// f3 / f2 helpers of the partial (Schur-mode) block LDL^T.
//
// PAPER.md:27 (§II): the arrowhead system "is then reduced in size by eliminating via many
// independent sparse direct factorizations the primal DoFs" -- after the partial factorization
// the kept (dual) blocks of each subdomain hold its dense Schur contribution
//     S_p = A_bb,p - C_p^T K_p^{-1} C_p,
// which k_schur_export writes out in the clique layout dd_aux_assemble consumes.  PAPER.md:29:
// "the solution of all or a subset of primal unknowns are recovered ... via many smaller size
// sparse forward backward substitutions": the condensation gathers the kept rows of the forward
// sweep into the auxiliary right-hand side (k_schur_gather, fixed order), the recovery scatters
// the auxiliary solution into the kept rows before the backward sweep (k_schur_scatter).
// All three are HBM-bound data movement.
#include <cuda_runtime.h>

#include "launch.hpp"

namespace ddk {

constexpr int XT = 32;  // export tile edge (32 x 32, 256 threads = 32 x 8)

// One CTA per 32x32 output tile of one (member a, member b) sub-block of S_g.  The element
// S_g[ra + r, cb + c] is the (r, c) element of the block A(I_a, I_b) of the updated arena:
//   mode 0: stored as is in the panel of I_b (rows of I_a):  src[r + c * ld]
//   mode 1: stored as A(I_b, I_a) in the panel of I_a:       src[c + r * ld]  (transposed read)
//   mode 2: the diagonal block of I_a (lower triangle valid): r >= c ? src[r + c ld] : src[c + r ld]
//   mode 3: no such block in the filled pattern -> 0
// Transposed reads go through a 32 x 33 shared tile so both the read and the write are coalesced.
template <bool C>
__global__ void __launch_bounds__(256) k_schur_export(SchurExportArgs a) {
  __shared__ double tr[XT][XT + 1], ti[XT][XT + 1];
  const SxTile T = a.tiles[blockIdx.x];
  const SxItem it = a.items[T.item];
  const int tx = threadIdx.x % XT, ty = threadIdx.x / XT;
  const double* src = a.arena + it.src;
  const int64_t base = a.soff[it.group] + it.dst;
  const int nr = min(XT, it.rows - T.r0), nc = min(XT, it.cols - T.c0);
  // mode 2: tiles strictly above the diagonal read the mirrored tile; the diagonal tile mixes
  const bool trans = it.mode == 1 || (it.mode == 2 && T.r0 < T.c0);
  if (trans) {  // stage the source tile rows (c0 + c) x cols (r0 + r) of the stored block, coalesced in c
    for (int q = ty; q < XT; q += 8) {  // q = r (source column)
      const int r = q, c = tx;
      double vr = 0.0, vi = 0.0;
      if (r < nr && c < nc) {
        const int64_t e = (int64_t)(T.c0 + c) + (int64_t)(T.r0 + r) * it.ld;
        vr = src[e];
        if (C) vi = src[e + a.aim];
      }
      tr[c][r] = vr;
      ti[c][r] = vi;
    }
    __syncthreads();
  }
  for (int q = ty; q < XT; q += 8) {  // q = c (output column), tx = r (output row): coalesced store
    const int r = tx, c = q;
    if (r >= nr || c >= nc) continue;
    double vr = 0.0, vi = 0.0;
    if (it.mode == 3) {
    } else if (trans) {
      vr = tr[c][r];
      vi = ti[c][r];
    } else {
      int64_t e;
      if (it.mode == 2 && T.r0 + r < T.c0 + c) e = (int64_t)(T.c0 + c) + (int64_t)(T.r0 + r) * it.ld;  // diagonal tile, upper
      else e = (int64_t)(T.r0 + r) + (int64_t)(T.c0 + c) * it.ld;
      vr = src[e];
      if (C) vi = src[e + a.aim];
    }
    const int64_t o = base + (int64_t)(T.r0 + r) + (int64_t)(T.c0 + c) * it.m;
    if (C) {
      a.S[2 * o] = vr;
      a.S[2 * o + 1] = vi;
    } else {
      a.S[o] = vr;
    }
  }
}

// Condensation: G[aux rows of I] += sum over the kept copies of I (ascending position) of their
// forward-sweep rows -- one CTA per (aux block, column), fixed order, no atomics.
template <bool C>
__global__ void k_schur_gather(SchurVecArgs a) {
  const SgItem it = a.items[blockIdx.x];
  for (int c = blockIdx.y; c < a.nrhs; c += gridDim.y) {
    for (int m = threadIdx.x; m < it.s; m += blockDim.x) {
      const int64_t g = it.aux_row + m + (int64_t)c * a.ldg;
      double re = C ? a.G[2 * g] : a.G[g], im = C ? a.G[2 * g + 1] : 0.0;
      for (int q = it.c0; q < it.c1; ++q) {
        const int64_t e = a.nd[a.contrib[q]].ydof + m + (int64_t)c * a.ldy;
        re += a.y[e];
        if (C) im += a.y[e + a.yim];
      }
      if (C) {
        a.G[2 * g] = re;
        a.G[2 * g + 1] = im;
      } else {
        a.G[g] = re;
      }
    }
  }
}

// Recovery: the kept rows of node t (item = its kept position in c0) <- x_b rows of its target.
template <bool C>
__global__ void k_schur_scatter(SchurVecArgs a) {
  const SgItem it = a.items[blockIdx.x];
  const int64_t yrow = a.nd[it.c0].ydof;
  for (int c = blockIdx.y; c < a.nrhs; c += gridDim.y)
    for (int m = threadIdx.x; m < it.s; m += blockDim.x) {
      const int64_t g = it.aux_row + m + (int64_t)c * a.ldg;
      const int64_t e = yrow + m + (int64_t)c * a.ldy;
      a.y[e] = C ? a.G[2 * g] : a.G[g];
      if (C) a.y[e + a.yim] = a.G[2 * g + 1];
    }
}

void launch_schur_export(bool cplx, const SchurExportArgs& a, int ntiles, cudaStream_t st) {
  if (ntiles == 0) return;
  if (cplx) k_schur_export<true><<<ntiles, 256, 0, st>>>(a);
  else k_schur_export<false><<<ntiles, 256, 0, st>>>(a);
}

void launch_schur_gather(bool cplx, const SchurVecArgs& a, int nitems, cudaStream_t st) {
  if (nitems == 0 || a.nrhs == 0) return;
  dim3 grid(nitems, a.nrhs < 1024 ? a.nrhs : 1024);
  if (cplx) k_schur_gather<true><<<grid, 128, 0, st>>>(a);
  else k_schur_gather<false><<<grid, 128, 0, st>>>(a);
}

void launch_schur_scatter(bool cplx, const SchurVecArgs& a, int nitems, cudaStream_t st) {
  if (nitems == 0 || a.nrhs == 0) return;
  dim3 grid(nitems, a.nrhs < 1024 ? a.nrhs : 1024);
  if (cplx) k_schur_scatter<true><<<grid, 128, 0, st>>>(a);
  else k_schur_scatter<false><<<grid, 128, 0, st>>>(a);
}

}  // namespace ddk
