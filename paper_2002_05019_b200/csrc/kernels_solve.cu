// Solve-phase kernels (sm_100a).  PAPER.md:29 (§II) "Once the auxiliary problem has been
// efficiently factorized" it is solved by forward/backward substitution for many
// excitations (Fig. 2c "200 excitations"); SURVEY.md §8(a) a7, a8.
//
//   y = P b              k_perm_in     (block order + in-block pivots, planar complex)
//   forward, per level:  k_fdiag       z_t = L_tt^{-1} y_t   (TB-tile inverses -> DMMA GEMMs)
//                        k_fupd        y_i -= sum_k L_ik z_k (owner-computes, gathered K)
//   y = D^{-1} y         k_dsolve      (1x1 / 2x2 closed form)
//   backward, per level: k_bupd        y_t -= sum_i L_it^T y_i   (pull, conflict-free)
//                        k_bdiag       y_t = L_tt^{-T} y_t
//   x = P^T y            k_perm_out    (store, or accumulate a refinement correction)
//   r = b - A x          k_spmv        (refinement residual over the ORIGINAL blocks, L7)
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "gemm_core.cuh"
#include "launch.hpp"

using namespace ddaux;

namespace ddk {

// Solve GEMM configurations: 64-row tiles; rhs tile 64 (real) / 32 (complex, so the 3M form's
// three accumulator sets fit at 4 CTAs per SM).  Real: per-warp masking; complex: per-sub-tile.
constexpr int SUBM = 64;
constexpr int BUPD_MAX_PARTS = 1024;  // split-K partial tiles of the backward update (workspace bound)
template <bool C>
struct SolveN {
  static constexpr int value = C ? 32 : 64;
};
#ifndef DDK_SOLVE_STAGES_REAL
#define DDK_SOLVE_STAGES_REAL 2
#endif
#ifndef DDK_SOLVE_RED
#define DDK_SOLVE_RED 1
#endif
template <bool C, bool M3>
struct SolveG {
  static constexpr int BN = SolveN<C>::value;
  static constexpr int ST = C ? 2 : DDK_SOLVE_STAGES_REAL;
#ifndef DDK_SOLVE_FAST_C
#define DDK_SOLVE_FAST_C 1
#endif
  static constexpr bool FAST = !C || DDK_SOLVE_FAST_C;  // fast loader (A/B switch for the complex kernels)
  using FU = Gemm<SUBM, BN, 16, 2, 2, ST, C, false, true, C && M3, C, false, false, false, FAST>;  // MK x KN (FINE = C)
  using BU = Gemm<SUBM, BN, 16, 2, 2, ST, C, true, true, C && M3, C, false, false, false, FAST>;   // KM x KN
};

// ---------------------------------------------------------------------------- permutations
template <bool C>
__global__ void k_perm_in(PermArgs a) {
  const int c = blockIdx.y;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < a.nrows; g += (int64_t)gridDim.x * blockDim.x) {
    const int o = a.gperm[g];
    double re = 0.0, im = 0.0;
    if (o >= 0 && (a.rowlim == 0 || g < a.rowlim)) {
      int64_t e = (int64_t)o + (int64_t)c * a.lds;
      if (C) {
        re = a.src[2 * e];
        im = a.src[2 * e + 1];
      } else {
        re = a.src[e];
      }
    }
    int64_t d = g + (int64_t)c * a.ldy;
    a.y[d] = re;
    if (C) a.y[d + a.yim] = im;
  }
}

template <bool C>
__global__ void k_perm_out(PermArgs a) {
  if (a.flag && *a.flag == 0) return;
  const int c = blockIdx.y;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < a.nrows; g += (int64_t)gridDim.x * blockDim.x) {
    const int o = a.gperm[g];
    if (o < 0) continue;
    int64_t s = g + (int64_t)c * a.ldy;
    int64_t e = (int64_t)o + (int64_t)c * a.ldd;
    if (C) {
      double re = a.y[s], im = a.y[s + a.yim];
      if (a.accumulate) {
        a.dst[2 * e] += re;
        a.dst[2 * e + 1] += im;
      } else {
        a.dst[2 * e] = re;
        a.dst[2 * e + 1] = im;
      }
    } else {
      if (a.accumulate) a.dst[e] += a.y[s];
      else a.dst[e] = a.y[s];
    }
  }
}

__global__ void k_copy(const double* __restrict__ src, int64_t lds, double* __restrict__ dst, int64_t ldd,
                       int64_t n, int w) {
  const int c = blockIdx.y;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n * w; r += (int64_t)gridDim.x * blockDim.x)
    dst[r + (int64_t)c * ldd * w] = src[r + (int64_t)c * lds * w];
}

// ---------------------------------------------------------------------------- diagonal solves (GEMM)
// z_t = L_tt^{-1} y_t (forward) or z_t = L_tt^{-T} y_t (backward) with the precomputed full
// inverse (k_linv): CTA (node, 64-row tile) x (64-rhs tile), K restricted to the triangle;
// results go to the level buffer T, then k_dcopy moves them back into y (no in-place hazard).
template <bool C, bool BWD, bool M3>
__global__ void __launch_bounds__(128, M3 ? 3 : 4) k_diag_g(SolveArgs a) {
  if (a.flag && *a.flag == 0) return;
  using G = typename std::conditional<BWD, typename SolveG<C, M3>::BU, typename SolveG<C, M3>::FU>::type;
  constexpr int SBN = SolveN<C>::value;
  extern __shared__ __align__(16) double smem[];
  const DTile D = a.dtiles[blockIdx.x];
  const NodeDev nd = a.nd[D.t];
  const int s = nd.s, m0 = D.tm * SUBM, n0 = blockIdx.y * SBN;
  const double* X = a.arena + nd.inv;
  Seg sg;
  if (!BWD) {  // A(m, k) = X(m0 + m, k), k < min(s, m0 + SUBM)   (MK)
    sg = Seg{X + m0, a.y + nd.ydof, nullptr, (int64_t)nd.ldi, a.ldy, min(s, m0 + SUBM)};
  } else {     // A(m, k') = X(m0 + k', m0 + m), k' < s - m0          (KM)
    sg = Seg{X + m0 + (int64_t)m0 * nd.ldi, a.y + nd.ydof + m0, nullptr, (int64_t)nd.ldi, a.ldy, s - m0};
  }
  typename G::Acc acc;
  G::zero(acc);
  G::run([&](int) { return sg; }, 1, 0, n0, s - m0, a.nrhs, a.aim, a.yim, smem, acc,
         G::tile_mask(s - m0, a.nrhs - n0, G::NO_DIAG));
  G::template store_tile<0>(acc, smem, a.T + D.toff + m0 + (int64_t)n0 * a.ldT, a.ldT, a.Tim, s - m0, a.nrhs - n0);
}

template <bool C>
__global__ void k_dcopy(SolveArgs a, int ntiles) {
  if (a.flag && *a.flag == 0) return;
  const int c = blockIdx.y;
  for (int q = blockIdx.x; q < ntiles; q += gridDim.x) {
    const DTile D = a.dtiles[q];
    const NodeDev nd = a.nd[D.t];
    const int m0 = D.tm * SUBM, m1 = min(nd.s, m0 + SUBM);
    for (int r = m0 + threadIdx.x; r < m1; r += blockDim.x) {
      const int64_t src = D.toff + r + (int64_t)c * a.ldT, dst = nd.ydof + r + (int64_t)c * a.ldy;
      a.y[dst] = a.T[src];
      if (C) a.y[dst + a.yim] = a.T[src + a.Tim];
    }
  }
}

// ---------------------------------------------------------------------------- level updates
template <bool C, bool M3>
__global__ void __launch_bounds__(128, M3 ? 3 : 4) k_fupd(SolveArgs a) {
  if (a.flag && *a.flag == 0) return;
  using G = typename SolveG<C, M3>::FU;
  constexpr int SBN = SolveN<C>::value;
  extern __shared__ __align__(16) double smem[];
  const SolveTarget T = a.ftargets[blockIdx.x];
  const NodeDev ni = a.nd[T.i];
  const int n0 = blockIdx.y * SBN, m0 = T.tm * SUBM;
  typename G::Acc acc;
  G::zero(acc);
  const SolveContrib* cl = a.fcontribs + T.c0;
  auto segfn = [&](int q) {
    const SolveContrib u = cl[q];
    const NodeDev nk = a.nd[u.k];
    Seg sg{a.arena + nk.panel + u.ro, a.y + nk.ydof, nullptr, (int64_t)nk.ld, a.ldy, nk.s};
    return sg;
  };
  G::run(segfn, T.c1 - T.c0, m0, n0, ni.s, a.nrhs, a.aim, a.yim, smem, acc,
         G::tile_mask(ni.s - m0, a.nrhs - n0, G::NO_DIAG));
  // y_i -= acc as L2 reductions: one reduction per element and launch (owner-computes tiles), so
  // the result is order-independent and bitwise the read-modify-write one (gemm_core.cuh MODE 2)
  G::template store_tile<DDK_SOLVE_RED ? 2 : 1>(acc, smem, a.y + ni.ydof + m0 + (int64_t)n0 * a.ldy, a.ldy, a.yim,
                                                 ni.s - m0, a.nrhs - n0);
}

// Backward pull update y_t -= sum_{i in struct(t)} L_it^T y_i.  With split-K (G > 1) CTA
// (tile, g) sums the g-th contiguous chunk of struct(t) into a partial buffer and
// k_bupd_reduce subtracts the G partials in fixed order g = 0..G-1 (deterministic).
// CL (thread-block cluster of the G chunk CTAs of one tile, G <= 8): the partial tiles are reduced
// through distributed shared memory in the same fixed order g = 0..G-1 (bitwise the same result
// as the two-kernel partial-buffer path, without its HBM round trip and second launch).
template <bool C, bool M3, bool CL, bool FOLD = false>
__global__ void __launch_bounds__(128, M3 ? 3 : 4) k_bupd(SolveArgs a, int G, double* part, int64_t pim) {
  if (a.flag && *a.flag == 0) return;
  using G_ = typename SolveG<C, M3>::BU;
  constexpr int SBN = SolveN<C>::value;
  extern __shared__ __align__(16) double smem[];
  const int tile = blockIdx.x / G, g = blockIdx.x % G;
  const int2 T = a.btiles[tile];  // (t, tm)
  const NodeDev nt = a.nd[T.x];
  const int n0 = blockIdx.y * SBN, m0 = T.y * SUBM;
  // chunk g = padded struct rows [R0, R1) (even bounds: 16-byte cp.async chunks), split inside
  // members so every chunk carries the same K; members qa..qb intersect it
  const int R0 = (int)((int64_t)nt.rp * g / G) & ~1;
  const int R1 = g == G - 1 ? nt.rp : ((int)((int64_t)nt.rp * (g + 1) / G) & ~1);
  auto member_of = [&](int r) {  // last member q with (st_row[q] - sp) <= r
    int lo = 0, hi = nt.nst - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (a.st_row[nt.st0 + mid] - nt.sp <= r) lo = mid;
      else hi = mid - 1;
    }
    return lo;
  };
  const int qa = R1 > R0 ? member_of(R0) : 0, qb = R1 > R0 ? member_of(R1 - 1) : -1;
  typename G_::Acc acc;
  G_::zero(acc);
  auto segfn = [&](int q) {
    const int ipos = a.st_pos[nt.st0 + qa + q];
    const int ro = a.st_row[nt.st0 + qa + q];
    const NodeDev ni = a.nd[ipos];
    const int o = ro - nt.sp;
    const int lo = max(0, R0 - o), hi = min(ni.s, R1 - o);
    // A(m, k) = L_it(lo + k, m) = panel_t[(ro + lo + k) + m*ld]  (KM)
    Seg sg{a.arena + nt.panel + ro + lo, a.y + ni.ydof + lo, nullptr, (int64_t)nt.ld, a.ldy, max(0, hi - lo)};
    return sg;
  };
  G_::run(segfn, qb - qa + 1, m0, n0, nt.s, a.nrhs, a.aim, a.yim, smem, acc,
          G_::tile_mask(nt.s - m0, a.nrhs - n0, G_::NO_DIAG));
  if (G == 1) {
    G_::template store_tile<DDK_SOLVE_RED ? 2 : 1>(acc, smem, a.y + nt.ydof + m0 + (int64_t)n0 * a.ldy, a.ldy, a.yim,
                                                    nt.s - m0, a.nrhs - n0);
  } else if constexpr (CL) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    constexpr int E = SUBM * SBN;
    double* Pr = smem;      // this CTA's partial tile, SUBM x SBN, ld SUBM (pipeline smem is idle)
    double* Pi = smem + E;
    G_::for_each(acc, [&](int r, int c, double vr, double vi) {
      Pr[r + c * SUBM] = vr;
      if (C) Pi[r + c * SUBM] = vi;
    });
    cl.sync();
    const int e0 = (int)((int64_t)E * g / G), e1 = (int)((int64_t)E * (g + 1) / G);
    for (int e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
      const int r = e % SUBM, c = e / SUBM;
      if (m0 + r >= nt.s || n0 + c >= a.nrhs) continue;
      double sr = 0.0, si = 0.0;
      for (int h = 0; h < G; ++h) {
        sr += cl.map_shared_rank(Pr, h)[e];
        if (C) si += cl.map_shared_rank(Pi, h)[e];
      }
      const int64_t o = nt.ydof + (int64_t)(m0 + r) + (int64_t)(n0 + c) * a.ldy;
      a.y[o] -= sr;
      if (C) a.y[o + a.yim] -= si;
    }
    cl.sync();  // the partial tiles stay alive until every remote read is done
  } else {
    double* P = part + (int64_t)blockIdx.x * SUBM * a.nrhs;  // SUBM x nrhs, ld SUBM
    G_::for_each(acc, [&](int r, int c, double vr, double vi) {
      if (n0 + c < a.nrhs) {
        int64_t e = (int64_t)r + (int64_t)(n0 + c) * SUBM;
        P[e] = vr;
        if (C) P[e + pim] = vi;
      }
    });
    if constexpr (FOLD) {
      // the last of the G chunk CTAs of this (tile, rhs tile) to finish reduces the partials in the
      // fixed order g = 0..G-1 (bitwise the sums of k_bupd_reduce, without its second launch)
      __shared__ int s_last;
      __threadfence();
      __syncthreads();
      int* cnt = a.cnt + (int64_t)tile * gridDim.y + blockIdx.y;
      if (threadIdx.x == 0) s_last = atomicAdd(cnt, 1) == G - 1;
      __syncthreads();
      if (!s_last) return;
      __threadfence();
      for (int e = threadIdx.x; e < SUBM * SBN; e += blockDim.x) {
        const int r = e % SUBM, c = e / SUBM;
        if (m0 + r >= nt.s || n0 + c >= a.nrhs) continue;
        const int64_t pe = (int64_t)r + (int64_t)(n0 + c) * SUBM;
        double sr = 0.0, si = 0.0;
        for (int h0 = 0; h0 < G; h0 += 8) {  // 8 partials in flight, added in the order h = 0..G-1
          double vr[8], vi[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const double* Q = part + (int64_t)(tile * G + min(h0 + u, G - 1)) * SUBM * a.nrhs;
            vr[u] = __ldcg(Q + pe);
            vi[u] = C ? __ldcg(Q + pe + pim) : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (h0 + u < G) {
              sr += vr[u];
              if (C) si += vi[u];
            }
        }
        const int64_t o = nt.ydof + (int64_t)(m0 + r) + (int64_t)(n0 + c) * a.ldy;
        a.y[o] -= sr;
        if (C) a.y[o + a.yim] -= si;
      }
      if (threadIdx.x == 0) *cnt = 0;  // ready for the next launch
    }
  }
}

template <bool C>
__global__ void k_bupd_reduce(SolveArgs a, int G, const double* __restrict__ part, int64_t pim) {
  if (a.flag && *a.flag == 0) return;
  const int tile = blockIdx.x;
  const int2 T = a.btiles[tile];
  const NodeDev nt = a.nd[T.x];
  const int m0 = T.y * SUBM;
  for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < SUBM * a.nrhs; e += gridDim.y * blockDim.x) {
    const int r = e % SUBM, c = e / SUBM;
    if (m0 + r >= nt.s) continue;
    double sr = 0.0, si = 0.0;
    for (int g = 0; g < G; ++g) {
      const double* P = part + (int64_t)(tile * G + g) * SUBM * a.nrhs;
      sr += P[e];
      if (C) si += P[e + pim];
    }
    int64_t o = nt.ydof + (int64_t)(m0 + r) + (int64_t)c * a.ldy;
    a.y[o] -= sr;
    if (C) a.y[o + a.yim] -= si;
  }
}

// ---------------------------------------------------------------------------- D solve
template <bool C>
__global__ void k_dsolve(SolveArgs a) {
  if (a.flag && *a.flag == 0) return;
  const int c = blockIdx.y;
  const double* dv_ = a.arena + a.d_off;
  const double* ev_ = a.arena + a.e_off;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < a.nrows; g += (int64_t)gridDim.x * blockDim.x) {
    const int pv = a.ipiv[g];
    if (pv == 0) continue;  // padding row
    int64_t e = g + (int64_t)c * a.ldy;
    if (pv > 0) {
      cz d = ld<C>(dv_, g, a.aim);
      if (d.r == 0.0 && d.i == 0.0) continue;
      st<C>(a.y, e, a.yim, dv<C>(ld<C>(a.y, e, a.yim), d));
    } else {
      cz ee = ld<C>(ev_, g, a.aim);
      if (ee.r == 0.0 && ee.i == 0.0) continue;  // second row of a pair: handled by the first
      cz d1 = ld<C>(dv_, g, a.aim), d2 = ld<C>(dv_, g + 1, a.aim);
      cz y1 = ld<C>(a.y, e, a.yim), y2 = ld<C>(a.y, e + 1, a.yim);
      // LAPACK xSYTRS scaled closed form
      cz akm1 = dv<C>(d1, ee), ak = dv<C>(d2, ee);
      cz den = mul<C>(akm1, ak) - mk(1.0, 0.0);
      cz bkm1 = dv<C>(y1, ee), bk = dv<C>(y2, ee);
      st<C>(a.y, e, a.yim, dv<C>(mul<C>(ak, bkm1) - bk, den));
      st<C>(a.y, e + 1, a.yim, dv<C>(mul<C>(akm1, bk) - bkm1, den));
    }
  }
}

// ---------------------------------------------------------------------------- residual SpMV
// R = Bsave - A X over the caller's original blocks (both triangles), SIMT FP64, written
// permuted into y.  CTA tile: 64 rows x 32 rhs; 256 threads, 4 x 2 outputs each.
constexpr int SPM = 64, SPN = 32, SPK = 16;
template <bool C>
__global__ void __launch_bounds__(256) k_spmv(SpmvArgs a) {
  __shared__ double Ar[SPK][SPM + 1], Ai[C ? SPK : 1][C ? SPM + 1 : 1];
  __shared__ double Xr[SPK][SPN + 1], Xi[C ? SPK : 1][C ? SPN + 1 : 1];
  const SpRow R = a.rows[blockIdx.x];
  const int I = R.I;
  const int sI = (int)a.blk_size[I];
  const int m0 = R.tm * SPM, n0 = blockIdx.y * SPN;
  const int tid = threadIdx.x;
  const int tr = tid % 16, tc = tid / 16;  // rows tr*4.., cols tc*2..
  double accr[4][2] = {}, acci[4][2] = {};
  for (int q = R.c0; q < R.c1; ++q) {
    const SpSeg sg = a.segs[q];
    const int sJ = (int)a.blk_size[sg.J];
    const int64_t oJ = a.odof[sg.J];
    for (int k0 = 0; k0 < sJ; k0 += SPK) {
      __syncthreads();
      for (int e = tid; e < SPM * SPK; e += 256) {
        int m = e % SPM, k = e / SPM;
        int gm = m0 + m, gk = k0 + k;
        double vr = 0.0, vi = 0.0;
        if (gm < sI && gk < sJ) {
          int64_t idx;
          if (sg.mode == 0) idx = gm + (int64_t)gk * sI;           // stored (I,J): s_I x s_J
          else if (sg.mode == 1) idx = gk + (int64_t)gm * sJ;      // stored (J,I): s_J x s_I, transposed
          else idx = gm >= gk ? gm + (int64_t)gk * sI : gk + (int64_t)gm * sI;  // diagonal, lower triangle
          idx += sg.voff;
          if (C) {
            vr = a.vals[2 * idx];
            vi = a.vals[2 * idx + 1];
          } else {
            vr = a.vals[idx];
          }
        }
        Ar[k][m] = vr;
        if (C) Ai[k][m] = vi;
      }
      for (int e = tid; e < SPK * SPN; e += 256) {
        int k = e % SPK, n = e / SPK;
        int gk = k0 + k, gn = n0 + n;
        double vr = 0.0, vi = 0.0;
        if (gk < sJ && gn < a.nrhs) {
          int64_t idx = oJ + gk + (int64_t)gn * a.ldx;
          if (C) {
            vr = a.X[2 * idx];
            vi = a.X[2 * idx + 1];
          } else {
            vr = a.X[idx];
          }
        }
        Xr[k][n] = vr;
        if (C) Xi[k][n] = vi;
      }
      __syncthreads();
#pragma unroll 4
      for (int k = 0; k < SPK; ++k) {
        double ar[4], ai[4], xr[2], xi[2];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          ar[u] = Ar[k][tr * 4 + u];
          if (C) ai[u] = Ai[k][tr * 4 + u];
        }
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          xr[v] = Xr[k][tc * 2 + v];
          if (C) xi[v] = Xi[k][tc * 2 + v];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            accr[u][v] = fma(ar[u], xr[v], accr[u][v]);
            if (C) {
              accr[u][v] = fma(-ai[u], xi[v], accr[u][v]);
              acci[u][v] = fma(ar[u], xi[v], acci[u][v]);
              acci[u][v] = fma(ai[u], xr[v], acci[u][v]);
            }
          }
      }
    }
  }
  const int64_t oI = a.odof[I];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      int gm = m0 + tr * 4 + u, gn = n0 + tc * 2 + v;
      if (gm < sI && gn < a.nrhs) {
        int64_t orow = oI + gm;
        int64_t bidx = orow + (int64_t)gn * a.ldb;
        int64_t yidx = (int64_t)a.ginv[orow] + (int64_t)gn * a.ldy;
        if (C) {
          a.y[yidx] = a.Bsave[2 * bidx] - accr[u][v];
          a.y[yidx + a.yim] = a.Bsave[2 * bidx + 1] - acci[u][v];
        } else {
          a.y[yidx] = a.Bsave[bidx] - accr[u][v];
        }
      }
    }
}

// ---------------------------------------------------------------------------- residual SpMV on DMMA
// Same product as k_spmv, on the FP64 tensor pipe: CTA tile 64 rows x 64 rhs, K = the columns of
// every stored block of block-row I (ascending J, fixed order).  The caller's blocks are read
// element-wise (interleaved complex at arbitrary offsets, so no 16-byte cp.async chunks): each
// thread gathers its 8 A and 8 B elements of the next K-chunk into registers while the DMMAs
// of the current chunk run, then stores them into the engine's MK / KN shared-memory tiles.
using SpG_R = Gemm<64, 64, 16, 2, 2, 2, false, false, true>;
using SpG_C = Gemm<64, 64, 16, 2, 2, 2, true, false, true>;
constexpr int SPT_M = 64, SPT_N = 64, SPT_K = 16;

template <bool C>
__global__ void __launch_bounds__(128) k_spmv_dmma(SpmvArgs a) {
  using G = typename std::conditional<C, SpG_C, SpG_R>::type;
  extern __shared__ __align__(16) double smem[];
  const SpRow R = a.rows[blockIdx.x];
  const int I = R.I, sI = (int)a.blk_size[I];
  const int m0 = R.tm * SPT_M, n0 = blockIdx.y * SPT_N;
  const int tid = threadIdx.x;
  constexpr int PER = SPT_M * SPT_K / 128;  // 8 elements of A and of B per thread per chunk
  double ra[PER], ia[PER], rb[PER], ib[PER];
  // chunk iterator over (segment, k0)
  int q = R.c0, k0 = 0;
  auto fetch = [&](int qq, int kk0) {
    const SpSeg sg = a.segs[qq];
    const int sJ = (int)a.blk_size[sg.J];
    const int64_t oJ = a.odof[sg.J];
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int e = tid + u * 128;
      // A(m, k): m fastest for stored / diagonal blocks, k fastest for transposed ones (coalescing)
      int m, k;
      if (sg.mode == 1) {
        k = e % SPT_K;
        m = e / SPT_K;
      } else {
        m = e % SPT_M;
        k = e / SPT_M;
      }
      const int gm = m0 + m, gk = kk0 + k;
      double vr = 0.0, vi = 0.0;
      if (gm < sI && gk < sJ) {
        int64_t idx;
        if (sg.mode == 0) idx = gm + (int64_t)gk * sI;
        else if (sg.mode == 1) idx = gk + (int64_t)gm * sJ;
        else idx = gm >= gk ? gm + (int64_t)gk * sI : gk + (int64_t)gm * sI;
        idx += sg.voff;
        if (C) {
          vr = a.vals[2 * idx];
          vi = a.vals[2 * idx + 1];
        } else {
          vr = a.vals[idx];
        }
      }
      ra[u] = vr;
      ia[u] = vi;
      // B(k, n) = X(oJ + k, n): k fastest
      const int kb = e % SPT_K, nb = e / SPT_K;
      const int gkb = kk0 + kb, gn = n0 + nb;
      double wr = 0.0, wi = 0.0;
      if (gkb < sJ && gn < a.nrhs) {
        int64_t idx = oJ + gkb + (int64_t)gn * a.ldx;
        if (C) {
          wr = a.X[2 * idx];
          wi = a.X[2 * idx + 1];
        } else {
          wr = a.X[idx];
        }
      }
      rb[u] = wr;
      ib[u] = wi;
    }
  };
  auto store = [&](double* st, int mode) {
    double* As = st;
    double* Bs = st + G::NPL * G::A_TILE;
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int e = tid + u * 128;
      int m, k;
      if (mode == 1) {
        k = e % SPT_K;
        m = e / SPT_K;
      } else {
        m = e % SPT_M;
        k = e / SPT_M;
      }
      As[k * G::A_LD + m] = ra[u];
      if (C) As[G::A_TILE + k * G::A_LD + m] = ia[u];
      const int kb = e % SPT_K, nb = e / SPT_K;
      Bs[nb * G::B_LD + kb] = rb[u];
      if (C) Bs[G::B_TILE + nb * G::B_LD + kb] = ib[u];
    }
  };
  typename G::Acc acc;
  G::zero(acc);
  if (q < R.c1) {
    fetch(q, k0);
    int buf = 0;
    for (;;) {
      const int mode = a.segs[q].mode;
      store(smem + buf * G::STAGE, mode);
      __syncthreads();
      // advance and prefetch the next chunk into registers
      const int sJ = (int)a.blk_size[a.segs[q].J];
      k0 += SPT_K;
      if (k0 >= sJ) {
        k0 = 0;
        ++q;
      }
      const bool more = q < R.c1;
      if (more) fetch(q, k0);
      G::compute_stage(smem + buf * G::STAGE, acc);
      buf ^= 1;
      if (!more) break;
    }
  }
  const int64_t oI = a.odof[I];
  G::for_each(acc, [&](int r, int c, double vr, double vi) {
    const int gm = m0 + r, gn = n0 + c;
    if (gm < sI && gn < a.nrhs) {
      const int64_t orow = oI + gm;
      const int64_t bidx = orow + (int64_t)gn * a.ldb;
      const int64_t yidx = (int64_t)a.ginv[orow] + (int64_t)gn * a.ldy;
      if (C) {
        a.y[yidx] = a.Bsave[2 * bidx] - vr;
        a.y[yidx + a.yim] = a.Bsave[2 * bidx + 1] - vi;
      } else {
        a.y[yidx] = a.Bsave[bidx] - vr;
      }
    }
  });
}

// ---------------------------------------------------------------------------- ||A||_inf, berr
template <bool C>
__global__ void k_norm_a(SpmvArgs a, unsigned long long* out) {
  __shared__ double red[256];
  const SpRow R = a.rows[blockIdx.x];
  const int I = R.I, sI = (int)a.blk_size[I];
  double best = 0.0;
  for (int m = R.tm * SPM + threadIdx.x; m < min(sI, (R.tm + 1) * SPM); m += blockDim.x) {
    double acc = 0.0;  // row sum of moduli over every block of block-row I (fixed order)
    for (int q = R.c0; q < R.c1; ++q) {
      const SpSeg sg = a.segs[q];
      const int sJ = (int)a.blk_size[sg.J];
      for (int k = 0; k < sJ; ++k) {
        int64_t idx;
        if (sg.mode == 0) idx = m + (int64_t)k * sI;
        else if (sg.mode == 1) idx = k + (int64_t)m * sJ;
        else idx = m >= k ? m + (int64_t)k * sI : k + (int64_t)m * sI;
        idx += sg.voff;
        acc += C ? hypot(a.vals[2 * idx], a.vals[2 * idx + 1]) : fabs(a.vals[idx]);
      }
    }
    best = fmax(best, acc);
  }
  red[threadIdx.x] = best;
  __syncthreads();
  for (int o = blockDim.x / 2; o; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) atomicMax(out, (unsigned long long)__double_as_longlong(red[0]));  // >= 0: bit order == value order
}

template <bool C>
__global__ void k_berr(const double* __restrict__ y, int64_t yim, int64_t ldy, int64_t nrows,
                       const double* __restrict__ X, int64_t ldx, int64_t n, const unsigned long long* normA,
                       double tol, double* berr, int* flag) {
  __shared__ double rr[256], rx[256];
  const int c = blockIdx.x;
  double mr = 0.0, mx = 0.0;
  for (int64_t g = threadIdx.x; g < nrows; g += blockDim.x) {
    int64_t e = g + (int64_t)c * ldy;
    mr = fmax(mr, C ? hypot(y[e], y[e + yim]) : fabs(y[e]));
  }
  for (int64_t g = threadIdx.x; g < n; g += blockDim.x) {
    int64_t e = g + (int64_t)c * ldx;
    mx = fmax(mx, C ? hypot(X[2 * e], X[2 * e + 1]) : fabs(X[e]));
  }
  rr[threadIdx.x] = mr;
  rx[threadIdx.x] = mx;
  __syncthreads();
  for (int o = blockDim.x / 2; o; o >>= 1) {
    if (threadIdx.x < o) {
      rr[threadIdx.x] = fmax(rr[threadIdx.x], rr[threadIdx.x + o]);
      rx[threadIdx.x] = fmax(rx[threadIdx.x], rx[threadIdx.x + o]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double na = __longlong_as_double((long long)*normA);
    const double den = na * rx[0];
    const double b = den > 0 ? rr[0] / den : (rr[0] > 0 ? INFINITY : 0.0);
    berr[c] = b;
    if (!(b <= tol)) atomicOr(flag, 1);
  }
}

// ---------------------------------------------------------------------------- launchers
template <class K>
static void set_smem(K kern, size_t bytes) {
  if (bytes > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

int solve_bm(bool) { return SUBM; }
size_t bupd_part_bytes(bool cplx, int nrhs) { return (size_t)BUPD_MAX_PARTS * SUBM * nrhs * (cplx ? 2 : 1) * 8; }
size_t bupd_cnt_bytes(bool cplx, int nrhs) {  // one arrival counter per (split tile, rhs tile)
  (void)cplx;
  return (size_t)BUPD_MAX_PARTS * ((nrhs + SolveN<true>::value - 1) / SolveN<true>::value) * sizeof(int);
}
int spmv_bm() { return SPM; }

static dim3 rows_grid(int64_t nrows, int nrhs) {
  int gx = (int)std::min<int64_t>((nrows + 255) / 256, 1024);
  return dim3(gx > 0 ? gx : 1, nrhs);
}

void launch_perm_in(bool cplx, const PermArgs& a, cudaStream_t st) {
  if (a.nrhs == 0) return;
  if (cplx) k_perm_in<true><<<rows_grid(a.nrows, a.nrhs), 256, 0, st>>>(a);
  else k_perm_in<false><<<rows_grid(a.nrows, a.nrhs), 256, 0, st>>>(a);
}
void launch_perm_out(bool cplx, const PermArgs& a, cudaStream_t st) {
  if (a.nrhs == 0) return;
  if (cplx) k_perm_out<true><<<rows_grid(a.nrows, a.nrhs), 256, 0, st>>>(a);
  else k_perm_out<false><<<rows_grid(a.nrows, a.nrhs), 256, 0, st>>>(a);
}
void launch_copy(bool cplx, const double* src, int64_t lds, double* dst, int64_t ldd, int64_t n, int nrhs,
                 cudaStream_t st) {
  if (nrhs == 0) return;
  int w = cplx ? 2 : 1;
  k_copy<<<rows_grid(n * w, nrhs), 256, 0, st>>>(src, lds, dst, ldd, n, w);
}

static int ntn(bool cplx, int nrhs) {
  const int bn = cplx ? SolveN<true>::value : SolveN<false>::value;
  return (nrhs + bn - 1) / bn;
}

template <class K>
static void launch_g(K kern, size_t smem, dim3 grid, cudaStream_t st, const SolveArgs& a) {
  set_smem(kern, smem);
  kern<<<grid, 128, smem, st>>>(a);
}

template <bool C, bool M3>
static void diag_t(bool backward, const SolveArgs& a, int ntiles, cudaStream_t st) {
  dim3 grid(ntiles, ntn(C, a.nrhs));
  if (!backward) launch_g(k_diag_g<C, false, M3>, SolveG<C, M3>::FU::SMEM_BYTES, grid, st, a);
  else launch_g(k_diag_g<C, true, M3>, SolveG<C, M3>::BU::SMEM_BYTES, grid, st, a);
  dim3 g2(std::min(ntiles, 256), a.nrhs);
  k_dcopy<C><<<g2, 64, 0, st>>>(a, ntiles);
}

void launch_diag_gemm(bool cplx, bool m3, bool backward, const SolveArgs& a, int ntiles, cudaStream_t st) {
  if (ntiles == 0 || a.nrhs == 0) return;
  if (!cplx) diag_t<false, false>(backward, a, ntiles, st);
  else if (m3) diag_t<true, true>(backward, a, ntiles, st);
  else diag_t<true, false>(backward, a, ntiles, st);
}

void launch_fupd(bool cplx, bool m3, const SolveArgs& a, int ntiles, cudaStream_t st) {
  if (ntiles == 0 || a.nrhs == 0) return;
  dim3 grid(ntiles, ntn(cplx, a.nrhs));
  if (!cplx) launch_g(k_fupd<false, false>, SolveG<false, false>::FU::SMEM_BYTES, grid, st, a);
  else if (m3) launch_g(k_fupd<true, true>, SolveG<true, true>::FU::SMEM_BYTES, grid, st, a);
  else launch_g(k_fupd<true, false>, SolveG<true, false>::FU::SMEM_BYTES, grid, st, a);
}

int bupd_split(bool cplx, int ntiles, int nrhs, int max_rp) {
  // enough CTAs to fill every SM at the backward-update kernel's occupancy (3 CTAs/SM) counting
  // one right-hand-side tile column, each chunk >= 128 rows of K; partial buffer bounded by
  // BUPD_MAX_PARTS tiles.  Independent of nrhs, so a column's result does not depend on how many
  // columns are solved together (bitwise).
  (void)cplx;
  (void)nrhs;
  const int want = 3 * 148;
  const int ctas = ntiles;
  if (ctas >= want) return 1;
  int G = (want + ctas - 1) / ctas;
  G = std::min(G, std::max(1, max_rp / 128));
  G = std::min(G, std::max(1, BUPD_MAX_PARTS / std::max(ntiles, 1)));
  static const int gmax = getenv("DD_AUX_BUPD_GMAX") ? atoi(getenv("DD_AUX_BUPD_GMAX")) : 32;  // A/B only
  return std::max(1, std::min(G, gmax));
}

template <bool C, bool M3>
static void bupd_t(const SolveArgs& a, int ntiles, int G, double* part, int64_t pim, bool cluster, cudaStream_t st) {
  using GB = typename SolveG<C, M3>::BU;
  dim3 grid(ntiles * G, ntn(C, a.nrhs));
#ifdef DD_AUX_AB
  if (cluster && G > 1) {
    set_smem(k_bupd<C, M3, true>, GB::SMEM_BYTES);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = GB::SMEM_BYTES;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)G;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_bupd<C, M3, true>, a, G, part, pim);
    return;
  }
#else
  (void)cluster;
#endif
  if (G > 1 && a.cnt) {  // split-K with the in-kernel (last-arriver) reduction
    set_smem(k_bupd<C, M3, false, true>, GB::SMEM_BYTES);
    k_bupd<C, M3, false, true><<<grid, 128, GB::SMEM_BYTES, st>>>(a, G, part, pim);
    return;
  }
  set_smem(k_bupd<C, M3, false>, GB::SMEM_BYTES);
  k_bupd<C, M3, false><<<grid, 128, GB::SMEM_BYTES, st>>>(a, G, part, pim);
}

void launch_bupd(bool cplx, bool m3, const SolveArgs& a, int ntiles, int max_rp, double* part, cudaStream_t st) {
  if (ntiles == 0 || a.nrhs == 0) return;
  // split-K reduction: partial buffer + fixed-order reduction kernel (default), or through a
  // thread-block cluster with distributed shared memory (DD_AUX_BUPD_CLUSTER=1, G capped at 8):
  // correct but measured slower -- cfg3 backward update 1518 -> 1620 ms, cfg2 528 -> 625 ms per
  // step (the cap on G costs more parallelism than the saved partial round trip gains)
#ifdef DD_AUX_AB
  static const bool cluster = getenv("DD_AUX_BUPD_CLUSTER") && atoi(getenv("DD_AUX_BUPD_CLUSTER")) == 1;
#else
  constexpr bool cluster = false;
#endif
  int G = part ? bupd_split(cplx, ntiles, a.nrhs, max_rp) : 1;
  if (cluster) G = std::min(G, 8);
  const int64_t pim = (int64_t)BUPD_MAX_PARTS * SUBM * a.nrhs;
  // The in-kernel (last-arriver) reduction is ONE CTA per (tile, rhs tile) reading G partial
  // tiles; the separate reduce kernel spreads the same fixed-order sums over the whole GPU.
  // Measured (solve ms per 1000 RHS, fold for G <= 0 / 4 / 8 / 32): cfg1 143 / 145 / 147 / 185,
  // cfg2 4,234 / 4,238 / 4,253 / 4,352, cfg3 3,504 / 3,539 / 3,551 / 3,599 -- the separate kernel
  // wins everywhere, so the fold is off (DDK_BUPD_FOLD_MAXG = 0; A/B switch).  Both forms add the
  // partials in the order g = 0..G-1: bitwise equal.
#ifndef DDK_BUPD_FOLD_MAXG
#define DDK_BUPD_FOLD_MAXG 0
#endif
  SolveArgs b = a;
  if (G > DDK_BUPD_FOLD_MAXG) b.cnt = nullptr;
  const SolveArgs& a_ = b;
  if (!cplx) bupd_t<false, false>(a_, ntiles, G, part, pim, cluster, st);
  else if (m3) bupd_t<true, true>(a_, ntiles, G, part, pim, cluster, st);
  else bupd_t<true, false>(a_, ntiles, G, part, pim, cluster, st);
  if (G > 1 && !cluster && !a_.cnt) {
    dim3 g2(ntiles, std::min(64, (SUBM * a.nrhs + 255) / 256));
    if (cplx) k_bupd_reduce<true><<<g2, 256, 0, st>>>(a, G, part, pim);
    else k_bupd_reduce<false><<<g2, 256, 0, st>>>(a, G, part, pim);
  }
}

void launch_dsolve(bool cplx, const SolveArgs& a, cudaStream_t st) {
  if (a.nrhs == 0) return;
  if (cplx) k_dsolve<true><<<rows_grid(a.nrows, a.nrhs), 256, 0, st>>>(a);
  else k_dsolve<false><<<rows_grid(a.nrows, a.nrhs), 256, 0, st>>>(a);
}
void launch_norm_a(bool cplx, const SpmvArgs& a, int nrow_tiles, unsigned long long* out, cudaStream_t st) {
  if (nrow_tiles == 0) return;
  if (cplx) k_norm_a<true><<<nrow_tiles, 64, 0, st>>>(a, out);
  else k_norm_a<false><<<nrow_tiles, 64, 0, st>>>(a, out);
}

void launch_berr(bool cplx, const double* y, int64_t yim, int64_t ldy, int64_t nrows, const double* X, int64_t ldx,
                 int64_t n, int nrhs, const unsigned long long* normA, double tol, double* berr, int* flag,
                 cudaStream_t st) {
  if (nrhs == 0) return;
  if (cplx) k_berr<true><<<nrhs, 256, 0, st>>>(y, yim, ldy, nrows, X, ldx, n, normA, tol, berr, flag);
  else k_berr<false><<<nrhs, 256, 0, st>>>(y, yim, ldy, nrows, X, ldx, n, normA, tol, berr, flag);
}

void launch_spmv(bool cplx, const SpmvArgs& a, int nrow_tiles, cudaStream_t st) {
  if (nrow_tiles == 0 || a.nrhs == 0) return;
  static const bool simt = getenv("DD_AUX_SPMV_SIMT") && atoi(getenv("DD_AUX_SPMV_SIMT"));
  if (simt) {
    dim3 grid(nrow_tiles, (a.nrhs + SPN - 1) / SPN);
    if (cplx) k_spmv<true><<<grid, 256, 0, st>>>(a);
    else k_spmv<false><<<grid, 256, 0, st>>>(a);
    return;
  }
  dim3 grid(nrow_tiles, (a.nrhs + SPT_N - 1) / SPT_N);
  if (cplx) {
    set_smem(k_spmv_dmma<true>, SpG_C::SMEM_BYTES);
    k_spmv_dmma<true><<<grid, 128, SpG_C::SMEM_BYTES, st>>>(a);
  } else {
    set_smem(k_spmv_dmma<false>, SpG_R::SMEM_BYTES);
    k_spmv_dmma<false><<<grid, 128, SpG_R::SMEM_BYTES, st>>>(a);
  }
}

}  // namespace ddk
