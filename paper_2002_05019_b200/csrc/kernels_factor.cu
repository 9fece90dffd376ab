// Factor-phase kernels (sm_100a).  PAPER.md:29 (§II): "custom block LDL^T with
// restricted Bunch-Kaufman pivoting"; SURVEY.md §8(a) rows a1-a6.
//
//   k0_*        a1  load caller blocks into the zeroed panel arena (planar, position order)
//   k1_diag_bk  a2  restricted BK LDL^T of each diagonal block of a level (one CTA per block),
//                   blocked dlasyf-style: left-looking panel of K1NB columns with warp-shuffle
//                   (value, index) pivot search, trailing update on DMMA; then the TB x TB
//                   inverse diagonal tiles of L_kk used by every TRSM
//   k_rowperm       apply P_t to the rows of block t inside earlier panels (explicit form, L5)
//   k2_panel    a3  W = (A P^T) L^{-T} by row strips (blocked TRSM as DMMA GEMMs), L = W D^{-1}
//   k3_update   a4  A_ij -= sum_k W_ik L_jk^T, owner-computes tiles with gathered K (DMMA)
//   k4_stats    a6  inertia / pivot statistics reduction
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "gemm_core.cuh"
#include "launch.hpp"

using namespace ddaux;

namespace ddk {

// ============================================================================ K0 load
// Copy input block (I,J) (caller layout, interleaved complex) into the arena block of the
// panel of the earlier-eliminated of the two, transposing when I is eliminated first.
template <bool C>
__global__ void k0_load(const double* __restrict__ vals, const LoadBlock* __restrict__ lb, int nblocks,
                        double* __restrict__ arena, int64_t aim) {
  for (int b = blockIdx.y; b < nblocks; b += gridDim.y) {  // grid-stride over blocks (gridDim.y <= 65535)
  LoadBlock L = lb[b];
  const int64_t total = (int64_t)L.rows * L.cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = e % L.rows, c = e / L.rows;  // source element (r, c) of the stored s_I x s_J block
    if (L.diag && r < c) continue;            // diagonal blocks: lower triangle only
    int64_t src = L.voff + e;
    double re, im = 0.0;
    if (C) {
      re = vals[2 * src];
      im = vals[2 * src + 1];
    } else {
      re = vals[src];
    }
    int64_t dst = L.trans ? (L.dst + c + r * L.ld) : (L.dst + r + c * L.ld);
    arena[dst] = re;
    if (C) arena[dst + aim] = im;
  }
  }
}

// ============================================================================ K1 diagonal BK
#ifndef DDK_NT1
#define DDK_NT1 256
#endif
constexpr int NT1 = DDK_NT1;  // K1 threads per CTA (one row each on the <=NT1 fast path)
constexpr size_t K1_SMEM_BUDGET = 210 * 1024;  // dynamic smem for the panel copy of L + W window

// Panel width: the widest of 64, 56, ..., 8 whose shared panel copy of L (s x NB) plus the W
// window cache (NB x (NB+1)) fits the budget; an explicit override (8..64) wins if it fits.
// fullw: the W cache holds ALL rows of the block (s x (NB+1)) instead of the NB-row window, so W
// never goes through global memory inside a panel (no row loads for an out-of-window imax, no
// global row interchanges); W is written to global memory once per panel for the trailing update
__host__ __device__ inline size_t k1_panel_bytes(int s, bool cplx, int nb, bool fullw = false) {
  return ((size_t)s * nb + (size_t)(fullw ? s : nb) * (nb + 1)) * (cplx ? 16 : 8);
}
__host__ __device__ inline int k1_panel_nb(int s, bool cplx, int req, bool fullw = false) {
  if (req >= 8 && req <= K1NB_MAX && k1_panel_bytes(s, cplx, req, fullw) <= K1_SMEM_BUDGET) return req;
  int nb = K1NB_MAX;
  while (nb > 8 && k1_panel_bytes(s, cplx, nb, fullw) > K1_SMEM_BUDGET) nb -= 8;
  return nb;
}
// rows per thread: s <= NT1 * MAXQ (4 -> 1024 on the fast path, 16 -> 4096 for larger interfaces)
using K1GemmR = Gemm<64, 64, 16, 2, NT1 / 64, 2, false, false, false>;
using K1GemmC = Gemm<64, 64, 16, 2, NT1 / 64, 2, true, false, false>;

// pivot-search magnitude with non-finite values mapped to +Inf (reading L4b): a NaN would be
// invisible to the (value desc, index asc) max reduction; as +Inf it makes colmax / rowmax non-finite
template <bool C>
__device__ __forceinline__ double mag_nf(cz v) {
  const double a = cabs1<C>(v);
  return a <= 1.79769313486231570e308 ? a : __longlong_as_double(0x7ff0000000000000LL);
}
__device__ __forceinline__ bool finite_d(double x) { return x <= 1.79769313486231570e308; }

// max |L| of the calling thread's values -> one atomicMax per warp on the factor-wide slot
__device__ __forceinline__ void warp_max_to(unsigned long long* slot, double m) {
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m > 0.0 && slot) atomicMax(slot, (unsigned long long)__double_as_longlong(m));
}
template <bool C>
__device__ __forceinline__ double modulus(cz v) {
  if constexpr (C) return hypot(v.r, v.i);
  else return fabs(v.r);
}

#ifndef DDK_REDUX
#define DDK_REDUX 1  // measured: cfg1 K1 30.1 -> 28.5 ms (factor 37.1 -> 35.9 ms) against the shuffle tree
#endif
__device__ __forceinline__ void warp_argmax(double& v, int& i) {
#if DDK_REDUX
  // (value desc, index asc) with three warp redux.sync ops: magnitudes are >= 0 (or -1 = no
  // candidate), so the IEEE bit pattern of a non-negative double orders like its value
  const bool cand = v >= 0.0;
  const unsigned hi = cand ? (unsigned)__double2hiint(v) : 0u, lo = cand ? (unsigned)__double2loint(v) : 0u;
  const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
  const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
  const unsigned mi = __reduce_min_sync(0xffffffffu, (cand && hi == mh && lo == ml) ? (unsigned)i : 0xffffffffu);
  v = (mh | ml) || mi != 0xffffffffu ? __hiloint2double((int)mh, (int)ml) : -1.0;
  i = mi == 0xffffffffu ? INT_MAX : (int)mi;
#else
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    double v2 = __shfl_xor_sync(0xffffffffu, v, o);
    int i2 = __shfl_xor_sync(0xffffffffu, i, o);
    if (v2 > v || (v2 == v && i2 < i)) {
      v = v2;
      i = i2;
    }
  }
#endif
}

// block-wide (max value, smallest index on ties): IDAMAX semantics (reading L3).  One barrier:
// consecutive calls alternate between two slot sets (a slot is rewritten only after every
// thread has passed the following call's barrier, i.e. finished reading it).
__device__ __forceinline__ void block_argmax(double& v, int& i, double (*shv)[NT1 / 32], int (*shi)[NT1 / 32],
                                             int& slot) {
  warp_argmax(v, i);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* sv = shv[slot];
  int* si = shi[slot];
  slot ^= 1;
  if (lane == 0) {
    sv[w] = v;
    si[w] = i;
  }
  __syncthreads();
  // every warp reduces the NT1/32 warp results with shuffles (one shared load per lane)
  constexpr int NW = NT1 / 32;
  v = sv[lane % NW];
  i = si[lane % NW];
#if DDK_REDUX
  warp_argmax(v, i);
#else
#pragma unroll
  for (int o = NW / 2; o; o >>= 1) {
    double v2 = __shfl_xor_sync(0xffffffffu, v, o);
    int i2 = __shfl_xor_sync(0xffffffffu, i, o);
    if (v2 > v || (v2 == v && i2 < i)) {
      v = v2;
      i = i2;
    }
  }
#endif
}

// Common tail of both K1 variants: TB x TB inverse diagonal tiles of L, the global permutation
// maps and the per-node statistics (inertia from D for real matrices, a6).
template <bool C>
__device__ void k1_finish(const K1Args& a, int t, const NodeDev& nd, double* A, double* smem, const int* perm,
                          const int* ipiv, const double* dv_, const double* ev_, int n2x2, int nswap, int zero_col,
                          int nperturbed = 0, int nonfinite = 0) {
  const int s = nd.s;
  const int64_t ldA = nd.ld, aim = a.aim;
  const int tid = threadIdx.x, nthr = blockDim.x;
  auto Ael = [&](int i, int j) { return (int64_t)i + (int64_t)j * ldA; };
  // ---------------------------------------------------------------- inverse diagonal tiles of L
  __threadfence_block();
  __syncthreads();
  {
    const int ntiles = (s + TB - 1) / TB;
    const int warp = tid >> 5, lane = tid & 31;
    double* Lr = smem + warp * (2 * TB * TB);  // per-warp staging (re, im)
    double* Li = Lr + TB * TB;
    double* Vb = a.arena + nd.linv;
    for (int p = warp; p < ntiles; p += nthr / 32) {
      const int r0 = p * TB, w = min(TB, s - r0);
      for (int e = lane; e < TB * TB; e += 32) {
        int i = e % TB, j = e / TB;
        cz v = (i < w && j < w && i > j) ? ld<C>(A, Ael(r0 + i, r0 + j), aim) : mk(0.0, 0.0);
        Lr[e] = v.r;
        Li[e] = v.i;
      }
      __syncwarp();
      // lane j computes column j of L_pp^{-1}: x_i = delta_ij - sum_{m<i} L(i,m) x_m
      cz x[TB];
#pragma unroll
      for (int i = 0; i < TB; ++i) {
        cz v = mk(i == lane ? 1.0 : 0.0, 0.0);
#pragma unroll
        for (int m = 0; m < i; ++m) v = fms<C>(v, mk(Lr[i + m * TB], Li[i + m * TB]), x[m]);
        x[i] = (i < lane) ? mk(0.0, 0.0) : v;
      }
#pragma unroll
      for (int i = 0; i < TB; ++i) st<C>(Vb, (int64_t)p * TB * TB + i + (int64_t)lane * TB, aim, x[i]);
      __syncwarp();
    }
  }
  __syncthreads();
  // ---------------------------------------------------------------- global permutation maps + stats
  for (int m = tid; m < nd.sp; m += nthr) {
    if (m < s) {
      int o = (int)(nd.odof + perm[m]);
      a.gperm[nd.ydof + m] = o;
      a.ginv[o] = (int)(nd.ydof + m);
    } else {
      a.gperm[nd.ydof + m] = -1;
    }
  }
  if (tid == 0) {
    int64_t np = 0, nn = 0, nz = 0;
    if (!C) {
      int q = 0;
      while (q < s) {
        if (ipiv[q] < 0) {
          double x = dv_[q], y = ev_[q], z = dv_[q + 1];
          double det = x * z - y * y;
          if (det < 0) {
            ++np;
            ++nn;
          } else if (det > 0) {
            if (x + z > 0) np += 2;
            else nn += 2;
          } else {
            ++nz;
            if (x + z > 0) ++np;
            else if (x + z < 0) ++nn;
            else ++nz;
          }
          q += 2;
        } else {
          double x = dv_[q];
          if (x > 0) ++np;
          else if (x < 0) ++nn;
          else ++nz;
          ++q;
        }
      }
    }
    int64_t* S = a.stats + (int64_t)t * 8;
    S[0] = np;
    S[1] = nn;
    S[2] = nz;
    S[3] = n2x2;
    S[4] = nswap;
    // first zero / non-finite pivot as an ELIMINATION-order key (padded position row + 1); k4 takes
    // the minimum over nodes and maps it to the original DoF through gperm (LAPACK INFO order)
    S[5] = zero_col >= 0 ? nd.ydof + zero_col + 1 : 0;
    S[6] = nperturbed;
    S[7] = nonfinite;
  }
}

template <bool C, int K1_MAXQ>
__global__ void __launch_bounds__(NT1) k1_diag_bk(K1Args a) {
  using G = typename std::conditional<C, K1GemmC, K1GemmR>::type;
  extern __shared__ __align__(16) double smem[];
  __shared__ double shv[2][NT1 / 32];
  __shared__ int shi[2][NT1 / 32];
  int aslot = 0;
  __shared__ double wrow_r[K1NB_MAX], wrow_i[K1NB_MAX];
  __shared__ int s_swa[K1NB_MAX], s_swb[K1NB_MAX], s_nswp;
  __shared__ double s_absakk2[2];  // parity-buffered: no barrier between a read and the next write
  __shared__ double s_xw[2][4];    // register copies (wv, wv2) of the two interchanged rows

  const int t = a.nodes[blockIdx.x];
  const NodeDev nd = a.nd[t];
  const int s = nd.s;
  const int64_t ldA = nd.ld;
  double* A = a.arena + nd.panel;  // diagonal block = panel rows [0, s)
  const int64_t aim = a.aim;
  double* W = a.work + nd.k1w;     // s x K1NB scratch, ld = sp
  const int64_t ldW = nd.sp;
  const int64_t wim = a.wim;
  int* perm = a.perm + nd.ydof;
  int* ipiv = a.ipiv + nd.ydof;
  double* dv_ = a.arena + a.d_off + nd.ydof;
  double* ev_ = a.arena + a.e_off + nd.ydof;
  const int tid = threadIdx.x;
  const double alpha = (1.0 + sqrt(17.0)) / 8.0;

  auto Ael = [&](int i, int j) { return (int64_t)i + (int64_t)j * ldA; };
  auto Wel = [&](int i, int m) { return (int64_t)i + (int64_t)m * ldW; };

  for (int i = tid; i < s; i += NT1) perm[i] = i;
  int n2x2 = 0, nswap = 0, zero_col = -1, nonfinite = 0, nperturbed = 0;
  double maxl = 0.0;  // max |L| of the entries this thread writes (SURVEY.md §8(b) max_abs_L)
  __syncthreads();

  // Panel width NB: the current panel's L columns live in shared memory (Lp, <= K1_LP_BUDGET
  // bytes; aliased later by the trailing-update GEMM and the inverse staging) and reach
  // global memory only at the panel end; W rows of the panel window [c0, c0+NB) are cached in
  // wt.  Thread tid owns rows tid + q*NT1 (q < K1_MAXQ) for the whole factorization and keeps
  // their current W values in registers, so a column without interchange costs two barriers.
  // Interchanges of rows inside L columns of EARLIER panels (explicit form, L5) are deferred
  // to the panel end (LAPACK xLASWP style): nothing in this kernel reads those columns before.
  // full-W mode when the panel width it allows is still >= 32 (a.fullw: 1 auto, 0 off)
  const bool FW = a.fullw != 0 && k1_panel_nb(s, C, a.nb, true) >= 32 &&
                  k1_panel_bytes(s, C, k1_panel_nb(s, C, a.nb, true), true) <= K1_SMEM_BUDGET;
  const int NB = FW ? k1_panel_nb(s, C, a.nb, true) : k1_panel_nb(s, C, a.nb);
  const int WIN = FW ? s : NB;               // rows held by the W cache, from c0
  double* Lpr = smem;                       // Lp(i, m) = Lpr[m * s + i]
  double* Lpi = smem + (size_t)s * NB;
  // W cache wt(r, m) = W(c0 + r, m), row stride NB+1 (after the panel copy of L)
  double* wtr = smem + (size_t)s * NB * (C ? 2 : 1);
  double* wti = wtr + (size_t)WIN * (NB + 1);
  const int WLD = NB + 1;
  auto LP = [&](int i, int m) { return (size_t)m * s + i; };
  cz Ak[K1_MAXQ], wv[K1_MAXQ], wv2[K1_MAXQ];
#pragma unroll
  for (int q = 0; q < K1_MAXQ; ++q) {
    const int i = tid + q * NT1;
    Ak[q] = i < s ? ld<C>(A, Ael(i, 0), aim) : mk(0.0, 0.0);
  }

  int k = 0;
  while (k < s) {
    const int c0 = k;
    const bool last_panel = (s - c0) <= NB;
    if (tid == 0) s_nswp = 0;
    // ------------------------------------------------------------ panel (left-looking)
    while (k < s) {
      const int kk = k - c0;
      if (!last_panel && kk >= NB - 1) break;
      // prefetch column k+1 of A now (its latency hides behind this column's work); it is kept
      // only if this step is a 1x1 pivot without interchange (which leaves column k+1 untouched)
      constexpr bool PF = K1_MAXQ <= 4;
      cz An[PF ? K1_MAXQ : 1];
      const bool pf = PF && k + 1 < s && !(kk + 1 >= NB - 1 && !last_panel);
      if constexpr (PF) {
        if (pf) {
#pragma unroll
          for (int q = 0; q < K1_MAXQ; ++q) {
            const int i = tid + q * NT1;
            if (i >= k + 1 && i < s) An[q] = ld<C>(A, Ael(i, k + 1), aim);
          }
        }
      }
      bool swapped = false;
      // updated column k:  W(k:s, kk) = A(k:s, k) - Lp(k:s, 0:kk) W(k, 0:kk)^T  (W row k: window)
      double bv = -1.0;
      int bi = INT_MAX;
#pragma unroll
      for (int q = 0; q < K1_MAXQ; ++q) {
        const int i = tid + q * NT1;
        if (i < k || i >= s) continue;
        // one FMA chain (DDK_K1_CHAINS=2 splits it in two: measured slower on cfg1, 35.1 vs 32.4 ms)
#ifndef DDK_K1_CHAINS
#define DDK_K1_CHAINS 1
#endif
        cz v = Ak[q], v1 = mk(0.0, 0.0);
        int m = 0;
        if (DDK_K1_CHAINS == 2)
        for (; m + 1 < kk; m += 2) {
          v = fms<C>(v, mk(Lpr[LP(i, m)], C ? Lpi[LP(i, m)] : 0.0), mk(wtr[(kk) * WLD + (m)], C ? wti[(kk) * WLD + (m)] : 0.0));
          v1 = fms<C>(v1, mk(Lpr[LP(i, m + 1)], C ? Lpi[LP(i, m + 1)] : 0.0),
                      mk(wtr[(kk) * WLD + (m + 1)], C ? wti[(kk) * WLD + (m + 1)] : 0.0));
        }
        for (; m < kk; ++m)
          v = fms<C>(v, mk(Lpr[LP(i, m)], C ? Lpi[LP(i, m)] : 0.0), mk(wtr[(kk) * WLD + (m)], C ? wti[(kk) * WLD + (m)] : 0.0));
        if (DDK_K1_CHAINS == 2) v = v + v1;
        wv[q] = v;
        if (!FW) st<C>(W, Wel(i, kk), wim, v);
        if (i - c0 < WIN) {
          wtr[(i - c0) * WLD + (kk)] = v.r;
          if constexpr (C) wti[(i - c0) * WLD + (kk)] = v.i;
        }
        double av = mag_nf<C>(v);
        if (i == k) s_absakk2[k & 1] = av;
        else if (av > bv) {
          bv = av;
          bi = i;
        }
      }
      block_argmax(bv, bi, shv, shi, aslot);
      // ---- pivot decision (Bunch-Kaufman, LAPACK xSYTF2 order)
      const double absakk = s_absakk2[k & 1];
      const double colmax = bv > 0.0 ? bv : 0.0;
      const int imax = bi;
      int kp, kstep = 1;
      bool zero = false, nonfin = !finite_d(absakk) || !finite_d(colmax), perturbed = false;
      if (!nonfin && fmax(absakk, colmax) == 0.0 && a.perturb_tau > 0.0) {
        perturbed = true;  // reading L4 (opt-in): 1x1 pivot d = tau * ||A||_inf, no swap
        kp = k;
      } else if (nonfin || fmax(absakk, colmax) == 0.0) {
        zero = true;  // LAPACK: zero (or, L4b, non-finite) pivot column, no elimination
        kp = k;
      } else if (absakk >= alpha * colmax) {
        kp = k;
      } else {
        // updated column imax -> W(:, kk+1) (symmetric access of the not-yet-updated trailing A)
        const bool inwin = imax - c0 < WIN;
        if (!inwin) {
          for (int m = tid; m < kk; m += NT1) {
            cz w = ld<C>(W, Wel(imax, m), wim);
            wrow_r[m] = w.r;
            wrow_i[m] = w.i;
          }
          __syncthreads();
        }
        double rv = -1.0;
        int ri = INT_MAX;
#pragma unroll
        for (int q = 0; q < K1_MAXQ; ++q) {
          const int i = tid + q * NT1;
          if (i < k || i >= s) continue;
          cz v = (i < imax) ? ld<C>(A, Ael(imax, i), aim) : ld<C>(A, Ael(i, imax), aim);
          cz v1 = mk(0.0, 0.0);
          const double* wr = inwin ? wtr + (imax - c0) * WLD : wrow_r;
          const double* wi = inwin ? wti + (imax - c0) * WLD : wrow_i;
          int m = 0;
          if (DDK_K1_CHAINS == 2)
          for (; m + 1 < kk; m += 2) {
            v = fms<C>(v, mk(Lpr[LP(i, m)], C ? Lpi[LP(i, m)] : 0.0), mk(wr[m], C ? wi[m] : 0.0));
            v1 = fms<C>(v1, mk(Lpr[LP(i, m + 1)], C ? Lpi[LP(i, m + 1)] : 0.0), mk(wr[m + 1], C ? wi[m + 1] : 0.0));
          }
          for (; m < kk; ++m) v = fms<C>(v, mk(Lpr[LP(i, m)], C ? Lpi[LP(i, m)] : 0.0), mk(wr[m], C ? wi[m] : 0.0));
          if (DDK_K1_CHAINS == 2) v = v + v1;
          wv2[q] = v;
          if (!FW) st<C>(W, Wel(i, kk + 1), wim, v);
          if (i - c0 < WIN) {
            wtr[(i - c0) * WLD + (kk + 1)] = v.r;
            if constexpr (C) wti[(i - c0) * WLD + (kk + 1)] = v.i;
          }
          if (i != imax) {
            double av = mag_nf<C>(v);
            if (av > rv) {
              rv = av;
              ri = i;
            }
          }
        }
        block_argmax(rv, ri, shv, shi, aslot);
        const double rowmax = rv;
        if (!finite_d(rowmax)) {  // L4b: the imax row holds a non-finite value
          zero = nonfin = true;
          kp = k;
        } else if (absakk >= alpha * colmax * (colmax / rowmax)) {
          kp = k;
        } else {
          const double aii = cabs1<C>(inwin ? mk(wtr[(imax - c0) * WLD + (kk + 1)], C ? wti[(imax - c0) * WLD + (kk + 1)] : 0.0)
                                            : ld<C>(W, Wel(imax, kk + 1), wim));
          kp = imax;
          if (aii >= alpha * rowmax) {  // 1x1 pivot on the imax column: it becomes column kk
#pragma unroll
            for (int q = 0; q < K1_MAXQ; ++q) {
              const int i = tid + q * NT1;
              if (i < k || i >= s) continue;
              wv[q] = wv2[q];
              if (!FW) st<C>(W, Wel(i, kk), wim, wv2[q]);
              if (i - c0 < WIN) {
                wtr[(i - c0) * WLD + (kk)] = wv2[q].r;
                if constexpr (C) wti[(i - c0) * WLD + (kk)] = wv2[q].i;
              }
            }
          } else {
            kstep = 2;
          }
        }
      }
      const int kkk = k + kstep - 1;
      if (kp != kkk) {
        swapped = true;
        __syncthreads();
        // move the non-updated column kkk of the trailing block to position kp (dlasyf).  The column
        // is already in registers (Ak = column k, the prefetched An = column k+1), so each row owner
        // stores its own element: no global round trip on the interchange path
        if constexpr (PF) {
          if (pf || kstep == 1) {
#pragma unroll
            for (int q = 0; q < K1_MAXQ; ++q) {
              const int i = tid + q * NT1;
              const cz cv = kstep == 1 ? Ak[q] : An[PF ? q : 0];
              if (i == kkk) st<C>(A, Ael(kp, kp), aim, cv);
              else if (i > kkk && i < kp) st<C>(A, Ael(kp, i), aim, cv);
              else if (i > kp && i < s) st<C>(A, Ael(i, kp), aim, cv);
            }
          } else {
            if (tid == 0) st<C>(A, Ael(kp, kp), aim, ld<C>(A, Ael(kkk, kkk), aim));
            for (int j = kkk + 1 + tid; j < kp; j += NT1) st<C>(A, Ael(kp, j), aim, ld<C>(A, Ael(j, kkk), aim));
            for (int j = kp + 1 + tid; j < s; j += NT1) st<C>(A, Ael(j, kp), aim, ld<C>(A, Ael(j, kkk), aim));
          }
        } else {
          if (tid == 0) st<C>(A, Ael(kp, kp), aim, ld<C>(A, Ael(kkk, kkk), aim));
          for (int j = kkk + 1 + tid; j < kp; j += NT1) st<C>(A, Ael(kp, j), aim, ld<C>(A, Ael(j, kkk), aim));
          for (int j = kp + 1 + tid; j < s; j += NT1) st<C>(A, Ael(j, kp), aim, ld<C>(A, Ael(j, kkk), aim));
        }
        // rows kkk, kp of the panel's L columns (shared copy) -- earlier panels: deferred
        for (int m = tid; m < kk; m += NT1) {
          double t0 = Lpr[LP(kkk, m)];
          Lpr[LP(kkk, m)] = Lpr[LP(kp, m)];
          Lpr[LP(kp, m)] = t0;
          if constexpr (C) {
            double t1 = Lpi[LP(kkk, m)];
            Lpi[LP(kkk, m)] = Lpi[LP(kp, m)];
            Lpi[LP(kp, m)] = t1;
          }
        }
        // rows kkk, kp of W columns 0..kk+kstep-1 (global, and the window cache)
        const bool kpwin = kp - c0 < WIN;
        for (int m = tid; m < kk + kstep; m += NT1) {
          cz x, y;
          if (FW) {  // the whole W lives in the cache
            x = mk(wtr[(kkk - c0) * WLD + m], C ? wti[(kkk - c0) * WLD + m] : 0.0);
            y = mk(wtr[(kp - c0) * WLD + m], C ? wti[(kp - c0) * WLD + m] : 0.0);
          } else {
            x = ld<C>(W, Wel(kkk, m), wim);
            y = ld<C>(W, Wel(kp, m), wim);
            st<C>(W, Wel(kkk, m), wim, y);
            st<C>(W, Wel(kp, m), wim, x);
          }
          wtr[(kkk - c0) * WLD + (m)] = y.r;
          if constexpr (C) wti[(kkk - c0) * WLD + (m)] = y.i;
          if (kpwin) {
            wtr[(kp - c0) * WLD + (m)] = x.r;
            if constexpr (C) wti[(kp - c0) * WLD + (m)] = x.i;
          }
        }
        if (tid == 0) {
          int x = perm[kkk];
          perm[kkk] = perm[kp];
          perm[kp] = x;
          s_swa[s_nswp] = kkk;
          s_swb[s_nswp] = kp;
          ++s_nswp;
        }
        // the owners of rows kkk and kp trade their register copies through shared memory (the
        // barrier orders this CTA's shared and global accesses; no fence or global reload needed)
#pragma unroll
        for (int q = 0; q < K1_MAXQ; ++q) {
          const int i = tid + q * NT1;
          if (i == kkk || i == kp) {
            double* x = s_xw[i == kkk ? 0 : 1];
            x[0] = wv[q].r;
            x[1] = wv[q].i;
            x[2] = wv2[q].r;
            x[3] = wv2[q].i;
          }
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < K1_MAXQ; ++q) {
          const int i = tid + q * NT1;
          if (i == kkk || i == kp) {
            const double* x = s_xw[i == kkk ? 1 : 0];
            wv[q] = mk(x[0], x[1]);
            if (kstep == 2) wv2[q] = mk(x[2], x[3]);
          }
        }
      }
      // ---- L columns (shared panel copy) and D; the next column is prefetched
      if (kstep == 1) {
        const cz D = perturbed ? mk(a.perturb_tau * __longlong_as_double((long long)*a.normA), 0.0)
                               : mk(wtr[(kk) * WLD + (kk)], C ? wti[(kk) * WLD + (kk)] : 0.0);
        const cz rD = zero ? mk(1.0, 0.0) : dv<C>(mk(1.0, 0.0), D);
#pragma unroll
        for (int q = 0; q < K1_MAXQ; ++q) {
          const int i = tid + q * NT1;
          if (i <= k || i >= s) continue;
          const cz l = mul<C>(wv[q], rD);
          Lpr[LP(i, kk)] = l.r;
          if constexpr (C) Lpi[LP(i, kk)] = l.i;
        }
        if (tid == 0) {
          st<C>(dv_, 0 + k, aim, D);
          st<C>(ev_, 0 + k, aim, mk(0.0, 0.0));
          ipiv[k] = kp + 1;
          if (zero && zero_col < 0) zero_col = k;
          nonfinite += nonfin;
          nperturbed += perturbed;
          if (kp != k) ++nswap;
        }
      } else {
        const cz w11 = mk(wtr[(kk) * WLD + (kk)], C ? wti[(kk) * WLD + (kk)] : 0.0), w21 = mk(wtr[(kk + 1) * WLD + (kk)], C ? wti[(kk + 1) * WLD + (kk)] : 0.0),
                 w22 = mk(wtr[(kk + 1) * WLD + (kk + 1)], C ? wti[(kk + 1) * WLD + (kk + 1)] : 0.0);
        // LAPACK dlasyf scaled closed form of [W_k W_k+1] D^{-1}
        const cz d11 = dv<C>(w22, w21), d22 = dv<C>(w11, w21);
        const cz tt = dv<C>(mk(1.0, 0.0), mul<C>(d11, d22) - mk(1.0, 0.0));
        const cz d21 = dv<C>(tt, w21);
#pragma unroll
        for (int q = 0; q < K1_MAXQ; ++q) {
          const int i = tid + q * NT1;
          if (i <= k || i >= s) continue;
          cz l0 = mk(0.0, 0.0), l1 = mk(0.0, 0.0);  // row k+1: identity 2x2 block of L
          if (i > k + 1) {
            l0 = mul<C>(d21, mul<C>(d11, wv[q]) - wv2[q]);
            l1 = mul<C>(d21, mul<C>(d22, wv2[q]) - wv[q]);
          }
          Lpr[LP(i, kk)] = l0.r;
          Lpr[LP(i, kk + 1)] = l1.r;
          if constexpr (C) {
            Lpi[LP(i, kk)] = l0.i;
            Lpi[LP(i, kk + 1)] = l1.i;
          }
        }
        if (tid == 0) {
          st<C>(dv_, k, aim, w11);
          st<C>(dv_, k + 1, aim, w22);
          st<C>(ev_, k, aim, w21);
          st<C>(ev_, k + 1, aim, mk(0.0, 0.0));
          ipiv[k] = ipiv[k + 1] = -(kp + 1);
          ++n2x2;
          if (kp != k + 1) ++nswap;
        }
      }
      k += kstep;
      if (k < s && !(kk + kstep >= NB - 1 && !last_panel)) {
        if (PF && pf && kstep == 1 && !swapped) {
#pragma unroll
          for (int q = 0; q < K1_MAXQ; ++q) Ak[q] = An[PF ? q : 0];
        } else {
#pragma unroll
          for (int q = 0; q < K1_MAXQ; ++q) {
            const int i = tid + q * NT1;
            if (i >= k && i < s) Ak[q] = ld<C>(A, Ael(i, k), aim);
          }
        }
      }
    }
    // ------------------------------------------------------------ panel end
    __syncthreads();
    {
      const int kb = k - c0;
      // the panel's L columns and D diagonal to global memory
      for (int m = 0; m < kb; ++m) {
        const int col = c0 + m;
        for (int i = col + 1 + tid; i < s; i += NT1) {
          const cz l = mk(Lpr[LP(i, m)], C ? Lpi[LP(i, m)] : 0.0);
          maxl = fmax(maxl, modulus<C>(l));
          st<C>(A, Ael(i, col), aim, l);
        }
        if (tid == 0) st<C>(A, Ael(col, col), aim, ld<C>(dv_, col, aim));
      }
      // deferred interchanges in the L columns of earlier panels (in pivot order)
      const int nsw = s_nswp;
      for (int j = tid; j < c0; j += NT1)
        for (int q = 0; q < nsw; ++q) {
          const int r0 = s_swa[q], r1 = s_swb[q];
          cz x = ld<C>(A, Ael(r0, j), aim), y = ld<C>(A, Ael(r1, j), aim);
          st<C>(A, Ael(r0, j), aim, y);
          st<C>(A, Ael(r1, j), aim, x);
        }
    }
    // ------------------------------------------------------------ trailing update (DMMA)
    if (k < s) {
      // A(k:s, k:s) -= L(k:s, c0:k) W(k:s, 0:kb)^T.  The GEMM window starts at the even
      // row ke <= k (16-byte aligned cp.async chunks); row/column ke < k is masked.
      const int kb = k - c0, ke = k & ~1, M = s - ke;
      if (FW) {  // W rows [ke, s) of this panel: cache -> global (the GEMM's B operand)
        for (int e = tid; e < (s - ke) * kb; e += NT1) {
          const int i = ke + e % (s - ke), m = e / (s - ke);
          st<C>(W, Wel(i, m), wim, mk(wtr[(i - c0) * WLD + m], C ? wti[(i - c0) * WLD + m] : 0.0));
        }
      }
      // the barrier orders this CTA's earlier global stores (L panel, W) before the cp.async reads
      __syncthreads();
      Seg sg;
      sg.a = A + Ael(ke, c0);
      sg.lda = ldA;
      sg.b = W + ke;  // B(q, n) = W(ke + n, q)
      sg.ldb = ldW;
      sg.acol = nullptr;
      sg.K = kb;
      const int nt = (M + 63) / 64;
      for (int tm = 0; tm < nt; ++tm)
        for (int tn = 0; tn <= tm; ++tn) {
          typename G::Acc acc;
          G::zero(acc);
          G::run([&](int) { return sg; }, 1, tm * 64, tn * 64, M, M, aim, wim, smem, acc,
                 G::tile_mask(M - tm * 64, M - tn * 64, tn * 64 - tm * 64));
          double* Cb = A + Ael(ke + tm * 64, ke + tn * 64);
          if (ke < k) {  // row / column ke (already eliminated) must stay: subtract exact zeros there
            G::for_each_mut(acc, [&](int r, int c, double& vr, double& vi) {
              if ((tm == 0 && r == 0) || (tn == 0 && c == 0)) vr = vi = 0.0;
            });
          }
          // coalesced read-modify-write (all loads of a batch in flight before the stores)
          G::template store_tile<1>(acc, smem, Cb, ldA, aim, M - tm * 64, M - tn * 64);
        }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < K1_MAXQ; ++q) {
        const int i = tid + q * NT1;
        if (i >= k && i < s) Ak[q] = ld<C>(A, Ael(i, k), aim);
      }
    }
  }

  warp_max_to(a.maxL, fmax(maxl, 1.0));  // unit diagonal included
  k1_finish<C>(a, t, nd, A, smem, perm, ipiv, dv_, ev_, n2x2, nswap, zero_col, nperturbed, nonfinite);
}

#ifdef DD_AUX_AB  // A/B-only variant (measured slower; not in the default build)
// ============================================================================ K1, warp variant
// For small diagonal blocks (real s <= 256, complex s <= 128) the column loop runs on ONE warp
// with the panel's L and W entirely in shared memory: argmax by shuffles, __syncwarp only, no
// block barrier per column.  The four warps of the CTA join at panel ends for the L/W write-back,
// the deferred interchanges and the DMMA trailing update.  Same decisions as k1_diag_bk.
constexpr int NT1W = 128;
using K1WGemmR = Gemm<64, 64, 16, 2, 2, 2, false, false, false>;
using K1WGemmC = Gemm<64, 64, 16, 2, 2, 2, true, false, false>;
// rows per lane: real s <= 256 -> 8, complex s <= 128 -> 4

template <bool C>
__global__ void __launch_bounds__(NT1W) k1_diag_bk_warp(K1Args a) {
  using G = typename std::conditional<C, K1WGemmC, K1WGemmR>::type;
  constexpr int K1W_Q = C ? 4 : 8;
  extern __shared__ __align__(16) double smem[];
  __shared__ int s_swa[K1NB], s_swb[K1NB], s_nswp, s_k;
  const int t = a.nodes[blockIdx.x];
  const NodeDev nd = a.nd[t];
  const int s = nd.s;
  const int64_t ldA = nd.ld, aim = a.aim;
  double* A = a.arena + nd.panel;
  double* Wg = a.work + nd.k1w;  // global W panel for the trailing GEMM, ld = sp
  const int64_t ldW = nd.sp, wim = a.wim;
  int* perm = a.perm + nd.ydof;
  int* ipiv = a.ipiv + nd.ydof;
  double* dv_ = a.arena + a.d_off + nd.ydof;
  double* ev_ = a.arena + a.e_off + nd.ydof;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const double alpha = (1.0 + sqrt(17.0)) / 8.0;
  constexpr int NB = K1NB;
  double* Lr = smem;                               // Lp(i, m) = Lr[m*s + i]
  double* Li = Lr + (size_t)s * NB;
  double* Wr = Lr + (size_t)s * NB * (C ? 2 : 1);  // Wp(i, m) = Wr[m*s + i]
  double* Wi = Wr + (size_t)s * NB;
  auto P = [&](int i, int m) { return (size_t)m * s + i; };
  auto Ael = [&](int i, int j) { return (int64_t)i + (int64_t)j * ldA; };
  auto Lget = [&](int i, int m) { return mk(Lr[P(i, m)], C ? Li[P(i, m)] : 0.0); };
  auto Wget = [&](int i, int m) { return mk(Wr[P(i, m)], C ? Wi[P(i, m)] : 0.0); };
  auto Lset = [&](int i, int m, cz v) {
    Lr[P(i, m)] = v.r;
    if constexpr (C) Li[P(i, m)] = v.i;
  };
  auto Wset = [&](int i, int m, cz v) {
    Wr[P(i, m)] = v.r;
    if constexpr (C) Wi[P(i, m)] = v.i;
  };

  for (int i = tid; i < s; i += NT1W) perm[i] = i;
  int n2x2 = 0, nswap = 0, zero_col = -1;
  __syncthreads();
  cz Ak[K1W_Q], wv[K1W_Q], wv2[K1W_Q];
  int k = 0;
  while (k < s) {
    const int c0 = k;
    const bool last_panel = (s - c0) <= NB;
    if (warp == 0) {
      int nsw = 0;
#pragma unroll
      for (int q = 0; q < K1W_Q; ++q) {
        const int i = lane + 32 * q;
        if (i >= k && i < s) Ak[q] = ld<C>(A, Ael(i, k), aim);
      }
      while (k < s) {
        const int kk = k - c0;
        if (!last_panel && kk >= NB - 1) break;
        double bv = -1.0, akk = 0.0;
        int bi = INT_MAX;
#pragma unroll
        for (int q = 0; q < K1W_Q; ++q) {
          const int i = lane + 32 * q;
          if (i < k || i >= s) continue;
          cz v = Ak[q];
          for (int m = 0; m < kk; ++m) v = fms<C>(v, Lget(i, m), Wget(k, m));
          wv[q] = v;
          Wset(i, kk, v);
          const double av = cabs1<C>(v);
          if (i == k) akk = av;
          else if (av > bv) {
            bv = av;
            bi = i;
          }
        }
        warp_argmax(bv, bi);
        const double absakk = __shfl_sync(0xffffffffu, akk, k & 31);
        const double colmax = bv > 0.0 ? bv : 0.0;
        const int imax = bi;
        int kp, kstep = 1;
        bool zero = false;
        if (fmax(absakk, colmax) == 0.0) {
          zero = true;
          kp = k;
        } else if (absakk >= alpha * colmax) {
          kp = k;
        } else {
          __syncwarp();
          double rv = -1.0;
          int ri = INT_MAX;
          cz ai[K1W_Q];  // column imax of the not-yet-updated trailing block: loads first
#pragma unroll
          for (int q = 0; q < K1W_Q; ++q) {
            const int i = lane + 32 * q;
            if (i >= k && i < s) ai[q] = (i < imax) ? ld<C>(A, Ael(imax, i), aim) : ld<C>(A, Ael(i, imax), aim);
          }
#pragma unroll
          for (int q = 0; q < K1W_Q; ++q) {
            const int i = lane + 32 * q;
            if (i < k || i >= s) continue;
            cz v = ai[q];
            for (int m = 0; m < kk; ++m) v = fms<C>(v, Lget(i, m), Wget(imax, m));
            wv2[q] = v;
            Wset(i, kk + 1, v);
            if (i != imax) {
              const double av = cabs1<C>(v);
              if (av > rv) {
                rv = av;
                ri = i;
              }
            }
          }
          warp_argmax(rv, ri);
          __syncwarp();
          const double rowmax = rv;
          if (absakk >= alpha * colmax * (colmax / rowmax)) {
            kp = k;
          } else {
            kp = imax;
            if (cabs1<C>(Wget(imax, kk + 1)) >= alpha * rowmax) {
#pragma unroll
              for (int q = 0; q < K1W_Q; ++q) {
                const int i = lane + 32 * q;
                if (i < k || i >= s) continue;
                wv[q] = wv2[q];
                Wset(i, kk, wv2[q]);
              }
            } else {
              kstep = 2;
            }
          }
        }
        __syncwarp();
        const int kkk = k + kstep - 1;
        if (kp != kkk) {
          {  // move column kkk of the trailing block to position kp: all loads first, then stores
            cz t0 = mk(0.0, 0.0), ta[K1W_Q], tb[K1W_Q];
            if (lane == 0) t0 = ld<C>(A, Ael(kkk, kkk), aim);
#pragma unroll
            for (int q = 0; q < K1W_Q; ++q) {
              const int j1 = kkk + 1 + lane + 32 * q, j2 = kp + 1 + lane + 32 * q;
              if (j1 < kp) ta[q] = ld<C>(A, Ael(j1, kkk), aim);
              if (j2 < s) tb[q] = ld<C>(A, Ael(j2, kkk), aim);
            }
            if (lane == 0) st<C>(A, Ael(kp, kp), aim, t0);
#pragma unroll
            for (int q = 0; q < K1W_Q; ++q) {
              const int j1 = kkk + 1 + lane + 32 * q, j2 = kp + 1 + lane + 32 * q;
              if (j1 < kp) st<C>(A, Ael(kp, j1), aim, ta[q]);
              if (j2 < s) st<C>(A, Ael(j2, kp), aim, tb[q]);
            }
          }
          for (int m = lane; m < kk; m += 32) {
            const cz x = Lget(kkk, m), y = Lget(kp, m);
            Lset(kkk, m, y);
            Lset(kp, m, x);
          }
          for (int m = lane; m < kk + kstep; m += 32) {
            const cz x = Wget(kkk, m), y = Wget(kp, m);
            Wset(kkk, m, y);
            Wset(kp, m, x);
          }
          if (lane == 0) {
            const int x = perm[kkk];
            perm[kkk] = perm[kp];
            perm[kp] = x;
            s_swa[nsw] = kkk;
            s_swb[nsw] = kp;
          }
          ++nsw;
          __syncwarp();
#pragma unroll
          for (int q = 0; q < K1W_Q; ++q) {
            const int i = lane + 32 * q;
            if (i == kkk || i == kp) {
              wv[q] = Wget(i, kk);
              if (kstep == 2) wv2[q] = Wget(i, kk + 1);
            }
          }
        }
        if (kstep == 1) {
          const cz D = Wget(k, kk);
          const cz rD = zero ? mk(1.0, 0.0) : dv<C>(mk(1.0, 0.0), D);
#pragma unroll
          for (int q = 0; q < K1W_Q; ++q) {
            const int i = lane + 32 * q;
            if (i <= k || i >= s) continue;
            Lset(i, kk, mul<C>(wv[q], rD));
          }
          if (lane == 0) {
            st<C>(dv_, k, aim, D);
            st<C>(ev_, k, aim, mk(0.0, 0.0));
            ipiv[k] = kp + 1;
            if (zero && zero_col < 0) zero_col = k;
            if (kp != k) ++nswap;
          }
        } else {
          const cz w11 = Wget(k, kk), w21 = Wget(k + 1, kk), w22 = Wget(k + 1, kk + 1);
          const cz d11 = dv<C>(w22, w21), d22 = dv<C>(w11, w21);
          const cz tt = dv<C>(mk(1.0, 0.0), mul<C>(d11, d22) - mk(1.0, 0.0));
          const cz d21 = dv<C>(tt, w21);
#pragma unroll
          for (int q = 0; q < K1W_Q; ++q) {
            const int i = lane + 32 * q;
            if (i <= k || i >= s) continue;
            cz l0 = mk(0.0, 0.0), l1 = mk(0.0, 0.0);
            if (i > k + 1) {
              l0 = mul<C>(d21, mul<C>(d11, wv[q]) - wv2[q]);
              l1 = mul<C>(d21, mul<C>(d22, wv2[q]) - wv[q]);
            }
            Lset(i, kk, l0);
            Lset(i, kk + 1, l1);
          }
          if (lane == 0) {
            st<C>(dv_, k, aim, w11);
            st<C>(dv_, k + 1, aim, w22);
            st<C>(ev_, k, aim, w21);
            st<C>(ev_, k + 1, aim, mk(0.0, 0.0));
            ipiv[k] = ipiv[k + 1] = -(kp + 1);
            ++n2x2;
            if (kp != k + 1) ++nswap;
          }
        }
        k += kstep;
        if (k < s && !(kk + kstep >= NB - 1 && !last_panel)) {
#pragma unroll
          for (int q = 0; q < K1W_Q; ++q) {
            const int i = lane + 32 * q;
            if (i >= k && i < s) Ak[q] = ld<C>(A, Ael(i, k), aim);
          }
        }
        __syncwarp();
      }
      if (lane == 0) {
        s_nswp = nsw;
        s_k = k;
      }
    }
    __syncthreads();
    k = s_k;
    // ------------------------------------------------------------ panel end (all warps)
    {
      const int kb = k - c0, nsw = s_nswp;
      for (int m = 0; m < kb; ++m) {
        const int col = c0 + m;
        for (int i = col + 1 + tid; i < s; i += NT1W) st<C>(A, Ael(i, col), aim, Lget(i, m));
        if (tid == 0) st<C>(A, Ael(col, col), aim, ld<C>(dv_, col, aim));
      }
      if (k < s)  // W panel rows >= k for the trailing GEMM
        for (int m = 0; m < kb; ++m)
          for (int i = k + tid; i < s; i += NT1W) st<C>(Wg, (int64_t)i + (int64_t)m * ldW, wim, Wget(i, m));
      for (int j = tid; j < c0; j += NT1W)
        for (int q = 0; q < nsw; ++q) {
          const int r0 = s_swa[q], r1 = s_swb[q];
          const cz x = ld<C>(A, Ael(r0, j), aim), y = ld<C>(A, Ael(r1, j), aim);
          st<C>(A, Ael(r0, j), aim, y);
          st<C>(A, Ael(r1, j), aim, x);
        }
    }
    __threadfence();
    __syncthreads();
    if (k < s) {  // trailing update A(k:s, k:s) -= L(k:s, c0:k) W(k:s, 0:kb)^T on DMMA (4 warps)
      const int kb = k - c0, ke = k & ~1, M = s - ke;
      Seg sg;
      sg.a = A + Ael(ke, c0);
      sg.lda = ldA;
      sg.b = Wg + ke;
      sg.ldb = ldW;
      sg.acol = nullptr;
      sg.K = kb;
      const int nt = (M + 63) / 64;
      for (int tm = 0; tm < nt; ++tm)
        for (int tn = 0; tn <= tm; ++tn) {
          typename G::Acc acc;
          G::zero(acc);
          G::run([&](int) { return sg; }, 1, tm * 64, tn * 64, M, M, aim, wim, smem, acc,
                 G::tile_mask(M - tm * 64, M - tn * 64, tn * 64 - tm * 64));
          double* Cb = A + Ael(ke + tm * 64, ke + tn * 64);
          if (ke < k) {  // row / column ke (already eliminated) must stay: subtract exact zeros there
            G::for_each_mut(acc, [&](int r, int c, double& vr, double& vi) {
              if ((tm == 0 && r == 0) || (tn == 0 && c == 0)) vr = vi = 0.0;
            });
          }
          // coalesced read-modify-write (all loads of a batch in flight before the stores)
          G::template store_tile<1>(acc, smem, Cb, ldA, aim, M - tm * 64, M - tn * 64);
        }
      __syncthreads();
    }
  }
  k1_finish<C>(a, t, nd, A, smem, perm, ipiv, dv_, ev_, n2x2, nswap, zero_col);
}

size_t k1w_smem(bool cplx, int max_s) {
  size_t lp = (size_t)max_s * K1NB * 8 * (cplx ? 2 : 1) * 2;  // Lp + Wp
  size_t g = cplx ? K1WGemmC::SMEM_BYTES : K1WGemmR::SMEM_BYTES;
  size_t inv = (size_t)(NT1W / 32) * 2 * TB * TB * sizeof(double);
  return std::max(lp, std::max(g, inv));
}

#endif  // DD_AUX_AB

// ============================================================================ full inverse of L_tt
// X = L_tt^{-1} (unit lower) by column tiles of width TB, one CTA per (node, column tile c):
//   X_cc = Linv_cc (the K1 tile inverse);  X_pc = -Linv_pp * sum_{q=c}^{p-1} L_pq X_qc  (p > c)
// (block forward substitution with identity right-hand side; strictly-upper part zeroed so the
// solve's diagonal GEMMs may read whole row panels).  Lets every diagonal solve of dd_aux_solve
// run as one parallel M-tiled DMMA GEMM instead of a sequential panel chain.
using LinvG_R = Gemm<32, 32, 16, 1, 4, 2, false, false, true>;
using LinvG_C = Gemm<32, 32, 16, 1, 4, 2, true, false, true>;

template <bool C>
__global__ void __launch_bounds__(128) k_linv(LinvArgs a) {
  using G = typename std::conditional<C, LinvG_C, LinvG_R>::type;
  extern __shared__ __align__(16) double smem[];
  const DTile it = a.items[blockIdx.x];
  const NodeDev nd = a.nd[it.t];
  const int s = nd.s, c = it.tm, c0 = c * TB, wc = min(TB, s - c0);
  const int64_t ldi = nd.ldi, ldA = nd.ld, aim = a.aim;
  double* X = a.arena + nd.inv;
  const double* P = a.arena + nd.panel;
  const double* Lt = a.arena + nd.linv;
  // zero rows [0, c0) of the column tile (strictly upper part) and write X_cc
  for (int e = threadIdx.x; e < c0 * wc; e += blockDim.x) {
    const int r = e % c0, q = e / c0;
    st<C>(X, r + (int64_t)(c0 + q) * ldi, aim, mk(0.0, 0.0));
  }
  for (int e = threadIdx.x; e < wc * wc; e += blockDim.x) {
    const int r = e % wc, q = e / wc;
    st<C>(X, (c0 + r) + (int64_t)(c0 + q) * ldi, aim, ld<C>(Lt, (int64_t)c * TB * TB + r + (int64_t)q * TB, aim));
  }
  __syncthreads();  // orders the CTA's global stores before its cp.async reads
  const int np = (s + TB - 1) / TB;
  for (int p = c + 1; p < np; ++p) {
    const int p0 = p * TB, wp = min(TB, s - p0);
    typename G::Acc acc;
    G::zero(acc);
    {  // acc = L(p0:p0+wp, c0:p0) X(c0:p0, c0:c0+wc)
      Seg sg{P + p0 + (int64_t)c0 * ldA, X + c0 + (int64_t)c0 * ldi, nullptr, ldA, ldi, p0 - c0};
      G::run([&](int) { return sg; }, 1, 0, 0, wp, wc, aim, aim, smem, acc);
    }
    double* Xp = X + p0 + (int64_t)c0 * ldi;
    G::for_each(acc, [&](int r, int q, double vr, double vi) {
      if (r < wp && q < wc) {
        Xp[r + (int64_t)q * ldi] = vr;
        if (C) Xp[r + (int64_t)q * ldi + aim] = vi;
      }
    });
    __syncthreads();
    G::zero(acc);
    {  // X_pc = -Linv_pp acc
      Seg sg{Lt + (int64_t)p * TB * TB, Xp, nullptr, (int64_t)TB, ldi, wp};
      G::run([&](int) { return sg; }, 1, 0, 0, wp, wc, aim, aim, smem, acc);
    }
    G::for_each(acc, [&](int r, int q, double vr, double vi) {
      if (r < wp && q < wc) {
        Xp[r + (int64_t)q * ldi] = -vr;
        if (C) Xp[r + (int64_t)q * ldi + aim] = -vi;
      }
    });
    __syncthreads();
  }
}

// ============================================================================ row permutation
// rows [ro, ro + s_t) of panel k are block t's rows of L_tk; reorder them by perm_t.
template <bool C>
__global__ void k_rowperm(RowpermArgs a, int nlist) {
  for (int li = blockIdx.y; li < nlist; li += gridDim.y) {  // grid-stride (gridDim.y <= 65535)
  const RowPerm R = a.list[li];
  const NodeDev nt = a.nd[R.t];
  const NodeDev nk = a.nd[R.k];
  const int s = nt.s;
  const int* perm = a.perm + nt.ydof;
  extern __shared__ __align__(16) double sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  double* br = sm + (size_t)warp * 2 * s;
  double* bi = br + s;
  for (int c = blockIdx.x * nw + warp; c < nk.s; c += gridDim.x * nw) {
    double* col = a.arena + nk.panel + R.ro + (int64_t)c * nk.ld;
    for (int m = lane; m < s; m += 32) {
      br[m] = col[perm[m]];
      if (C) bi[m] = col[perm[m] + a.aim];
    }
    __syncwarp();
    for (int m = lane; m < s; m += 32) {
      col[m] = br[m];
      if (C) col[m + a.aim] = bi[m];
    }
    __syncwarp();
  }
  }
}

// ============================================================================ K3 Schur update
// Tile configurations (selected at analyze time; env DD_AUX_K3CFG):
//   0: real 128x128 / complex 64x128, 8 warps, 1 CTA per SM
//   1: real 128x64  / complex 64x64,  4 warps, 2 CTAs per SM (prologue/epilogue of one CTA
//      overlap the MMA of the other)
template <bool C, int CFG>
struct K3Cfg;
#ifdef DD_AUX_AB
template <>
struct K3Cfg<false, 0> {
  using G = Gemm<128, 128, 16, 2, 4, 4, false, false, false>;
  static constexpr int NT = 256, BM = 128, BN = 128, MINB = 1;
};
#endif
#ifdef DD_AUX_AB
template <>
struct K3Cfg<true, 0> {
  using G = Gemm<64, 128, 16, 2, 4, 3, true, false, false>;
  static constexpr int NT = 256, BM = 64, BN = 128, MINB = 1;
};
#endif
#ifdef DD_AUX_AB
template <>
struct K3Cfg<false, 1> {
  using G = Gemm<128, 64, 16, 2, 2, 3, false, false, false>;
  static constexpr int NT = 128, BM = 128, BN = 64, MINB = 2;
};
#endif
#ifdef DD_AUX_AB
template <>
struct K3Cfg<true, 1> {
  using G = Gemm<64, 64, 16, 2, 2, 3, true, false, false>;
  static constexpr int NT = 128, BM = 64, BN = 64, MINB = 2;
};
#endif

#ifdef DD_AUX_AB
template <>
struct K3Cfg<false, 2> {  // real 128x64, 4 stages (deeper prefetch for DRAM-resident W panels)
  using G = Gemm<128, 64, 16, 2, 2, 4, false, false, false>;
  static constexpr int NT = 128, BM = 128, BN = 64, MINB = 2;
};
#endif
#ifdef DD_AUX_AB
template <>
struct K3Cfg<true, 2> {
  using G = Gemm<64, 64, 16, 2, 2, 4, true, false, false>;
  static constexpr int NT = 128, BM = 64, BN = 64, MINB = 1;
};
#endif

#ifdef DD_AUX_AB
template <>
struct K3Cfg<false, 3> {  // real 128x64, register-capped for 3 CTAs per SM (12 warps)
  using G = Gemm<128, 64, 16, 2, 2, 3, false, false, false>;
  static constexpr int NT = 128, BM = 128, BN = 64, MINB = 3;
};
#endif
#ifdef DD_AUX_AB
template <>
struct K3Cfg<true, 3> {
  using G = Gemm<64, 64, 16, 2, 2, 3, true, false, false>;
  static constexpr int NT = 128, BM = 64, BN = 64, MINB = 2;
};
#endif
#ifdef DD_AUX_AB
template <>
struct K3Cfg<false, 4> {  // real 64x64, 4 CTAs per SM (16 warps), least ragged-tile padding
  using G = Gemm<64, 64, 16, 2, 2, 3, false, false, false>;
  static constexpr int NT = 128, BM = 64, BN = 64, MINB = 4;
};
#endif
#ifdef DD_AUX_AB
template <>
struct K3Cfg<true, 4> {
  using G = Gemm<64, 64, 16, 2, 2, 3, true, false, false>;
  static constexpr int NT = 128, BM = 64, BN = 64, MINB = 2;
};
#endif

#ifdef DD_AUX_AB
template <>
struct K3Cfg<false, 5> {  // real 64x32, 3 stages, 5 CTAs per SM
  using G = Gemm<64, 32, 16, 2, 2, 3, false, false, false>;
  static constexpr int NT = 128, BM = 64, BN = 32, MINB = 5;
};
#endif
#ifdef DD_AUX_AB
template <>
struct K3Cfg<true, 5> {  // complex 64x32, 2 stages, 4 CTAs per SM (dense microbench: 94% of ZGEMM)
  using G = Gemm<64, 32, 16, 2, 2, 2, true, false, false>;
  static constexpr int NT = 128, BM = 64, BN = 32, MINB = 4;
};
#endif

#ifdef DD_AUX_AB
template <>
struct K3Cfg<false, 6> {
  using G = Gemm<64, 64, 16, 2, 2, 3, false, false, false>;
  static constexpr int NT = 128, BM = 64, BN = 64, MINB = 4;
};
#endif
#ifdef DD_AUX_AB
template <>
struct K3Cfg<true, 6> {  // complex 64x32 3M (Gauss): 3 real DMMA products per complex product
  using G = Gemm<64, 32, 16, 2, 2, 2, true, false, false, true>;
  static constexpr int NT = 128, BM = 64, BN = 32, MINB = 4;
};
#endif

#ifdef DD_AUX_AB
template <>
struct K3Cfg<false, 7> {  // real 64x64, coarse (per-warp) masking
  using G = Gemm<64, 64, 16, 2, 2, 3, false, false, false, false, false>;
  static constexpr int NT = 128, BM = 64, BN = 64, MINB = 4;
};
#endif
#ifdef DD_AUX_AB
template <>
struct K3Cfg<true, 7> {  // complex 64x32 4M, coarse masking
  using G = Gemm<64, 32, 16, 2, 2, 2, true, false, false, false, false>;
  static constexpr int NT = 128, BM = 64, BN = 32, MINB = 4;
};
#endif
#ifdef DD_AUX_AB
template <>
struct K3Cfg<false, 8> {
  using G = Gemm<64, 64, 16, 2, 2, 3, false, false, false, false, false>;
  static constexpr int NT = 128, BM = 64, BN = 64, MINB = 4;
};
#endif
#ifdef DD_AUX_AB
template <>
struct K3Cfg<true, 8> {  // complex 64x32 3M, coarse masking
  using G = Gemm<64, 32, 16, 2, 2, 2, true, false, false, true, false>;
  static constexpr int NT = 128, BM = 64, BN = 32, MINB = 4;
};
#endif

template <>
struct K3Cfg<false, 9> {  // real 64x64, coarse masking, vectorised (16-byte) fragment loads
  using G = Gemm<64, 64, 16, 2, 2, 3, false, false, false, false, false, true>;
  static constexpr int NT = 128, BM = 64, BN = 64, MINB = 4;
};
template <>
struct K3Cfg<true, 9> {  // complex 64x32 3M, vectorised fragment loads, fast loader at 3 CTAs/SM (162 registers, no spills; at 4 CTAs/SM the fast loader spills: 21 TF/s; generic loader at 4 CTAs/SM: 38.5 vs 40.0 effective TF/s on cfg3)
  using G = Gemm<64, 32, 16, 2, 2, 2, true, false, false, true, true, true>;
  static constexpr int NT = 128, BM = 64, BN = 32, MINB = 3;
};
template <>
struct K3Cfg<false, 10> {  // real 64x64, per-sub-tile masking, vectorised fragment loads
  using G = Gemm<64, 64, 16, 2, 2, 3, false, false, false, false, true, true>;
  static constexpr int NT = 128, BM = 64, BN = 64, MINB = 4;
};
template <>
struct K3Cfg<true, 10> {  // complex 64x32 4M, coarse masking, vectorised fragment loads
  using G = Gemm<64, 32, 16, 2, 2, 2, true, false, false, false, false, true>;
  static constexpr int NT = 128, BM = 64, BN = 32, MINB = 4;
};

#ifdef DD_AUX_AB
template <>
struct K3Cfg<false, 11> {  // real 64x64, VEC, rectangular 16x16-granular edge masking (RECT)
  using G = Gemm<64, 64, 16, 2, 2, 3, false, false, false, false, false, true, true>;
  static constexpr int NT = 128, BM = 64, BN = 64, MINB = 4;
};
#endif
#ifdef DD_AUX_AB
template <>
struct K3Cfg<true, 11> {  // complex 64x32 3M, VEC, RECT
  using G = Gemm<64, 32, 16, 2, 2, 2, true, false, false, true, false, true, true>;
  static constexpr int NT = 128, BM = 64, BN = 32, MINB = 4;
};
#endif
#ifdef DD_AUX_AB
template <>
struct K3Cfg<false, 12> {  // real 64x64, scalar fragments, RECT (16x8-granular)
  using G = Gemm<64, 64, 16, 2, 2, 3, false, false, false, false, false, false, true>;
  static constexpr int NT = 128, BM = 64, BN = 64, MINB = 4;
};
#endif
#ifdef DD_AUX_AB
template <>
struct K3Cfg<true, 12> {  // complex 64x32 4M, VEC, RECT
  using G = Gemm<64, 32, 16, 2, 2, 2, true, false, false, false, false, true, true>;
  static constexpr int NT = 128, BM = 64, BN = 32, MINB = 4;
};
#endif

template <>
struct K3Cfg<false, 13> {  // real 64x64, RECT, BK = 24, 2 stages (52 KB smem, 4 CTAs/SM): 2/3 of the stage barriers per flop of BK = 16 (cfg2: 29.9 -> 30.5 TF/s; BK = 32 only fits 3 CTAs/SM: 26.4)
  using G = Gemm<64, 64, 24, 2, 2, 2, false, false, false, false, false, false, true>;
  static constexpr int NT = 128, BM = 64, BN = 64, MINB = 4;
};
template <>
struct K3Cfg<true, 13> {  // complex 64x32 3M, 2 stages, coarse masking (no per-mma predicates)
  using G = Gemm<64, 32, 16, 2, 2, 2, true, false, false, true, false, false, false, false, false>;
  static constexpr int NT = 128, BM = 64, BN = 32, MINB = 4;
};

#ifdef DD_AUX_AB
template <>
struct K3Cfg<false, 14> {  // real 64x64, RECT, 3 stages, mbarrier pipeline (no CTA barrier per stage)
  using G = Gemm<64, 64, 16, 2, 2, 3, false, false, false, false, false, false, true, true>;
  static constexpr int NT = 128, BM = 64, BN = 64, MINB = 4;
};
#endif
#ifdef DD_AUX_AB
template <>
struct K3Cfg<true, 14> {  // complex 64x32 3M VEC, 3 stages, mbarrier pipeline
  using G = Gemm<64, 32, 16, 2, 2, 3, true, false, false, true, true, true, false, true>;
  static constexpr int NT = 128, BM = 64, BN = 32, MINB = 3;
};
#endif

#ifdef DD_AUX_AB
template <>
struct K3Cfg<false, 15> {  // cfg 13 register-capped for 5 CTAs per SM (20 warps)
  using G = Gemm<64, 64, 16, 2, 2, 2, false, false, false, false, false, false, true>;
  static constexpr int NT = 128, BM = 64, BN = 64, MINB = 5;
};
#endif
#ifdef DD_AUX_AB
template <>
struct K3Cfg<true, 15> {  // complex 64x32 3M VEC, 5 CTAs per SM
  using G = Gemm<64, 32, 16, 2, 2, 2, true, false, false, true, true, true>;
  static constexpr int NT = 128, BM = 64, BN = 32, MINB = 5;
};
#endif
#ifdef DD_AUX_AB
template <>
struct K3Cfg<false, 16> {  // real 64x64, RECT, BK = 16, 2 stages (the default before BK = 24)
  using G = Gemm<64, 64, 16, 2, 2, 2, false, false, false, false, false, false, true>;
  static constexpr int NT = 128, BM = 64, BN = 64, MINB = 4;
};
template <>
struct K3Cfg<true, 16> {
  using G = Gemm<64, 32, 32, 2, 2, 2, true, false, false, true, false, false, false>;
  static constexpr int NT = 128, BM = 64, BN = 32, MINB = 3;
};
template <>
struct K3Cfg<false, 17> {  // real 128x64, 8 warps of 32x32, 3 stages, RECT (2 CTAs/SM, 16 warps; 4 warps of 64x32: 24.5 TF/s on cfg2)
  using G = Gemm<128, 64, 16, 4, 2, 3, false, false, false, false, false, false, true>;
  static constexpr int NT = 256, BM = 128, BN = 64, MINB = 2;
};
template <>
struct K3Cfg<true, 17> {
  using G = Gemm<64, 64, 16, 2, 2, 2, true, false, false, true, false, false, false>;
  static constexpr int NT = 128, BM = 64, BN = 64, MINB = 2;
};
template <>
struct K3Cfg<false, 18> {  // real 64x64, 8 warps of 32x16, 2 stages, RECT (3 CTAs/SM, 24 warps; 64x128 with 4 warps: 22.9 TF/s on cfg2)
  using G = Gemm<64, 64, 16, 2, 4, 2, false, false, false, false, false, false, true>;
  static constexpr int NT = 256, BM = 64, BN = 64, MINB = 3;
};
template <>
struct K3Cfg<true, 18> {
  using G = Gemm<64, 32, 16, 2, 2, 2, true, false, false, true, true, true>;
  static constexpr int NT = 128, BM = 64, BN = 32, MINB = 4;
};
template <>
struct K3Cfg<false, 19> {  // = 13
  using G = Gemm<64, 64, 16, 2, 2, 2, false, false, false, false, false, false, true>;
  static constexpr int NT = 128, BM = 64, BN = 64, MINB = 4;
};
template <>
struct K3Cfg<true, 19> {  // complex 64x32 3M VEC, generic loader, 4 CTAs/SM (the default before the fast loader at 3 CTAs/SM)
  using G = Gemm<64, 32, 16, 2, 2, 2, true, false, false, true, true, true, false, false, false>;
  static constexpr int NT = 128, BM = 64, BN = 32, MINB = 4;
};
#endif

// One output tile of the Schur update (the body of both K3 launch forms).
template <bool C, int CFG>
__device__ __forceinline__ void k3_tile(const K3Args& a, int64_t blk, double* smem) {
  using Cf = K3Cfg<C, CFG>;
  using G = typename Cf::G;
  constexpr int BM = Cf::BM, BN = Cf::BN;
  // implicit tiles: find this CTA's target (last t with tprefix[t] <= gid) and its (tm, tn)
  const int64_t gid = a.tile0 + blk;
  int lo = 0, hi = a.ntargets - 1;
#ifndef DDK_K3_SEARCH32
#define DDK_K3_SEARCH32 1
#endif
  if (DDK_K3_SEARCH32) {
    // 32-ary search: each round every lane probes one of 32 evenly spaced candidates at once (one
    // dependent global latency per round instead of one per halving); every warp finds the same t
    const int lane = threadIdx.x & 31;
    while (lo < hi) {
      const int step = (hi - lo + 31) >> 5;  // >= 1
      const int pidx = lo + 1 + lane * step;
      const bool ok = pidx <= hi && a.tprefix[pidx] <= gid;
      const unsigned m = __ballot_sync(0xffffffffu, ok);
      if (m == 0u) {
        hi = lo;
      } else {
        const int j = 31 - __clz(m);  // the last candidate with tprefix <= gid (tprefix ascending)
        lo = lo + 1 + j * step;
        hi = min(hi, lo + step - 1);
      }
    }
  } else {
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (a.tprefix[mid] <= gid) lo = mid;
      else hi = mid - 1;
    }
  }
  const UpdTarget tg = a.targets[lo];
  Tile T;
  {
    int local = (int)(gid - a.tprefix[lo]);
    const int ntn = (tg.N + BN - 1) / BN;
    T.tm = 0;
    if (!tg.diag) {
      T.tm = local / ntn;
      T.tn = local % ntn;
    } else {
      for (;;) {
        const int rowt = min(ntn, (T.tm * BM + BM - 1) / BN + 1);
        if (local < rowt) break;
        local -= rowt;
        ++T.tm;
      }
      T.tn = local;
    }
  }
  const NodeDev nj = a.nd[tg.j];
  typename G::Acc acc;
  G::zero(acc);
  const UpdContrib* cl = a.contribs + tg.c0;
  auto gseg = [&](int q) {
    const UpdContrib u = cl[q];
    const NodeDev nk = a.nd[u.k];
    Seg sg;
    sg.a = a.work + nk.w + u.arow;          // W_ik
    sg.lda = nk.ldw;
    sg.b = a.arena + nk.panel + u.brow;     // B(q, n) = L_jk(n, q)
    sg.ldb = nk.ld;
    sg.acol = nullptr;
    sg.K = nk.s;
    return sg;
  };
  // the first K3_SEGC contributor descriptors are fetched once, in parallel, into shared memory
  // (a segment switch inside the pipeline then costs no dependent global round trips)
#ifndef DDK_SEGC
#define DDK_SEGC 0
#endif
  constexpr int K3_SEGC = DDK_SEGC > 0 ? DDK_SEGC : 1;
  __shared__ Seg segc[K3_SEGC];
  const int ncon = tg.c1 - tg.c0;
  if (DDK_SEGC > 0) {
    if ((int)threadIdx.x < min(ncon, K3_SEGC)) segc[threadIdx.x] = gseg(threadIdx.x);
    __syncthreads();
  }
  auto segfn = [&](int q) { return (DDK_SEGC > 0 && q < K3_SEGC) ? segc[q] : gseg(q); };
  const int mlim = tg.M - T.tm * BM, nlim = tg.N - T.tn * BN;
#ifndef DDK_K3_ALIAS
#define DDK_K3_ALIAS 0  // measured slower on cfg2 (30.16 -> 29.64 TF/s: register spills on the aliased path, 2-4 extra barriers in its epilogue); A/B switch
#endif
  // ragged tiles (valid rows / columns within one warp row / column): the otherwise idle warps
  // share the k-steps of the occupied warp tiles (gemm_core.cuh "warp aliasing")
  const unsigned amap = DDK_K3_ALIAS ? G::alias_map(mlim, nlim) : 0u;
  const int diag_off = tg.diag ? T.tn * BN - T.tm * BM : G::NO_DIAG;
  double* Cb = a.arena + nj.panel + tg.ro + (int64_t)T.tm * BM + (int64_t)T.tn * BN * nj.ld;
#ifndef DDK_K3_RED
#define DDK_K3_RED 1
#endif
  constexpr int EPI = DDK_K3_RED ? 2 : 1;  // 2: L2 reductions (no C read round trip); 1: read-modify-write
  if (EPI == 1) G::prefetch_tile_l2(Cb, nj.ld, a.aim, mlim, nlim);
  unsigned mask;
  if (amap) {  // CTA-uniform
    mask = G::tile_mask(mlim, nlim, diag_off, true);
    G::template run<true>(segfn, tg.c1 - tg.c0, T.tm * BM, T.tn * BN, tg.M, tg.N, a.wim, a.aim, smem, acc, mask);
  } else {
    mask = G::tile_mask(mlim, nlim, diag_off);
    G::run(segfn, tg.c1 - tg.c0, T.tm * BM, T.tn * BN, tg.M, tg.N, a.wim, a.aim, smem, acc, mask);
  }
  G::template store_tile<EPI>(acc, smem, Cb, nj.ld, a.aim, mlim, nlim, amap, mask != 0u);
}

template <bool C, int CFG>
__global__ void __launch_bounds__(K3Cfg<C, CFG>::NT, K3Cfg<C, CFG>::MINB) k3_update(K3Args a) {
  extern __shared__ __align__(16) double smem[];
  k3_tile<C, CFG>(a, blockIdx.x, smem);
}

#ifdef DD_AUX_AB
// Persistent form (A/B, DD_AUX_K3PERSIST=1): one CTA per resident slot, tiles taken from a
// dynamic counter in launch (cost-descending) order, so no CTA is launched per tile and the
// largest-K tiles start first (LPT-like load balance across the SMs).
template <bool C, int CFG>
__global__ void __launch_bounds__(K3Cfg<C, CFG>::NT, K3Cfg<C, CFG>::MINB) k3_update_persist(K3Args a) {
  extern __shared__ __align__(16) double smem[];
  __shared__ long long s_tile;
  for (;;) {
    if (threadIdx.x == 0) s_tile = (long long)atomicAdd(a.counter, 1ull);
    __syncthreads();
    const long long t = s_tile;
    __syncthreads();
    if (t >= a.ntiles) return;
    k3_tile<C, CFG>(a, t, smem);
  }
}
#endif  // DD_AUX_AB

// ============================================================================ K2 panel TRSM
// W_t = (A_struct,t P_t^T) L_tt^{-T} as ONE tiled DMMA GEMM per level using the full inverse
// X = L_tt^{-1} from k_linv: W(m, n) = sum_{k <= n} Ahat(m, perm[k]) X(n, k) -- the column
// permutation P_t^T is a gather in the A loader, the triangle of X bounds K per column tile.
// Then k2_dinv forms L = W D^{-1} (1x1 / 2x2, LAPACK scaled form) in place of A_struct,t.
template <bool C, int CFG>
__global__ void __launch_bounds__(K3Cfg<C, CFG>::NT, K3Cfg<C, CFG>::MINB) k2_gemm(K2Args a) {
  using Cf = K3Cfg<C, CFG>;
  using G = typename Cf::G;
  constexpr int BM = Cf::BM, BN = Cf::BN;
  extern __shared__ __align__(16) double smem[];
  const Tile T = a.items[blockIdx.x];
  const NodeDev nd = a.nd[T.target];
  const int s = nd.s, m0 = T.tm * BM, n0 = T.tn * BN;
  // the column gather map (P_t) of the K range goes to shared memory first: the loader then
  // never waits on a dependent global load before its cp.async
  int* pcol = reinterpret_cast<int*>(smem + G::SMEM_BYTES / sizeof(double));
  const int kmax = min(s, n0 + BN);
  for (int q = threadIdx.x; q < kmax; q += blockDim.x) pcol[q] = a.perm[nd.ydof + q];
  __syncthreads();
  Seg sg;
  sg.a = a.arena + nd.panel + nd.sp;   // Ahat rows (struct part), columns gathered by perm
  sg.lda = nd.ld;
  sg.acol = pcol;
  sg.b = a.arena + nd.inv;             // B(k, n) = X(n, k)
  sg.ldb = nd.ldi;
  sg.K = min(s, n0 + BN);
  typename G::Acc acc;
  G::zero(acc);
  const int mlim = nd.rp - m0, nlim = s - n0;
  G::run([&](int) { return sg; }, 1, m0, n0, nd.rp, s, a.aim, a.aim, smem, acc,
         G::tile_mask(mlim, nlim, G::NO_DIAG));
  double* W = a.work + nd.w + m0 + (int64_t)n0 * nd.ldw;
  G::template store_tile<0>(acc, smem, W, nd.ldw, a.wim, mlim, nlim);
}

constexpr int NT2 = 128;
template <bool C>
__global__ void __launch_bounds__(NT2) k2_dinv(K2Args a) {
  const Strip S = a.strips[blockIdx.x];
  const NodeDev nd = a.nd[S.t];
  const int s = nd.s, M = S.nrows;
  const int64_t ldA = nd.ld, ldW = nd.ldw, aim = a.aim, wim = a.wim;
  double* Ahat = a.arena + nd.panel + nd.sp + S.row0;
  const double* W = a.work + nd.w + S.row0;
  const double* dv_ = a.arena + a.d_off + nd.ydof;
  const double* ev_ = a.arena + a.e_off + nd.ydof;
  const int* ipiv = a.ipiv + nd.ydof;
  double maxl = 0.0;
  for (int c = blockIdx.y; c < s; c += gridDim.y) {
    const bool two = ipiv[c] < 0;
    // a 2x2 pivot is only taken when colmax > 0, so e != 0 exactly on the first column of a pair
    const cz e0 = ld<C>(ev_, c, aim);
    const int c1 = (two && (e0.r != 0.0 || e0.i != 0.0)) ? c : c - 1;
    for (int r = threadIdx.x; r < M; r += NT2) {
      const int64_t e = (int64_t)r + (int64_t)c * ldW;
      cz out;
      if (!two) {
        const cz d = ld<C>(dv_, c, aim), wv = ld<C>(W, e, wim);
        out = (d.r == 0.0 && d.i == 0.0) ? wv : dv<C>(wv, d);
      } else {
        const cz d11 = ld<C>(dv_, c1, aim), d22 = ld<C>(dv_, c1 + 1, aim), d21 = ld<C>(ev_, c1, aim);
        const cz wk = ld<C>(W, (int64_t)r + (int64_t)c1 * ldW, wim),
                 wk1 = ld<C>(W, (int64_t)r + (int64_t)(c1 + 1) * ldW, wim);
        const cz a11 = dv<C>(d22, d21), a22 = dv<C>(d11, d21);
        const cz tt = dv<C>(mk(1.0, 0.0), mul<C>(a11, a22) - mk(1.0, 0.0));
        const cz s21 = dv<C>(tt, d21);
        out = (c == c1) ? mul<C>(s21, mul<C>(a11, wk) - wk1) : mul<C>(s21, mul<C>(a22, wk1) - wk);
      }
      maxl = fmax(maxl, modulus<C>(out));
      st<C>(Ahat, (int64_t)r + (int64_t)c * ldA, aim, out);
    }
  }
  warp_max_to(a.maxL, maxl);
}

// ============================================================================ K4 stats
__global__ void k4_stats(const int64_t* __restrict__ node_stats, int nnodes, const int* __restrict__ gperm,
                         int64_t* __restrict__ out) {
  constexpr int NQ = 8;  // npos, nneg, nzero, n2x2, nswaps, first-zero key (min), nperturbed, nonfinite
  __shared__ int64_t sh[8][NQ];
  int64_t acc[NQ] = {0, 0, 0, 0, 0, INT64_MAX, 0, 0};
  for (int t = threadIdx.x; t < nnodes; t += blockDim.x) {
    const int64_t* S = node_stats + (int64_t)t * 8;
    for (int q = 0; q < NQ; ++q)
      if (q != 5) acc[q] += S[q];
    if (S[5] > 0 && S[5] < acc[5]) acc[5] = S[5];  // elimination-order key of the first zero pivot
  }
  // simple two-level reduction (256 threads)
  for (int q = 0; q < NQ; ++q) {
    int64_t v = acc[q];
    for (int o = 16; o; o >>= 1) {
      int64_t u = __shfl_xor_sync(0xffffffffu, v, o);
      v = (q == 5) ? (u < v ? u : v) : v + u;
    }
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5][q] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t r[NQ] = {0, 0, 0, 0, 0, INT64_MAX, 0, 0};
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w)
      for (int q = 0; q < NQ; ++q) r[q] = (q == 5) ? (sh[w][q] < r[q] ? sh[w][q] : r[q]) : r[q] + sh[w][q];
    for (int q = 0; q < NQ; ++q) out[q] = r[q];
    // position row -> 1 + original DoF (gperm is final once every level's K1 has run)
    out[5] = r[5] == INT64_MAX ? 0 : (int64_t)gperm[r[5] - 1] + 1;
  }
}

// ============================================================================ launchers
template <class K>
static void set_smem(K kern, size_t bytes) {
  if (bytes > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

void launch_load(bool cplx, const double* vals, const LoadBlock* lb, int nblocks, int64_t max_elems, double* arena,
                 int64_t aim, cudaStream_t st) {
  if (nblocks == 0) return;
  int gx = (int)std::min<int64_t>((max_elems + 255) / 256, 64);
  dim3 grid(gx, std::min(nblocks, 65535));
  if (cplx) k0_load<true><<<grid, 256, 0, st>>>(vals, lb, nblocks, arena, aim);
  else k0_load<false><<<grid, 256, 0, st>>>(vals, lb, nblocks, arena, aim);
}

size_t k1_smem(bool cplx, int max_s, int nb_req) {
  size_t g = cplx ? K1GemmC::SMEM_BYTES : K1GemmR::SMEM_BYTES;
  size_t inv = (size_t)(NT1 / 32) * 2 * TB * TB * sizeof(double);
  size_t m = g > inv ? g : inv;
  // the budget covers the largest block of the launch; smaller blocks pick widths that fit it too
  const size_t lp = k1_panel_bytes(max_s, cplx, k1_panel_nb(max_s, cplx, nb_req));
  return std::max<size_t>(std::max(m, lp), (size_t)K1_SMEM_BUDGET);
}

template <bool C, int Q>
static void launch_k1_t(const K1Args& a, int nnodes, int max_s, cudaStream_t st) {
  const size_t sm = k1_smem(C, max_s, a.nb);
  set_smem(k1_diag_bk<C, Q>, sm);
  k1_diag_bk<C, Q><<<nnodes, NT1, sm, st>>>(a);
}

void launch_k1(bool cplx, const K1Args& a, int nnodes, int max_s, cudaStream_t st) {
  // warp variant: opt-in (DD_AUX_K1WARP=1); measured slower than the 256-thread kernel on cfg1
  // (59 vs 42 ms), kept for the next round's latency work
#ifdef DD_AUX_AB
  static const bool warp = getenv("DD_AUX_K1WARP") && atoi(getenv("DD_AUX_K1WARP"));
  if (warp && max_s <= (cplx ? 128 : 256)) {
    const size_t sm = k1w_smem(cplx, max_s);
    if (cplx) {
      set_smem(k1_diag_bk_warp<true>, sm);
      k1_diag_bk_warp<true><<<nnodes, NT1W, sm, st>>>(a);
    } else {
      set_smem(k1_diag_bk_warp<false>, sm);
      k1_diag_bk_warp<false><<<nnodes, NT1W, sm, st>>>(a);
    }
    return;
  }
#endif
  // rows per thread sized to the level's largest block: the per-row loops are unrolled over
  // K1_MAXQ, so a tighter bound removes dead per-column work for small interfaces
  static const int maxq_env = getenv("DD_AUX_K1MAXQ") ? atoi(getenv("DD_AUX_K1MAXQ")) : 0;
  if (max_s <= NT1 && maxq_env != 4) {
    if (cplx) launch_k1_t<true, 1>(a, nnodes, max_s, st);
    else launch_k1_t<false, 1>(a, nnodes, max_s, st);
  } else if (max_s <= NT1 * 2 && maxq_env != 4) {
    if (cplx) launch_k1_t<true, 2>(a, nnodes, max_s, st);
    else launch_k1_t<false, 2>(a, nnodes, max_s, st);
  } else if (max_s <= NT1 * 4) {
    if (cplx) launch_k1_t<true, 4>(a, nnodes, max_s, st);
    else launch_k1_t<false, 4>(a, nnodes, max_s, st);
  } else {
    if (cplx) launch_k1_t<true, 16>(a, nnodes, max_s, st);
    else launch_k1_t<false, 16>(a, nnodes, max_s, st);
  }
}

void launch_linv(bool cplx, const LinvArgs& a, int nitems, cudaStream_t st) {
  if (nitems == 0) return;
  if (cplx) {
    set_smem(k_linv<true>, LinvG_C::SMEM_BYTES);
    k_linv<true><<<nitems, 128, LinvG_C::SMEM_BYTES, st>>>(a);
  } else {
    set_smem(k_linv<false>, LinvG_R::SMEM_BYTES);
    k_linv<false><<<nitems, 128, LinvG_R::SMEM_BYTES, st>>>(a);
  }
}

void launch_rowperm(bool cplx, const RowpermArgs& a, int nlist, int max_s, cudaStream_t st) {
  if (nlist == 0) return;
  size_t sm = (size_t)4 * 2 * max_s * sizeof(double);  // 4 warps
  dim3 grid(8, std::min(nlist, 65535));
  // the attribute is set once to the largest size any handle can need (a replayed CUDA graph is
  // checked against the attribute's value at replay time); each launch uses its own size
  const size_t sm_max = (size_t)4 * 2 * K1_MAX_BLOCK * sizeof(double);
  if (cplx) {
    static bool once = (set_smem(k_rowperm<true>, sm_max), true);
    (void)once;
    k_rowperm<true><<<grid, 128, sm, st>>>(a, nlist);
  } else {
    static bool once = (set_smem(k_rowperm<false>, sm_max), true);
    (void)once;
    k_rowperm<false><<<grid, 128, sm, st>>>(a, nlist);
  }
}

template <int CFG>
static int bm_of(bool cplx) { return cplx ? K3Cfg<true, CFG>::BM : K3Cfg<false, CFG>::BM; }
template <int CFG>
static int bn_of(bool cplx) { return cplx ? K3Cfg<true, CFG>::BN : K3Cfg<false, CFG>::BN; }

int k3_bm(bool cplx, int cfg) {
  switch (cfg) {
#ifdef DD_AUX_AB
    case 0: return bm_of<0>(cplx);
#endif
#ifdef DD_AUX_AB
    case 2: return bm_of<2>(cplx);
#endif
#ifdef DD_AUX_AB
    case 3: return bm_of<3>(cplx);
#endif
#ifdef DD_AUX_AB
    case 4: return bm_of<4>(cplx);
#endif
#ifdef DD_AUX_AB
    case 5: return bm_of<5>(cplx);
#endif
#ifdef DD_AUX_AB
    case 6: return bm_of<6>(cplx);
#endif
#ifdef DD_AUX_AB
    case 7: return bm_of<7>(cplx);
#endif
#ifdef DD_AUX_AB
    case 8: return bm_of<8>(cplx);
#endif
    case 9: return bm_of<9>(cplx);
    case 10: return bm_of<10>(cplx);
#ifdef DD_AUX_AB
    case 11: return bm_of<11>(cplx);
#endif
#ifdef DD_AUX_AB
    case 12: return bm_of<12>(cplx);
#endif
    case 13: return bm_of<13>(cplx);
#ifdef DD_AUX_AB
    case 14: return bm_of<14>(cplx);
#endif
#ifdef DD_AUX_AB
    case 15: return bm_of<15>(cplx);
    case 16: return bm_of<16>(cplx);
    case 17: return bm_of<17>(cplx);
    case 18: return bm_of<18>(cplx);
    case 19: return bm_of<19>(cplx);
#endif
    default: return bm_of<13>(cplx);
  }
}
int k3_bn(bool cplx, int cfg) {
  switch (cfg) {
#ifdef DD_AUX_AB
    case 0: return bn_of<0>(cplx);
#endif
#ifdef DD_AUX_AB
    case 2: return bn_of<2>(cplx);
#endif
#ifdef DD_AUX_AB
    case 3: return bn_of<3>(cplx);
#endif
#ifdef DD_AUX_AB
    case 4: return bn_of<4>(cplx);
#endif
#ifdef DD_AUX_AB
    case 5: return bn_of<5>(cplx);
#endif
#ifdef DD_AUX_AB
    case 6: return bn_of<6>(cplx);
#endif
#ifdef DD_AUX_AB
    case 7: return bn_of<7>(cplx);
#endif
#ifdef DD_AUX_AB
    case 8: return bn_of<8>(cplx);
#endif
    case 9: return bn_of<9>(cplx);
    case 10: return bn_of<10>(cplx);
#ifdef DD_AUX_AB
    case 11: return bn_of<11>(cplx);
#endif
#ifdef DD_AUX_AB
    case 12: return bn_of<12>(cplx);
#endif
    case 13: return bn_of<13>(cplx);
#ifdef DD_AUX_AB
    case 14: return bn_of<14>(cplx);
#endif
#ifdef DD_AUX_AB
    case 15: return bn_of<15>(cplx);
    case 16: return bn_of<16>(cplx);
    case 17: return bn_of<17>(cplx);
    case 18: return bn_of<18>(cplx);
    case 19: return bn_of<19>(cplx);
#endif
    default: return bn_of<13>(cplx);
  }
}

template <bool C, int CFG>
static void launch_k3_t(const K3Args& a, int ntiles, cudaStream_t st, bool persistent) {
  using Cf = K3Cfg<C, CFG>;
#ifdef DD_AUX_AB
  if (persistent) {
    static int slots = 0;
    if (!slots) {
      set_smem(k3_update_persist<C, CFG>, Cf::G::SMEM_BYTES);
      int per = 0, dev = 0, nsm = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k3_update_persist<C, CFG>, Cf::NT, Cf::G::SMEM_BYTES);
      slots = std::max(1, per) * nsm;
    }
    K3Args b = a;
    b.ntiles = ntiles;
    cudaMemsetAsync(b.counter, 0, sizeof(unsigned long long), st);
    k3_update_persist<C, CFG><<<std::min(ntiles, slots), Cf::NT, Cf::G::SMEM_BYTES, st>>>(b);
    return;
  }
#else
  (void)persistent;  // measured slower: A/B builds only
#endif
  set_smem(k3_update<C, CFG>, Cf::G::SMEM_BYTES);
  k3_update<C, CFG><<<ntiles, Cf::NT, Cf::G::SMEM_BYTES, st>>>(a);
}

template <int CFG>
static void launch_k3_c(bool cplx, const K3Args& a, int ntiles, cudaStream_t st, bool persistent = false) {
  if (cplx) launch_k3_t<true, CFG>(a, ntiles, st, persistent);
  else launch_k3_t<false, CFG>(a, ntiles, st, persistent);
}

void launch_k3(bool cplx, int cfg, const K3Args& a, int ntiles, cudaStream_t st, bool persistent) {
  if (ntiles == 0) return;
  persistent = persistent && a.counter != nullptr;
  if (cfg == 9 || cfg == 10 || cfg == 13) {  // the default-build configurations (persistent-capable)
    if (cfg == 9) launch_k3_c<9>(cplx, a, ntiles, st, persistent);
    else if (cfg == 10) launch_k3_c<10>(cplx, a, ntiles, st, persistent);
    else launch_k3_c<13>(cplx, a, ntiles, st, persistent);
    return;
  }
  switch (cfg) {
#ifdef DD_AUX_AB
    case 0: launch_k3_c<0>(cplx, a, ntiles, st); break;
#endif
#ifdef DD_AUX_AB
    case 2: launch_k3_c<2>(cplx, a, ntiles, st); break;
#endif
#ifdef DD_AUX_AB
    case 3: launch_k3_c<3>(cplx, a, ntiles, st); break;
#endif
#ifdef DD_AUX_AB
    case 4: launch_k3_c<4>(cplx, a, ntiles, st); break;
#endif
#ifdef DD_AUX_AB
    case 5: launch_k3_c<5>(cplx, a, ntiles, st); break;
#endif
#ifdef DD_AUX_AB
    case 6: launch_k3_c<6>(cplx, a, ntiles, st); break;
#endif
#ifdef DD_AUX_AB
    case 7: launch_k3_c<7>(cplx, a, ntiles, st); break;
#endif
#ifdef DD_AUX_AB
    case 8: launch_k3_c<8>(cplx, a, ntiles, st); break;
#endif
    case 9: launch_k3_c<9>(cplx, a, ntiles, st); break;
    case 10: launch_k3_c<10>(cplx, a, ntiles, st); break;
#ifdef DD_AUX_AB
    case 11: launch_k3_c<11>(cplx, a, ntiles, st); break;
#endif
#ifdef DD_AUX_AB
    case 12: launch_k3_c<12>(cplx, a, ntiles, st); break;
#endif
    case 13: launch_k3_c<13>(cplx, a, ntiles, st); break;
#ifdef DD_AUX_AB
    case 14: launch_k3_c<14>(cplx, a, ntiles, st); break;
#endif
#ifdef DD_AUX_AB
    case 15: launch_k3_c<15>(cplx, a, ntiles, st); break;
    case 16: launch_k3_c<16>(cplx, a, ntiles, st); break;
    case 17: launch_k3_c<17>(cplx, a, ntiles, st); break;
    case 18: launch_k3_c<18>(cplx, a, ntiles, st); break;
    case 19: launch_k3_c<19>(cplx, a, ntiles, st); break;
#endif
    default: launch_k3_c<13>(cplx, a, ntiles, st); break;
  }
}

template <bool C, int CFG>
static void launch_k2_t(const K2Args& a, int nitems, int max_s, cudaStream_t st) {
  using Cf = K3Cfg<C, CFG>;
  const size_t sm = Cf::G::SMEM_BYTES + (size_t)((max_s + 3) & ~3) * sizeof(int);  // + column map
  // the attribute is set to the largest size any level may use (a replayed CUDA graph checks every
  // node against the attribute's final value); occupancy follows each launch's own size
  set_smem(k2_gemm<C, CFG>, Cf::G::SMEM_BYTES + (size_t)K1_MAX_BLOCK * sizeof(int));
  k2_gemm<C, CFG><<<nitems, Cf::NT, sm, st>>>(a);
}

void launch_k2(bool cplx, int cfg, const K2Args& a, int nitems, int nstrips, int max_s, cudaStream_t st) {
  if (nitems > 0) {
    switch (cfg) {  // same tile shapes as the Schur update
      case 9: cplx ? launch_k2_t<true, 9>(a, nitems, max_s, st) : launch_k2_t<false, 9>(a, nitems, max_s, st); break;
      case 10: cplx ? launch_k2_t<true, 10>(a, nitems, max_s, st) : launch_k2_t<false, 10>(a, nitems, max_s, st); break;
#ifdef DD_AUX_AB
      case 11: cplx ? launch_k2_t<true, 11>(a, nitems, max_s, st) : launch_k2_t<false, 11>(a, nitems, max_s, st); break;
#endif
#ifdef DD_AUX_AB
      case 12: cplx ? launch_k2_t<true, 12>(a, nitems, max_s, st) : launch_k2_t<false, 12>(a, nitems, max_s, st); break;
#endif
      case 13: cplx ? launch_k2_t<true, 13>(a, nitems, max_s, st) : launch_k2_t<false, 13>(a, nitems, max_s, st); break;
#ifdef DD_AUX_AB
      case 6: cplx ? launch_k2_t<true, 6>(a, nitems, max_s, st) : launch_k2_t<false, 6>(a, nitems, max_s, st); break;
#endif
#ifdef DD_AUX_AB
      case 5: cplx ? launch_k2_t<true, 5>(a, nitems, max_s, st) : launch_k2_t<false, 5>(a, nitems, max_s, st); break;
#endif
#ifdef DD_AUX_AB
      case 4: cplx ? launch_k2_t<true, 4>(a, nitems, max_s, st) : launch_k2_t<false, 4>(a, nitems, max_s, st); break;
#endif
#ifdef DD_AUX_AB
      case 1: cplx ? launch_k2_t<true, 1>(a, nitems, max_s, st) : launch_k2_t<false, 1>(a, nitems, max_s, st); break;
#endif
#ifdef DD_AUX_AB
      case 16: cplx ? launch_k2_t<true, 16>(a, nitems, max_s, st) : launch_k2_t<false, 16>(a, nitems, max_s, st); break;
      case 17: cplx ? launch_k2_t<true, 17>(a, nitems, max_s, st) : launch_k2_t<false, 17>(a, nitems, max_s, st); break;
      case 18: cplx ? launch_k2_t<true, 18>(a, nitems, max_s, st) : launch_k2_t<false, 18>(a, nitems, max_s, st); break;
      case 19: cplx ? launch_k2_t<true, 19>(a, nitems, max_s, st) : launch_k2_t<false, 19>(a, nitems, max_s, st); break;
#endif
      default: cplx ? launch_k2_t<true, 13>(a, nitems, max_s, st) : launch_k2_t<false, 13>(a, nitems, max_s, st); break;
    }
  }
  if (nstrips > 0) {
    dim3 grid(nstrips, 8);
    if (cplx) k2_dinv<true><<<grid, NT2, 0, st>>>(a);
    else k2_dinv<false><<<grid, NT2, 0, st>>>(a);
  }
}

void launch_k4(const int64_t* node_stats, int nnodes, const int* gperm, int64_t* out, cudaStream_t st) {
  k4_stats<<<1, 256, 0, st>>>(node_stats, nnodes, gperm, out);
}

}  // namespace ddk
