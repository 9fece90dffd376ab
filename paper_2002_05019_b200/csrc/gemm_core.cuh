// FP64 tensor-core (DMMA) tile engine for sm_100a.
//
// On sm_100a the FP64 tensor path is reachable only through warp-level
// mma.sync ... .f64 (tcgen05.mma has no f64 kind; wgmma is sm_90a-only), which
// lowers to SASS DMMA.8x8x4.  This engine computes one BM x BN
// output tile of   C (+)= sum_seg A_seg * B_seg   where the K dimension is the
// concatenation of a list of segments ("gathered K", SURVEY.md §8(a) a4:
// owner-computes target tiles summing all contributors of a level in a fixed
// order -- deterministic, no atomics).  Operands are staged into shared memory by
// cp.async (LDGSTS, 16-byte chunks; zero-filled along K outside the logical shape,
// rows / columns outside it are never stored) in a STAGES-deep pipeline and fed to
// mma.sync.m16n8k4.f64 from registers.  The copies go through per-thread running
// pointers (the "fast loader" below); the tile can be subtracted from C by L2
// reductions (store_tile MODE 2).
//
// Operand layouts (all column-major storage in HBM):
//   A "MK": A(m,k) = a[m + col(k)*lda]   (m contiguous; optional column gather map)
//   A "KM": A(m,k) = a[k + m*lda]        (k contiguous; i.e. a transposed view)
//   B "NK": B(k,n) = b[n + k*ldb]        (n contiguous; B = L^T of a col-major L)
//   B "KN": B(k,n) = b[k + n*ldb]        (k contiguous; a col-major K x N block)
// Complex (complex symmetric, no conjugation) is planar: imaginary planes at a
// fixed element offset; products use the 4M real formulation
//   Cr += Ar Br - Ai Bi,  Ci += Ar Bi + Ai Br.
// Alignment contract: every segment base, lda/ldb and row offsets are even
// (16-byte aligned chunks); the library's layout guarantees it.
#pragma once
#include <cstdint>

namespace ddk {

struct Seg {
  const double* a;   // A(0,0) (re plane)
  const double* b;   // B(0,0) (re plane)
  const int* acol;   // MK only: column gather map (k -> column), or nullptr
  int64_t lda, ldb;
  int K;
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
// fixed 16-byte copy to a shared-window address, skipped when !pred (the destination keeps its
// old contents: only for rows / columns whose results are never stored)
__device__ __forceinline__ void cp_async16_if(unsigned saddr, const void* gmem, int pred) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %2, 0;\n"
      " @p cp.async.cg.shared.global [%0], [%1], 16;\n}\n" ::"r"(saddr),
      "l"(gmem), "r"(pred)
      : "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// mbarrier helpers (MBAR pipeline): per-stage "full" barriers completed by the threads' cp.async
// groups (cp.async.mbarrier.arrive.noinc), "empty" barriers completed by one arrival per warp
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_cpasync_arrive(uint64_t* b) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared.b64 [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared.b64 _, [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred P;\n"
      "DD_MBAR_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared.b64 P, [%0], %1;\n"
      " @!P bra DD_MBAR_WAIT_%=;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void dmma16x8x4(double (&c)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

__device__ __forceinline__ double dneg(double x) {  // sign flip on the integer pipe (keeps DMMA pipe free)
  return __longlong_as_double(__double_as_longlong(x) ^ (long long)0x8000000000000000ull);
}

// C3M (complex only): 3M / Gauss formulation -- T1 = Ar Br, T2 = Ai Bi, T3 = (Ar+Ai)(Br+Bi),
// Cr = T1 - T2, Ci = T3 - T1 - T2: three real DMMA products instead of four.
// FINE: per-16x8-sub-tile DMMA masking (one predicate per mma) vs coarse per-warp masking (a warp
// whose whole warp tile is outside the valid region skips the stage; otherwise branch-free).
// VEC (MK x NK only): vectorised fragment loads.  The mma's row slots g / g+8 of a 16-row sub-tile
// map to tile rows 2g / 2g+1 and its column slot g of sub-tile b to tile column
// 16*(b/2) + 2g + (b%2), so a thread's two A values and the B values of a sub-tile pair are
// adjacent in shared memory: one 16-byte LDS each instead of two 8-byte ones (bank-conflict free
// with the ld = 4 (mod 16) padding).  The accumulator mapping (for_each, masks) follows.
template <int BM, int BN, int BK, int WARPS_M, int WARPS_N, int STAGES, bool CPLX, bool A_KM, bool B_KN,
          bool C3M = false, bool FINE = true, bool VEC = false, bool RECT = false, bool MBAR = false,
          bool FAST = true>
struct Gemm {
  static constexpr int NTHR = WARPS_M * WARPS_N * 32;
  static constexpr int WTM = BM / WARPS_M, WTN = BN / WARPS_N;
  static constexpr int MI = WTM / 16, NI = WTN / 8;
  static constexpr int NPL = CPLX ? 2 : 1;
  static constexpr int A_LD = A_KM ? (BK + 4) : (BM + 4);
  static constexpr int A_TILE = A_KM ? BM * (BK + 4) : BK * (BM + 4);
  static constexpr int B_LD = B_KN ? (BK + 4) : (BN + 4);
  static constexpr int B_TILE = B_KN ? BN * (BK + 4) : BK * (BN + 4);
  static constexpr int STAGE = NPL * (A_TILE + B_TILE);
  static constexpr size_t SMEM_BYTES = (size_t)STAGES * STAGE * sizeof(double);
  static_assert(WTM % 16 == 0 && WTN % 8 == 0 && BK % 4 == 0, "tile shape");
  static_assert((A_LD % 16) == 4 && (B_LD % 16) == 4, "bank-conflict-free padding");
  static_assert(!VEC || (!A_KM && !B_KN && NI % 2 == 0), "VEC needs MK x NK and an even NI");

  static_assert(!C3M || CPLX, "3M needs complex operands");
  struct Acc {
    double r[MI][NI][4];                       // real part (4M) / T1 (3M)
    double i[CPLX ? MI : 1][CPLX ? NI : 1][4];  // imaginary part (4M) / T2 (3M)
    double t[C3M ? MI : 1][C3M ? NI : 1][4];    // T3 (3M)
  };

  __device__ static void zero(Acc& acc) {
#pragma unroll
    for (int a = 0; a < MI; ++a)
#pragma unroll
      for (int b = 0; b < NI; ++b)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          acc.r[a][b][v] = 0.0;
          if constexpr (CPLX) acc.i[a][b][v] = 0.0;
          if constexpr (C3M) acc.t[a][b][v] = 0.0;
        }
  }

  // Warp aliasing for ragged tiles (RECT, 2 x 2 warps, tile_mask(.., alias = true)): when only warp
  // row 0 (and / or warp column 0) of a tile holds valid rows (columns), the warps of row 1
  // (column 1) would idle.  They are mapped onto the same warp tile as their row-0 (column-0)
  // sibling instead and the k-steps of every stage are dealt round-robin over the 2 (4) aliases;
  // store_tile adds the partial sums in a fixed order.
  __device__ static int alias_nsplit(unsigned amap) { return ((amap & 1u) ? 2 : 1) * ((amap & 2u) ? 2 : 1); }
  __device__ static int alias_part(unsigned amap) {
    const int warp = threadIdx.x >> 5;
    return ((amap & 1u) ? warp % WARPS_M : 0) + ((amap & 2u) ? (warp / WARPS_M) * ((amap & 1u) ? 2 : 1) : 0);
  }

  // Visit every accumulator element: f(row_in_tile, col_in_tile, re, im)
  // amap (RECT + alias, see tile_mask): bit 0 / 1 = this tile's warps all work on warp row / column 0
  template <class F>
  __device__ static void for_each(const Acc& acc, F f, unsigned amap = 0u) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wm = (amap & 1u) ? 0 : warp % WARPS_M, wn = (amap & 2u) ? 0 : warp / WARPS_M;
    const int g = lane >> 2, tg = lane & 3;
#pragma unroll
    for (int a = 0; a < MI; ++a)
#pragma unroll
      for (int b = 0; b < NI; ++b)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          int row = VEC ? wm * WTM + a * 16 + 2 * g + (v >> 1) : wm * WTM + a * 16 + g + ((v >> 1) << 3);
          int col = VEC ? wn * WTN + (b >> 1) * 16 + 4 * tg + 2 * (v & 1) + (b & 1) : wn * WTN + b * 8 + 2 * tg + (v & 1);
          if constexpr (C3M) {
            const double t1 = acc.r[a][b][v], t2 = acc.i[a][b][v], t3 = acc.t[a][b][v];
            f(row, col, t1 - t2, t3 - t1 - t2);
          } else {
            f(row, col, acc.r[a][b][v], CPLX ? acc.i[CPLX ? a : 0][CPLX ? b : 0][v] : 0.0);
          }
        }
  }

  // Mutable visit (not 3M): f(row_in_tile, col_in_tile, re&, im&)
  template <class F>
  __device__ static void for_each_mut(Acc& acc, F f) {
    static_assert(!C3M, "for_each_mut: 3M accumulators hold products, not the result");
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wm = warp % WARPS_M, wn = warp / WARPS_M;
    const int g = lane >> 2, tg = lane & 3;
    double dummy = 0.0;
#pragma unroll
    for (int a = 0; a < MI; ++a)
#pragma unroll
      for (int b = 0; b < NI; ++b)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          int row = VEC ? wm * WTM + a * 16 + 2 * g + (v >> 1) : wm * WTM + a * 16 + g + ((v >> 1) << 3);
          int col = VEC ? wn * WTN + (b >> 1) * 16 + 4 * tg + 2 * (v & 1) + (b & 1) : wn * WTN + b * 8 + 2 * tg + (v & 1);
          if constexpr (CPLX) f(row, col, acc.r[a][b][v], acc.i[a][b][v]);
          else f(row, col, acc.r[a][b][v], dummy);
        }
  }

  // Epilogue through shared memory: the accumulator tile is staged in the (idle) pipeline buffers
  // and written back column-coalesced with all loads of a batch in flight before the stores
  // (the fragment-order read-modify-write serialised ~32 dependent L2 round trips per tile).
  // MODE 0: C = acc, 1: C -= acc.  Call after run() (which ends with a barrier); ends with one.
  static constexpr int ELD = BM + 2;
  static_assert((size_t)BN * ELD * (CPLX ? 2 : 1) <= (size_t)STAGES * STAGE, "epilogue tile fits the pipeline smem");
  // MODE 2: C -= acc as fire-and-forget reductions at L2 (red.global.add.f64 of -acc): no C load,
  // no round trip before the CTA retires.  Every element of C gets exactly ONE reduction per
  // launch (owner-computes tiles; aliased warps are summed in shared memory first), so the result
  // does not depend on the order the reductions arrive in, and C + (-v) rounds as C - v does:
  // bitwise the read-modify-write result.  `active` = this warp holds a computed warp tile.
  template <int MODE>
  __device__ static void store_tile(const Acc& acc, double* smem, double* C, int64_t ldc, int64_t cim, int mlim,
                                    int nlim, unsigned amap = 0u, bool active = true) {
    double* Sr = smem;
    double* Si = smem + BN * ELD;
    if constexpr (MODE == 2) {
      if (amap == 0u) {  // straight from the accumulator fragments (8 rows x 1 column = two full sectors)
        if (active)
          for_each(acc, [&](int r, int c, double vr, double vi) {
            if (r < mlim && c < nlim) {
              atomicAdd(C + r + (int64_t)c * ldc, -vr);
              if constexpr (CPLX) atomicAdd(C + r + (int64_t)c * ldc + cim, -vi);
            }
          });
        return;
      }
    }
    if (amap == 0u) {
      for_each(acc, [&](int r, int c, double vr, double vi) {
        Sr[c * ELD + r] = vr;
        if constexpr (CPLX) Si[c * ELD + r] = vi;
      });
      __syncthreads();
    } else {
      // aliased warps hold partial sums (their share of the k-steps) of the same warp tile: added
      // in the fixed order part 0, 1, .. (deterministic)
      const int nsplit = alias_nsplit(amap), part = alias_part(amap);
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        if (p >= nsplit) break;  // CTA-uniform
        if (part == p)
          for_each(
              acc,
              [&](int r, int c, double vr, double vi) {
                if (p == 0) {
                  Sr[c * ELD + r] = vr;
                  if constexpr (CPLX) Si[c * ELD + r] = vi;
                } else {
                  Sr[c * ELD + r] += vr;
                  if constexpr (CPLX) Si[c * ELD + r] += vi;
                }
              },
              amap);
        __syncthreads();
      }
    }
    constexpr int PER = (BM * BN + NTHR - 1) / NTHR;
    // the accumulator registers are dead once staged, so a whole tile's loads fit in flight
#ifndef DDK_EPI_BATCH
#define DDK_EPI_BATCH 16
#endif
    constexpr int EB = CPLX ? 8 : DDK_EPI_BATCH;  // complex: two planes in flight per element
    constexpr int BATCH = PER < EB ? PER : EB;
#pragma unroll 1
    for (int q0 = 0; q0 < PER; q0 += BATCH) {
      double old_r[BATCH], old_i[CPLX ? BATCH : 1];
#pragma unroll
      for (int u = 0; u < BATCH; ++u) {
        const int e = threadIdx.x + (q0 + u) * NTHR;
        const int r = e % BM, c = e / BM;
        if (MODE == 1 && q0 + u < PER && c < BN && r < mlim && c < nlim) {
          old_r[u] = C[r + (int64_t)c * ldc];
          if constexpr (CPLX) old_i[u] = C[r + (int64_t)c * ldc + cim];
        }
      }
      if constexpr (MODE == 2) {  // aliased tile: the summed staging tile goes out as reductions
#pragma unroll
        for (int u = 0; u < BATCH; ++u) {
          const int e = threadIdx.x + (q0 + u) * NTHR;
          const int r = e % BM, c = e / BM;
          if (q0 + u < PER && c < BN && r < mlim && c < nlim) {
            atomicAdd(C + r + (int64_t)c * ldc, -Sr[c * ELD + r]);
            if constexpr (CPLX) atomicAdd(C + r + (int64_t)c * ldc + cim, -Si[c * ELD + r]);
          }
        }
        continue;
      }
#pragma unroll
      for (int u = 0; u < BATCH; ++u) {
        const int e = threadIdx.x + (q0 + u) * NTHR;
        const int r = e % BM, c = e / BM;
        if (q0 + u < PER && c < BN && r < mlim && c < nlim) {
          const double vr = Sr[c * ELD + r];
          C[r + (int64_t)c * ldc] = MODE == 1 ? old_r[u] - vr : vr;
          if constexpr (CPLX) {
            const double vi = Si[c * ELD + r];
            C[r + (int64_t)c * ldc + cim] = MODE == 1 ? old_i[u] - vi : vi;
          }
        }
      }
    }
    __syncthreads();
  }

  // Pull the C tile (valid region) into L2 ahead of the epilogue's read-modify-write: one
  // prefetch per 128-byte line, issued at tile start so the epilogue's loads hit L2.
  __device__ static void prefetch_tile_l2(const double* C, int64_t ldc, int64_t cim, int mlim, int nlim) {
#ifndef DDK_PREFETCH_C
#define DDK_PREFETCH_C 1
#endif
    if (!DDK_PREFETCH_C) return;
    const int rows = mlim < BM ? mlim : BM, cols = nlim < BN ? nlim : BN;
    if (rows <= 0 || cols <= 0) return;
    const int lpc = (rows + 15) / 16;  // 128-byte lines per column (lines may straddle: +1 below)
    const int nl = (lpc + 1) * cols * (CPLX ? 2 : 1);
    for (int q = threadIdx.x; q < nl; q += NTHR) {
      int x = q;
      const int pl = CPLX ? (x % 2) : 0;
      if (CPLX) x /= 2;
      const int c = x / (lpc + 1), l = x % (lpc + 1);
      const double* col = C + (int64_t)c * ldc + pl * cim;
      const uintptr_t a0 = (uintptr_t)col & ~uintptr_t(127);
      const uintptr_t a = a0 + (uintptr_t)l * 128;
      if (a <= (uintptr_t)(col + rows - 1)) asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
    }
  }

  __device__ static void load_stage(double* st, const Seg& sg, int kofs, int m0, int n0, int M, int N,
                                    int64_t aim, int64_t bim) {
    double* As = st;
    double* Bs = st + NPL * A_TILE;
    const int tid = threadIdx.x;
    // ---- A tile
    if constexpr (!A_KM) {
      constexpr int CH = BK * (BM / 2);
#pragma unroll
      for (int c = tid; c < CH; c += NTHR) {
        int kk = c / (BM / 2), mm = (c % (BM / 2)) * 2;
        int gm = m0 + mm, gk = kofs + kk;
        int bytes = (gk < sg.K && gm < M) ? (gm + 1 < M ? 16 : 8) : 0;
        const double* src = sg.a;
        if (bytes) src = sg.a + gm + (int64_t)(sg.acol ? sg.acol[gk] : gk) * sg.lda;
        cp_async16(As + kk * A_LD + mm, src, bytes);
        if constexpr (CPLX) cp_async16(As + A_TILE + kk * A_LD + mm, bytes ? src + aim : src, bytes);
      }
    } else {
      constexpr int CH = BM * (BK / 2);
#pragma unroll
      for (int c = tid; c < CH; c += NTHR) {
        int mm = c / (BK / 2), kk = (c % (BK / 2)) * 2;
        int gm = m0 + mm, gk = kofs + kk;
        int bytes = (gk < sg.K && gm < M) ? (gk + 1 < sg.K ? 16 : 8) : 0;
        const double* src = bytes ? sg.a + gk + (int64_t)gm * sg.lda : sg.a;
        cp_async16(As + mm * A_LD + kk, src, bytes);
        if constexpr (CPLX) cp_async16(As + A_TILE + mm * A_LD + kk, bytes ? src + aim : src, bytes);
      }
    }
    // ---- B tile
    if constexpr (!B_KN) {
      constexpr int CH = BK * (BN / 2);
#pragma unroll
      for (int c = tid; c < CH; c += NTHR) {
        int kk = c / (BN / 2), nn = (c % (BN / 2)) * 2;
        int gn = n0 + nn, gk = kofs + kk;
        int bytes = (gk < sg.K && gn < N) ? (gn + 1 < N ? 16 : 8) : 0;
        const double* src = bytes ? sg.b + gn + (int64_t)gk * sg.ldb : sg.b;
        cp_async16(Bs + kk * B_LD + nn, src, bytes);
        if constexpr (CPLX) cp_async16(Bs + B_TILE + kk * B_LD + nn, bytes ? src + bim : src, bytes);
      }
    } else {
      constexpr int CH = BN * (BK / 2);
#pragma unroll
      for (int c = tid; c < CH; c += NTHR) {
        int nn = c / (BK / 2), kk = (c % (BK / 2)) * 2;
        int gn = n0 + nn, gk = kofs + kk;
        int bytes = (gk < sg.K && gn < N) ? (gk + 1 < sg.K ? 16 : 8) : 0;
        const double* src = bytes ? sg.b + gk + (int64_t)gn * sg.ldb : sg.b;
        cp_async16(Bs + nn * B_LD + kk, src, bytes);
        if constexpr (CPLX) cp_async16(Bs + B_TILE + nn * B_LD + kk, bytes ? src + bim : src, bytes);
      }
    }
  }

  // ---- Fast loader (all four operand layouts; segments without a column gather).  load_stage
  // recomputes every chunk's source address and bounds from scratch (~26 SASS instructions and a
  // 6-deep dependent chain per cp.async: more issue slots per stage than the DMMAs themselves,
  // and with 16 warps per SM the kernels were bound by each warp's serial instruction latency).
  // A thread's chunks of a stage share one row (or k) offset and sit a fixed distance apart, so
  // inside a segment the thread keeps ONE running pointer per operand (pa, pb): a full stage
  // costs one 64-bit add per chunk.  The row predicate is constant per tile; only a segment's
  // last partial stage (pk + BK > K) and gathered segments go through load_stage.  The chunks of
  // the next stage are issued in parts between the k-steps of the current stage (part<KS>).
#ifndef DDK_FASTLD
#define DDK_FASTLD 1
#endif
  static constexpr int KSTEPS = BK / 4;
  static_assert(KSTEPS >= 1 && KSTEPS <= 8, "StageLd::part_rt / all() and the 4-bit k-step counts cover BK <= 32");
  // The copies of a stage go out in the first SPREAD k-steps (0 = all KSTEPS).  Measured with
  // 2-stage pipelines: real K3 (MK x NK) on cfg2, BK = 16: 29.3 / 29.8 / 29.9 TF/s with SPREAD
  // 1 / 2 / 4; BK = 24: 30.1 / 30.3 / 30.4 with 4 / 3 / 6; the solve (.. x KN) 4,405 / 4,367 /
  // 4,505 ms per 1000 RHS with 1 / 2 / 4 -- copies issued in the last k-steps have little time
  // to land before the next stage's wait.
#ifndef DDK_FASTLD_SPREAD
#define DDK_FASTLD_SPREAD 0
#endif
#ifndef DDK_FASTLD_SPREAD_KN
#define DDK_FASTLD_SPREAD_KN 2
#endif
#ifndef DDK_FASTLD_SPREAD_CPLX
#define DDK_FASTLD_SPREAD_CPLX 1  // complex (cfg3): 3M K3 at 3 CTAs/SM 40.0 / 39.5 / 37.4 effective TF/s with SPREAD 1 / 2 / 4; solve 3,439 / 3,523 / 3,799 ms per 1000 RHS
#endif
  static constexpr int SPREAD_REQ = CPLX ? DDK_FASTLD_SPREAD_CPLX : (B_KN ? DDK_FASTLD_SPREAD_KN : DDK_FASTLD_SPREAD);
  static constexpr int SPREAD = (SPREAD_REQ > 0 && SPREAD_REQ < KSTEPS) ? SPREAD_REQ : KSTEPS;
  // One operand's copy pattern.  RC (row-contiguous: A "MK" / B "NK"): a thread's chunks share one
  // row pair and sit KS k-columns apart, the running pointer walks through them and through the
  // stages.  KC (k-contiguous: A "KM" / B "KN"): a thread's chunks share one k pair and sit RS
  // rows apart (pointer p0 + j * RS * ld, one row-predicate bit per chunk); a stage advances p0
  // by BK elements.
  template <int R, int LD, bool KC>
  struct Pat {
    static constexpr int GRP = KC ? BK / 2 : R / 2;          // threads along the contiguous direction
    static constexpr int STEP = NTHR / (GRP > 0 ? GRP : 1);  // k columns (RC) or rows (KC) between chunks
    static constexpr int CH = (KC ? R : BK) / (STEP > 0 ? STEP : 1);
    static constexpr bool OK = GRP > 0 && NTHR % GRP == 0 && (KC ? R : BK) % STEP == 0 && CH >= 1 && CH <= 32;
    __device__ static int off(int tid) {  // offset of the thread's first chunk inside the operand's stage tile
      const int c = (tid % GRP) * 2, o = tid / GRP;
      return o * LD + c;  // RC: k column o, row pair c; KC: row o, k pair c
    }
    static constexpr int DSTEP = STEP * LD;  // smem distance between a thread's successive chunks
  };
  using PA = Pat<BM, A_LD, A_KM>;
  using PB = Pat<BN, B_LD, B_KN>;
  static constexpr bool FASTLD_ANY = DDK_FASTLD && FAST && PA::OK && PB::OK;
  static constexpr bool FASTLD = FASTLD_ANY && !MBAR;
  struct FastLd {
    const double* pa;  // this thread's first A chunk of the next full stage
    const double* pb;
    int64_t ia, ib;    // element stride between the thread's successive chunks
    unsigned ba, bb;   // row predicate(s): RC one flag, KC bit j = chunk j's row lies inside the operand
    unsigned sa, sb;   // shared-window address of this thread's first A / B chunk in stage slot 0
  };
  // Rows m >= M of A (columns n >= N of B) are NOT zero-filled here, and a last odd row is copied
  // as a full 16-byte chunk: row m of the product depends on row m of A only, rows >= M are never
  // stored, and the extra element lies inside the operand's (even) leading dimension.  Zero fill
  // matters along K only, which the generic loader handles (partial last stage of a segment).
  template <class P, bool KC>
  __device__ static unsigned fast_pred(int r0, int lim) {
    const int tid = threadIdx.x;
    if constexpr (!KC) {
      return (unsigned)(r0 + (tid % P::GRP) * 2 < lim);
    } else {
      unsigned m = 0;
#pragma unroll
      for (int j = 0; j < P::CH; ++j) m |= (unsigned)(r0 + tid / P::GRP + j * P::STEP < lim) << j;
      return m;
    }
  }
  __device__ static void fast_tile(FastLd& f, double* smem, int m0, int n0, int M, int N) {
    f.ba = fast_pred<PA, A_KM>(m0, M);
    f.bb = fast_pred<PB, B_KN>(n0, N);
    f.sa = smem_u32(smem + PA::off(threadIdx.x));
    f.sb = smem_u32(smem + NPL * A_TILE + PB::off(threadIdx.x));
  }
  // pointer to the thread's first chunk at k offset 0 of a segment + the chunk stride
  template <class P, bool KC>
  __device__ static void fast_ptr(const double*& p, int64_t& inc, unsigned pred, const double* base, int64_t ld,
                                  int r0) {
    const int tid = threadIdx.x;
    const int c = (tid % P::GRP) * 2, o = tid / P::GRP;
    if constexpr (!KC) {
      p = pred ? base + (r0 + c) + (int64_t)o * ld : base;
      inc = pred ? (int64_t)P::STEP * ld : 0;
    } else {
      p = base + c + (int64_t)(r0 + o) * ld;  // chunks whose row is outside are predicated off
      inc = (int64_t)P::STEP * ld;
    }
  }
  __device__ static void fast_seg(FastLd& f, const Seg& sg, int m0, int n0) {
    fast_ptr<PA, A_KM>(f.pa, f.ia, f.ba, sg.a, sg.lda, m0);
    fast_ptr<PB, B_KN>(f.pb, f.ib, f.bb, sg.b, sg.ldb, n0);
  }
  template <class P, bool KC, int KS, int TILE>
  __device__ static void fast_op(const double*& p, int64_t inc, unsigned pred, unsigned sdst, int64_t im) {
#pragma unroll
    for (int j = 0; j < P::CH; ++j)
      if (j * SPREAD / P::CH == KS) {
        const unsigned d = sdst + (unsigned)(j * P::DSTEP * sizeof(double));
        if constexpr (!KC) {
          cp_async16_if(d, p, pred);
          if constexpr (CPLX) cp_async16_if(d + (unsigned)(TILE * sizeof(double)), p + im, pred);
          p += inc;
        } else {
          const double* q = p + j * inc;
          cp_async16_if(d, q, (pred >> j) & 1u);
          if constexpr (CPLX) cp_async16_if(d + (unsigned)(TILE * sizeof(double)), q + im, (pred >> j) & 1u);
        }
      }
    if constexpr (KC && KS == SPREAD - 1) p += BK;
  }
  // part KS (of KSTEPS) of a full stage's copies into stage slot `slot`
  template <int KS>
  __device__ static void fast_part(FastLd& f, int slot, int64_t aim, int64_t bim) {
    const unsigned so = (unsigned)slot * (unsigned)(STAGE * sizeof(double));
    fast_op<PA, A_KM, KS, A_TILE>(f.pa, f.ia, f.ba, f.sa + so, aim);
    fast_op<PB, B_KN, KS, B_TILE>(f.pb, f.ib, f.bb, f.sb + so, bim);
  }
  // What the copy engine of run() does during one compute stage: mode 0 nothing, 1 a full stage
  // through the running pointers (in parts, between the k-steps), 2 the generic loader (all of
  // it ahead of the compute stage: one inlined copy, not one per compute body).
  struct StageLd {
    int mode, slot;
    double* st;
    FastLd* f;
    const Seg* sg;
    int kofs, m0, n0, M, N;
    int64_t aim, bim;
    template <int KS>
    __device__ __forceinline__ void part() const {
      if (mode == 1) fast_part<KS>(*f, slot, aim, bim);
    }
    __device__ __forceinline__ void generic() const {  // mode 2: ahead of the compute stage
      if (mode == 2) load_stage(st, *sg, kofs, m0, n0, M, N, aim, bim);
    }
    __device__ __forceinline__ void part_rt(int ks) const {  // ks is a constant after unrolling
      switch (ks) {
        case 0: part<0>(); break;
        case 1: if constexpr (KSTEPS > 1) part<1 % KSTEPS>(); break;
        case 2: if constexpr (KSTEPS > 2) part<2 % KSTEPS>(); break;
        case 3: if constexpr (KSTEPS > 3) part<3 % KSTEPS>(); break;
        case 4: if constexpr (KSTEPS > 4) part<4 % KSTEPS>(); break;
        case 5: if constexpr (KSTEPS > 5) part<5 % KSTEPS>(); break;
        case 6: if constexpr (KSTEPS > 6) part<6 % KSTEPS>(); break;
        case 7: if constexpr (KSTEPS > 7) part<7 % KSTEPS>(); break;
      }
    }
    __device__ __forceinline__ void all() const {
      part<0>();
      if constexpr (KSTEPS > 1) part<1 % KSTEPS>();
      if constexpr (KSTEPS > 2) part<2 % KSTEPS>();
      if constexpr (KSTEPS > 3) part<3 % KSTEPS>();
      if constexpr (KSTEPS > 4) part<4 % KSTEPS>();
      if constexpr (KSTEPS > 5) part<5 % KSTEPS>();
      if constexpr (KSTEPS > 6) part<6 % KSTEPS>();
      if constexpr (KSTEPS > 7) part<7 % KSTEPS>();
    }
  };

  // Bit (a*NI + b) set = this warp's 16x8 sub-tile (a, b) intersects the valid region: rows
  // < mlim, cols < nlim and, when diag_off != NO_DIAG, not strictly above the diagonal
  // col - row == diag_off (diagonal target blocks store only their lower triangle).  Masked
  // sub-tiles issue no DMMA, which the co-resident CTA's warps pick up.
  static constexpr int NO_DIAG = -(1 << 30);
  // RECT: the valid part of a warp tile is a rectangle of whole 16-row groups x whole column
  // groups (8 columns; 16 with VEC) -- code = 1 | na << 4 | ncg << 8, 0 = skip the warp tile
  // (entirely outside, or strictly above a diagonal target's diagonal).
  static constexpr int CG = VEC ? 16 : 8;    // columns per column group
  static constexpr int NCG = WTN / CG;       // column groups per warp tile
  static constexpr bool ALIAS_OK = RECT && WARPS_M == 2 && WARPS_N == 2;
  // CTA-uniform alias map of a tile with mlim valid rows and nlim valid columns
  __device__ static unsigned alias_map(int mlim, int nlim) {
    return ALIAS_OK ? (unsigned)(mlim <= WTM) | ((unsigned)(nlim <= WTN) << 1) : 0u;
  }
  __device__ static unsigned tile_mask(int mlim, int nlim, int diag_off, bool alias = false) {
    const int warp = threadIdx.x >> 5;
    int wm = warp % WARPS_M, wn = warp / WARPS_M;
    if constexpr (RECT) {
      unsigned amap = 0u;
      if constexpr (ALIAS_OK) {
        if (alias && mlim <= WTM) amap |= 1u, wm = 0;
        if (alias && nlim <= WTN) amap |= 2u, wn = 0;
      }
      const int r0 = wm * WTM, c0 = wn * WTN;
      if (r0 >= mlim || c0 >= nlim) return 0u;
      if (diag_off != NO_DIAG && r0 + WTM - 1 < c0 + diag_off) return 0u;
      const int na = min(MI, (mlim - r0 + 15) / 16), ncg = min(NCG, (nlim - c0 + CG - 1) / CG);
      return 1u | ((unsigned)na << 4) | ((unsigned)ncg << 8) | (amap << 12);
    }
    unsigned m = 0;
#pragma unroll
    for (int a = 0; a < MI; ++a)
#pragma unroll
      for (int b = 0; b < NI; ++b) {
        const int r0 = wm * WTM + a * 16, c0 = VEC ? wn * WTN + (b >> 1) * 16 + (b & 1) : wn * WTN + b * 8;
        bool on = r0 < mlim && c0 < nlim;
        if (diag_off != NO_DIAG && r0 + 15 < c0 + diag_off) on = false;
        if (on) m |= 1u << (a * NI + b);
      }
    return m;
  }

  // Sub-tiles a < NA, b < NB of the warp tile; PRED: per-mma predicate from mask (FINE mode).
  // nks: k-steps of 4 holding data in this stage (a segment's last stage may be partly
  // zero-filled: its empty k-steps issue no DMMA)
  // LD: the copies of the next stage (ld) are issued in parts between the k-steps
  template <int NA, int NB, bool PRED, bool LD = false>
  __device__ static void compute_body(const double* st, Acc& acc, unsigned mask, int nks = BK / 4,
                                      const StageLd* ld = nullptr, unsigned amap = 0u) {
    if constexpr (!PRED) mask = ~0u;  // constant: the per-mma predicates fold away
    const double* As = st;
    const double* Bs = st + NPL * A_TILE;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wm = (amap & 1u) ? 0 : warp % WARPS_M, wn = (amap & 2u) ? 0 : warp / WARPS_M;
    // live k-steps of this warp: those holding data (k tail) and, for aliased warps, ks = part (mod nsplit)
    unsigned lm = (1u << (nks > 0 ? nks : 1)) - 1u;
    if (amap) {
      const int ns = alias_nsplit(amap), pt = alias_part(amap);
      unsigned pm = 0u;
#pragma unroll
      for (int ks = 0; ks < BK / 4; ++ks)
        if ((ks & (ns - 1)) == pt) pm |= 1u << ks;
      lm &= pm;
    }
    const int g = lane >> 2, tg = lane & 3;
    struct Frag {
      double ar[MI][2], br[NI];
      double ai[CPLX ? MI : 1][2], bi[CPLX ? NI : 1];
    };
    auto load = [&](int ks, Frag& f) {
      const int k = ks * 4 + tg;
      auto& ar = f.ar;
      auto& br = f.br;
      auto& ai = f.ai;
      auto& bi = f.bi;
      (void)ai;
      (void)bi;
      if constexpr (VEC) {
#pragma unroll
        for (int a = 0; a < NA; ++a) {
          const int o = k * A_LD + wm * WTM + a * 16 + 2 * g;
          const double2 v = *reinterpret_cast<const double2*>(As + o);
          ar[a][0] = v.x;
          ar[a][1] = v.y;
          if constexpr (CPLX) {
            const double2 w = *reinterpret_cast<const double2*>(As + A_TILE + o);
            ai[a][0] = w.x;
            ai[a][1] = w.y;
          }
        }
#pragma unroll
        for (int p = 0; p < NB / 2; ++p) {
          const int o = k * B_LD + wn * WTN + p * 16 + 2 * g;
          const double2 v = *reinterpret_cast<const double2*>(Bs + o);
          br[2 * p] = v.x;
          br[2 * p + 1] = v.y;
          if constexpr (CPLX) {
            const double2 w = *reinterpret_cast<const double2*>(Bs + B_TILE + o);
            bi[2 * p] = w.x;
            bi[2 * p + 1] = w.y;
          }
        }
      } else {
#pragma unroll
        for (int a = 0; a < NA; ++a) {
          int m = wm * WTM + a * 16 + g;
          int o0 = A_KM ? (m * A_LD + k) : (k * A_LD + m);
          int o1 = A_KM ? ((m + 8) * A_LD + k) : (k * A_LD + m + 8);
          ar[a][0] = As[o0];
          ar[a][1] = As[o1];
          if constexpr (CPLX) {
            ai[a][0] = As[A_TILE + o0];
            ai[a][1] = As[A_TILE + o1];
          }
        }
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          int n = wn * WTN + b * 8 + g;
          int o = B_KN ? (n * B_LD + k) : (k * B_LD + n);
          br[b] = Bs[o];
          if constexpr (CPLX) bi[b] = Bs[B_TILE + o];
        }
      }
    };
    auto issue = [&](Frag& f) {
      auto& ar = f.ar;
      auto& br = f.br;
      auto& ai = f.ai;
      auto& bi = f.bi;
      (void)ai;
      (void)bi;
      // Issue order: every product class over all (a, b) before the next class, so two
      // DMMAs into the same accumulator are MI*NI instructions apart (no dependency stall).
      if constexpr (C3M) {
        double sa[MI][2], sb[NI];
#pragma unroll
        for (int a = 0; a < NA; ++a) {
          sa[a][0] = ar[a][0] + ai[a][0];
          sa[a][1] = ar[a][1] + ai[a][1];
        }
#pragma unroll
        for (int b = 0; b < NB; ++b) sb[b] = br[b] + bi[b];
#pragma unroll
        for (int a = 0; a < NA; ++a)
#pragma unroll
          for (int b = 0; b < NB; ++b)
            if ((mask >> (a * NI + b)) & 1u) dmma16x8x4(acc.r[a][b], ar[a][0], ar[a][1], br[b]);
#pragma unroll
        for (int a = 0; a < NA; ++a)
#pragma unroll
          for (int b = 0; b < NB; ++b)
            if ((mask >> (a * NI + b)) & 1u) dmma16x8x4(acc.i[a][b], ai[a][0], ai[a][1], bi[b]);
#pragma unroll
        for (int a = 0; a < NA; ++a)
#pragma unroll
          for (int b = 0; b < NB; ++b)
            if ((mask >> (a * NI + b)) & 1u) dmma16x8x4(acc.t[a][b], sa[a][0], sa[a][1], sb[b]);
      } else {
#pragma unroll
      for (int a = 0; a < NA; ++a)
#pragma unroll
        for (int b = 0; b < NB; ++b)
          if ((mask >> (a * NI + b)) & 1u) dmma16x8x4(acc.r[a][b], ar[a][0], ar[a][1], br[b]);
      if constexpr (CPLX) {
#pragma unroll
        for (int a = 0; a < NA; ++a)
#pragma unroll
          for (int b = 0; b < NB; ++b)
            if ((mask >> (a * NI + b)) & 1u) dmma16x8x4(acc.i[a][b], ar[a][0], ar[a][1], bi[b]);
        double nai[MI][2];
#pragma unroll
        for (int a = 0; a < NA; ++a) {
          nai[a][0] = dneg(ai[a][0]);
          nai[a][1] = dneg(ai[a][1]);
        }
#pragma unroll
        for (int a = 0; a < NA; ++a)
#pragma unroll
          for (int b = 0; b < NB; ++b)
            if ((mask >> (a * NI + b)) & 1u) dmma16x8x4(acc.r[a][b], nai[a][0], nai[a][1], bi[b]);
#pragma unroll
        for (int a = 0; a < NA; ++a)
#pragma unroll
          for (int b = 0; b < NB; ++b)
            if ((mask >> (a * NI + b)) & 1u) dmma16x8x4(acc.i[a][b], ai[a][0], ai[a][1], br[b]);
      }
      }  // 4M / real
    };
#ifndef DDK_KSTEP_BREAK
#define DDK_KSTEP_BREAK 1
#endif
#ifndef DDK_FRAG_DB
#define DDK_FRAG_DB 0
#endif
    if constexpr (LD) {
#pragma unroll
      for (int ks = 0; ks < BK / 4; ++ks) {
        // warp-uniform; an empty k-step (k tail, or another alias's share) loads and issues nothing
        const bool live = (lm >> ks) & 1u;
        Frag f;
        if (live) load(ks, f);
        ld->part_rt(ks);
        if (live) issue(f);
      }
    } else if constexpr (DDK_FRAG_DB != 0) {
      // register double-buffered fragments: the loads of k-step ks+1 are issued before the DMMAs
      // of k-step ks (the k-tail skip is kept: an empty k-step loads and issues nothing)
      Frag fr[2];
      load(0, fr[0]);
#pragma unroll
      for (int ks = 0; ks < BK / 4; ++ks) {
        if (ks > 0 && ks >= nks) break;  // warp-uniform
        if (ks + 1 < BK / 4 && ks + 1 < nks) load(ks + 1, fr[(ks + 1) & 1]);
        issue(fr[ks & 1]);
      }
    } else {
#pragma unroll
      for (int ks = 0; ks < BK / 4; ++ks) {
        if (DDK_KSTEP_BREAK && ks > 0 && ks >= nks) break;  // warp-uniform
        if (!((lm >> ks) & 1u)) continue;
        Frag f;
        load(ks, f);
        issue(f);
      }
    }
  }

  // AL: the tile's warps may be aliased (runtime amap from the mask); otherwise amap is the
  // constant 0 and the alias logic folds away (its runtime form costs registers: spills at 128)
  template <bool LD = false, bool AL = false>
  __device__ static void compute_stage(const double* st, Acc& acc, unsigned mask = ~0u, int nks = BK / 4,
                                       const StageLd* ld = nullptr) {
    if constexpr (RECT) {
      if (mask == 0u) {  // warp-uniform
        if constexpr (LD) ld->all();
        return;
      }
      const int na = (mask >> 4) & 15, ncg = (mask >> 8) & 15;
      constexpr int BPG = VEC ? 2 : 1;  // sub-tiles per column group
      if constexpr (AL) {  // ragged tiles only: two bodies (code size)
        const unsigned amap = (mask >> 12) & 3u;
        if constexpr (MI >= 2) {
          if (na == 1) return compute_body<1, NI, false, LD>(st, acc, ~0u, nks, ld, amap);
        }
        return compute_body<MI, NI, false, LD>(st, acc, ~0u, nks, ld, amap);
      }
      if (na == MI && ncg == NCG) return compute_body<MI, NI, false, LD>(st, acc, ~0u, nks, ld);
      if constexpr (MI >= 2) {
        if (na == 1 && ncg == NCG) return compute_body<1, NI, false, LD>(st, acc, ~0u, nks, ld);
      }
      if constexpr (NCG >= 2) {
        if (na == MI && ncg == 1) return compute_body<MI, BPG, false, LD>(st, acc, ~0u, nks, ld);
        if (na == 1 && ncg == 1) return compute_body<1, BPG, false, LD>(st, acc, ~0u, nks, ld);
      }
      return compute_body<MI, NI, false, LD>(st, acc, ~0u, nks, ld);  // other shapes: full warp tile
    } else if constexpr (!FINE) {
      if (mask == 0u) {  // warp-uniform
        if constexpr (LD) ld->all();
        return;
      }
      compute_body<MI, NI, false, LD>(st, acc, ~0u, nks, ld);
    } else {
      compute_body<MI, NI, true, LD>(st, acc, mask, nks, ld);
    }
  }

  // Main loop over a segment list. SegFn: Seg(int idx). All threads of the CTA call this
  // with identical arguments.  smem: STAGES*STAGE doubles.  Ends with a __syncthreads().
  template <bool AL = false, class SegFn>
  __device__ static void run(SegFn segfn, int nseg, int m0, int n0, int M, int N, int64_t aim, int64_t bim,
                             double* smem, Acc& acc, unsigned mask = ~0u) {
    if constexpr (MBAR) {
      run_mbar(segfn, nseg, m0, n0, M, N, aim, bim, smem, acc, mask);
      return;
    }
    int pseg = 0, pk = 0;
    Seg cur;
    while (pseg < nseg) {  // skip empty segments
      cur = segfn(pseg);
      if (cur.K > 0) break;
      ++pseg;
    }
    auto advance = [&]() {
      pk += BK;
      if (pk >= cur.K) {
        pk = 0;
        ++pseg;
        while (pseg < nseg) {
          cur = segfn(pseg);
          if (cur.K > 0) break;
          ++pseg;
        }
      }
    };
    int issued = 0;
    unsigned kvpack = 0;  // per stage slot: k-steps of 4 holding data (4 bits each)
#ifndef DDK_KSKIP
#define DDK_KSKIP 1
#endif
    auto note_k = [&](int slot) {
      const int kv = DDK_KSKIP ? min(BK, cur.K - pk) : BK;
      kvpack = (kvpack & ~(15u << (4 * slot))) | ((unsigned)((kv + 3) / 4) << (4 * slot));
    };
    if constexpr (FASTLD) {
      FastLd f;
      fast_tile(f, smem, m0, n0, M, N);
      if (pseg < nseg) fast_seg(f, cur, m0, n0);
      StageLd sl;
      sl.f = &f;
      sl.sg = &cur;
      sl.m0 = m0, sl.n0 = n0, sl.M = M, sl.N = N, sl.aim = aim, sl.bim = bim;
      // choose how the next stage is copied (before the copies), then step to the stage after it
      auto plan = [&]() {
        sl.mode = 0;
        if (pseg < nseg) {
          sl.mode = (cur.acol == nullptr && pk + BK <= cur.K) ? 1 : 2;
          sl.slot = issued % STAGES;
          sl.st = smem + sl.slot * STAGE;
          sl.kofs = pk;
          note_k(issued % STAGES);
        }
      };
      auto step = [&]() {
        if (sl.mode) {
          const int was = pseg;
          advance();
          ++issued;
          if (pseg != was && pseg < nseg) fast_seg(f, cur, m0, n0);
        }
      };
#pragma unroll 1
      for (int s = 0; s < STAGES - 1; ++s) {
        plan();
        sl.generic();
        sl.all();
        step();
        cp_async_commit();
      }
      int done = 0;
#pragma unroll 1
      while (done < issued) {
        cp_async_wait<STAGES - 2>();
        __syncthreads();
        plan();
        sl.generic();
        const int slot = done % STAGES;
        compute_stage<true, AL>(smem + slot * STAGE, acc, mask, (int)((kvpack >> (4 * slot)) & 15u), &sl);
        step();
        cp_async_commit();
        ++done;
      }
      cp_async_wait<0>();
      __syncthreads();
      return;
    }
#pragma unroll 1
    for (int s = 0; s < STAGES - 1; ++s) {
      if (pseg < nseg) {
        load_stage(smem + (issued % STAGES) * STAGE, cur, pk, m0, n0, M, N, aim, bim);
        note_k(issued % STAGES);
        advance();
        ++issued;
      }
      cp_async_commit();
    }
    int done = 0;
#pragma unroll 1
    while (done < issued) {
      cp_async_wait<STAGES - 2>();
      __syncthreads();
      if (pseg < nseg) {
        load_stage(smem + (issued % STAGES) * STAGE, cur, pk, m0, n0, M, N, aim, bim);
        note_k(issued % STAGES);
        advance();
        ++issued;
      }
      cp_async_commit();
      const int slot = done % STAGES;
      compute_stage<false, AL>(smem + slot * STAGE, acc, mask, (int)((kvpack >> (4 * slot)) & 15u));
      ++done;
    }
    cp_async_wait<0>();
    __syncthreads();
  }

  // MBAR main loop: no CTA-wide barrier per stage.  A warp waits only for the data of the stage
  // it computes (full[s]) and, before refilling a buffer, for every warp to have consumed it
  // (empty[s], one stage of slack with STAGES >= 3), so warps drift within the pipeline depth.
  template <class SegFn>
  __device__ static void run_mbar(SegFn segfn, int nseg, int m0, int n0, int M, int N, int64_t aim, int64_t bim,
                                  double* smem, Acc& acc, unsigned mask) {
    static_assert(STAGES >= 3, "MBAR pipeline needs >= 3 stages");
    __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
    if (threadIdx.x == 0) {
#pragma unroll
      for (int q = 0; q < STAGES; ++q) {
        mbar_init(&full[q], NTHR);
        mbar_init(&empty[q], NTHR / 32);
      }
    }
    __syncthreads();
    int pseg = 0, pk = 0;
    Seg cur;
    while (pseg < nseg) {
      cur = segfn(pseg);
      if (cur.K > 0) break;
      ++pseg;
    }
    auto advance = [&]() {
      pk += BK;
      if (pk >= cur.K) {
        pk = 0;
        ++pseg;
        while (pseg < nseg) {
          cur = segfn(pseg);
          if (cur.K > 0) break;
          ++pseg;
        }
      }
    };
    int issued = 0;
    unsigned kvpack = 0;  // per stage slot: k-steps of 4 holding data (4 bits each)
    auto note_k = [&](int slot) {
      const int kv = DDK_KSKIP ? min(BK, cur.K - pk) : BK;
      kvpack = (kvpack & ~(15u << (4 * slot))) | ((unsigned)((kv + 3) / 4) << (4 * slot));
    };
    FastLd f;
    if constexpr (FASTLD_ANY) {
      fast_tile(f, smem, m0, n0, M, N);
      if (pseg < nseg) fast_seg(f, cur, m0, n0);
    }
    // one stage's copies (all at once: the interleaved form would have to wait for the buffer's
    // previous readers before the compute stage, i.e. a CTA-wide barrier again)
    auto load_next = [&](int slot) {
      note_k(slot);
      if constexpr (FASTLD_ANY) {
        StageLd sl;
        sl.f = &f, sl.sg = &cur, sl.slot = slot, sl.st = smem + slot * STAGE, sl.kofs = pk;
        sl.m0 = m0, sl.n0 = n0, sl.M = M, sl.N = N, sl.aim = aim, sl.bim = bim;
        sl.mode = (cur.acol == nullptr && pk + BK <= cur.K) ? 1 : 2;
        sl.generic();
        sl.all();
      } else {
        load_stage(smem + slot * STAGE, cur, pk, m0, n0, M, N, aim, bim);
      }
      mbar_cpasync_arrive(&full[slot]);
      const int was = pseg;
      advance();
      ++issued;
      if constexpr (FASTLD_ANY) {
        if (pseg != was && pseg < nseg) fast_seg(f, cur, m0, n0);
      }
    };
#pragma unroll 1
    for (int q = 0; q < STAGES - 1 && pseg < nseg; ++q) load_next(q);
    const int lane = threadIdx.x & 31;
    int done = 0;
#pragma unroll 1
    while (done < issued) {
      const int sb = done % STAGES;
      mbar_wait(&full[sb], (unsigned)((done / STAGES) & 1));
      compute_stage(smem + sb * STAGE, acc, mask, (int)((kvpack >> (4 * sb)) & 15u));
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[sb]);
      ++done;
      if (pseg < nseg) {
        const int nb = issued % STAGES;
        if (issued >= STAGES) mbar_wait(&empty[nb], (unsigned)(((issued - STAGES) / STAGES) & 1));
        load_next(nb);
      }
    }
    cp_async_wait<0>();
    __syncthreads();
  }
};

}  // namespace ddk
