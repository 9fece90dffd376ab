// f1: on-device clique assembly of the auxiliary matrix.
//
// PAPER.md:27 (§II): eliminating each subdomain's primal unknowns leaves a dense
// contribution over the dual DoFs of the interfaces the subdomain touches; PAPER.md:29:
// the auxiliary matrix is the resulting "sparse collection of dense blocks", one dense
// clique per subdomain.  Assembly is the plain sum
//     A_IJ = sum_{p : I, J in clique p} S_p[rows of I, cols of J]        (I >= J, lower blocks)
// with the optional symmetric part (S_p + S_p^T)/2 taken first (reading L12).
//
// HBM-bound: every S_p entry that lands in an output block is read once (for an off-diagonal
// block with the symmetric part also its mirror S_p[J, I], through a 32x32 shared tile so both
// reads are coalesced; a diagonal block computes its lower tiles and stores each mirrored, so its
// S_p entries are read once as well) and every output element is written once.  Owner-computes over output tiles
// with the contributors summed in ascending clique order (deterministic, no atomics); the
// additions are explicitly rounded (__dadd_rn / __dmul_rn) so no FMA contraction changes them.
#include <cuda_runtime.h>

#include "launch.hpp"

namespace ddk {

namespace {

template <bool C>
struct Elem;
template <>
struct Elem<false> {
  using T = double;
  __device__ static T zero() { return 0.0; }
  __device__ static T add(T a, T b) { return __dadd_rn(a, b); }
  __device__ static T half_sum(T a, T b) { return __dmul_rn(0.5, __dadd_rn(a, b)); }
};
template <>
struct Elem<true> {
  using T = double2;  // (re, im) interleaved, like torch.complex128
  __device__ static T zero() { return make_double2(0.0, 0.0); }
  __device__ static T add(T a, T b) { return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y)); }
  __device__ static T half_sum(T a, T b) {
    return make_double2(__dmul_rn(0.5, __dadd_rn(a.x, b.x)), __dmul_rn(0.5, __dadd_rn(a.y, b.y)));
  }
};

constexpr int AT = 32;     // output tile edge
constexpr int ATY = 8;     // thread rows (256 threads: 32 x 8, 4 columns each)

}  // namespace

// One CTA per (output block, 32-column chunk); loops over 32-row tiles of the block.
// ACC (SYM = false only): accumulate onto the block's current values; a template parameter so the
// plain assembly carries no per-element branch for it (as a runtime flag it cost cfg2's assembly
// 11.5 -> 12.3 ms).
template <bool C, bool SYM, bool ACC = false>
__global__ void __launch_bounds__(AT * ATY) k_assemble(AsmArgs a) {
  using E = Elem<C>;
  using T = typename E::T;
  __shared__ T tileT[AT][AT + 1];
  const AsmItem it = a.items[blockIdx.x];
  const T* S = reinterpret_cast<const T*>(a.S);
  T* out = reinterpret_cast<T*>(a.vals) + it.dst;
  const int tx = threadIdx.x % AT, ty = threadIdx.x / AT;
  // diagonal block with the symmetric part: the result is symmetric, so only the tiles on and
  // below the diagonal are computed and each off-diagonal one is also stored mirrored -- every
  // S_p element of the block is then read from HBM once (the pair S[r0, c0] / S[c0, r0] is read by
  // this CTA only)
  const bool mirror = SYM && it.pad;
  if (ACC && it.k0 == it.k1) return;  // accumulate mode: blocks no clique covers keep their values
  for (int r0 = mirror ? it.c0 : 0; r0 < it.rows; r0 += AT) {
    T acc[AT / ATY];
#pragma unroll
    for (int j = 0; j < AT / ATY; ++j) {
      const int row = r0 + tx, col = it.c0 + ty + ATY * j;  // accumulate (SYM = false only): start from the block
      acc[j] = (ACC && row < it.rows && col < it.cols) ? out[row + (int64_t)col * it.rows] : E::zero();
    }
    for (int q = it.k0; q < it.k1; ++q) {
      const AsmContrib c = a.con[q];
      const T* Sp = S + c.soff;
      T v[AT / ATY];
#pragma unroll
      for (int j = 0; j < AT / ATY; ++j) {
        const int row = r0 + tx, col = it.c0 + ty + ATY * j;
        v[j] = (row < it.rows && col < it.cols) ? Sp[(c.ra + row) + (int64_t)(c.cb + col) * c.ld] : E::zero();
      }
      if constexpr (SYM) {
        // S_p^T entry (row, col) = S_p[cb + col, ra + row]: read row-wise (coalesced over col)
        __syncthreads();
#pragma unroll
        for (int j = 0; j < AT / ATY; ++j) {
          const int row = r0 + ty + ATY * j, col = it.c0 + tx;
          tileT[ty + ATY * j][tx] =
              (row < it.rows && col < it.cols) ? Sp[(c.cb + col) + (int64_t)(c.ra + row) * c.ld] : E::zero();
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < AT / ATY; ++j) v[j] = E::half_sum(v[j], tileT[tx][ty + ATY * j]);
      }
#pragma unroll
      for (int j = 0; j < AT / ATY; ++j) acc[j] = E::add(acc[j], v[j]);
    }
#pragma unroll
    for (int j = 0; j < AT / ATY; ++j) {
      const int row = r0 + tx, col = it.c0 + ty + ATY * j;
      if (row < it.rows && col < it.cols) out[row + (int64_t)col * it.rows] = acc[j];
    }
    if (SYM && mirror && r0 > it.c0) {  // the mirrored tile (c0.., r0..) = this tile transposed
      __syncthreads();
#pragma unroll
      for (int j = 0; j < AT / ATY; ++j) tileT[ty + ATY * j][tx] = acc[j];
      __syncthreads();
#pragma unroll
      for (int j = 0; j < AT / ATY; ++j) {
        const int row = it.c0 + tx, col = r0 + ty + ATY * j;
        if (row < it.rows && col < it.cols) out[row + (int64_t)col * it.rows] = tileT[tx][ty + ATY * j];
      }
    }
  }
}

int asm_chunk() { return AT; }

void launch_assemble(bool cplx, bool sym, const AsmArgs& a, int nitems, cudaStream_t st) {
  if (nitems <= 0) return;
  const dim3 grid(nitems), block(AT * ATY);
  const bool acc = a.accumulate != 0;  // api.cu only passes accumulate with sym off
  if (cplx) {
    if (sym) k_assemble<true, true><<<grid, block, 0, st>>>(a);
    else if (acc) k_assemble<true, false, true><<<grid, block, 0, st>>>(a);
    else k_assemble<true, false><<<grid, block, 0, st>>>(a);
  } else {
    if (sym) k_assemble<false, true><<<grid, block, 0, st>>>(a);
    else if (acc) k_assemble<false, false, true><<<grid, block, 0, st>>>(a);
    else k_assemble<false, false><<<grid, block, 0, st>>>(a);
  }
}

}  // namespace ddk
