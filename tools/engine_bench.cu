// Microbenchmark of the DMMA tile engine (paper_2002_05019_b200/csrc/gemm_core.cuh) on a dense
// C -= A B^T (M = N = K = 8192), no sparsity, to separate engine efficiency from the
// block-sparse workload's tile structure.  Build + run (GPU box):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2002_05019_b200/csrc \
//        tools/engine_bench.cu -o /tmp/engine_bench && /tmp/engine_bench
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "gemm_core.cuh"

using namespace ddk;

// Fixed-cost probes (K3 regime): EPI 0 = fragment-order RMW, 1 = store_tile<1> (coalesced, + C-tile L2 prefetch),
// 2 = no read-modify-write (one guarded store); PERSIST = one CTA per resident slot striding over the tiles
template <class G, bool C, int BM, int BN, int EPI, bool PERSIST>
__global__ void __launch_bounds__(G::NTHR, 4) dense2(const double* A, const double* B, double* Cm, int M, int N, int K,
                                                     int ksplit) {
  extern __shared__ __align__(16) double smem[];
  const int ntile = (M / BM) * (N / BN);
  for (int tile = blockIdx.x; tile < ntile; tile += PERSIST ? gridDim.x : ntile) {
    const int tm = tile % (M / BM), tn = tile / (M / BM);
    typename G::Acc acc;
    G::zero(acc);
    auto segfn = [&](int q) {
      Seg s;
      s.a = A + (int64_t)q * ksplit * M;
      s.b = B + (int64_t)q * ksplit * N;
      s.acol = nullptr;
      s.lda = M;
      s.ldb = N;
      s.K = ksplit;
      return s;
    };
    double* Cb = Cm + (int64_t)tm * BM + (int64_t)tn * BN * M;
    if (EPI == 1) G::prefetch_tile_l2(Cb, M, 0, BM, BN);
    G::run(segfn, K / ksplit, tm * BM, tn * BN, M, N, 0, 0, smem, acc);
    if (EPI == 0) {
      G::for_each(acc, [&](int r, int c, double vr, double vi) { Cb[(int64_t)r + (int64_t)c * M] -= vr; });
    } else if (EPI == 1) {
      G::template store_tile<1>(acc, smem, Cb, M, 0, BM, BN);
    } else if (EPI == 3) {
      G::template store_tile<2>(acc, smem, Cb, M, 0, BM, BN);
    } else {
      double sum = 0.0;
      G::for_each(acc, [&](int r, int c, double vr, double vi) { sum += vr; });
      if (sum == 123.456) Cb[threadIdx.x] = sum;
    }
  }
}

template <class G, bool C, int BM, int BN, int EPI, bool PERSIST>
void run2(const char* name, int M, int K, int ksplit) {
  const int N = M;
  double *A, *B, *Cm;
  cudaMalloc(&A, (size_t)M * K * 8);
  cudaMalloc(&B, (size_t)N * K * 8);
  cudaMalloc(&Cm, (size_t)M * N * 8);
  cudaMemset(A, 0, (size_t)M * K * 8);
  cudaMemset(B, 0, (size_t)N * K * 8);
  cudaMemset(Cm, 0, (size_t)M * N * 8);
  auto kern = dense2<G, C, BM, BN, EPI, PERSIST>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM_BYTES);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, G::NTHR, G::SMEM_BYTES);
  const int ntile = (M / BM) * (N / BN);
  const int grid = PERSIST ? occ * 148 : ntile;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int it = 0; it < 2; ++it) kern<<<grid, G::NTHR, G::SMEM_BYTES>>>(A, B, Cm, M, N, K, ksplit);
  cudaEventRecord(e0);
  const int reps = 3;
  for (int it = 0; it < reps; ++it) kern<<<grid, G::NTHR, G::SMEM_BYTES>>>(A, B, Cm, M, N, K, ksplit);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  double flops = 2.0 * M * N * (double)K * reps;
  printf("%-44s M=N=%d K=%d occ=%d/SM grid=%d  %.2f TF/s  err=%s\n", name, M, K, occ, grid,
         flops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  cudaFree(A);
  cudaFree(B);
  cudaFree(Cm);
}

template <class G, bool C, int BM, int BN, bool AKM = false, bool BKN = false>
__global__ void __launch_bounds__(G::NTHR) dense(const double* A, const double* B, double* Cm, int M, int N, int K,
                                                 int64_t aim, int64_t bim, int64_t cim, int ksplit) {
  extern __shared__ __align__(16) double smem[];
  const int tm = blockIdx.x % (M / BM), tn = blockIdx.x / (M / BM);
  typename G::Acc acc;
  G::zero(acc);
  // K split into segments of ksplit columns (exercises the gathered-K path like k3_update)
  auto segfn = [&](int q) {
    Seg s;
    // MK: a[m + k*M]; KM: a[k + m*K]  /  NK: b[n + k*N]; KN: b[k + n*K]
    s.a = AKM ? A + (int64_t)q * ksplit : A + (int64_t)q * ksplit * M;
    s.b = BKN ? B + (int64_t)q * ksplit : B + (int64_t)q * ksplit * N;
    s.acol = nullptr;
    s.lda = AKM ? K : M;
    s.ldb = BKN ? K : N;
    s.K = ksplit;
    return s;
  };
  G::run(segfn, K / ksplit, tm * BM, tn * BN, M, N, aim, bim, smem, acc);
  double* Cb = Cm + (int64_t)tm * BM + (int64_t)tn * BN * M;
  G::for_each(acc, [&](int r, int c, double vr, double vi) {
    int64_t e = (int64_t)r + (int64_t)c * M;
    Cb[e] -= vr;
    if (C) Cb[e + cim] -= vi;
  });
}

template <class G, bool C, int BM, int BN, bool AKM = false, bool BKN = false>
void run(const char* name, int M, int K, int ksplit) {
  const int N = M;
  const int pl = C ? 2 : 1;
  double *A, *B, *Cm;
  cudaMalloc(&A, (size_t)M * K * pl * 8);
  cudaMalloc(&B, (size_t)N * K * pl * 8);
  cudaMalloc(&Cm, (size_t)M * N * pl * 8);
  cudaMemset(A, 0, (size_t)M * K * pl * 8);
  cudaMemset(B, 0, (size_t)N * K * pl * 8);
  cudaMemset(Cm, 0, (size_t)M * N * pl * 8);
  auto kern = dense<G, C, BM, BN, AKM, BKN>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM_BYTES);
  int grid = (M / BM) * (N / BN);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, G::NTHR, G::SMEM_BYTES);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int it = 0; it < 2; ++it)
    kern<<<grid, G::NTHR, G::SMEM_BYTES>>>(A, B, Cm, M, N, K, (int64_t)M * K, (int64_t)N * K, (int64_t)M * N, ksplit);
  cudaEventRecord(e0);
  const int reps = 3;
  for (int it = 0; it < reps; ++it)
    kern<<<grid, G::NTHR, G::SMEM_BYTES>>>(A, B, Cm, M, N, K, (int64_t)M * K, (int64_t)N * K, (int64_t)M * N, ksplit);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  double flops = 2.0 * M * N * (double)K * (C ? 4 : 1) * reps;
  printf("%-34s M=N=%d K=%d ksplit=%d occ=%d/SM smem=%zuKB  %.2f TF/s  err=%s\n", name, M, K, ksplit, occ,
         G::SMEM_BYTES / 1024, flops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  cudaFree(A);
  cudaFree(B);
  cudaFree(Cm);
}

int main(int argc, char** argv) {
  if (argc > 1) {  // fixed-cost probes only
    using G13 = Gemm<64, 64, 16, 2, 2, 2, false, false, false, false, false, false, true>;
    using G24 = Gemm<64, 64, 24, 2, 2, 2, false, false, false, false, false, false, true>;
    for (int K : {576, 2304, 9216}) {
      run2<G13, false, 64, 64, 0, false>("64x64 2st frag-RMW", 8192, K, 576);
      run2<G13, false, 64, 64, 1, false>("64x64 2st store_tile+prefetch", 8192, K, 576);
      run2<G13, false, 64, 64, 2, false>("64x64 2st no epilogue", 8192, K, 576);
      run2<G13, false, 64, 64, 3, false>("64x64 2st L2 reductions (red.add.f64)", 8192, K, 576);
      run2<G24, false, 64, 64, 3, false>("64x64 BK24 2st L2 reductions", 8192, K, 576);
      run2<G13, false, 64, 64, 1, true>("64x64 2st store_tile persistent", 8192, K, 576);
      run2<G13, false, 64, 64, 2, true>("64x64 2st no epilogue persistent", 8192, K, 576);
      run2<G24, false, 64, 64, 1, false>("64x64 BK24 2st store_tile+prefetch", 8192, K, 576);
    }
    return 0;
  }
  // configurations used by k3_update (see kernels_factor.cu K3Cfg)
  run<Gemm<128, 64, 16, 2, 2, 3, false, false, false>, false, 128, 64>("real 128x64 4w 3st (cfg1)", 8192, 8192, 512);
  run<Gemm<128, 64, 16, 2, 2, 4, false, false, false>, false, 128, 64>("real 128x64 4w 4st (cfg2)", 8192, 8192, 512);
  run<Gemm<128, 128, 16, 2, 4, 4, false, false, false>, false, 128, 128>("real 128x128 8w 4st (cfg0)", 8192, 8192, 512);
  run<Gemm<64, 64, 16, 2, 2, 3, false, false, false>, false, 64, 64>("real 64x64 4w 3st", 8192, 8192, 512);
  run<Gemm<128, 64, 32, 2, 2, 3, false, false, false>, false, 128, 64>("real 128x64 4w BK32 3st", 8192, 8192, 512);
  run<Gemm<64, 128, 16, 2, 2, 3, false, false, false>, false, 64, 128>("real 64x128 4w 3st", 8192, 8192, 512);
  run<Gemm<64, 64, 16, 2, 2, 3, true, false, false>, true, 64, 64>("cplx 64x64 4w 3st (cfg1)", 8192, 4096, 512);
  run<Gemm<64, 128, 16, 2, 4, 3, true, false, false>, true, 64, 128>("cplx 64x128 8w 3st (cfg0)", 8192, 4096, 512);
  run<Gemm<128, 64, 16, 2, 2, 3, false, false, false>, false, 128, 64>("real 128x64 4w 3st ksplit 8192", 8192, 8192, 8192);
  // solve-kernel layouts (fupd: MK x KN, bupd: KM x KN)
  run<Gemm<64, 64, 16, 2, 2, 3, true, false, true>, true, 64, 64, false, true>("cplx 64x64 MKxKN (fupd)", 8192, 4096, 512);
  run<Gemm<64, 64, 16, 2, 2, 3, true, true, true>, true, 64, 64, true, true>("cplx 64x64 KMxKN (bupd)", 8192, 4096, 512);
  run<Gemm<64, 64, 16, 2, 2, 3, false, false, true>, false, 64, 64, false, true>("real 64x64 MKxKN (fupd)", 8192, 8192, 512);
  run<Gemm<64, 64, 16, 2, 2, 3, false, true, true>, false, 64, 64, true, true>("real 64x64 KMxKN (bupd)", 8192, 8192, 512);
  run<Gemm<64, 64, 32, 2, 2, 3, true, true, true>, true, 64, 64, true, true>("cplx 64x64 KMxKN BK32", 8192, 4096, 512);
  run<Gemm<64, 32, 16, 2, 2, 2, true, false, false>, true, 64, 32>("cplx 64x32 2st", 8192, 4096, 512);
  // short K per tile (the K3 regime: one contributor of ~512-600 columns)
  run<Gemm<64, 64, 16, 2, 2, 3, false, false, false>, false, 64, 64>("real 64x64 K=512", 8192, 512, 512);
  run<Gemm<64, 64, 16, 2, 2, 3, false, false, false>, false, 64, 64>("real 64x64 K=1024", 8192, 1024, 512);
  run<Gemm<64, 32, 16, 2, 2, 2, true, false, false>, true, 64, 32>("cplx 64x32 K=512", 8192, 512, 512);
  // mbarrier pipeline (no CTA barrier per stage) vs __syncthreads pipeline, K3 real regime
  run<Gemm<64, 64, 16, 2, 2, 2, false, false, false, false, false, false, true>, false, 64, 64>("real 64x64 RECT 2st K=576", 8192, 576, 576);
  run<Gemm<64, 64, 16, 2, 2, 3, false, false, false, false, false, false, true>, false, 64, 64>("real 64x64 RECT 3st K=576", 8192, 576, 576);
  run<Gemm<64, 64, 16, 2, 2, 2, false, false, false, false, false, false, true>, false, 64, 64>("real 64x64 RECT 2st K=8192", 8192, 8192, 512);
  run<Gemm<64, 64, 16, 2, 2, 3, false, false, false, false, false, false, true, true>, false, 64, 64>("real 64x64 RECT 3st MBAR K=576", 8192, 576, 576);
  run<Gemm<64, 64, 16, 2, 2, 4, false, false, false, false, false, false, true, true>, false, 64, 64>("real 64x64 RECT 4st MBAR K=576", 8192, 576, 576);
  run<Gemm<64, 64, 16, 2, 2, 3, false, false, false, false, false, false, true, true>, false, 64, 64>("real 64x64 RECT 3st MBAR K=8192", 8192, 8192, 512);
  run<Gemm<64, 32, 16, 2, 2, 2, true, false, false, true, true, true>, true, 64, 32>("cplx 64x32 3M VEC 2st K=512", 8192, 512, 512);
  run<Gemm<64, 32, 16, 2, 2, 3, true, false, false, true, true, true, false, true>, true, 64, 32>("cplx 64x32 3M VEC 3st MBAR K=512", 8192, 512, 512);
  // more warps per tile (latency hiding): 8 warps of 32x16 on a 64x64 tile; 128x64 with 8 warps of 32x32
  run<Gemm<64, 64, 16, 2, 4, 2, false, false, false, false, false, false, true>, false, 64, 64>("real 64x64 8w RECT 2st K=576", 8192, 576, 576);
  run<Gemm<64, 64, 16, 2, 4, 3, false, false, false, false, false, false, true>, false, 64, 64>("real 64x64 8w RECT 3st K=576", 8192, 576, 576);
  run<Gemm<64, 64, 16, 2, 4, 2, false, false, false, false, false, false, true>, false, 64, 64>("real 64x64 8w RECT 2st K=8192", 8192, 8192, 512);
  run<Gemm<128, 64, 16, 4, 2, 3, false, false, false, false, false, false, true>, false, 128, 64>("real 128x64 8w RECT 3st K=576", 8192, 576, 576);
  run<Gemm<128, 64, 16, 4, 2, 3, false, false, false, false, false, false, true>, false, 128, 64>("real 128x64 8w RECT 3st K=8192", 8192, 8192, 512);
  run<Gemm<128, 128, 16, 4, 4, 4, false, false, false, false, false, false, true>, false, 128, 128>("real 128x128 16w RECT 4st K=576", 8192, 576, 576);
  return 0;
}
