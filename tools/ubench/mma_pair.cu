// tcgen05.mma.cta_group::2 (CTA pair, M = 256) throughput per N on a 2-CTA
// cluster vs cta_group::1 M = 128 (tools/ubench/mma.cu): does the pair form
// lift the ~45-clk per-instruction floor of N = 64? The leader CTA issues R
// back-to-back MMAs, commits (multicast to both CTAs), waits; SM clocks per
// MMA = per-SM time for a 128-row share. Operands: uninitialised smem.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mma_pair mma_pair.cu
#include <cstdio>
#include <cstdint>
#include "../../paper_2605_04569_b200/csrc/isa_ptx.cuh"
using namespace isa;

template <int N, int TS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) pair_bench(long long* out, int reps) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = cluster_ctarank();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc2<512>(&slot);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = slot;
  long long t = 0;
  if (rank == 0 && threadIdx.x == 0) {
    constexpr uint32_t idesc = idesc_bf16_f32(256, N, 0, TS ? 1 : 0);
    const uint64_t da = sdesc_sw128_base(smem_u32(smem), 16, 1024);
    const uint64_t db = sdesc_sw128_base(smem_u32(smem + 65536), TS ? 16384 : 16, 1024);
    for (int w = 0; w < 2; ++w) {
      const long long t0 = clock64();
      for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          if (TS)
            mma_ts2(tmem + 256, tmem + 64 + kk * 8, db + kk * 128, idesc, (r | kk) != 0);
          else
            mma_ss2(tmem, da + kk * 2, db + kk * 2, idesc, (r | kk) != 0);
        }
      }
      mma_commit_pair(&bar);
      mbar_wait(&bar, w & 1);
      t = clock64() - t0;
    }
    out[blockIdx.x / 2] = t;
  } else if (rank == 1 && threadIdx.x == 0) {
    for (int w = 0; w < 2; ++w) mbar_wait(&bar, w & 1);
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc2<512>(tmem);
  }
}

template <int N, int TS>
void run(long long* d, int clusters) {
  const int reps = 512;
  cudaFuncSetAttribute(pair_bench<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  pair_bench<N, TS><<<2 * clusters, 128, 200 * 1024>>>(d, reps);
  cudaError_t e = cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const double per = (double)h / (reps * 8.0);
  const double flop_per_sm = 2.0 * 128 * N * 16;  // each SM's 128-row share
  printf("pair M=256 N=%3d %s clusters=%2d: %.1f clk/MMA  %.0f FLOP/clk/SM  (%s)\n", N, TS ? "TS" : "SS", clusters, per,
         flop_per_sm / per, cudaGetErrorString(e));
}

int main() {
  long long* d;
  cudaMalloc(&d, 1024 * 8);
  for (int c : {1, 74}) {
    run<64, 0>(d, c);
    run<128, 0>(d, c);
    run<256, 0>(d, c);
    run<64, 1>(d, c);
    run<128, 1>(d, c);
  }
  return 0;
}
