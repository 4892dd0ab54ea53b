// tcgen05.mma throughput per shape on one SM (sm_100a): issue R MMAs
// back-to-back from one thread, commit, wait; SM clocks per MMA. Operands are
// uninitialised shared memory (throughput only).
#include <cstdio>
#include <cstdint>
#include "../../paper_2605_04569_b200/csrc/isa_ptx.cuh"
using namespace isa;

template <int M, int N, int TS, int BMN>
__global__ void __launch_bounds__(128, 1) mma_bench(long long* out, int reps) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  long long t = 0;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = idesc_bf16_f32(M, N, 0, BMN);
    const uint64_t da = sdesc_sw128_base(smem_u32(smem), 16, 1024);
    const uint64_t db = sdesc_sw128_base(smem_u32(smem + 65536), BMN ? 16384 : 16, 1024);
    for (int w = 0; w < 2; ++w) {
      const long long t0 = clock64();
      for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          if (TS)
            mma_ts(tmem + 256, tmem + 64 + kk * 8, db + (BMN ? kk * 128 : kk * 2), idesc, (r | kk) != 0);
          else
            mma_ss(tmem, da + kk * 2, db + kk * 2, idesc, (r | kk) != 0);
        }
      }
      mma_commit(&bar);
      mbar_wait(&bar, w & 1);
      t = clock64() - t0;
    }
    out[blockIdx.x] = t;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <int M, int N, int TS, int BMN = TS>
void run(long long* d, int ctas) {
  const int reps = 512;
  cudaFuncSetAttribute(mma_bench<M, N, TS, BMN>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  mma_bench<M, N, TS, BMN><<<ctas, 128, 200 * 1024>>>(d, reps);
  cudaError_t e = cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const double per = (double)h / (reps * 8.0);
  const double flop = 2.0 * M * N * 16;
  printf("M=%3d N=%3d %s%s ctas=%3d: %.1f clk/MMA  %.0f FLOP/clk/SM  (%s)\n", M, N, TS ? "TS" : "SS", BMN ? "(B MN-major)" : "", ctas, per,
         flop / per, cudaGetErrorString(e));
}

int main() {
  long long* d;
  cudaMalloc(&d, 1024 * 8);
  for (int ctas : {1, 148}) {
    run<128, 256, 0>(d, ctas);
    run<128, 128, 0>(d, ctas);
    run<128, 64, 0>(d, ctas);
    run<64, 256, 0>(d, ctas);
    run<64, 128, 0>(d, ctas);
    run<64, 64, 0>(d, ctas);
    run<128, 128, 1>(d, ctas);
    run<64, 128, 1>(d, ctas);
    run<128, 64, 1, 0>(d, ctas);
    run<128, 128, 1, 0>(d, ctas);
    run<128, 256, 1, 0>(d, ctas);
  }
  return 0;
}
