// L2 -> SM bandwidth on B200 (the roofline of the L2-resident operand streams
// of K7T): every CTA streams an L2-resident buffer into shared memory with
// (a) 16-byte LDG per thread and (b) cp.async.bulk (TMA bulk copies of 16 KB
// chunks, 4 in flight per CTA, mbarrier completion). Bytes moved / time.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2bw l2bw.cu && ./l2bw
#include <cstdio>
#include <cstdint>

__global__ void __launch_bounds__(512) ldg_kernel(const int4* __restrict__ buf, size_t n16, int reps, int4* sink) {
  int4 acc = make_int4(0, 0, 0, 0);
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
      int4 v = __ldcg(buf + i);
      acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
  if (acc.x == 0x12345678) sink[threadIdx.x] = acc;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

constexpr int kChunk = 16384, kSlots = 4;
__global__ void __launch_bounds__(32) bulk_kernel(const char* __restrict__ buf, size_t bytes, int reps, int* sink) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) uint64_t bar[kSlots];
  if (threadIdx.x == 0) {
    for (int s = 0; s < kSlots; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncwarp();
  if (threadIdx.x != 0) return;
  const size_t chunks = bytes / kChunk;
  uint32_t phase[kSlots] = {0, 0, 0, 0};
  long long issued = 0;
  const long long total = (long long)reps * ((chunks - blockIdx.x + gridDim.x - 1) / gridDim.x);
  long long done = 0;
  auto issue = [&](long long it) {
    const int s = it % kSlots;
    const size_t c = blockIdx.x + (size_t)(it % ((chunks - blockIdx.x + gridDim.x - 1) / gridDim.x)) * gridDim.x;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"(kChunk));
    asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(sm + s * kChunk)),
                 "l"(buf + c * kChunk), "r"(kChunk), "r"(smem_u32(&bar[s]))
                 : "memory");
  };
  for (; issued < total && issued < kSlots; ++issued) issue(issued);
  for (; done < total; ++done) {
    const int s = done % kSlots;
    asm volatile(
        "{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(smem_u32(&bar[s])),
        "r"(phase[s]));
    phase[s] ^= 1;
    if (issued < total) issue(issued++);
  }
  if (sm[0] == 123 && sm[1] == 45) sink[blockIdx.x] = 1;
}

int main() {
  const size_t bytes = 64ull << 20;  // L2-resident (126 MB L2)
  char* buf;
  int* sink;
  cudaMalloc(&buf, bytes);
  cudaMalloc(&sink, 1 << 20);
  cudaMemset(buf, 1, bytes);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int reps = 20;
  for (int blocks_per_sm : {1, 2, 4}) {
    ldg_kernel<<<148 * blocks_per_sm, 512>>>((const int4*)buf, bytes / 16, 2, (int4*)sink);
    cudaEventRecord(a);
    ldg_kernel<<<148 * blocks_per_sm, 512>>>((const int4*)buf, bytes / 16, reps, (int4*)sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("LDG.128   %d x 512 threads/SM: %8.1f GB/s (%.1f B/clk/SM at 1.965 GHz)\n", blocks_per_sm,
           bytes * (double)reps / ms / 1e6, bytes * (double)reps / (ms * 1e-3) / 148 / 1.965e9);
  }
  cudaFuncSetAttribute(bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kChunk * kSlots);
  for (int ctas : {1, 2, 3}) {
    bulk_kernel<<<148 * ctas, 32, kChunk * kSlots>>>(buf, bytes, 2, sink);
    cudaEventRecord(a);
    bulk_kernel<<<148 * ctas, 32, kChunk * kSlots>>>(buf, bytes, reps, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("TMA bulk  %d CTA/SM x %d x 16 KB in flight: %8.1f GB/s (%.1f B/clk/SM at 1.965 GHz)\n", ctas, kSlots,
           bytes * (double)reps / ms / 1e6, bytes * (double)reps / (ms * 1e-3) / 148 / 1.965e9);
  }
  cudaError_t e = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(e));
}
