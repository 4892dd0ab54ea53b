// mma.sync m16n8k16 bf16->f32 throughput on sm_100a (legacy warp MMA path).
#include <cstdio>
#include <cstdint>
__global__ void k(float* out, long long* clk, int n) {
  uint32_t a[4] = {threadIdx.x, threadIdx.x * 3u, threadIdx.x * 5u, threadIdx.x * 7u};
  uint32_t b0 = threadIdx.x * 11u, b1 = threadIdx.x * 13u;
  float c[8][4] = {};
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                   : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  }
  long long t1 = clock64();
  float s = 0;
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}
int main() {
  float* o; long long* c;
  cudaMalloc(&o, 148 * 1024 * 4); cudaMalloc(&c, 148 * 8);
  for (int w : {4, 8, 16}) {
    const int n = 4096;
    k<<<148, 32 * w>>>(o, c, 16);
    k<<<148, 32 * w>>>(o, c, n);
    cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    double flop = 2.0 * 16 * 8 * 16 * 8.0 * n * w;  // per SM
    printf("warps/SM=%2d: %.1f clk per mma per SM, %.0f FLOP/clk/SM (tcgen05 peak 8192)\n", w,
           (double)h / (8.0 * n * w), flop / h);
  }
}
