// fp64 throughput on sm_100a: DMMA m8n8k4 vs DFMA.
#include <cstdio>
__global__ void kd(double* out, long long* clk, int n) {
  double a = threadIdx.x * 1e-3, b = threadIdx.x * 2e-3;
  double c[8][2] = {};
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
  }
  long long t1 = clock64();
  double s = 0;
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}
__global__ void kf(double* out, long long* clk, int n) {
  double a = threadIdx.x * 1e-3, b = threadIdx.x * 2e-3;
  double c[8] = {};
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) asm volatile("fma.rn.f64 %0, %1, %2, %0;" : "+d"(c[j]) : "d"(a), "d"(b));
  }
  long long t1 = clock64();
  double s = 0;
  for (int j = 0; j < 8; ++j) s += c[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}
int main() {
  double* o; long long* c;
  cudaMalloc(&o, 148 * 1024 * 8); cudaMalloc(&c, 148 * 8);
  for (int w : {4, 8, 16}) {
    const int n = 2048;
    kd<<<148, 32 * w>>>(o, c, 16); kd<<<148, 32 * w>>>(o, c, n); cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("DMMA m8n8k4 warps/SM=%2d: %.1f FMA/clk/SM\n", w, 256.0 * 8 * n * w / h);
    kf<<<148, 32 * w>>>(o, c, 16); kf<<<148, 32 * w>>>(o, c, n); cudaDeviceSynchronize();
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("DFMA        warps/SM=%2d: %.1f FMA/clk/SM\n", w, 32.0 * 8 * n * w / h);
  }
}
