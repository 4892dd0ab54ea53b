// Does mma.sync.m8n8k4 f64 (DMMA) accumulate its k = 4 products as the
// sequential FMA chain c = fma(a3, b3, fma(a2, b2, fma(a1, b1, fma(a0, b0, c))))?
// Random fp32-representable operands (like the coarse scores' fp32 means);
// counts bit mismatches against both chain orders.
#include <cstdio>
#include <cstdint>

__global__ void k(const double* A, const double* B, const double* C, double* D, double* F, double* R, int trials) {
  const int lane = threadIdx.x;
  for (int t = 0; t < trials; ++t) {
    const double* a = A + t * 32;  // 8 x 4 row-major
    const double* b = B + t * 32;  // 4 x 8 (k x n)
    const double* c = C + t * 64;  // 8 x 8
    // fragments: A row = lane/4, col = lane%4; B row(k) = lane%4, col = lane/4; C rows lane/4, cols 2*(lane%4)+{0,1}
    double af = a[(lane >> 2) * 4 + (lane & 3)];
    double bf = b[(lane & 3) * 8 + (lane >> 2)];
    double c0 = c[(lane >> 2) * 8 + 2 * (lane & 3)], c1 = c[(lane >> 2) * 8 + 2 * (lane & 3) + 1];
    double d0, d1;
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};"
                 : "=d"(d0), "=d"(d1) : "d"(af), "d"(bf), "d"(c0), "d"(c1));
    D[t * 64 + (lane >> 2) * 8 + 2 * (lane & 3)] = d0;
    D[t * 64 + (lane >> 2) * 8 + 2 * (lane & 3) + 1] = d1;
    if (lane < 64 / 2) {
      for (int e = lane; e < 64; e += 32) {
        const int i = e / 8, j = e % 8;
        double f = c[e], r = c[e];
        for (int kk = 0; kk < 4; ++kk) f = fma(a[i * 4 + kk], b[kk * 8 + j], f);
        for (int kk = 3; kk >= 0; --kk) r = fma(a[i * 4 + kk], b[kk * 8 + j], r);
        F[t * 64 + e] = f;
        R[t * 64 + e] = r;
      }
    }
  }
}

int main() {
  const int T = 4096;
  double *hA = new double[T * 32], *hB = new double[T * 32], *hC = new double[T * 64];
  uint64_t s = 12345;
  auto rnd = [&]() {
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    return (float)((int64_t)(s >> 11) - (1ll << 52)) / (float)(1ll << 52);  // fp32 value in (-1, 1)
  };
  for (int i = 0; i < T * 32; ++i) hA[i] = rnd(), hB[i] = rnd();
  for (int i = 0; i < T * 64; ++i) hC[i] = (double)rnd() * 3.0 + (double)rnd() * 1e-9;
  double *A, *B, *C, *D, *F, *R;
  cudaMalloc(&A, T * 32 * 8); cudaMalloc(&B, T * 32 * 8); cudaMalloc(&C, T * 64 * 8);
  cudaMalloc(&D, T * 64 * 8); cudaMalloc(&F, T * 64 * 8); cudaMalloc(&R, T * 64 * 8);
  cudaMemcpy(A, hA, T * 32 * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(B, hB, T * 32 * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(C, hC, T * 64 * 8, cudaMemcpyHostToDevice);
  k<<<1, 32>>>(A, B, C, D, F, R, T);
  double *hD = new double[T * 64], *hF = new double[T * 64], *hR = new double[T * 64];
  cudaMemcpy(hD, D, T * 64 * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(hF, F, T * 64 * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(hR, R, T * 64 * 8, cudaMemcpyDeviceToHost);
  int mf = 0, mr = 0;
  for (int i = 0; i < T * 64; ++i) mf += hD[i] != hF[i], mr += hD[i] != hR[i];
  printf("DMMA vs chain k=0..3: %d / %d mismatches; vs chain k=3..0: %d / %d (%s)\n", mf, T * 64, mr, T * 64,
         cudaGetErrorString(cudaGetLastError()));
}
