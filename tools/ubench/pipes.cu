// Per-SMSP issue throughput of the softmax instruction mix on sm_100a.
// One CTA per SM, W warps per SMSP (4*W warps/CTA); each warp runs N
// iterations of 8 independent chains of one instruction kind. Reports
// SM clocks per warp-instruction per SMSP (= 1 / throughput).
#include <cstdio>
#include <cuda_bf16.h>

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(*reinterpret_cast<unsigned long long*>(&d))
      : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)),
        "l"(*reinterpret_cast<unsigned long long*>(&c)));
  return d;
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  float2 d;
  asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(*reinterpret_cast<unsigned long long*>(&d))
      : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)));
  return d;
}

template <int KIND>
__global__ void bench(float* out, long long* clk, int n) {
  float a[8];
  float2 b[8];
  unsigned u[8];
  for (int j = 0; j < 8; ++j) {
    a[j] = -0.001f * (threadIdx.x + j);
    b[j] = make_float2(a[j], a[j] * 0.5f);
    u[j] = threadIdx.x * 7 + j;
  }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (KIND == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[j]));
      if (KIND == 1) b[j] = ffma2(b[j], make_float2(0.999f, 0.999f), make_float2(-0.001f, -0.001f));
      if (KIND == 2) b[j] = fadd2(b[j], make_float2(-0.001f, 0.001f));
      if (KIND == 3) {
        unsigned r;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[j]), "f"(__uint_as_float(u[j])));
        u[j] ^= r;
      }
      if (KIND == 4) asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(a[j]) : "f"(b[j].x), "f"(b[j].y));
      if (KIND == 5) asm volatile("fma.rn.f32 %0, %0, 0f3F7FBE77, 0fBA83126F;" : "+f"(a[j]));
      if (KIND == 6) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(u[j]));
      if (KIND == 7) asm volatile("mad.lo.u32 %0, %0, 3, 7;" : "+r"(u[j]));
      if (KIND >= 8) {
        const int k1 = KIND / 10 - 1, k2 = KIND % 10;  // pairs: 1 instr of each kind
        auto one = [&](int k) {
          if (k == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[j]));
          if (k == 1) b[j] = ffma2(b[j], make_float2(0.999f, 0.999f), make_float2(-0.001f, -0.001f));
          if (k == 3) {
            unsigned r;
            asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b[j].x), "f"(__uint_as_float(u[j])));
            u[j] ^= r;
          }
          if (k == 4) asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(b[j].y) : "f"(b[j].x), "f"(a[j]));
          if (k == 7) asm volatile("mad.lo.u32 %0, %0, 3, 7;" : "+r"(u[j]));
        };
        one(k1);
        one(k2);
      }
    }
  }
  long long t1 = clock64();
  float s = 0;
  for (int j = 0; j < 8; ++j) s += a[j] + b[j].x + b[j].y + __uint_as_float(u[j]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

int main() {
  const char* names[] = {"MUFU.EX2 f32", "FFMA2", "FADD2", "F2FP.BF16 pack", "FMNMX3", "FFMA", "MUFU.EX2 bf16x2", "IMAD"};
  const int pairs[] = {13, 11, 14, 43, 41, 44, 23, 24, 48, 47, 21, 27, 22};
  const char* pnames[] = {"MUFU+F2FP", "MUFU+FFMA2", "MUFU+FMNMX3", "F2FP+F2FP(2x)", "F2FP+FFMA2", "F2FP+FMNMX3",
                          "FFMA2+F2FP", "FFMA2+FMNMX3", "F2FP+IMAD", "F2FP+IMAD?", "FFMA2+FFMA2(2x)", "FFMA2+IMAD", "FFMA2+FADD2?"};
  float* out;
  long long* clk;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&clk, 148 * 8);
  const int n = 4096;
  for (int kind = 0; kind < 8; ++kind) {
    for (int w : {1, 2, 4}) {
      int threads = 128 * w;
      void (*fn)(float*, long long*, int);
      switch (kind) {
        case 0: fn = bench<0>; break; case 1: fn = bench<1>; break; case 2: fn = bench<2>; break;
        case 3: fn = bench<3>; break; case 4: fn = bench<4>; break; case 5: fn = bench<5>; break;
        case 6: fn = bench<6>; break; default: fn = bench<7>; break;
      }
      fn<<<148, threads>>>(out, clk, 16);
      fn<<<148, threads>>>(out, clk, n);
      cudaDeviceSynchronize();
      long long c;
      cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
      // per SMSP: w warps x n x 8 instructions
      printf("%-18s warps/SMSP=%d  clk per warp-instr per SMSP = %.2f\n", names[kind], w,
             (double)c / (double(w) * n * 8));
    }
  }
  for (int pi = 0; pi < 13; ++pi) {
    void (*fn)(float*, long long*, int) = nullptr;
    switch (pairs[pi]) {
      case 13: fn = bench<13>; break; case 11: fn = bench<11>; break; case 14: fn = bench<14>; break;
      case 43: fn = bench<43>; break; case 41: fn = bench<41>; break; case 44: fn = bench<44>; break;
      case 23: fn = bench<23>; break; case 24: fn = bench<24>; break; case 48: fn = bench<48>; break;
      case 47: fn = bench<47>; break; case 21: fn = bench<21>; break; case 27: fn = bench<27>; break;
      default: fn = bench<22>; break;
    }
    fn<<<148, 256>>>(out, clk, 16);
    fn<<<148, 256>>>(out, clk, n);
    cudaDeviceSynchronize();
    long long c;
    cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
    printf("%-18s (kinds %d) warps/SMSP=2  clk per PAIR per SMSP = %.2f\n", pnames[pi], pairs[pi], (double)c / (2.0 * n * 8));
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
