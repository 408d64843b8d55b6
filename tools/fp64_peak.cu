// FP64 throughput microbenchmark for B200 (sm_100a): DFMA vs mma.sync .f64 shapes.
// Measures the FP64 roofline denominator that MEASURED_PEAKS.json lacks.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA error %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void dfma_kernel(double* out, int iters, double s) {
  double a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = fma(a[i], s, 1e-9);
    }
  }
  double t = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) t += a[i];
  if (t == 12345.678) out[0] = t;
}

__global__ void dmma_m8n8k4(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double t = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) t += c[i][0] + c[i][1];
  if (t == 12345.678) out[0] = t;
}

__global__ void dmma_m16n8k4(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b = 1.0 - threadIdx.x * 1e-4;
  double c[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 2; ++r) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b));
    }
  }
  double t = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) t += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (t == 12345.678) out[0] = t;
}

__global__ void dmma_m16n8k16(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - threadIdx.x * 1e-4 + i;
  double c[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double t = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) t += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (t == 12345.678) out[0] = t;
}

template <typename F>
static double time_it(F launch, int reps) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  launch();
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  for (int i = 0; i < reps; ++i) launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms / reps;
}

int main() {
  double* out; CK(cudaMalloc(&out, 8));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"sms\": %d, \"clock_khz\": %d", sms, clk);
  const int iters = 2000;
  for (int bpsm = 4; bpsm <= 8; bpsm *= 2) {
    int blocks = sms * bpsm, threads = 256;
    double ms = time_it([&] { dfma_kernel<<<blocks, threads>>>(out, iters, 0.999999); }, 5);
    double flops = 2.0 * blocks * threads * (double)iters * 16 * 8;
    printf(", \"dfma_bpsm%d_tflops\": %.3f", bpsm, flops / ms / 1e9);
    ms = time_it([&] { dmma_m8n8k4<<<blocks, threads>>>(out, iters); }, 5);
    flops = 2.0 * (blocks * threads / 32) * (double)iters * 16 * (8 * 8 * 4);
    printf(", \"dmma_m8n8k4_bpsm%d_tflops\": %.3f", bpsm, flops / ms / 1e9);
    ms = time_it([&] { dmma_m16n8k4<<<blocks, threads>>>(out, iters); }, 5);
    flops = 2.0 * (blocks * threads / 32) * (double)iters * 8 * (16 * 8 * 4);
    printf(", \"dmma_m16n8k4_bpsm%d_tflops\": %.3f", bpsm, flops / ms / 1e9);
    ms = time_it([&] { dmma_m16n8k16<<<blocks, threads>>>(out, iters); }, 5);
    flops = 2.0 * (blocks * threads / 32) * (double)iters * 4 * (16 * 8 * 16);
    printf(", \"dmma_m16n8k16_bpsm%d_tflops\": %.3f", bpsm, flops / ms / 1e9);
  }
  CK(cudaGetLastError());
  printf("}\n");
  return 0;
}
