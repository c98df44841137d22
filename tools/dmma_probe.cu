// FP64 throughput probe on sm_100a: DFMA vs mma.sync f64 (m8n8k4, m16n8k4,
// m16n8k8, m16n8k16). Prints TFLOP/s per variant.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_k(double* out, int iters) {
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + 1e-9 * (threadIdx.x + i);
  for (int k = 0; k < iters; ++k)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], 0.999999999, 1e-12);
  double s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 1234.5) out[0] = s;
}

__global__ void m884_k(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.5;
  double c[8][2];
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  for (int k = 0; k < iters; ++k) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 1234.5) out[0] = s;
}

__global__ void m1684_k(double* out, int iters) {
  double a0 = 1.0 + threadIdx.x * 1e-9, a1 = 0.7, b = 0.5;
  double c[8][4];
  for (int i = 0; i < 8; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0.0;
  for (int k = 0; k < iters; ++k) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) for (int j = 0; j < 4; ++j) s += c[i][j];
  if (s == 1234.5) out[0] = s;
}

__global__ void m16816_k(double* out, int iters) {
  double a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + threadIdx.x * 1e-9 + i;
  for (int i = 0; i < 4; ++i) b[i] = 0.5 + i;
  double c[4][4];
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0.0;
  for (int k = 0; k < iters; ++k) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) s += c[i][j];
  if (s == 1234.5) out[0] = s;
}

template <class F>
double run(F k, double flops_per_thread_iter, int blocks, int threads, int iters) {
  double* out;
  cudaMalloc(&out, 8);
  k<<<blocks, threads>>>(out, 16);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int r = 0; r < 3; ++r) k<<<blocks, threads>>>(out, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaFree(out);
  return 3.0 * flops_per_thread_iter * iters * (double)blocks * threads / (ms * 1e-3) / 1e12;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int it = 2000;
  for (int wpsm : {4, 8, 16, 32}) {
    const int blocks = sms * wpsm / 4, threads = 128;
    printf("warps/SM %2d: DFMA %.1f TF  m8n8k4 %.1f TF  m16n8k4 %.1f TF  m16n8k16 %.1f TF\n", wpsm,
           run(dfma_k, 8 * 2.0, blocks, threads, it),
           run(m884_k, 8 * 2.0 * 256 / 32, blocks, threads, it),
           run(m1684_k, 8 * 2.0 * 512 / 32, blocks, threads, it),
           run(m16816_k, 4 * 2.0 * 2048 / 32, blocks, threads, it));
  }
  cudaError_t e = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
