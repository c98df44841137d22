// Do DFMA (FP64 pipe) and DMMA (tensor pipe) issue concurrently on sm_100a?
// Kernels: DMMA only, DFMA only, and both interleaved in each warp; prints
// TFLOP/s of each part. nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

template <int NMMA, int NFMA>
__global__ void mix_k(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.5;
  double c[NMMA > 0 ? NMMA : 1][2];
  double f[NFMA > 0 ? NFMA : 1];
  for (int i = 0; i < (NMMA > 0 ? NMMA : 1); ++i) c[i][0] = c[i][1] = 0.0;
  for (int i = 0; i < (NFMA > 0 ? NFMA : 1); ++i) f[i] = 1.0 + 1e-9 * (threadIdx.x + i);
  for (int k = 0; k < iters; ++k) {
#pragma unroll
    for (int i = 0; i < NMMA; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
#pragma unroll
    for (int i = 0; i < NFMA; ++i) f[i] = fma(f[i], 0.999999999, 1e-12);
  }
  double s = 0;
  for (int i = 0; i < NMMA; ++i) s += c[i][0] + c[i][1];
  for (int i = 0; i < NFMA; ++i) s += f[i];
  if (s == 1234.5) out[0] = s;
}

template <int NMMA, int NFMA>
void run(const char* name, int blocks, int threads, int iters) {
  double* out;
  cudaMalloc(&out, 8);
  mix_k<NMMA, NFMA><<<blocks, threads>>>(out, 16);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  mix_k<NMMA, NFMA><<<blocks, threads>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double warps = double(blocks) * threads / 32;
  const double mma_fl = warps * iters * NMMA * 512.0, fma_fl = double(blocks) * threads * iters * NFMA * 2.0;
  printf("%-34s %8.3f ms  DMMA %6.2f TF  DFMA %6.2f TF  sum %6.2f TF\n", name, ms, mma_fl / ms / 1e9,
         fma_fl / ms / 1e9, (mma_fl + fma_fl) / ms / 1e9);
  cudaFree(out);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int it = 20000;
  for (int wps : {4, 8, 16, 32}) {
    printf("-- %d warps/SM\n", wps);
    run<8, 0>("dmma x8", sms, 32 * wps, it);
    run<0, 8>("dfma x8", sms, 32 * wps, it * 8);
    run<8, 8>("dmma x8 + dfma x8", sms, 32 * wps, it);
    run<8, 16>("dmma x8 + dfma x16", sms, 32 * wps, it);
    run<8, 32>("dmma x8 + dfma x32", sms, 32 * wps, it);
  }
  return 0;
}
