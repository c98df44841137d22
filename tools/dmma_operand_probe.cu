// DMMA.8x8x4 throughput on sm_100a vs operand pattern (12 warps/SM, like the
// contraction's consumers): same A/B registers every instruction, distinct
// A/B registers per instruction, distinct + one DADD per 2 DMMAs, and the
// contraction's 3M pattern (A shared by pairs, B distinct).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_operand_probe dmma_operand_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int MODE>
__global__ void k(double* out, int iters) {
  double a[8], b[8], c[6][2];
  for (int i = 0; i < 8; ++i) { a[i] = 1.0 + 1e-9 * (threadIdx.x + i); b[i] = 0.5 + 1e-9 * i; }
  for (int i = 0; i < 6; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      if (MODE == 0) {
#pragma unroll
        for (int i = 0; i < 6; ++i) dmma(c[i][0], c[i][1], a[0], b[0]);
      } else if (MODE == 1) {
#pragma unroll
        for (int i = 0; i < 6; ++i) dmma(c[i][0], c[i][1], a[(s + i) & 7], b[(s * 3 + i) & 7]);
      } else if (MODE == 2) {
        double sa = a[s] + a[s + 1];
        double sb0 = b[s] + b[s + 2], sb1 = b[s + 1] + b[s + 3];
        dmma(c[0][0], c[0][1], a[s], b[s]);
        dmma(c[1][0], c[1][1], a[s], b[s + 1]);
        dmma(c[2][0], c[2][1], a[s + 1], b[s + 2]);
        dmma(c[3][0], c[3][1], a[s + 1], b[s + 3]);
        dmma(c[4][0], c[4][1], sa, sb0);
        dmma(c[5][0], c[5][1], sa, sb1);
        a[s] += 1e-30; b[s] += 1e-30;  // keep the sums live per iteration
      } else if (MODE == 3) {  // 3M pattern without sums: A shared by pairs
        dmma(c[0][0], c[0][1], a[s], b[s]);
        dmma(c[1][0], c[1][1], a[s], b[s + 1]);
        dmma(c[2][0], c[2][1], a[s + 1], b[s + 2]);
        dmma(c[3][0], c[3][1], a[s + 1], b[s + 3]);
        dmma(c[4][0], c[4][1], a[s + 2], b[s + 4]);
        dmma(c[5][0], c[5][1], a[s + 2], b[s + 1]);
      } else if (MODE == 4) {  // 4M pattern: every operand used twice
        dmma(c[0][0], c[0][1], a[s], b[s]);
        dmma(c[1][0], c[1][1], a[s + 1], b[s + 1]);
        dmma(c[2][0], c[2][1], a[s], b[s + 1]);
        dmma(c[3][0], c[3][1], a[s + 1], b[s]);
        dmma(c[4][0], c[4][1], a[s], b[s + 2]);
        dmma(c[5][0], c[5][1], a[s + 1], b[s + 3]);
      }
    }
  }
  double t = 0;
  for (int i = 0; i < 6; ++i) t += c[i][0] + c[i][1];
  if (t == 1234.5) out[0] = t;
}

template <class F>
void run(const char* name, F kern, int warps) {
  double* out;
  cudaMalloc(&out, 8);
  const int iters = 4000, blocks = 148;
  kern<<<blocks, warps * 32>>>(out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<<<blocks, warps * 32>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 512.0 * 24 * iters * blocks * warps;  // 24 DMMA per iteration per warp
  printf("%-28s warps/SM %2d  %6.2f TF/s\n", name, warps, flops / (ms * 1e-3) / 1e12);
  cudaFree(out);
}

int main() {
  for (int w : {4, 8, 12, 16}) {
    run("same A/B", k<0>, w);
    run("distinct A/B", k<1>, w);
    run("3M with DADD sums", k<2>, w);
    run("3M pattern, no sums", k<3>, w);
    run("4M pattern", k<4>, w);
  }
  return 0;
}
