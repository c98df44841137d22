// DMMA.8x8x4 dependent-chain latency and chains needed for peak (1 SM).
#include <cstdio>
#include <cuda_runtime.h>
template <int C>
__global__ void k(double* out, int iters, long long* cyc) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.5;
  double c[C][2];
  for (int i = 0; i < C; ++i) c[i][0] = c[i][1] = 0.0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < C; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < C; ++i) s += c[i][0] + c[i][1];
  if (s == 1234.5) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int C>
void run(int warps) {
  double* o; long long* cyc;
  cudaMalloc(&o, 8); cudaMalloc(&cyc, 8);
  const int iters = 2000;
  k<C><<<1, 32 * warps>>>(o, iters, cyc);
  k<C><<<1, 32 * warps>>>(o, iters, cyc);
  long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("chains/warp %2d warps/SM %d: %.1f clk per DMMA per warp, %.2f clk per DMMA per SM\n", C, warps,
         (double)h / (iters * C), (double)h / (iters * C * warps));
}
int main() {
  run<1>(1); run<2>(1); run<4>(1); run<8>(1); run<16>(1);
  run<1>(4); run<4>(4); run<8>(4); run<9>(4); run<12>(4); run<16>(4);
  run<4>(8); run<8>(8);
  return 0;
}
