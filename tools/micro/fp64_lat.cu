// fp64 latency / throughput probe: dependent DADD / DMUL chains and the
// orientation-style loop (LDS + I2D + DMUL + DADD chain), clock64 per warp.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chain(double* out, long long* cyc, double a, int n, int mode)
{
  double x = a + threadIdx.x, y = a * 0.5;
  long long t0 = clock64();
  if (mode == 0) { for (int i = 0; i < n; i++) x = x + y; }
  else if (mode == 1) { for (int i = 0; i < n; i++) x = x * y; }
  else { for (int i = 0; i < n; i++) x = fma(x, y, y); }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void chain2(double* out, long long* cyc, double a, int n)
{
  // two interleaved chains (gx, gy)
  double x = a + threadIdx.x, z = a - threadIdx.x, y = a * 0.5;
  long long t0 = clock64();
  for (int i = 0; i < n; i++) { x = x + y; z = z + y; }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = x + z;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main()
{
  double* d; long long* c;
  cudaMalloc(&d, 1 << 24); cudaMalloc(&c, 1 << 20);
  long long h[1024];
  const int n = 4096;
  const char* names[3] = {"DADD", "DMUL", "DFMA"};
  for (int m = 0; m < 3; m++) {
    chain<<<1, 32>>>(d, c, 1.0000001, n, m);
    cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
    printf("%s dependent latency: %.2f cycles\n", names[m], (double)h[0] / n);
  }
  chain2<<<1, 32>>>(d, c, 1.0000001, n);
  cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
  printf("2 interleaved DADD chains: %.2f cycles per iteration\n", (double)h[0] / n);
  // throughput: many warps per SM, DADD chains
  for (int w : {4, 8, 16, 32}) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    chain<<<148, 32 * w>>>(d, c, 1.0000001, n, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
    printf("%2d warps/SM: %.2f cycles per dependent DADD per warp, %.3f ms, %.1f GDADD/s\n", w, (double)h[0] / n, ms,
           148.0 * 32 * w * n / (ms * 1e6));
  }
  return 0;
}
