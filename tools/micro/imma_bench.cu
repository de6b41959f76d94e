// Microbenchmark: warp-level IMMA (mma.sync m16n8k32 u8, s32 accumulate) throughput on sm_100a.
#include <cstdio>
#include <cstdint>
__global__ void k_imma(const uint32_t* in, int* out, int iters) {
  uint32_t a0 = in[threadIdx.x], a1 = in[threadIdx.x + 1], a2 = in[threadIdx.x + 2], a3 = in[threadIdx.x + 3];
  uint32_t b0 = in[threadIdx.x + 4], b1 = in[threadIdx.x + 5];
  int c[8][4] = {};
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int k = 0; k < 8; k++)
      asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+r"(c[k][0]), "+r"(c[k][1]), "+r"(c[k][2]), "+r"(c[k][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0 + k), "r"(b1));
  }
  int s = 0;
  for (int k = 0; k < 8; k++) s += c[k][0] + c[k][1] + c[k][2] + c[k][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  uint32_t* in; int* out;
  cudaMalloc(&in, 4096); cudaMalloc(&out, 148 * 8 * 1024 * 4);
  cudaMemset(in, 0x01, 4096);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4000, blocks = 148 * 4, threads = 256;
  k_imma<<<blocks, threads>>>(in, out, 10);
  cudaEventRecord(e0);
  k_imma<<<blocks, threads>>>(in, out, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double macs = (double)blocks * (threads / 32) * iters * 8 * (16.0 * 8 * 32);
  printf("mma.sync m16n8k32 u8: %.3f ms  %.1f TMAC/s = %.1f TOPS  (%.0f MAC/clk/SM at 1.965 GHz)  err=%s\n", ms,
         macs / ms / 1e9, 2 * macs / ms / 1e9, macs / (ms * 1e-3) / 148 / 1.965e9, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
