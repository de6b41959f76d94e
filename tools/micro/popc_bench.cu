// Microbenchmark: POPC / LOP3 throughput and b1 mma.sync (xor.popc) on sm_100a.
#include <cstdio>
#include <cstdint>
__global__ void k_popc(const uint32_t* in, uint32_t* out, int iters) {
  uint32_t a = in[threadIdx.x], b = in[threadIdx.x + 1], c = a ^ 0x55, d = b ^ 0x33;
  uint32_t s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int k = 0; k < 16; k++) {
      s0 += __popc(a ^ (b + k)); s1 += __popc(c ^ (d + k)); s2 += __popc(a ^ (d + k)); s3 += __popc(c ^ (b + k));
    }
    a += s0; c += s1;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s0 + s1 + s2 + s3;
}
__global__ void k_mma_b1(const uint32_t* in, int* out, int iters) {
  uint32_t a0 = in[threadIdx.x], a1 = in[threadIdx.x + 1], a2 = in[threadIdx.x + 2], a3 = in[threadIdx.x + 3];
  uint32_t b0 = in[threadIdx.x + 4], b1 = in[threadIdx.x + 5];
  int c0 = 0, c1 = 0, c2 = 0, c3 = 0, e0 = 0, e1 = 0, e2 = 0, e3 = 0;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int k = 0; k < 8; k++) {
      asm volatile("mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.xor.popc {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+r"(c0), "+r"(c1), "+r"(c2), "+r"(c3) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
      asm volatile("mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.xor.popc {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+r"(e0), "+r"(e1), "+r"(e2), "+r"(e3) : "r"(a1), "r"(a2), "r"(a3), "r"(a0), "r"(b1), "r"(b0));
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = c0 + c1 + c2 + c3 + e0 + e1 + e2 + e3;
}
int main() {
  uint32_t* in; uint32_t* out;
  cudaMalloc(&in, 4096); cudaMalloc(&out, 148 * 8 * 1024 * 4);
  cudaMemset(in, 0x5a, 4096);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 2000, blocks = 148 * 8, threads = 256;
  k_popc<<<blocks, threads>>>(in, out, 10);
  cudaEventRecord(e0);
  k_popc<<<blocks, threads>>>(in, out, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double pops = (double)blocks * threads * iters * 64;
  printf("popc: %.3f ms  %.1f Gpopc/s  %.2f popc/clk/SM (at 1.965 GHz)\n", ms, pops / ms / 1e6, pops / (ms * 1e-3) / 148 / 1.965e9);
  k_mma_b1<<<blocks, threads>>>(in, (int*)out, 10);
  cudaEventRecord(e0);
  k_mma_b1<<<blocks, threads>>>(in, (int*)out, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  double bops = (double)blocks * (threads / 32) * iters * 16 * (16.0 * 8 * 256);
  printf("mma b1 xor.popc: %.3f ms  %.1f Tbitop/s (16x8x256 per mma)  err=%s\n", ms, bops / ms / 1e9,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
