// tc_i8_peak.cu -- tcgen05.mma.kind::i8 issue-rate microbenchmark: one CTA per
// SM, one thread issuing back-to-back M x N x 32 MMAs from shared memory into
// TMEM (no loads), for N = 64 / 128 / 256.  Prints MAC/clk/SM and POPS.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tc_i8_peak.cu -o tc_i8_peak
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t a)
{
  return (uint64_t)((a >> 4) & 0x3fff) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) |
         ((uint64_t)2 << 61);
}

__device__ volatile int g_stop;
template <int N, bool WALK, int LDMODE>
__global__ void __launch_bounds__(128, 1) k_peak(int iters, unsigned long long* clk)
{
  extern __shared__ uint8_t dsm[];
  uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsm) + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t mb;
  __shared__ uint32_t slot;
  __shared__ volatile int stop;
  __shared__ __align__(16) uint8_t spare[96 * 16 * 16];
  if (threadIdx.x == 0) stop = 0;
  const int bytes = WALK ? (128 + N) * 512 : (128 + N) * 128;
  for (int i = threadIdx.x; i < bytes / 4; i += 128) reinterpret_cast<uint32_t*>(s)[i] = 0x01010101u;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(LDMODE ? 2 * N : (N < 32 ? 32 : N)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mb)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  const uint32_t idesc = (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  if (threadIdx.x == 0) {
    const uint64_t da = sdesc(smem_u32(s)), db = sdesc(smem_u32(s + (WALK ? 128 * 512 : 128 * 128)));
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
      asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(LDMODE == 3 ? tmem + (uint32_t)((i & 1) * N) : tmem),
                   "l"(WALK ? da + (uint64_t)((((i >> 2) & 3) * 128 * 128 + (i & 3) * 32) >> 4) + (LDMODE == 3 ? (uint64_t)(((i & 1) * 8192) >> 4) : 0ull) : da + 2 * (i & 3)),
                   "l"(WALK ? db + (uint64_t)((((i >> 2) & 3) * N * 128 + (i & 3) * 32) >> 4) : db + 2 * (i & 3)),
                   "r"(idesc), "r"(i));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mb)));
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}"
                   : "=r"(done) : "r"(smem_u32(&mb)));
    unsigned long long t1 = clock64();
    if (blockIdx.x == 0) *clk = t1 - t0;
    stop = 1;
  } else if ((LDMODE == 1 || LDMODE == 2) && threadIdx.x >= 32) {
    // warps 1..3: tcgen05.ld of the other accumulator (LDMODE 1) or shared
    // stores (LDMODE 2) until the MMAs finish
    const int w = threadIdx.x >> 5;
    uint32_t acc = 0;
    while (!stop) {
      if (LDMODE == 1) {
        uint32_t v[32];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                     "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                       "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                       "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
                       "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
                       "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                     : "r"(tmem + ((uint32_t)(32 * w) << 16) + N));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        for (int k = 0; k < 32; k++) acc += v[k];
      } else {
        uint4* p = reinterpret_cast<uint4*>(spare) + (threadIdx.x & 31) + 32 * (w - 1);
        for (int k = 0; k < 16; k++) p[96 * k] = make_uint4(acc, k, acc, k);
        acc++;
      }
    }
    if (acc == 0x12345) *clk = acc;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(LDMODE ? 2 * N : (N < 32 ? 32 : N)));
}

template <int N, bool WALK, int LDMODE = 0>
void run(int sms)
{
  const int iters = 200000, smem = (WALK ? (128 + N) * 512 : (128 + N) * 128) + 1024;
  cudaFuncSetAttribute(k_peak<N, WALK, LDMODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* clk;
  cudaMalloc(&clk, 8);
  k_peak<N, WALK, LDMODE><<<sms, 128, smem>>>(1000, clk);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k_peak<N, WALK, LDMODE><<<sms, 128, smem>>>(iters, clk);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  unsigned long long c = 0;
  cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
  const double macs = (double)iters * 128 * N * 32;
  printf("%s M=128 N=%3d K=32 i8: %.3f ms, %.1f MAC/clk/SM (clock64), %.0f TOPS over %d SMs (%s)\n",
         LDMODE == 3 ? "walk, 2 accumulators alternating" : LDMODE == 1 ? "walk + 3 warps tcgen05.ld" : (LDMODE == 2 ? "walk + 3 warps st.shared" : (WALK ? "walk 64KB images" : "same 4 slices  ")), N, ms, macs / c,
         2.0 * macs * sms / (ms * 1e-3) / 1e12, sms, cudaGetErrorString(cudaGetLastError()));
}

int main()
{
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<64, false>(sms);
  run<128, false>(sms);
  run<256, false>(sms);
  run<128, true>(sms);
  run<256, true>(sms);
  run<128, true, 1>(sms);
  run<128, true, 2>(sms);
  run<128, true, 3>(sms);
  return 0;
}
