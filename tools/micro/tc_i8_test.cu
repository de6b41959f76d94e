// tc_i8_test.cu -- standalone check of a tcgen05 kind::i8 Hamming tile kernel
// (bits expanded to 0/1 bytes, d = |q| + |r| - 2 q.r) against a CPU popcount.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tc_i8_test.cu -o tc_i8_test
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

constexpr int TM = 128, TN = 256, KB = 512;   // tile rows (query), tile cols (reference), bits
constexpr int A_BYTES = TM * KB, B_BYTES = TN * KB;  // expanded 0/1 bytes

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// K-major SWIZZLE_128B operand: K block kb (128 bytes of K) is a [rows][128 B]
// region; 16-byte chunk c of row r sits at chunk c ^ (r & 7).
__device__ __forceinline__ uint32_t sw_off(int rows, int r, int kbyte)
{
  const int kb = kbyte >> 7, c = (kbyte >> 4) & 7;
  return (uint32_t)(kb * rows * 128 + r * 128 + ((c ^ (r & 7)) << 4) + (kbyte & 15));
}

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr)
{
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3fff);        // start address
  d |= (uint64_t)1 << 16;                        // LBO = 1 (16 B units; unused for SW128 K-major)
  d |= (uint64_t)(1024 >> 4) << 32;              // SBO = 1024 B between 8-row groups
  d |= (uint64_t)1 << 46;                        // version = 1 (sm100)
  d |= (uint64_t)2 << 61;                        // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ uint32_t idesc_i8(int M, int N)
{
  uint32_t d = 0;
  d |= 2u << 4;                 // C = S32
  d |= 0u << 7;                 // A = unsigned 8-bit
  d |= 0u << 10;                // B = unsigned 8-bit
  d |= (uint32_t)(N >> 3) << 17;
  d |= (uint32_t)(M >> 4) << 24;
  return d;
}

__device__ __forceinline__ void expand_word(uint8_t* base, int rows, int r, int w, uint32_t v)
{
  // 32 bits of word w -> bytes 32w .. 32w + 31 (bit j of the word -> byte 32w + j)
  uint32_t o[8];
#pragma unroll
  for (int q = 0; q < 8; q++) o[q] = (((v >> (4 * q)) & 15u) * 0x00204081u) & 0x01010101u;
  *reinterpret_cast<uint4*>(base + sw_off(rows, r, 32 * w)) = make_uint4(o[0], o[1], o[2], o[3]);
  *reinterpret_cast<uint4*>(base + sw_off(rows, r, 32 * w + 16)) = make_uint4(o[4], o[5], o[6], o[7]);
}

__global__ void __launch_bounds__(256, 1) k_tc(const uint32_t* q, int nq, const uint32_t* rr, int nr, int32_t* out,
                                               int* err, int mode)
{
  extern __shared__ __align__(1024) uint8_t dsm[];
  uint8_t* sA = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsm) + 1023) & ~(uintptr_t)1023);
  uint8_t* sB = sA + A_BYTES;
  __shared__ uint64_t mbar;
  __shared__ uint32_t tslot;
  __shared__ int pq[TM], pr[TN];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int i0 = blockIdx.y * TM, j0 = blockIdx.x * TN;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  // expand: 16 words per row
  for (int i = tid; i < TM * 16; i += 256) {
    const int r = i >> 4, w = i & 15;
    const uint32_t v = i0 + r < nq ? q[(long long)(i0 + r) * 16 + w] : 0u;
    expand_word(sA, TM, r, w, v);
  }
  for (int i = tid; i < TN * 16; i += 256) {
    const int r = i >> 4, w = i & 15;
    const uint32_t v = j0 + r < nr ? rr[(long long)(j0 + r) * 16 + w] : 0u;
    expand_word(sB, TN, r, w, v);
  }
  if (tid < TM) {
    int c = 0;
    for (int w = 0; w < 16; w++) c += i0 + tid < nq ? __popc(q[(long long)(i0 + tid) * 16 + w]) : 0;
    pq[tid] = c;
  }
  {
    int c = 0;
    for (int w = 0; w < 16; w++) c += j0 + tid < nr ? __popc(rr[(long long)(j0 + tid) * 16 + w]) : 0;
    pr[tid] = c;
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (mode == 2) {   // expansion only
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tslot), "r"(256));
    return;
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  if (tid == 0) {
    const uint32_t id = idesc_i8(TM, TN);
#pragma unroll 1
    for (int k = 0; k < KB / 32; k++) {
      const int kb = k >> 2, sub = k & 3;
      const uint64_t da = sdesc(smem_u32(sA + kb * TM * 128 + sub * 32));
      const uint64_t db = sdesc(smem_u32(sB + kb * TN * 128 + sub * 32));
      const uint32_t acc = k > 0;
      asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                   " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
                   "l"(da), "l"(db), "r"(id), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar)));
  }
  // wait (bounded)
  {
    uint32_t done = 0;
    long long spins = 0;
    while (!done) {
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                   : "=r"(done) : "r"(smem_u32(&mbar)), "r"(0));
      if (++spins > (1ll << 26)) { if (lane == 0) atomicAdd(err, 1); break; }
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  // epilogue: warp w reads TMEM lanes 32 (w % 4) .., columns 128 (w / 4) .. + 127
  const int row = 32 * (warp & 3) + lane, cb = 128 * (warp >> 2);
#pragma unroll 1
  for (int c0 = 0; c0 < 128; c0 += 32) {
    uint32_t v[32];
    const uint32_t ta = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(cb + c0);
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                 "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                   "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
                   "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
                   "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                 : "r"(ta));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    if (mode == 1) {   // count only (no matrix store)
      int c = 0;
#pragma unroll
      for (int j = 0; j < 32; j++) c += pq[row] + pr[cb + c0 + j] - 2 * (int)v[j] <= 102;
      if (c == 12345) atomicAdd(err, 0);
      continue;
    }
    if (i0 + row < nq)
#pragma unroll
      for (int j = 0; j < 32; j++) {
        const int col = cb + c0 + j;
        if (j0 + col < nr) out[(long long)(i0 + row) * nr + j0 + col] = pq[row] + pr[col] - 2 * (int)v[j];
      }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

int main(int argc, char** argv)
{
  const int nq = argc > 1 ? atoi(argv[1]) : 300, nr = argc > 2 ? atoi(argv[2]) : 517;
  std::vector<uint32_t> q((size_t)nq * 16), r((size_t)nr * 16);
  uint64_t s = 88172645463325252ull;
  auto rnd = [&]() { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return (uint32_t)s; };
  for (auto& x : q) x = rnd();
  for (auto& x : r) x = rnd();
  for (int w = 0; w < 16; w++) r[w] = q[w];   // one exact duplicate: distance 0
  uint32_t *dq, *dr;
  int32_t* dout;
  int* derr;
  CK(cudaMalloc(&dq, q.size() * 4));
  CK(cudaMalloc(&dr, r.size() * 4));
  CK(cudaMalloc(&dout, (size_t)nq * nr * 4));
  CK(cudaMalloc(&derr, 4));
  CK(cudaMemset(derr, 0, 4));
  CK(cudaMemcpy(dq, q.data(), q.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dr, r.data(), r.size() * 4, cudaMemcpyHostToDevice));
  const int smem = A_BYTES + B_BYTES + 1024;
  CK(cudaFuncSetAttribute(k_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  dim3 grid((nr + TN - 1) / TN, (nq + TM - 1) / TM);
  k_tc<<<grid, 256, smem>>>(dq, nq, dr, nr, dout, derr, 0);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  int herr = 0;
  CK(cudaMemcpy(&herr, derr, 4, cudaMemcpyDeviceToHost));
  std::vector<int32_t> out((size_t)nq * nr);
  CK(cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost));
  long long bad = 0;
  for (int i = 0; i < nq; i++)
    for (int j = 0; j < nr; j++) {
      int d = 0;
      for (int w = 0; w < 16; w++) d += __builtin_popcount(q[(size_t)i * 16 + w] ^ r[(size_t)j * 16 + w]);
      if (d != out[(size_t)i * nr + j]) {
        if (bad < 5) printf("mismatch %d %d: %d vs %d\n", i, j, out[(size_t)i * nr + j], d);
        bad++;
      }
    }
  printf("nq %d nr %d timeouts %d mismatches %lld  d(0,0)=%d\n", nq, nr, herr, bad, out[0]);
  // timing on a frame-sized problem
  if (argc > 3) {
    const int N = atoi(argv[3]);
    uint32_t *bq;
    int32_t* bo;
    CK(cudaMalloc(&bq, (size_t)N * 64));
    CK(cudaMemset(bq, 0x5a, (size_t)N * 64));
    CK(cudaMalloc(&bo, (size_t)N * N * 4));
    dim3 g2((N + TN - 1) / TN, (N + TM - 1) / TM);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int mode = 0; mode < 3; mode++) {
      k_tc<<<g2, 256, smem>>>(bq, N, bq, N, bo, derr, mode);
      cudaEventRecord(e0);
      for (int it = 0; it < 5; it++) k_tc<<<g2, 256, smem>>>(bq, N, bq, N, bo, derr, mode);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("mode %d (0 store, 1 count, 2 expand only) N %d: %.3f ms, %.1f G pairs/s\n", mode, N, ms / 5,
             (double)N * N / (ms / 5 * 1e-3) / 1e9);
    }
  }
  return bad != 0 || herr != 0;
}
