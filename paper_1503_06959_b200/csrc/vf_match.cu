// vf_match.cu -- descriptor matching on packed binary descriptors
// (SURVEY.md 8(f) rank 1): hamming_matrix and radius_match of
// /root/reference/pkg/src/vidfeat/matching.py:47-94.
//
// Three paths, by row width: 512-bit rows run on the 5th-generation tensor
// cores (tcgen05.mma.kind::i8, TMEM accumulator; k_hamming_tc), other whole-
// word widths on mma.sync u8 (k_hamming_mma), anything else on POPC.
// All-pairs Hamming distance is compute-bound integer work: per pair,
// popcount(q XOR r) over the descriptor words.  CTA tile 128 queries x 128
// references, 256 threads, each thread 8 x 8 pairs in registers; the tile's
// descriptor words are staged word-major in shared memory so a thread reads
// its 8 query words and 8 reference words of one descriptor word with four
// 16-byte loads.  POPC (quarter-rate, 16 / clk / SM measured) bounds it:
// 16 POPC per pair for 512-bit descriptors.
//
// radius_match appends (q << 32 | r, d) for d <= t_m with warp-aggregated
// atomics, then one device radix sort on the 64-bit key gives np.nonzero's
// (query, reference) order.
#include <cstdint>
#include <cstdlib>
#include <cub/device/device_radix_sort.cuh>
#include "../../include/vidfeat_b200.h"

#define HM_T 128                 // queries / references per CTA tile
#define HM_THREADS 256
#define HM_MAXW 16               // descriptor words staged per pass (64 bytes = one 512-bit descriptor)

namespace {

// Stage rows [base, base + 128) x words [w0, w0 + nw) word-major into s[w][row]
// (bytes past nbytes and rows past n read as zero: XOR of zeros adds nothing).
__device__ __forceinline__ void stage_rows(const uint8_t* src, long long n, int nbytes, long long base, int w0, int nw,
                                           uint32_t* s)
{
  const bool aligned = ((reinterpret_cast<uintptr_t>(src) | (uintptr_t)nbytes) & 3) == 0;
  for (int i = threadIdx.x; i < HM_T * nw; i += HM_THREADS) {
    const int row = i / nw, w = i - row * nw;   // consecutive threads: consecutive words of a row
    const long long gr = base + row;
    uint32_t v = 0;
    if (gr < n) {
      const uint8_t* p = src + gr * nbytes;
      const int b0 = 4 * (w0 + w);
      if (aligned && b0 + 4 <= nbytes) {
        v = __ldg(reinterpret_cast<const uint32_t*>(p + b0));
      } else {
        for (int k = 0; k < 4; k++)
          if (b0 + k < nbytes) v |= (uint32_t)__ldg(p + b0 + k) << (8 * k);
      }
    }
    s[w * HM_T + row] = v;
  }
}

// acc[i][j] = distance between query ty * 8 + i and reference tx * 8 + j of the tile.
__device__ __forceinline__ void tile_distances(const uint8_t* q, long long nq, const uint8_t* r, long long nr,
                                               int nbytes, long long q0, long long r0, uint32_t* sq, uint32_t* sr,
                                               int acc[8][8])
{
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
#pragma unroll
  for (int i = 0; i < 8; i++)
#pragma unroll
    for (int j = 0; j < 8; j++) acc[i][j] = 0;
  const int nwords = (nbytes + 3) / 4;
  for (int w0 = 0; w0 < nwords; w0 += HM_MAXW) {
    const int nw = min(HM_MAXW, nwords - w0);
    __syncthreads();
    stage_rows(q, nq, nbytes, q0, w0, nw, sq);
    stage_rows(r, nr, nbytes, r0, w0, nw, sr);
    __syncthreads();
#pragma unroll 2
    for (int w = 0; w < nw; w++) {
      const uint4 qa = *reinterpret_cast<const uint4*>(sq + w * HM_T + 8 * ty);
      const uint4 qb = *reinterpret_cast<const uint4*>(sq + w * HM_T + 8 * ty + 4);
      const uint4 ra = *reinterpret_cast<const uint4*>(sr + w * HM_T + 8 * tx);
      const uint4 rb = *reinterpret_cast<const uint4*>(sr + w * HM_T + 8 * tx + 4);
      const uint32_t qv[8] = {qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w};
      const uint32_t rv[8] = {ra.x, ra.y, ra.z, ra.w, rb.x, rb.y, rb.z, rb.w};
#pragma unroll
      for (int i = 0; i < 8; i++)
#pragma unroll
        for (int j = 0; j < 8; j++) acc[i][j] += __popc(qv[i] ^ rv[j]);
    }
  }
}

__global__ void __launch_bounds__(HM_THREADS) k_hamming_matrix(const uint8_t* q, long long nq, const uint8_t* r,
                                                              long long nr, int nbytes, int32_t* out, long long ld)
{
  __shared__ __align__(16) uint32_t sq[HM_MAXW * HM_T];
  __shared__ __align__(16) uint32_t sr[HM_MAXW * HM_T];
  const long long q0 = (long long)blockIdx.y * HM_T, r0 = (long long)blockIdx.x * HM_T;
  int acc[8][8];
  tile_distances(q, nq, r, nr, nbytes, q0, r0, sq, sr, acc);
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const bool vec = (ld & 3) == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0;
#pragma unroll
  for (int i = 0; i < 8; i++) {
    const long long qi = q0 + 8 * ty + i;
    if (qi >= nq) break;
    const long long rj = r0 + 8 * tx;
    int32_t* o = out + qi * ld + rj;
    if (vec && rj + 8 <= nr) {
      reinterpret_cast<int4*>(o)[0] = make_int4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
      reinterpret_cast<int4*>(o)[1] = make_int4(acc[i][4], acc[i][5], acc[i][6], acc[i][7]);
    } else {
#pragma unroll
      for (int j = 0; j < 8; j++)
        if (rj + j < nr) o[j] = acc[i][j];
    }
  }
}

__global__ void __launch_bounds__(HM_THREADS) k_radius_match(const uint8_t* q, long long nq, const uint8_t* r,
                                                            long long nr, int nbytes, int t_m,
                                                            unsigned long long* keys, int32_t* dist, long long cap,
                                                            unsigned long long* count)
{
  __shared__ __align__(16) uint32_t sq[HM_MAXW * HM_T];
  __shared__ __align__(16) uint32_t sr[HM_MAXW * HM_T];
  const long long q0 = (long long)blockIdx.y * HM_T, r0 = (long long)blockIdx.x * HM_T;
  int acc[8][8];
  tile_distances(q, nq, r, nr, nbytes, q0, r0, sq, sr, acc);
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4, lane = threadIdx.x & 31;
#pragma unroll
  for (int i = 0; i < 8; i++)
#pragma unroll
    for (int j = 0; j < 8; j++) {
      const long long qi = q0 + 8 * ty + i, rj = r0 + 8 * tx + j;
      const bool hit = qi < nq && rj < nr && acc[i][j] <= t_m;
      const unsigned m = __ballot_sync(0xffffffffu, hit);
      if (!m) continue;
      unsigned long long pos = 0;
      if (lane == __ffs(m) - 1) pos = atomicAdd(count, (unsigned long long)__popc(m));
      pos = __shfl_sync(0xffffffffu, pos, __ffs(m) - 1) + __popc(m & ((1u << lane) - 1));
      if (hit && (long long)pos < cap) {
        keys[pos] = ((unsigned long long)qi << 32) | (unsigned long long)rj;
        dist[pos] = acc[i][j];
      }
    }
}

// ---------------------------------------------------------------------------
// Tensor-core path (rows of 4 * NW bytes, NW <= 16 words): the Hamming distance
// of 0/1 vectors is |q| + |r| - 2 q.r, and q.r is an integer GEMM over the
// bits.  Warp-level IMMA (mma.sync m16n8k32 u8 -> s32) with K = 32 bits = one
// descriptor word per k-step; A/B fragments are expanded from packed bits in
// registers (nibble * 0x00204081 & 0x01010101 puts bit j in byte j; A and B
// use the same bit -> k mapping, so the dot product is exact).  CTA tile 128 x
// 128, 8 warps of 32 x 64 (2 x 8 MMA tiles); rows padded to 17 words in shared
// memory so the 8 rows a fragment load touches sit in distinct banks.
// ---------------------------------------------------------------------------
#define MM_PAD 17

__device__ __forceinline__ uint32_t nib_bytes(uint32_t w, int sh)
{
  return (((w >> sh) & 0xfu) * 0x00204081u) & 0x01010101u;
}

template <bool RADIUS>
__global__ void __launch_bounds__(HM_THREADS) k_hamming_mma(const uint8_t* q, long long nq, const uint8_t* r,
                                                           long long nr, int nbytes, int32_t* out, long long ld,
                                                           int t_m, unsigned long long* keys, int32_t* dist,
                                                           long long cap, unsigned long long* count)
{
  __shared__ uint32_t sq[HM_T * MM_PAD], sr[HM_T * MM_PAD];
  __shared__ int pq[HM_T], prr[HM_T];
  const long long q0 = (long long)blockIdx.y * HM_T, r0 = (long long)blockIdx.x * HM_T;
  const int nw = nbytes >> 2;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int i = tid; i < HM_T * nw; i += HM_THREADS) {
    const int row = i / nw, w = i - row * nw;
    const long long gq = q0 + row, gr = r0 + row;
    sq[row * MM_PAD + w] = gq < nq ? __ldg(reinterpret_cast<const uint32_t*>(q + gq * nbytes) + w) : 0u;
    sr[row * MM_PAD + w] = gr < nr ? __ldg(reinterpret_cast<const uint32_t*>(r + gr * nbytes) + w) : 0u;
  }
  __syncthreads();
  if (tid < HM_T) {
    int a = 0, c = 0;
    for (int w = 0; w < nw; w++) { a += __popc(sq[tid * MM_PAD + w]); c += __popc(sr[tid * MM_PAD + w]); }
    pq[tid] = a;
    prr[tid] = c;
  }
  __syncthreads();
  const int wm = (wid & 3) * 32, wn = (wid >> 2) * 64;   // warp tile origin in the CTA tile
  const int gid = lane >> 2, tig = lane & 3;
  int acc[2][8][4];
#pragma unroll
  for (int i = 0; i < 2; i++)
#pragma unroll
    for (int j = 0; j < 8; j++)
#pragma unroll
      for (int k = 0; k < 4; k++) acc[i][j][k] = 0;
#pragma unroll 2
  for (int ks = 0; ks < nw; ks++) {
    uint32_t a[2][4], bb[8][2];
#pragma unroll
    for (int i = 0; i < 2; i++) {
      const uint32_t w0 = sq[(wm + 16 * i + gid) * MM_PAD + ks], w1 = sq[(wm + 16 * i + gid + 8) * MM_PAD + ks];
      a[i][0] = nib_bytes(w0, 4 * tig);          // row gid,     k = 4 tig .. 4 tig + 3
      a[i][1] = nib_bytes(w1, 4 * tig);          // row gid + 8
      a[i][2] = nib_bytes(w0, 4 * tig + 16);     // row gid,     k = 16 + 4 tig ..
      a[i][3] = nib_bytes(w1, 4 * tig + 16);     // row gid + 8
    }
#pragma unroll
    for (int j = 0; j < 8; j++) {
      const uint32_t w = sr[(wn + 8 * j + gid) * MM_PAD + ks];
      bb[j][0] = nib_bytes(w, 4 * tig);          // column gid, k = 4 tig ..
      bb[j][1] = nib_bytes(w, 4 * tig + 16);
    }
#pragma unroll
    for (int i = 0; i < 2; i++)
#pragma unroll
      for (int j = 0; j < 8; j++)
        asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                     "{%0,%1,%2,%3};"
                     : "+r"(acc[i][j][0]), "+r"(acc[i][j][1]), "+r"(acc[i][j][2]), "+r"(acc[i][j][3])
                     : "r"(a[i][0]), "r"(a[i][1]), "r"(a[i][2]), "r"(a[i][3]), "r"(bb[j][0]), "r"(bb[j][1]));
  }
  // epilogue: d = |q| + |r| - 2 q.r; C fragment: c0, c1 -> (row gid, cols 2 tig, 2 tig + 1), c2, c3 -> row gid + 8
  if (RADIUS) {
    // matches are sparse: skip the append loop unless some lane of the warp has one
    bool any = false;
#pragma unroll
    for (int i = 0; i < 2; i++)
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int lr = wm + 16 * i + gid + 8 * h;
        const int pa = pq[lr];
#pragma unroll
        for (int j = 0; j < 8; j++) {
          const int lc = wn + 8 * j + 2 * tig;
          any |= pa + prr[lc] - 2 * acc[i][j][2 * h] <= t_m;
          any |= pa + prr[lc + 1] - 2 * acc[i][j][2 * h + 1] <= t_m;
        }
      }
    if (!__any_sync(0xffffffffu, any)) return;
  }
#pragma unroll
  for (int i = 0; i < 2; i++)
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const int lr = wm + 16 * i + gid + 8 * h;
      const long long qi = q0 + lr;
      const int pa = pq[lr];
#pragma unroll
      for (int j = 0; j < 8; j++) {
        const int lc = wn + 8 * j + 2 * tig;
        const long long rj = r0 + lc;
        const int d0 = pa + prr[lc] - 2 * acc[i][j][2 * h], d1 = pa + prr[lc + 1] - 2 * acc[i][j][2 * h + 1];
        if (!RADIUS) {
          if (qi < nq) {
            int32_t* o = out + qi * ld + rj;
            if (rj + 1 < nr && ((reinterpret_cast<uintptr_t>(o) & 7) == 0)) {
              *reinterpret_cast<int2*>(o) = make_int2(d0, d1);
            } else {
              if (rj < nr) o[0] = d0;
              if (rj + 1 < nr) o[1] = d1;
            }
          }
        } else {
#pragma unroll
          for (int e = 0; e < 2; e++) {
            const int d = e ? d1 : d0;
            const bool hit = qi < nq && rj + e < nr && d <= t_m;
            const unsigned m = __ballot_sync(0xffffffffu, hit);
            if (!m) continue;
            unsigned long long pos = 0;
            if (lane == __ffs(m) - 1) pos = atomicAdd(count, (unsigned long long)__popc(m));
            pos = __shfl_sync(0xffffffffu, pos, __ffs(m) - 1) + __popc(m & ((1u << lane) - 1));
            if (hit && (long long)pos < cap) {
              keys[pos] = ((unsigned long long)qi << 32) | (unsigned long long)(rj + e);
              dist[pos] = d;
            }
          }
        }
      }
    }
}

// ---------------------------------------------------------------------------
// tcgen05 path (512-bit descriptors): the 5th-generation tensor cores with the
// accumulator in TMEM.  q.r of the 0/1 bits is a u8 x u8 -> s32 GEMM with
// K = 512: the packed rows are expanded to 0/1 bytes straight into shared
// memory in the canonical K-major SWIZZLE_128B layout (K block kb = bytes
// 128 kb .. of every row is a [rows][128 B] region, 16-byte chunk c of row r
// at c ^ (r & 7)), one elected thread issues 16 tcgen05.mma.kind::i8
// (M = 128, N = 256, K = 32 each) into a 128 x 256 s32 TMEM accumulator and
// commits to an mbarrier, and the epilogue reads it back with tcgen05.ld
// (warp w: TMEM lanes 32 (w % 4).., columns TC_COLS (w / 4)..), d = |q| + |r| -
// 2 q.r.  Persistent CTAs keep their 128-query tile A resident and walk a
// strided set of 256-reference tiles B.
// ---------------------------------------------------------------------------
#define TC_M 128
#define TC_N 256
#define TC_THREADS 512
#define TC_COLS (TC_N / (TC_THREADS / 128))   // accumulator columns per epilogue warp
#define TC_SMEM (TC_M * 512 + TC_N * 512 + 1024)

__device__ __forceinline__ uint32_t tc_smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// UMMA shared-memory descriptor, K-major SWIZZLE_128B: start >> 4, LBO 1,
// SBO 1024 B (8-row groups), version 1 (sm100), layout 2 (128B swizzle)
__device__ __forceinline__ uint64_t tc_sdesc(uint32_t saddr)
{
  return (uint64_t)((saddr >> 4) & 0x3fff) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) |
         ((uint64_t)2 << 61);
}

// instruction descriptor kind::i8: C = s32, A = B = unsigned 8-bit, both
// K-major, N >> 3, M >> 4
constexpr uint32_t TC_IDESC = (2u << 4) | ((uint32_t)(TC_N >> 3) << 17) | ((uint32_t)(TC_M >> 4) << 24);

// Packed rows [base, base + R) of a 64-byte-row matrix, one uint4 (16 bytes =
// one 128-byte K-block row once expanded) per (row, K block); thread t holds
// items t, t + TC_THREADS, ... (all loads in flight together).  Item i: lanes
// 8k .. 8k + 7 of a warp take 8 consecutive rows of K block k, so a warp
// reads 8 whole 64-byte rows and each quarter-warp's 16-byte smem stores
// land in 8 distinct swizzled chunk slots (no bank conflicts).
__device__ __forceinline__ void tc_item(int i, int& r, int& kb)
{
  r = (i & 7) + 8 * (i >> 5);
  kb = (i >> 3) & 3;
}

template <int R>
struct TcRows {
  uint4 v[R * 4 / TC_THREADS];
};

template <int R>
__device__ __forceinline__ void tc_load(const uint8_t* src, long long n, long long base, TcRows<R>& t)
{
#pragma unroll
  for (int u = 0; u < R * 4 / TC_THREADS; u++) {
    int r, kb;
    tc_item(threadIdx.x + u * TC_THREADS, r, kb);
    t.v[u] = base + r < n ? __ldg(reinterpret_cast<const uint4*>(src + (base + r) * 64) + kb) : make_uint4(0, 0, 0, 0);
  }
}

// expanded 0/1 bytes into `sm` (R rows, K-major SWIZZLE_128B) + per-row
// popcounts into `pc`
template <int R>
__device__ __forceinline__ void tc_expand(const TcRows<R>& t, uint32_t sm, int* pc)
{
#pragma unroll
  for (int u = 0; u < R * 4 / TC_THREADS; u++) {
    int r, kb;
    tc_item(threadIdx.x + u * TC_THREADS, r, kb);
    const uint4 v = t.v[u];
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    const uint32_t row = sm + kb * (R * 128) + r * 128;
#pragma unroll
    for (int c = 0; c < 8; c++) {   // chunk c: bits 16 c .. 16 c + 15 of the block
      const uint32_t x = w[c >> 1] >> (16 * (c & 1));
      const uint32_t o0 = ((x & 0xfu) * 0x00204081u) & 0x01010101u;
      const uint32_t o1 = (((x >> 4) & 0xfu) * 0x00204081u) & 0x01010101u;
      const uint32_t o2 = (((x >> 8) & 0xfu) * 0x00204081u) & 0x01010101u;
      const uint32_t o3 = (((x >> 12) & 0xfu) * 0x00204081u) & 0x01010101u;
      asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(row + ((c ^ (r & 7)) << 4)), "r"(o0), "r"(o1),
                   "r"(o2), "r"(o3));
    }
    int cnt = __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
    cnt += __shfl_xor_sync(0xffffffffu, cnt, 8);
    cnt += __shfl_xor_sync(0xffffffffu, cnt, 16);
    if (kb == 0) pc[r] = cnt;
  }
}
static_assert((TC_M * 4) % TC_THREADS == 0 && (TC_N * 4) % TC_THREADS == 0, "whole (row, K block) items per thread");

__device__ __forceinline__ void tc_wait(uint32_t mbar, uint32_t phase, unsigned* err)
{
  uint32_t done = 0;
  long long spins = 0;
  while (!done) {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(done)
                 : "r"(mbar), "r"(phase));
    if (!done && ++spins > (1ll << 28)) {   // never expected: report instead of hanging the GPU
      atomicOr(err, 1u);
      return;
    }
  }
}

template <bool RADIUS>
__global__ void __launch_bounds__(TC_THREADS, 1) k_hamming_tc(const uint8_t* q, long long nq, const uint8_t* r,
                                                              long long nr, int32_t* out, long long ld, int t_m,
                                                              unsigned long long* keys, int32_t* dist, long long cap,
                                                              unsigned long long* count, unsigned* err)
{
  extern __shared__ uint8_t tc_dsm[];
  uint8_t* sA = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(tc_dsm) + 1023) & ~(uintptr_t)1023);
  uint8_t* sB = sA + TC_M * 512;
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tslot;
  __shared__ int pq[TC_M];
  __shared__ __align__(16) int pr[TC_N];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long q0 = (long long)blockIdx.y * TC_M;
  const long long n_ct = (nr + TC_N - 1) / TC_N;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc_smem_u32(&tslot)),
                 "r"(TC_N));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tc_smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  {
    TcRows<TC_M> ta;
    tc_load<TC_M>(q, nq, q0, ta);
    tc_expand<TC_M>(ta, tc_smem_u32(sA), pq);
  }
  TcRows<TC_N> tb;   // packed rows of the next reference tile (prefetched)
  tc_load<TC_N>(r, nr, (long long)blockIdx.x * TC_N, tb);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot, mb = tc_smem_u32(&mbar);
  const int row = 32 * (warp & 3) + lane, cb = TC_COLS * (warp >> 2);
  const long long qi = q0 + row;
  uint32_t phase = 0;
#pragma unroll 1
  for (long long ct = blockIdx.x; ct < n_ct; ct += gridDim.x, phase ^= 1u) {
    const long long r0 = ct * TC_N;
    tc_expand<TC_N>(tb, tc_smem_u32(sB), pr);
    asm volatile("fence.proxy.async.shared::cta;");   // generic-proxy smem writes -> tensor core
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll 1
      for (int k = 0; k < 16; k++) {
        const int kb = k >> 2, sub = k & 3;
        const uint64_t da = tc_sdesc(tc_smem_u32(sA + kb * TC_M * 128 + sub * 32));
        const uint64_t db = tc_sdesc(tc_smem_u32(sB + kb * TC_N * 128 + sub * 32));
        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                     " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
                     "l"(da), "l"(db), "r"(TC_IDESC), "r"((uint32_t)k));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mb));
    }
    if (ct + gridDim.x < n_ct) tc_load<TC_N>(r, nr, (ct + gridDim.x) * TC_N, tb);   // overlaps MMA + epilogue
    tc_wait(mb, phase, err);
    asm volatile("tcgen05.fence::after_thread_sync;");
    const int pa = pq[row];
#pragma unroll 1
    for (int c0 = 0; c0 < TC_COLS; c0 += 32) {
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
      const long long rj0 = r0 + cb + c0;
      if (!RADIUS) {
        // transpose the warp's 32 x 32 block through smem (the B operand
        // region: the MMA reading it has completed) so every store writes one
        // 128-byte row segment
        int* st = reinterpret_cast<int*>(sB) + warp * (32 * 33);
        const int4* pr4 = reinterpret_cast<const int4*>(pr + cb + c0);
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          const int4 p4 = pr4[j >> 2];
          st[lane * 33 + j] = pa + p4.x - 2 * (int)v[j];
          st[lane * 33 + j + 1] = pa + p4.y - 2 * (int)v[j + 1];
          st[lane * 33 + j + 2] = pa + p4.z - 2 * (int)v[j + 2];
          st[lane * 33 + j + 3] = pa + p4.w - 2 * (int)v[j + 3];
        }
        __syncwarp();
        const long long qb = q0 + 32 * (warp & 3);
        if (rj0 + lane < nr)
#pragma unroll 4
          for (int rr = 0; rr < 32; rr++)
            if (qb + rr < nq) out[(qb + rr) * ld + rj0 + lane] = st[rr * 33 + lane];
        __syncwarp();
      } else {
        uint32_t hits = 0;
        const int4* pr4 = reinterpret_cast<const int4*>(pr + cb + c0);
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          const int4 p4 = pr4[j >> 2];
          hits |= (uint32_t)(pa + p4.x - 2 * (int)v[j] <= t_m) << j;
          hits |= (uint32_t)(pa + p4.y - 2 * (int)v[j + 1] <= t_m) << (j + 1);
          hits |= (uint32_t)(pa + p4.z - 2 * (int)v[j + 2] <= t_m) << (j + 2);
          hits |= (uint32_t)(pa + p4.w - 2 * (int)v[j + 3] <= t_m) << (j + 3);
        }
        if (rj0 + 32 > nr) hits &= nr - rj0 >= 32 ? 0xffffffffu : (nr - rj0 <= 0 ? 0u : (1u << (nr - rj0)) - 1u);
        if (qi >= nq) hits = 0;
        if (__any_sync(0xffffffffu, hits != 0)) {   // matches are sparse
          for (int j = 0; j < 32; j++) {
            const bool hit = (hits >> j) & 1u;
            const unsigned m = __ballot_sync(0xffffffffu, hit);
            if (!m) continue;
            unsigned long long pos = 0;
            if (lane == __ffs(m) - 1) pos = atomicAdd(count, (unsigned long long)__popc(m));
            pos = __shfl_sync(0xffffffffu, pos, __ffs(m) - 1) + __popc(m & ((1u << lane) - 1));
            if (hit && (long long)pos < cap) {
              keys[pos] = ((unsigned long long)qi << 32) | (unsigned long long)(rj0 + j);
              dist[pos] = pa + pr[cb + c0 + j] - 2 * (int)v[j];
            }
          }
        }
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();   // TMEM reads and sB reads of this tile are done before the next one
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TC_N));
}

__global__ void k_split_keys(const unsigned long long* keys, long long n, int32_t* qi, int32_t* ri)
{
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const unsigned long long k = keys[i];
    qi[i] = (int32_t)(k >> 32);
    ri[i] = (int32_t)(k & 0xffffffffu);
  }
}

int match_status(cudaError_t e) { return e == cudaSuccess ? VF_OK : VF_ERR_CUDA; }

// tcgen05 path: 512-bit rows, 16-byte aligned; VF_MATCH_NO_TC=1 forces the
// mma.sync path (A/B comparison)
bool use_tc(const void* q, const void* r, int nbytes)
{
  static const bool off = getenv("VF_MATCH_NO_TC") != nullptr || getenv("VF_MATCH_POPC") != nullptr;
  return !off && nbytes == 64 && ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(r)) & 15) == 0;
}

// wait-timeout flag of the asynchronous matrix path (never expected to trip)
unsigned* tc_err()
{
  static unsigned* p = nullptr;
  if (!p && cudaMalloc(&p, sizeof(unsigned)) == cudaSuccess) cudaMemset(p, 0, sizeof(unsigned));
  return p;
}

// launch geometry of k_hamming_tc: grid.y = query tiles, grid.x = reference
// tile stride, about two waves of one CTA per SM in total
dim3 tc_grid(long long nq, long long nr)
{
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(k_hamming_tc<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_SMEM);
    cudaFuncSetAttribute(k_hamming_tc<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_SMEM);
  }
  const long long qt = (nq + TC_M - 1) / TC_M, rt = (nr + TC_N - 1) / TC_N;
  const long long gx = std::max<long long>(1, std::min<long long>(rt, (2LL * sms + qt - 1) / qt));
  return dim3((unsigned)gx, (unsigned)qt);
}

// mma.sync path: whole 32-bit words (<= 16 per row) and 4-byte aligned rows;
// VF_MATCH_POPC=1 forces the POPC kernels (A/B comparison)
bool use_mma(const void* q, const void* r, int nbytes)
{
  static const bool popc = getenv("VF_MATCH_POPC") != nullptr;
  return !popc && nbytes % 4 == 0 && nbytes <= 64 &&
         ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(r)) & 3) == 0;
}

}  // namespace

extern "C" int vf_hamming_matrix(const uint8_t* q_dev, int64_t nq, const uint8_t* r_dev, int64_t nr, int nbytes,
                                 int32_t* out_dev, int64_t ld, void* stream)
{
  if (nq < 0 || nr < 0 || nbytes < 1 || ld < nr) return VF_ERR_ARG;
  if (nq == 0 || nr == 0) return VF_OK;
  if (!q_dev || !r_dev || !out_dev || nq > INT32_MAX || nr > INT32_MAX) return VF_ERR_ARG;
  const dim3 grid((unsigned)((nr + HM_T - 1) / HM_T), (unsigned)((nq + HM_T - 1) / HM_T));
  if (grid.y > 65535) return VF_ERR_ARG;
  if (use_tc(q_dev, r_dev, nbytes))
    k_hamming_tc<false><<<tc_grid(nq, nr), TC_THREADS, TC_SMEM, (cudaStream_t)stream>>>(
        q_dev, nq, r_dev, nr, out_dev, ld, 0, nullptr, nullptr, 0, nullptr, tc_err());
  else if (use_mma(q_dev, r_dev, nbytes))
    k_hamming_mma<false><<<grid, HM_THREADS, 0, (cudaStream_t)stream>>>(q_dev, nq, r_dev, nr, nbytes, out_dev, ld, 0,
                                                                       nullptr, nullptr, 0, nullptr);
  else
    k_hamming_matrix<<<grid, HM_THREADS, 0, (cudaStream_t)stream>>>(q_dev, nq, r_dev, nr, nbytes, out_dev, ld);
  return match_status(cudaGetLastError());
}

extern "C" int vf_radius_match(const uint8_t* q_dev, int64_t nq, const uint8_t* r_dev, int64_t nr, int nbytes,
                               int t_m, int32_t* q_idx_dev, int32_t* r_idx_dev, int32_t* dist_dev, int64_t cap,
                               int64_t* n_matches, void* stream)
{
  if (!n_matches || nq < 0 || nr < 0 || nbytes < 1 || cap < 0) return VF_ERR_ARG;
  *n_matches = 0;
  if (nq == 0 || nr == 0) return VF_OK;                 // matching.py:84-85
  if (!q_dev || !r_dev || nq > INT32_MAX || nr > INT32_MAX) return VF_ERR_ARG;
  if (cap > 0 && (!q_idx_dev || !r_idx_dev || !dist_dev)) return VF_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const dim3 grid((unsigned)((nr + HM_T - 1) / HM_T), (unsigned)((nq + HM_T - 1) / HM_T));
  if (grid.y > 65535) return VF_ERR_ARG;
  const long long kcap = cap > 0 ? cap : 1;
  unsigned long long *keys = nullptr, *keys_sorted = nullptr, *count = nullptr;
  int32_t* dist_tmp = nullptr;
  cudaError_t e = cudaMallocAsync(&keys, kcap * sizeof(unsigned long long), st);
  if (e == cudaSuccess) e = cudaMallocAsync(&keys_sorted, kcap * sizeof(unsigned long long), st);
  if (e == cudaSuccess) e = cudaMallocAsync(&dist_tmp, kcap * sizeof(int32_t), st);
  if (e == cudaSuccess) e = cudaMallocAsync(&count, 2 * sizeof(unsigned long long), st);
  if (e == cudaSuccess) e = cudaMemsetAsync(count, 0, 2 * sizeof(unsigned long long), st);
  unsigned* err = reinterpret_cast<unsigned*>(count + 1);
  if (e == cudaSuccess) {
    if (use_tc(q_dev, r_dev, nbytes))
      k_hamming_tc<true><<<tc_grid(nq, nr), TC_THREADS, TC_SMEM, st>>>(q_dev, nq, r_dev, nr, nullptr, 0, t_m, keys,
                                                                       dist_tmp, cap, count, err);
    else if (use_mma(q_dev, r_dev, nbytes))
      k_hamming_mma<true><<<grid, HM_THREADS, 0, st>>>(q_dev, nq, r_dev, nr, nbytes, nullptr, 0, t_m, keys, dist_tmp,
                                                       cap, count);
    else
      k_radius_match<<<grid, HM_THREADS, 0, st>>>(q_dev, nq, r_dev, nr, nbytes, t_m, keys, dist_tmp, cap, count);
    e = cudaGetLastError();
  }
  unsigned long long n2[2] = {0, 0};
  if (e == cudaSuccess) e = cudaMemcpyAsync(n2, count, sizeof(n2), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  const unsigned long long n = n2[0];
  int rc = match_status(e);
  if (rc == VF_OK && (n2[1] & 0xffffffffull)) rc = VF_ERR_CUDA;   // a tensor-core wait timed out
  if (rc == VF_OK) {
    *n_matches = (int64_t)n;
    if ((long long)n > cap) {
      rc = VF_ERR_MATCH_CAPACITY;
    } else if (n > 0) {
      // (query, reference) order of np.nonzero: sort the 64-bit keys
      int end_bit = 64;
      while (end_bit > 1 && !(((unsigned long long)(nq - 1) << 32) >> (end_bit - 1))) end_bit--;
      size_t tmp_bytes = 0;
      cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys, keys_sorted, dist_tmp, dist_dev, (int64_t)n, 0,
                                      end_bit, st);
      void* tmp = nullptr;
      e = cudaMallocAsync(&tmp, tmp_bytes, st);
      if (e == cudaSuccess)
        e = cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, keys_sorted, dist_tmp, dist_dev, (int64_t)n, 0,
                                            end_bit, st);
      if (e == cudaSuccess) {
        k_split_keys<<<(unsigned)std::min<long long>(4096, ((long long)n + 255) / 256), 256, 0, st>>>(
            keys_sorted, (long long)n, q_idx_dev, r_idx_dev);
        e = cudaGetLastError();
      }
      if (tmp) cudaFreeAsync(tmp, st);
      if (e == cudaSuccess) e = cudaStreamSynchronize(st);
      rc = match_status(e);
    }
  }
  if (keys) cudaFreeAsync(keys, st);
  if (keys_sorted) cudaFreeAsync(keys_sorted, st);
  if (dist_tmp) cudaFreeAsync(dist_tmp, st);
  if (count) cudaFreeAsync(count, st);
  return rc;
}
