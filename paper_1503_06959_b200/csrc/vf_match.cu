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
#include <climits>
#include <cstdio>
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

// Wait for the phase of parity `phase` of an mbarrier.  SLEEP: back off
// between polls (waiting warps leave their scheduler's issue slots to the
// single-thread producer lanes).
template <bool SLEEP = false>
__device__ __forceinline__ void tc_wait(uint32_t mbar, uint32_t phase, unsigned* err)
{
  uint32_t done = 0;
  long long spins = 0;
  while (!done) {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(done)
                 : "r"(mbar), "r"(phase));
    if (!done) {
      if (SLEEP) __nanosleep(64);
      if (++spins > (1ll << 28)) {   // never expected: report instead of hanging the GPU
        atomicOr(err, 1u);
        return;
      }
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

// ---------------------------------------------------------------------------
// Pipelined tcgen05 radius match (512-bit rows).  The packed rows of both
// sides are first expanded ONCE (k_tc_images) into per-128-row tile images:
// the exact shared-memory image the UMMA descriptors expect (K-major,
// SWIZZLE_128B: K block kb = [128 rows][128 B], 16-B chunk c of row r at
// c ^ (r & 7)), 64 KB per 128 rows, plus per-row popcounts.  k_radius_tc
// then runs a warp-specialised pipeline, one persistent CTA per SM owning a
// contiguous range of the (256-query, 128-reference) tile grid:
//   * load lane: streams reference K blocks (16 KB each, 1-D bulk TMA,
//     mbarrier complete_tx) through a ring of RT_STAGES stages;
//   * MMA lane: keeps the 256-row query block A (128 KB) resident (reloaded
//     when the range moves to the next query block) and issues, per K block,
//     2 x 4 tcgen05.mma.kind::i8 (M = N = 128, K = 32) into two 128 x 128 s32
//     TMEM accumulators; each K block's commit frees its stage, each tile's
//     commit publishes the accumulator pair (double-buffered: 512 columns);
//   * 16 epilogue warps: tcgen05.ld, a max-of-(2 v - |r|) test per 32
//     columns (matches are sparse), exact hits buffered per warp in shared
//     memory and flushed with one reservation per batch.
// Reusing each reference block for 256 query rows halves the L2 -> SM traffic
// of the expanded operands relative to a 128-row block.
// ---------------------------------------------------------------------------
#define RT_ROWS 128
#define RT_IMG (RT_ROWS * 512)            // bytes per 128-row tile image
#define RT_KBLK (RT_ROWS * 128)           // bytes per K block of a tile image (one ring stage)
#define RT_STAGES 5
#define RT_EPI 16                         // epilogue warps
#define RT_THREADS (32 * RT_EPI + 64)     // + load warp + MMA warp
#define RT_SMEM (2 * RT_IMG + RT_STAGES * RT_KBLK + 1024)
#define RT_MBUF 32                        // matches buffered per epilogue warp

constexpr uint32_t RT_IDESC = (2u << 4) | ((uint32_t)(RT_ROWS >> 3) << 17) | ((uint32_t)(RT_ROWS >> 4) << 24);

// rows [0, n) of 64-byte packed rows -> tile images (rows past n are zero)
// and popcounts; item = (row, K block), 16 packed bytes -> 128 expanded bytes
__global__ void k_tc_images(const uint8_t* src, long long n, long long n_pad, uint8_t* img, int* pc)
{
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n_pad * 4; i += (long long)gridDim.x * blockDim.x) {
    const long long row = i >> 2;
    const int kb = (int)(i & 3);
    const uint4 v = row < n ? __ldg(reinterpret_cast<const uint4*>(src + row * 64) + kb) : make_uint4(0, 0, 0, 0);
    const int r = (int)(row & (RT_ROWS - 1));
    uint8_t* dst = img + (row / RT_ROWS) * RT_IMG + kb * (RT_ROWS * 128) + r * 128;
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int c = 0; c < 8; c++) {
      const uint32_t x = w[c >> 1] >> (16 * (c & 1));
      uint4 o;
      o.x = ((x & 0xfu) * 0x00204081u) & 0x01010101u;
      o.y = (((x >> 4) & 0xfu) * 0x00204081u) & 0x01010101u;
      o.z = (((x >> 8) & 0xfu) * 0x00204081u) & 0x01010101u;
      o.w = (((x >> 12) & 0xfu) * 0x00204081u) & 0x01010101u;
      *reinterpret_cast<uint4*>(dst + ((c ^ (r & 7)) << 4)) = o;
    }
    int cnt = __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
    cnt += __shfl_xor_sync(0xffffffffu, cnt, 1);
    cnt += __shfl_xor_sync(0xffffffffu, cnt, 2);
    if (kb == 0) pc[row] = cnt;
  }
}

__device__ __forceinline__ void rt_expect_load(uint32_t mbar, uint32_t sdst, const void* gsrc, uint32_t bytes)
{
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sdst),
               "l"(gsrc), "r"(bytes), "r"(mbar)
               : "memory");
}

__global__ void __launch_bounds__(RT_THREADS, 1) k_radius_tc(const uint8_t* qimg, const int* qpc, long long nq,
                                                             const uint8_t* rimg, const int* rpc, long long nr,
                                                             int t_m, unsigned long long* keys, int32_t* dist,
                                                             long long cap, unsigned long long* count, unsigned* err)
{
  extern __shared__ uint8_t rt_dsm[];
  uint8_t* sA = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(rt_dsm) + 1023) & ~(uintptr_t)1023);
  uint8_t* sR = sA + 2 * RT_IMG;   // ring of RT_STAGES K blocks
  __shared__ __align__(8) uint64_t mb_full[RT_STAGES], mb_empty[RT_STAGES], mb_mma[2], mb_free[2], mb_a;
  __shared__ uint32_t tslot;
  __shared__ __align__(16) uint32_t prs[RT_EPI][32];            // per epilogue warp: column popcount pairs
  __shared__ unsigned long long mkey[RT_EPI][RT_MBUF];          // per epilogue warp: buffered matches
  __shared__ int mdist[RT_EPI][RT_MBUF];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long qt = (nq + 2 * RT_ROWS - 1) / (2 * RT_ROWS), rt = (nr + RT_ROWS - 1) / RT_ROWS;
  const long long T = qt * rt;
  const long long j0 = T * blockIdx.x / gridDim.x, j1 = T * (blockIdx.x + 1) / gridDim.x;
  if (j0 >= j1) return;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc_smem_u32(&tslot)),
                 "r"(4 * RT_ROWS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  const uint32_t full0 = tc_smem_u32(&mb_full[0]), empty0 = tc_smem_u32(&mb_empty[0]);
  const uint32_t mma0 = tc_smem_u32(&mb_mma[0]), free0 = tc_smem_u32(&mb_free[0]), mba = tc_smem_u32(&mb_a);
  if (tid == 0) {
    for (int k = 0; k < RT_STAGES; k++) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(full0 + 8 * k));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(empty0 + 8 * k));
    }
    for (int k = 0; k < 2; k++) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mma0 + 8 * k));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(free0 + 8 * k), "r"(RT_EPI));
    }
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mba));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  const uint32_t sa = tc_smem_u32(sA), sr = tc_smem_u32(sR);
  const long long n_loads = (j1 - j0) * 4;   // K blocks of the range, in order
  if (warp == RT_EPI) {
    // ---- load lane: reference K blocks through the ring ----
    if (lane == 0) {
      long long rtile = j0 % rt;
      int kb = 0, st = 0;
      uint32_t ph = 1;   // parity of the empty phase to wait for (none in the first pass over the ring)
#pragma unroll 1
      for (long long i = 0; i < n_loads; i++) {
        if (i >= RT_STAGES) tc_wait(empty0 + 8 * st, ph, err);   // freed by the MMAs of load i - S
        rt_expect_load(full0 + 8 * st, sr + st * RT_KBLK, rimg + rtile * RT_IMG + kb * RT_KBLK, RT_KBLK);
        if (++st == RT_STAGES) { st = 0; ph ^= 1u; }
        if (++kb == 4) {
          kb = 0;
          if (++rtile == rt) rtile = 0;
        }
      }
    }
  } else if (warp == RT_EPI + 1) {
    // ---- MMA lane ----
    if (lane == 0) {
      uint32_t a_phase = 0;
      long long a_tile = -1;
      const uint64_t dA0 = tc_sdesc(sa), dR0 = tc_sdesc(sr);
#ifdef RT_PROBE
      unsigned long long probe_full = 0, probe_free = 0, probe_issue = 0, probe_a = 0, probe_start = clock64();
#endif
      long long qtile = j0 / rt, rtile = j0 - qtile * rt;
      int st = 0;
      uint32_t fph = 0;   // parity of the next full phase of stage st
#pragma unroll 1
      for (long long j = j0; j < j1; j++) {
        const long long jj = j - j0;
        const int buf = (int)(jj & 1);
        if (qtile != a_tile) {
          // A is read by the MMAs of tile j - 1: wait for them before reloading
          if (jj > 0) tc_wait(mma0 + 8 * (buf ^ 1), (uint32_t)(((jj - 1) >> 1) & 1), err);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mba), "r"(2 * RT_IMG) : "memory");
          for (int m = 0; m < 2; m++)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             sa + m * RT_IMG),
                         "l"(qimg + (2 * qtile + m) * RT_IMG), "r"(RT_IMG), "r"(mba)
                         : "memory");
          tc_wait(mba, a_phase, err);
          a_phase ^= 1u;
          a_tile = qtile;
        }
#ifdef RT_PROBE
        unsigned long long pt0 = clock64();
#endif
        if (jj >= 2) tc_wait(free0 + 8 * buf, (uint32_t)(((jj - 2) >> 1) & 1), err);   // accumulators read
#ifdef RT_PROBE
        probe_free += clock64() - pt0;
#endif
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t acc0 = tmem + (uint32_t)(2 * buf * RT_ROWS);
#pragma unroll
        for (int kb = 0; kb < 4; kb++) {
#ifdef RT_PROBE
          unsigned long long pt1 = clock64();
#endif
          tc_wait(full0 + 8 * st, fph, err);
#ifdef RT_PROBE
          unsigned long long pt2 = clock64();
          probe_full += pt2 - pt1;
#endif
          asm volatile("tcgen05.fence::after_thread_sync;");
          // descriptors: the start-address field is addr >> 4 (< 2^14), so
          // offsets add to the base descriptor directly
          const uint64_t db = dR0 + (uint64_t)((st * RT_KBLK) >> 4);
#pragma unroll
          for (int m = 0; m < 2; m++)
#pragma unroll
            for (int sub = 0; sub < 4; sub++) {
              const uint64_t da = dA0 + (uint64_t)((m * RT_IMG + kb * RT_KBLK + sub * 32) >> 4);
              asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                           " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(acc0 + m * RT_ROWS),
                           "l"(da), "l"(db + (uint64_t)(sub * 2)), "r"(RT_IDESC), "r"((uint32_t)(kb | sub)));
            }
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(empty0 + 8 * st));
#ifdef RT_PROBE
          probe_issue += clock64() - pt2;
#endif
          if (++st == RT_STAGES) { st = 0; fph ^= 1u; }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mma0 + 8 * buf));
        if (++rtile == rt) { rtile = 0; qtile++; }
      }
#ifdef RT_PROBE
      if (blockIdx.x < 4)
        printf("cta %d tiles %lld: total %llu clk, wait full %llu, wait free %llu, issue %llu\n", blockIdx.x, j1 - j0,
               clock64() - probe_start, probe_full, probe_free, probe_issue);
#endif
    }
  } else {
    // ---- epilogue warps: warp w reads TMEM lanes 32 (w & 3) .. of sub-tile
    // m = w >> 3 (query rows 128 m + ..), accumulator columns 64 ((w >> 2) & 1)
    // .. + 64 in two 32-column chunks ----
    const int m = warp >> 3, erow = 128 * m + 32 * (warp & 3) + lane, ecol = 64 * ((warp >> 2) & 1);
    uint32_t* pw = prs[warp];
    unsigned long long* bk = mkey[warp];
    int* bd = mdist[warp];
    int nb = 0;   // matches buffered by this warp (warp-uniform)
    auto flush = [&]() {
      unsigned long long pos = 0;
      if (lane == 0) pos = atomicAdd(count, (unsigned long long)nb);
      pos = __shfl_sync(0xffffffffu, pos, 0);
      for (int i = lane; i < nb; i += 32)
        if ((long long)(pos + i) < cap) {
          keys[pos + i] = bk[i];
          dist[pos + i] = bd[i];
        }
      __syncwarp();
      nb = 0;
    };
    long long qtile = j0 / rt, rtile = j0 - qtile * rt;
    auto col_pc = [&](long long c) { return c < nr ? __ldg(rpc + c) : 0x7ff; };   // past nr: never passes the fast test
    int prA = col_pc(rtile * RT_ROWS + ecol + lane), prB = col_pc(rtile * RT_ROWS + ecol + 32 + lane);
    long long qi = -1;
    int pa = 0, lim = INT_MAX;
#pragma unroll 1
    for (long long j = j0; j < j1; j++) {
      const long long jj = j - j0;
      const int buf = (int)(jj & 1);
      if (qtile * 2 * RT_ROWS + erow != qi) {   // the query rows change with the query block only
        qi = qtile * 2 * RT_ROWS + erow;
        pa = qi < nq ? __ldg(qpc + qi) : 0;
        lim = qi < nq ? pa - t_m : INT_MAX;   // hit iff pa + pr - 2 v <= t_m iff 2 v - pr >= pa - t_m
      }
      const long long rc0 = rtile * RT_ROWS + ecol;
      // column popcounts of the two chunks as 16x2 pairs (col k | col 32 + k)
      pw[lane] = (uint32_t)prA | ((uint32_t)prB << 16);
      __syncwarp();
      const long long qtile_n = rtile + 1 == rt ? qtile + 1 : qtile, rtile_n = rtile + 1 == rt ? 0 : rtile + 1;
      tc_wait(mma0 + 8 * buf, (uint32_t)((jj >> 1) & 1), err);
      asm volatile("tcgen05.fence::after_thread_sync;");
      // both 32-column chunks into registers as 16x2 pairs (q.r <= 512), then
      // the accumulator pair is released: the MMAs of tile j + 2 overlap this
      // tile's tests
      uint32_t w[32];
      {
        uint32_t t[32];
        const uint32_t ta = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((2 * buf + m) * RT_ROWS + ecol);
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                   "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                   : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7]),
                     "=r"(w[8]), "=r"(w[9]), "=r"(w[10]), "=r"(w[11]), "=r"(w[12]), "=r"(w[13]), "=r"(w[14]),
                     "=r"(w[15]), "=r"(w[16]), "=r"(w[17]), "=r"(w[18]), "=r"(w[19]), "=r"(w[20]), "=r"(w[21]),
                     "=r"(w[22]), "=r"(w[23]), "=r"(w[24]), "=r"(w[25]), "=r"(w[26]), "=r"(w[27]), "=r"(w[28]),
                     "=r"(w[29]), "=r"(w[30]), "=r"(w[31])
                   : "r"(ta));
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                   "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                   : "=r"(t[0]), "=r"(t[1]), "=r"(t[2]), "=r"(t[3]), "=r"(t[4]), "=r"(t[5]), "=r"(t[6]), "=r"(t[7]),
                     "=r"(t[8]), "=r"(t[9]), "=r"(t[10]), "=r"(t[11]), "=r"(t[12]), "=r"(t[13]), "=r"(t[14]),
                     "=r"(t[15]), "=r"(t[16]), "=r"(t[17]), "=r"(t[18]), "=r"(t[19]), "=r"(t[20]), "=r"(t[21]),
                     "=r"(t[22]), "=r"(t[23]), "=r"(t[24]), "=r"(t[25]), "=r"(t[26]), "=r"(t[27]), "=r"(t[28]),
                     "=r"(t[29]), "=r"(t[30]), "=r"(t[31])
                   : "r"(ta + 32));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
        for (int k = 0; k < 32; k++) w[k] |= t[k] << 16;
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(free0 + 8 * buf) : "memory");
      if (j + 1 < j1) {   // next tile's column popcounts, in flight during the tests
        prA = col_pc(rtile_n * RT_ROWS + ecol + lane);
        prB = col_pc(rtile_n * RT_ROWS + ecol + 32 + lane);
      }
      // fast test: max over the 64 columns of 2 q.r - |r| (matches are sparse)
      const uint4* p4 = reinterpret_cast<const uint4*>(pw);
      uint32_t mx = 0x80008000u;
#pragma unroll
      for (int k = 0; k < 32; k += 4) {
        const uint4 p = p4[k >> 2];
        mx = __vimax3_s16x2(mx, __vsub2(__vadd2(w[k], w[k]), p.x), __vsub2(__vadd2(w[k + 1], w[k + 1]), p.y));
        mx = __vimax3_s16x2(mx, __vsub2(__vadd2(w[k + 2], w[k + 2]), p.z), __vsub2(__vadd2(w[k + 3], w[k + 3]), p.w));
      }
      const unsigned cand = (__ballot_sync(0xffffffffu, (int)(short)(mx & 0xffffu) >= lim) ? 1u : 0u) |
                            (__ballot_sync(0xffffffffu, (int)(short)(mx >> 16) >= lim) ? 2u : 0u);
      if (cand) {
#pragma unroll 1
        for (int c = 0; c < 2; c++) {
          if (!((cand >> c) & 1u)) continue;
          const int c0 = 32 * c, sh = 16 * c;
          const long long left = nr - (rc0 + c0);   // columns of the chunk inside the reference set
          const uint32_t valid = left >= 32 ? 0xffffffffu : (left <= 0 ? 0u : (1u << left) - 1u);
          uint32_t hits = 0;
          const uint4* q4 = reinterpret_cast<const uint4*>(pw);
#pragma unroll
          for (int k = 0; k < 32; k += 4) {
            const uint4 p = q4[k >> 2];
            hits |= (uint32_t)(2 * (int)((w[k] >> sh) & 0xffffu) - (int)((p.x >> sh) & 0xffffu) >= lim) << k;
            hits |= (uint32_t)(2 * (int)((w[k + 1] >> sh) & 0xffffu) - (int)((p.y >> sh) & 0xffffu) >= lim) << (k + 1);
            hits |= (uint32_t)(2 * (int)((w[k + 2] >> sh) & 0xffffu) - (int)((p.z >> sh) & 0xffffu) >= lim) << (k + 2);
            hits |= (uint32_t)(2 * (int)((w[k + 3] >> sh) & 0xffffu) - (int)((p.w >> sh) & 0xffffu) >= lim) << (k + 3);
          }
          hits &= valid;
          if (!__any_sync(0xffffffffu, hits != 0)) continue;
          // buffer the chunk's matches (order is restored by the sort)
          const int nh = __popc(hits);
          int off = nh;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, off, o);
            if (lane >= o) off += y;
          }
          const int tot = __shfl_sync(0xffffffffu, off, 31);
          off -= nh;
          if (nb + tot > RT_MBUF) flush();
          unsigned long long* kd = bk;
          int* dd = bd;
          long long pos = nb + off;
          if (tot > RT_MBUF) {   // more matches in one chunk than the buffer holds: direct
            unsigned long long p0 = 0;
            if (lane == 0) p0 = atomicAdd(count, (unsigned long long)tot);
            pos = (long long)__shfl_sync(0xffffffffu, p0, 0) + off;
            kd = keys;
            dd = dist;
          }
          for (uint32_t h = hits; h; h &= h - 1) {
            const int k = __ffs(h) - 1;
            uint32_t wk = 0;   // w[k] without dynamic register indexing
#pragma unroll
            for (int kk = 0; kk < 32; kk++) wk = kk == k ? w[kk] : wk;
            const int vk = (int)((wk >> sh) & 0xffffu), pk = (int)((pw[k] >> sh) & 0xffffu);
            if (tot <= RT_MBUF || pos < cap) {
              kd[pos] = ((unsigned long long)qi << 32) | (unsigned long long)(rc0 + c0 + k);
              dd[pos] = pa + pk - 2 * vk;
            }
            pos++;
          }
          __syncwarp();
          if (tot <= RT_MBUF) nb += tot;
        }
      }
      __syncwarp();   // pw is rewritten for the next tile
      qtile = qtile_n;
      rtile = rtile_n;
    }
    if (nb) flush();
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(4 * RT_ROWS));
  }
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

// Stream-ordered scratch from a private pool that keeps its memory (release
// threshold = max): repeated calls reuse it instead of remapping pages at
// every synchronisation.
cudaMemPool_t mt_pool()
{
  static cudaMemPool_t pool = [] {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaMemPoolProps pp = {};
    pp.allocType = cudaMemAllocationTypePinned;
    pp.location.type = cudaMemLocationTypeDevice;
    pp.location.id = dev;
    cudaMemPool_t p = nullptr;
    if (cudaMemPoolCreate(&p, &pp) != cudaSuccess) return (cudaMemPool_t) nullptr;
    uint64_t keep = ~0ull;
    cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &keep);
    return p;
  }();
  return pool;
}

template <typename T>
cudaError_t mt_alloc(T** p, size_t bytes, cudaStream_t st)
{
  cudaMemPool_t pool = mt_pool();
  if (!pool) return cudaErrorMemoryAllocation;
  return cudaMallocFromPoolAsync(reinterpret_cast<void**>(p), bytes, pool, st);
}

// tile images of both sides, then the pipelined tensor-core radius kernel
cudaError_t radius_tc(const uint8_t* q, long long nq, const uint8_t* r, long long nr, int t_m, unsigned long long* keys,
                      int32_t* dist, long long cap, unsigned long long* count, unsigned* err, cudaStream_t st)
{
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(k_radius_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, RT_SMEM);
  }
  const long long qt = 2 * ((nq + 2 * RT_ROWS - 1) / (2 * RT_ROWS)), rt = (nr + RT_ROWS - 1) / RT_ROWS;   // qt: 128-row images, even
  uint8_t *qi = nullptr, *ri = nullptr;
  int *qp = nullptr, *rp = nullptr;
  cudaError_t e = mt_alloc(&qi, qt * RT_IMG, st);
  if (e == cudaSuccess) e = mt_alloc(&ri, rt * RT_IMG, st);
  if (e == cudaSuccess) e = mt_alloc(&qp, qt * RT_ROWS * sizeof(int), st);
  if (e == cudaSuccess) e = mt_alloc(&rp, rt * RT_ROWS * sizeof(int), st);
  if (e == cudaSuccess) {
    k_tc_images<<<(unsigned)std::min<long long>(4 * sms, (qt * RT_ROWS * 4 + 255) / 256), 256, 0, st>>>(
        q, nq, qt * RT_ROWS, qi, qp);
    k_tc_images<<<(unsigned)std::min<long long>(4 * sms, (rt * RT_ROWS * 4 + 255) / 256), 256, 0, st>>>(
        r, nr, rt * RT_ROWS, ri, rp);
    const long long grid = std::min<long long>(qt / 2 * rt, sms);
    k_radius_tc<<<(unsigned)grid, RT_THREADS, RT_SMEM, st>>>(qi, qp, nq, ri, rp, nr, t_m, keys, dist, cap, count, err);
    e = cudaGetLastError();
  }
  if (qi) cudaFreeAsync(qi, st);
  if (ri) cudaFreeAsync(ri, st);
  if (qp) cudaFreeAsync(qp, st);
  if (rp) cudaFreeAsync(rp, st);
  return e;
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

// vf_match_timing state (benchmarks only)
struct MatchTiming {
  bool on = false;
  double ms = 0.0;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
};
MatchTiming g_mt;

extern "C" int vf_match_timing(int enable, double* ms)
{
  if (enable) {
    if (!g_mt.e0 && (cudaEventCreate(&g_mt.e0) != cudaSuccess || cudaEventCreate(&g_mt.e1) != cudaSuccess))
      return VF_ERR_CUDA;
    g_mt.ms = 0.0;
    g_mt.on = true;
  } else {
    g_mt.on = false;
  }
  if (ms) *ms = g_mt.ms;
  return VF_OK;
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
  cudaError_t e = mt_alloc(&keys, kcap * sizeof(unsigned long long), st);
  if (e == cudaSuccess) e = mt_alloc(&keys_sorted, kcap * sizeof(unsigned long long), st);
  if (e == cudaSuccess) e = mt_alloc(&dist_tmp, kcap * sizeof(int32_t), st);
  if (e == cudaSuccess) e = mt_alloc(&count, 2 * sizeof(unsigned long long), st);
  if (e == cudaSuccess) e = cudaMemsetAsync(count, 0, 2 * sizeof(unsigned long long), st);
  unsigned* err = reinterpret_cast<unsigned*>(count + 1);
  if (e == cudaSuccess) {
    if (g_mt.on) cudaEventRecord(g_mt.e0, st);
    if (use_tc(q_dev, r_dev, nbytes))
      e = radius_tc(q_dev, nq, r_dev, nr, t_m, keys, dist_tmp, cap, count, err, st);
    else if (use_mma(q_dev, r_dev, nbytes))
      k_hamming_mma<true><<<grid, HM_THREADS, 0, st>>>(q_dev, nq, r_dev, nr, nbytes, nullptr, 0, t_m, keys, dist_tmp,
                                                       cap, count);
    else
      k_radius_match<<<grid, HM_THREADS, 0, st>>>(q_dev, nq, r_dev, nr, nbytes, t_m, keys, dist_tmp, cap, count);
    e = cudaGetLastError();
  }
  if (g_mt.on) cudaEventRecord(g_mt.e1, st);
  unsigned long long n2[2] = {0, 0};
  if (e == cudaSuccess) e = cudaMemcpyAsync(n2, count, sizeof(n2), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (g_mt.on && e == cudaSuccess) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, g_mt.e0, g_mt.e1) == cudaSuccess) g_mt.ms += ms;
  }
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
      // never below the 32 reference-index bits (a single query still sorts by r)
      while (end_bit > 32 && !(((unsigned long long)(nq - 1) << 32) >> (end_bit - 1))) end_bit--;
      size_t tmp_bytes = 0;
      cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys, keys_sorted, dist_tmp, dist_dev, (int64_t)n, 0,
                                      end_bit, st);
      void* tmp = nullptr;
      e = mt_alloc(&tmp, tmp_bytes, st);
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
