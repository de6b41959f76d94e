// vf_match.cu -- descriptor matching on packed binary descriptors
// (SURVEY.md 8(f) rank 1): hamming_matrix and radius_match of
// /root/reference/pkg/src/vidfeat/matching.py:47-94.
//
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

__global__ void k_split_keys(const unsigned long long* keys, long long n, int32_t* qi, int32_t* ri)
{
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const unsigned long long k = keys[i];
    qi[i] = (int32_t)(k >> 32);
    ri[i] = (int32_t)(k & 0xffffffffu);
  }
}

int match_status(cudaError_t e) { return e == cudaSuccess ? VF_OK : VF_ERR_CUDA; }

// tensor-core path: whole 32-bit words (<= 16 per row) and 4-byte aligned rows;
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
  if (use_mma(q_dev, r_dev, nbytes))
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
  if (e == cudaSuccess) e = cudaMallocAsync(&count, sizeof(unsigned long long), st);
  if (e == cudaSuccess) e = cudaMemsetAsync(count, 0, sizeof(unsigned long long), st);
  if (e == cudaSuccess) {
    if (use_mma(q_dev, r_dev, nbytes))
      k_hamming_mma<true><<<grid, HM_THREADS, 0, st>>>(q_dev, nq, r_dev, nr, nbytes, nullptr, 0, t_m, keys, dist_tmp,
                                                       cap, count);
    else
      k_radius_match<<<grid, HM_THREADS, 0, st>>>(q_dev, nq, r_dev, nr, nbytes, t_m, keys, dist_tmp, cap, count);
    e = cudaGetLastError();
  }
  unsigned long long n = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&n, count, sizeof(n), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  int rc = match_status(e);
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
