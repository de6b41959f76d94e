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

__global__ void k_split_keys(const unsigned long long* keys, long long n, int32_t* qi, int32_t* ri)
{
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const unsigned long long k = keys[i];
    qi[i] = (int32_t)(k >> 32);
    ri[i] = (int32_t)(k & 0xffffffffu);
  }
}

int match_status(cudaError_t e) { return e == cudaSuccess ? VF_OK : VF_ERR_CUDA; }

}  // namespace

extern "C" int vf_hamming_matrix(const uint8_t* q_dev, int64_t nq, const uint8_t* r_dev, int64_t nr, int nbytes,
                                 int32_t* out_dev, int64_t ld, void* stream)
{
  if (nq < 0 || nr < 0 || nbytes < 1 || ld < nr) return VF_ERR_ARG;
  if (nq == 0 || nr == 0) return VF_OK;
  if (!q_dev || !r_dev || !out_dev || nq > INT32_MAX || nr > INT32_MAX) return VF_ERR_ARG;
  const dim3 grid((unsigned)((nr + HM_T - 1) / HM_T), (unsigned)((nq + HM_T - 1) / HM_T));
  if (grid.y > 65535) return VF_ERR_ARG;
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
