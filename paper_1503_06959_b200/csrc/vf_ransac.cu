// vf_ransac.cu -- batched geometric verification on the GPU (SURVEY.md 8(f)
// rank 4): ransac_homography (/root/reference/pkg/src/vidfeat/matching.py:
// 151-192) for many match sets in one call, as count_mpr / locate_object
// (matching.py:209-220, evaluation.py:95-121) consume it.
//
// Per call (all problems at once, four launches on `stream`):
//   k_rs_samples   thread per (problem, iteration): the reference's minimal
//                  samples, rng.choice(n, 4, replace=False) of
//                  default_rng(seed), by PCG64 jump-ahead (vf_rng.cuh)
//   k_rs_fixup     thread per problem: iterations after a (rare) Lemire
//                  rejection regenerated sequentially
//   k_rs_score     CTA per (problem, 64 iterations): 64 minimal homographies
//                  solved into shared memory, then every match point scored
//                  against all 64 (thread per point, ballot + popc counts);
//                  best (max count, first iteration) by a 64-bit atomicMax
//   k_rs_refit     CTA per problem: the best consensus set, the normalized DLT
//                  refit (matching.py:109-137) as the least eigenvector of the
//                  9x9 normal matrix, the usable test (matching.py:140-146),
//                  the final inlier mask and count (matching.py:187-192)
// Minimal models: for 4 points the normalized DLT's null vector is the
// homography through the 4 correspondences; it is computed in closed form
// (unit square -> quad maps, H = Q_dst adj(Q_src)) on centred, scaled
// coordinates and normalized by h22 as _dlt does.  Float results differ from
// numpy's LAPACK path by rounding only (parity tolerance in tests/).
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>

#include "../../include/vidfeat_b200.h"
#include "vf_rng.cuh"

namespace {

constexpr int RS_HB = 64;        // hypotheses per scoring CTA
constexpr int RS_THREADS = 256;

// ---- 3x3 helpers ---------------------------------------------------------
__device__ __forceinline__ void mat3mul(const double* a, const double* b, double* c)
{
#pragma unroll
  for (int i = 0; i < 3; i++)
#pragma unroll
    for (int j = 0; j < 3; j++)
      c[3 * i + j] = __fma_rn(a[3 * i], b[j], __fma_rn(a[3 * i + 1], b[3 + j], __dmul_rn(a[3 * i + 2], b[6 + j])));
}

__device__ __forceinline__ double det3(const double* h)
{
  return h[0] * (h[4] * h[8] - h[5] * h[7]) - h[1] * (h[3] * h[8] - h[5] * h[6]) + h[2] * (h[3] * h[7] - h[4] * h[6]);
}

// 2-norm condition number (largest / smallest singular value) by one-sided
// Jacobi on the columns: the smallest singular value keeps absolute accuracy
// ~eps * sigma_max, as LAPACK's (np.linalg.cond, matching.py:146)
__device__ double cond3(const double* h)
{
  double c[3][3];
#pragma unroll
  for (int i = 0; i < 3; i++)
#pragma unroll
    for (int j = 0; j < 3; j++) c[j][i] = h[3 * i + j];
  for (int sweep = 0; sweep < 40; sweep++) {
    bool rot = false;
#pragma unroll
    for (int pq = 0; pq < 3; pq++) {
      const int p = pq == 2 ? 1 : 0, q = pq == 0 ? 1 : 2;
      double a = 0, b = 0, g = 0;
#pragma unroll
      for (int k = 0; k < 3; k++) {
        a += c[p][k] * c[p][k];
        b += c[q][k] * c[q][k];
        g += c[p][k] * c[q][k];
      }
      if (fabs(g) > 1e-15 * sqrt(a * b) && g != 0.0) {
        rot = true;
        const double zeta = (b - a) / (2.0 * g);
        const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / sqrt(1.0 + t * t), sn = cs * t;
#pragma unroll
        for (int k = 0; k < 3; k++) {
          const double u = c[p][k], v = c[q][k];
          c[p][k] = cs * u - sn * v;
          c[q][k] = sn * u + cs * v;
        }
      }
    }
    if (!rot) break;
  }
  double smax = 0.0, smin = INFINITY;
#pragma unroll
  for (int j = 0; j < 3; j++) {
    const double s = sqrt(c[j][0] * c[j][0] + c[j][1] * c[j][1] + c[j][2] * c[j][2]);
    smax = fmax(smax, s);
    smin = fmin(smin, s);
  }
  return smin > 0.0 ? smax / smin : INFINITY;
}

// _dlt's tail + _usable (matching.py:134-146): finite, scaled by h22 when
// |h22| > 1e-12, |det| >= 1e-12, cond < 1e12
__device__ bool finish_usable(double* h)
{
  for (int i = 0; i < 9; i++)
    if (!isfinite(h[i])) return false;
  if (fabs(h[8]) > 1e-12) {
    const double d = h[8];
    for (int i = 0; i < 9; i++) h[i] = h[i] / d;
  }
  if (fabs(det3(h)) < 1e-12) return false;
  return cond3(h) < 1e12;
}

// projective map of the unit square corners (0,0),(1,0),(1,1),(0,1) onto
// the quad (x[k], y[k])
__device__ __forceinline__ void square_to_quad(const double* x, const double* y, double* m)
{
  const double sx = (x[0] - x[1]) + (x[2] - x[3]), sy = (y[0] - y[1]) + (y[2] - y[3]);
  const double dx1 = x[1] - x[2], dx2 = x[3] - x[2], dy1 = y[1] - y[2], dy2 = y[3] - y[2];
  const double den = dx1 * dy2 - dx2 * dy1;
  const double g = (sx * dy2 - dx2 * sy) / den, h = (dx1 * sy - sx * dy1) / den;
  m[0] = x[1] - x[0] + g * x[1]; m[1] = x[3] - x[0] + h * x[3]; m[2] = x[0];
  m[3] = y[1] - y[0] + g * y[1]; m[4] = y[3] - y[0] + h * y[3]; m[5] = y[0];
  m[6] = g;                      m[7] = h;                      m[8] = 1.0;
}

// centroid / sqrt(2)-mean-distance conditioning of 4 points (as
// _normalize_points, matching.py:97-106); false if the points coincide
__device__ __forceinline__ bool cond4(const double* x, const double* y, double* u, double* v, double& s, double& cx,
                                      double& cy)
{
  cx = ((x[0] + x[1]) + (x[2] + x[3])) * 0.25;
  cy = ((y[0] + y[1]) + (y[2] + y[3])) * 0.25;
  double d = 0.0;
  for (int k = 0; k < 4; k++) d += sqrt((x[k] - cx) * (x[k] - cx) + (y[k] - cy) * (y[k] - cy));
  d *= 0.25;
  if (d < 1e-12) return false;
  s = 1.4142135623730951 / d;
  for (int k = 0; k < 4; k++) { u[k] = s * (x[k] - cx); v[k] = s * (y[k] - cy); }
  return true;
}

// Homography through 4 correspondences (the minimal-sample _dlt); false if
// the sample is degenerate or the model is not usable.  Not inlined, so the
// scoring and refit kernels evaluate the very same instructions.
__device__ __noinline__ bool minimal_h(const double2* src, const double2* dst, const int32_t* idx, double* h)
{
  double sx[4], sy[4], dx[4], dy[4];
  for (int k = 0; k < 4; k++) {
    const double2 a = src[idx[k]], b = dst[idx[k]];
    sx[k] = a.x; sy[k] = a.y; dx[k] = b.x; dy[k] = b.y;
  }
  double su[4], sv[4], du[4], dv[4], ss, scx, scy, ds, dcx, dcy;
  if (!cond4(sx, sy, su, sv, ss, scx, scy) || !cond4(dx, dy, du, dv, ds, dcx, dcy)) return false;
  double qs[9], qd[9], adj[9], hn[9];
  square_to_quad(su, sv, qs);
  square_to_quad(du, dv, qd);
  adj[0] = qs[4] * qs[8] - qs[5] * qs[7]; adj[1] = qs[2] * qs[7] - qs[1] * qs[8]; adj[2] = qs[1] * qs[5] - qs[2] * qs[4];
  adj[3] = qs[5] * qs[6] - qs[3] * qs[8]; adj[4] = qs[0] * qs[8] - qs[2] * qs[6]; adj[5] = qs[2] * qs[3] - qs[0] * qs[5];
  adj[6] = qs[3] * qs[7] - qs[4] * qs[6]; adj[7] = qs[1] * qs[6] - qs[0] * qs[7]; adj[8] = qs[0] * qs[4] - qs[1] * qs[3];
  mat3mul(qd, adj, hn);
  // h = inv(T_d) hn T_s (matching.py:131)
  const double ts[9] = {ss, 0.0, -ss * scx, 0.0, ss, -ss * scy, 0.0, 0.0, 1.0};
  const double tdi[9] = {1.0 / ds, 0.0, dcx, 0.0, 1.0 / ds, dcy, 0.0, 0.0, 1.0};
  double t[9];
  mat3mul(hn, ts, t);
  mat3mul(tdi, t, h);
  return finish_usable(h);
}

// project_points + the reprojection test (matching.py:149-156,177-179):
// err = |(h [x y 1])_xy / z - d| with |z| < 1e-12 -> 1e-12, inlier iff err < tol
__device__ __forceinline__ bool reproj_inlier(const double* h, double2 s, double2 d, double tol)
{
  const double px = __fma_rn(s.x, h[0], __fma_rn(s.y, h[1], h[2]));
  const double py = __fma_rn(s.x, h[3], __fma_rn(s.y, h[4], h[5]));
  double z = __fma_rn(s.x, h[6], __fma_rn(s.y, h[7], h[8]));
  z = fabs(z) < 1e-12 ? 1e-12 : z;
  const double ex = __dsub_rn(__ddiv_rn(px, z), d.x), ey = __dsub_rn(__ddiv_rn(py, z), d.y);
  return __dsqrt_rn(__fma_rn(ex, ex, __dmul_rn(ey, ey))) < tol;
}

struct RsProb {
  const int64_t* off;      // [P + 1] point offsets
  const double2* src;      // query points
  const double2* dst;      // reference points
  int32_t* table;          // [P][iters][4] minimal samples
  unsigned long long* best;  // [P] (count << 32) | ~iteration
  int32_t* first_rej;      // [P] first iteration whose draws rejected
  int P, iters;
  uint64_t seed;
  double tol;
};

__global__ void k_rs_samples(RsProb q)
{
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)q.P * q.iters) return;
  const int p = (int)(t / q.iters), k = (int)(t - (long long)p * q.iters);
  const int64_t n = q.off[p + 1] - q.off[p];
  if (n < 4) return;
  vfr::Pcg g = vfr::pcg_seed(q.seed);
  vfr::seek32(g, (uint64_t)k * vfr::words_per_choice(n));
  if (vfr::choice4(g, (uint32_t)n, q.table + ((long long)p * q.iters + k) * 4)) atomicMin(q.first_rej + p, k);
}

__global__ void k_rs_fixup(RsProb q)
{
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= q.P) return;
  const int k0 = q.first_rej[p];
  if (k0 >= q.iters) return;
  const int64_t n = q.off[p + 1] - q.off[p];
  vfr::Pcg g = vfr::pcg_seed(q.seed);
  vfr::seek32(g, (uint64_t)k0 * vfr::words_per_choice(n));
  for (int k = k0; k < q.iters; k++) vfr::choice4(g, (uint32_t)n, q.table + ((long long)p * q.iters + k) * 4);
}

__global__ void __launch_bounds__(RS_THREADS) k_rs_score(RsProb q)
{
  __shared__ __align__(16) double hs[RS_HB][10];
  __shared__ int cnt[RS_HB];
  __shared__ unsigned vm32[2];
  const int p = blockIdx.y, k0 = blockIdx.x * RS_HB;
  const int64_t base = q.off[p], n = q.off[p + 1] - base;
  if (n < 4 || k0 >= q.iters) return;
  const double2* src = q.src + base;
  const double2* dst = q.dst + base;
  const int tid = threadIdx.x, lane = tid & 31;
  if (tid < RS_HB) {   // warps 0 and 1: one minimal model each
    const int k = k0 + tid;
    bool ok = false;
    cnt[tid] = 0;
    if (k < q.iters) ok = minimal_h(src, dst, q.table + ((long long)p * q.iters + k) * 4, hs[tid]);
    const unsigned b = __ballot_sync(0xffffffffu, ok);
    if (lane == 0) vm32[tid >> 5] = b;
  }
  __syncthreads();
  const unsigned long long vm = (unsigned long long)vm32[0] | ((unsigned long long)vm32[1] << 32);
  int c0 = 0, c1 = 0;
  for (int64_t i0 = 0; i0 < n; i0 += RS_THREADS) {
    const int64_t i = i0 + tid;
    const bool in = i < n;
    const double2 s = in ? src[i] : make_double2(0.0, 0.0), d = in ? dst[i] : make_double2(0.0, 0.0);
    for (unsigned long long m = vm; m; m &= m - 1) {
      const int h = __ffsll((long long)m) - 1;
      const unsigned b = __ballot_sync(0xffffffffu, in && reproj_inlier(hs[h], s, d, q.tol));
      if (lane == (h & 31)) {
        if (h < 32) c0 += __popc(b);
        else c1 += __popc(b);
      }
    }
  }
  atomicAdd(&cnt[lane], c0);
  atomicAdd(&cnt[lane + 32], c1);
  __syncthreads();
  if (tid < RS_HB) {
    const int k = k0 + tid, c = cnt[tid];
    unsigned long long key = ((vm >> tid) & 1ull) && c > 0 ? ((unsigned long long)c << 32) | (0xffffffffu - (unsigned)k) : 0ull;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const unsigned long long other = __shfl_xor_sync(0xffffffffu, key, o);
      key = other > key ? other : key;
    }
    if (lane == 0 && key) atomicMax(q.best + p, key);
  }
}

// block-wide sum of NV doubles per thread (RS_THREADS threads)
template <int NV>
__device__ void block_sum(double* v, double* red /* [RS_THREADS / 32][NV] */)
{
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < NV; j++) {
    double x = v[j];
#pragma unroll
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    v[j] = x;
  }
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int j = 0; j < NV; j++) red[wid * NV + j] = v[j];
  __syncthreads();
#pragma unroll
  for (int j = 0; j < NV; j++) {
    double x = 0.0;
    for (int w = 0; w < RS_THREADS / 32; w++) x += red[w * NV + j];
    v[j] = x;
  }
  __syncthreads();
}

// least eigenvector of the symmetric 9x9 A (cyclic Jacobi); A destroyed
__device__ void least_eigvec9(double (*A)[9], double* out)
{
  double V[9][9];
  for (int i = 0; i < 9; i++)
    for (int j = 0; j < 9; j++) V[i][j] = i == j ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 60; sweep++) {
    double off = 0.0, dia = 0.0;
    for (int p = 0; p < 9; p++) {
      dia += A[p][p] * A[p][p];
      for (int r = p + 1; r < 9; r++) off += A[p][r] * A[p][r];
    }
    if (off <= 1e-34 * dia || off == 0.0) break;
    for (int p = 0; p < 8; p++)
      for (int r = p + 1; r < 9; r++) {
        const double apq = A[p][r];
        if (apq == 0.0) continue;
        const double theta = (A[r][r] - A[p][p]) / (2.0 * apq);
        const double t = copysign(1.0, theta) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < 9; k++) {   // A <- A J
          const double akp = A[k][p], akq = A[k][r];
          A[k][p] = c * akp - s * akq;
          A[k][r] = s * akp + c * akq;
        }
        for (int k = 0; k < 9; k++) {   // A <- J^T A
          const double apk = A[p][k], aqk = A[r][k];
          A[p][k] = c * apk - s * aqk;
          A[r][k] = s * apk + c * aqk;
        }
        for (int k = 0; k < 9; k++) {
          const double vkp = V[k][p], vkq = V[k][r];
          V[k][p] = c * vkp - s * vkq;
          V[k][r] = s * vkp + c * vkq;
        }
      }
  }
  int m = 0;
  for (int i = 1; i < 9; i++)
    if (A[i][i] < A[m][m]) m = i;
  for (int i = 0; i < 9; i++) out[i] = V[i][m];
}

__global__ void __launch_bounds__(RS_THREADS) k_rs_refit(RsProb q, double* H_out, uint8_t* inl_out, int32_t* n_out)
{
  __shared__ double red[RS_THREADS / 32 * 24];
  __shared__ double hsm[9];
  __shared__ double G[9][9];
  __shared__ int ok;
  const int p = blockIdx.x, tid = threadIdx.x;
  const int64_t base = q.off[p], n = q.off[p + 1] - base;
  const double2* src = q.src + base;
  const double2* dst = q.dst + base;
  uint8_t* mask = inl_out + base;
  const unsigned long long key = n >= 4 ? q.best[p] : 0ull;
  const int bc = (int)(key >> 32);
  auto fail = [&]() {
    for (int64_t i = tid; i < n; i += RS_THREADS) mask[i] = 0;
    if (tid < 9) H_out[9 * p + tid] = NAN;
    if (tid == 0) n_out[p] = -1;
  };
  if (bc < 4) { fail(); return; }   // matching.py:183-184
  if (tid == 0) {
    const int kb = (int)(0xffffffffu - (unsigned)(key & 0xffffffffu));
    ok = minimal_h(src, dst, q.table + ((long long)p * q.iters + kb) * 4, hsm);
  }
  __syncthreads();
  double hb[9];
  for (int j = 0; j < 9; j++) hb[j] = hsm[j];
  // consensus set of the best model: centroids (matching.py:98)
  double v[24];
  for (int j = 0; j < 5; j++) v[j] = 0.0;
  for (int64_t i = tid; i < n; i += RS_THREADS) {
    const double2 s = src[i], d = dst[i];
    const bool in = reproj_inlier(hb, s, d, q.tol);
    mask[i] = in;
    if (in) { v[0] += 1.0; v[1] += s.x; v[2] += s.y; v[3] += d.x; v[4] += d.y; }
  }
  block_sum<5>(v, red);
  const double m = v[0];
  const double scx = v[1] / m, scy = v[2] / m, dcx = v[3] / m, dcy = v[4] / m;
  // mean distances (matching.py:99)
  v[0] = v[1] = 0.0;
  for (int64_t i = tid; i < n; i += RS_THREADS)
    if (mask[i]) {
      const double2 s = src[i], d = dst[i];
      v[0] += sqrt((s.x - scx) * (s.x - scx) + (s.y - scy) * (s.y - scy));
      v[1] += sqrt((d.x - dcx) * (d.x - dcx) + (d.y - dcy) * (d.y - dcy));
    }
  block_sum<2>(v, red);
  const double sd_s = v[0] / m, sd_d = v[1] / m;
  if (sd_s < 1e-12 || sd_d < 1e-12) { fail(); return; }   // _normalize_points -> None
  const double ss = 1.4142135623730951 / sd_s, ds = 1.4142135623730951 / sd_d;
  // normal matrix A^T A of the DLT rows (matching.py:114-119): with
  // s = (u, v, 1) and d = (a, b), it is built from sum w * s s^T for
  // w in {1, a, b, a^2 + b^2} (4 x 6 distinct sums)
  for (int j = 0; j < 24; j++) v[j] = 0.0;
  for (int64_t i = tid; i < n; i += RS_THREADS)
    if (mask[i]) {
      const double2 s = src[i], d = dst[i];
      const double u = ss * s.x - ss * scx, w = ss * s.y - ss * scy;
      const double a = ds * d.x - ds * dcx, b = ds * d.y - ds * dcy;
      const double ssT[6] = {u * u, u * w, u, w * w, w, 1.0};
      const double wt[4] = {1.0, a, b, a * a + b * b};
#pragma unroll
      for (int c = 0; c < 4; c++)
#pragma unroll
        for (int e = 0; e < 6; e++) v[6 * c + e] += wt[c] * ssT[e];
    }
  block_sum<24>(v, red);
  if (tid == 0) {
    auto S = [&](int c, int i, int j) {   // (sum w_c s s^T)[i][j]
      const int lo = i < j ? i : j, hi = i < j ? j : i;
      const int e = lo == 0 ? hi : (lo == 1 ? 2 + hi : 5);
      return v[6 * c + e];
    };
    for (int i = 0; i < 9; i++)
      for (int j = 0; j < 9; j++) G[i][j] = 0.0;
    for (int i = 0; i < 3; i++)
      for (int j = 0; j < 3; j++) {
        G[i][j] = G[3 + i][3 + j] = S(0, i, j);
        G[i][6 + j] = G[6 + j][i] = -S(1, i, j);
        G[3 + i][6 + j] = G[6 + j][3 + i] = -S(2, i, j);
        G[6 + i][6 + j] = S(3, i, j);
      }
    double hn[9], t[9], h[9];
    least_eigvec9(G, hn);
    const double ts[9] = {ss, 0.0, -ss * scx, 0.0, ss, -ss * scy, 0.0, 0.0, 1.0};
    const double tdi[9] = {1.0 / ds, 0.0, dcx, 0.0, 1.0 / ds, dcy, 0.0, 0.0, 1.0};
    mat3mul(hn, ts, t);
    mat3mul(tdi, t, h);
    ok = finish_usable(h);
    for (int j = 0; j < 9; j++) hsm[j] = h[j];
  }
  __syncthreads();
  if (!ok) { fail(); return; }
  for (int j = 0; j < 9; j++) hb[j] = hsm[j];
  int c = 0;
  for (int64_t i = tid; i < n; i += RS_THREADS) {
    const bool in = reproj_inlier(hb, src[i], dst[i], q.tol);
    mask[i] = in;
    c += in;
  }
  c = __reduce_add_sync(0xffffffffu, c);
  __shared__ int csum;
  if (tid == 0) csum = 0;
  __syncthreads();
  if ((tid & 31) == 0) atomicAdd(&csum, c);
  __syncthreads();
  if (tid < 9) H_out[9 * p + tid] = hb[tid];
  if (tid == 0) n_out[p] = csum;
}

__global__ void k_rs_init(int P, unsigned long long* best, int32_t* first_rej, int iters)
{
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < P) { best[p] = 0ull; first_rej[p] = iters; }
}

int rs_scratch(int P, int iters, const int64_t* off_host, cudaStream_t st, void** mem, RsProb& q)
{
  const size_t o_off = 0, o_best = ((size_t)(P + 1) * 8 + 255) & ~(size_t)255;
  const size_t o_rej = o_best + (((size_t)P * 8 + 255) & ~(size_t)255);
  const size_t o_tab = o_rej + (((size_t)P * 4 + 255) & ~(size_t)255);
  const size_t bytes = o_tab + (size_t)P * iters * 16 + 16;
  char* m = nullptr;
  if (cudaMallocAsync((void**)&m, bytes, st) != cudaSuccess) return VF_ERR_CUDA;
  if (cudaMemcpyAsync(m + o_off, off_host, (size_t)(P + 1) * 8, cudaMemcpyHostToDevice, st) != cudaSuccess) {
    cudaFreeAsync(m, st);
    return VF_ERR_CUDA;
  }
  q.off = reinterpret_cast<const int64_t*>(m + o_off);
  q.best = reinterpret_cast<unsigned long long*>(m + o_best);
  q.first_rej = reinterpret_cast<int32_t*>(m + o_rej);
  q.table = reinterpret_cast<int32_t*>(m + o_tab);
  *mem = m;
  return VF_OK;
}

void rs_samples(const RsProb& q, cudaStream_t st)
{
  k_rs_init<<<(q.P + 255) / 256, 256, 0, st>>>(q.P, q.best, q.first_rej, q.iters);
  const long long nt = (long long)q.P * q.iters;
  if (nt > 0) k_rs_samples<<<(unsigned)((nt + 255) / 256), 256, 0, st>>>(q);
  k_rs_fixup<<<(q.P + 127) / 128, 128, 0, st>>>(q);
}

bool offsets_ok(int P, const int64_t* off)
{
  if (off[0] != 0) return false;
  for (int p = 0; p < P; p++)
    if (off[p + 1] < off[p] || off[p + 1] - off[p] > INT32_MAX) return false;
  return true;
}

}  // namespace

extern "C" int vf_ransac_homography(int n_problems, const int64_t* offsets, const double* src_dev,
                                    const double* dst_dev, int iters, double reproj_tol, uint64_t seed, double* H_dev,
                                    uint8_t* inlier_dev, int32_t* n_inliers_dev, void* stream)
{
  if (n_problems < 0 || iters < 0 || !offsets) return VF_ERR_ARG;
  if (n_problems == 0) return VF_OK;
  if (n_problems > 65535 || !offsets_ok(n_problems, offsets) || !H_dev || !n_inliers_dev) return VF_ERR_ARG;
  if (offsets[n_problems] > 0 && (!src_dev || !dst_dev || !inlier_dev)) return VF_ERR_ARG;
  if (((uintptr_t)src_dev | (uintptr_t)dst_dev) & 15) return VF_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  RsProb q;
  void* mem = nullptr;
  const int rc = rs_scratch(n_problems, iters, offsets, st, &mem, q);
  if (rc != VF_OK) return rc;
  q.src = reinterpret_cast<const double2*>(src_dev);
  q.dst = reinterpret_cast<const double2*>(dst_dev);
  q.P = n_problems;
  q.iters = iters;
  q.seed = seed;
  q.tol = reproj_tol;
  rs_samples(q, st);
  if (iters > 0) k_rs_score<<<dim3((unsigned)((iters + RS_HB - 1) / RS_HB), (unsigned)n_problems), RS_THREADS, 0, st>>>(q);
  k_rs_refit<<<n_problems, RS_THREADS, 0, st>>>(q, H_dev, inlier_dev, n_inliers_dev);
  cudaFreeAsync(mem, st);
  return cudaGetLastError() == cudaSuccess ? VF_OK : VF_ERR_CUDA;
}

extern "C" int vf_ransac_samples(uint64_t seed, int64_t n, int iters, int32_t* out_dev, void* stream)
{
  if (n < 4 || n > INT32_MAX || iters < 0 || (iters > 0 && !out_dev)) return VF_ERR_ARG;
  if (iters == 0) return VF_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t off[2] = {0, n};
  RsProb q;
  void* mem = nullptr;
  const int rc = rs_scratch(1, iters, off, st, &mem, q);
  if (rc != VF_OK) return rc;
  q.P = 1;
  q.iters = iters;
  q.seed = seed;
  rs_samples(q, st);
  cudaMemcpyAsync(out_dev, q.table, (size_t)iters * 16, cudaMemcpyDeviceToDevice, st);
  cudaFreeAsync(mem, st);
  return cudaGetLastError() == cudaSuccess ? VF_OK : VF_ERR_CUDA;
}

extern "C" int vf_ransac_samples_host(uint64_t seed, int64_t n, int iters, int32_t* out)
{
  if (n < 4 || n > INT32_MAX || iters < 0 || (iters > 0 && !out)) return VF_ERR_ARG;
  vfr::Pcg g = vfr::pcg_seed(seed);
  for (int k = 0; k < iters; k++) vfr::choice4(g, (uint32_t)n, out + 4 * (int64_t)k);
  return VF_OK;
}
