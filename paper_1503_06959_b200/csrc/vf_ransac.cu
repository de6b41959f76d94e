// vf_ransac.cu -- batched geometric verification on the GPU (SURVEY.md 8(f)
// rank 4): ransac_homography (/root/reference/pkg/src/vidfeat/matching.py:
// 151-192) for many match sets in one call, as count_mpr / locate_object
// (matching.py:209-220, evaluation.py:95-121) consume it.
//
// Per call (all problems at once, on `stream`):
//   k_rs_samples   thread per (problem, iteration): the reference's minimal
//                  samples, rng.choice(n, 4, replace=False) of
//                  default_rng(seed), by PCG64 jump-ahead (vf_rng.cuh)
//   k_rs_fixup     thread per problem: iterations after a (rare) Lemire
//                  rejection regenerated sequentially
//   k_rs_score     CTA per (problem, 64 iterations, 4096-point chunk): 64
//                  minimal homographies solved into shared memory, then every
//                  point of the chunk scored against all 64 (thread per point,
//                  ballot + popc counts), counts added per iteration
//   refit          k_rs_best (CTA per problem: the best iteration, max count /
//                  first index, and its model), then grid-wide passes over
//                  4096-point chunks with per-chunk partials summed in chunk
//                  order (bitwise reproducible): k_rs_pass<0> consensus set +
//                  centroids, <1> mean distances, <2> the 9x9 normal matrix of
//                  the normalized DLT (matching.py:109-137); k_rs_solve (warp
//                  per problem: least eigenvector by inverse iteration,
//                  de-normalize, the
//                  usable test, matching.py:140-146); k_rs_pass<3> final
//                  inlier mask + counts; k_rs_out (matching.py:187-192)
// Minimal models: for 4 points the normalized DLT's null vector is the
// homography through the 4 correspondences; it is computed in closed form
// (unit square -> quad maps, H = Q_dst adj(Q_src)) on centred, scaled
// coordinates and normalized by h22 as _dlt does.  Float results differ from
// numpy's LAPACK path by rounding only (parity tolerance in tests/).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>

#include "../../include/vidfeat_b200.h"
#include "vf_rng.cuh"

namespace {

constexpr int RS_HB = 64;        // hypotheses per scoring CTA
constexpr int RS_PCH = 4096;     // points per scoring CTA
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

// The same decision without the divisions and the square root, when it is
// clear: with z the (unclamped) denominator, err < tol <=> |p - d z|^2 <
// tol^2 z^2.  Taken only when both sides differ by more than 1e-6 relative
// (fp64 rounding of either form is ~1e-13 here), z is not near its clamp or
// cancelling, and the coordinates are below 1e7 (`plain`); every other case
// -- and any NaN -- goes to the exact reference form above.  So each
// decision equals reproj_inlier's.
__device__ __forceinline__ bool reproj_inlier_fast(const double* h, double2 s, double2 d, double tol, double tol2,
                                                   bool plain)
{
  if (plain) {
    const double px = __fma_rn(s.x, h[0], __fma_rn(s.y, h[1], h[2]));
    const double py = __fma_rn(s.x, h[3], __fma_rn(s.y, h[4], h[5]));
    const double z = __fma_rn(s.x, h[6], __fma_rn(s.y, h[7], h[8]));
    const double zb = __fma_rn(fabs(s.x), fabs(h[6]), __fma_rn(fabs(s.y), fabs(h[7]), fabs(h[8])));
    if (fabs(z) > 1e-6 * zb && fabs(z) >= 1e-9) {
      const double ex = __fma_rn(-d.x, z, px), ey = __fma_rn(-d.y, z, py);
      const double e = __fma_rn(ex, ex, __dmul_rn(ey, ey)), t = __dmul_rn(tol2, __dmul_rn(z, z));
      if (e < t * (1.0 - 1e-6)) return true;
      if (e > t * (1.0 + 1e-6)) return false;
    }
  }
  return reproj_inlier(h, s, d, tol);
}

__device__ __forceinline__ bool plain_point(double2 s, double2 d)
{
  return fmax(fmax(fabs(s.x), fabs(s.y)), fmax(fabs(d.x), fabs(d.y))) < 1e7;
}

struct RsProb {
  const int64_t* off;      // [P + 1] point offsets
  const double2* src;      // query points
  const double2* dst;      // reference points
  int32_t* table;          // [P][iters][4] minimal samples
  int32_t* cnt;            // [P][iters] inlier count per iteration (0 if not usable)
  int32_t* first_rej;      // [P] first iteration whose draws rejected
  int P, iters, chunks;    // chunks: point chunks of the largest problem
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

constexpr int RS_PPT = 4;   // points per thread per hypothesis in k_rs_score

static_assert(RS_HB * 4 == RS_THREADS, "one model per 4 threads");
__global__ void __launch_bounds__(RS_THREADS, 2) k_rs_score(RsProb q)
{
  __shared__ __align__(16) double hs[RS_HB][12];
  __shared__ int cnt[RS_HB];
  __shared__ int vlist[RS_HB];
  __shared__ int nvalid;
  const int p = blockIdx.y, kb = blockIdx.x / q.chunks, ch = blockIdx.x - kb * q.chunks, k0 = kb * RS_HB;
  const int64_t base = q.off[p], n = q.off[p + 1] - base;
  const int64_t c_lo = (int64_t)ch * RS_PCH, c_hi = min(n, c_lo + RS_PCH);
  if (n < 4 || k0 >= q.iters || c_lo >= n) return;
  const double2* src = q.src + base;
  const double2* dst = q.dst + base;
  const int tid = threadIdx.x, lane = tid & 31;
  __shared__ unsigned vb[RS_THREADS / 32];
  // model h is solved by thread 4 h (8 lanes in each of the 8 warps)
  const int hm = tid >> 2;
  const bool solver = (tid & 3) == 0;
  bool ok = false;
  if (tid < RS_HB) cnt[tid] = 0;
  if (solver) {
    const int k = k0 + hm;
    if (k < q.iters) ok = minimal_h(src, dst, q.table + ((long long)p * q.iters + k) * 4, hs[hm]);
    if (ok) {   // z-guard coefficients (see the point loop)
      hs[hm][9] = 1e-6 * (fabs(hs[hm][6]) + fabs(hs[hm][7]));
      hs[hm][10] = 1e-6 * fabs(hs[hm][8]);
      hs[hm][11] = 0.0;
    }
  }
  const unsigned b = __ballot_sync(0xffffffffu, ok);
  if (lane == 0) vb[tid >> 5] = b;
  __syncthreads();
  if (ok) {   // compacted list of the usable models, in model order
    int before = __popc(b & ((1u << lane) - 1));
    for (int w = 0; w < (tid >> 5); w++) before += __popc(vb[w]);
    vlist[before] = hm;
  }
  if (tid == 0) {
    int t = 0;
    for (int w = 0; w < RS_THREADS / 32; w++) t += __popc(vb[w]);
    nvalid = t;
  }
  __syncthreads();
  const int nv = nvalid;
  // Decisions without division / square root (as reproj_inlier_fast): with
  // z unclamped, err < tol <=> |p - d z|^2 < tol^2 z^2, taken when the two
  // sides differ by > 1e-6 relative and |z| > zt = 1e-6 ((|h6| + |h7|) B +
  // |h8|) (>= 1e-6 (|h6 x| + |h7 y| + |h8|) for the thread's points, |x|, |y|
  // <= B: no cancellation in z) and > 1e-9 (far from the clamp); all else,
  // and coordinates >= 1e7, by the exact form.
  const bool fast = q.tol > 0.0;
  const double tlo = q.tol * q.tol * (1.0 - 1e-6), thi = q.tol * q.tol * (1.0 + 1e-6);
  int c0 = 0, c1 = 0;
  for (int64_t i0 = c_lo; i0 < c_hi; i0 += RS_THREADS * RS_PPT) {
    double2 s[RS_PPT], d[RS_PPT];
    unsigned live = 0, plain = 0;
    double bnd = 0.0;
#pragma unroll
    for (int u = 0; u < RS_PPT; u++) {
      const int64_t i = i0 + tid + u * RS_THREADS;
      const bool in = i < c_hi;
      s[u] = in ? src[i] : make_double2(0.0, 0.0);
      d[u] = in ? dst[i] : make_double2(0.0, 0.0);
      live |= (unsigned)in << u;
      const bool pl = in && fast && plain_point(s[u], d[u]);
      plain |= (unsigned)pl << u;
      if (pl) bnd = fmax(bnd, fmax(fabs(s[u].x), fabs(s[u].y)));
    }
    for (int j = 0; j < nv; j++) {
      const int h = vlist[j];
      double hv[12];
#pragma unroll
      for (int e = 0; e < 12; e += 2) {
        const double2 w = *reinterpret_cast<const double2*>(&hs[h][e]);
        hv[e] = w.x;
        hv[e + 1] = w.y;
      }
      double zt = __fma_rn(hv[9], bnd, hv[10]);
      zt = zt > 1e-9 ? zt : 1e-9;
      int c = 0;
      unsigned dec = 0;
#pragma unroll
      for (int u = 0; u < RS_PPT; u++) {
        const double px = __fma_rn(s[u].x, hv[0], __fma_rn(s[u].y, hv[1], hv[2]));
        const double py = __fma_rn(s[u].x, hv[3], __fma_rn(s[u].y, hv[4], hv[5]));
        const double z = __fma_rn(s[u].x, hv[6], __fma_rn(s[u].y, hv[7], hv[8]));
        const double ex = __fma_rn(-d[u].x, z, px), ey = __fma_rn(-d[u].y, z, py);
        const double e = __fma_rn(ex, ex, __dmul_rn(ey, ey)), z2 = __dmul_rn(z, z);
        const bool zok = fabs(z) > zt;
        const bool inl = zok && e < tlo * z2, outl = zok && e > thi * z2;
        const bool pl = (plain >> u) & 1;
        c += inl && pl;
        dec |= (unsigned)((inl || outl) && pl) << u;
      }
      const unsigned und = live & ~dec;
      if (__any_sync(0xffffffffu, und != 0)) {   // rare: the exact reference form
#pragma unroll
        for (int u = 0; u < RS_PPT; u++)
          if ((und >> u) & 1) c += reproj_inlier(hv, s[u], d[u], q.tol);
      }
      const int tot = __reduce_add_sync(0xffffffffu, c);
      if (lane == (h & 31)) {
        if (h < 32) c0 += tot;
        else c1 += tot;
      }
    }
  }
  atomicAdd(&cnt[lane], c0);
  atomicAdd(&cnt[lane + 32], c1);
  __syncthreads();
  if (tid < RS_HB && cnt[tid] > 0) atomicAdd(q.cnt + (long long)p * q.iters + k0 + tid, cnt[tid]);
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

// Least eigenvector of the symmetric positive semi-definite 9x9 G by inverse
// iteration on G + mu I (mu = 1e-12 trace keeps the Cholesky factor real
// under rounding; the shift does not move eigenvectors), started from x0
// (the best minimal model in the same coordinates).  Iterates until the
// unit iterate changes by < 1e-15 (the accuracy limit eps ||G|| / gap of any
// method on G); false if G is zero or not finite.  One thread, registers.
__device__ bool least_eigvec9(const double (*G)[9], const double* x0, double* out)
{
  double L[9][9];
  double tr = 0.0;
#pragma unroll
  for (int i = 0; i < 9; i++) tr += G[i][i];
  if (!(tr > 0.0) || !isfinite(tr)) return false;
  const double mu = 1e-12 * tr;
#pragma unroll
  for (int i = 0; i < 9; i++)
#pragma unroll
    for (int j = 0; j <= i; j++) {
      double s = G[i][j] + (i == j ? mu : 0.0);
#pragma unroll
      for (int k = 0; k < j; k++) s -= L[i][k] * L[j][k];
      if (i == j) L[i][i] = sqrt(s > 0.0 ? s : mu);
      else L[i][j] = s / L[j][j];
    }
  double x[9], n0 = 0.0;
#pragma unroll
  for (int i = 0; i < 9; i++) n0 += x0[i] * x0[i];
  n0 = n0 > 0.0 && isfinite(n0) ? 1.0 / sqrt(n0) : 0.0;
#pragma unroll
  for (int i = 0; i < 9; i++) x[i] = n0 > 0.0 ? x0[i] * n0 : 1.0 / 3.0;
  for (int it = 0; it < 300; it++) {
    double z[9], y[9];
#pragma unroll
    for (int i = 0; i < 9; i++) {   // L z = x
      double s = x[i];
#pragma unroll
      for (int k = 0; k < i; k++) s -= L[i][k] * z[k];
      z[i] = s / L[i][i];
    }
#pragma unroll
    for (int i = 8; i >= 0; i--) {   // L^T y = z
      double s = z[i];
#pragma unroll
      for (int k = i + 1; k < 9; k++) s -= L[k][i] * y[k];
      y[i] = s / L[i][i];
    }
    double nrm = 0.0, dot = 0.0;
#pragma unroll
    for (int i = 0; i < 9; i++) { nrm += y[i] * y[i]; dot += y[i] * x[i]; }
    const double inv = (dot < 0.0 ? -1.0 : 1.0) / sqrt(nrm);
    double diff = 0.0;
#pragma unroll
    for (int i = 0; i < 9; i++) {
      const double v = y[i] * inv;
      diff = fmax(diff, fabs(v - x[i]));
      x[i] = v;
    }
    if (!(diff >= 1e-15) && it > 0) break;
  }
#pragma unroll
  for (int i = 0; i < 9; i++) out[i] = x[i];
  return true;
}

// ---- refit (matching.py:183-192), split into grid-wide passes ------------
// Per problem: status 0 = (None, []), 1 = best model found, 2 = final model.
// Every pass sums the per-chunk partials of the earlier passes in chunk
// order, so results are bitwise reproducible (no floating-point atomics).
constexpr int RS_RCH = 4096;   // points per refit-pass CTA
constexpr int RS_NPART = 32;   // partial slots per (problem, chunk)
//   [0] m  [1..4] sum x, y, dx, dy  [5, 6] sum distances  [7] final count
//   [8..31] normal-matrix sums

struct RsRefit {
  double* part;     // [P][rchunks][RS_NPART]
  double* hbest;    // [P][9]
  double* hfin;     // [P][9]
  int32_t* status;  // [P]
  int rchunks;
};

__global__ void __launch_bounds__(RS_THREADS) k_rs_best(RsProb q, RsRefit r)
{
  __shared__ unsigned long long wkey[RS_THREADS / 32];
  const int p = blockIdx.x, tid = threadIdx.x;
  const int64_t base = q.off[p], n = q.off[p + 1] - base;
  // best iteration: max count, first index (the strict > of matching.py:180)
  unsigned long long key = 0ull;
  if (n >= 4)
    for (int k = tid; k < q.iters; k += RS_THREADS) {
      const int c = q.cnt[(long long)p * q.iters + k];
      const unsigned long long kk = ((unsigned long long)(unsigned)c << 32) | (0xffffffffu - (unsigned)k);
      key = c > 0 && kk > key ? kk : key;
    }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const unsigned long long other = __shfl_xor_sync(0xffffffffu, key, o);
    key = other > key ? other : key;
  }
  if ((tid & 31) == 0) wkey[tid >> 5] = key;
  __syncthreads();
  if (tid == 0) {
    for (int w = 0; w < RS_THREADS / 32; w++) key = wkey[w] > key ? wkey[w] : key;
    int st = 0;
    if ((int)(key >> 32) >= 4) {   // matching.py:183-184
      const int kb = (int)(0xffffffffu - (unsigned)(key & 0xffffffffu));
      st = minimal_h(q.src + base, q.dst + base, q.table + ((long long)p * q.iters + kb) * 4, r.hbest + 9 * p) ? 1 : 0;
    }
    r.status[p] = st;
  }
}

// Sum of NV partial slots over the problem's chunks by one full warp: lane l
// takes chunks l, l + 32, ...; the 32 lane sums are then added in lane order
// by every lane, so the result is the same in all lanes and in every run.
template <int NV>
__device__ __forceinline__ void part_sum(const RsRefit& r, int p, int slot, double* out)
{
  const int lane = threadIdx.x & 31;
  double acc[NV];
#pragma unroll
  for (int j = 0; j < NV; j++) acc[j] = 0.0;
  const double* pp = r.part + (long long)p * r.rchunks * RS_NPART + slot;
  for (int c = lane; c < r.rchunks; c += 32)
#pragma unroll
    for (int j = 0; j < NV; j++) acc[j] += pp[(long long)c * RS_NPART + j];
#pragma unroll
  for (int j = 0; j < NV; j++) {
    double t = 0.0;
#pragma unroll
    for (int l = 0; l < 32; l++) t += __shfl_sync(0xffffffffu, acc[j], l);
    out[j] = t;
  }
}

// conditioning of the consensus set from the pass-0 / pass-1 partials
struct RsNorm {
  double m, scx, scy, dcx, dcy, ss, ds;
  bool ok;
};

__device__ __forceinline__ RsNorm rs_norm(const RsRefit& r, int p, bool with_scale)
{
  double v[7];
  part_sum<7>(r, p, 0, v);
  RsNorm o;
  o.m = v[0];
  o.scx = v[1] / o.m; o.scy = v[2] / o.m; o.dcx = v[3] / o.m; o.dcy = v[4] / o.m;
  o.ok = true;
  o.ss = o.ds = 0.0;
  if (with_scale) {
    const double sd_s = v[5] / o.m, sd_d = v[6] / o.m;
    o.ok = !(sd_s < 1e-12 || sd_d < 1e-12);   // _normalize_points -> None (matching.py:100-101)
    o.ss = 1.4142135623730951 / sd_s;
    o.ds = 1.4142135623730951 / sd_d;
  }
  return o;
}

template <int PASS>
__global__ void __launch_bounds__(RS_THREADS) k_rs_pass(RsProb q, RsRefit r, uint8_t* inl_out)
{
  __shared__ double red[RS_THREADS / 32 * 24];
  const int p = blockIdx.y, ch = blockIdx.x, tid = threadIdx.x;
  const int64_t base = q.off[p], n = q.off[p + 1] - base;
  const int64_t lo = (int64_t)ch * RS_RCH, hi = min(n, lo + RS_RCH);
  if (lo >= n) return;
  const double2* src = q.src + base;
  const double2* dst = q.dst + base;
  uint8_t* mask = inl_out + base;
  const int st = r.status[p];
  double* out = r.part + ((long long)p * r.rchunks + ch) * RS_NPART;
  const double tol2 = q.tol * q.tol;
  const bool fast = q.tol > 0.0;
  if (PASS == 3) {   // final inliers (matching.py:190-192)
    int c = 0;
    double h[9];
    for (int j = 0; j < 9; j++) h[j] = st == 2 ? r.hfin[9 * p + j] : 0.0;
    for (int64_t i = lo + tid; i < hi; i += RS_THREADS) {
      bool in = false;
      if (st == 2) {
        const double2 s = src[i], d = dst[i];
        in = reproj_inlier_fast(h, s, d, q.tol, tol2, fast && plain_point(s, d));
      }
      mask[i] = in;
      c += in;
    }
    double v[1] = {(double)c};
    block_sum<1>(v, red);
    if (tid == 0) out[7] = v[0];
    return;
  }
  if (st != 1) return;
  if (PASS == 0) {   // consensus set of the best model + centroid sums (matching.py:98,177-182)
    double h[9], v[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    for (int j = 0; j < 9; j++) h[j] = r.hbest[9 * p + j];
    for (int64_t i = lo + tid; i < hi; i += RS_THREADS) {
      const double2 s = src[i], d = dst[i];
      const bool in = reproj_inlier_fast(h, s, d, q.tol, tol2, fast && plain_point(s, d));
      mask[i] = in;
      if (in) { v[0] += 1.0; v[1] += s.x; v[2] += s.y; v[3] += d.x; v[4] += d.y; }
    }
    block_sum<5>(v, red);
    if (tid < 5) out[tid] = v[tid];
  } else if (PASS == 1) {   // mean distances to the centroids (matching.py:99)
    const RsNorm nm = rs_norm(r, p, false);
    double v[2] = {0.0, 0.0};
    for (int64_t i = lo + tid; i < hi; i += RS_THREADS)
      if (mask[i]) {
        const double2 s = src[i], d = dst[i];
        v[0] += sqrt((s.x - nm.scx) * (s.x - nm.scx) + (s.y - nm.scy) * (s.y - nm.scy));
        v[1] += sqrt((d.x - nm.dcx) * (d.x - nm.dcx) + (d.y - nm.dcy) * (d.y - nm.dcy));
      }
    block_sum<2>(v, red);
    if (tid < 2) out[5 + tid] = v[tid];
  } else {   // PASS 2: normal matrix A^T A of the DLT rows (matching.py:114-119)
    const RsNorm nm = rs_norm(r, p, true);
    // with s = (u, v, 1) and d = (a, b): sums of w s s^T, w in {1, a, b, a^2 + b^2}
    double v[24];
    for (int j = 0; j < 24; j++) v[j] = 0.0;
    if (nm.ok)
      for (int64_t i = lo + tid; i < hi; i += RS_THREADS)
        if (mask[i]) {
          const double2 s = src[i], d = dst[i];
          const double u = nm.ss * s.x - nm.ss * nm.scx, w = nm.ss * s.y - nm.ss * nm.scy;
          const double a = nm.ds * d.x - nm.ds * nm.dcx, b = nm.ds * d.y - nm.ds * nm.dcy;
          const double ssT[6] = {u * u, u * w, u, w * w, w, 1.0};
          const double wt[4] = {1.0, a, b, a * a + b * b};
#pragma unroll
          for (int c = 0; c < 4; c++)
#pragma unroll
            for (int e = 0; e < 6; e++) v[6 * c + e] += wt[c] * ssT[e];
        }
    block_sum<24>(v, red);
    if (tid < 24) out[8 + tid] = v[tid];
  }
}

// warp per problem: assemble A^T A, least eigenvector (inverse iteration),
// de-normalize, _usable
__global__ void __launch_bounds__(32) k_rs_solve(RsProb q, RsRefit r)
{
  __shared__ double G[9][9];
  const int p = blockIdx.x, lane = threadIdx.x;
  if (r.status[p] != 1) return;
  const RsNorm nm = rs_norm(r, p, true);
  if (!nm.ok) {
    if (lane == 0) r.status[p] = 0;
    return;
  }
  double v[24];
  part_sum<24>(r, p, 8, v);
  auto S = [&](int c, int i, int j) {   // (sum w_c s s^T)[i][j]
    const int lo = i < j ? i : j, hi = i < j ? j : i;
    const int e = lo == 0 ? hi : (lo == 1 ? 2 + hi : 5);
    return v[6 * c + e];
  };
  if (lane < 9) {
    const int i = lane;
    for (int j = 0; j < 9; j++) G[i][j] = 0.0;
    if (i < 3) {
      for (int j = 0; j < 3; j++) { G[i][j] = S(0, i, j); G[i][6 + j] = -S(1, i, j); }
    } else if (i < 6) {
      for (int j = 0; j < 3; j++) { G[i][3 + j] = S(0, i - 3, j); G[i][6 + j] = -S(2, i - 3, j); }
    } else {
      for (int j = 0; j < 3; j++) {
        G[i][j] = -S(1, j, i - 6);
        G[i][3 + j] = -S(2, j, i - 6);
        G[i][6 + j] = S(3, i - 6, j);
      }
    }
  }
  __syncwarp();
  if (lane == 0) {
    double h[9], t[9], hh[9], x0[9];
    {   // warm start: T_d H_best T_s^-1
      const double* hb = r.hbest + 9 * p;
      const double tsi[9] = {1.0 / nm.ss, 0.0, nm.scx, 0.0, 1.0 / nm.ss, nm.scy, 0.0, 0.0, 1.0};
      const double td[9] = {nm.ds, 0.0, -nm.ds * nm.dcx, 0.0, nm.ds, -nm.ds * nm.dcy, 0.0, 0.0, 1.0};
      double hb9[9];
      for (int j = 0; j < 9; j++) hb9[j] = hb[j];
      mat3mul(hb9, tsi, t);
      mat3mul(td, t, x0);
    }
    const bool eig = least_eigvec9(G, x0, hh);
    const double ts[9] = {nm.ss, 0.0, -nm.ss * nm.scx, 0.0, nm.ss, -nm.ss * nm.scy, 0.0, 0.0, 1.0};
    const double tdi[9] = {1.0 / nm.ds, 0.0, nm.dcx, 0.0, 1.0 / nm.ds, nm.dcy, 0.0, 0.0, 1.0};
    mat3mul(hh, ts, t);
    mat3mul(tdi, t, h);
    const bool ok = eig && finish_usable(h);
    for (int j = 0; j < 9; j++) r.hfin[9 * p + j] = h[j];
    r.status[p] = ok ? 2 : 0;
  }
}

__global__ void __launch_bounds__(32) k_rs_out(RsRefit r, double* H_out, int32_t* n_out)
{
  const int p = blockIdx.x, lane = threadIdx.x;
  if (r.status[p] != 2) {
    if (lane < 9) H_out[9 * p + lane] = NAN;
    if (lane == 0) n_out[p] = -1;
    return;
  }
  double c[1];
  part_sum<1>(r, p, 7, c);
  if (lane < 9) H_out[9 * p + lane] = r.hfin[9 * p + lane];
  if (lane == 0) n_out[p] = (int32_t)c[0];
}

__global__ void k_rs_init(int P, int32_t* first_rej, int iters)
{
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < P) first_rej[p] = iters;
}

// Stream-ordered scratch from a private pool that keeps its memory (release
// threshold = max), so repeated calls reuse it without remapping.
cudaMemPool_t rs_pool()
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

int rs_scratch(int P, int iters, const int64_t* off_host, cudaStream_t st, void** mem, RsProb& q, RsRefit* rf = nullptr,
               int rchunks = 0)
{
  const size_t o_off = 0, o_cnt = ((size_t)(P + 1) * 8 + 255) & ~(size_t)255;
  const size_t o_rej = o_cnt + (((size_t)P * iters * 4 + 255) & ~(size_t)255);
  const size_t o_tab = o_rej + (((size_t)P * 4 + 255) & ~(size_t)255);
  const size_t o_part = o_tab + (((size_t)P * iters * 16 + 255) & ~(size_t)255);
  const size_t o_hb = o_part + (size_t)P * rchunks * RS_NPART * 8;
  const size_t o_hf = o_hb + (size_t)P * 9 * 8, o_st = o_hf + (size_t)P * 9 * 8;
  const size_t bytes = o_st + (size_t)P * 4 + 16;
  char* m = nullptr;
  cudaMemPool_t pool = rs_pool();
  if (!pool || cudaMallocFromPoolAsync((void**)&m, bytes, pool, st) != cudaSuccess) return VF_ERR_CUDA;
  if (cudaMemcpyAsync(m + o_off, off_host, (size_t)(P + 1) * 8, cudaMemcpyHostToDevice, st) != cudaSuccess) {
    cudaFreeAsync(m, st);
    return VF_ERR_CUDA;
  }
  q.off = reinterpret_cast<const int64_t*>(m + o_off);
  q.cnt = reinterpret_cast<int32_t*>(m + o_cnt);
  if (cudaMemsetAsync(m + o_cnt, 0, (size_t)P * iters * 4, st) != cudaSuccess) {
    cudaFreeAsync(m, st);
    return VF_ERR_CUDA;
  }
  q.first_rej = reinterpret_cast<int32_t*>(m + o_rej);
  q.table = reinterpret_cast<int32_t*>(m + o_tab);
  if (rf) {
    rf->part = reinterpret_cast<double*>(m + o_part);
    rf->hbest = reinterpret_cast<double*>(m + o_hb);
    rf->hfin = reinterpret_cast<double*>(m + o_hf);
    rf->status = reinterpret_cast<int32_t*>(m + o_st);
    rf->rchunks = rchunks;
  }
  *mem = m;
  return VF_OK;
}

void rs_samples(const RsProb& q, cudaStream_t st)
{
  k_rs_init<<<(q.P + 255) / 256, 256, 0, st>>>(q.P, q.first_rej, q.iters);
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
  int64_t n_max = 0;
  for (int p = 0; p < n_problems; p++) n_max = std::max(n_max, offsets[p + 1] - offsets[p]);
  const int rchunks = (int)std::max<int64_t>(1, (n_max + RS_RCH - 1) / RS_RCH);
  RsProb q;
  RsRefit rf;
  void* mem = nullptr;
  const int rc = rs_scratch(n_problems, iters, offsets, st, &mem, q, &rf, rchunks);
  if (rc != VF_OK) return rc;
  q.src = reinterpret_cast<const double2*>(src_dev);
  q.dst = reinterpret_cast<const double2*>(dst_dev);
  q.P = n_problems;
  q.iters = iters;
  q.seed = seed;
  q.tol = reproj_tol;
  rs_samples(q, st);
  q.chunks = (int)std::max<int64_t>(1, (n_max + RS_PCH - 1) / RS_PCH);
  const long long gx = (long long)((iters + RS_HB - 1) / RS_HB) * q.chunks;
  if (gx > INT32_MAX) { cudaFreeAsync(mem, st); return VF_ERR_ARG; }
  if (iters > 0) k_rs_score<<<dim3((unsigned)gx, (unsigned)n_problems), RS_THREADS, 0, st>>>(q);
  const dim3 pg((unsigned)rchunks, (unsigned)n_problems);
  k_rs_best<<<n_problems, RS_THREADS, 0, st>>>(q, rf);
  k_rs_pass<0><<<pg, RS_THREADS, 0, st>>>(q, rf, inlier_dev);
  k_rs_pass<1><<<pg, RS_THREADS, 0, st>>>(q, rf, inlier_dev);
  k_rs_pass<2><<<pg, RS_THREADS, 0, st>>>(q, rf, inlier_dev);
  k_rs_solve<<<n_problems, 32, 0, st>>>(q, rf);
  k_rs_pass<3><<<pg, RS_THREADS, 0, st>>>(q, rf, inlier_dev);
  k_rs_out<<<n_problems, 32, 0, st>>>(rf, H_dev, n_inliers_dev);
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
