// vf_temporal.cuh -- temporal block-matching baseline:
// /root/reference/pkg/src/vidfeat/temporal.py (spiral_search :183-226,
// baseline_step :229-308) and pipeline.py:281-345 (_run_temporal).
//
// Off GOP starts every previous feature is chased into the current frame by a
// two-stage spiral SAD search of its patch x patch block.  One warp per
// feature, lanes = search offsets:
//   * the block and a search window (search radius + refinement margin) are
//     staged in shared memory;
//   * coarse stage: lane k takes spiral offset 32 j + k of round j; integer
//     SADs with the native 4-byte SAD (VABSDIFF4 accumulate) on funnel-shifted
//     window words.  The reference's sequential rule (update on a strictly
//     smaller SAD, stop at the first SAD < t_et) is: the first offset in
//     spiral order with SAD < t_et, else the first offset attaining the
//     minimum -- a ballot per round, then an argmin;
//   * fine stage (quarter-pixel bilinear): when every coarse offset is an
//     integer and every fine offset a multiple of 1/4, the fp64 SADs of
//     _fine_search_jit are exact multiples of 1/16, so 16 x SAD is computed
//     in integers -- horizontally interpolated tables for the 4 phases, then
//     one packed 16x2 IMAD pair per two pixels for the vertical phase and the
//     native VIMNMX3.U16x2 for |16 p - v|.  Any other configuration runs the
//     reference's fp64 expression per pixel, in its order;
//   * rows are abandoned when every lane's partial SAD already reaches the
//     best SAD of earlier rounds (the reference abandons per candidate; the
//     outcome is the same).

#include <algorithm>
#include <vector>

namespace vft {

// temporal.py:46-61: grid offsets within +/-radius at `step`, Chebyshev rings
// from the centre, counterclockwise from +x within a ring (ties impossible).
inline std::vector<double> spiral_offsets(double radius, double step)
{
  const int n = (int)std::floor(radius / step + 1e-9);
  struct P { double x, y, cheb, ang; };
  std::vector<P> pts;
  for (int iy = -n; iy <= n; iy++)
    for (int ix = -n; ix <= n; ix++) {
      const double x = step * ix, y = step * iy;
      double a = std::atan2(y, x);
      if (a < -1e-12) a += 2.0 * M_PI;
      pts.push_back({x, y, std::max(std::fabs(x), std::fabs(y)), a});
    }
  std::stable_sort(pts.begin(), pts.end(), [](const P& a, const P& b) {
    return a.cheb != b.cheb ? a.cheb < b.cheb : a.ang < b.ang;
  });
  std::vector<double> out;
  for (const P& p : pts) { out.push_back(p.x); out.push_back(p.y); }
  return out;
}

struct Setup {
  int P, nc, nf, rc, rfc, dyadic;
  double t_bm, t_et;
  const double* coarse;   // nc (x, y) pairs, spiral order
  const double* fine;     // nf (x, y) pairs, spiral order without (0, 0)
  int M;                  // window margin around the block: rc + rfc + 1
  int win_w, win_words;   // window bytes per row (P + 2M), words per row (+1 for funnel reads)
  int ht_w, ht_rows;      // fine tables: values per row (P + 2 rfc), rows (P + 2 rfc + 1)
  int shmask;             // byte shifts (xr & 3) of coarse candidates: window copies kept
  int sm_words;           // shared words per warp
};

inline void layout(Setup& q)
{
  q.M = q.rc + q.rfc + 1;
  q.win_w = q.P + 2 * q.M;
  q.win_words = (q.win_w + 3) / 4 + 1;
  q.ht_w = q.P + 2 * q.rfc;
  q.ht_rows = q.P + 2 * q.rfc + 1;
  const int patch_words = (q.P * q.P + 3) / 4, p16_words = (q.P * q.P + 1) / 2;
  const int win = q.win_w * q.win_words;
  const int tables = q.dyadic ? 4 * q.ht_rows * (q.ht_w / 2) * 2 : 0;
  // copy 0 is the window itself; copies for the other shifts coarse candidates use
  const int ncopy = 1 + __builtin_popcount(q.shmask & 0xe);
  q.sm_words = patch_words + p16_words + win * ncopy + tables;
}

#define BM_WARPS 4

// One feature, whole warp.  Returns found (warp-uniform) and the new position
// and SAD.  `sm` = this warp's shared words.
__device__ bool search(const Setup& q, uint32_t* sm, const uint8_t* prev, long long prev_pitch, const uint8_t* cur,
                       long long pitch, int w, int h, double x, double y, double& nx, double& ny, double& sad_out)
{
  const int lane = threadIdx.x & 31, P = q.P;
  // temporal.py:280-287 / 208-211: rounded centre, block top-left
  const double cxd = floor(x + 0.5), cyd = floor(y + 0.5);
  if (!(cxd > -1e9 && cxd < 1e9 && cyd > -1e9 && cyd < 1e9)) return false;
  const int cxi = (int)cxd, cyi = (int)cyd;
  const int tlx = cxi - P / 2, tly = cyi - P / 2;
  if (tlx < 0 || tly < 0 || tlx + P > w || tly + P > h) return false;
  uint32_t* pw = sm;                                   // block bytes, row-major, as words
  uint32_t* p16 = pw + (P * P + 3) / 4;                // 16 * block value, 16x2 pairs
  uint32_t* win = p16 + (P * P + 1) / 2;               // window rows
  const int wsz = q.win_w * q.win_words;
  uint32_t* ht = win + wsz * (1 + __popc(q.shmask & 0xe));   // fine tables (dyadic path)
  // copy c (c = 1..3, when used) holds the window shifted left by c bytes
  auto copy_of = [&](int c) -> uint32_t* { return c == 0 ? win : win + wsz * __popc(q.shmask & 0xe & ((2 << c) - 1)); };
  uint8_t* pb = reinterpret_cast<uint8_t*>(pw);
  // word (r, k) of a w-word-wide region at (x0, y0) of a frame: aligned 4-byte
  // loads + funnel shift when the row span lies inside the frame and rows are
  // 4-byte aligned, else bytes (zero outside the frame)
  auto fetch = [&](const uint8_t* f, long long fp, int x0, int yy, int k) -> uint32_t {
    if (yy < 0 || yy >= h) return 0u;
    const uint8_t* row = f + (long long)yy * fp;
    const int xb = x0 + 4 * k;
    // w % 4 == 0: the second aligned word of an in-row span never passes the row's end
    if (xb >= 0 && xb + 4 <= w && (w & 3) == 0 && ((reinterpret_cast<uintptr_t>(row) | (uintptr_t)fp) & 3) == 0) {
      const uint32_t* r32 = reinterpret_cast<const uint32_t*>(row) + (xb >> 2);
      const uint32_t lo = __ldg(r32), hi = (xb & 3) ? __ldg(r32 + 1) : 0u;
      return __funnelshift_r(lo, hi, 8 * (xb & 3));
    }
    uint32_t v = 0;
#pragma unroll
    for (int c = 0; c < 4; c++) {
      const int xx = xb + c;
      if (xx >= 0 && xx < w) v |= (uint32_t)__ldg(row + xx) << (8 * c);
    }
    return v;
  };
  if ((P & 3) == 0) {
    const int pwr0 = P / 4;
    for (int i = lane; i < P * pwr0; i += 32) pw[i] = fetch(prev, prev_pitch, tlx, tly + i / pwr0, i % pwr0);
  } else {
    for (int i = lane; i < P * P; i += 32) pb[i] = __ldg(prev + (long long)(tly + i / P) * prev_pitch + tlx + i % P);
  }
  // window [tlx - M, tlx + P + M) x [tly - M, tly + P + M) of cur, zero outside the frame;
  // (row, word) of element i advanced incrementally (no division)
  const int wx0 = tlx - q.M, wy0 = tly - q.M;
  {
    const int dr = 32 / q.win_words, dk = 32 - dr * q.win_words;
    int r = lane / q.win_words, k = lane - r * q.win_words;
    const bool inside = wx0 >= 0 && wy0 >= 0 && wx0 + 4 * q.win_words + 4 <= w && wy0 + q.win_w <= h && (w & 3) == 0 &&
                        ((reinterpret_cast<uintptr_t>(cur) | (uintptr_t)pitch) & 3) == 0;
    if (inside) {                                      // whole window in the frame: aligned funnel loads
      const uint32_t* b32 = reinterpret_cast<const uint32_t*>(cur + (long long)wy0 * pitch) + (wx0 >> 2);
      const int ps = (int)(pitch >> 2), sh = 8 * (wx0 & 3);
      for (int i = lane; i < wsz; i += 32) {
        const uint32_t* a = b32 + r * ps + k;
        win[i] = __funnelshift_r(__ldg(a), __ldg(a + 1), sh);
        r += dr;
        k += dk;
        if (k >= q.win_words) { k -= q.win_words; r++; }
      }
    } else {
      for (int i = lane; i < wsz; i += 32) {
        win[i] = fetch(cur, pitch, wx0, wy0 + r, k);
        r += dr;
        k += dk;
        if (k >= q.win_words) { k -= q.win_words; r++; }
      }
    }
  }
  __syncwarp();
  for (int c = 1; c < 4; c++) {                        // shifted copies (last word of a row: pad)
    if (!((q.shmask >> c) & 1)) continue;
    uint32_t* dst = copy_of(c);
    for (int i = lane; i < wsz; i += 32) {
      const bool last = (i + 1) % q.win_words == 0;
      dst[i] = __funnelshift_r(win[i], last ? 0u : win[i + 1], 8 * c);
    }
  }
  __syncwarp();
  for (int i = lane; i < (P * P + 1) / 2; i += 32) {
    const uint32_t a = 16u * pb[2 * i], b = 2 * i + 1 < P * P ? 16u * pb[2 * i + 1] : 0u;
    p16[i] = a | (b << 16);
  }
  __syncwarp();

  // ---- coarse stage (temporal.py:125-145) ----
  int best = INT_MAX, bestk = -1;
  bool early = false;
  const int pwr = P / 4;                               // whole block words per row
  for (int base = 0; base < q.nc && !early; base += 32) {
    const int k = base + lane;
    bool valid = k < q.nc;
    int dx = 0, dy = 0;
    if (valid) {
      dx = (int)q.coarse[2 * k];                       // np.int64(offs): truncation
      dy = (int)q.coarse[2 * k + 1];
      const int cx = tlx + dx, cy = tly + dy;
      valid = cx >= 0 && cy >= 0 && cx + P <= w && cy + P <= h;
    }
    const int xr = q.M + dx, yr = q.M + dy;            // window coordinates of the candidate
    const int o = xr >> 2, sh = 8 * (xr & 3);
    const uint32_t* cw = copy_of(0) + yr * q.win_words + o;
    int sad = 0;
    for (int r = 0; r < P; r++) {
      if (valid) {
        const uint32_t* row = cw + r * q.win_words;
        const uint32_t* pr = pw + r * P / 4;
        if ((P & 3) == 0) {
          for (int t = 0; t < pwr; t++) {
            const uint32_t a = __funnelshift_r(row[t], row[t + 1], sh);
            asm("vabsdiff4.u32.u32.u32.add %0, %1, %2, %0;" : "+r"(sad) : "r"(a), "r"(pr[t]));
          }
        } else {
          const uint8_t* wb = reinterpret_cast<const uint8_t*>(win + (yr + r) * q.win_words) + xr;
          const uint8_t* bb = pb + r * P;
          for (int c = 0; c < P; c++) sad += abs((int)bb[c] - (int)wb[c]);
        }
      }
      if ((r & 3) == 3 && __all_sync(0xffffffffu, !valid || sad >= best)) break;
    }
    // first offset with SAD < t_et (it beats every earlier SAD, all >= t_et)
    const unsigned e = __ballot_sync(0xffffffffu, valid && sad < best && (double)sad < q.t_et);
    if (e) {
      const int src = __ffs(e) - 1;
      best = __shfl_sync(0xffffffffu, sad, src);
      bestk = base + src;
      early = true;
      break;
    }
    // otherwise the round's smallest SAD below the incumbent, first lane on ties
    unsigned key = (valid && sad < best) ? ((unsigned)sad << 5) | (unsigned)lane : 0xffffffffu;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) key = min(key, __shfl_xor_sync(0xffffffffu, key, off));
    if (key != 0xffffffffu) {
      best = (int)(key >> 5);
      bestk = base + (int)(key & 31);
    }
  }
  if (bestk < 0) return false;
  double ox = q.coarse[2 * bestk], oy = q.coarse[2 * bestk + 1];
  double bestd = (double)best;

  // ---- fine stage (temporal.py:147-180, 214-222) ----
  if (!early && q.nf > 0) {
    const double bfx = (double)tlx + ox, bfy = (double)tly + oy;
    int fk = -1;
    if (q.dyadic) {
      // integer block origin of the refinement (coarse offsets are integers)
      const int bx = tlx + (int)ox, by = tly + (int)oy;
      // H_a(y, x) = (4 - a) I(y, x) + a I(y, x + 1), x in [bx - rfc, bx + rfc + P), a = 0..3,
      // stored as 16x2 pairs at even (x, x+1) and odd (x+1, x+2) alignment
      const int hx0 = bx - q.rfc, hy0 = by - q.rfc;
      const int pairs = q.ht_w / 2;
      const uint8_t* wb = reinterpret_cast<const uint8_t*>(win);
      const int wbp = 4 * q.win_words;
      auto raw = [&](int yy, int xx) -> uint32_t { return wb[(yy - wy0) * wbp + (xx - wx0)]; };
      const int dr = 32 / pairs, dk = 32 - dr * pairs;
      int rr = lane / pairs, kk = lane - rr * pairs;   // (phase-major row, pair) of element i
      for (int i = lane; i < 4 * q.ht_rows * pairs; i += 32) {
        const int a = rr / q.ht_rows, r = rr - a * q.ht_rows, k = kk, yy = hy0 + r, xx = hx0 + 2 * k;
        kk += dk;
        rr += dr;
        if (kk >= pairs) { kk -= pairs; rr++; }
        const uint32_t i0 = raw(yy, xx), i1 = raw(yy, xx + 1), i2 = raw(yy, xx + 2), i3 = raw(yy, xx + 3);
        const uint32_t h0 = (4 - a) * i0 + a * i1, h1 = (4 - a) * i1 + a * i2, h2 = (4 - a) * i2 + a * i3;
        uint32_t* te = ht + (a * q.ht_rows + r) * pairs * 2;
        te[k] = h0 | (h1 << 16);                       // even alignment: (x, x+1)
        te[pairs + k] = h1 | (h2 << 16);               // odd alignment: (x+1, x+2)
      }
      __syncwarp();
      const double best16_init = bestd * 16.0;
      double best16 = best16_init;
      for (int base = 0; base < q.nf; base += 32) {
        const int j = base + lane;
        bool valid = j < q.nf;
        int a = 0, bq = 0, xr = 0, yr = 0;
        if (valid) {
          const double fx = bfx + q.fine[2 * j], fy = bfy + q.fine[2 * j + 1];
          const double flx = floor(fx), fly = floor(fy);
          const int ix = (int)flx, iy = (int)fly;
          valid = ix >= 0 && iy >= 0 && ix + P < w && iy + P < h;
          a = (int)((fx - flx) * 4.0);
          bq = (int)((fy - fly) * 4.0);
          xr = ix - hx0;
          yr = iy - hy0;
        }
        const uint32_t* t0 = ht + (a * q.ht_rows + yr) * pairs * 2 + ((xr & 1) ? pairs : 0) + (xr >> 1);
        const uint32_t wa = 4u - (uint32_t)bq, wb2 = (uint32_t)bq;
        int sad16 = 0;
        for (int r = 0; r < P; r++) {
          if (valid) {
            const uint32_t* h0 = t0 + r * pairs * 2;
            const uint32_t* h1 = h0 + pairs * 2;
            const uint32_t* pp = p16 + r * (P / 2);
            uint32_t acc = 0;
            for (int t = 0; t < P / 2; t++) {
              const uint32_t v = h0[t] * wa + h1[t] * wb2;          // 16 x bilinear value, two pixels
              acc += __vimax3_u16x2(pp[t], v, v) - __vimin3_u16x2(pp[t], v, v);
            }
            sad16 += (int)(acc & 0xffffu) + (int)(acc >> 16);
          }
          if ((r & 3) == 3 && __all_sync(0xffffffffu, !valid || (double)sad16 >= best16)) break;
        }
        const double sd = (double)sad16 * 0.0625;
        const unsigned e = __ballot_sync(0xffffffffu, valid && sd < bestd && sd < q.t_et);
        if (e) {
          const int src = __ffs(e) - 1;
          bestd = __shfl_sync(0xffffffffu, sd, src);
          fk = base + src;
          break;
        }
        unsigned key = (valid && sd < bestd) ? ((unsigned)sad16 << 5) | (unsigned)lane : 0xffffffffu;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) key = min(key, __shfl_xor_sync(0xffffffffu, key, off));
        if (key != 0xffffffffu) {
          bestd = (double)(key >> 5) * 0.0625;
          best16 = (double)(key >> 5);
          fk = base + (int)(key & 31);
        }
      }
    } else {
      // the reference's fp64 expression, per pixel in its order
      const uint8_t* wb = reinterpret_cast<const uint8_t*>(win);
      const int wbp = 4 * q.win_words;
      for (int base = 0; base < q.nf; base += 32) {
        const int j = base + lane;
        bool valid = j < q.nf;
        double sad = 0.0;
        if (valid) {
          const double fx = bfx + q.fine[2 * j], fy = bfy + q.fine[2 * j + 1];
          const double flx = floor(fx), fly = floor(fy);
          const long long ix = (long long)flx, iy = (long long)fly;
          valid = ix >= 0 && iy >= 0 && ix + P < w && iy + P < h;
          if (valid) {
            const double ax = fx - (double)ix, ay = fy - (double)iy;
            const double w00 = (1.0 - ax) * (1.0 - ay), w10 = ax * (1.0 - ay), w01 = (1.0 - ax) * ay, w11 = ax * ay;
            const int xr = (int)(ix - wx0), yr = (int)(iy - wy0);
            for (int r = 0; r < P; r++) {
              const uint8_t* f0 = wb + (yr + r) * wbp + xr;
              const uint8_t* f1 = f0 + wbp;
              for (int c = 0; c < P; c++) {
                const double v = w00 * f0[c] + w10 * f0[c + 1] + w01 * f1[c] + w11 * f1[c + 1];
                sad += fabs((double)pb[r * P + c] - v);
              }
              if (sad >= bestd) break;                  // abandoned (temporal.py:170-172)
            }
          }
        }
        const unsigned e = __ballot_sync(0xffffffffu, valid && sad < bestd && sad < q.t_et);
        if (e) {
          const int src = __ffs(e) - 1;
          bestd = __shfl_sync(0xffffffffu, sad, src);
          fk = base + src;
          break;
        }
        // round argmin: smallest SAD below the incumbent, first lane on ties
        double m = (valid && sad < bestd) ? sad : INFINITY;
        int ml = lane;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          const double om = __shfl_xor_sync(0xffffffffu, m, off);
          const int ol = __shfl_xor_sync(0xffffffffu, ml, off);
          if (om < m || (om == m && ol < ml)) { m = om; ml = ol; }
        }
        if (m < bestd) { bestd = m; fk = base + ml; }
      }
    }
    if (fk >= 0) { ox += q.fine[2 * fk]; oy += q.fine[2 * fk + 1]; }
  }
  if (bestd >= q.t_bm) return false;                   // temporal.py:223-224
  nx = (double)cxi + ox;
  ny = (double)cyi + oy;
  sad_out = bestd;
  return true;
}

}  // namespace vft

// Stand-alone batch (vf_block_match): warp per feature.
__global__ void __launch_bounds__(32 * BM_WARPS) k_block_match(const vft::Setup q, const uint8_t* prev,
                                                               const uint8_t* cur, int w, int h, long long pitch,
                                                               int n, const double* x, const double* y, double* nx,
                                                               double* ny, double* sad, uint8_t* found)
{
  extern __shared__ uint32_t bm_sm[];
  uint32_t* sm = bm_sm + (threadIdx.x >> 5) * q.sm_words;
  for (int i = blockIdx.x * BM_WARPS + (threadIdx.x >> 5); i < n; i += gridDim.x * BM_WARPS) {
    double ax = 0, ay = 0, as = 0;
    const bool f = vft::search(q, sm, prev, pitch, cur, pitch, w, h, __ldg(x + i), __ldg(y + i), ax, ay, as);
    if ((threadIdx.x & 31) == 0) {
      found[i] = f ? 1 : 0;
      nx[i] = f ? ax : 0.0;
      ny[i] = f ? ay : 0.0;
      sad[i] = f ? as : 0.0;
    }
    __syncwarp();
  }
}

// Engine, off-GOP step: the previous features of every stream (flattened),
// results to staging (x, y) + flags, found counts per 1024-feature chunk.
__global__ void __launch_bounds__(32 * BM_WARPS) k_blockmatch(const __grid_constant__ Geo g,
                                                              const __grid_constant__ Bufs b, const vft::Setup q,
                                                              int n_streams)
{
  extern __shared__ uint32_t bm_sm[];
  __shared__ int sm_warp[32];
  int* pre = reinterpret_cast<int*>(bm_sm + BM_WARPS * q.sm_words);
  stream_prefix(n_streams, pre, sm_warp, [&](int sl) {
    const int* ctr = b.ctr + (b.s0 + sl) * C_NCTR;
    return ctr[C_NFEAT0 + ((ctr[C_FRAME] & 1) ^ 1)];
  });
  const int total = pre[n_streams];
  uint32_t* sm = bm_sm + (threadIdx.x >> 5) * q.sm_words;
  for (int gi = blockIdx.x * BM_WARPS + (threadIdx.x >> 5); gi < total; gi += gridDim.x * BM_WARPS) {
    // stream of gi: number of stream starts <= gi, minus one (lanes test 32 starts at a time)
    int lo = -1;
    for (int base = 0; base < n_streams; base += 32) {
      const int sl = base + (threadIdx.x & 31);
      lo += __popc(__ballot_sync(0xffffffffu, sl < n_streams && pre[sl] <= gi));
    }
    const int s = b.s0 + lo, i = gi - pre[lo];
    const int prevbuf = (b.ctr[s * C_NCTR + C_FRAME] & 1) ^ 1;
    const long long p = feat_base(g, s, prevbuf, b.ctr[s * C_NCTR + C_NFEAT0 + prevbuf]) + i;
    const uint8_t* cur = b.frames + (long long)(s - b.s0) * b.frame_stride;
    const uint8_t* prv = b.prev_frame + (long long)s * g.W * g.H;
    double ax = 0, ay = 0, as = 0;
    // the previous frame is stored unpitched (W bytes per row); the current one at frame_pitch
    const bool f = vft::search(q, sm, prv, g.W, cur, b.frame_pitch, g.W, g.H, b.fx[p], b.fy[p], ax, ay, as);
    if ((threadIdx.x & 31) == 0) {
      const long long o = (long long)s * g.kp_cap + i;
      b.bm_found[o] = f ? 1 : 0;
      b.st_x[o] = ax;
      b.st_y[o] = ay;
      if (f) atomicAdd(b.bm_chunk + (long long)s * g.prop_chunks + i / 1024, 1);
    }
    __syncwarp();
  }
}

// Engine, off-GOP step: matched features in previous-list order (temporal.py:
// 300-307): origin propagated, age + 1, descriptor / sigma / theta / score
// unchanged, position from the search.  CTA per 1024-feature chunk; the chunk
// offset is the sum of the earlier chunks' counts; chunk 0 writes the report
// (pipeline.py:322-341: n_detected 0, coverage 0).
__global__ void __launch_bounds__(256) k_bm_write(const __grid_constant__ Geo g, const __grid_constant__ Bufs b)
{
  __shared__ int wsum[4][8];
  __shared__ int base_sm;
  const int s = b.s0 + blockIdx.y, c = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  int* ctr = b.ctr + s * C_NCTR;
  const int cur = ctr[C_FRAME] & 1, prev = cur ^ 1;
  const int n_prev = ctr[C_NFEAT0 + prev];
  const int nch = (n_prev + 1023) / 1024;
  if (c >= max(nch, 1)) return;
  const int* cnt = b.bm_chunk + (long long)s * g.prop_chunks;
  __shared__ int tot_sm;
  if (wid == 0) {
    int before = 0, all = 0;
    for (int k = lane; k < nch; k += 32) {
      const int v = cnt[k];
      all += v;
      before += k < c ? v : 0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      before += __shfl_xor_sync(0xffffffffu, before, o);
      all += __shfl_xor_sync(0xffffffffu, all, o);
    }
    if (lane == 0) { base_sm = before; tot_sm = all; }
  }
  __syncthreads();
  if (c == 0) {
    const int total = tot_sm;
    if (tid == 0) {
      ctr[C_NDET] = 0; ctr[C_NPROP] = total; ctr[C_NTOTAL] = total; ctr[C_NDROP] = 0; ctr[C_NSURV] = 0;
      double* rp = b.report + (long long)s * 16;
      rp[0] = 0; rp[1] = total; rp[2] = total; rp[3] = 0; rp[4] = 0.0;
      rp[5] = ctr[C_FRAME]; rp[6] = 0; rp[7] = 0;
      rp[9] += total; rp[11] += 1.0;
    }
  }
  if (nch == 0) return;
  const long long fb = feat_base(g, s, prev, n_prev), ob = feat_base(g, s, cur, tot_sm);
  const long long so = (long long)s * g.kp_cap;
  int f[4];
#pragma unroll
  for (int j = 0; j < 4; j++) {
    const int e = c * 1024 + j * 256 + tid;
    f[j] = e < n_prev && b.bm_found[so + e];
    const unsigned bal = __ballot_sync(0xffffffffu, f[j]);
    if (lane == 0) wsum[j][wid] = __popc(bal);
    f[j] |= __popc(bal & ((1u << lane) - 1)) << 1;
  }
  __syncthreads();
  int acc = base_sm;
#pragma unroll
  for (int j = 0; j < 4; j++) {
    int before = 0, grp = 0;
#pragma unroll
    for (int w8 = 0; w8 < 8; w8++) { before += w8 < wid ? wsum[j][w8] : 0; grp += wsum[j][w8]; }
    if (f[j] & 1) {
      const int e = c * 1024 + j * 256 + tid;
      const long long o = ob + acc + before + (f[j] >> 1), p = fb + e;
      b.fx[o] = b.st_x[so + e]; b.fy[o] = b.st_y[so + e];
      b.fs[o] = b.fs[p]; b.ft[o] = b.ft[p]; b.fv[o] = b.fv[p];
      b.forg[o] = 1; b.fage[o] = b.fage[p] + 1;
      const uint4* sd = reinterpret_cast<const uint4*>(b.fdesc + p * 64);
      uint4* dd = reinterpret_cast<uint4*>(b.fdesc + o * 64);
      dd[0] = sd[0]; dd[1] = sd[1]; dd[2] = sd[2]; dd[3] = sd[3];
    }
    acc += grp;
  }
}

// The current frames become the next step's previous frames (temporal mode).
__global__ void k_copy_frames(const __grid_constant__ Geo g, const __grid_constant__ Bufs b)
{
  const int s = b.s0 + blockIdx.y;
  const uint8_t* src = b.frames + (long long)(s - b.s0) * b.frame_stride;
  uint8_t* dst = b.prev_frame + (long long)s * g.W * g.H;
  const bool vec = ((reinterpret_cast<uintptr_t>(src) | (uintptr_t)b.frame_pitch | (uintptr_t)g.W) & 15) == 0;
  if (vec) {
    const int per_row = g.W / 16;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < (long long)g.H * per_row;
         i += (long long)gridDim.x * blockDim.x) {
      const long long y = i / per_row, k = i - y * per_row;
      reinterpret_cast<uint4*>(dst + y * g.W)[k] = __ldg(reinterpret_cast<const uint4*>(src + y * b.frame_pitch) + k);
    }
  } else {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < (long long)g.H * g.W;
         i += (long long)gridDim.x * blockDim.x) {
      const long long y = i / g.W, x = i - y * g.W;
      dst[i] = __ldg(src + y * b.frame_pitch + x);
    }
  }
}
