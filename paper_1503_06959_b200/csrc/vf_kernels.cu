// vf_kernels.cu -- sm_100a kernels of the per-frame detect+describe hot path.
//
// One launch per stage, each over ALL streams of the batch (blockIdx.z / .y =
// stream), so a step processes frame n of every stream with 7 launches:
//
//   k_binmask   (binning mode) previous-feature histogram -> cell mask
//   k_pyramid   octave/intra-octave pyramid + IDDM cell mask + tile SAT
//   k_worklist  active FAST tiles -> compacted work list (+ per_layer coverage)
//   k_fast      segment-test scores over active tiles (persistent CTAs)
//   k_nms       scale-space NMS + fp64 refinement + border/merge filters,
//               deterministic (layer, y, x) compaction; last CTA scans
//   k_describe  orientation + 512-bit descriptor of kept keypoints, and
//               Eq. 1 propagation of the previous features
//   k_finalize  per-stream counters, buffer flip
//
// Reference: /root/reference/pkg/src/vidfeat/{pyramid,detector,descriptor,
// masking,pipeline}.py (cited file:line).  fp64 code is compiled with
// -fmad=false so the operation sequence matches numba's (no contraction).
#include "vf_common.cuh"
#include <math_constants.h>
#include <climits>
#include <cstdio>

// Descriptor sampling pattern (pattern.py:21-106), uploaded by vf_set_pattern.
#define VF_NPTS 60
#define VF_NBITS 512
#define VF_MAXLONG 512
__constant__ double c_px[VF_NPTS], c_py[VF_NPTS], c_rad[VF_NPTS];
__constant__ short c_si[VF_NBITS], c_sj[VF_NBITS];
__constant__ short c_li[VF_MAXLONG], c_lj[VF_MAXLONG];
__constant__ double c_wx[VF_MAXLONG], c_wy[VF_MAXLONG];
__constant__ int c_nlong;
__constant__ double c_pmax, c_radmax;        // pattern footprint: max |p|, max smoothing radius
// The same pattern as plain global tables for per-thread (divergent) reads in
// kernel prologues: a constant-bank read with 32 different addresses per warp
// is serialised, a global read is one coalesced request.
__device__ uint32_t g_pairs[VF_NBITS];      // si | sj << 16
__device__ double g_ptab[64][3];            // point x, y, smoothing radius (rows 60..63 repeat point 0)
__device__ uint32_t g_lpair[VF_MAXLONG];     // long pairs li | lj << 16 (lane-strided reads: global, not constant)
__device__ double2 g_lw[VF_MAXLONG];         // orientation weights (wx, wy) of the long pairs
// Orientation as a linear form of the 60 box means: gx = sum_i v_i Wx_i with
// Wx_i = sum over long pairs (i, j) of wx - sum over pairs (j, i) of wx (fp64
// sums on the host), and the bound weights Ax_i = sum of |wx| over the pairs
// touching i (same for y).  Rows 60..63 are zero.  [point][Wx, Wy, Ax, Ay]
__device__ double g_ow[64][4];
__constant__ double c_ogam;                  // certificate factor, see dr_orient_lin

// ============================================================================
// k_pyramid: pyramid.py:67-125 + masking.py:84-93 + descriptor.py:28-32
// ============================================================================
// One CTA per (pyramid tile, stream).  The tile is ptw x pth o0 pixels with
// ptw, pth multiples of 3 * 2^(O-1), so every derived pixel of every layer
// is a function of this tile only (2x2 halving blocks, 3x3 -> 2x2 resample
// blocks).  The o0 tile is read from HBM once; all 2(O)-1 derived tiles are
// built in shared memory and stored; the IDDM compare runs on the mask
// source octave while it is in smem; the tile-local summed-area table for the
// descriptor is built from the same smem tile.
__device__ __forceinline__ void lvl_dims(const Geo& g, int l, int& lw, int& lh)
{
  int o = l >> 1;
  if (l & 1) { lw = (2 * g.ptw / 3) >> o; lh = (2 * g.pth / 3) >> o; }
  else { lw = g.ptw >> o; lh = g.pth >> o; }
}

// ----------------------------------------------------------------------------
// Summed-area tables for the descriptor's box means (descriptor.py:28-32,85-92).
// The reference builds one (H+1) x (W+1) int64 SAT of the frame.  Here:
//   L(y, x)  = sum of o0 over [Y0, y] x [X0, x] inside its VF_ST x VF_ST tile
//   K(y, tx) = sum of o0 over [Y0, y] x [0, X0(tx))        (strip carry)
// so S(y, x) = L + K is the SAT of the VF_ST-row strip the pixel lies in, and
// a box sum is 4 strip-SAT corners per strip it spans (<= 2 strips for box
// radii < VF_ST / 2, i.e. sigma < ~9 with the default pattern).
// All values < 2^32 and box sums are exact in uint32.
// ----------------------------------------------------------------------------
// Strip carries of SAT strip ty of stream s: one warp, lanes over tile columns.
__device__ void strip_carries(const Geo& g, const Bufs& b, int s, int ty)
{
  // K[y][t] = sum over rows y' <= y of the strip and tiles t' < t of the row
  // sums.  Warp per strip; 32 tile columns per chunk (warp scan across lanes),
  // rows accumulated per lane.  Chunk c hands its per-row inclusive total to
  // chunk c + 1 through K[y][32(c+1)] (the value that slot takes anyway).
  // Row loads are issued RB at a time so the strip is not a chain of latencies.
  const int lane = threadIdx.x & 31;
  const int Y0 = ty * VF_ST, th = min(VF_ST, g.H - Y0);
  const uint32_t* rs = b.rowsum + ((long long)s * g.H + Y0) * g.stx;
  uint32_t* K = b.carry + ((long long)s * g.H + Y0) * g.stx;
  const int nch = (g.stx + 31) / 32;
  const int P = g.stx;
  constexpr int RB = 16;
#pragma unroll 1
  for (int c = 0; c < nch; c++) {
    const int t = 32 * c + lane;
    const bool in = t < P;
    const bool hand = lane == 31 && t + 1 < P;
    const uint32_t* rsp = rs + (in ? t : 0);
    const uint32_t* lp = K + 32 * c;
    uint32_t* kp = K + t;
    uint32_t acc = 0;
#pragma unroll 1
    for (int y0 = 0; y0 < th; y0 += RB) {
      uint32_t v[RB], left[RB];
#pragma unroll
      for (int k = 0; k < RB; k++) {
        const bool r = y0 + k < th;
        const int off = (y0 + k) * P;
        v[k] = (in && r) ? rsp[off] : 0u;
        left[k] = (c > 0 && r) ? lp[off] : 0u;
      }
#pragma unroll
      for (int k = 0; k < RB; k++) {
        acc += v[k];
        uint32_t inc = acc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
          if (lane >= o) inc += u;
        }
        if (y0 + k < th) {
          const int off = (y0 + k) * P;
          if (in) kp[off] = left[k] + inc - acc;
          if (hand) kp[off + 1] = left[k] + inc;
        }
      }
    }
    __syncwarp();
  }
}

// Box sum over [x0, x1] x [y0, y1] (inclusive, inside the frame) from the
// strip SATs S: per strip the box spans, 4 corners (corners above the strip
// start or left of column 0 are 0).
__device__ __forceinline__ uint32_t box_sum(const uint32_t* S, const Geo& g, int x0, int x1, int y0, int y1)
{
  const int TH = VF_ST;
  int ys = (int)__umulhi((uint32_t)y0, (uint32_t)g.sth_magic) * TH;   // strip start of y0
  const bool left = x0 > 0;
  int yb = min(y1, ys + TH - 1);
  const uint32_t* rb = S + (long long)yb * g.W;
  uint32_t sum = __ldg(rb + x1) - (left ? __ldg(rb + x0 - 1) : 0u);
  if (y0 > ys) {
    const uint32_t* ra = S + (long long)(y0 - 1) * g.W;
    sum -= __ldg(ra + x1) - (left ? __ldg(ra + x0 - 1) : 0u);
  }
  while (yb < y1) {                 // next strip(s): rows start at the strip top
    ys += TH;
    yb = min(y1, ys + TH - 1);
    const uint32_t* r2 = S + (long long)yb * g.W;
    sum += __ldg(r2 + x1) - (left ? __ldg(r2 + x0 - 1) : 0u);
  }
  return sum;
}

// o0 tile [X0, X0+ptw) x [Y0, Y0+pth) of stream s into smem (pitch ptw),
// 16-byte loads when the frame rows allow it.
// rowsum (nullable, zeroed smem [pth][ptw / VF_ST]) accumulates the tile's
// row sums per SAT-tile column.
__device__ __forceinline__ void load_o0_tile(const Geo& g, const Bufs& b, int s, int X0, int Y0, int tw, int th,
                                             uint8_t* t0, uint32_t* rowsum = nullptr)
{
  const int tid = threadIdx.x, nt = blockDim.x;
  const uint8_t* src = b.frames + (long long)(s - b.s0) * b.frame_stride + (long long)Y0 * b.frame_pitch + X0;
  const bool vec = ((reinterpret_cast<uintptr_t>(src) | (uintptr_t)b.frame_pitch) & 15) == 0 && tw == g.ptw;
  if (vec) {
    const int per_row = g.ptw / 16;
    for (int i = tid; i < th * per_row; i += nt) {
      const int y = i / per_row, c = i - y * per_row;
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(src + (long long)y * b.frame_pitch) + c);
      *reinterpret_cast<uint4*>(t0 + y * g.ptw + 16 * c) = v;
      if (rowsum) {
        uint32_t a = __dp4a(v.x, 0x01010101u, 0u);
        a = __dp4a(v.y, 0x01010101u, a);
        a = __dp4a(v.z, 0x01010101u, a);
        a = __dp4a(v.w, 0x01010101u, a);
        atomicAdd(rowsum + y * (g.ptw / VF_ST) + (16 * c) / VF_ST, a);
      }
    }
  } else {
    for (int i = tid; i < th * g.ptw; i += nt) {
      const int y = i / g.ptw, x = i - y * g.ptw;
      const uint8_t v = x < tw ? __ldg(src + (long long)y * b.frame_pitch + x) : 0;
      t0[i] = v;
      if (rowsum && v) atomicAdd(rowsum + y * (g.ptw / VF_ST) + x / VF_ST, (uint32_t)v);
    }
  }
}

__global__ void __launch_bounds__(256) k_pyramid(const __grid_constant__ Geo g, const __grid_constant__ Bufs b)
{
  extern __shared__ __align__(16) uint8_t smem[];
  const int s = b.s0 + blockIdx.z;
  const int X0 = blockIdx.x * g.ptw, Y0 = blockIdx.y * g.pth;
  const int tid = threadIdx.x, nt = blockDim.x;
  // carve smem: level tiles then SAT
  int off[VF_MAXL];
  int acc = 0;
  for (int l = 0; l < g.NL; l++) {
    int lw, lh;
    lvl_dims(g, l, lw, lh);
    off[l] = acc;
    acc += (lw * lh + 15) & ~15;
  }

  if (blockIdx.x == 0 && blockIdx.y == 0) {
    if (tid == 0) {
      b.ctr[s * C_NCTR + C_STAGE] = 0;
      b.ctr[s * C_NCTR + C_NGLOB] = 0;
      b.nms_cnt[4 * s] = 0; b.nms_cnt[4 * s + 1] = 0;
      b.sat_count[s] = 0;
      b.work_count[s] = 0;
    }
    for (int i = tid; i < g.sty * g.stw_words; i += blockDim.x) b.sat_bits[(long long)s * g.sty * g.stw_words + i] = 0u;
  }

  // ---- load the o0 tile ------------------------------------------------------
  const int tw = min(g.ptw, g.W - X0), th = min(g.pth, g.H - Y0);
  uint8_t* t0 = smem + off[0];
  uint32_t* rsum = reinterpret_cast<uint32_t*>(smem + acc);   // [pth][ptw / VF_ST] row sums
  const int nseg = g.ptw / VF_ST;
  for (int y = tid; y < g.pth * nseg; y += nt) rsum[y] = 0;
  __syncthreads();
  load_o0_tile(g, b, s, X0, Y0, tw, th, t0, rsum);
  __syncthreads();

  // ---- derived layers: level by level, octave and intra chains together ------
  for (int o = 0; o < g.O; o++) {
    for (int k = 0; k < 2; k++) {
      int l = 2 * o + k;
      if (l == 0) continue;
      int lw, lh;
      lvl_dims(g, l, lw, lh);
      int gx0 = k ? ((2 * X0 / 3) >> o) : (X0 >> o);
      int gy0 = k ? ((2 * Y0 / 3) >> o) : (Y0 >> o);
      int vw = min(lw, g.L[l].w - gx0), vh = min(lh, g.L[l].h - gy0);
      if (vw <= 0 || vh <= 0) continue;
      uint8_t* dst = smem + off[l];
      uint8_t* gdst = b.layers + (long long)s * g.layer_slab + g.L[l].layer_off + (long long)gy0 * g.L[l].pitch + gx0;
      const int gp = g.L[l].pitch;
      if (l == 1) {
        // i0: area-weighted 2/3 resample of o0 (pyramid.py:76-94): per axis
        // even output 2a+b, odd a+2b, then (v+4)//9.  A thread makes a 2 x 4
        // output block from 3 rows x 6 columns.
        if ((lw & 3) == 0 && (lh & 1) == 0) {
          const int wpr = lw >> 2, nblk = (lh >> 1) * wpr;
          for (int i = tid; i < nblk; i += nt) {
            const int p = i / wpr, q = i - p * wpr;
            const int base = 6 * q, al = base & ~3, sh = 8 * (base & 3);
            uint32_t hsum[3][4];
#pragma unroll
            for (int r = 0; r < 3; r++) {
              const uint8_t* row = t0 + (3 * p + r) * g.ptw + al;
              // base & 3 is 0 or 2, so the aligned 8 bytes al..al+7 cover base..base+5
              const uint32_t w0 = *reinterpret_cast<const uint32_t*>(row);
              const uint32_t w1 = *reinterpret_cast<const uint32_t*>(row + 4);
              const unsigned long long lo = ((unsigned long long)w1 << 32 | w0) >> sh;
              const uint32_t c0 = lo & 0xff, c1 = (lo >> 8) & 0xff, c2 = (lo >> 16) & 0xff, c3 = (lo >> 24) & 0xff;
              const uint32_t c4 = (lo >> 32) & 0xff, c5 = (lo >> 40) & 0xff;
              hsum[r][0] = 2 * c0 + c1; hsum[r][1] = c1 + 2 * c2;
              hsum[r][2] = 2 * c3 + c4; hsum[r][3] = c4 + 2 * c5;
            }
            uint32_t e = 0, o = 0;
#pragma unroll
            for (int c = 0; c < 4; c++) {
              e |= ((2 * hsum[0][c] + hsum[1][c] + 4) / 9) << (8 * c);
              o |= ((hsum[1][c] + 2 * hsum[2][c] + 4) / 9) << (8 * c);
            }
            const int y = 2 * p, x = 4 * q;
            *reinterpret_cast<uint32_t*>(dst + y * lw + x) = e;
            *reinterpret_cast<uint32_t*>(dst + (y + 1) * lw + x) = o;
            if (x + 4 <= vw) {
              if (y < vh) *reinterpret_cast<uint32_t*>(gdst + (long long)y * gp + x) = e;
              if (y + 1 < vh) *reinterpret_cast<uint32_t*>(gdst + (long long)(y + 1) * gp + x) = o;
            } else {
              for (int c = 0; c < 4 && x + c < vw; c++) {
                if (y < vh) gdst[(long long)y * gp + x + c] = (uint8_t)(e >> (8 * c));
                if (y + 1 < vh) gdst[(long long)(y + 1) * gp + x + c] = (uint8_t)(o >> (8 * c));
              }
            }
          }
        } else {
          for (int i = tid; i < vw * vh; i += nt) {
            int y = i / vw, x = i - y * vw;
            int ky = y >> 1, kx = x >> 1;
            int ry0 = (y & 1) ? 3 * ky + 1 : 3 * ky, cy0 = (y & 1) ? 1 : 2, cy1 = (y & 1) ? 2 : 1;
            int rx0 = (x & 1) ? 3 * kx + 1 : 3 * kx, cx0 = (x & 1) ? 1 : 2, cx1 = (x & 1) ? 2 : 1;
            const uint8_t* r0 = t0 + ry0 * g.ptw;
            const uint8_t* r1 = r0 + g.ptw;
            uint32_t a0 = cy0 * r0[rx0] + cy1 * r1[rx0];
            uint32_t a1 = cy0 * r0[rx0 + 1] + cy1 * r1[rx0 + 1];
            uint8_t q = (uint8_t)((cx0 * a0 + cx1 * a1 + 4) / 9);
            dst[y * lw + x] = q;
            gdst[(long long)y * gp + x] = q;
          }
        }
      } else {
        // halving of the same chain's previous level (pyramid.py:67-73):
        // 4 outputs per thread, pair sums in 16-bit lanes
        int pl = l - 2, pw, ph;
        lvl_dims(g, pl, pw, ph);
        const uint8_t* sp = smem + off[pl];
        if ((lw & 3) == 0) {
          const int wpr = lw >> 2;
          for (int i = tid; i < lh * wpr; i += nt) {
            const int y = i / wpr, q = i - y * wpr;
            const uint2 r0 = *reinterpret_cast<const uint2*>(sp + (2 * y) * pw + 8 * q);
            const uint2 r1 = *reinterpret_cast<const uint2*>(sp + (2 * y + 1) * pw + 8 * q);
            uint32_t a0 = (r0.x & 0x00ff00ffu) + ((r0.x >> 8) & 0x00ff00ffu) + (r1.x & 0x00ff00ffu) + ((r1.x >> 8) & 0x00ff00ffu);
            uint32_t a1 = (r0.y & 0x00ff00ffu) + ((r0.y >> 8) & 0x00ff00ffu) + (r1.y & 0x00ff00ffu) + ((r1.y >> 8) & 0x00ff00ffu);
            a0 = ((a0 + 0x00020002u) >> 2) & 0x00ff00ffu;
            a1 = ((a1 + 0x00020002u) >> 2) & 0x00ff00ffu;
            const uint32_t wv = __byte_perm(a0, a1, 0x6420);
            const int x = 4 * q;
            *reinterpret_cast<uint32_t*>(dst + y * lw + x) = wv;
            if (y < vh) {
              if (x + 4 <= vw) *reinterpret_cast<uint32_t*>(gdst + (long long)y * gp + x) = wv;
              else for (int c = 0; c < 4 && x + c < vw; c++) gdst[(long long)y * gp + x + c] = (uint8_t)(wv >> (8 * c));
            }
          }
        } else {
          for (int i = tid; i < vw * vh; i += nt) {
            int y = i / vw, x = i - y * vw;
            const uint8_t* r0 = sp + (2 * y) * pw + 2 * x;
            uint32_t sum = r0[0] + r0[1] + r0[pw] + r0[pw + 1];
            uint8_t q = (uint8_t)((sum + 2) >> 2);
            dst[y * lw + x] = q;
            gdst[(long long)y * gp + x] = q;
          }
        }
      }
    }
    __syncthreads();
  }

  // ---- IDDM (masking.py:84-93) on the mask-source octave(s) -------------------
  if (g.mask_mode == 1) {
    const int um = use_mask(g, b, s);
    unsigned long long covered = 0;
    int lv0 = g.per_layer ? 0 : g.mask_level, lv1 = g.per_layer ? g.O - 1 : g.mask_level;
    for (int lv = lv0; lv <= lv1; lv++) {
      int l = 2 * lv, lw, lh;
      lvl_dims(g, l, lw, lh);
      int gx0 = X0 >> lv, gy0 = Y0 >> lv;
      int vw = min(lw, g.L[l].w - gx0), vh = min(lh, g.L[l].h - gy0);
      if (vw <= 0 || vh <= 0) continue;
      const GridGeo& G = g.grid[g.per_layer ? lv : 0];
      const uint8_t* cur = smem + off[l];
      uint8_t* st = iddm_state(g, b, s, lv, 0);
      const uint8_t* stp = iddm_state(g, b, s, lv, 1);
      uint8_t* cells = b.cells + (long long)s * g.cell_slab + G.cell_off;
      for (int i = tid; i < vw * vh; i += nt) {
        int y = i / vw, x = i - y * vw;
        long long gi = (long long)(gy0 + y) * g.L[l].w + gx0 + x;
        int c = cur[y * lw + x];
        if (um) {
          int p = stp[gi];
          int d = c - p;
          d = d < 0 ? -d : d;
          int bit = (double)d > g.t_i;   // int16 diff vs float t_i, strict
          cells[gi] = (uint8_t)bit;
          if (bit && !g.per_layer) {
            long long ay = (long long)(gy0 + y) * G.ch, ax = (long long)(gx0 + x) * G.cw;
            long long hy = g.H - ay, hx = g.W - ax;
            hy = hy < G.ch ? hy : G.ch;
            hx = hx < G.cw ? hx : G.cw;
            if (hy > 0 && hx > 0) covered += (unsigned long long)(hy * hx);
          }
        }
        st[gi] = (uint8_t)c;
      }
    }
    if (um && !g.per_layer) {
      for (int o = 16; o > 0; o >>= 1) covered += __shfl_down_sync(0xffffffffu, covered, o);
      if ((tid & 31) == 0 && covered) atomicAdd(b.cov + s, covered);
    }
  }

  // ---- summed-area data of the descriptor (descriptor.py:28-32) --------------
  // Per-row sums of this tile feed the strip carries (k_worklist); the strip
  // SATs themselves are built by k_sat for the tiles the descriptor reads.
  for (int i = tid; i < th * nseg; i += nt) {
    const int y = i / nseg, k = i - y * nseg, col = blockIdx.x * nseg + k;
    if (col < g.stx) b.rowsum[((long long)s * g.H + Y0 + y) * g.stx + col] = rsum[i];
  }
}

// Flattened item index -> stream via the per-stream prefix (stream_prefix).
__device__ __forceinline__ int find_stream(const int* pre, int n_streams, int gi)
{
  int lo = 0, hi = n_streams;
  while (hi - lo > 1) { int m = (lo + hi) >> 1; if (pre[m] <= gi) lo = m; else hi = m; }
  return lo;
}

// Same, for a persistent loop that visits increasing items: start from the
// previous item's stream (usually 0 or 1 steps instead of a binary search).
__device__ __forceinline__ int find_stream_from(const int* pre, int n_streams, int gi, int& hint)
{
  int lo = hint;
  while (lo + 1 < n_streams && pre[lo + 1] <= gi) lo++;
  hint = lo;
  return lo;
}

// Exclusive prefix over streams of a per-stream count, computed by the whole
// block (one load per thread), into pre[0..n_streams].
template <typename F>
__device__ __forceinline__ void stream_prefix(int n_streams, int* pre, int* sm_warp, F count)
{
  int carry = 0;
  for (int base = 0; base < n_streams; base += blockDim.x) {
    const int s = base + threadIdx.x;
    const int v = s < n_streams ? count(s) : 0;
    int tot;
    const int ex = block_excl_scan<int>(v, sm_warp, tot);
    if (s < n_streams) pre[s] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) pre[n_streams] = carry;
  __syncthreads();
}

// ============================================================================
// k_sat: strip SATs for the descriptor.  Dense frames (no mask): every tile;
// masked frames: the tiles kept keypoints' footprints touch (marked by k_nms).
// Persistent CTAs, one warp per VF_ST x VF_ST tile, flattened over streams:
//   lane r: row r of the tile (two 16-B loads), its running row prefix plus
//           d(r) = K(r) - K(r-1) (the part of row r left of the tile), into a
//           padded smem tile;
//   lane x: column x accumulated down the rows = L(y, x) + K(y, tx), stored as
//           one coalesced 128-B row segment per row.
// ============================================================================
#define SAT_WARPS 8
#define SAT_PITCH (VF_ST + 4)   // words; 16-B row stores of 8 lanes hit distinct banks
__global__ void __launch_bounds__(32 * SAT_WARPS) k_sat(const __grid_constant__ Geo g, const __grid_constant__ Bufs b,
                                                        int n_streams, int all)
{
  extern __shared__ __align__(16) uint8_t smem[];
  uint32_t* tile = reinterpret_cast<uint32_t*>(smem) + (threadIdx.x >> 5) * VF_ST * SAT_PITCH;
  int* pre = reinterpret_cast<int*>(smem + SAT_WARPS * VF_ST * SAT_PITCH * 4);
  __shared__ int sm_warp[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  // all = 1 (stand-alone describe): every tile of a stream with keypoints;
  // else the tiles k_nms marked for the strip-SAT path's keypoints
  stream_prefix(n_streams, pre, sm_warp, [&](int sl) {
    const int s = b.s0 + sl;
    return all ? (b.ctr[s * C_NCTR + C_NDET] == 0 ? 0 : g.sat_tiles)
               : (!b.sat_early && b.ctr[s * C_NCTR + C_NGLOB] == 0 ? 0 : b.sat_count[s]);
  });
  const int n = pre[n_streams];
  // one-tile software pipeline per warp: tile k + 1's work-list entry, carry
  // word and row loads are in flight while tile k is built
  struct TileIn { int s, X0, Y0, tw, th; uint32_t kr, w[8]; };
  const bool vec = ((reinterpret_cast<uintptr_t>(b.frames) | (uintptr_t)b.frame_pitch | (uintptr_t)b.frame_stride) &
                    15) == 0;
  int shint = 0;
  auto fetch = [&](int item, TileIn& in) {
    const int lo = find_stream_from(pre, n_streams, item, shint);
    const int s = b.s0 + lo, i = item - pre[lo];
    const int t = all ? i : b.sat_work[(long long)s * g.sat_tiles + i];
    const int ty = t / g.stx, tx = t - ty * g.stx;
    in.s = s; in.X0 = tx * VF_ST; in.Y0 = ty * VF_ST;
    in.tw = min(VF_ST, g.W - in.X0); in.th = min(VF_ST, g.H - in.Y0);
    const bool rin = lane < in.th;
    const uint8_t* src = b.frames + (long long)(s - b.s0) * b.frame_stride + (long long)(in.Y0 + lane) * b.frame_pitch +
                         in.X0;
    in.kr = rin ? __ldg(b.carry + ((long long)s * g.H + in.Y0 + lane) * g.stx + tx) : 0u;
    if (in.tw == VF_ST && vec) {
      uint4 v0 = make_uint4(0, 0, 0, 0), v1 = v0;
      if (rin) { v0 = __ldg(reinterpret_cast<const uint4*>(src)); v1 = __ldg(reinterpret_cast<const uint4*>(src) + 1); }
      in.w[0] = v0.x; in.w[1] = v0.y; in.w[2] = v0.z; in.w[3] = v0.w;
      in.w[4] = v1.x; in.w[5] = v1.y; in.w[6] = v1.z; in.w[7] = v1.w;
    } else {
#pragma unroll
      for (int q = 0; q < 8; q++) {
        uint32_t v = 0;
#pragma unroll
        for (int c = 0; c < 4; c++) {
          const int x = 4 * q + c;
          if (rin && x < in.tw) v |= (uint32_t)src[x] << (8 * c);
        }
        in.w[q] = v;
      }
    }
  };
  const int stride = gridDim.x * SAT_WARPS;
  int item = blockIdx.x * SAT_WARPS + wid;
  TileIn cur;
  if (item < n) fetch(item, cur);
  for (; item < n; item += stride) {
    TileIn nxt;
    if (item + stride < n) fetch(item + stride, nxt);
    // ---- lane = row: running row prefix + d(r) = K(r) - K(r - 1) ----
    const uint32_t kp = __shfl_up_sync(0xffffffffu, cur.kr, 1);
    uint32_t run = lane == 0 ? cur.kr : cur.kr - kp;
    uint32_t* trow = tile + lane * SAT_PITCH;
#pragma unroll
    for (int q = 0; q < 8; q++) {
      uint4 o;
      run += cur.w[q] & 0xff;         o.x = run;
      run += (cur.w[q] >> 8) & 0xff;  o.y = run;
      run += (cur.w[q] >> 16) & 0xff; o.z = run;
      run += cur.w[q] >> 24;          o.w = run;
      *reinterpret_cast<uint4*>(trow + 4 * q) = o;
    }
    __syncwarp();
    // ---- lane = column ----
    uint32_t* dst = b.sat + (long long)cur.s * g.W * g.H + (long long)cur.Y0 * g.W + cur.X0 + lane;
    uint32_t col = 0;
    const bool cin = lane < cur.tw;
#pragma unroll 8
    for (int r = 0; r < cur.th; r++) {
      col += tile[r * SAT_PITCH + lane];
      if (cin) dst[(long long)r * g.W] = col;
    }
    __syncwarp();
    cur = nxt;
  }
}

// Strip carries for stand-alone use (the pipeline computes them in k_worklist).
__global__ void k_carries(const __grid_constant__ Geo g, const __grid_constant__ Bufs b)
{
  strip_carries(g, b, b.s0 + blockIdx.y, blockIdx.x);
}

// ============================================================================
// k_pyramid4: k_pyramid specialised for the benchmark geometry -- O = 4,
// 96 x 48 o0 tiles, IDDM on the top octave.  Same arithmetic, static thread
// maps: the eight levels are produced in four phases (level pairs that do not
// depend on each other share a phase), four pixels per 32-bit word.
// ============================================================================
// 2x2 rounded halving of two rows of 4 bytes: the two outputs sit in bytes 0
// and 2 of the result (16-bit lanes; bits above a lane's byte are garbage, the
// callers extract bytes).  Byte gathers by PRMT instead of shift + mask.
__device__ __forceinline__ uint32_t halve_w(uint32_t a, uint32_t c)
{
  const uint32_t e = __byte_perm(a, 0u, 0x4240) + __byte_perm(a, 0u, 0x4341) + __byte_perm(c, 0u, 0x4240) +
                     __byte_perm(c, 0u, 0x4341) + 0x00020002u;   // lane sums <= 1022
  return e >> 2;
}
__device__ __forceinline__ uint32_t halve4(const uint2 r0, const uint2 r1)
{
  return __byte_perm(halve_w(r0.x, r1.x), halve_w(r0.y, r1.y), 0x6420);
}

__device__ __forceinline__ void store_word(uint8_t* gdst, int gp, int y, int x, int vw, int vh, uint32_t w)
{
  if (y >= vh || x >= vw) return;
  if (x + 4 <= vw) *reinterpret_cast<uint32_t*>(gdst + (long long)y * gp + x) = w;
  else for (int c = 0; c < 4 && x + c < vw; c++) gdst[(long long)y * gp + x + c] = (uint8_t)(w >> (8 * c));
}

// PART selects the work (the split pyramid of masked frames):
//   PYR_FULL   every level (frame 0, mode none, binning);
//   PYR_OCHAIN o1, o2, o3 + IDDM + SAT row sums for every tile; streams whose
//              frame is unmasked also get the intra-octave chain here;
//   PYR_ICHAIN i0..i3 of masked streams, only for tiles whose derived pixels a
//              FAST score can read: an active top-octave cell within
//              g.pyr_halo o0 pixels of the tile (a FAST ring reaches 3 layer
//              pixels, <= 3 * W / w_i3 o0 pixels).  FAST reads the other
//              pixels only for gated-off positions, whose results are dropped.
#define PYR_FULL 0
#define PYR_OCHAIN 1
#define PYR_ICHAIN 2
template <int PART>
__global__ void __launch_bounds__(256) k_pyramid4(const __grid_constant__ Geo g, const __grid_constant__ Bufs b)
{
  constexpr int TW = 96, TH = 48;
  __shared__ __align__(16) uint8_t t0[TH * TW];
  __shared__ __align__(16) uint8_t si0[32 * 64], so1[24 * 48], si1[16 * 32], so2[12 * 24], si2[8 * 16];
  __shared__ __align__(16) uint8_t so3[6 * 12 + 8];
  const int s = b.s0 + blockIdx.z, tid = threadIdx.x;
  const int X0 = blockIdx.x * TW, Y0 = blockIdx.y * TH;
  const bool masked = PART != PYR_FULL && use_mask(g, b, s);
  const bool do_o = PART != PYR_ICHAIN;
  const bool do_i = PART != PYR_OCHAIN || !masked;
  if (PART == PYR_ICHAIN) {
    if (!masked) return;   // built by the PYR_OCHAIN launch
    const GridGeo& G = g.grid[0];
    const int cx0 = max(0, X0 - g.pyr_halo) / G.cw, cx1 = min(G.cols - 1, (X0 + TW - 1 + g.pyr_halo) / G.cw);
    const int cy0 = max(0, Y0 - g.pyr_halo) / G.ch, cy1 = min(G.rows - 1, (Y0 + TH - 1 + g.pyr_halo) / G.ch);
    const int wa = cx0 >> 5, nwd = (cx1 >> 5) - wa + 1, n = (cy1 - cy0 + 1) * nwd;
    uint32_t any = 0;
    if (tid < n) {
      const int r = tid / nwd, k = tid - r * nwd;
      const uint32_t* bits = b.cbits + ((long long)s * 2 + (stream_epoch(b, s) & 1)) * G.rows * g.cbits_words;
      uint32_t v = __ldcg(bits + (long long)(cy0 + r) * g.cbits_words + wa + k);
      if (k == 0) v &= 0xffffffffu << (cx0 & 31);
      if (k == nwd - 1) v &= 0xffffffffu >> (31 - (cx1 & 31));
      any = v;
    }
    if (!__syncthreads_or(any != 0)) return;
  }
  if (PART != PYR_ICHAIN && blockIdx.x == 0 && blockIdx.y == 0) {
    if (tid == 0) {
      b.ctr[s * C_NCTR + C_STAGE] = 0;
      b.ctr[s * C_NCTR + C_NGLOB] = 0;
      b.nms_cnt[4 * s] = 0; b.nms_cnt[4 * s + 1] = 0;
      b.sat_count[s] = 0;
      b.work_count[s] = 0;
    }
    for (int i = tid; i < g.sty * g.stw_words; i += blockDim.x) b.sat_bits[(long long)s * g.sty * g.stw_words + i] = 0u;
    if (g.use_cbits) {
      // the other parity's bit mask, written by the next step (this step's
      // other CTAs write parity epoch & 1)
      const int nw = g.grid[0].rows * g.cbits_words;
      uint32_t* nb = b.cbits + ((long long)s * 2 + ((stream_epoch(b, s) + 1) & 1)) * nw;
      for (int i = tid; i < nw; i += blockDim.x) nb[i] = 0u;
    }
  }
  const int tw = min(TW, g.W - X0), th = min(TH, g.H - Y0);
  // an o0 tile inside the frame has every derived tile inside its layer (the
  // tile origin is a multiple of 3 * 2^(O-1)): plain word stores, no bounds
  const bool interior = tw == TW && th == TH;
  // derived tile origins of layer l (o0 tile origin x 2/3 and / 2^k; multiples
  // of 3 * 2^(O-1) divide exactly) and their global base pointers, once per CTA
  __shared__ uint8_t* lbase[8];
  __shared__ int lgx[8], lgy[8];
  if (tid >= 1 && tid < 8) {
    const int k = (tid - 1) >> 1;                        // i_k (odd l) / o_(k+1) (even l)
    const int gx0 = (tid & 1) ? (2 * X0 / 3) >> k : X0 >> (k + 1);
    const int gy0 = (tid & 1) ? (2 * Y0 / 3) >> k : Y0 >> (k + 1);
    const LayerGeo& L = g.L[tid];
    lgx[tid] = gx0;
    lgy[tid] = gy0;
    lbase[tid] = b.layers + (long long)s * g.layer_slab + L.layer_off + (long long)gy0 * L.pitch + gx0;
  }
  auto put = [&](int l, int gx0, int gy0, int y, int x, uint32_t w) {
    (void)gx0;
    (void)gy0;
    const LayerGeo& L = g.L[l];
    uint8_t* gd = lbase[l];
    if (interior) *reinterpret_cast<uint32_t*>(gd + y * L.pitch + x) = w;
    else store_word(gd, L.pitch, y, x, L.w - lgx[l], L.h - lgy[l], w);
  };
  // ---- o0 tile ----
  {
    const uint8_t* src = b.frames + (long long)(s - b.s0) * b.frame_stride + (long long)Y0 * b.frame_pitch + X0;
    const bool vec = ((reinterpret_cast<uintptr_t>(src) | (uintptr_t)b.frame_pitch) & 15) == 0 && tw == TW;
    if (vec) {
      for (int i = tid; i < th * (TW / 16); i += 256) {
        const int y = i / (TW / 16), c = i - y * (TW / 16);
        *reinterpret_cast<uint4*>(t0 + y * TW + 16 * c) =
            __ldg(reinterpret_cast<const uint4*>(src + (long long)y * b.frame_pitch) + c);
      }
    } else {
      for (int i = tid; i < th * TW; i += 256) {
        const int y = i / TW, x = i - y * TW;
        t0[i] = x < tw ? __ldg(src + (long long)y * b.frame_pitch + x) : 0;
      }
    }
  }
  __syncthreads();
  // ---- phase 1: i0 (2/3 resample) + o1 (halving) + row sums ----
  if (do_i) {
    // i0: 16 row pairs x 16 words, one 2x4 block per thread
    const int p = tid >> 4, q = tid & 15;
    const int base = 6 * q, al = base & ~3, sh = 8 * (base & 3);
    // row r's six input bytes c0..c5 as L = (c0, c1, c2, c3), M = (c3, c4, c5, -)
    uint32_t L[3], M[3];
#pragma unroll
    for (int r = 0; r < 3; r++) {
      const uint32_t* row = reinterpret_cast<const uint32_t*>(t0 + (3 * p + r) * TW + al);
      const uint32_t w0 = row[0], w1 = row[1];   // the group starts at byte 0 or 2 of w0 (6q mod 4)
      L[r] = __funnelshift_r(w0, w1, sh);
      M[r] = sh == 0 ? (w1 << 8 | w0 >> 24) : (w1 >> 8);
    }
    // each output is one dp4a of a 2x2 input block with the separable weights
    // (2, 1) x (2, 1) of _two_thirds (pyramid.py:76-94): even output row from
    // rows 0-1, odd from rows 1-2; left output column of a pair from columns
    // (0, 1), right from (1, 2) of its 3-column group
    auto div9 = [](uint32_t v) { return (v * 7282u + 29128u) >> 16; };   // (v + 4) // 9, v + 4 < 32768
    const uint32_t WL = 0x01020204u, WR = 0x02010402u;                   // bytes (a0 a1 b0 b1): 4 2 2 1 | 2 4 1 2
    const uint32_t WLo = 0x02040102u, WRo = 0x04020201u;                 // odd rows: 2 1 4 2 | 1 2 2 4
    const uint32_t e0 = div9(__dp4a(__byte_perm(L[0], L[1], 0x5410), WL, 0u));
    const uint32_t e1 = div9(__dp4a(__byte_perm(L[0], L[1], 0x6521), WR, 0u));
    const uint32_t e2 = div9(__dp4a(__byte_perm(M[0], M[1], 0x5410), WL, 0u));
    const uint32_t e3 = div9(__dp4a(__byte_perm(M[0], M[1], 0x6521), WR, 0u));
    const uint32_t o0 = div9(__dp4a(__byte_perm(L[1], L[2], 0x5410), WLo, 0u));
    const uint32_t o1 = div9(__dp4a(__byte_perm(L[1], L[2], 0x6521), WRo, 0u));
    const uint32_t o2 = div9(__dp4a(__byte_perm(M[1], M[2], 0x5410), WLo, 0u));
    const uint32_t o3 = div9(__dp4a(__byte_perm(M[1], M[2], 0x6521), WRo, 0u));
    const uint32_t e = __byte_perm(__byte_perm(e0, e1, 0x0040), __byte_perm(e2, e3, 0x0040), 0x5410);
    const uint32_t o = __byte_perm(__byte_perm(o0, o1, 0x0040), __byte_perm(o2, o3, 0x0040), 0x5410);
    *reinterpret_cast<uint32_t*>(si0 + (2 * p) * 64 + 4 * q) = e;
    *reinterpret_cast<uint32_t*>(si0 + (2 * p + 1) * 64 + 4 * q) = o;
    put(1, 2 * X0 / 3, 2 * Y0 / 3, 2 * p, 4 * q, e);
    put(1, 2 * X0 / 3, 2 * Y0 / 3, 2 * p + 1, 4 * q, o);
  }
  for (int i = tid; do_o && i < 24 * 12; i += 256) {
    const int y = i / 12, q = i - y * 12;
    const uint32_t w = halve4(*reinterpret_cast<const uint2*>(t0 + (2 * y) * TW + 8 * q),
                              *reinterpret_cast<const uint2*>(t0 + (2 * y + 1) * TW + 8 * q));
    *reinterpret_cast<uint32_t*>(so1 + y * 48 + 4 * q) = w;
    put(2, X0 >> 1, Y0 >> 1, y, 4 * q, w);
  }
  if (do_o && tid < 3 * th) {
    // row sums per 32-px SAT column of the tile (strip carries of the SATs)
    const int y = tid / 3, k = tid - 3 * y, col = 3 * blockIdx.x + k;
    const uint32_t* row = reinterpret_cast<const uint32_t*>(t0 + y * TW + VF_ST * k);
    uint32_t a = 0;
#pragma unroll
    for (int q = 0; q < VF_ST / 4; q++) a = __dp4a(row[q], 0x01010101u, a);
    if (col < g.stx) b.rowsum[((long long)s * g.H + Y0 + y) * g.stx + col] = a;
  }
  __syncthreads();
  // ---- phase 2: i1 from i0, o2 from o1 ----
  if (tid < 128) {
    if (do_i) {
    const int y = tid >> 3, q = tid & 7;
    const uint32_t w = halve4(*reinterpret_cast<const uint2*>(si0 + (2 * y) * 64 + 8 * q),
                              *reinterpret_cast<const uint2*>(si0 + (2 * y + 1) * 64 + 8 * q));
    *reinterpret_cast<uint32_t*>(si1 + y * 32 + 4 * q) = w;
    put(3, (2 * X0 / 3) >> 1, (2 * Y0 / 3) >> 1, y, 4 * q, w);
    }
  } else if (do_o && tid < 128 + 72) {
    const int i = tid - 128, y = i / 6, q = i - y * 6;
    const uint32_t w = halve4(*reinterpret_cast<const uint2*>(so1 + (2 * y) * 48 + 8 * q),
                              *reinterpret_cast<const uint2*>(so1 + (2 * y + 1) * 48 + 8 * q));
    *reinterpret_cast<uint32_t*>(so2 + y * 24 + 4 * q) = w;
    put(4, X0 >> 2, Y0 >> 2, y, 4 * q, w);
  }
  __syncthreads();
  // ---- phase 3: i2 from i1, o3 from o2 ----
  if (do_i && tid < 32) {
    const int y = tid >> 2, q = tid & 3;
    const uint32_t w = halve4(*reinterpret_cast<const uint2*>(si1 + (2 * y) * 32 + 8 * q),
                              *reinterpret_cast<const uint2*>(si1 + (2 * y + 1) * 32 + 8 * q));
    *reinterpret_cast<uint32_t*>(si2 + y * 16 + 4 * q) = w;
    put(5, (2 * X0 / 3) >> 2, (2 * Y0 / 3) >> 2, y, 4 * q, w);
  } else if (do_o && tid >= 32 && tid < 32 + 18) {
    const int i = tid - 32, y = i / 3, q = i - y * 3;
    const uint32_t w = halve4(*reinterpret_cast<const uint2*>(so2 + (2 * y) * 24 + 8 * q),
                              *reinterpret_cast<const uint2*>(so2 + (2 * y + 1) * 24 + 8 * q));
    *reinterpret_cast<uint32_t*>(so3 + y * 12 + 4 * q) = w;
    put(6, X0 >> 3, Y0 >> 3, y, 4 * q, w);
  }
  __syncthreads();
  // ---- phase 4: i3 from i2; IDDM on o3 (masking.py:84-93) ----
  if (do_i && tid < 8) {
    const int y = tid >> 1, q = tid & 1;
    const uint32_t w = halve4(*reinterpret_cast<const uint2*>(si2 + (2 * y) * 16 + 8 * q),
                              *reinterpret_cast<const uint2*>(si2 + (2 * y + 1) * 16 + 8 * q));
    put(7, (2 * X0 / 3) >> 3, (2 * Y0 / 3) >> 3, y, 4 * q, w);
  }
  if (do_o && g.mask_mode == 1 && tid >= 32 && tid < 128) {
    unsigned long long covered = 0;
    const int i = tid - 32;
    const LayerGeo& L = g.L[6];
    const int gx0 = X0 >> 3, gy0 = Y0 >> 3;
    const bool um = use_mask(g, b, s);
    int mybit = 0;
    if (i < 72) {
      const int y = i / 12, x = i - y * 12;
      if (gy0 + y < L.h && gx0 + x < L.w) {
        const GridGeo& G = g.grid[0];
        const long long gi = (long long)(gy0 + y) * L.w + gx0 + x;
        uint8_t* st = iddm_state(g, b, s, 3, 0);
        const int c = so3[y * 12 + x];
        if (um) {
          int d = c - (int)iddm_state(g, b, s, 3, 1)[gi];
          d = d < 0 ? -d : d;
          const int bit = (double)d > g.t_i;   // int16 diff vs float t_i, strict
          b.cells[(long long)s * g.cell_slab + G.cell_off + gi] = (uint8_t)bit;
          mybit = bit;
          if (bit) {
            long long hy = g.H - (long long)(gy0 + y) * G.ch, hx = g.W - (long long)(gx0 + x) * G.cw;
            hy = hy < G.ch ? hy : G.ch;
            hx = hx < G.cw ? hx : G.cw;
            if (hy > 0 && hx > 0) covered = (unsigned long long)(hy * hx);
          }
        }
        st[gi] = (uint8_t)c;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) covered += __shfl_down_sync(0xffffffffu, covered, o);
    if ((tid & 31) == 0 && covered) atomicAdd(b.cov + s, covered);
    if (g.use_cbits && um) {
      // cells i = 32 (w - 1) + lane of this warp as bits: the pieces of tile
      // rows (12 cells each) OR-ed into the stream's cell-row words
      const unsigned bal = __ballot_sync(0xffffffffu, mybit);
      const int lane = tid & 31, ibase = i - lane;
      if (bal && lane < 4) {
        const int y = ibase / 12 + lane;            // rows meeting this warp's 32 cells
        const int a = max(12 * y, ibase), e = min(min(12 * y + 12, ibase + 32), 72);
        if (a < e && gy0 + y < g.grid[0].rows) {
          const uint32_t piece = (bal >> (a - ibase)) & ((1u << (e - a)) - 1u);
          if (piece) {
            const int gx = gx0 + (a - 12 * y), sh = gx & 31;
            uint32_t* row = b.cbits + ((long long)s * 2 + (stream_epoch(b, s) & 1)) * g.grid[0].rows * g.cbits_words +
                            (long long)(gy0 + y) * g.cbits_words + (gx >> 5);
            atomicOr(row, piece << sh);
            if (sh + (e - a) > 32) atomicOr(row + 1, piece >> (32 - sh));
          }
        }
      }
    }
  }
}

// ============================================================================
// Warp-strip pyramid (O = 4): two launches without shared memory or block
// barriers, every lane loading all of its input bytes at once.
//
// k_pyr_o: warp per strip of 8 o0 rows x 512 o0 columns (lane: 16 columns).
//   o1 (4 rows x 8 px per lane), o2 (2 rows x 4 px), o3 (2 px) by the 2x2
//   rounded halving of pyramid.py:67-73; the IDDM of masking.py:84-93 on o3
//   (two top-octave cells per lane; two ballots are the strip's two words of
//   the bit mask);
//   the per-32-column SAT row sums of the 8 rows.  Block 0 of each stream
//   also resets the per-step counters.
// k_pyr_i: warp per unit of 48 o0 rows x 96 o0 columns (lane: a 12 x 12 block;
//   PYI_LPR lanes side by side, 32 / PYI_LPR row groups).  The unit is the
//   granularity of the activity gate below: a compact unit plus its halo
//   covers ~3x fewer o0 pixels per active cell than a 12 x 384 strip did.
//   i0 (8 rows x 8 px per lane) by the 2/3 area resample of pyramid.py:76-94
//   (one dp4a of a 2x2 input block with the separable (2, 1) x (2, 1)
//   weights, then (v + 4) // 9 by multiply-shift), i1 (4 x 4), i2 (2 x 2),
//   i3 (1) by halving.  In masked frames only units with an active top-octave
//   cell within g.pyr_halo o0 pixels run (a FAST ring reaches 3 layer pixels
//   of a gated pixel, <= 3 W / w_i3 o0 pixels); FAST reads the other pixels
//   only for gated-off positions, whose scores are dropped.
// ============================================================================
#define PYO_COLS 512
#ifndef PYI_LPR
#define PYI_LPR 8                 // lanes per row group of a k_pyr_i warp unit
#endif
#define PYI_COLS (12 * PYI_LPR)   // unit width (o0 columns)
#define PYI_RG (32 / PYI_LPR)     // row groups (12 o0 rows each) per unit
__device__ __forceinline__ void store_bytes(uint8_t* row, int x, int valid, uint32_t w, int n)
{
  // n bytes of w at row[x..x+n) (x aligned to n), clipped to `valid` columns
  if (x + n <= valid) {
#ifdef VF_DEBUG
    if (reinterpret_cast<uintptr_t>(row + x) & (n - 1)) printf("store_bytes x %d n %d\n", x, n);
#endif
    if (n == 4) *reinterpret_cast<uint32_t*>(row + x) = w;
    else if (n == 2) *reinterpret_cast<uint16_t*>(row + x) = (uint16_t)w;
    else row[x] = (uint8_t)w;
  } else {
    for (int c = 0; c < n && x + c < valid; c++) row[x + c] = (uint8_t)(w >> (8 * c));
  }
}

// Up to 4 bytes at p (clipped to `valid` bytes), packed little-endian: the
// edge lanes of the strip kernels (kept out of line; returns a value so the
// callers' row arrays stay in registers).
__device__ __noinline__ uint32_t load_edge4(const uint8_t* p, int valid)
{
  uint32_t w = 0u;
  for (int c = 0; c < 4 && c < valid; c++) w |= (uint32_t)__ldg(p + c) << (8 * c);
  return w;
}

// 2x2 rounded halving of two rows of 16 bytes -> 8 bytes (pyramid.py:67-73)
__device__ __forceinline__ uint2 halve8(const uint4 a, const uint4 c)
{
  return make_uint2(halve4(make_uint2(a.x, a.y), make_uint2(c.x, c.y)), halve4(make_uint2(a.z, a.w), make_uint2(c.z, c.w)));
}

__global__ void __launch_bounds__(256) k_pyr_o(const __grid_constant__ Geo g, const __grid_constant__ Bufs b)
{
  const int s = b.s0 + blockIdx.y, lane = threadIdx.x & 31;
  if (blockIdx.x == 0) {
    if (threadIdx.x == 0) {
      b.ctr[s * C_NCTR + C_STAGE] = 0;
      b.ctr[s * C_NCTR + C_NGLOB] = 0;
      b.nms_cnt[4 * s] = 0; b.nms_cnt[4 * s + 1] = 0;
      b.sat_count[s] = 0;
      b.work_count[s] = 0;
    }
    for (int i = threadIdx.x; i < g.sty * g.stw_words; i += blockDim.x) b.sat_bits[(long long)s * g.sty * g.stw_words + i] = 0u;
  }
  const int nsx = (g.W + PYO_COLS - 1) / PYO_COLS;
  const int strip = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int sy = strip / nsx, sx = strip - sy * nsx;
  const int h1 = g.L[2].h;
  if (sy * 4 >= h1) return;
  const int X = sx * PYO_COLS + 16 * lane, Y = sy * 8, W = g.W, H = g.H;
  const int nr = min(8, H - Y);              // o0 rows present (>= 2)
  // ---- 8 o0 rows x 16 columns of this lane ----
  const uint8_t* src = b.frames + (long long)(s - b.s0) * b.frame_stride + (long long)Y * b.frame_pitch + X;
  const int pitch = (int)b.frame_pitch;
  const bool vec = ((reinterpret_cast<uintptr_t>(b.frames) | (uintptr_t)b.frame_pitch | (uintptr_t)b.frame_stride) & 15) == 0;
  uint4 r[8];
  if (vec && X + 16 <= W && nr == 8) {
#pragma unroll
    for (int k = 0; k < 8; k++) r[k] = __ldg(reinterpret_cast<const uint4*>(src + k * pitch));
  } else {
#pragma unroll
    for (int k = 0; k < 8; k++) {
      const bool ok = k < nr && X < W;
      const uint8_t* p = src + k * pitch;
      r[k] = make_uint4(ok ? load_edge4(p, W - X) : 0u, ok && X + 4 < W ? load_edge4(p + 4, W - X - 4) : 0u,
                        ok && X + 8 < W ? load_edge4(p + 8, W - X - 8) : 0u,
                        ok && X + 12 < W ? load_edge4(p + 12, W - X - 12) : 0u);
    }
  }
  // the previous frame's top-octave pixels for the IDDM, loaded beside the rows
  const LayerGeo& L3 = g.L[6];
  const int x3 = X / 8, y3 = sy;
  const bool in3a = x3 < L3.w && y3 < L3.h, in3b = x3 + 1 < L3.w && y3 < L3.h;
  const int gi = y3 * L3.w + x3;
  const bool um = g.mask_mode == 1 && use_mask(g, b, s);
  int p3a = 0, p3b = 0;
  if (um) {
    const uint8_t* stp = iddm_state(g, b, s, 3, 1);
    if (in3a) p3a = stp[gi];
    if (in3b) p3b = stp[gi + 1];
  }
  // ---- SAT row sums: 32-column segments = 2 lanes ----
  {
    const int col = X / VF_ST;
    uint32_t* rs = b.rowsum + ((long long)s * H + Y) * g.stx + col;
    const bool wr = (lane & 1) == 0 && col < g.stx;
#pragma unroll
    for (int k = 0; k < 8; k++) {
      uint32_t a = __dp4a(r[k].w, 0x01010101u, __dp4a(r[k].z, 0x01010101u,
                   __dp4a(r[k].y, 0x01010101u, __dp4a(r[k].x, 0x01010101u, 0u))));
      a += __shfl_xor_sync(0xffffffffu, a, 1);
      if (wr && k < nr) rs[k * g.stx] = a;
    }
  }
  uint8_t* lay = b.layers + (long long)s * g.layer_slab;
  // ---- o1: 4 rows x 8 px ----
  const LayerGeo& L1 = g.L[2];
  uint2 w1[4];
  {
    const int x1 = X / 2;
    uint8_t* o1 = lay + L1.layer_off + (long long)(4 * sy) * L1.pitch + x1;
    const int n1 = min(4, h1 - 4 * sy);
    const bool full = x1 + 8 <= L1.w;
#pragma unroll
    for (int k = 0; k < 4; k++) {
      w1[k] = halve8(r[2 * k], r[2 * k + 1]);
      if (k < n1) {
        if (full) *reinterpret_cast<uint2*>(o1 + k * L1.pitch) = w1[k];
        else if (x1 < L1.w) {
          store_bytes(o1 + k * L1.pitch - x1, x1, L1.w, w1[k].x, 4);
          if (x1 + 4 < L1.w) store_bytes(o1 + k * L1.pitch - x1, x1 + 4, L1.w, w1[k].y, 4);
        }
      }
    }
  }
  // ---- o2: 2 rows x 4 px ----
  const LayerGeo& L2 = g.L[4];
  uint32_t w2[2];
  {
    const int x2 = X / 4;
    uint8_t* o2 = lay + L2.layer_off + (long long)(2 * sy) * L2.pitch + x2;
    const int n2 = min(2, L2.h - 2 * sy);
#pragma unroll
    for (int k = 0; k < 2; k++) {
      w2[k] = halve4(w1[2 * k], w1[2 * k + 1]);
      if (k < n2 && x2 < L2.w) store_bytes(o2 + k * L2.pitch - x2, x2, L2.w, w2[k], 4);
    }
  }
  // ---- o3: 1 row x 2 px ----
  const uint32_t q3 = halve_w(w2[0], w2[1]);
  const int c3a = (int)(q3 & 0xffu), c3b = (int)((q3 >> 16) & 0xffu);
  uint8_t* o3 = lay + L3.layer_off + (long long)y3 * L3.pitch + x3;
  if (in3b) *reinterpret_cast<uint16_t*>(o3) = (uint16_t)(c3a | (c3b << 8));
  else if (in3a) *o3 = (uint8_t)c3a;
  // ---- IDDM on o3 (masking.py:84-93): int16 diff vs float t_i, strict ----
  if (g.mask_mode == 1) {
    const GridGeo& G = g.grid[0];
    uint8_t* st = iddm_state(g, b, s, 3, 0);
    int bits = 0;
    unsigned covered = 0;
    if (um) {
      uint8_t* cl = b.cells + (long long)s * g.cell_slab + G.cell_off;
      if (in3a) {
        const int d = abs(c3a - p3a);
        const int bit = (double)d > g.t_i;
        cl[gi] = (uint8_t)bit;
        bits = bit;
        if (bit) covered += (unsigned)(min(G.ch, H - y3 * G.ch) * min(G.cw, W - x3 * G.cw));
      }
      if (in3b) {
        const int d = abs(c3b - p3b);
        const int bit = (double)d > g.t_i;
        cl[gi + 1] = (uint8_t)bit;
        bits |= bit << 1;
        if (bit) covered += (unsigned)(min(G.ch, H - y3 * G.ch) * min(G.cw, W - (x3 + 1) * G.cw));
      }
    }
    if (in3a) st[gi] = (uint8_t)c3a;
    if (in3b) st[gi + 1] = (uint8_t)c3b;
    if (um) {
      // cell 32 k + lane of the strip belongs to lane (32 k + lane) / 2, pixel lane & 1
      const uint32_t wk0 = __ballot_sync(0xffffffffu, (__shfl_sync(0xffffffffu, bits, lane >> 1) >> (lane & 1)) & 1);
      const uint32_t wk1 = __ballot_sync(0xffffffffu, (__shfl_sync(0xffffffffu, bits, 16 + (lane >> 1)) >> (lane & 1)) & 1);
      if (wk0 | wk1) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) covered += __shfl_down_sync(0xffffffffu, covered, o);
      }
      if (lane < 2) {
        if (lane == 0 && covered) atomicAdd(b.cov + s, (unsigned long long)covered);
        const int wd = 2 * sx + lane;   // cells 32 wd .. 32 wd + 31 of row y3
        if (g.use_cbits && y3 < G.rows && wd < g.cbits_words)
          b.cbits[((long long)s * 2 + (stream_epoch(b, s) & 1)) * G.rows * g.cbits_words + (long long)y3 * g.cbits_words +
                  wd] = lane ? wk1 : wk0;
      }
    }
  }
}

__device__ __forceinline__ uint32_t div9x(uint32_t v) { return (v * 7282u + 29128u) >> 16; }   // (v + 4) // 9

__global__ void __launch_bounds__(256) k_pyr_i(const __grid_constant__ Geo g, const __grid_constant__ Bufs b)
{
  const int s = b.s0 + blockIdx.y, lane = threadIdx.x & 31;
  const int nsx = (g.W + PYI_COLS - 1) / PYI_COLS;
  const int strip = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int sy = strip / nsx, sx = strip - sy * nsx;
  const LayerGeo& Li0 = g.L[1];
  if (sy * PYI_RG * 8 >= Li0.h) return;
  // the lane's 12 x 12 o0 block: row group ry (12 o0 rows -> 8 i0 rows),
  // column group cx (12 o0 columns -> 8 i0 columns)
  const int ry = sy * PYI_RG + lane / PYI_LPR, cx = sx * PYI_LPR + lane % PYI_LPR;
  const int X = 12 * cx, Y = 12 * ry;
  if (g.use_cbits && use_mask(g, b, s)) {
    // any active top-octave cell within pyr_halo o0 pixels of the unit?
    const GridGeo& G = g.grid[0];
    const int X0 = sx * PYI_COLS, Y0 = sy * PYI_RG * 12;
    const int cx0 = max(0, X0 - g.pyr_halo) / G.cw, cx1 = min(G.cols - 1, (X0 + PYI_COLS - 1 + g.pyr_halo) / G.cw);
    const int cy0 = max(0, Y0 - g.pyr_halo) / G.ch, cy1 = min(G.rows - 1, (Y0 + 12 * PYI_RG - 1 + g.pyr_halo) / G.ch);
    const int wa = cx0 >> 5, wb = cx1 >> 5;
    const uint32_t mh = 0xffffffffu << (cx0 & 31), mt = 0xffffffffu >> (31 - (cx1 & 31));
    const uint32_t* bits = b.cbits + ((long long)s * 2 + (stream_epoch(b, s) & 1)) * G.rows * g.cbits_words + wa;
    uint32_t any = 0;
    for (int r = cy0 + lane; r <= cy1; r += 32) {   // lane per cell row
      const uint32_t* rw = bits + (long long)r * g.cbits_words;
      for (int k = 0; k <= wb - wa; k++) {
        uint32_t v = __ldcg(rw + k);
        if (k == 0) v &= mh;
        if (k == wb - wa) v &= mt;
        any |= v;
      }
    }
    if (!__any_sync(0xffffffffu, any != 0u)) return;
  }
  if (ry * 8 >= Li0.h) return;
  // ---- 12 o0 rows x 12 columns of this lane (3 words per row) ----
  const uint8_t* src = b.frames + (long long)(s - b.s0) * b.frame_stride + (long long)Y * b.frame_pitch + X;
  const int pitch = (int)b.frame_pitch;
  const bool vec = ((reinterpret_cast<uintptr_t>(b.frames) | (uintptr_t)b.frame_pitch | (uintptr_t)b.frame_stride) & 3) == 0;
  uint32_t r[12][3];
  if (vec && X + 12 <= g.W && Y + 12 <= g.H) {
#pragma unroll
    for (int k = 0; k < 12; k++)
#pragma unroll
      for (int q = 0; q < 3; q++) {
#ifdef VF_DEBUG
        if ((reinterpret_cast<uintptr_t>(src + k * pitch) & 3)) printf("pyr_i load X %d\n", X);
#endif
        r[k][q] = __ldg(reinterpret_cast<const uint32_t*>(src + k * pitch) + q);
      }
  } else {
#pragma unroll
    for (int k = 0; k < 12; k++) {
      const bool ok = Y + k < g.H && X < g.W;
#pragma unroll
      for (int q = 0; q < 3; q++) r[k][q] = ok ? load_edge4(src + k * pitch + 4 * q, g.W - X - 4 * q) : 0u;
    }
  }
  // ---- i0: 8 rows x 8 px (2 words) per lane ----
  // a 3-row x 6-column group gives a 2 x 4 output block: row bytes c0..c5 as
  // L = (c0, c1, c2, c3), M = (c3, c4, c5, -); each output is one dp4a of a
  // 2x2 input block with the weights 4 2 2 1 (and mirrors), then // 9
  const uint32_t WL = 0x01020204u, WR = 0x02010402u, WLo = 0x02040102u, WRo = 0x04020201u;
  uint32_t i0w[8][2];
#pragma unroll
  for (int t = 0; t < 4; t++) {          // row triple t -> i0 rows 2t, 2t + 1
#pragma unroll
    for (int h = 0; h < 2; h++) {        // 6-column half h -> i0 px 4h .. 4h + 3
      uint32_t Lr[3], Mr[3];
#pragma unroll
      for (int k = 0; k < 3; k++) {
        const uint32_t* rw = r[3 * t + k];
        // columns 6h .. 6h + 5: h = 0 -> bytes 0..5 (word 0, word 1 low half); h = 1 -> bytes 6..11
        Lr[k] = h == 0 ? rw[0] : __funnelshift_r(rw[1], rw[2], 16);
        Mr[k] = h == 0 ? __funnelshift_r(rw[0], rw[1], 24) : (rw[2] >> 8);
      }
      const uint32_t e0 = div9x(__dp4a(__byte_perm(Lr[0], Lr[1], 0x5410), WL, 0u));
      const uint32_t e1 = div9x(__dp4a(__byte_perm(Lr[0], Lr[1], 0x6521), WR, 0u));
      const uint32_t e2 = div9x(__dp4a(__byte_perm(Mr[0], Mr[1], 0x5410), WL, 0u));
      const uint32_t e3 = div9x(__dp4a(__byte_perm(Mr[0], Mr[1], 0x6521), WR, 0u));
      const uint32_t o0 = div9x(__dp4a(__byte_perm(Lr[1], Lr[2], 0x5410), WLo, 0u));
      const uint32_t o1 = div9x(__dp4a(__byte_perm(Lr[1], Lr[2], 0x6521), WRo, 0u));
      const uint32_t o2 = div9x(__dp4a(__byte_perm(Mr[1], Mr[2], 0x5410), WLo, 0u));
      const uint32_t o3 = div9x(__dp4a(__byte_perm(Mr[1], Mr[2], 0x6521), WRo, 0u));
      i0w[2 * t][h] = __byte_perm(__byte_perm(e0, e1, 0x0040), __byte_perm(e2, e3, 0x0040), 0x5410);
      i0w[2 * t + 1][h] = __byte_perm(__byte_perm(o0, o1, 0x0040), __byte_perm(o2, o3, 0x0040), 0x5410);
    }
  }
  uint8_t* lay = b.layers + (long long)s * g.layer_slab;
  const int xi0 = 8 * cx;   // = 2 X / 3
  {
    uint8_t* row = lay + Li0.layer_off + (long long)(8 * ry) * Li0.pitch;
    const int n0 = min(8, Li0.h - 8 * ry);
#pragma unroll
    for (int k = 0; k < 8; k++) {
      if (k < n0 && xi0 < Li0.w) {
#ifdef VF_DEBUG
        if (xi0 + 8 <= Li0.w && (reinterpret_cast<uintptr_t>(row + xi0) & 7)) printf("pyr_i i0 store xi0 %d\n", xi0);
#endif
        if (xi0 + 8 <= Li0.w) *reinterpret_cast<uint2*>(row + xi0) = make_uint2(i0w[k][0], i0w[k][1]);
        else { store_bytes(row, xi0, Li0.w, i0w[k][0], 4); if (xi0 + 4 < Li0.w) store_bytes(row, xi0 + 4, Li0.w, i0w[k][1], 4); }
      }
      row += Li0.pitch;
    }
  }
  // ---- i1: 4 rows x 4 px ----
  const LayerGeo& Li1 = g.L[3];
  uint32_t i1w[4];
#pragma unroll
  for (int k = 0; k < 4; k++) {
    i1w[k] = halve4(make_uint2(i0w[2 * k][0], i0w[2 * k][1]), make_uint2(i0w[2 * k + 1][0], i0w[2 * k + 1][1]));
    const int y = 4 * ry + k, x = 4 * cx;
    if (y < Li1.h && x < Li1.w) store_bytes(lay + Li1.layer_off + (long long)y * Li1.pitch, x, Li1.w, i1w[k], 4);
  }
  // ---- i2: 2 rows x 2 px ----
  const LayerGeo& Li2 = g.L[5];
  uint32_t i2w[2];
#pragma unroll
  for (int k = 0; k < 2; k++) {
    const uint32_t a = i1w[2 * k], c = i1w[2 * k + 1];
    i2w[k] = __byte_perm(halve_w(a, c), 0u, 0x4420);
    const int y = 2 * ry + k, x = 2 * cx;
    if (y < Li2.h && x < Li2.w) store_bytes(lay + Li2.layer_off + (long long)y * Li2.pitch, x, Li2.w, i2w[k], 2);
  }
  // ---- i3: 1 px ----
  const LayerGeo& Li3 = g.L[7];
  const int y3 = ry, x3 = cx;
  if (y3 < Li3.h && x3 < Li3.w) {
    const uint32_t sum = (i2w[0] & 0xffu) + (i2w[0] >> 8) + (i2w[1] & 0xffu) + (i2w[1] >> 8);
    lay[Li3.layer_off + (long long)y3 * Li3.pitch + x3] = (uint8_t)((sum + 2) >> 2);
  }
}

// ============================================================================
// k_binmask: masking.py:96-136 (histogram of the previous MERGED features,
// pipeline.py:184-185), thresholded at t_h; coverage = covered pixels / WH.
// ============================================================================
__global__ void __launch_bounds__(1024) k_binmask(const __grid_constant__ Geo g, const __grid_constant__ Bufs b)
{
  extern __shared__ int hist[];
  const int s = b.s0 + blockIdx.x;
  if (!use_mask(g, b, s)) return;
  const GridGeo& G = g.grid[0];
  const int n_cells = G.rows * G.cols;
  for (int i = threadIdx.x; i < n_cells; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  const int* ctr = b.ctr + s * C_NCTR;
  const int prev = (ctr[C_FRAME] & 1) ^ 1;
  const int n_prev = ctr[C_NFEAT0 + prev];
  const long long fb = feat_base(g, s, prev, n_prev);
  const double sx = (double)G.cw, sy = (double)G.ch;   // ceil(W/cols), ceil(H/rows)
  for (int i = threadIdx.x; i < n_prev; i += blockDim.x) {
    double fx = floor(b.fx[fb + i] / sx), fy = floor(b.fy[fb + i] / sy);
    long long k = (long long)fx, r = (long long)fy;
    k = k < 0 ? 0 : (k > G.cols - 1 ? G.cols - 1 : k);
    r = r < 0 ? 0 : (r > G.rows - 1 ? G.rows - 1 : r);
    atomicAdd(&hist[r * G.cols + k], 1);
  }
  __syncthreads();
  uint8_t* cells = b.cells + (long long)s * g.cell_slab + G.cell_off;
  unsigned long long covered = 0;
  for (int i = threadIdx.x; i < n_cells; i += blockDim.x) {
    int bit = hist[i] >= g.t_h;
    cells[i] = (uint8_t)bit;
    if (bit) {
      int r = i / G.cols, c = i - r * G.cols;
      long long hy = (long long)g.H - (long long)r * G.ch, hx = (long long)g.W - (long long)c * G.cw;
      hy = hy < G.ch ? hy : G.ch;
      hx = hx < G.cw ? hx : G.cw;
      if (hy > 0 && hx > 0) covered += (unsigned long long)(hy * hx);
    }
  }
  for (int o = 16; o > 0; o >>= 1) covered += __shfl_down_sync(0xffffffffu, covered, o);
  if ((threadIdx.x & 31) == 0 && covered) atomicAdd(b.cov + s, covered);
}

// ============================================================================
// k_worklist: active-tile compaction.  A FAST tile (128 x 8 layer pixels) is
// active when any cell its pixels project to (detector.py:175-181) is set;
// inactive tiles are never read or written (pipeline.py:104-117 skips).
// Extra CTAs compute the union coverage in per_layer mode.
// ============================================================================
#define PROP_CHUNK 1024
#ifndef PROP_CTAS
#define PROP_CTAS 16
#endif
#define VF_CLEAR (1 << 30)   // work-list flag: zero the tile's scores and bitmap words
__global__ void __launch_bounds__(256) k_worklist(const __grid_constant__ Geo g, const __grid_constant__ Bufs b,
                                                   int tile_ctas, int cov_ctas, int carry_ctas)
{
  const int s = b.s0 + blockIdx.y;
  const int epoch = stream_epoch(b, s);
  const int um = use_mask(g, b, s);
  const int lane = threadIdx.x & 31;
  if ((int)blockIdx.x >= tile_ctas + cov_ctas && (int)blockIdx.x < tile_ctas + cov_ctas + carry_ctas) {
    const int ty = (blockIdx.x - tile_ctas - cov_ctas) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (ty < g.sty) strip_carries(g, b, s, ty);
    return;
  }
  if ((int)blockIdx.x >= tile_ctas + cov_ctas + carry_ctas) {
    // Eq. 1 propagation counts: previous features under a 0 mask bit, per
    // 1024-feature chunk of the previous list (masking.py:176-183)
    if (!um) return;
    __shared__ int sm_warp[32];
    __shared__ int last_sm;
    int* ctr = b.ctr + s * C_NCTR;
    const int prev = (ctr[C_FRAME] & 1) ^ 1;
    const int n_prev = ctr[C_NFEAT0 + prev];
    const int nch = (n_prev + PROP_CHUNK - 1) / PROP_CHUNK;
    const long long fb = feat_base(g, s, prev, n_prev);
    for (int c = blockIdx.x - tile_ctas - cov_ctas - carry_ctas; c < nch; c += PROP_CTAS) {
      int cnt = 0;
      const int e0 = c * PROP_CHUNK + threadIdx.x * (PROP_CHUNK / 256);
#pragma unroll
      for (int k = 0; k < PROP_CHUNK / 256; k++)
        if (e0 + k < n_prev) cnt += !merge_mask_at(g, b, s, b.fx[fb + e0 + k], b.fy[fb + e0 + k]);
      int tot;
      block_excl_scan<int>(cnt, sm_warp, tot);
      if (threadIdx.x == 0) b.prop_cnt[(long long)s * g.prop_chunks + c] = tot;
    }
    // the last of the stream's count CTAs scans the chunk counts into output
    // offsets and the propagated total (known before the detection finishes)
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      last_sm = atomicAdd(ctr + C_PTICKET, 1) == PROP_CTAS - 1;
      if (last_sm) ctr[C_PTICKET] = 0;
    }
    __syncthreads();
    if (!last_sm || threadIdx.x >= 32) return;
    __threadfence();
    const int* pc = b.prop_cnt + (long long)s * g.prop_chunks;
    int* po = b.prop_out + (long long)s * g.prop_chunks;
    int carry = 0, tot;
    for (int base = 0; base < nch; base += 32) {
      const int i = base + lane;
      const int k = i < nch ? __ldcg(pc + i) : 0;
      const int ex = warp_excl_scan(k, lane, tot);
      if (i < nch) po[i] = carry + ex;
      carry += tot;
    }
    if (lane == 0) ctr[C_NPROP] = carry;
    return;
  }
  if ((int)blockIdx.x >= tile_ctas) {
    // per_layer union coverage: one warp per full-res row (masking.py:44-46)
    if (!um || !g.per_layer) return;
    const int rows_per_cta = 8;
    int y = (blockIdx.x - tile_ctas) * rows_per_cta + (threadIdx.x >> 5);
    if (y >= g.H) return;
    const uint8_t* cells = b.cells + (long long)s * g.cell_slab;
    unsigned long long cnt = 0;
    for (int x = lane; x < g.W; x += 32) {
      int v = 0;
      for (int k = 0; k < g.n_grids; k++) {
        const GridGeo& G = g.grid[k];
        v |= cells[G.cell_off + (y / G.ch) * G.cols + x / G.cw];
      }
      cnt += v;
    }
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_down_sync(0xffffffffu, cnt, o);
    if (lane == 0 && cnt) atomicAdd(b.cov + s, cnt);
    return;
  }
  // ---- FAST-tile activity (detector.py:175-181, pipeline.py:104-117) -------
  // Lane per tile: a tile is active when any cell its pixels project to is
  // set.  The default IDDM mask is read as bits (k_pyramid4), other masks as
  // bytes; the rectangle's words are loaded four at a time.
  const int tile = blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = tile < g.tiles_per_stream;
  int* st = b.tile_stamp + (long long)s * g.tiles_per_stream + tile;
  const int old_stamp = valid ? *st : 0;   // issued with the mask loads below
  int l = 0, ty = 0;
  bool active = false;
  if (valid) {
    while (l + 1 < g.NL && tile >= g.L[l + 1].tile_base) l++;
    const LayerGeo& Lg = g.L[l];
    const int t = tile - Lg.tile_base;
    ty = t / Lg.tiles_x;
    const int tx = t - ty * Lg.tiles_x;
    active = true;
    if (um) {
      const int y0 = ty * VF_TILE_H, y1 = min(Lg.h, y0 + VF_TILE_H) - 1;
      const int x0 = tx * VF_TILE_W, x1 = min(Lg.w, x0 + VF_TILE_W) - 1;
      const int* lut = b.lut + Lg.rc_off;
      const int r0 = __ldg(lut + y0), r1 = __ldg(lut + y1);
      const int c0 = __ldg(lut + Lg.h + x0), c1 = __ldg(lut + Lg.h + x1);
      const int nrow = r1 - r0 + 1;
      uint32_t any = 0;
      if (g.use_cbits) {
        const GridGeo& G = g.grid[0];
        const uint32_t* bits = b.cbits + ((long long)s * 2 + (epoch & 1)) * G.rows * g.cbits_words +
                               (long long)r0 * g.cbits_words;
        const int wa = c0 >> 5, nwd = (c1 >> 5) - wa + 1, n = nrow * nwd;
        const uint32_t mh = 0xffffffffu << (c0 & 31), mt = 0xffffffffu >> (31 - (c1 & 31));
        int r = 0, k = 0;
#pragma unroll 1
        for (int i = 0; i < n; i += 4) {
          uint32_t w[4];
#pragma unroll
          for (int j = 0; j < 4; j++) {
            uint32_t v = 0;
            if (i + j < n) {
              v = __ldcg(bits + r * g.cbits_words + wa + k);
              if (k == 0) v &= mh;
              if (k == nwd - 1) v &= mt;
            }
            w[j] = v;
            if (++k == nwd) { k = 0; r++; }
          }
          any |= w[0] | w[1] | w[2] | w[3];
        }
      } else {
        const GridGeo& G = g.grid[grid_of_layer(g, l)];
        const uint8_t* cells = b.cells + (long long)s * g.cell_slab + G.cell_off;
        // aligned 32-bit words (the cell slab is padded), partial words masked
        const uintptr_t first = reinterpret_cast<uintptr_t>(cells + c0) & ~(uintptr_t)3;
        const int nwd = (int)(((reinterpret_cast<uintptr_t>(cells + c1) & ~(uintptr_t)3) - first) / 4) + 1;
        const int head = (int)(reinterpret_cast<uintptr_t>(cells + c0) & 3);
        const int tail = (int)(reinterpret_cast<uintptr_t>(cells + c1) & 3);
        const int n = nrow * nwd;
        int r = r0, k = 0;
#pragma unroll 1
        for (int i = 0; i < n; i += 4) {
          uint32_t w[4];
#pragma unroll
          for (int j = 0; j < 4; j++) {
            uint32_t v = 0;
            if (i + j < n) {
              v = *(reinterpret_cast<const uint32_t*>(first + (uintptr_t)r * G.cols) + k);
              if (k == 0) v &= 0xffffffffu << (8 * head);
              if (k == nwd - 1) v &= 0xffffffffu >> (8 * (3 - tail));
            }
            w[j] = v;
            if (++k == nwd) { k = 0; r++; }
          }
          any |= w[0] | w[1] | w[2] | w[3];
        }
      }
      active = any != 0;
    }
  }
  // Invariant: a tile not active this step holds zero scores and bitmap words,
  // so k_nms reads maps without activity checks.  A tile active last step but
  // not now becomes a clear item (tile | VF_CLEAR) that k_fast zeroes.
  bool clear = false;
  if (valid) {
    if (active) {
      const LayerGeo& Lg = g.L[l];
      *st = epoch;
      b.band_stamp[(long long)s * g.bands_per_stream + Lg.band_base + ty] = epoch;
      b.band_cand[(long long)s * g.bands_per_stream + Lg.band_base + ty] = 0;
    } else {
      clear = old_stamp == epoch - 1;
    }
  }
  // warp-aggregated append to the work list
  const bool item = active || clear;
  const unsigned m = __ballot_sync(0xffffffffu, item);
  int pos = 0;
  if (lane == 0 && m) pos = atomicAdd(b.work_count + s, __popc(m));
  pos = __shfl_sync(0xffffffffu, pos, 0);
  if (item)
    b.worklist[(long long)s * g.tiles_per_stream + pos + __popc(m & ((1u << lane) - 1))] = tile | (clear ? VF_CLEAR : 0);
}

// ============================================================================
// k_fast: segment-test score map (detector.py:107-158) over active tiles.
// ============================================================================
// Tile 128 x 8 staged with a 3-row / 16-byte halo in smem by 16-byte loads.
// Pass 1 runs the exact 4-point necessary test (detector.py:117-125) on
// packed bytes (4 pixels per 32-bit word: saturating byte differences vs t);
// survivors go to an smem queue; pass 2 scores each queued pixel with packed
// sliding-window minima over the 16-pixel ring (max over 16 arcs of the min
// of 9 consecutive saturating differences, bright and dark), which equals
// _score_map_jit exactly.  Scores >= t are stored as
// uint8 (<= 254) plus a 1-bit candidate bitmap for the NMS.
#define FT_ROWS (VF_TILE_H + 6)
#define FT_COLS (VF_TILE_W + 32)
// Exact FAST score of one pixel from its 16-pixel ring (detector.py:127-158):
// with d_i = r_i - c, the best arc of 9 is max(max_arcs min9(r) - c,
// c - min_arcs max9(r), 0) (saturating differences are monotone in r).  The
// ring is held as 8 words of 16x2 lanes (r_2k, r_2k+1); sliding minima and
// maxima of 9 use the native 3-input VIMNMX3.U16x2.
__device__ __forceinline__ uint32_t pair_shift1(uint32_t a, uint32_t b) { return __byte_perm(a, b, 0x5432); }
__device__ __forceinline__ int fast_best(const uint32_t w[8], int c)
{
  uint32_t s1[8], mn3[8], mx3[8];
#pragma unroll
  for (int k = 0; k < 8; k++) s1[k] = pair_shift1(w[k], w[(k + 1) & 7]);
#pragma unroll
  for (int k = 0; k < 8; k++) {
    mn3[k] = __vimin3_u16x2(w[k], s1[k], w[(k + 1) & 7]);
    mx3[k] = __vimax3_u16x2(w[k], s1[k], w[(k + 1) & 7]);
  }
  uint32_t mn9[8], mx9[8];
#pragma unroll
  for (int k = 0; k < 8; k++) {
    mn9[k] = __vimin3_u16x2(mn3[k], pair_shift1(mn3[(k + 1) & 7], mn3[(k + 2) & 7]), mn3[(k + 3) & 7]);
    mx9[k] = __vimax3_u16x2(mx3[k], pair_shift1(mx3[(k + 1) & 7], mx3[(k + 2) & 7]), mx3[(k + 3) & 7]);
  }
  uint32_t hi = __vimax3_u16x2(__vimax3_u16x2(mn9[0], mn9[1], mn9[2]), __vimax3_u16x2(mn9[3], mn9[4], mn9[5]),
                               __vimax3_u16x2(mn9[6], mn9[7], mn9[7]));
  uint32_t lo = __vimin3_u16x2(__vimin3_u16x2(mx9[0], mx9[1], mx9[2]), __vimin3_u16x2(mx9[3], mx9[4], mx9[5]),
                               __vimin3_u16x2(mx9[6], mx9[7], mx9[7]));
  const int bmax = (int)max(hi & 0xffffu, hi >> 16), dmin = (int)min(lo & 0xffffu, lo >> 16);
  return max(max(bmax - c, c - dmin), 0);
}

// OR the SAT tiles covering the o0 pixel box [xa, xb] x [ya, yb] (clamped to
// the frame) into the stream's tile bitmap: one atomic per tile row and word.
__device__ __forceinline__ void mark_sat_box(const Geo& g, const Bufs& b, int s, int xa, int xb, int ya, int yb)
{
  xa = max(0, xa); xb = min(g.W - 1, xb);
  ya = max(0, ya); yb = min(g.H - 1, yb);
  const int txa = xa / VF_ST, txb = xb / VF_ST, tya = ya / VF_ST, tyb = yb / VF_ST;
  const int wa = txa >> 5, wb = txb >> 5;
  unsigned* bits = b.sat_bits + (long long)s * g.sty * g.stw_words;
  for (int ty = tya; ty <= tyb; ty++)
    for (int w = wa; w <= wb; w++) {
      const int lo = max(txa, 32 * w) - 32 * w, hi = min(txb, 32 * w + 31) - 32 * w;
      const unsigned m = (hi == 31 ? 0xffffffffu : ((1u << (hi + 1)) - 1u)) & ~((1u << lo) - 1u);
      atomicOr(bits + ty * g.stw_words + w, m);
    }
}

// True when every SAT tile of the box is set in the bitmap (VF_SAT_CHECK).
__device__ __forceinline__ bool sat_box_marked(const Geo& g, const Bufs& b, int s, int xa, int xb, int ya, int yb)
{
  xa = max(0, xa); xb = min(g.W - 1, xb);
  ya = max(0, ya); yb = min(g.H - 1, yb);
  const unsigned* bits = b.sat_bits + (long long)s * g.sty * g.stw_words;
  bool ok = true;
  for (int ty = ya / VF_ST; ty <= yb / VF_ST; ty++)
    for (int tx = xa / VF_ST; tx <= xb / VF_ST; tx++) ok &= (__ldcg(bits + ty * g.stw_words + (tx >> 5)) >> (tx & 31)) & 1u;
  return ok;
}

// Warp per tile (no block barriers): each warp stages its tile, runs the
// pre-test, scores its queue and stores, with __syncwarp only.
#define FAST_WARPS 8
struct FastWarp {
  uint8_t tile[FT_ROWS][FT_COLS];
  uint8_t sc[VF_TILE_H][VF_TILE_W];
  uint16_t queue[VF_TILE_H * VF_TILE_W];
  uint32_t drop[VF_TILE_H][VF_TILE_W / 32];   // candidates dropped by the in-tile 3x3 test
  int rc[VF_TILE_H];          // cell row of each tile row (gating)
  uint16_t cc[VF_TILE_W];     // cell column of each tile column
};

__global__ void __launch_bounds__(32 * FAST_WARPS) k_fast(const __grid_constant__ Geo g, const __grid_constant__ Bufs b,
                                                          int n_streams)
{
  extern __shared__ __align__(16) uint8_t fsm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  FastWarp& fw = reinterpret_cast<FastWarp*>(fsm)[wid];
  int* pre = reinterpret_cast<int*>(fsm + sizeof(FastWarp) * FAST_WARPS);   // [n_streams + 1]
  __shared__ int sm_warp[32];
  stream_prefix(n_streams, pre, sm_warp, [&](int sl) { return b.work_count[b.s0 + sl]; });
  const int n_work = pre[n_streams];
  const int t = g.threshold;
  for (int item = blockIdx.x * FAST_WARPS + wid; item < n_work; item += gridDim.x * FAST_WARPS) {
    int lo = -1;                           // stream of item: stream starts <= item, minus one
    for (int sb = 0; sb < n_streams; sb += 32)
      lo += __popc(__ballot_sync(0xffffffffu, sb + lane < n_streams && pre[sb + lane] <= item));
    const int s = b.s0 + lo;
    const int witem = b.worklist[(long long)s * g.tiles_per_stream + (item - pre[lo])];
    const bool clear_only = (witem & VF_CLEAR) != 0;
    const int tile_id = witem & (VF_CLEAR - 1);
    int l = 0;
    while (l + 1 < g.NL && tile_id >= g.L[l + 1].tile_base) l++;
    const LayerGeo& Lg = g.L[l];
    const int tl = tile_id - Lg.tile_base;
    const int ty = tl / Lg.tiles_x, tx = tl - ty * Lg.tiles_x;
    const int y0 = ty * VF_TILE_H, x0 = tx * VF_TILE_W;
    const int w = Lg.w, h = Lg.h;
    int pitch;
    const uint8_t* lp = layer_ptr(g, b, s, l, pitch);
    for (int i = lane; i < VF_TILE_H * VF_TILE_W / 16; i += 32)
      reinterpret_cast<uint4*>(&fw.sc[0][0])[i] = make_uint4(0, 0, 0, 0);
    (&fw.drop[0][0])[lane] = 0u;
    if (!clear_only) {
    const int um = use_mask(g, b, s);
    const uint8_t* cells = nullptr;
    int cols = 0;
    if (um) {
      const GridGeo& G = g.grid[grid_of_layer(g, l)];
      cells = b.cells + (long long)s * g.cell_slab + G.cell_off;
      cols = G.cols;
      const int* lut = b.lut + Lg.rc_off;
      if (lane < VF_TILE_H) fw.rc[lane] = y0 + lane < h ? __ldg(lut + y0 + lane) : 0;
#pragma unroll
      for (int k = 0; k < VF_TILE_W / 32; k++) {
        const int x = x0 + 32 * k + lane;
        fw.cc[32 * k + lane] = (uint16_t)(x < w ? __ldg(lut + h + x) : 0);
      }
    }
    // ---- stage rows y0-3 .. y0+10, cols x0-16 .. x0+143 ----
    // interior 16-B chunks by cp.async (global -> shared, no register round
    // trip, all of a lane's copies in flight together); chunks at the layer
    // edge bytewise, chunks outside the layer zero
    const bool vec_ok = ((reinterpret_cast<uintptr_t>(lp) | (uintptr_t)pitch) & 15) == 0;
    for (int i = lane; i < FT_ROWS * (FT_COLS / 16); i += 32) {
      const int rr = i / (FT_COLS / 16), c16 = i - rr * (FT_COLS / 16);
      const int y = y0 - 3 + rr, x = x0 - 16 + 16 * c16;
      uint8_t* dst = &fw.tile[rr][16 * c16];
      if (y >= 0 && y < h && x + 16 > 0 && x < w) {
        const uint8_t* row = lp + (long long)y * pitch;
        if (vec_ok && x >= 0 && x + 16 <= pitch && x + 16 <= ((w + 15) & ~15)) {
          const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(row + x) : "memory");
        } else {
          uint8_t tmp[16];
#pragma unroll
          for (int k = 0; k < 16; k++) tmp[k] = (x + k >= 0 && x + k < w) ? __ldg(row + x + k) : 0;
          *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<uint4*>(tmp);
        }
      } else {
        *reinterpret_cast<uint4*>(dst) = make_uint4(0, 0, 0, 0);
      }
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncwarp();
    // ---- pass 1: 4-point necessary test (detector.py:117-125) ----
    // A 9-arc covers two adjacent compass points, both brighter than C + t or
    // both darker than C - t, so both have |X - C| > t: the test below (an
    // adjacent pair over the threshold in absolute difference) keeps every
    // corner; pass 2 decides exactly.  Four pixels per word: VABSDIFF4, then
    // a borrow-free per-byte compare a > t into bit 7 of each byte.
    const uint32_t T4 = (uint32_t)(t < 128 ? t + 1 : t - 127) * 0x01010101u;
    const bool lowT = t < 128;
    auto over = [&](uint32_t X, uint32_t C) {
      const uint32_t a = __vabsdiffu4(X, C);
      return lowT ? (((a | 0x80808080u) - T4) | a) & 0x80808080u
                  : ((((a & 0x7f7f7f7fu) | 0x80808080u) - T4) & a) & 0x80808080u;
    };
    uint32_t inb = 0;                       // this lane's pixels inside [3, w - 3)
#pragma unroll
    for (int i = 0; i < 4; i++) {
      const int x = x0 + 4 * lane + i;
      inb |= (x >= 3 && x < w - 3) ? (0x80u << (8 * i)) : 0u;
    }
    int qn = 0;
    // queue slots: exclusive prefix of the per-lane counts (0..4) from
    // bit-plane ballots; only set pass bits are written
    auto enqueue = [&](uint32_t pass, int r, int k) {
      const int np = __popc(pass);
      const unsigned b0 = __ballot_sync(0xffffffffu, np & 1), b1 = __ballot_sync(0xffffffffu, np & 2),
                     b2 = __ballot_sync(0xffffffffu, np & 4);
      const unsigned lt = (1u << lane) - 1u;
      int pos = qn + __popc(b0 & lt) + 2 * __popc(b1 & lt) + 4 * __popc(b2 & lt);
      for (uint32_t pm = pass; pm; pm &= pm - 1u)
        fw.queue[pos++] = (uint16_t)(r * VF_TILE_W + 4 * k + ((__ffs(pm) - 1) >> 3));
      qn += __popc(b0) + 2 * __popc(b1) + 4 * __popc(b2);
    };
    // the 4-point test of word k of row r (pixels x0 + 4k .. +3)
    auto pretest = [&](int r, int k) {
      const int cb = 16 + 4 * k;
      const uint32_t C = *reinterpret_cast<const uint32_t*>(&fw.tile[r + 3][cb]);
      const uint32_t P = *reinterpret_cast<const uint32_t*>(&fw.tile[r + 3][cb - 4]);
      const uint32_t B = *reinterpret_cast<const uint32_t*>(&fw.tile[r + 3][cb + 4]);
      const uint32_t N = *reinterpret_cast<const uint32_t*>(&fw.tile[r][cb]);
      const uint32_t S = *reinterpret_cast<const uint32_t*>(&fw.tile[r + 6][cb]);
      const uint32_t E = __byte_perm(C, B, 0x6543), Wd = __byte_perm(P, C, 0x4321);   // x + 3, x - 3
      return (over(N, C) | over(S, C)) & (over(E, C) | over(Wd, C));
    };
    if (!um) {
      for (int r = 0; r < VF_TILE_H; r++) {
        const int y = y0 + r;
        const uint32_t pass = (y >= 3 && y < h - 3) ? pretest(r, lane) & inb : 0u;
        enqueue(pass, r, lane);
      }
    } else {
      // Gated tile: most words of an active tile lie in inactive cells
      // (detector.py:112-114 scores them 0).  List the (row, word) items with
      // an active in-bounds pixel -- lane k looks up the cells of its four
      // pixels once per cell row -- and run the 4-point test on the list only,
      // 32 items per round, with the per-pixel gate folded in.
      uint16_t* items = reinterpret_cast<uint16_t*>(&fw.sc[0][0]);   // zeroed again below
      uint32_t inb4 = 0;
#pragma unroll
      for (int i = 0; i < 4; i++) inb4 |= ((inb >> (8 * i + 7)) & 1u) << i;
      int n_items = 0, prev_rc = -1;
      uint32_t g4 = 0;
      for (int r = 0; r < VF_TILE_H; r++) {
        const int y = y0 + r;
        uint32_t gr = 0;
        if (y >= 3 && y < h - 3 && inb4) {
          if (fw.rc[r] != prev_rc) {
            prev_rc = fw.rc[r];
            const uint8_t* crow = cells + (long long)prev_rc * cols;
            g4 = 0;
#pragma unroll
            for (int i = 0; i < 4; i++) g4 |= (crow[fw.cc[4 * lane + i]] ? 1u : 0u) << i;
          }
          gr = g4 & inb4;
        }
        const unsigned m = __ballot_sync(0xffffffffu, gr != 0);
        if (gr) items[n_items + __popc(m & ((1u << lane) - 1u))] = (uint16_t)((r << 12) | (lane << 4) | gr);
        n_items += __popc(m);
      }
      __syncwarp();
      for (int base = 0; base < n_items; base += 32) {
        uint32_t pass = 0;
        int r = 0, k = 0;
        if (base + lane < n_items) {
          const int it = items[base + lane];
          r = it >> 12;
          k = (it >> 4) & 31;
          const uint32_t gate = ((((uint32_t)it & 15u) * 0x00204081u) & 0x01010101u) * 0x80u;
          pass = pretest(r, k) & gate;
        }
        enqueue(pass, r, k);
      }
      __syncwarp();
      for (int i = lane; i < (n_items + 7) / 8; i += 32) reinterpret_cast<uint4*>(items)[i] = make_uint4(0, 0, 0, 0);
    }
    __syncwarp();
    // ---- pass 2: exact score of queued pixels ----
    for (int qi = lane; qi < qn; qi += 32) {
      const int p = fw.queue[qi];
      const int r = p / VF_TILE_W, c = p - r * VF_TILE_W;
      const int R = r + 3, Cc = 16 + c;
      // ring order of detector.py:34-40 (clockwise from north), as 16x2 pairs
      const uint8_t* t0p = &fw.tile[0][0];
      auto px = [&](int dy, int dx) { return (uint32_t)t0p[(R + dy) * FT_COLS + Cc + dx]; };
      uint32_t wr[8];
      wr[0] = px(-3, 0) | (px(-3, 1) << 16);
      wr[1] = px(-2, 2) | (px(-1, 3) << 16);
      wr[2] = px(0, 3) | (px(1, 3) << 16);
      wr[3] = px(2, 2) | (px(3, 1) << 16);
      wr[4] = px(3, 0) | (px(3, -1) << 16);
      wr[5] = px(2, -2) | (px(1, -3) << 16);
      wr[6] = px(0, -3) | (px(-1, -3) << 16);
      wr[7] = px(-2, -2) | (px(-3, -1) << 16);
      const int score = fast_best(wr, (int)px(0, 0)) - 1;
      if (score >= t) fw.sc[r][c] = (uint8_t)score;
    }
    __syncwarp();
    // ---- pass 3 (b.nms_pre): a candidate whose 8 neighbours all lie in this
    // tile and that is not their strict maximum would fail k_nms_test's strict
    // 3x3 test (detector.py:255-262): drop it from the bitmap here, so only the
    // NMS work shrinks.  Candidates on the tile's border wait for k_nms_test.
    if (b.nms_pre) {
      for (int qi = lane; qi < qn; qi += 32) {
        const int p = fw.queue[qi];
        const int r = p / VF_TILE_W, c = p - r * VF_TILE_W;
        const int sv = fw.sc[r][c];
        if (sv == 0 || r == 0 || r == VF_TILE_H - 1 || c == 0 || c == VF_TILE_W - 1) continue;
        int m = 0;
#pragma unroll
        for (int dy = -1; dy <= 1; dy++)
#pragma unroll
          for (int dx = -1; dx <= 1; dx++)
            if (dy || dx) m = max(m, (int)fw.sc[r + dy][c + dx]);
        if (m >= sv) atomicOr(&fw.drop[r][c >> 5], 1u << (c & 31));
      }
      __syncwarp();
    }
    }
    __syncwarp();
    // ---- store scores (whole tile: gated pixels read back as 0) + bitmap ----
    uint8_t* smap = b.scores + (long long)s * g.sm_slab + Lg.sm_off;
    for (int i = lane; i < VF_TILE_H * (VF_TILE_W / 16); i += 32) {
      const int r = i >> 3, cc = i & 7;
      const int y = y0 + r, x = x0 + 16 * cc;
      if (y >= h || x >= w) continue;
      *reinterpret_cast<uint4*>(smap + (long long)y * Lg.pitch + x) = *reinterpret_cast<const uint4*>(&fw.sc[r][16 * cc]);
    }
    {
      // Candidate bitmap (score >= t), minus the candidates pass 3 dropped.
      const int r = lane >> 2, kw = lane & 3;
      const int y = y0 + r;
      uint32_t word_all = 0;
#pragma unroll
      for (int q = 0; q < 8; q++) {
        const uint32_t v = *reinterpret_cast<const uint32_t*>(&fw.sc[r][32 * kw + 4 * q]);
        const uint32_t nz = __vcmpne4(v, 0u);
        word_all |= (((nz >> 7) & 1u) | ((nz >> 14) & 2u) | ((nz >> 21) & 4u) | ((nz >> 28) & 8u)) << (4 * q);
      }
      const uint32_t word = word_all & ~fw.drop[r][kw];
      if (y < h && x0 + 32 * kw < w)
        b.bitmaps[(long long)s * g.bm_slab_words + Lg.bm_off + (long long)y * Lg.bm_words + 4 * tx + kw] = word;
      if (b.sat_early && __any_sync(0xffffffffu, word != 0u)) {
        // SAT tiles any keypoint kept from this tile's candidates can read: the
        // bounding box of the candidates, widened by LayerGeo.sat_reach (float
        // positions are within 1 pixel, inside its margin).  One (tile row,
        // word) pair per lane.
        const bool hasc = word != 0u;
        const int xl = __reduce_min_sync(0xffffffffu, hasc ? x0 + 32 * kw + __ffs(word) - 1 : INT_MAX);
        const int xh = __reduce_max_sync(0xffffffffu, hasc ? x0 + 32 * kw + 31 - __clz(word) : -1);
        const int yl = __reduce_min_sync(0xffffffffu, hasc ? y : INT_MAX);
        const int yh = __reduce_max_sync(0xffffffffu, hasc ? y : -1);
        const float inv = Lg.inv_scale;
        const int F = Lg.sat_reach;
        const int xa = max(0, (int)((float)xl * inv) - F), xb = min(g.W - 1, (int)((float)xh * inv) + F);
        const int ya = max(0, (int)((float)yl * inv) - F), yb = min(g.H - 1, (int)((float)yh * inv) + F);
        const int txa = xa / VF_ST, txb = xb / VF_ST, tya = ya / VF_ST, tyb = yb / VF_ST;
        const int wa = txa >> 5, nw = (txb >> 5) - wa + 1, np = (tyb - tya + 1) * nw;
        unsigned* bits = b.sat_bits + (long long)s * g.sty * g.stw_words;
        for (int i = lane; i < np; i += 32) {
          const int ty = tya + i / nw, wd = wa + i % nw;
          const int lo = max(txa, 32 * wd) - 32 * wd, hi = min(txb, 32 * wd + 31) - 32 * wd;
          const unsigned m = (hi == 31 ? 0xffffffffu : ((1u << (hi + 1)) - 1u)) & ~((1u << lo) - 1u);
          atomicOr(bits + ty * g.stw_words + wd, m);   // no return value: fire and forget
        }
      }
      int n = __popc(word), na = __popc(word_all);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        n += __shfl_down_sync(0xffffffffu, n, o);
        na += __shfl_down_sync(0xffffffffu, na, o);
      }
      if (lane == 0) {
        if (na) atomicAdd(&b.ctr[s * C_NCTR + C_NCAND], na);
        if (n) atomicAdd(&b.band_cand[(long long)s * g.bands_per_stream + Lg.band_base + ty], n);
      }
    }
    __syncwarp();
  }
}

// ============================================================================
// k_nms: detector.py:239-307 over one band (8 rows of one layer) per CTA.
// ============================================================================
// Candidates come from the FAST bitmap in row-major order (block scan over
// per-thread word ranges), so kept keypoints leave each band in (y, x) order
// and bands are ordered (layer, y): the reference order.  Each candidate:
// strict 3x3 max, strict vs the rounded-projected pixel of layers i+-1, fp64
// quadratic refinement of itself and its neighbours (op order of
// detector.py:207-228, 277-302), border filter (pipeline.py:148-161) and the
// Eq. 1 merge filter (masking.py:176-178, applied before describing: a
// dropped detection's descriptor is never observable).  The last CTA of each
// stream scans band counts and propagation-chunk counts into offsets.

// Score of layer l at (y, x); 0 outside the layer.  Gated pixels score 0
// (detector.py:112-114): k_fast stores whole active tiles with 0 at gated
// pixels, and tiles not active this step hold zeros (cleared by k_fast when
// they stop being active), so a map read needs no activity check.  Branch-free:
// the load uses a clamped in-bounds address, so a caller's reads overlap.
__device__ __forceinline__ int score_read(const Geo& g, const Bufs& b, int s, int um, int l, int y, int x)
{
  (void)um;
  const LayerGeo& Lg = g.L[l];
  const bool in = (unsigned)y < (unsigned)Lg.h && (unsigned)x < (unsigned)Lg.w;
  const int off = in ? y * Lg.pitch + x : 0;
  const int v = __ldg(b.scores + (long long)s * g.sm_slab + Lg.sm_off + off);
  return in ? v : 0;
}

// floor((n + d / 2) / d) for 0 <= n < 2^40 (detector.py:266-269 rounding of
// the projected coordinate), exact: fp64 reciprocal estimate, one correction.
__device__ __forceinline__ int round_div(int y, int num, int d, double rd)
{
  const long long n = (long long)y * num + (d >> 1);
  long long q = (long long)((double)n * rd);
  if (q * d > n) q--;
  else if ((q + 1) * d <= n) q++;
  return (int)q;
}

__device__ __forceinline__ void fit_peak(const double p[3][3], double& ox, double& oy, double& val, int& okp)
{
  // detector.py:207-228, same operation order (no FMA: -fmad=false)
  double gx = 0.5 * (p[1][2] - p[1][0]);
  double gy = 0.5 * (p[2][1] - p[0][1]);
  double dxx = p[1][2] - 2.0 * p[1][1] + p[1][0];
  double dyy = p[2][1] - 2.0 * p[1][1] + p[0][1];
  double dxy = 0.25 * (p[2][2] - p[2][0] - p[0][2] + p[0][0]);
  double det = dxx * dyy - dxy * dxy;
  int ok = (dxx < 0.0) && (det > 0.0);
  double safe = ok ? det : 1.0;
  double x = ok ? -(dyy * gx - dxy * gy) / safe : 0.0;
  double y = ok ? -(dxx * gy - dxy * gx) / safe : 0.0;
  ok = ok && (fabs(x) < 1.0) && (fabs(y) < 1.0);
  x = ok ? x : 0.0;
  y = ok ? y : 0.0;
  val = p[1][1] + 0.5 * (gx * x + gy * y);
  ox = x; oy = y; okp = ok;
}

__device__ __forceinline__ void patch_load(const Geo& g, const Bufs& b, int s, int um, int l, int y, int x, int v[9])
{
#pragma unroll
  for (int dy = -1; dy <= 1; dy++)
#pragma unroll
    for (int dx = -1; dx <= 1; dx++) v[(dy + 1) * 3 + dx + 1] = score_read(g, b, s, um, l, y + dy, x + dx);
}

__device__ __forceinline__ int patch_to_double(const int v[9], double p[3][3])
{
  int mx = INT_MIN;
#pragma unroll
  for (int i = 0; i < 9; i++) {
    p[i / 3][i % 3] = (double)v[i];
    mx = v[i] > mx ? v[i] : mx;
  }
  return mx;
}

struct NmsOut { double x, y, sig, v; int flags; };  // flags: 1 survivor, 2 border ok, 4 kept

// Batch 1 of detector.py:251-275: strict 3x3 maximum and strict vs the rounded
// projection into layers l-1, l+1.
__device__ __forceinline__ bool nms_test(const Geo& g, const Bufs& b, int s, int um, int l, int y, int x)
{
  const LayerGeo& Lg = g.L[l];
  // batch 1: centre, 8 neighbours, projected pixels of layers l-1, l+1
  const int sv = score_read(g, b, s, um, l, y, x);
  int nb[8];
#pragma unroll
  for (int i = 0; i < 8; i++) {
    const int dy = i < 3 ? -1 : (i < 5 ? 0 : 1);
    const int dx = i < 3 ? i - 1 : (i == 3 ? -1 : (i == 4 ? 1 : i - 6));
    int yy = y + dy, xx = x + dx;
    if (g.nms_wrap) {                                    // smap[ys+dy, xs+dx] (detector.py:260-262)
      yy = yy < 0 ? yy + Lg.h : yy;
      xx = xx < 0 ? xx + Lg.w : xx;
    }
    nb[i] = score_read(g, b, s, um, l, yy, xx);
  }
  int yj[2] = {0, 0}, xj[2] = {0, 0}, cj[2] = {0, 0};
  const bool has[2] = {l >= 1, l + 1 < g.NL};
#pragma unroll
  for (int k = 0; k < 2; k++) {                          // detector.py:264-273
    if (!has[k]) continue;
    const int j = l - 1 + 2 * k;
    const int hj = g.L[j].h, wj = g.L[j].w;
    const int a = round_div(y, hj, Lg.h, Lg.rinv_h), c = round_div(x, wj, Lg.w, Lg.rinv_w);
    yj[k] = a < hj - 1 ? a : hj - 1;
    xj[k] = c < wj - 1 ? c : wj - 1;
    cj[k] = score_read(g, b, s, um, j, yj[k], xj[k]);
  }
  bool keep = sv > 0;
#pragma unroll
  for (int i = 0; i < 8; i++) keep &= sv > nb[i];
#pragma unroll
  for (int k = 0; k < 2; k++) keep &= !has[k] || sv > cj[k];
  return keep;
}

// Survivor refinement (detector.py:277-302) + border / merge filters.
__device__ NmsOut nms_refine(const Geo& g, const Bufs& b, int s, int um, int l, int y, int x)
{
  NmsOut o;
  o.flags = 1;
  const LayerGeo& Lg = g.L[l];
  const bool has[2] = {l >= 1, l + 1 < g.NL};
  int yj[2] = {0, 0}, xj[2] = {0, 0};
#pragma unroll
  for (int k = 0; k < 2; k++) {
    if (!has[k]) continue;
    const int j = l - 1 + 2 * k;
    const int hj = g.L[j].h, wj = g.L[j].w;
    const int a = round_div(y, hj, Lg.h, Lg.rinv_h), c = round_div(x, wj, Lg.w, Lg.rinv_w);
    yj[k] = a < hj - 1 ? a : hj - 1;
    xj[k] = c < wj - 1 ? c : wj - 1;
  }
  // batch 2: the three 3x3 patches (zero-padded maps, detector.py:231-236)
  int pv[3][9];
  patch_load(g, b, s, um, l, y, x, pv[0]);
#pragma unroll
  for (int k = 0; k < 2; k++)
    if (has[0] && has[1]) patch_load(g, b, s, um, l - 1 + 2 * k, yj[k], xj[k], pv[1 + k]);
  double p[3][3], ox, oy, v0;
  int ok;
  patch_to_double(pv[0], p);
  fit_peak(p, ox, oy, v0, ok);
  double nv[2] = {0.0, 0.0};
  const bool both = has[0] && has[1];                    // neighbour values only feed the scale fit
#pragma unroll
  for (int k = 0; k < 2; k++) {                          // detector.py:281-285
    if (!both) continue;
    double pj[3][3], tx, ty, vj;
    int okj;
    const int pmax = patch_to_double(pv[1 + k], pj);
    fit_peak(pj, tx, ty, vj, okj);
    nv[k] = okj ? vj : (double)pmax;
  }
  double sig = Lg.sigma;
  if (l >= 1 && l + 1 < g.NL) {                          // detector.py:287-297
    const double vb = nv[0], va = nv[1];
    const double denom = vb - 2.0 * v0 + va;
    double delta = denom < 0.0 ? 0.5 * (vb - va) / denom : 0.0;
    delta = fabs(delta) < 1.0 ? delta : 0.0;
    const double up = g.L[l + 1].sigma / Lg.sigma;
    const double down = g.L[l - 1].sigma / Lg.sigma;
    // sigma_i * up^a * down^c with a = max(delta, 0), c = max(-delta, 0): one
    // factor is x^0 = 1 exactly, so one pow gives the same product
    const double f = pow(delta > 0.0 ? up : down, fabs(delta));
    sig = delta > 0.0 ? Lg.sigma * f * 1.0 : Lg.sigma * 1.0 * f;
  }
  // detector.py:299-302; dividing by an octave scale 2^-o is exactly x * 2^o
  double xf, yf;
  if ((l & 1) == 0) {
    const double inv = (double)(1 << (l >> 1));
    xf = ((double)x + ox) * inv;
    yf = ((double)y + oy) * inv;
  } else {
    xf = ((double)x + ox) / Lg.scale;
    yf = ((double)y + oy) / Lg.scale;
  }
  const double xhi = (double)g.W - 1e-6, yhi = (double)g.H - 1e-6;
  xf = xf < 0.0 ? 0.0 : (xf > xhi ? xhi : xf);
  yf = yf < 0.0 ? 0.0 : (yf > yhi ? yhi : yf);
  o.x = xf; o.y = yf; o.sig = sig; o.v = v0;
  if (g.nms_raw) { o.flags |= 6; return o; }
  const double m = 3.0 * sig;                            // pipeline.py:148-161
  if (xf >= m && yf >= m && xf <= (double)(g.W - 1) - m && yf <= (double)(g.H - 1) - m) {
    o.flags |= 2;
    if (!um || merge_mask_at(g, b, s, xf, yf)) o.flags |= 4;   // masking.py:176-178
  }
  return o;
}

// Mark the SAT tiles a keypoint's descriptor footprint touches: samples lie
// within 10.8 sigma (+0.5 rounding) of the centre and boxes add <= 1.69 sigma
// + 0.5 (pattern.py:22-23,58), plus one pixel for the SAT corner.
__device__ __forceinline__ void mark_sat_tiles(const Geo& g, const Bufs& b, int s, double x, double y, double sg,
                                               int epoch)
{
  // footprint bound of the 60 boxes (|p| <= 10.8, radius <= 1.69 sigma)
  (void)epoch;
  const int F = (int)ceil(12.5 * sg) + 2;
  const int xi = (int)x, yi = (int)y;
  if (!b.sat_early) mark_sat_box(g, b, s, xi - F, xi + F + 1, yi - F, yi + F + 1);
  else if (b.sat_check && !sat_box_marked(g, b, s, xi - F, xi + F + 1, yi - F, yi + F + 1))
    atomicOr(b.ctr + s * C_NCTR + C_ERR, VF_ERRBIT_SATMARK);
}

// Warp-collective, at k_nms_test's kept-keypoint site: append the kept
// keypoints (candidate index c) to the stream's describe list (warp-aggregated
// atomic) and mark the SAT tiles of their footprints.
__device__ __forceinline__ void desc_list_kept(const Geo& g, const Bufs& b, int s, bool kp, double x, double y,
                                               double sg, int c, int lane)
{
  const unsigned gm = __ballot_sync(0xffffffffu, kp);
  if (gm) {
    const int leader = __ffs(gm) - 1;
    int gb = 0;
    if (lane == leader) gb = atomicAdd(b.ctr + s * C_NCTR + C_NGLOB, __popc(gm));
    gb = __shfl_sync(0xffffffffu, gb, leader);
    if (kp) {
      b.gidx[(long long)s * g.kp_cap + gb + __popc(gm & ((1u << lane) - 1))] = c;
      mark_sat_tiles(g, b, s, x, y, sg, 0);
    }
  }
}

// Block-wide exclusive scan (blockDim.x = NF_THREADS) of one value per thread.
#define NF_THREADS 256
#define NMS_CHUNK_THREADS (1 << NMS_CHUNK_LOG)
__device__ __forceinline__ int block_excl_scan(int v, int& total, int* sm)
{
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int wt;
  const int ex = warp_excl_scan(v, lane, wt);
  if (lane == 31) sm[wid] = wt;
  __syncthreads();
  int off = 0;
  total = 0;
#pragma unroll
  for (int w = 0; w < NF_THREADS / 32; w++) {
    const int t = sm[w];
    off += w < wid ? t : 0;
    total += t;
  }
  __syncthreads();
  return off + ex;
}


// Warp per NMS unit: R consecutive rows of a band (R = VF_TILE_H / b.nms_u;
// R = 8 when many streams fill the GPU, fewer rows per warp for single-stream
// batches so more warps share the work).  The unit's FAST bitmap words are
// walked 32 at a time in row-major order, one word per lane: a warp scan of
// the popcounts gives every candidate its rank and the lanes write their
// candidates (row, x) into a per-warp list.  The list is tested 32 at a time
// (lane = candidate: strict 3x3 + cross-layer), survivors are queued FIFO and
// refined 32 at a time (fp64), and kept keypoints are compacted with ballots,
// so each unit emits its keypoints in (y, x) order and units are ordered
// (layer, y): the reference order (detector.py:251-253,303-306).
#define NMS_WARPS 4
#define NMS_THREADS (32 * NMS_WARPS)
#define NMS_PF 16       // bitmap words per lane staged at once
#define NMS_LIST (1024 + 32)   // candidates of 32 bitmap words + an untested remainder
__global__ void __launch_bounds__(NMS_THREADS, 8) k_nms(const __grid_constant__ Geo g, const __grid_constant__ Bufs b)
{
  // (row offset << 13) | x as 16 bits (x < 8192, row offset < 8): a small
  // footprint leaves the L1 to the score-map reads
  __shared__ uint16_t cand[NMS_WARPS][NMS_LIST];
  __shared__ uint16_t sq[NMS_WARPS][64];      // survivor queue, same encoding
  __shared__ uint32_t wbuf[NMS_WARPS][32 * NMS_PF];   // staged bitmap words of the unit
  const int s = b.s0 + blockIdx.y, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int U = b.nms_u, R = VF_TILE_H / U;
  const int unit = blockIdx.x * NMS_WARPS + w;
  if (unit >= g.bands_per_stream * U) return;
  const int bid = unit / U, sub = unit - bid * U;
  int4* rec = reinterpret_cast<int4*>(b.unit_rec) + ((long long)s * g.bands_per_stream * U + unit);
  const int epoch = stream_epoch(b, s);
  int kept = 0, n_ok = 0, n_drop = 0, base = 0;
  if (b.band_stamp[(long long)s * g.bands_per_stream + bid] == epoch &&
      __ldcg(b.band_cand + (long long)s * g.bands_per_stream + bid) > 0) {
    const int um = use_mask(g, b, s) ? epoch : 0;
    int* ctr = b.ctr + s * C_NCTR;
    int l = 0;
    while (l + 1 < g.NL && bid >= g.L[l + 1].band_base) l++;
    const LayerGeo& Lg = g.L[l];
    const int ys = (bid - Lg.band_base) * VF_TILE_H + sub * R;
    const int nrows = max(0, min(Lg.h - ys, R));
    const int bmw = Lg.bm_words, nw = nrows * bmw;
    const uint32_t* bm = b.bitmaps + (long long)s * g.bm_slab_words + Lg.bm_off + (long long)ys * bmw;
    // candidates of the unit: the band's count from k_fast when the unit is the
    // whole band, else the popcount of the unit's words (inactive tiles hold zero words)
    int total = 0;
    if (U == 1) {
      total = __ldcg(b.band_cand + (long long)s * g.bands_per_stream + bid);
    } else {
      for (int k = lane; k < nw; k += 32) total += __popc(__ldg(bm + k));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) total += __shfl_xor_sync(0xffffffffu, total, o);
    }
    if (total > 0) {
      int bs = 0;
      if (lane == 0) {
        bs = atomicAdd(&ctr[C_STAGE], total);
        if (bs + total > g.kp_cap) { atomicOr(&ctr[C_ERR], VF_ERRBIT_STAGING); bs = -1; }
      }
      base = __shfl_sync(0xffffffffu, bs, 0);
    }
    if (total > 0 && base >= 0) {
      // One loop with a single test site and a single refine site (the fp64
      // refinement is large: inlining it twice made the kernel i-cache bound).
      // cand[head, tail) holds listed, untested candidates; sq[0, qn) survivors.
      int qn = 0, head = 0, tail = 0, k0 = 0;   // warp-uniform
      int kb = 0, ke = 0;                       // words [kb, ke) of the unit are staged in wbuf
      for (;;) {
        if (tail - head < 32 && k0 < nw) {
          if (k0 == ke) {
            // stage the next 512 bitmap words, 16 independent loads per lane in flight
            kb = k0;
            ke = min(nw, k0 + 32 * NMS_PF);
#pragma unroll
            for (int j = 0; j < NMS_PF; j++) {
              const int k = kb + 32 * j + lane;
              wbuf[w][32 * j + lane] = k < ke ? __ldg(bm + k) : 0u;
            }
            __syncwarp();
          }
          const int k = k0 + lane;
          const uint32_t word = wbuf[w][k0 - kb + lane];   // zero past ke
          k0 = min(ke, k0 + 32);
          if (!__any_sync(0xffffffffu, word != 0u)) continue;   // 32 empty words (gated tiles)
          // refill: move the (< 32) untested remainder to the front, list this pass
          if (head) {
            const int rem = tail - head;
            const uint16_t v = lane < rem ? cand[w][head + lane] : (uint16_t)0;
            __syncwarp();
            if (lane < rem) cand[w][lane] = v;
            head = 0;
            tail = rem;
          }
          int tot;
          int pos = tail + warp_excl_scan(__popc(word), lane, tot);
          if (word) {
            const int r = k / bmw, cw = k - r * bmw;
            for (uint32_t m = word; m; m &= m - 1u) cand[w][pos++] = (uint16_t)((r << 13) | (32 * cw + __ffs(m) - 1));
          }
          tail += tot;
          __syncwarp();
          continue;
        }
        if (tail > head) {
          // test up to 32 listed candidates (lane = candidate), queue the survivors
          const int nr = min(32, tail - head);
          bool keep = false;
          int v = 0;
          if (lane < nr) {
            v = cand[w][head + lane];
            keep = nms_test(g, b, s, um, l, ys + (v >> 13), v & 0x1fff);
          }
          const unsigned sm = __ballot_sync(0xffffffffu, keep);
          if (keep) sq[w][qn + __popc(sm & ((1u << lane) - 1))] = (uint16_t)v;
          qn += __popc(sm);
          head += nr;
          __syncwarp();
        }
        const bool fin = k0 >= nw && head == tail;
        if (qn >= 32 || (fin && qn > 0)) {
          // refine the oldest nb survivors (FIFO keeps the (y, x) order)
          const int nb = min(32, qn);
          NmsOut o;
          o.flags = 0;
          if (lane < nb) {
            const int v = sq[w][lane];
            o = nms_refine(g, b, s, um, l, ys + (v >> 13), v & 0x1fff);
          }
          const unsigned kb = __ballot_sync(0xffffffffu, o.flags & 4);
          n_ok += __popc(__ballot_sync(0xffffffffu, o.flags & 2));
          n_drop += __popc(__ballot_sync(0xffffffffu, (o.flags & 1) && !(o.flags & 2)));
          if (o.flags & 4) {
            const long long dst = (long long)s * g.kp_cap + base + kept + __popc(kb & ((1u << lane) - 1));
            b.st_x[dst] = o.x; b.st_y[dst] = o.y; b.st_s[dst] = o.sig; b.st_v[dst] = o.v;
          }
          kept += __popc(kb);
          __syncwarp();
          const uint16_t rest = lane + nb < qn ? sq[w][lane + nb] : (uint16_t)0;
          __syncwarp();
          if (lane + nb < qn) sq[w][lane] = rest;
          qn -= nb;
          __syncwarp();
        } else if (fin) {
          break;
        }
      }
    } else {
      base = 0;
    }
  }
  if (lane == 0) *rec = make_int4(base, kept, n_ok, n_drop);
}

// ============================================================================
// Candidate-parallel scale-space NMS of the pipeline (detector.py:239-307):
//   k_nms_list   warp per active band: the band's FAST bitmap words in
//                row-major order -> candidate codes (layer, y, x) at the
//                band's offset (prefix of the active bands' k_fast counts), so
//                the list is in the reference's (layer, y, x) order;
//   k_nms_test   thread per candidate, NMS_CHUNK candidates per CTA pass:
//                nms_test + nms_refine (strict 3x3 + cross-layer maximum,
//                fp64 refinement, border and merge filters), kept records in
//                the candidate's staging slot, rank within the chunk by a
//                block scan, the chunk's kept count; kept keypoints join the
//                describe list and mark their SAT tiles;
//   k_nms_finish chunk counts -> output offsets (k_desc_fused: rank = chunk
//                offset + rank in chunk), FrameReport, SAT-tile work list.
// ============================================================================
#define NL_WARPS 8
__device__ __forceinline__ int band_count(const Bufs& b, const Geo& g, int s, int bid, int epoch)
{
  // both loads issued together (a stale count of an inactive band is discarded)
  const long long i = (long long)s * g.bands_per_stream + bid;
  const int st = b.band_stamp[i], cnt = __ldcg(b.band_cand + i);
  return st == epoch ? cnt : 0;
}

__global__ void __launch_bounds__(32 * NL_WARPS) k_nms_list(const __grid_constant__ Geo g,
                                                            const __grid_constant__ Bufs b)
{
  __shared__ int red[NL_WARPS], cnt[NL_WARPS];
  const int s = b.s0 + blockIdx.y, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int epoch = stream_epoch(b, s);
  const int band0 = blockIdx.x * NL_WARPS, nb = g.bands_per_stream;
  // candidates of the active bands before this CTA's
  int part = 0;
#pragma unroll 2
  for (int i = tid; i < band0; i += 32 * NL_WARPS) part += band_count(b, g, s, i, epoch);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  const int bid = band0 + w;
  const int mine = bid < nb ? band_count(b, g, s, bid, epoch) : 0;
  if (lane == 0) { red[w] = part; cnt[w] = mine; }
  __syncthreads();
  int off = 0, tot = 0;
#pragma unroll
  for (int k = 0; k < NL_WARPS; k++) {
    off += red[k] + (k < w ? cnt[k] : 0);
    tot += cnt[k];
  }
  int* ctr = b.ctr + s * C_NCTR;
  if (blockIdx.x == gridDim.x - 1 && tid == 0) {
    int all = tot;
#pragma unroll
    for (int k = 0; k < NL_WARPS; k++) all += red[k];
    ctr[C_STAGE] = all;   // the stream's candidates (capacity retry sizing)
    if (all > g.kp_cap) atomicOr(&ctr[C_ERR], VF_ERRBIT_STAGING);
  }
  if (mine == 0 || off + mine > g.kp_cap) return;
  int l = 0;
  while (l + 1 < g.NL && bid >= g.L[l + 1].band_base) l++;
  const LayerGeo& Lg = g.L[l];
  const int ys = (bid - Lg.band_base) * VF_TILE_H;
  const int bmw = Lg.bm_words, nw = min(VF_TILE_H, Lg.h - ys) * bmw;
  const uint32_t* bm = b.bitmaps + (long long)s * g.bm_slab_words + Lg.bm_off + (long long)ys * bmw;
  uint32_t* out = b.cand + (long long)s * g.kp_cap;
  const uint32_t lcode = (uint32_t)l << 26;
  int pos = off;
  for (int k0 = 0; k0 < nw; k0 += 128) {
    uint32_t wd[4];
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const int k = k0 + 32 * q + lane;
      wd[q] = k < nw ? __ldcg(bm + k) : 0u;
    }
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const unsigned any = __ballot_sync(0xffffffffu, wd[q] != 0u);
      if (!any) continue;
      const int k = k0 + 32 * q + lane;
      int t;
      int p = pos + warp_excl_scan(__popc(wd[q]), lane, t);
      if (wd[q]) {
        const int r = k / bmw, cw = k - r * bmw;
        const uint32_t base = lcode | ((uint32_t)(ys + r) << 13) | (uint32_t)(32 * cw);
        for (uint32_t m = wd[q]; m; m &= m - 1u) out[p++] = base + (uint32_t)(__ffs(m) - 1);
      }
      pos += t;
    }
  }
}

// The set tiles of a stream's SAT-tile bitmap, in bitmap order -> the k_sat
// work list (whole CTA of NF_THREADS threads).
__device__ __forceinline__ void sat_work_list(const Geo& g, const Bufs& b, int s, int* sm)
{
  const int tid = threadIdx.x;
  const int nw = g.sty * g.stw_words;
  const unsigned* bits = b.sat_bits + (long long)s * nw;
  int* work = b.sat_work + (long long)s * g.sat_tiles;
  int cnt = 0;
  for (int w0 = 0; w0 < nw; w0 += NF_THREADS) {
    const int wi = w0 + tid;
    unsigned v = wi < nw ? __ldcg(bits + wi) : 0u;
    int tot;
    int pos = cnt + block_excl_scan(__popc(v), tot, sm);
    const int ty = wi / g.stw_words, t0 = ty * g.stx + 32 * (wi - ty * g.stw_words);
    for (; v; v &= v - 1u) work[pos++] = t0 + __ffs(v) - 1;
    cnt += tot;
  }
  if (tid == 0) b.sat_count[s] = cnt;
}

// Early SAT (b.sat_early): the work list of the tiles k_fast marked, one CTA
// per stream, launched on the describe stream right after k_fast.
__global__ void __launch_bounds__(NF_THREADS) k_sat_list(const __grid_constant__ Geo g, const __grid_constant__ Bufs b)
{
  __shared__ int sm[NF_THREADS / 32];
  sat_work_list(g, b, b.s0 + blockIdx.x, sm);
}

// After k_nms (stream order), one CTA per stream: band output offsets (scan
// of the kept counts in band order), the SAT-tile work list (the bitmap's set
// tiles in bitmap order) and the FrameReport.  Every load is issued up front.
__device__ __forceinline__ void nms_finish_stream(const Geo& g, const Bufs& b, int s, int* sm, int (*red)[NF_THREADS / 32])
{
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int um = use_mask(g, b, s);
  int n_det, n_drop = 0, n_surv = 0;
  if (b.desc_bin) {
    // ---- pipeline (k_nms_test): chunk kept counts -> output offsets, in place ----
    const int* ctr = b.ctr + s * C_NCTR;
    const int nch = (ctr[C_ERR] & VF_ERRBIT_STAGING) ? 0 : (ctr[C_STAGE] + NMS_CHUNK_THREADS - 1) >> NMS_CHUNK_LOG;
    int* co = b.chunk_off + (long long)s * g.nms_chunks;
    int carry = 0;
    for (int c0 = 0; c0 < nch; c0 += NF_THREADS) {
      const int i = c0 + tid;
      const int v = i < nch ? __ldcg(co + i) : 0;
      int tot;
      const int ex = block_excl_scan(v, tot, sm);
      if (i < nch) co[i] = carry + ex;
      carry += tot;
    }
    n_det = carry;
    if (tid == 0) {
      const int n_ok = __ldcg(b.nms_cnt + 4 * s), n_dr = __ldcg(b.nms_cnt + 4 * s + 1);
      n_drop = n_dr;
      n_surv = n_ok + n_dr;
    }
  } else {
    // ---- stand-alone (k_nms): unit offsets, thread t owns units [t * per, t * per + per) ----
    const int nb = g.bands_per_stream * b.nms_u;   // NMS units, (layer, y) order
    const int4* rec = reinterpret_cast<const int4*>(b.unit_rec) + (long long)s * nb;
    int* bout = b.unit_out + (long long)s * nb;
    const int per = (nb + NF_THREADS - 1) / NF_THREADS;
    int kept = 0;
    for (int k = 0; k < per; k++) {
      const int i = tid * per + k;
      if (i < nb) {
        const int4 r = __ldcg(rec + i);
        kept += r.y;
        n_drop += r.w;
        n_surv += r.z + r.w;
      }
    }
    int run = block_excl_scan(kept, n_det, sm);
    for (int k = 0; k < per; k++) {
      const int i = tid * per + k;
      if (i < nb) {
        bout[i] = run;
        run += __ldcg(rec + i).y;
      }
    }
  }
  // ---- SAT tiles marked by the stream's bands (k_nms ORs footprints into
  // the bitmap) -> the k_sat work list ----
  if ((um || b.desc_bin) && !b.sat_early) sat_work_list(g, b, s, sm);
  // ---- FrameReport ----
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    n_drop += __shfl_down_sync(0xffffffffu, n_drop, o);
    n_surv += __shfl_down_sync(0xffffffffu, n_surv, o);
  }
  if (lane == 0) { red[0][wid] = n_drop; red[1][wid] = n_surv; }
  __syncthreads();
  if (tid == 0) {
    n_drop = 0;
    n_surv = 0;
    for (int w = 0; w < NF_THREADS / 32; w++) { n_drop += red[0][w]; n_surv += red[1][w]; }
    // propagated total: scanned by k_worklist (joined before k_nms)
    const int n_prop = um ? __ldcg(b.ctr + s * C_NCTR + C_NPROP) : 0;
    int* ctr = b.ctr + s * C_NCTR;
    int n_total = n_det + n_prop;
    int n_desc = n_det;   // detected records the describe kernels write
    if (n_total > g.kp_cap) {
      // overflow: flagged (vf_process_checked grows the capacity and replays);
      // the describe writes are clamped so they cannot overlap the propagated tail
      ctr[C_ERR] |= VF_ERRBIT_CAPACITY;
      n_total = g.kp_cap;
      n_desc = max(0, g.kp_cap - n_prop);
    }
    ctr[C_NDET] = n_desc; ctr[C_NPROP] = n_prop; ctr[C_NTOTAL] = n_total; ctr[C_NDROP] = n_drop;
    ctr[C_NSURV] = n_surv;
    ctr[C_TICKET] = 0;
    const double cov = um ? (double)__ldcg(b.cov + s) / ((double)g.W * (double)g.H) : 1.0;   // masking.py:44-46
    double* rp = b.report + (long long)s * 16;
    rp[0] = n_det; rp[1] = n_prop; rp[2] = n_total; rp[3] = n_drop; rp[4] = cov;
    rp[5] = ctr[C_FRAME]; rp[6] = n_surv; rp[7] = __ldcg(&ctr[C_NCAND]);
    rp[8] += n_det; rp[9] += n_total; rp[10] += cov; rp[11] += 1.0;
  }
}

__global__ void __launch_bounds__(NF_THREADS) k_nms_finish(const __grid_constant__ Geo g, const __grid_constant__ Bufs b)
{
  __shared__ int sm[NF_THREADS / 32];
  __shared__ int red[2][NF_THREADS / 32];
  nms_finish_stream(g, b, b.s0 + blockIdx.x, sm, red);
}

#ifndef NMS_TEST_MINB
#define NMS_TEST_MINB 6   // 40 registers (152 B of spills): 888 resident CTAs take a dense step's chunks in fewer waves (config 5 none 2807 -> 2754 us)
#endif
__global__ void __launch_bounds__(NMS_CHUNK_THREADS, NMS_TEST_MINB) k_nms_test(const __grid_constant__ Geo g,
                                                                const __grid_constant__ Bufs b, int n_streams)
{
  __shared__ int sm_warp[32];
  __shared__ int red[2][NMS_CHUNK_THREADS / 32];
  __shared__ short sq[NMS_CHUNK_THREADS];   // survivors of the chunk (offsets in the chunk)
  extern __shared__ int pre[];   // [n_streams + 1]
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  stream_prefix(n_streams, pre, sm_warp, [&](int sl) {
    const int* ctr = b.ctr + (b.s0 + sl) * C_NCTR;
    return (ctr[C_ERR] & VF_ERRBIT_STAGING) ? 0 : (ctr[C_STAGE] + NMS_CHUNK_THREADS - 1) >> NMS_CHUNK_LOG;
  });
  const int total = pre[n_streams];
  int shint = 0;
  for (int item = blockIdx.x; item < total; item += gridDim.x) {
    const int sl = find_stream_from(pre, n_streams, item, shint), s = b.s0 + sl, ch = item - pre[sl];
    const int c = (ch << NMS_CHUNK_LOG) + tid;
    const int ncand = b.ctr[s * C_NCTR + C_STAGE];
    const int um = use_mask(g, b, s);
    const uint32_t* cl = b.cand + (long long)s * g.kp_cap;
    bool surv = false;
    if (c < ncand) {
      const uint32_t code = __ldcg(cl + c);
      surv = nms_test(g, b, s, um, (int)(code >> 26), (int)((code >> 13) & 0x1fffu), (int)(code & 0x1fffu));
    }
    // survivors compacted in candidate order, so the refinement runs on full warps
    int nsurv;
    const int sr = block_excl_scan<int>(surv ? 1 : 0, sm_warp, nsurv);
    if (surv) sq[sr] = (short)tid;
    __syncthreads();
    NmsOut o;
    o.flags = 0;
    int cs = 0;
    if (tid < nsurv) {
      cs = (ch << NMS_CHUNK_LOG) + sq[tid];
      const uint32_t code = __ldcg(cl + cs);
      o = nms_refine(g, b, s, um, (int)(code >> 26), (int)((code >> 13) & 0x1fffu), (int)(code & 0x1fffu));
    }
    const bool kp = (o.flags & 4) != 0;
    int nk;
    const int r = block_excl_scan<int>(kp ? 1 : 0, sm_warp, nk);
    const long long si = (long long)s * g.kp_cap + cs;
    if (kp) {
      b.st_x[si] = o.x; b.st_y[si] = o.y; b.st_s[si] = o.sig; b.st_v[si] = o.v;
      b.cand_rank[si] = r;
    }
    desc_list_kept(g, b, s, kp, o.x, o.y, o.sig, cs, lane);
    // FrameReport counts: survivors inside / outside the border margin
    int n_ok = __popc(__ballot_sync(0xffffffffu, o.flags & 2));
    int n_dr = __popc(__ballot_sync(0xffffffffu, (o.flags & 1) && !(o.flags & 2)));
    if (lane == 0) { red[0][wid] = n_ok; red[1][wid] = n_dr; }
    __syncthreads();
    if (tid == 0) {
      n_ok = 0; n_dr = 0;
#pragma unroll
      for (int k = 0; k < NMS_CHUNK_THREADS / 32; k++) { n_ok += red[0][k]; n_dr += red[1][k]; }
      b.chunk_off[(long long)s * g.nms_chunks + ch] = nk;
      if (n_ok) atomicAdd(b.nms_cnt + 4 * s + 0, n_ok);
      if (n_dr) atomicAdd(b.nms_cnt + 4 * s + 1, n_dr);
    }
    __syncthreads();
  }
}


// ============================================================================
// k_describe: descriptor.py:85-144 + pipeline.py:164-170 for kept keypoints,
// and masking.py:179-183 propagation of previous features.
// ============================================================================

// _box_mean_jit (descriptor.py:85-92) at a sample position: clamped box,
// sum // area (exact: float quotient, then a one-step integer correction).
__device__ __forceinline__ int box_mean(const uint32_t* S, const Geo& g, long long x, long long y, long long r)
{
  const int x0 = (int)max(x - r, 0LL), x1 = (int)min(x + r, (long long)g.W - 1);
  const int y0 = (int)max(y - r, 0LL), y1 = (int)min(y + r, (long long)g.H - 1);
  const uint32_t sm = box_sum(S, g, x0, x1, y0, y1);
  const uint32_t area = (uint32_t)((x1 - x0 + 1) * (y1 - y0 + 1));
  uint32_t q = (uint32_t)((float)sm * __frcp_rn((float)area));
  if (q * area > sm) q--;
  else if ((q + 1) * area <= sm) q++;
  return (int)q;
}

// ---------------------------------------------------------------------------
// Warp-batched describe: one warp takes up to 32 keypoints.
//   A. lanes sample (keypoint, point) pairs at theta = 0: 60 box means each
//      (descriptor.py:94-115 with cos 0 = 1, sin 0 = 0: the rotation is exact)
//   B. lane k runs keypoint k's orientation sum sequentially in long-pair
//      order, fp64 without FMA, exactly as _orientations_jit (:128-144)
//   C. lanes sample the rotated points (cos/sin of keypoint k's theta)
//   D. 16 __ballot_sync per keypoint build the 512 bits
//      (_describe_batch_jit :117-126), bit-reversed per byte into the
//      MSB-first packing of pack_descriptor (:271-275); 16 lanes store 64 B.
// ---------------------------------------------------------------------------
#define DW_WARPS 4
#define DS_THREADS (32 * DW_WARPS)
#define DW_ROW 68   // bytes per keypoint row (17 words: odd, so lane k's rows fall in distinct banks)

struct DescWarp {
  uint8_t v[32 * DW_ROW];   // box means are 0..255 (sum // area of uint8 pixels)
  double kx[32], ky[32], sg[32], cs[32], sn[32];
  const uint32_t* sat[32];
};

// Sample (keypoint, point) pairs into w.v: 4 pairs per lane per iteration,
// every SAT corner load issued before any is consumed (branch-free: a masked
// corner re-reads corner A and is multiplied by 0).  Boxes spanning three or
// more strips (boxes taller than VF_ST rows) take box_sum.
__device__ __forceinline__ void sample_pass(const Geo& g, DescWarp& w, int nk, int lane, bool rotated)
{
  const int npair = nk * VF_NPTS;
  const int TH = VF_ST;
  for (int q0 = lane; q0 < npair; q0 += 128) {
    const uint32_t* rowp[4][3];
    int xa[4], xb[4], area[4], dst[4];
    uint32_t msk[4];
    bool slow[4];
    int bx0[4], bx1[4], by0[4], by1[4];
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const int q = q0 + 32 * u;
      const bool valid = q < npair;
      const int k = valid ? q / VF_NPTS : 0, j = valid ? q - k * VF_NPTS : 0;
      const double sg = w.sg[k];
      double fx, fy;
      if (rotated) {
        const double c = w.cs[k], sn = w.sn[k], px = g_ptab[j][0], py = g_ptab[j][1];
        fx = w.kx[k] + sg * (c * px - sn * py) + 0.5;
        fy = w.ky[k] + sg * (sn * px + c * py) + 0.5;
      } else {
        fx = w.kx[k] + sg * g_ptab[j][0] + 0.5;
        fy = w.ky[k] + sg * g_ptab[j][1] + 0.5;
      }
      long long x = (long long)floor(fx), y = (long long)floor(fy);
      x = x < 0 ? 0 : (x > g.W - 1 ? g.W - 1 : x);
      y = y < 0 ? 0 : (y > g.H - 1 ? g.H - 1 : y);
      const int r = (int)floor(g_ptab[j][2] * sg + 0.5);
      const int x0 = max((int)x - r, 0), x1 = min((int)x + r, g.W - 1);
      const int y0 = max((int)y - r, 0), y1 = min((int)y + r, g.H - 1);
      const int ys = (int)__umulhi((uint32_t)y0, g.sth_magic) * TH;
      const int yb = min(y1, ys + TH - 1);
      const bool left = x0 > 0, top = y0 > ys, cross = y1 > yb;
      slow[u] = y1 > ys + 2 * TH - 1;
      const uint32_t* S = w.sat[k];
      rowp[u][0] = S + (long long)yb * g.W;
      rowp[u][1] = top ? S + (long long)(y0 - 1) * g.W : rowp[u][0];
      rowp[u][2] = cross ? S + (long long)y1 * g.W : rowp[u][0];
      xa[u] = left ? x0 - 1 : x1;
      xb[u] = x1;
      msk[u] = (left ? 1u : 0u) | (top ? 2u : 0u) | (cross ? 4u : 0u) | (valid ? 8u : 0u);
      area[u] = (x1 - x0 + 1) * (y1 - y0 + 1);
      dst[u] = k * DW_ROW + j;
      bx0[u] = x0; bx1[u] = x1; by0[u] = y0; by1[u] = y1;
    }
    uint32_t v[4][6];
#pragma unroll
    for (int u = 0; u < 4; u++) {
      v[u][0] = __ldca(rowp[u][0] + xb[u]);
      v[u][1] = __ldca(rowp[u][0] + xa[u]);
      v[u][2] = __ldca(rowp[u][1] + xb[u]);
      v[u][3] = __ldca(rowp[u][1] + xa[u]);
      v[u][4] = __ldca(rowp[u][2] + xb[u]);
      v[u][5] = __ldca(rowp[u][2] + xa[u]);
    }
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const uint32_t m = msk[u];
      const uint32_t L = m & 1u, T = (m >> 1) & 1u, C = (m >> 2) & 1u;
      uint32_t sm = v[u][0] - L * v[u][1] - T * (v[u][2] - L * v[u][3]) + C * (v[u][4] - L * v[u][5]);
      if (slow[u]) sm = box_sum(w.sat[dst[u] / DW_ROW], g, bx0[u], bx1[u], by0[u], by1[u]);
      const uint32_t a = (uint32_t)area[u];
      uint32_t qv = (uint32_t)((float)sm * __frcp_rn((float)a));
      if (qv * a > sm) qv--;
      else if ((qv + 1) * a <= sm) qv++;
      if (m & 8u) w.v[dst[u]] = (uint8_t)qv;
    }
  }
}

// theta_given: w.cs/w.sn already hold cos/sin of the caller's angles.
// Returns theta of lane's keypoint (lane < nk) via *theta_lane; desc_lane[q]
// (lane q < 16) receives descriptor word q of each keypoint through `emit`.
template <typename Emit>
__device__ __forceinline__ void describe_warp(const Geo& g, DescWarp& w, const uint32_t* pairs, int nk, int lane,
                                              bool theta_given, double& theta_lane, Emit emit)
{
  if (!theta_given) {
    sample_pass(g, w, nk, lane, false);
    __syncwarp();
    if (lane < nk) {
      const uint8_t* v = w.v + lane * DW_ROW;
      double gx = 0.0, gy = 0.0;
      const int L = c_nlong;
      for (int p = 0; p < L; p++) {
        const double dv = (double)(v[c_li[p]] - v[c_lj[p]]);
        gx += dv * c_wx[p];
        gy += dv * c_wy[p];
      }
      double th = atan2(gy, gx);
      th = th <= -CUDART_PI ? CUDART_PI : th;
      theta_lane = th;
      double sn, cs;
      sincos(th, &sn, &cs);
      w.cs[lane] = cs;
      w.sn[lane] = sn;
    }
    __syncwarp();
  }
  sample_pass(g, w, nk, lane, true);
  __syncwarp();
  for (int k = 0; k < nk; k++) {
    const uint8_t* v = w.v + k * DW_ROW;
    uint32_t mine = 0;
#pragma unroll
    for (int q = 0; q < 16; q++) {
      const uint32_t pr = pairs[32 * q + lane];           // si | sj << 16 (smem, conflict-free)
      const uint32_t word = __ballot_sync(0xffffffffu, v[pr & 0xffff] > v[pr >> 16]);
      if (lane == q) mine = word;
    }
    emit(k, __byte_perm(__brev(mine), 0, 0x0123));
  }
}

// Corner addresses of the box of one sample point (descriptor.py:94-115):
// fp64 position in the reference's op order, clamped box, strip-SAT corners.
struct BoxQ {
  double dist;   // distance of the unrounded sample position (x or y) to the nearest integer
  const uint32_t *r0, *r1, *r2;
  int xa, xb, area;
  uint32_t L, T, C;
  bool slow;
  int x0, x1, y0, y1;
};

__device__ __forceinline__ BoxQ box_query(const uint32_t* S, const Geo& g, double kx, double ky, double sg, double cs,
                                         double sn, double px, double py, double rad, bool rotated)
{
  double fx, fy;
  if (rotated) {
    fx = kx + sg * (cs * px - sn * py) + 0.5;
    fy = ky + sg * (sn * px + cs * py) + 0.5;
  } else {
    fx = kx + sg * px + 0.5;
    fy = ky + sg * py + 0.5;
  }
  // floor to int in one conversion (positions are within +/-2^31), then clamp
  const int x = min(max(__double2int_rd(fx), 0), g.W - 1);
  const int y = min(max(__double2int_rd(fy), 0), g.H - 1);
  const int r = __double2int_rd(rad * sg + 0.5);
  BoxQ q;
  q.dist = fmin(fabs(fx - rint(fx)), fabs(fy - rint(fy)));
  q.x0 = max(x - r, 0); q.x1 = min(x + r, g.W - 1);
  q.y0 = max(y - r, 0); q.y1 = min(y + r, g.H - 1);
  const int TH = VF_ST;
  const int ys = (int)__umulhi((uint32_t)q.y0, g.sth_magic) * TH;
  const int yb = min(q.y1, ys + TH - 1);
  q.L = q.x0 > 0; q.T = q.y0 > ys; q.C = q.y1 > yb;
  q.slow = q.y1 > ys + 2 * TH - 1;
  q.r0 = S + (long long)yb * g.W;
  q.r1 = q.T ? S + (long long)(q.y0 - 1) * g.W : q.r0;
  q.r2 = q.C ? S + (long long)q.y1 * g.W : q.r0;
  q.xa = q.L ? q.x0 - 1 : q.x1;
  q.xb = q.x1;
  q.area = (q.x1 - q.x0 + 1) * (q.y1 - q.y0 + 1);
  return q;
}

// sum // area, exact (float quotient + one-step integer correction)
__device__ __forceinline__ uint32_t exact_div(uint32_t sm, uint32_t a)
{
  uint32_t q = (uint32_t)((float)sm * __frcp_rn((float)a));
  if (q * a > sm) q--;
  else if ((q + 1) * a <= sm) q++;
  return q;
}

// Box means of two sample points: both points' corners are computed first and
// all 12 loads issued together (masked corners re-read corner A, times 0).
__device__ __forceinline__ void point_means2(const uint32_t* S, const Geo& g, double kx, double ky, double sg,
                                             double cs, double sn, const double* pa, const double* pb, bool rotated,
                                             uint32_t& ma, uint32_t& mb, double* da = nullptr, double* db = nullptr)
{
  const BoxQ a = box_query(S, g, kx, ky, sg, cs, sn, pa[0], pa[1], pa[2], rotated);
  const BoxQ c = box_query(S, g, kx, ky, sg, cs, sn, pb[0], pb[1], pb[2], rotated);
  if (da) { *da = a.dist; *db = c.dist; }
  // predicated corner loads: a corner the box does not use issues no request
  auto ld = [](bool p, const uint32_t* q) -> uint32_t { return p ? __ldg(q) : 0u; };
  const uint32_t a0 = __ldg(a.r0 + a.xb), a1 = ld(a.L, a.r0 + a.xa), a2 = ld(a.T, a.r1 + a.xb);
  const uint32_t a3 = ld(a.T && a.L, a.r1 + a.xa), a4 = ld(a.C, a.r2 + a.xb), a5 = ld(a.C && a.L, a.r2 + a.xa);
  const uint32_t c0 = __ldg(c.r0 + c.xb), c1 = ld(c.L, c.r0 + c.xa), c2 = ld(c.T, c.r1 + c.xb);
  const uint32_t c3 = ld(c.T && c.L, c.r1 + c.xa), c4 = ld(c.C, c.r2 + c.xb), c5 = ld(c.C && c.L, c.r2 + c.xa);
  uint32_t sa = a0 - a1 - (a2 - a3) + (a4 - a5);
  uint32_t sc = c0 - c1 - (c2 - c3) + (c4 - c5);
  if (__any_sync(0xffffffffu, a.slow || c.slow)) {   // a box over >= 3 strips (sigma >~ 9): rare
    if (a.slow) sa = box_sum(S, g, a.x0, a.x1, a.y0, a.y1);
    if (c.slow) sc = box_sum(S, g, c.x0, c.x1, c.y0, c.y1);
  }
  ma = exact_div(sa, (uint32_t)a.area);
  mb = exact_div(sc, (uint32_t)c.area);
}

#ifndef DSW
#define DSW 8   // warps per CTA of k_desc_fused
#endif

// ============================================================================
// Orientation helpers of k_desc_fused
// ============================================================================
__device__ __forceinline__ double dr_i2d(int n)   // exact int -> double without I2F
{
  return __hiloint2double(0x43380000, (int)(0x80000000u + (unsigned)n)) - 6755401588539392.0;
}

// Orientation from the lane's two box means m0 (point lane) and m1 (point
// lane + 32) as the linear form sum_i v_i W_i, warp-reduced (every lane ends
// with identical values).  The reference sums the 393 rounded products
// dv_p * w_p sequentially (descriptor.py:132-144); the linear form, the host
// rounding of W_i and that sequential order are all within c_ogam * sum_i v_i
// A_i of the exact sum of the products (standard recursive / pairwise
// summation bounds, c_ogam = 2 (L + 80) u), so |g_lin - g_seq| <= b per
// component.  Returns false when that bound is not small against |g| or theta
// may sit on the -pi / pi branch cut; else cs, sn = g / |g| and dth bounds the
// angle between g_lin and g_seq plus the libm and rounding differences.
__device__ __forceinline__ bool dr_orient_lin(uint32_t m0, uint32_t m1, const double (*ow)[4], int lane, double& gx,
                                              double& gy, double& cs, double& sn, double& dth)
{
  const int l1 = lane + 32;
  const double v0 = (double)m0, v1 = (double)m1;   // exact (<= 255)
  double sx = v0 * ow[lane][0] + v1 * ow[l1][0];
  double sy = v0 * ow[lane][1] + v1 * ow[l1][1];
  double ax = v0 * ow[lane][2] + v1 * ow[l1][2];
  double ay = v0 * ow[lane][3] + v1 * ow[l1][3];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sx += __shfl_xor_sync(0xffffffffu, sx, o);
    sy += __shfl_xor_sync(0xffffffffu, sy, o);
    ax += __shfl_xor_sync(0xffffffffu, ax, o);
    ay += __shfl_xor_sync(0xffffffffu, ay, o);
  }
  gx = sx;
  gy = sy;
  const double bx = c_ogam * ax, by = c_ogam * ay;
  const double g2 = sx * sx + sy * sy;
  const double rn = rsqrt(g2);
  const double gn = g2 * rn;
  if (!(bx + by < 1e-3 * gn)) return false;                // includes g == 0
  if (sx < 0.0 && fabs(sy) <= by) return false;            // theta near the +-pi cut
  cs = sx * rn;
  sn = sy * rn;
  dth = 2.02 * (bx + by) * rn + 1e-14;   // rn = 1 / |g| (to ~1 ulp)
  return true;
}

// The reference's sequential sums (one lane): the rare fallback of dr_orient_lin.
__device__ __noinline__ void dr_orient_seq_g(const uint8_t* v, double& gx_out, double& gy_out)
{
  double gx = 0.0, gy = 0.0;
  const int L = c_nlong;
  for (int p = 0; p < L; p++) {
    const double dv = dr_i2d((int)v[c_li[p]] - (int)v[c_lj[p]]);
    gx += dv * c_wx[p];
    gy += dv * c_wy[p];
  }
  gx_out = gx;
  gy_out = gy;
}

// ============================================================================
// k_desc_fused: the strip-SAT describe of one keypoint per warp in a single
// pass (descriptor.py:85-144,271-275): theta = 0 box means -> orientation
// (dr_orient_warp, certified against the sequential sum; dr_orient_seq when
// the certificate fails) -> rotated box means -> 16 ballots.  The rotated
// samples cover the same disk as the theta = 0 ones, so their SAT corners are
// mostly L1 hits of the first pass.  Keypoints: the describe list b.gidx
// (candidate indices, from k_nms_test) of the streams [s0, s0 + n).
// ============================================================================
#ifndef FUSED_PAIRS_REG
#define FUSED_PAIRS_REG 1
#endif
#ifndef FUSED_MINB
#define FUSED_MINB 2
#endif
__global__ void __launch_bounds__(32 * DSW, FUSED_MINB) k_desc_fused(const __grid_constant__ Geo g,
                                                         const __grid_constant__ Bufs b, int n_streams)
{
  __shared__ __align__(16) uint8_t vals[DSW][DW_ROW];
  __shared__ uint32_t pairs[VF_NBITS];
  __shared__ double ptab[64][3];   // pattern point x, y, smoothing radius
  __shared__ double ow[64][4];     // orientation linear form (g_ow)
  __shared__ int sm_warp[32];
  extern __shared__ int pre[];     // [n_streams + 1]
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int k = threadIdx.x; k < VF_NBITS; k += 32 * DSW) pairs[k] = g_pairs[k];
  stream_prefix(n_streams, pre, sm_warp, [&](int sl) { return b.ctr[(b.s0 + sl) * C_NCTR + C_NGLOB]; });
  const int total = pre[n_streams];
  for (int j = threadIdx.x; j < 64; j += 32 * DSW) {
    ptab[j][0] = g_ptab[j][0]; ptab[j][1] = g_ptab[j][1]; ptab[j][2] = g_ptab[j][2];
    ow[j][0] = g_ow[j][0]; ow[j][1] = g_ow[j][1]; ow[j][2] = g_ow[j][2]; ow[j][3] = g_ow[j][3];
  }
  __syncthreads();
  const int j1 = lane + 32 < VF_NPTS ? lane + 32 : lane;
  const bool has1 = lane + 32 < VF_NPTS;
  const double pn0 = sqrt(ptab[lane][0] * ptab[lane][0] + ptab[lane][1] * ptab[lane][1]);
  const double pn1 = has1 ? sqrt(ptab[j1][0] * ptab[j1][0] + ptab[j1][1] * ptab[j1][1]) : 0.0;
  uint8_t* v = vals[wid];
#if FUSED_PAIRS_REG
  uint32_t preg[16];   // this lane's 16 short pairs (bits 32 q + lane), in registers
#pragma unroll
  for (int q = 0; q < 16; q++) preg[q] = pairs[32 * q + lane];
#endif
  // The warp's keypoints are gi = g0 + k * Wt; their headers (position, scale,
  // output slot) are fetched 32 at a time, lane k for keypoint k, and lane k
  // computes keypoint k's theta = atan2(gy, gx) after the batch.
  const int Wt = gridDim.x * DSW;
  int shint = 0;   // each lane's items increase (by 32 Wt per batch)
  for (int g0 = blockIdx.x * DSW + wid; g0 < total; g0 += 32 * Wt) {
    const int gl = g0 + lane * Wt;
    long long o_l = -1;
    int s_l = 0;
    double kx_l = 0.0, ky_l = 0.0, sg_l = 0.0;
    if (gl < total) {
      const int sl = find_stream_from(pre, n_streams, gl, shint), i = gl - pre[sl];
      s_l = b.s0 + sl;
      const int* ctr = b.ctr + s_l * C_NCTR;
      // describe-list entry = candidate index c (staging slot); output rank =
      // kept keypoints of the earlier candidate chunks + rank within the chunk
      const int c = __ldcg(b.gidx + (long long)s_l * g.kp_cap + i);
      const long long si = (long long)s_l * g.kp_cap + c;
      const int rank = __ldcg(b.chunk_off + (long long)s_l * g.nms_chunks + (c >> NMS_CHUNK_LOG)) +
                       __ldcg(b.cand_rank + si);
      kx_l = __ldcg(b.st_x + si); ky_l = __ldcg(b.st_y + si); sg_l = __ldcg(b.st_s + si);
      if (rank < ctr[C_NDET]) {   // ranks past the capacity-clamped count are not written
        o_l = feat_base(g, s_l, ctr[C_FRAME] & 1, ctr[C_NTOTAL]) + rank;
        b.fx[o_l] = kx_l; b.fy[o_l] = ky_l; b.fs[o_l] = sg_l; b.fv[o_l] = __ldcg(b.st_v + si);
        b.forg[o_l] = 0; b.fage[o_l] = 0;
      }
    }
    const int nk = min(32, (total - g0 + Wt - 1) / Wt);
    double gx_l = 0.0, gy_l = 0.0;
#pragma unroll 1
    for (int k = 0; k < nk; k++) {
      const long long o = __shfl_sync(0xffffffffu, o_l, k);
      if (o < 0) continue;   // warp-uniform
      const int s = __shfl_sync(0xffffffffu, s_l, k);
      const double kx = __shfl_sync(0xffffffffu, kx_l, k), ky = __shfl_sync(0xffffffffu, ky_l, k);
      const double sg = __shfl_sync(0xffffffffu, sg_l, k);
      const uint32_t* S = b.sat + (long long)s * g.W * g.H;
      uint32_t m0, m1;
      point_means2(S, g, kx, ky, sg, 1.0, 0.0, ptab[lane], ptab[j1], false, m0, m1);
      if (!has1) m1 = 0u;
      const uint32_t z0 = m0, z1 = m1;   // theta = 0 means (for the fallback)
      double gx, gy, cs = 1.0, sn = 0.0, dth = 0.0;
      bool ok = dr_orient_lin(m0, m1, ow, lane, gx, gy, cs, sn, dth) && !b.orient_seq;
      if (ok) {
        double d0, d1;
        point_means2(S, g, kx, ky, sg, cs, sn, ptab[lane], ptab[j1], true, m0, m1, &d0, &d1);
        const double ue = 1.5 * sg * dth;
        const bool near0 = pn0 > 0.0 && d0 < ue * pn0 + 1e-11;
        const bool near1 = has1 && pn1 > 0.0 && d1 < ue * pn1 + 1e-11;
        ok = !__any_sync(0xffffffffu, near0 || near1);
      }
      if (!ok) {   // rare: the reference's sequential sum and the device libm
        v[lane] = (uint8_t)z0;
        if (has1) v[lane + 32] = (uint8_t)z1;
        __syncwarp();
        double tx = 0.0, ty = 0.0;
        if (lane == 0) dr_orient_seq_g(v, tx, ty);
        gx = __shfl_sync(0xffffffffu, tx, 0);
        gy = __shfl_sync(0xffffffffu, ty, 0);
        double th = atan2(gy, gx);
        th = th <= -CUDART_PI ? CUDART_PI : th;
        sincos(th, &sn, &cs);
        point_means2(S, g, kx, ky, sg, cs, sn, ptab[lane], ptab[j1], true, m0, m1);
      }
      if (lane == k) { gx_l = gx; gy_l = gy; }
      __syncwarp();
      v[lane] = (uint8_t)m0;
      if (has1) v[lane + 32] = (uint8_t)m1;
      __syncwarp();
      uint32_t mine = 0u;
#pragma unroll
      for (int q = 0; q < 16; q++) {
#if FUSED_PAIRS_REG
        const uint32_t pr = preg[q];
#else
        const uint32_t pr = pairs[32 * q + lane];   // si | sj << 16 (smem, conflict-free)
#endif
        const uint32_t word = __ballot_sync(0xffffffffu, v[pr & 0xffff] > v[pr >> 16]);
        if (lane == q) mine = word;
      }
      if (lane < 16) reinterpret_cast<uint32_t*>(b.fdesc + o * 64)[lane] = __byte_perm(__brev(mine), 0, 0x0123);
      __syncwarp();
    }
    if (o_l >= 0) {   // theta of lane's keypoint (descriptor.py:142-143)
      double th = atan2(gy_l, gx_l);
      b.ft[o_l] = th <= -CUDART_PI ? CUDART_PI : th;
    }
  }
}

// Eq. 1: previous features under a 0 mask bit, in previous-list order, origin
// -> propagated, age + 1 (masking.py:179-183).  CTA per 1024-feature chunk of
// the previous list (chunk output offsets from k_worklist's counts): every
// field of the chunk is loaded up front (most features propagate), one
// ballot-based chunk scan gives the destinations, then the 64-B descriptors
// are copied by the whole CTA as consecutive 16-B words (coalesced).
#define PROP_PER (PROP_CHUNK / 256)
static_assert(PROP_PER * 7 <= 32, "flag + rank packing");
__global__ void __launch_bounds__(256, 4) k_propagate(const __grid_constant__ Geo g, const __grid_constant__ Bufs b)
{
  __shared__ int wsum[PROP_PER][8];
  __shared__ int dsts[PROP_CHUNK];
  const int s = b.s0 + blockIdx.y, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (!use_mask(g, b, s)) return;
  const int* ctr = b.ctr + s * C_NCTR;
  const int cur = ctr[C_FRAME] & 1, prev = cur ^ 1;
  const int n_prev = ctr[C_NFEAT0 + prev];
  const int n_prop = ctr[C_NPROP];                       // from k_worklist (same stream, earlier)
  const int nch = (n_prev + PROP_CHUNK - 1) / PROP_CHUNK;
  const long long fb = feat_base(g, s, prev, n_prev);
  const long long ob = feat_base(g, s, cur, n_prop);     // the propagated segment: the last n_prop slots
  for (int c = blockIdx.x; c < nch; c += gridDim.x) {
    const int base = c * PROP_CHUNK;
    // phase 1: the merge bit of every feature of the chunk -> destination slots
    double xs[PROP_PER], ys[PROP_PER];
#pragma unroll
    for (int j = 0; j < PROP_PER; j++) {
      const int e = base + j * 256 + tid;
      const long long p = fb + (e < n_prev ? e : 0);
      xs[j] = b.fx[p];
      ys[j] = b.fy[p];
    }
    unsigned fl = 0;
#pragma unroll
    for (int j = 0; j < PROP_PER; j++) {
      const int e = base + j * 256 + tid;
      const bool f = e < n_prev && !merge_mask_at(g, b, s, xs[j], ys[j]);
      const unsigned bal = __ballot_sync(0xffffffffu, f);
      if (lane == 0) wsum[j][wid] = __popc(bal);
      // keep mask of features e - lane .. e - lane + 31 (the delta result of vf_pipeline_collect_delta)
      if (b.keep_bits && lane == 0 && e < n_prev) b.keep_bits[(long long)s * b.keep_words + (e >> 5)] = bal;
      fl |= (f ? 1u : 0u) << j;
      fl |= (unsigned)__popc(bal & ((1u << lane) - 1)) << (4 + 6 * j);   // rank within the warp (<= 31)
    }
    __syncthreads();
    // element (j, tid) goes after all of group j' < j and warps w < wid of group j
    int acc = 0;
    const long long dst0 = b.prop_out[(long long)s * g.prop_chunks + c];
#pragma unroll
    for (int j = 0; j < PROP_PER; j++) {
      int inwarp = 0, grp = 0;
#pragma unroll
      for (int w = 0; w < 8; w++) {
        const int v = wsum[j][w];
        inwarp += w < wid ? v : 0;
        grp += v;
      }
      const long long dst = dst0 + acc + inwarp + ((fl >> (4 + 6 * j)) & 0x3fu);
      acc += grp;
      dsts[j * 256 + tid] = ((fl >> j) & 1u) && dst < n_prop ? (int)dst : -1;
    }
    __syncthreads();
    // phase 2: every field copied by the whole CTA in source order (loads
    // independent of each other, stores mostly contiguous)
    const int nvalid = min(PROP_CHUNK, n_prev - base);
#pragma unroll
    for (int j = 0; j < PROP_PER; j++) {
      const int f = j * 256 + tid;
      const int dst = f < nvalid ? dsts[f] : -1;
      if (dst >= 0) {
        const long long p = fb + base + f, o = ob + dst;   // ob: segment start
        const double x = b.fx[p], y = b.fy[p], sg = b.fs[p], th = b.ft[p], v = b.fv[p];
        const int ag = b.fage[p];
        b.fx[o] = x; b.fy[o] = y; b.fs[o] = sg; b.ft[o] = th; b.fv[o] = v;
        b.forg[o] = 1; b.fage[o] = ag + 1;
      }
    }
    // descriptors: 4 x 16 B per feature, word q = feature q / 4, part q % 4
    const uint4* src = reinterpret_cast<const uint4*>(b.fdesc + (fb + base) * 64);
    uint4* dstd = reinterpret_cast<uint4*>(b.fdesc + ob * 64);   // segment start
#pragma unroll
    for (int half = 0; half < 2; half++) {
      uint4 d[8];
      int dq[8];
#pragma unroll
      for (int i = 0; i < 8; i++) {
        const int q = (half * 8 + i) * 256 + tid, f = q >> 2;
        const int dst = f < nvalid ? dsts[f] : -1;
        dq[i] = dst < 0 ? -1 : dst * 4 + (q & 3);
        if (dst >= 0) d[i] = src[q];
      }
#pragma unroll
      for (int i = 0; i < 8; i++)
        if (dq[i] >= 0) dstd[dq[i]] = d[i];
    }
    __syncthreads();
  }
}

// ============================================================================
// k_pack: features of streams [0, n) into one contiguous SoA (for a single
// device->host copy per field); pre[s] = first index of stream s.
// ============================================================================
__global__ void __launch_bounds__(256) k_pack(const __grid_constant__ Geo g, const __grid_constant__ Bufs b,
                                              int n_streams, int buf_override, double* px, double* py, double* ps,
                                              double* pt, double* pv, uint8_t* po, int* pa, uint8_t* pd,
                                              int* pre_out, long long pack_cap, int* err_out)
{
  __shared__ int sm_warp[32];
  extern __shared__ int pre[];
  stream_prefix(n_streams, pre, sm_warp, [&](int s) {
    const int* ctr = b.ctr + s * C_NCTR;
    const int buf = buf_override >= 0 ? buf_override : ((ctr[C_FRAME] - 1) & 1);   // last finished frame
    return ctr[C_NFEAT0 + buf];
  });
  if (blockIdx.x == 0)
    for (int s = threadIdx.x; s <= n_streams; s += blockDim.x) {
      pre_out[s] = pre[s];
      if (err_out && s < n_streams) err_out[s] = b.ctr[s * C_NCTR + C_ERR];   // sticky capacity flags
    }
  const int total = pre[n_streams];
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total && i < pack_cap;
       i += (long long)gridDim.x * blockDim.x) {
    int lo = 0, hi = n_streams;
    while (hi - lo > 1) { int m = (lo + hi) >> 1; if (pre[m] <= i) lo = m; else hi = m; }
    const int s = lo, k = (int)(i - pre[s]);
    const int* ctr = b.ctr + s * C_NCTR;
    const int buf = buf_override >= 0 ? buf_override : ((ctr[C_FRAME] - 1) & 1);
    const long long f = feat_base(g, s, buf, ctr[C_NFEAT0 + buf]) + k;
    px[i] = b.fx[f]; py[i] = b.fy[f]; ps[i] = b.fs[f]; pt[i] = b.ft[f]; pv[i] = b.fv[f];
    po[i] = b.forg[f]; pa[i] = b.fage[f];
    const uint4* sd = reinterpret_cast<const uint4*>(b.fdesc + f * 64);
    uint4* dd = reinterpret_cast<uint4*>(pd + i * 64);
    dd[0] = sd[0]; dd[1] = sd[1]; dd[2] = sd[2]; dd[3] = sd[3];
  }
}

// ============================================================================
// k_pack_delta: the step's result as a delta against the previous lists
// (vf_pipeline_collect_delta): every stream's DETECTED records (the head of
// its list) packed contiguously, plus the Eq. 1 keep mask of its previous
// list (masking.py:176-183).  With the previous list on the host, list n =
// detected ++ [previous[i], origin propagated, age + 1, for each kept i],
// exactly the merged list.  Runs after k_finalize (counters of frame f).
// ============================================================================
__global__ void __launch_bounds__(256) k_pack_delta(const __grid_constant__ Geo g, const __grid_constant__ Bufs b,
                                                    int n_streams, double* px, double* py, double* ps, double* pt,
                                                    double* pv, uint8_t* pd, uint32_t* pk, int* pre_det,
                                                    int* pre_kw, int* counts, long long cap, long long kcap,
                                                    int* err_out)
{
  __shared__ int sm_warp[32];
  extern __shared__ int pre[];   // [2][n_streams + 1]: detected, keep words
  int* pw = pre + n_streams + 1;
  auto nbits = [&](int s) {
    const int* ctr = b.ctr + s * C_NCTR;
    const bool masked = (g.mask_mode == 1 || g.mask_mode == 2) && ctr[C_FRAME] >= 2;
    return masked ? ctr[C_NFEAT0 + (ctr[C_FRAME] & 1)] : 0;   // the previous list's length
  };
  stream_prefix(n_streams, pre, sm_warp, [&](int s) { return b.ctr[s * C_NCTR + C_NDET]; });
  stream_prefix(n_streams, pw, sm_warp, [&](int s) { return (nbits(s) + 31) >> 5; });
  if (blockIdx.x == 0)
    for (int s = threadIdx.x; s <= n_streams; s += blockDim.x) {
      pre_det[s] = pre[s];
      pre_kw[s] = pw[s];
      if (s < n_streams) {
        const int* ctr = b.ctr + s * C_NCTR;
        counts[3 * s] = ctr[C_NDET]; counts[3 * s + 1] = ctr[C_NPROP]; counts[3 * s + 2] = nbits(s);
        if (err_out) err_out[s] = ctr[C_ERR];   // sticky capacity flags
      }
    }
  const int total = pre[n_streams], words = pw[n_streams];
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total && i < cap;
       i += (long long)gridDim.x * blockDim.x) {
    const int s = find_stream(pre, n_streams, (int)i), k = (int)(i - pre[s]);
    const int* ctr = b.ctr + s * C_NCTR;
    const int buf = (ctr[C_FRAME] - 1) & 1;
    const long long f = feat_base(g, s, buf, ctr[C_NFEAT0 + buf]) + k;
    px[i] = b.fx[f]; py[i] = b.fy[f]; ps[i] = b.fs[f]; pt[i] = b.ft[f]; pv[i] = b.fv[f];
    const uint4* sd = reinterpret_cast<const uint4*>(b.fdesc + f * 64);
    uint4* dd = reinterpret_cast<uint4*>(pd + i * 64);
    dd[0] = sd[0]; dd[1] = sd[1]; dd[2] = sd[2]; dd[3] = sd[3];
  }
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < words && i < kcap;
       i += (long long)gridDim.x * blockDim.x) {
    const int s = find_stream(pw, n_streams, (int)i), k = (int)(i - pw[s]);
    const int nb = nbits(s);
    uint32_t v = b.keep_bits[(long long)s * b.keep_words + k];
    if (32 * k + 32 > nb) v &= (1u << (nb - 32 * k)) - 1u;   // bits past the list (last word)
    pk[i] = v;
  }
}

// ============================================================================
// k_copy_out: the packed fields of a step -> the caller's host arrays in one
// launch (vf_pipeline_collect*, when every destination is pinned host memory
// the device can address): the SMs write over PCIe, so a step's result costs
// one launch instead of one DMA copy (~10 us of fixed cost each) per field.
// ============================================================================
struct CopySeg { const uint8_t* src; uint8_t* dst; long long bytes; };
struct CopySegs { CopySeg seg[8]; int n; };
__global__ void __launch_bounds__(256) k_copy_out(const __grid_constant__ CopySegs cs)
{
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x, nt = (long long)gridDim.x * blockDim.x;
  for (int k = 0; k < cs.n; k++) {
    const CopySeg sg = cs.seg[k];
    if (((reinterpret_cast<uintptr_t>(sg.src) | reinterpret_cast<uintptr_t>(sg.dst)) & 15) == 0) {
      const long long nv = sg.bytes >> 4;
      for (long long i = tid; i < nv; i += nt)
        reinterpret_cast<uint4*>(sg.dst)[i] = __ldcs(reinterpret_cast<const uint4*>(sg.src) + i);
      for (long long i = (nv << 4) + tid; i < sg.bytes; i += nt) sg.dst[i] = sg.src[i];
    } else {
      for (long long i = tid; i < sg.bytes; i += nt) sg.dst[i] = sg.src[i];
    }
  }
}

// ============================================================================
// k_finalize: state carried to the next frame (pipeline.py:276-277)
// ============================================================================
__global__ void k_finalize(const __grid_constant__ Geo g, const __grid_constant__ Bufs b, int n_streams)
{
  const int sl = blockIdx.x * blockDim.x + threadIdx.x;
  if (sl < n_streams) {
    const int s = b.s0 + sl;
    int* ctr = b.ctr + s * C_NCTR;
    const int cur = ctr[C_FRAME] & 1;
    if (b.hist && ctr[C_FRAME] < b.hist_frames) {   // per-frame FrameReport history (end-of-run gather)
      const double* rp = b.report + (long long)s * 16;
      double* h = b.hist + ((long long)s * b.hist_frames + ctr[C_FRAME]) * 8;
#pragma unroll
      for (int k = 0; k < 8; k++) h[k] = rp[k];
    }
    ctr[C_NFEAT0 + cur] = ctr[C_NTOTAL];
    ctr[C_FRAME] += 1;
    ctr[C_EPOCH] += 1;
    ctr[C_NCAND] = 0;
    b.cov[s] = 0ull;
  }
}

// vf_reset: forget the temporal state; the activity epoch stays monotonic so
// stamps written before the reset can never match again.
__global__ void k_reset(int* ctr, unsigned long long* cov, double* report, int n_streams)
{
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_streams) return;
  for (int k = 0; k < C_NCTR; k++)
    if (k != C_EPOCH) ctr[s * C_NCTR + k] = 0;
  ctr[s * C_NCTR + C_EPOCH] += 1;
  cov[s] = 0ull;
  for (int k = 0; k < 16; k++) report[(long long)s * 16 + k] = 0.0;
}

// Capacity retry (vf_process_checked): undo the counters of the step just run
// on streams [s0, s0 + n) so it can be replayed from the same state.  The
// previous feature buffer and the previous IDDM octave (the other parity)
// were only read by the step; activity stamps are epoch-based and the epoch
// stays monotonic.
__global__ void k_rollback(int* ctr, double* report, int s0, int n)
{
  const int s = s0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= s0 + n) return;
  int* c = ctr + s * C_NCTR;
  c[C_FRAME] -= 1;
  c[C_ERR] = 0;
  double* rp = report + (long long)s * 16;
  rp[8] -= rp[0]; rp[9] -= rp[2]; rp[10] -= rp[4]; rp[11] -= 1.0;
}

// ============================================================================
// Stand-alone stage kernels (drop-in for the reference's per-stage public
// functions; they share the device code above).
// ============================================================================
// intensity_diff_mask (masking.py:84-93)
__global__ void k_intensity_mask(const uint8_t* prev, const uint8_t* cur, long long n, double t_i, uint8_t* out)
{
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    int d = (int)cur[i] - (int)prev[i];
    d = d < 0 ? -d : d;
    out[i] = (double)d > t_i;
  }
}

// ast_corner_score (detector.py:58-71) at any arc length: the largest t with
// arc_len contiguous circle pixels (arc starts 0..15, indices mod 16) all
// > c + t or all < c - t, i.e. max over starts of (min over the arc) - 1,
// clipped at 0.  Thread per query point (validated on the host).
__constant__ signed char c_circle[16][2] = {{0, -3}, {1, -3}, {2, -2}, {3, -1}, {3, 0}, {3, 1}, {2, 2}, {1, 3},
                                            {0, 3}, {-1, 3}, {-2, 2}, {-3, 1}, {-3, 0}, {-3, -1}, {-2, -2}, {-1, -3}};
__global__ void k_ast_score(const uint8_t* layer, long long pitch, int n, const int* xs, const int* ys, int arc,
                            int* out)
{
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int x = xs[i], y = ys[i];
  const int c = layer[(long long)y * pitch + x];
  int d[16];
#pragma unroll
  for (int k = 0; k < 16; k++) d[k] = (int)layer[(long long)(y + c_circle[k][1]) * pitch + x + c_circle[k][0]] - c;
  // an arc of >= 16 pixels covers the whole circle (indices repeat mod 16)
  const int a = arc < 16 ? arc : 16;
  int best = 0;
#pragma unroll 1
  for (int st = 0; st < 16; st++) {
    int mb = d[st], md = -d[st];
#pragma unroll 1
    for (int k = 1; k < a; k++) {
      int j = st + k;
      j = j >= 16 ? j - 16 : j;
      mb = min(mb, d[j]);
      md = min(md, -d[j]);
    }
    best = max(best, max(mb - 1, md - 1));
  }
  out[i] = max(best, 0);
}

// sad_block (temporal.py:63-67): sum of |a - b| of n-byte patches, CTA per patch.
__global__ void k_sad_block(const uint8_t* a, const uint8_t* b, long long n, int count, long long* out)
{
  __shared__ unsigned long long part[32];
  const uint8_t* pa = a + (long long)blockIdx.x * n;
  const uint8_t* pb = b + (long long)blockIdx.x * n;
  unsigned long long acc = 0;
  for (long long k = threadIdx.x; k < n; k += blockDim.x) acc += (unsigned)abs((int)pa[k] - (int)pb[k]);
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) t += part[w];
    out[blockIdx.x] = (long long)t;
  }
  (void)count;
}

// binning_histogram (masking.py:96-119)
__global__ void k_binning_hist(int n, const double* xs, const double* ys, int W, int H, int rows, int cols,
                               unsigned long long* hist)
{
  const double sx = (double)((W + cols - 1) / cols), sy = (double)((H + rows - 1) / rows);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    long long k = (long long)floor(xs[i] / sx), r = (long long)floor(ys[i] / sy);
    k = k < 0 ? 0 : (k > cols - 1 ? cols - 1 : k);
    r = r < 0 ? 0 : (r > rows - 1 ? rows - 1 : r);
    atomicAdd(hist + r * cols + k, 1ull);
  }
}

// upsample_mask (masking.py:139-148)
__global__ void k_upsample(const uint8_t* bits, int cols, int cw, int ch, int W, int H, uint8_t* full)
{
  const long long n = (long long)W * H;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    int y = (int)(i / W), x = (int)(i - (long long)y * W);
    full[i] = bits[(y / ch) * cols + x / cw];
  }
}

// _mask_values (masking.py:157-165) on a full-resolution mask
__global__ void k_mask_values(const uint8_t* full, int W, int H, int n, const double* xs, const double* ys, uint8_t* out)
{
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    long long xi = (long long)floor(xs[i] + 0.5), yi = (long long)floor(ys[i] + 0.5);
    xi = xi < 0 ? 0 : (xi > W - 1 ? W - 1 : xi);
    yi = yi < 0 ? 0 : (yi > H - 1 ? H - 1 : yi);
    out[i] = full[yi * W + xi];
  }
}

// orientations_batch / describe_batch (descriptor.py:194-232) on caller keypoints.
// theta_in == nullptr: estimate orientation first; else describe at the given angles.
__global__ void __launch_bounds__(DS_THREADS) k_describe_batch(const __grid_constant__ Geo g, const uint32_t* sat, int n,
                                                               const double* kx, const double* ky, const double* sg,
                                                               const double* theta_in, double* theta_out, uint8_t* desc)
{
  __shared__ DescWarp ws[DW_WARPS];
  __shared__ uint32_t pairs[VF_NBITS];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int k = threadIdx.x; k < VF_NBITS; k += DS_THREADS) pairs[k] = g_pairs[k];
  __syncthreads();
  DescWarp& w = ws[wid];
  const int base = (blockIdx.x * DW_WARPS + wid) * 32;
  if (base >= n) return;
  const int nk = min(32, n - base);
  double th = 0.0;
  if (lane < nk) {
    w.kx[lane] = kx[base + lane]; w.ky[lane] = ky[base + lane]; w.sg[lane] = sg[base + lane];
    w.sat[lane] = sat;
    if (theta_in) {
      th = theta_in[base + lane];
      double sn, cs;
      sincos(th, &sn, &cs);
      w.cs[lane] = cs; w.sn[lane] = sn;
    }
  }
  __syncwarp();
  describe_warp(g, w, pairs, nk, lane, theta_in != nullptr, th, [&](int k, uint32_t word) {
    if (desc && lane < 16) reinterpret_cast<uint32_t*>(desc + (long long)(base + k) * 64)[lane] = word;
  });
  if (lane < nk && theta_out) theta_out[base + lane] = th;
}

// Candidate bitmap from caller score maps (nms_and_refine, detector.py:310-324):
// every nonzero pixel is a candidate; all tiles active.
__global__ void k_bitmap_from_maps(const __grid_constant__ Geo g, const __grid_constant__ Bufs b)
{
  const int l = blockIdx.y;
  const LayerGeo& Lg = g.L[l];
  const long long nw = (long long)Lg.h * Lg.bm_words;
  const uint8_t* sm = b.scores + Lg.sm_off;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nw; i += (long long)gridDim.x * blockDim.x) {
    int y = (int)(i / Lg.bm_words), k = (int)(i - (long long)y * Lg.bm_words);
    uint32_t word = 0;
    for (int bit = 0; bit < 32; bit++) {
      int x = 32 * k + bit;
      if (x < Lg.w && sm[(long long)y * Lg.pitch + x]) word |= 1u << bit;
    }
    b.bitmaps[Lg.bm_off + i] = word;
  }
}
