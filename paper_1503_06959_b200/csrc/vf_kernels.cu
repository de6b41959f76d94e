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

// Descriptor sampling pattern (pattern.py:21-106), uploaded by vf_set_pattern.
#define VF_NPTS 60
#define VF_NBITS 512
#define VF_MAXLONG 512
__constant__ double c_px[VF_NPTS], c_py[VF_NPTS], c_rad[VF_NPTS];
__constant__ short c_si[VF_NBITS], c_sj[VF_NBITS];
__constant__ short c_li[VF_MAXLONG], c_lj[VF_MAXLONG];
__constant__ double c_wx[VF_MAXLONG], c_wy[VF_MAXLONG];
__constant__ int c_nlong;

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

__global__ void __launch_bounds__(256) k_pyramid(const __grid_constant__ Geo g, const __grid_constant__ Bufs b)
{
  extern __shared__ __align__(16) uint8_t smem[];
  const int s = blockIdx.z;
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
  uint32_t* ssat = reinterpret_cast<uint32_t*>(smem + acc);

  if (blockIdx.x == 0 && blockIdx.y == 0 && tid == 0) {
    b.ctr[s * C_NCTR + C_STAGE] = 0;
    if (s == 0) *b.work_count = 0;
  }

  // ---- load the o0 tile ------------------------------------------------------
  const int tw = min(g.ptw, g.W - X0), th = min(g.pth, g.H - Y0);
  const uint8_t* src = b.frames + (long long)s * b.frame_stride + (long long)Y0 * b.frame_pitch + X0;
  uint8_t* t0 = smem + off[0];
  const bool vec = ((reinterpret_cast<uintptr_t>(src) | (uintptr_t)b.frame_pitch) & 15) == 0 && tw == g.ptw;
  if (vec) {
    const int per_row = g.ptw / 16;
    for (int i = tid; i < th * per_row; i += nt) {
      int y = i / per_row, c = i - y * per_row;
      uint4 v = __ldg(reinterpret_cast<const uint4*>(src + (long long)y * b.frame_pitch) + c);
      *reinterpret_cast<uint4*>(t0 + y * g.ptw + 16 * c) = v;
    }
  } else {
    for (int i = tid; i < th * g.ptw; i += nt) {
      int y = i / g.ptw, x = i - y * g.ptw;
      t0[i] = x < tw ? __ldg(src + (long long)y * b.frame_pitch + x) : 0;
    }
  }
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
      if (l == 1) {
        // i0: area-weighted 2/3 resample of o0 (pyramid.py:76-94): per axis
        // even output 2a+b, odd a+2b, then (v+4)//9.
        for (int i = tid; i < vw * vh; i += nt) {
          int y = i / vw, x = i - y * vw;
          int ky = y >> 1, kx = x >> 1;
          int ry0 = (y & 1) ? 3 * ky + 1 : 3 * ky, cy0 = (y & 1) ? 1 : 2, cy1 = (y & 1) ? 2 : 1;
          int rx0 = (x & 1) ? 3 * kx + 1 : 3 * kx, cx0 = (x & 1) ? 1 : 2, cx1 = (x & 1) ? 2 : 1;
          const uint8_t* r0 = t0 + ry0 * g.ptw;
          const uint8_t* r1 = r0 + g.ptw;
          uint32_t a0 = cy0 * r0[rx0] + cy1 * r1[rx0];
          uint32_t a1 = cy0 * r0[rx0 + 1] + cy1 * r1[rx0 + 1];
          uint32_t v = cx0 * a0 + cx1 * a1;
          uint8_t q = (uint8_t)((v + 4) / 9);
          dst[y * lw + x] = q;
          gdst[(long long)y * g.L[l].pitch + x] = q;
        }
      } else {
        // halving of the same chain's previous level (pyramid.py:67-73)
        int pl = l - 2, pw, ph;
        lvl_dims(g, pl, pw, ph);
        const uint8_t* sp = smem + off[pl];
        for (int i = tid; i < vw * vh; i += nt) {
          int y = i / vw, x = i - y * vw;
          const uint8_t* r0 = sp + (2 * y) * pw + 2 * x;
          uint32_t sum = r0[0] + r0[1] + r0[pw] + r0[pw + 1];
          uint8_t q = (uint8_t)((sum + 2) >> 2);
          dst[y * lw + x] = q;
          gdst[(long long)y * g.L[l].pitch + x] = q;
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
      uint8_t* st = b.state + (long long)s * g.state_slab + g.state_off[lv];
      uint8_t* cells = b.cells + (long long)s * g.cell_slab + G.cell_off;
      for (int i = tid; i < vw * vh; i += nt) {
        int y = i / vw, x = i - y * vw;
        long long gi = (long long)(gy0 + y) * g.L[l].w + gx0 + x;
        int c = cur[y * lw + x];
        if (um) {
          int p = st[gi];
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

  // ---- tile-local summed-area table (descriptor.py:28-32) ---------------------
  // L(y, x) = sum of o0 over [tile_y0, y] x [tile_x0, x]; box sums decompose
  // over the <= 4 tiles a box touches (see box_sum).  Values < 2^32.
  {
    const int lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
    const int per = (g.ptw + 31) / 32;
    for (int y = wid; y < th; y += nw) {
      uint32_t run = 0;
      int xb = lane * per;
      for (int k = 0; k < per; k++) {
        int x = xb + k;
        if (x < tw) run += t0[y * g.ptw + x];
      }
      uint32_t inc = run;
      for (int o = 1; o < 32; o <<= 1) {
        uint32_t v = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += v;
      }
      uint32_t r = inc - run;
      for (int k = 0; k < per; k++) {
        int x = xb + k;
        if (x < tw) { r += t0[y * g.ptw + x]; ssat[y * g.ptw + x] = r; }
      }
    }
    __syncthreads();
    for (int x = tid; x < tw; x += nt) {
      uint32_t run = 0;
      for (int y = 0; y < th; y++) { run += ssat[y * g.ptw + x]; ssat[y * g.ptw + x] = run; }
    }
    __syncthreads();
    uint32_t* gs = b.sat + (long long)s * g.W * g.H;
    for (int i = tid; i < th * tw; i += nt) {
      int y = i / tw, x = i - y * tw;
      gs[(long long)(Y0 + y) * g.W + X0 + x] = ssat[y * g.ptw + x];
    }
  }
}

// ============================================================================
// k_binmask: masking.py:96-136 (histogram of the previous MERGED features,
// pipeline.py:184-185), thresholded at t_h; coverage = covered pixels / WH.
// ============================================================================
__global__ void __launch_bounds__(1024) k_binmask(const __grid_constant__ Geo g, const __grid_constant__ Bufs b)
{
  extern __shared__ int hist[];
  const int s = blockIdx.x;
  if (!use_mask(g, b, s)) return;
  const GridGeo& G = g.grid[0];
  const int n_cells = G.rows * G.cols;
  for (int i = threadIdx.x; i < n_cells; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  const int* ctr = b.ctr + s * C_NCTR;
  const int prev = (ctr[C_FRAME] & 1) ^ 1;
  const int n_prev = ctr[C_NFEAT0 + prev];
  const long long fb = ((long long)s * 2 + prev) * g.kp_cap;
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
__global__ void __launch_bounds__(256) k_worklist(const __grid_constant__ Geo g, const __grid_constant__ Bufs b,
                                                   int tile_ctas)
{
  const int s = blockIdx.y;
  const int* ep = b.epoch;
  const int epoch = *ep;
  const int um = use_mask(g, b, s);
  const int lane = threadIdx.x & 31;
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
  const int tile = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (tile >= g.tiles_per_stream) return;
  int l = 0;
  while (l + 1 < g.NL && tile >= g.L[l + 1].tile_base) l++;
  const LayerGeo& Lg = g.L[l];
  const int t = tile - Lg.tile_base;
  const int ty = t / Lg.tiles_x, tx = t - ty * Lg.tiles_x;
  int active = 1;
  if (um) {
    const int y0 = ty * VF_TILE_H, y1 = min(Lg.h, y0 + VF_TILE_H) - 1;
    const int x0 = tx * VF_TILE_W, x1 = min(Lg.w, x0 + VF_TILE_W) - 1;
    const int* lut = b.lut + Lg.rc_off;
    const int r0 = __ldg(lut + y0), r1 = __ldg(lut + y1);
    const int c0 = __ldg(lut + Lg.h + x0), c1 = __ldg(lut + Lg.h + x1);
    const GridGeo& G = g.grid[grid_of_layer(g, l)];
    const uint8_t* cells = b.cells + (long long)s * g.cell_slab + G.cell_off;
    const int nc = c1 - c0 + 1, ncell = (r1 - r0 + 1) * nc;
    int any = 0;
    for (int i = lane; i < ncell && !any; i += 32) {
      int r = r0 + i / nc, c = c0 + i % nc;
      any = cells[(long long)r * G.cols + c];
    }
    active = __any_sync(0xffffffffu, any);
  }
  if (lane == 0) {
    if (active) {
      b.tile_stamp[(long long)s * g.tiles_per_stream + tile] = epoch;
      b.band_stamp[(long long)s * g.bands_per_stream + Lg.band_base + ty] = epoch;
      int pos = atomicAdd(b.work_count, 1);
      b.worklist[pos] = s * g.tiles_per_stream + tile;
    }
  }
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
__device__ __forceinline__ uint32_t arc_max_min9(const uint32_t w[4])
{
  uint32_t m2[4], m4[4], m9[4];
#pragma unroll
  for (int q = 0; q < 4; q++) m2[q] = __vminu4(w[q], __byte_perm(w[q], w[(q + 1) & 3], 0x4321));
#pragma unroll
  for (int q = 0; q < 4; q++) m4[q] = __vminu4(m2[q], __byte_perm(m2[q], m2[(q + 1) & 3], 0x5432));
#pragma unroll
  for (int q = 0; q < 4; q++) m9[q] = __vminu4(__vminu4(m4[q], m4[(q + 1) & 3]), w[(q + 2) & 3]);
  uint32_t m = __vmaxu4(__vmaxu4(m9[0], m9[1]), __vmaxu4(m9[2], m9[3]));
  m = __vmaxu4(m, m >> 16);
  m = __vmaxu4(m, m >> 8);
  return m & 0xffu;
}

__global__ void __launch_bounds__(128) k_fast(const __grid_constant__ Geo g, const __grid_constant__ Bufs b)
{
  __shared__ __align__(16) uint8_t tile[FT_ROWS][FT_COLS];
  __shared__ __align__(16) uint8_t sc[VF_TILE_H][VF_TILE_W];
  __shared__ uint16_t queue[VF_TILE_H * VF_TILE_W];
  __shared__ int qn;
  const int tid = threadIdx.x;
  const int n_work = *b.work_count;
  const int t = g.threshold;
  const uint32_t tt = (uint32_t)t * 0x01010101u;
  for (int item = blockIdx.x; item < n_work; item += gridDim.x) {
    const int code = b.worklist[item];
    const int s = code / g.tiles_per_stream, tile_id = code - s * g.tiles_per_stream;
    int l = 0;
    while (l + 1 < g.NL && tile_id >= g.L[l + 1].tile_base) l++;
    const LayerGeo& Lg = g.L[l];
    const int tl = tile_id - Lg.tile_base;
    const int ty = tl / Lg.tiles_x, tx = tl - ty * Lg.tiles_x;
    const int y0 = ty * VF_TILE_H, x0 = tx * VF_TILE_W;
    const int w = Lg.w, h = Lg.h;
    int pitch;
    const uint8_t* lp = layer_ptr(g, b, s, l, pitch);
    const int um = use_mask(g, b, s);
    // ---- stage rows y0-3 .. y0+10, cols x0-16 .. x0+143 ----
    const bool vec_ok = ((reinterpret_cast<uintptr_t>(lp) | (uintptr_t)pitch) & 15) == 0;
    for (int i = tid; i < FT_ROWS * (FT_COLS / 16); i += blockDim.x) {
      int rr = i / (FT_COLS / 16), cc = i - rr * (FT_COLS / 16);
      int y = y0 - 3 + rr, x = x0 - 16 + 16 * cc;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (y >= 0 && y < h) {
        const uint8_t* row = lp + (long long)y * pitch;
        if (vec_ok && x >= 0 && x + 16 <= pitch && x + 16 <= ((w + 15) & ~15)) {
          v = __ldg(reinterpret_cast<const uint4*>(row + x));
        } else {
          uint8_t tmp[16];
#pragma unroll
          for (int k = 0; k < 16; k++) tmp[k] = (x + k >= 0 && x + k < w) ? __ldg(row + x + k) : 0;
          v = *reinterpret_cast<uint4*>(tmp);
        }
      }
      *reinterpret_cast<uint4*>(&tile[rr][16 * cc]) = v;
    }
    for (int i = tid; i < VF_TILE_H * VF_TILE_W / 16; i += blockDim.x)
      reinterpret_cast<uint4*>(&sc[0][0])[i] = make_uint4(0, 0, 0, 0);
    if (tid == 0) qn = 0;
    __syncthreads();
    // ---- pass 1: 4-point necessary test, 4 pixels per word ----
    for (int wi = tid; wi < VF_TILE_H * (VF_TILE_W / 4); wi += blockDim.x) {
      const int r = wi >> 5, k = wi & 31;
      const int y = y0 + r;
      uint32_t pass = 0;
      if (y >= 3 && y < h - 3) {
        const int cb = 16 + 4 * k;
        const uint32_t C = *reinterpret_cast<const uint32_t*>(&tile[r + 3][cb]);
        const uint32_t P = *reinterpret_cast<const uint32_t*>(&tile[r + 3][cb - 4]);
        const uint32_t B = *reinterpret_cast<const uint32_t*>(&tile[r + 3][cb + 4]);
        const uint32_t N = *reinterpret_cast<const uint32_t*>(&tile[r][cb]);
        const uint32_t S = *reinterpret_cast<const uint32_t*>(&tile[r + 6][cb]);
        const uint32_t E = __byte_perm(C, B, 0x6543), Wd = __byte_perm(P, C, 0x4321);
        const uint32_t br = (__vcmpgtu4(__vsubus4(N, C), tt) | __vcmpgtu4(__vsubus4(S, C), tt)) &
                            (__vcmpgtu4(__vsubus4(E, C), tt) | __vcmpgtu4(__vsubus4(Wd, C), tt));
        const uint32_t dk = (__vcmpgtu4(__vsubus4(C, N), tt) | __vcmpgtu4(__vsubus4(C, S), tt)) &
                            (__vcmpgtu4(__vsubus4(C, E), tt) | __vcmpgtu4(__vsubus4(C, Wd), tt));
        pass = br | dk;
        if (pass) {
#pragma unroll
          for (int i = 0; i < 4; i++) {
            const int x = x0 + 4 * k + i;
            bool ok = x >= 3 && x < w - 3;
            if (ok && um) ok = gate_at(g, b, s, l, y, x);
            if (!ok) pass &= ~(0xffu << (8 * i));
          }
        }
      }
      const int np = __popc(pass) >> 3;
      // warp-aggregated queue append
      int incl = np;
      const int lane = tid & 31;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      int wbase = 0;
      const int wtot = __shfl_sync(0xffffffffu, incl, 31);
      if (lane == 31 && wtot) wbase = atomicAdd(&qn, wtot);
      wbase = __shfl_sync(0xffffffffu, wbase, 31);
      int pos = wbase + incl - np;
#pragma unroll
      for (int i = 0; i < 4; i++)
        if (pass & (0xffu << (8 * i))) queue[pos++] = (uint16_t)(r * VF_TILE_W + 4 * k + i);
    }
    __syncthreads();
    // ---- pass 2: exact score of queued pixels ----
    const int nq = qn;
    for (int qi = tid; qi < nq; qi += blockDim.x) {
      const int p = queue[qi];
      const int r = p / VF_TILE_W, c = p - r * VF_TILE_W;
      const int R = r + 3, Cc = 16 + c;
      const uint32_t ctr = tile[R][Cc];
      uint32_t ring[4];
      ring[0] = tile[R - 3][Cc] | (tile[R - 3][Cc + 1] << 8) | (tile[R - 2][Cc + 2] << 16) | (tile[R - 1][Cc + 3] << 24);
      ring[1] = tile[R][Cc + 3] | (tile[R + 1][Cc + 3] << 8) | (tile[R + 2][Cc + 2] << 16) | (tile[R + 3][Cc + 1] << 24);
      ring[2] = tile[R + 3][Cc] | (tile[R + 3][Cc - 1] << 8) | (tile[R + 2][Cc - 2] << 16) | (tile[R + 1][Cc - 3] << 24);
      ring[3] = tile[R][Cc - 3] | (tile[R - 1][Cc - 3] << 8) | (tile[R - 2][Cc - 2] << 16) | (tile[R - 3][Cc - 1] << 24);
      const uint32_t c4 = ctr * 0x01010101u;
      uint32_t bw[4], dw[4];
#pragma unroll
      for (int q = 0; q < 4; q++) { bw[q] = __vsubus4(ring[q], c4); dw[q] = __vsubus4(c4, ring[q]); }
      const int best = (int)max(arc_max_min9(bw), arc_max_min9(dw));
      const int score = best - 1;
      if (score >= t) sc[r][c] = (uint8_t)score;
    }
    __syncthreads();
    // ---- store scores (whole tile: gated pixels read back as 0) + bitmap ----
    uint8_t* smap = b.scores + (long long)s * g.sm_slab + Lg.sm_off;
    for (int i = tid; i < VF_TILE_H * (VF_TILE_W / 16); i += blockDim.x) {
      const int r = i >> 3, cc = i & 7;
      const int y = y0 + r, x = x0 + 16 * cc;
      if (y >= h || x >= w) continue;
      uint8_t* dst = smap + (long long)y * Lg.pitch + x;
      *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(&sc[r][16 * cc]);  // pitch padded to 16
    }
    if (tid < VF_TILE_H * VF_TILE_WORDS) {
      const int r = tid >> 2, kw = tid & 3;
      const int y = y0 + r;
      if (y < h && x0 + 32 * kw < w) {
        uint32_t word = 0;
#pragma unroll
        for (int q = 0; q < 8; q++) {
          uint32_t v = *reinterpret_cast<const uint32_t*>(&sc[r][32 * kw + 4 * q]);
          uint32_t nz = __vcmpne4(v, 0u);
          // bytes 0xff/0x00 -> 4 bits
          uint32_t bits = ((nz >> 7) & 1u) | ((nz >> 14) & 2u) | ((nz >> 21) & 4u) | ((nz >> 28) & 8u);
          word |= bits << (4 * q);
        }
        b.bitmaps[(long long)s * g.bm_slab_words + Lg.bm_off + (long long)y * Lg.bm_words + 4 * tx + kw] = word;
        const int n = __popc(word);
        if (n) atomicAdd(&b.ctr[s * C_NCTR + C_NCAND], n);
      }
    }
    __syncthreads();
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
#define NMS_THREADS 128
#define NMS_ROUND 512

__device__ __forceinline__ int score_read(const Geo& g, const Bufs& b, int s, int um, int l, int y, int x)
{
  const LayerGeo& Lg = g.L[l];
  if (y < 0 || y >= Lg.h || x < 0 || x >= Lg.w) return 0;
  if (um && !gate_at(g, b, s, l, y, x)) return 0;    // gated pixels score 0 (detector.py:112-114)
  return b.scores[(long long)s * g.sm_slab + Lg.sm_off + (long long)y * Lg.pitch + x];
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

__device__ __forceinline__ int patch_read(const Geo& g, const Bufs& b, int s, int um, int l, int y, int x, double p[3][3])
{
  int mx = INT_MIN;
#pragma unroll
  for (int dy = -1; dy <= 1; dy++)
#pragma unroll
    for (int dx = -1; dx <= 1; dx++) {
      int v = score_read(g, b, s, um, l, y + dy, x + dx);
      p[dy + 1][dx + 1] = (double)v;
      mx = v > mx ? v : mx;
    }
  return mx;
}

struct NmsOut { double x, y, sig, v; int flags; };  // flags: 1 survivor, 2 border ok, 4 kept

__device__ NmsOut nms_one(const Geo& g, const Bufs& b, int s, int um, int l, int y, int x)
{
  NmsOut o; o.flags = 0; o.x = o.y = o.sig = o.v = 0.0;
  const LayerGeo& Lg = g.L[l];
  const int sv = score_read(g, b, s, um, l, y, x);
  if (sv == 0) return o;
  bool keep = true;
#pragma unroll
  for (int dy = -1; dy <= 1; dy++)
#pragma unroll
    for (int dx = -1; dx <= 1; dx++)
      if (dx || dy) {
        int yy = y + dy, xx = x + dx;
        if (g.nms_wrap) {                                // smap[ys+dy, xs+dx] (detector.py:260-262)
          yy = yy < 0 ? yy + Lg.h : yy;
          xx = xx < 0 ? xx + Lg.w : xx;
        }
        keep &= sv > score_read(g, b, s, um, l, yy, xx);
      }
  int yj[2], xj[2];
#pragma unroll
  for (int k = 0; k < 2; k++) {                          // detector.py:264-273
    const int j = l - 1 + 2 * k;
    if (j < 0 || j >= g.NL) continue;
    const int hj = g.L[j].h, wj = g.L[j].w;
    long long a = ((long long)y * hj + (Lg.h >> 1)) / Lg.h;
    long long c = ((long long)x * wj + (Lg.w >> 1)) / Lg.w;
    yj[k] = (int)(a < hj - 1 ? a : hj - 1);
    xj[k] = (int)(c < wj - 1 ? c : wj - 1);
    keep &= sv > score_read(g, b, s, um, j, yj[k], xj[k]);
  }
  if (!keep) return o;
  o.flags = 1;
  double p[3][3], ox, oy, v0;
  int ok;
  patch_read(g, b, s, um, l, y, x, p);
  fit_peak(p, ox, oy, v0, ok);
  double nv[2] = {0.0, 0.0};
#pragma unroll
  for (int k = 0; k < 2; k++) {                          // detector.py:281-285
    const int j = l - 1 + 2 * k;
    if (j < 0 || j >= g.NL) continue;
    double pj[3][3], tx, ty, vj;
    int okj;
    int pmax = patch_read(g, b, s, um, j, yj[k], xj[k], pj);
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
    const double a = delta > 0.0 ? delta : 0.0;
    const double c = -delta > 0.0 ? -delta : 0.0;
    sig = Lg.sigma * pow(up, a) * pow(down, c);
  }
  double xf = ((double)x + ox) / Lg.scale;               // detector.py:299-302
  double yf = ((double)y + oy) / Lg.scale;
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

__device__ void nms_last_cta(const Geo& g, const Bufs& b, int s, int* sm_warp)
{
  // exclusive scans over band records and propagation chunks of stream s
  __shared__ int carry;
  const int tid = threadIdx.x;
  int* rec = b.band_rec + (long long)s * g.bands_per_stream * 4;
  int* bout = b.band_out + (long long)s * g.bands_per_stream;
  int tot;
  if (tid == 0) carry = 0;
  __syncthreads();
  int n_drop = 0, n_surv = 0;
  for (int base = 0; base < g.bands_per_stream; base += blockDim.x) {
    int i = base + tid;
    int k = 0;
    if (i < g.bands_per_stream) {
      k = __ldcg(rec + 4 * i + 1);
      n_drop += __ldcg(rec + 4 * i + 3);
      n_surv += __ldcg(rec + 4 * i + 2) + __ldcg(rec + 4 * i + 3);
    }
    int ex = block_excl_scan<int>(k, sm_warp, tot);
    if (i < g.bands_per_stream) bout[i] = carry + ex;
    __syncthreads();
    if (tid == 0) carry += tot;
    __syncthreads();
  }
  const int n_det = carry;
  __syncthreads();
  if (tid == 0) carry = 0;
  __syncthreads();
  int* pc = b.prop_cnt + (long long)s * g.prop_chunks;
  int* po = b.prop_out + (long long)s * g.prop_chunks;
  for (int base = 0; base < g.prop_chunks; base += blockDim.x) {
    int i = base + tid;
    int k = i < g.prop_chunks ? __ldcg(pc + i) : 0;
    int ex = block_excl_scan<int>(k, sm_warp, tot);
    if (i < g.prop_chunks) po[i] = carry + ex;
    __syncthreads();
    if (tid == 0) carry += tot;
    __syncthreads();
  }
  const int n_prop = carry;
  // block reduce n_drop, n_surv
  for (int o = 16; o > 0; o >>= 1) {
    n_drop += __shfl_down_sync(0xffffffffu, n_drop, o);
    n_surv += __shfl_down_sync(0xffffffffu, n_surv, o);
  }
  __shared__ int red[2][32];
  if ((tid & 31) == 0) { red[0][tid >> 5] = n_drop; red[1][tid >> 5] = n_surv; }
  __syncthreads();
  if (tid == 0) {
    int d = 0, sv = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) { d += red[0][w]; sv += red[1][w]; }
    int* ctr = b.ctr + s * C_NCTR;
    int n_total = n_det + n_prop;
    if (n_total > g.kp_cap) { ctr[C_ERR] |= VF_ERRBIT_CAPACITY; n_total = g.kp_cap; }
    ctr[C_NDET] = n_det; ctr[C_NPROP] = n_prop; ctr[C_NTOTAL] = n_total; ctr[C_NDROP] = d;
    ctr[C_NSURV] = sv;
    ctr[C_TICKET] = 0;
    const int um = use_mask(g, b, s);
    double cov = um ? (double)__ldcg(b.cov + s) / ((double)g.W * (double)g.H) : 1.0;   // masking.py:44-46
    double* rp = b.report + (long long)s * 16;
    rp[0] = n_det; rp[1] = n_prop; rp[2] = n_total; rp[3] = d; rp[4] = cov;
    rp[5] = ctr[C_FRAME]; rp[6] = sv; rp[7] = __ldcg(&ctr[C_NCAND]);
    rp[8] += n_det; rp[9] += n_total; rp[10] += cov; rp[11] += 1.0;
  }
}

__global__ void __launch_bounds__(NMS_THREADS) k_nms(const __grid_constant__ Geo g, const __grid_constant__ Bufs b)
{
  __shared__ int sm_warp[32];
  __shared__ int sh_base, sh_last;
  __shared__ int cand_yx[NMS_ROUND];
  __shared__ double r_x[NMS_ROUND], r_y[NMS_ROUND], r_s[NMS_ROUND], r_v[NMS_ROUND];
  __shared__ uint8_t r_f[NMS_ROUND];
  const int s = blockIdx.y, bid = blockIdx.x, tid = threadIdx.x;
  const int epoch = *b.epoch;
  const int um = use_mask(g, b, s);
  int* ctr = b.ctr + s * C_NCTR;
  const int cur = ctr[C_FRAME] & 1, prev = cur ^ 1;

  if (bid < g.bands_per_stream) {
    int* rec = b.band_rec + ((long long)s * g.bands_per_stream + bid) * 4;
    int kept = 0, n_ok = 0, n_drop = 0, base = 0;
    if (b.band_stamp[(long long)s * g.bands_per_stream + bid] == epoch) {
      int l = 0;
      while (l + 1 < g.NL && bid >= g.L[l + 1].band_base) l++;
      const LayerGeo& Lg = g.L[l];
      const int ty = bid - Lg.band_base;
      const int y0 = ty * VF_TILE_H, nrows = min(Lg.h - y0, VF_TILE_H);
      const int nwords = nrows * Lg.bm_words;
      const uint32_t* bm = b.bitmaps + (long long)s * g.bm_slab_words + Lg.bm_off + (long long)y0 * Lg.bm_words;
      const int* tst = b.tile_stamp + (long long)s * g.tiles_per_stream + Lg.tile_base + ty * Lg.tiles_x;
      const int per = (nwords + NMS_THREADS - 1) / NMS_THREADS;
      const int w0 = tid * per, w1 = min(nwords, w0 + per);
      int cnt = 0;
      for (int i = w0; i < w1; i++) {
        const int k = i % Lg.bm_words;
        if (tst[k / VF_TILE_WORDS] == epoch) cnt += __popc(__ldcg(bm + i));
      }
      int total;
      const int ex = block_excl_scan<int>(cnt, sm_warp, total);
      if (total > 0) {
        if (tid == 0) {
          int bs = atomicAdd(&ctr[C_STAGE], total);
          if (bs + total > g.kp_cap) { atomicOr(&ctr[C_ERR], VF_ERRBIT_STAGING); bs = -1; }
          sh_base = bs;
        }
        __syncthreads();
        base = sh_base;
        if (base >= 0) {
          for (int r0 = 0; r0 < total; r0 += NMS_ROUND) {
            // enumerate this round's candidates in row-major order
            int idx = ex;
            for (int i = w0; i < w1 && idx < r0 + NMS_ROUND; i++) {
              const int k = i % Lg.bm_words;
              if (tst[k / VF_TILE_WORDS] != epoch) continue;
              uint32_t word = __ldcg(bm + i);
              while (word) {
                const int bit = __ffs(word) - 1;
                word &= word - 1;
                if (idx >= r0 && idx < r0 + NMS_ROUND) {
                  const int yy = y0 + i / Lg.bm_words, xx = 32 * k + bit;
                  cand_yx[idx - r0] = (yy << 16) | xx;
                }
                idx++;
              }
            }
            __syncthreads();
            const int nr = min(NMS_ROUND, total - r0);
            for (int e = tid; e < nr; e += NMS_THREADS) {
              const int yx = cand_yx[e];
              NmsOut o = nms_one(g, b, s, um, l, yx >> 16, yx & 0xffff);
              r_x[e] = o.x; r_y[e] = o.y; r_s[e] = o.sig; r_v[e] = o.v; r_f[e] = (uint8_t)o.flags;
            }
            __syncthreads();
            // ordered compaction of kept entries
            const int per2 = (nr + NMS_THREADS - 1) / NMS_THREADS;
            const int e0 = tid * per2, e1 = min(nr, e0 + per2);
            int kc = 0, okc = 0, dc = 0;
            for (int e = e0; e < e1; e++) {
              const int f = r_f[e];
              kc += (f >> 2) & 1;
              okc += (f >> 1) & 1;
              dc += (f & 1) && !(f & 2);
            }
            int rtot;
            int kex = block_excl_scan<int>(kc, sm_warp, rtot);
            long long dst = (long long)s * g.kp_cap + base + kept + kex;
            for (int e = e0; e < e1; e++) {
              if (r_f[e] & 4) {
                b.st_x[dst] = r_x[e]; b.st_y[dst] = r_y[e]; b.st_s[dst] = r_s[e]; b.st_v[dst] = r_v[e];
                dst++;
              }
            }
            int t2;
            okc = block_excl_scan<int>(okc, sm_warp, t2), n_ok += t2;
            dc = block_excl_scan<int>(dc, sm_warp, t2), n_drop += t2;
            kept += rtot;
            __syncthreads();
          }
        } else {
          base = 0;
        }
      }
    }
    if (tid == 0) { rec[0] = base; rec[1] = kept; rec[2] = n_ok; rec[3] = n_drop; }
  } else {
    // propagation chunk: count previous features under a 0 mask bit (masking.py:179-183)
    const int c = bid - g.bands_per_stream;
    const int n_prev = ctr[C_NFEAT0 + prev];
    int cnt = 0;
    if (um) {
      const long long fb = ((long long)s * 2 + prev) * g.kp_cap;
      const int e0 = c * 1024 + tid * 8;
      for (int e = e0; e < min(n_prev, e0 + 8); e++)
        cnt += !merge_mask_at(g, b, s, b.fx[fb + e], b.fy[fb + e]);
    }
    int tot;
    block_excl_scan<int>(cnt, sm_warp, tot);
    if (tid == 0) b.prop_cnt[(long long)s * g.prop_chunks + c] = tot;
  }
  // ---- last CTA of the stream scans ----
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    int tk = atomicAdd(&ctr[C_TICKET], 1);
    sh_last = (tk == (int)gridDim.x - 1);
  }
  __syncthreads();
  if (sh_last) {
    __threadfence();
    nms_last_cta(g, b, s, sm_warp);
  }
}

// ============================================================================
// k_describe: descriptor.py:85-144 + pipeline.py:164-170 for kept keypoints,
// and masking.py:179-183 propagation of previous features.
// ============================================================================
#define DS_THREADS 128

// Box sum over [x0,x1] x [y0,y1] from the tile-local SATs (mod 2^32 exact).
__device__ __forceinline__ uint32_t box_sum(const uint32_t* sat, const Geo& g, int x0, int x1, int y0, int y1)
{
  uint32_t sum = 0;
  const int TW = g.ptw, TH = g.pth, W = g.W;
  for (int ty = y0 / TH; ty <= y1 / TH; ty++) {
    const int ty0 = ty * TH;
    const int ya = max(y0, ty0), yb = min(y1, ty0 + TH - 1);
    for (int tx = x0 / TW; tx <= x1 / TW; tx++) {
      const int tx0 = tx * TW;
      const int xa = max(x0, tx0), xb = min(x1, tx0 + TW - 1);
      uint32_t A = __ldg(sat + (long long)yb * W + xb);
      uint32_t Bv = ya > ty0 ? __ldg(sat + (long long)(ya - 1) * W + xb) : 0u;
      uint32_t Cv = xa > tx0 ? __ldg(sat + (long long)yb * W + xa - 1) : 0u;
      uint32_t Dv = (ya > ty0 && xa > tx0) ? __ldg(sat + (long long)(ya - 1) * W + xa - 1) : 0u;
      sum += A - Bv - Cv + Dv;
    }
  }
  return sum;
}

// _box_mean_jit (descriptor.py:85-92) at a sample position
__device__ __forceinline__ int box_mean(const uint32_t* sat, const Geo& g, long long x, long long y, long long r)
{
  const int x0 = (int)max(x - r, 0LL), x1 = (int)min(x + r, (long long)g.W - 1);
  const int y0 = (int)max(y - r, 0LL), y1 = (int)min(y + r, (long long)g.H - 1);
  const uint32_t s = box_sum(sat, g, x0, x1, y0, y1);
  return (int)(s / (uint32_t)((x1 - x0 + 1) * (y1 - y0 + 1)));
}

// One keypoint: theta (descriptor.py:128-144) then 512 bits (descriptor.py:117-126).
__device__ void describe_one(const Geo& g, const uint32_t* sat, double kx, double ky, double sg, int* sv,
                             double& theta_out, uint32_t bits[16])
{
  const int stride = DS_THREADS;
  // pass 1: theta = 0 (cos 0 = 1, sin 0 = 0 make the rotation exact)
  for (int j = 0; j < VF_NPTS; j++) {
    long long x = (long long)floor(kx + sg * c_px[j] + 0.5);
    long long y = (long long)floor(ky + sg * c_py[j] + 0.5);
    x = x < 0 ? 0 : (x > g.W - 1 ? g.W - 1 : x);
    y = y < 0 ? 0 : (y > g.H - 1 ? g.H - 1 : y);
    long long r = (long long)floor(c_rad[j] * sg + 0.5);
    sv[j * stride] = box_mean(sat, g, x, y, r);
  }
  // sequential fp64 sums in long-pair order (no FMA), as _orientations_jit
  double gx = 0.0, gy = 0.0;
  const int L = c_nlong;
  for (int p = 0; p < L; p++) {
    const double dv = (double)(sv[c_li[p] * stride] - sv[c_lj[p] * stride]);
    gx += dv * c_wx[p];
    gy += dv * c_wy[p];
  }
  double th = atan2(gy, gx);
  th = th <= -CUDART_PI ? CUDART_PI : th;
  theta_out = th;
  // pass 2: rotated samples
  double sn, cs;
  sincos(th, &sn, &cs);
  for (int j = 0; j < VF_NPTS; j++) {
    const double px = c_px[j], py = c_py[j];
    long long x = (long long)floor(kx + sg * (cs * px - sn * py) + 0.5);
    long long y = (long long)floor(ky + sg * (sn * px + cs * py) + 0.5);
    x = x < 0 ? 0 : (x > g.W - 1 ? g.W - 1 : x);
    y = y < 0 ? 0 : (y > g.H - 1 ? g.H - 1 : y);
    long long r = (long long)floor(c_rad[j] * sg + 0.5);
    sv[j * stride] = box_mean(sat, g, x, y, r);
  }
#pragma unroll
  for (int q = 0; q < 16; q++) bits[q] = 0;
  for (int k = 0; k < VF_NBITS; k++) {
    if (sv[c_si[k] * stride] > sv[c_sj[k] * stride]) {
      // MSB-first bytes (descriptor.py:271-275): bit k -> byte k>>3, mask 0x80>>(k&7)
      const int B = k >> 3;
      bits[B >> 2] |= (0x80u >> (k & 7)) << (8 * (B & 3));
    }
  }
}

__global__ void __launch_bounds__(DS_THREADS) k_describe(const __grid_constant__ Geo g, const __grid_constant__ Bufs b)
{
  __shared__ int sv_all[VF_NPTS * DS_THREADS];
  __shared__ int sm_warp[32];
  const int s = blockIdx.y, bid = blockIdx.x, tid = threadIdx.x;
  const int* ctr = b.ctr + s * C_NCTR;
  const int cur = ctr[C_FRAME] & 1, prev = cur ^ 1;
  const long long ob = ((long long)s * 2 + cur) * g.kp_cap;
  if (bid < g.bands_per_stream) {
    const int* rec = b.band_rec + ((long long)s * g.bands_per_stream + bid) * 4;
    const int kept = rec[1];
    if (kept == 0) return;
    const long long sb = (long long)s * g.kp_cap + rec[0];
    const int out0 = b.band_out[(long long)s * g.bands_per_stream + bid];
    const uint32_t* sat = b.sat + (long long)s * g.W * g.H;
    int* sv = sv_all + tid;
    for (int i = tid; i < kept; i += DS_THREADS) {
      const double kx = b.st_x[sb + i], ky = b.st_y[sb + i], sg = b.st_s[sb + i];
      double th;
      uint32_t bits[16];
      describe_one(g, sat, kx, ky, sg, sv, th, bits);
      const long long o = ob + out0 + i;
      if (out0 + i >= g.kp_cap) continue;
      b.fx[o] = kx; b.fy[o] = ky; b.fs[o] = sg; b.ft[o] = th; b.fv[o] = b.st_v[sb + i];
      b.forg[o] = 0; b.fage[o] = 0;
      uint4* d = reinterpret_cast<uint4*>(b.fdesc + o * 64);
      d[0] = make_uint4(bits[0], bits[1], bits[2], bits[3]);
      d[1] = make_uint4(bits[4], bits[5], bits[6], bits[7]);
      d[2] = make_uint4(bits[8], bits[9], bits[10], bits[11]);
      d[3] = make_uint4(bits[12], bits[13], bits[14], bits[15]);
    }
  } else {
    // Eq. 1: previous features under a 0 mask bit, in previous-list order,
    // origin -> propagated, age + 1 (masking.py:179-183)
    if (!use_mask(g, b, s)) return;
    const int c = bid - g.bands_per_stream;
    const int n_prev = ctr[C_NFEAT0 + prev];
    if (c * 1024 >= n_prev) return;
    const long long fb = ((long long)s * 2 + prev) * g.kp_cap;
    const int e0 = c * 1024 + tid * 8, e1 = min(n_prev, e0 + 8);
    uint32_t flags = 0;
    int cnt = 0;
    for (int e = e0; e < e1; e++)
      if (!merge_mask_at(g, b, s, b.fx[fb + e], b.fy[fb + e])) { flags |= 1u << (e - e0); cnt++; }
    int tot;
    int ex = block_excl_scan<int>(cnt, sm_warp, tot);
    long long dst = (long long)ctr[C_NDET] + b.prop_out[(long long)s * g.prop_chunks + c] + ex;
    for (int e = e0; e < e1; e++) {
      if (!(flags & (1u << (e - e0)))) continue;
      if (dst < g.kp_cap) {
        const long long o = ob + dst, p = fb + e;
        b.fx[o] = b.fx[p]; b.fy[o] = b.fy[p]; b.fs[o] = b.fs[p]; b.ft[o] = b.ft[p]; b.fv[o] = b.fv[p];
        b.forg[o] = 1; b.fage[o] = b.fage[p] + 1;
        const uint4* sd = reinterpret_cast<const uint4*>(b.fdesc + p * 64);
        uint4* dd = reinterpret_cast<uint4*>(b.fdesc + o * 64);
        dd[0] = sd[0]; dd[1] = sd[1]; dd[2] = sd[2]; dd[3] = sd[3];
      }
      dst++;
    }
  }
}

// ============================================================================
// k_finalize: state carried to the next frame (pipeline.py:276-277)
// ============================================================================
__global__ void k_finalize(const __grid_constant__ Geo g, const __grid_constant__ Bufs b, int n_streams)
{
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < n_streams) {
    int* ctr = b.ctr + s * C_NCTR;
    const int cur = ctr[C_FRAME] & 1;
    ctr[C_NFEAT0 + cur] = ctr[C_NTOTAL];
    ctr[C_FRAME] += 1;
    ctr[C_NCAND] = 0;
    b.cov[s] = 0ull;
  }
  if (s == 0) *b.epoch += 1;
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
// theta_in == nullptr: estimate orientation, else describe at the given angles.
__global__ void __launch_bounds__(DS_THREADS) k_describe_batch(const __grid_constant__ Geo g, const uint32_t* sat, int n,
                                                               const double* kx, const double* ky, const double* sg,
                                                               const double* theta_in, double* theta_out, uint8_t* desc)
{
  __shared__ int sv_all[VF_NPTS * DS_THREADS];
  const int i = blockIdx.x * DS_THREADS + threadIdx.x;
  if (i >= n) return;
  int* sv = sv_all + threadIdx.x;
  double th;
  uint32_t bits[16];
  if (theta_in == nullptr) {
    describe_one(g, sat, kx[i], ky[i], sg[i], sv, th, bits);
    if (theta_out) theta_out[i] = th;
    if (desc) {
      uint4* d = reinterpret_cast<uint4*>(desc + (long long)i * 64);
      for (int q = 0; q < 4; q++) d[q] = make_uint4(bits[4 * q], bits[4 * q + 1], bits[4 * q + 2], bits[4 * q + 3]);
    }
    return;
  }
  // describe at a given theta: reuse pass 2 of describe_one
  const double t = theta_in[i];
  double sn, cs;
  sincos(t, &sn, &cs);
  const int stride = DS_THREADS;
  for (int j = 0; j < VF_NPTS; j++) {
    const double px = c_px[j], py = c_py[j];
    long long x = (long long)floor(kx[i] + sg[i] * (cs * px - sn * py) + 0.5);
    long long y = (long long)floor(ky[i] + sg[i] * (sn * px + cs * py) + 0.5);
    x = x < 0 ? 0 : (x > g.W - 1 ? g.W - 1 : x);
    y = y < 0 ? 0 : (y > g.H - 1 ? g.H - 1 : y);
    long long r = (long long)floor(c_rad[j] * sg[i] + 0.5);
    sv[j * stride] = box_mean(sat, g, x, y, r);
  }
  for (int q = 0; q < 16; q++) bits[q] = 0;
  for (int k = 0; k < VF_NBITS; k++)
    if (sv[c_si[k] * stride] > sv[c_sj[k] * stride]) {
      const int B = k >> 3;
      bits[B >> 2] |= (0x80u >> (k & 7)) << (8 * (B & 3));
    }
  if (theta_out) theta_out[i] = t;
  uint4* d = reinterpret_cast<uint4*>(desc + (long long)i * 64);
  for (int q = 0; q < 4; q++) d[q] = make_uint4(bits[4 * q], bits[4 * q + 1], bits[4 * q + 2], bits[4 * q + 3]);
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
