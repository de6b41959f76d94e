// vf_common.cuh -- shared device-side definitions of the B200 detect+describe path.
//
// Geometry, per-stream slab layout and device helpers shared by every kernel.
// The reference is a CPU package (vidfeat 0.1.0); citations are file:line in
// /root/reference/pkg/src/vidfeat/.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define VF_MAXO 8                 // max octaves
#define VF_MAXL (2 * VF_MAXO)     // layers o0,i0,o1,i1,...
#define VF_MAXG VF_MAXO           // mask grids (per_layer: one per octave level)

// FAST tiles (layer coordinates): 128 columns x 8 rows.  An NMS band is one
// row of tiles (8 layer rows, full layer width), so bands emit keypoints in
// the reference's (layer, y, x) order (detector.py:251-253,303-306).
#define VF_TILE_W 128
#define VF_TILE_H 8
#define VF_TILE_WORDS (VF_TILE_W / 32)

// per-stream int32 counters
enum {
  C_FRAME = 0,      // frames processed on this stream
  C_NFEAT0 = 1,     // features in buffer 0
  C_NFEAT1 = 2,     // features in buffer 1
  C_NDET = 3, C_NPROP = 4, C_NTOTAL = 5, C_NDROP = 6,
  C_STAGE = 7,      // staging bump allocator
  C_TICKET = 8,     // last-CTA ticket (NMS launch)
  C_ERR = 9,        // sticky error bits
  C_NSURV = 10,     // NMS survivors (before border filter)
  C_NCAND = 11,     // FAST candidates
  C_EPOCH = 12,     // monotonic step id (activity stamps), survives vf_reset
  C_PTICKET = 13,   // last-CTA ticket of the propagation-count CTAs (k_worklist)
  C_NGLOB = 14,     // kept keypoints in the describe list (b.gidx) this step
  C_NCTR = 16
};
#define VF_ERRBIT_CAPACITY 1
#define VF_ERRBIT_STAGING 2
#define VF_ERRBIT_INDEX 4
#define VF_ERRBIT_SATMARK 8   // VF_SAT_CHECK=1: a kept keypoint's footprint tile was not marked by k_fast

#define VF_ST 32   // strip-SAT tile edge and strip height (o0 pixels)

#define NMS_CHUNK_LOG 8          // NMS candidates per k_nms_test CTA pass: 256

struct LayerGeo {
  int w, h;
  int pitch;            // derived-layer / score-map pitch (bytes)
  int tiles_x, tiles_y; // FAST tiles
  int tile_base;        // first tile id of this layer within a stream
  int band_base;        // first band id (== tile row) of this layer
  int row_base;         // first NMS row id of this layer (rows of all layers, layer order)
  int bm_words;         // candidate-bitmap words per row
  long long layer_off;  // byte offset of the derived layer in the layer slab (l >= 1)
  long long sm_off;     // byte offset of the score map in the score slab
  long long bm_off;     // word offset of the bitmap in the bitmap slab
  int rc_off, cc_off;   // offsets of the row/col -> cell LUTs (per grid, see Geo)
  double scale, sigma;  // pyramid.py:122-124; detector.py:243
  double rinv_h, rinv_w;  // 1 / h, 1 / w (exact integer division by h, w)
  int sat_reach;        // o0 pixels around floor(x / scale) that a kept keypoint's footprint box stays within
  float inv_scale;      // 1 / scale (k_fast's early SAT-tile marks)
};

struct GridGeo {          // a cell grid of the detection mask (masking.py:30-55)
  int rows, cols, cw, ch; // cell size in full-res pixels (masking.py:143-144)
  long long cell_off;     // byte offset in the cell slab
};

struct Geo {
  int W, H, O, NL;
  int threshold;
  int mask_mode;        // 0 none, 1 intensity, 2 binning
  int per_layer;        // intensity per octave level (pipeline.py:188-200)
  int mask_level;       // octave level of the IDDM source (pipeline.py:187)
  double t_i;           // masking.py:26
  int t_h;              // masking.py:70
  int n_grids;
  GridGeo grid[VF_MAXG];
  LayerGeo L[VF_MAXL];
  int tiles_per_stream, bands_per_stream, rows_per_stream;
  long long layer_slab, sm_slab, bm_slab_words, cell_slab, lut_len;
  // pyramid tiles (kernel k_pyramid), also the SAT tiles
  int ptw, pth, ptx, pty;   // pyramid tiles (o0 pixels)
  int stx, sty;             // strip-SAT tiles: VF_ST x VF_ST o0 pixels, stx x sty per frame
  int stw_words;            // 32-bit words per tile row of the SAT-tile bitmap
  int use_cbits;            // IDDM mask also emitted as bits by k_pyramid4 (grid 0)
  int cbits_words;          // 32-bit words per cell row of the bit mask
  // IDDM state: octave levels kept for the next frame
  long long state_off[VF_MAXO]; long long state_slab;
  int kp_cap;           // feature capacity per stream and buffer
  // temporal baseline (mask_mode 3, temporal.py:23-43): GOP and search set-up
  int gop_delta, gop_patch, bm_nc, bm_nf, bm_rc, bm_rf, bm_dyadic;
  double gop_t_bm, gop_t_et;
  int prop_chunks;      // CTAs reserved for propagation chunks
  int sat_tiles;        // stx * sty
  unsigned sth_magic;   // ceil(2^32 / VF_ST): y / VF_ST == umulhi(y, sth_magic) for y < 2^16
  int nms_raw;          // stand-alone nms_and_refine: no border / merge filter
  int pyr_split;        // masked frames build the intra-octave chain only near active cells (k_pyramid4)
  int pyr_halo;         // o0 pixels a FAST ring reaches around a tile's derived pixels
  int nms_wrap;         // stand-alone: numpy negative-index wrap in the 3x3 test
  int nms_chunks;       // NMS candidate chunks per stream: kp_cap / NMS_CHUNK_THREADS
};

// Per-launch stream-batch pointers.
struct Bufs {
  int s0;               // first stream of this launch (stream groups run on separate CUDA streams)
  const uint8_t* frames; long long frame_stride; long long frame_pitch; // o0 of stream s (relative to s0)
  uint8_t* layers;      // [S][layer_slab]
  uint8_t* scores;      // [S][sm_slab]
  uint32_t* bitmaps;    // [S][bm_slab_words]
  int* tile_stamp;      // [S][tiles_per_stream]
  int* band_stamp;      // [S][bands_per_stream]
  int nms_u;            // NMS units per band (1, 2, 4 or 8): a unit is VF_TILE_H / nms_u rows
  int* unit_rec;        // [S][bands_per_stream * nms_u][4]: staging base, kept, border-ok, dropped per NMS unit
  int* unit_out;        // [S][bands_per_stream * nms_u]: output offset of the unit's kept keypoints
  int* band_cand;       // [S][bands_per_stream]: FAST candidates of the band this step
  int* gidx;            // [S][kp_cap] describe list: candidate indices of the kept keypoints (k_nms_test)
  int desc_bin;         // 1: pipeline NMS (k_nms_list / k_nms_test, describe list); 0: stand-alone k_nms
  uint32_t* cand;       // [S][kp_cap] NMS candidates (layer << 26 | y << 13 | x) in (layer, y, x) order
  int* cand_rank;       // [S][kp_cap] kept candidate's rank within its NMS chunk
  int* chunk_off;       // [S][nms_chunks] kept count of each chunk (k_nms_test), then its output offset
  int* nms_cnt;         // [S][4] survivors inside / outside the border margin (FrameReport)
  int nms_pre;          // k_fast drops candidates that fail the strict 3x3 test inside their tile (VF_NMS_PRE=0: off)
  int orient_seq;       // k_desc_fused: always take the sequential-sum orientation (test hook, VF_ORIENT_SEQ=1)
  int sat_early;        // 1: k_fast marks the SAT tiles (candidate footprint bounds) and k_sat runs beside the NMS
  int sat_check;        // VF_SAT_CHECK=1: k_nms_test asserts every kept footprint tile was marked (VF_ERRBIT_SATMARK)
  int* prop_cnt;        // [S][prop_chunks]
  int* prop_out;        // [S][prop_chunks]
  uint8_t* cells;       // [S][cell_slab]
  int* cell_row_stamp;  // [S][n_grids][max rows] "row has an active cell" stamps
  uint8_t* state;       // [S][state_slab]
  const int* lut;       // [lut_len] row/col -> cell maps (shared by all streams)
  uint32_t* sat;        // [max_streams][W*H] strip SATs
  uint32_t* rowsum;     // [S][H][stx] row sums of o0 per SAT-tile column
  uint32_t* carry;      // [S][H][stx] strip carries K(y, tx) (see strip_carries)
  uint32_t* cbits;      // [S][2 (epoch parity)][rows][cbits_words] IDDM cells as bits
  unsigned* sat_bits;   // [S][sty][stw_words] SAT tiles marked this step (cleared by k_pyramid)
  int* sat_work; int* sat_count;   // [S][sat_tiles] / [S]: SAT tiles marked this step (masked frames)
  double* st_x; double* st_y; double* st_s; double* st_v;   // staging [S][kp_cap]
  const double* bm_coarse; const double* bm_fine;         // spiral offsets (x, y) pairs (temporal mode)
  uint8_t* prev_frame;     // [S][H][W] previous frame (temporal mode)
  uint8_t* bm_found;       // [S][kp_cap] block-match result flags
  int* bm_chunk;           // [S][prop_chunks] found counts per 1024-feature chunk
  // double-buffered features [S][2][kp_cap]
  double* fx; double* fy; double* fs; double* ft; double* fv;
  uint8_t* forg; int* fage; uint8_t* fdesc;  // desc: [S][2][kp_cap][64]
  int* ctr;             // [S][C_NCTR]
  unsigned long long* cov;  // [S] covered full-res pixels of this frame
  double* report;       // [S][8]: n_det, n_prop, n_total, n_dropped, coverage, frame, n_surv, n_cand
  int* worklist; int* work_count;  // [S][tiles_per_stream] / [S]: active FAST tiles per stream
  double* hist; int hist_frames;  // optional [S][hist_frames][8]: report rows of every frame (vf_set_history)
  uint32_t* keep_bits;  // optional [S][keep_words]: Eq. 1 keep mask of the previous list (delta collect)
  int keep_words;
};

// --------------------------------------------------------------------------
// small helpers
// --------------------------------------------------------------------------
// Per-stream monotonic step id: activity stamps compare against it, so nothing
// has to be cleared between steps (or across vf_reset).
__device__ __forceinline__ int stream_epoch(const Bufs& b, int s) { return b.ctr[s * C_NCTR + C_EPOCH] + 1; }

__device__ __forceinline__ const uint8_t* layer_ptr(const Geo& g, const Bufs& b, int s, int l, int& pitch)
{
  if (l == 0) { pitch = (int)b.frame_pitch; return b.frames + (long long)(s - b.s0) * b.frame_stride; }
  pitch = g.L[l].pitch;
  return b.layers + (long long)s * g.layer_slab + g.L[l].layer_off;
}

// IDDM state of octave level lv: the source octave of frame f is kept at
// parity f & 1 (prev = 1 reads the previous frame's, parity (f & 1) ^ 1), so a
// step can be replayed (capacity retry) without losing the previous octave.
__device__ __forceinline__ uint8_t* iddm_state(const Geo& g, const Bufs& b, int s, int lv, int prev)
{
  const int par = (b.ctr[s * C_NCTR + C_FRAME] & 1) ^ prev;
  return b.state + ((long long)s * 2 + par) * g.state_slab + g.state_off[lv];
}

// Grid used to gate layer l (per_layer: its octave level's grid, else grid 0).
__device__ __forceinline__ int grid_of_layer(const Geo& g, int l) { return g.per_layer ? (l >> 1) : 0; }

// Gate of layer pixel (y, x): the full-res mask sampled by floor mapping
// (detector.py:175-181) of the block-replicated cell mask (masking.py:139-148).
__device__ __forceinline__ int gate_at(const Geo& g, const Bufs& b, int s, int l, int y, int x)
{
  const int gi = grid_of_layer(g, l);
  const int* lut = b.lut + g.L[l].rc_off;      // rows then cols
  int r = __ldg(lut + y);
  int c = __ldg(lut + g.L[l].h + x);
  const GridGeo& G = g.grid[gi];
  return b.cells[(long long)s * g.cell_slab + G.cell_off + (long long)r * G.cols + c];
}

// Merge-mask bit at full-res position (masking.py:151-165); per_layer uses the
// union of the level masks (pipeline.py:196-199).
__device__ __forceinline__ int merge_mask_at(const Geo& g, const Bufs& b, int s, double x, double y)
{
  // clamp in fp64 first (same result as clamping the rounded integer), then
  // 32-bit integer cell arithmetic
  double xr = floor(x + 0.5), yr = floor(y + 0.5);
  xr = xr < 0.0 ? 0.0 : (xr > (double)(g.W - 1) ? (double)(g.W - 1) : xr);
  yr = yr < 0.0 ? 0.0 : (yr > (double)(g.H - 1) ? (double)(g.H - 1) : yr);
  const int xi = (int)xr, yi = (int)yr;
  const uint8_t* cells = b.cells + (long long)s * g.cell_slab;
  int v = 0;
  for (int k = 0; k < g.n_grids; k++) {
    const GridGeo& G = g.grid[k];
    v |= cells[G.cell_off + (yi / G.ch) * G.cols + xi / G.cw];
  }
  return v;
}

// Feature lists are stored at the END of their buffer: buffer `buf` of stream s
// holding n features uses slots [kp_cap - n, kp_cap), detected first, then
// propagated.  Propagated features (slots >= kp_cap - n_prop) can then be
// written before the detected count is known.
__device__ __forceinline__ long long feat_base(const Geo& g, int s, int buf, int n)
{
  return ((long long)s * 2 + buf) * g.kp_cap + (g.kp_cap - n);
}

__device__ __forceinline__ int use_mask(const Geo& g, const Bufs& b, int s)
{
  // pipeline.py:234; temporal mode detects without a mask at GOP starts (temporal.py:287-288)
  return g.mask_mode != 0 && g.mask_mode != 3 && b.ctr[s * C_NCTR + C_FRAME] > 0;
}

__device__ __forceinline__ int warp_excl_scan(int v, int lane, int& total)
{
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  total = __shfl_sync(0xffffffffu, x, 31);
  return x - v;
}

template <typename T>
__device__ __forceinline__ T block_excl_scan(T v, T* sm_warp, T& total)
{
  // blockDim.x multiple of 32, <= 1024
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  T x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sm_warp[wid] = x;
  __syncthreads();
  if (wid == 0) {
    T w = lane < nw ? sm_warp[lane] : T(0);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      T y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < nw) sm_warp[lane] = w;
  }
  __syncthreads();
  T base = wid > 0 ? sm_warp[wid - 1] : T(0);
  total = sm_warp[nw - 1];
  __syncthreads();
  return base + x - v;
}
