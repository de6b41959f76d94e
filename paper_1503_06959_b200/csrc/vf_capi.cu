// vf_capi.cu -- C ABI (include/vidfeat_b200.h): contexts, HBM layout, launches.
//
// Single translation unit: includes the kernels.  Built by
// paper_1503_06959_b200/build.py (nvcc -gencode arch=compute_100a,code=sm_100a).
#include "vf_kernels.cu"
#include "vf_temporal.cuh"
#include "../../include/vidfeat_b200.h"

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <algorithm>
#include <climits>
#include <type_traits>

#define VF_VERSION "vidfeat-b200 0.1.0 (sm_100a)"
#ifdef VF_DEBUG
#define DBG_SYNC(st, name) do { (void)(st); cudaError_t e_ = cudaDeviceSynchronize(); if (e_ != cudaSuccess) fprintf(stderr, "vidfeat_b200 debug: %s after %s\n", cudaGetErrorString(e_), name); } while (0)
#else
#define DBG_SYNC(st, name) do { } while (0)
#endif

namespace {

int g_pattern_ok = 0;

struct Alloc {
  std::vector<void*> ptrs;
  cudaError_t err = cudaSuccess;
  template <typename T>
  T* get(size_t n) {
    void* p = nullptr;
    if (n == 0) n = 1;
    cudaError_t e = cudaMalloc(&p, n * sizeof(T));
    if (e != cudaSuccess) { err = e; return nullptr; }
    cudaMemset(p, 0, n * sizeof(T));
    ptrs.push_back(p);
    return static_cast<T*>(p);
  }
  void release() {
    for (void* p : ptrs) cudaFree(p);
    ptrs.clear();
  }
  void drop(void* p) {   // free one allocation made by get()
    for (auto& q : ptrs)
      if (q == p) { cudaFree(p); q = ptrs.back(); ptrs.pop_back(); return; }
  }
};

inline long long align_up(long long v, long long a) { return (v + a - 1) / a * a; }
inline int cdiv(long long a, long long b) { return (int)((a + b - 1) / b); }

// pyramid.py:97-125 geometry (+ validation in the reference's order)
int layer_dims(int W, int H, int O, int* ws, int* hs, double* scales)
{
  if (O < 1) return VF_ERR_OCTAVES;
  if (O > VF_MAXO) return VF_ERR_ARG;
  int need = 1 << (O - 1);
  if (W < need || H < need) return VF_ERR_FRAME_SMALL;
  int ow = W, oh = H, iw = (2 * W) / 3, ih = (2 * H) / 3;
  if (iw < 1 || ih < 1) return VF_ERR_UNDERFLOW;
  for (int o = 0; o < O; o++) {
    if (o > 0) {
      ow /= 2; oh /= 2; iw /= 2; ih /= 2;
      if (ow < 1 || oh < 1 || iw < 1 || ih < 1) return VF_ERR_UNDERFLOW;
    }
    ws[2 * o] = ow; hs[2 * o] = oh; ws[2 * o + 1] = iw; hs[2 * o + 1] = ih;
    double sc = ldexp(1.0, -o);
    scales[2 * o] = sc;
    scales[2 * o + 1] = sc / 1.5;
  }
  return VF_OK;
}

// GopConfig (temporal.py:23-43): all gop_* fields zero = the defaults;
// otherwise validated in the reference's order.
struct Gop { int delta, patch; double t_bm, t_et, cw, cs, fw, fs; };
int gop_from_config(const vf_config& c, Gop& o)
{
  const bool zero = !c.gop_delta && !c.gop_patch && c.gop_t_bm == 0.0 && c.gop_t_et == 0.0 &&
                    c.gop_coarse_window == 0.0 && c.gop_coarse_step == 0.0 && c.gop_fine_window == 0.0 &&
                    c.gop_fine_step == 0.0;
  if (zero) { o = Gop{10, 16, 1800.0, 1000.0, 12.0, 2.0, 1.75, 0.25}; return VF_OK; }
  o = Gop{c.gop_delta, c.gop_patch, c.gop_t_bm, c.gop_t_et, c.gop_coarse_window, c.gop_coarse_step,
          c.gop_fine_window, c.gop_fine_step};
  if (o.delta < 1) return VF_ERR_GOP_DELTA;
  if (o.patch % 2 != 0 || o.patch < 2) return VF_ERR_GOP_PATCH;
  if (o.fs > o.cs) return VF_ERR_GOP_STEP;
  if (o.t_bm <= 0 || o.t_et <= 0) return VF_ERR_GOP_SAD;
  if (!(o.cs > 0) || !(o.fs > 0) || o.cw < 0 || o.fw < 0 || o.cw / o.cs > 4096 || o.fw / o.fs > 4096) return VF_ERR_ARG;
  return VF_OK;
}

// Spiral offsets + search set-up of a GopConfig; offsets stay on the host in co / fi.
void gop_setup(const Gop& o, vft::Setup& q, std::vector<double>& co, std::vector<double>& fi)
{
  co = vft::spiral_offsets(o.cw, o.cs);
  fi = vft::spiral_offsets(o.fw, o.fs);
  fi.erase(fi.begin(), fi.begin() + 2);             // skip (0, 0) (temporal.py:216)
  q.P = o.patch; q.nc = (int)co.size() / 2; q.nf = (int)fi.size() / 2;
  q.t_bm = o.t_bm; q.t_et = o.t_et;
  double mc = 0, mf = 0;
  bool dy = true;
  for (double v : co) { mc = std::max(mc, std::fabs(v)); dy = dy && v == std::floor(v); }
  for (double v : fi) { mf = std::max(mf, std::fabs(v)); dy = dy && v * 4.0 == std::floor(v * 4.0); }
  q.rc = (int)std::ceil(mc);
  q.rfc = std::max(1, (int)std::ceil(mf));
  q.dyadic = dy && o.patch * o.patch * 255LL * 16 < (1LL << 24);
  const int M = q.rc + q.rfc + 1;
  (void)M;
  q.shmask = 1;                                      // window only (shifted copies measured slower)
  vft::layout(q);
}

// Fill Geo for a frame size and config.  lut is filled on the host.
int make_geo(const vf_config& c, Geo& g, std::vector<int>& lut)
{
  memset(&g, 0, sizeof(g));
  if (c.threshold < 1) return VF_ERR_THRESHOLD;
  if (c.mask_mode < 0 || c.mask_mode > 3) return VF_ERR_MODE;
  if (c.t_h < 0) return VF_ERR_T_H;
  if (c.grid_rows < 1 || c.grid_cols < 1) return VF_ERR_GRID;
  int ws[VF_MAXL], hs[VF_MAXL];
  double sc[VF_MAXL];
  int rc = layer_dims(c.width, c.height, c.n_octaves, ws, hs, sc);
  if (rc) return rc;
  if (c.width > 8192) return VF_ERR_ARG;   // NMS candidate encoding: x < 2^13
  g.W = c.width; g.H = c.height; g.O = c.n_octaves; g.NL = 2 * c.n_octaves;
  g.threshold = c.threshold;
  g.mask_mode = c.mask_mode;
  g.per_layer = c.mask_mode == 1 ? c.per_layer : 0;
  if (c.mask_mode == 3) {
    Gop o;
    const int grc = gop_from_config(c, o);
    if (grc) return grc;
    g.gop_delta = o.delta; g.gop_patch = o.patch; g.gop_t_bm = o.t_bm; g.gop_t_et = o.t_et;
  }
  g.mask_level = c.octave_for_mask < 0 ? g.O - 1 : c.octave_for_mask;
  if (c.mask_mode == 1 && (g.mask_level < 0 || g.mask_level >= g.O)) return VF_ERR_OCTAVE_KEY;
  g.t_i = c.t_i; g.t_h = c.t_h;
  long long lay = 0, smo = 0, bmo = 0;
  int tb = 0, bb = 0, rb = 0;
  for (int l = 0; l < g.NL; l++) {
    LayerGeo& L = g.L[l];
    L.w = ws[l]; L.h = hs[l];
    L.pitch = (int)align_up(L.w, 16);
    L.scale = sc[l];
    L.sigma = 1.0 / sc[l];
    L.rinv_h = 1.0 / L.h; L.rinv_w = 1.0 / L.w;
    L.tiles_x = cdiv(L.w, VF_TILE_W); L.tiles_y = cdiv(L.h, VF_TILE_H);
    L.tile_base = tb; tb += L.tiles_x * L.tiles_y;
    L.band_base = bb; bb += L.tiles_y;
    L.row_base = rb; rb += L.h;
    L.bm_words = cdiv(L.w, 32);
    if (l >= 1) { L.layer_off = lay; lay += align_up((long long)L.pitch * L.h, 256); }
    L.sm_off = smo; smo += align_up((long long)L.pitch * L.h + 16, 256);
    L.bm_off = bmo; bmo += align_up((long long)L.bm_words * L.h, 64);
  }
  // Early SAT marks (k_fast): bound of the descriptor footprint of any keypoint
  // the NMS can keep from a candidate of layer l.  The refined sigma lies
  // between the layer's and a neighbour's (|delta| < 1, detector.py:287-297;
  // layers 0 and NL - 1 keep theirs); the refined position is within one layer
  // pixel of the candidate (|ox|, |oy| < 1, detector.py:207-228); + 3 covers
  // the float candidate position (< 1 px) and the (int) truncations.
  for (int l = 0; l < g.NL; l++) {
    const double sg = (l >= 1 && l + 1 < g.NL) ? std::max(g.L[l].sigma, g.L[l + 1].sigma) : g.L[l].sigma;
    g.L[l].sat_reach = (int)ceil(12.5 * sg) + 2 + (int)ceil(1.0 / g.L[l].scale) + 3;
    g.L[l].inv_scale = (float)(1.0 / g.L[l].scale);
  }
  g.tiles_per_stream = tb; g.bands_per_stream = bb; g.rows_per_stream = rb;
  g.layer_slab = std::max(lay, 256LL); g.sm_slab = smo; g.bm_slab_words = bmo;
  // mask grids (masking.py:139-148 cell geometry; binning masking.py:132-136)
  long long co = 0;
  if (g.mask_mode == 1) {
    int lv0 = g.per_layer ? 0 : g.mask_level, lv1 = g.per_layer ? g.O - 1 : g.mask_level;
    for (int lv = lv0; lv <= lv1; lv++) {
      GridGeo& G = g.grid[g.n_grids++];
      G.rows = hs[2 * lv]; G.cols = ws[2 * lv];
      G.cw = cdiv(g.W, G.cols); G.ch = cdiv(g.H, G.rows);
      G.cell_off = co; co += align_up((long long)G.rows * G.cols + 4, 64);
    }
  } else if (g.mask_mode == 2) {
    GridGeo& G = g.grid[g.n_grids++];
    G.rows = c.grid_rows; G.cols = c.grid_cols;
    G.cw = cdiv(g.W, G.cols); G.ch = cdiv(g.H, G.rows);
    G.cell_off = co; co += align_up((long long)G.rows * G.cols + 4, 64);
    if ((long long)G.rows * G.cols * 4 > 200 * 1024) return VF_ERR_GRID;
  }
  g.cell_slab = std::max(co, 64LL);
  // row/col -> cell LUTs per layer (detector.py:175-181 floor mapping, then // cell)
  lut.clear();
  for (int l = 0; l < g.NL; l++) {
    LayerGeo& L = g.L[l];
    L.rc_off = (int)lut.size();
    L.cc_off = L.rc_off + L.h;
    if (g.n_grids == 0) { lut.resize(lut.size() + L.h + L.w, 0); continue; }
    const GridGeo& G = g.grid[g.per_layer ? (l >> 1) : 0];
    for (int y = 0; y < L.h; y++) lut.push_back((int)(((long long)y * g.H / L.h) / G.ch));
    for (int x = 0; x < L.w; x++) lut.push_back((int)(((long long)x * g.W / L.w) / G.cw));
  }
  g.lut_len = (long long)lut.size();
  // IDDM state (previous frame's mask-source octave levels)
  long long so = 0;
  if (g.mask_mode == 1) {
    int lv0 = g.per_layer ? 0 : g.mask_level, lv1 = g.per_layer ? g.O - 1 : g.mask_level;
    for (int lv = lv0; lv <= lv1; lv++) { g.state_off[lv] = so; so += align_up((long long)ws[2 * lv] * hs[2 * lv], 64); }
  }
  g.state_slab = std::max(so, 64LL);
  // pyramid / SAT tiles: multiples of 3 * 2^(O-1)
  const int unit = 3 << (g.O - 1);
  g.ptw = unit * std::max(1, 96 / unit);
  g.pth = unit * std::max(1, 48 / unit);
  g.ptx = cdiv(g.W, g.ptw); g.pty = cdiv(g.H, g.pth);
  // strip-SAT tiles, independent of the pyramid tiles (ptw is a multiple of VF_ST)
  g.stx = cdiv(g.W, VF_ST); g.sty = cdiv(g.H, VF_ST);
  g.sat_tiles = g.stx * g.sty;
  g.stw_words = cdiv(g.stx, 32);
  g.sth_magic = (unsigned)((0x100000000ULL + VF_ST - 1) / VF_ST);
  // bit-packed IDDM mask from k_pyramid4 (its geometry, default mask source)
  g.use_cbits = g.mask_mode == 1 && !g.per_layer && g.mask_level == 3 && g.O == 4 && g.ptw == 96 && g.pth == 48;
  g.cbits_words = g.use_cbits ? cdiv(g.grid[0].cols, 32) : 0;
  // the warp-strip pyramid (k_pyr_o + k_pyr_i) for O = 4; VF_PYR_SPLIT=0 keeps the smem-tile k_pyramid4
  g.pyr_split = g.O == 4 && (g.mask_mode != 1 || g.use_cbits) &&
                !(getenv("VF_PYR_SPLIT") && atoi(getenv("VF_PYR_SPLIT")) == 0);
  g.pyr_halo = 4 * std::max(cdiv(g.W, g.L[g.NL - 1].w), cdiv(g.H, g.L[g.NL - 1].h)) + 2;
  if (g.ptw % VF_ST) return VF_ERR_ARG;
  long long cap = c.kp_capacity > 0 ? c.kp_capacity : std::max(65536LL, (long long)g.W * g.H / 8);
  g.kp_cap = (int)std::min(cap, 1LL << 28);
  g.prop_chunks = cdiv(g.kp_cap, 1024);
  g.nms_chunks = cdiv(g.kp_cap, 1 << NMS_CHUNK_LOG);
  if (g.W > 8192 || g.H > 8192 || g.NL > 16) return VF_ERR_ARG;   // NMS candidate code: layer << 26 | y << 13 | x
  return VF_OK;
}

int pyramid_smem(const Geo& g)
{
  int acc = 0;
  for (int l = 0; l < g.NL; l++) {
    int lw, lh, o = l >> 1;
    if (l & 1) { lw = (2 * g.ptw / 3) >> o; lh = (2 * g.pth / 3) >> o; }
    else { lw = g.ptw >> o; lh = g.pth >> o; }
    acc += (lw * lh + 15) & ~15;
  }
  return acc + g.pth * (g.ptw / VF_ST) * 4;   // + row-sum accumulators per SAT column
}

int g_num_sms = 0;

int cuda_status(cudaError_t e)
{
  if (e == cudaSuccess) return VF_OK;
  fprintf(stderr, "vidfeat_b200: CUDA error %s\n", cudaGetErrorString(e));
  return VF_ERR_CUDA;
}

}  // namespace

// Steps the pipelined API keeps in flight (vf_pipeline_submit before a collect
// is due): with 3, the upload of step n + 2 is queued while step n + 1 computes
// and step n's result is copied out, so the slowest of the three sets the pace.
#define VF_PIPE_DEPTH 3

struct vf_ctx {
  vf_config cfg;
  Geo g;
  Bufs b;
  Alloc mem;
  int S;
  std::vector<long long> frames_done;   // host mirror of per-stream frame counters
  int pyr_smem;
  int fast_grid;
  int desc_grid;
  int sat_grid, sat_smem, desc_smem, dfused_grid, nmst_grid;
  vft::Setup bmq{};                     // temporal mode: block-match set-up (device offsets)
  int bm_grid = 0, bm_smem = 0;
  // host-input staging (vf_process_host)
  uint8_t* hstage[2] = {nullptr, nullptr};
  long long hstage_bytes = 0;
  int hstage_k = 0;
  cudaEvent_t hstage_free[2] = {nullptr, nullptr};
  // packed feature output (vf_fetch_features): device SoA + host-visible prefix
  struct Pack {
    double *x = nullptr, *y, *s, *t, *v;
    uint8_t *o, *d;
    int* a;
    int* pre = nullptr;        // device [S + 1]
    int* pre_host = nullptr;   // pinned [S + 1]
    long long cap = 0;
  } pack;
  // pipelined host API (vf_pipeline_submit / vf_pipeline_collect)
  struct Pipe {
    bool init = false;
    cudaStream_t h2d = nullptr, comp = nullptr, d2h = nullptr;
    uint8_t* frames[VF_PIPE_DEPTH] = {};
    long long frame_bytes = 0;
    double *x[VF_PIPE_DEPTH], *y[VF_PIPE_DEPTH], *s[VF_PIPE_DEPTH], *t[VF_PIPE_DEPTH], *v[VF_PIPE_DEPTH];
    uint8_t *o[VF_PIPE_DEPTH], *d[VF_PIPE_DEPTH];
    int* a[VF_PIPE_DEPTH];
    int* pre[VF_PIPE_DEPTH];
    int* pre_host[VF_PIPE_DEPTH];
    int* meta[VF_PIPE_DEPTH] = {};        // device blob: pre | kpre | cnt | err (pointers below point into it)
    int* meta_host[VF_PIPE_DEPTH] = {};   // pinned copy, one D2H per step
    int* err[VF_PIPE_DEPTH] = {};
    int* err_host[VF_PIPE_DEPTH] = {};    // sticky capacity flags of each stream after the step
    size_t meta_ints = 0;
    long long cap = 0;
    cudaEvent_t ev_h2d[VF_PIPE_DEPTH], ev_comp[VF_PIPE_DEPTH], ev_pre[VF_PIPE_DEPTH], ev_d2h[VF_PIPE_DEPTH];
    long long submitted = 0, collected = 0;
    int n_streams[VF_PIPE_DEPTH];
    // delta results (vf_pipeline_set_delta): keep masks of the previous lists
    bool delta = false;
    uint32_t* kb[VF_PIPE_DEPTH] = {};
    int* kpre[VF_PIPE_DEPTH] = {};
    int* kpre_host[VF_PIPE_DEPTH] = {};
    int* cnt[VF_PIPE_DEPTH] = {};
    int* cnt_host[VF_PIPE_DEPTH] = {};
    long long kcap = 0;
  } pipe;
  // live per-stage timing (vf_set_timing): one event before each stage + end
  int timing = 0;
  std::vector<cudaEvent_t> ev_pool, ev_used;
  std::vector<int> ev_stage;   // stage index of each recorded interval start
  std::vector<int> ev_group;   // stream group of each mark
  // side-stream kernel intervals (k_propagate): (stage, start, end) on the aux stream
  std::vector<int> side_stage;
  std::vector<cudaEvent_t> side_ev;
  int cur_group = 0;
  // stream groups: independent stream ranges launched on their own CUDA streams
  int n_groups_max = 0;
  // side stream per launch group: the worklist's carries / propagation counts
  // run concurrently with k_fast and join before k_nms
  std::vector<cudaStream_t> aux;
  std::vector<cudaEvent_t> aux_in, aux_mid, aux_out;
  std::vector<cudaStream_t> gstreams;
  std::vector<cudaEvent_t> gjoin;
  cudaEvent_t gfork = nullptr;
  cudaStream_t hp = nullptr;
  cudaEvent_t hp_in = nullptr, hp_out = nullptr;
  std::vector<cudaStream_t> dstreams;
  std::vector<cudaEvent_t> djoin;
  std::vector<cudaEvent_t> dfork_g;     // per stream group
  std::vector<cudaEvent_t> dsat_e;      // per describe stream: its k_sat done (VF_DESC_STAGGER)
  std::vector<cudaEvent_t> dfast_e, dsatall_e;   // per group: k_fast done / the early k_sat done (sat_early)
  std::vector<cudaStream_t> sat_s;               // per group: lowest-priority stream of the early k_sat (VF_SAT_LOW=1)
  std::vector<cudaStream_t> pyi_s;      // per stream group: k_pyr_i beside the main work list
  std::vector<cudaEvent_t> pyi_e;
  // CUDA graph of one step (small batches): the step's launches (all its
  // streams) captured once per batch size and replayed; inputs are copied
  // into a context-owned buffer first so the graph's pointers stay fixed
#ifdef VF_DEBUG
  int graphs = 0;                       // debug builds synchronize after every launch: no capture
#else
  int graphs = 1;                       // vf_set_graphs
#endif
  cudaGraphExec_t gexec = nullptr;
  cudaGraph_t graph = nullptr;          // kept alive: its kernel nodes own the captured argument storage
  std::vector<cudaGraphNode_t> gnodes;  // kernel nodes of the step graph (Bufs is argument 1 of each)
  std::vector<Bufs> gbufs;              // their captured Bufs (frames re-pointed per step)
  const uint8_t* g_frames = nullptr;    // frames / stride of the capture
  long long g_stride = 0;
  int g_n = 0;
  int eager_n = 0;                      // batch size of the last eager step (streams / events exist)
  bool capturing = false;
  cudaStream_t cap = nullptr;           // capture stream
};

static void pack_free(vf_ctx* c)
{
  auto& P = c->pack;
  for (void* p : {(void*)P.x, (void*)P.y, (void*)P.s, (void*)P.t, (void*)P.v, (void*)P.o, (void*)P.d, (void*)P.a})
    if (p) cudaFree(p);
  P.x = P.y = P.s = P.t = P.v = nullptr;
  P.o = P.d = nullptr;
  P.a = nullptr;
  P.cap = 0;
}

#define VF_NSTAGES 9   // binmask, pyramid, worklist, fast, nms, sat, describe, propagate, finalize
static cudaEvent_t pool_event(vf_ctx* c)
{
  cudaEvent_t e;
  if (c->ev_pool.empty()) cudaEventCreate(&e);
  else { e = c->ev_pool.back(); c->ev_pool.pop_back(); }
  return e;
}

static void stage_mark(vf_ctx* c, int stage, cudaStream_t st)
{
  if (!c->timing) return;
  cudaEvent_t e = pool_event(c);
  cudaEventRecord(e, st);
  c->ev_used.push_back(e);
  c->ev_stage.push_back(stage);
  c->ev_group.push_back(c->cur_group);
}

extern "C" {

const char* vf_version(void) { return VF_VERSION; }

const char* vf_strerror(int code)
{
  switch (code) {
    case VF_OK: return "ok";
    case VF_ERR_THRESHOLD: return "detection threshold must be >= 1";
    case VF_ERR_OCTAVES: return "n_octaves must be >= 1";
    case VF_ERR_FRAME_SMALL: return "frame too small for the requested octaves";
    case VF_ERR_UNDERFLOW: return "dimension underflow while building the pyramid";
    case VF_ERR_MODE: return "unknown mask mode";
    case VF_ERR_T_H: return "histogram threshold must be >= 0";
    case VF_ERR_GRID: return "binning grid must be at least 1x1";
    case VF_ERR_EMPTY: return "empty frame sequence";
    case VF_ERR_CAPACITY: return "keypoint capacity exceeded";
    case VF_ERR_CUDA: return "CUDA runtime error";
    case VF_ERR_ARG: return "invalid argument";
    case VF_ERR_INDEX: return "index out of bounds";
    case VF_ERR_OCTAVE_KEY: return "no octave layer at octave_for_mask";
    case VF_ERR_PATTERN: return "sampling pattern not set or malformed";
    case VF_ERR_MATCH_CAPACITY: return "match buffer capacity exceeded";
    case VF_ERR_GOP_DELTA: return "GOP length must be >= 1";
    case VF_ERR_GOP_PATCH: return "patch side must be even and positive";
    case VF_ERR_GOP_STEP: return "fine_step must not exceed coarse_step";
    case VF_ERR_GOP_SAD: return "SAD thresholds must be positive";
    default: return "unknown error";
  }
}

int vf_set_pattern(const double* points, const double* radii, int m, const int32_t* short_pairs, int nbits,
                   const int32_t* long_pairs, int L)
{
  if (m != VF_NPTS || nbits != VF_NBITS || L < 1 || L > VF_MAXLONG) return VF_ERR_PATTERN;
  double px[VF_NPTS], py[VF_NPTS];
  short si[VF_NBITS], sj[VF_NBITS], li[VF_MAXLONG], lj[VF_MAXLONG];
  double wx[VF_MAXLONG], wy[VF_MAXLONG];
  for (int j = 0; j < m; j++) { px[j] = points[2 * j]; py[j] = points[2 * j + 1]; }
  for (int k = 0; k < nbits; k++) {
    if (short_pairs[2 * k] < 0 || short_pairs[2 * k] >= m || short_pairs[2 * k + 1] < 0 || short_pairs[2 * k + 1] >= m)
      return VF_ERR_PATTERN;
    si[k] = (short)short_pairs[2 * k]; sj[k] = (short)short_pairs[2 * k + 1];
  }
  for (int p = 0; p < L; p++) {
    int a = long_pairs[2 * p], c = long_pairs[2 * p + 1];
    if (a < 0 || a >= m || c < 0 || c >= m) return VF_ERR_PATTERN;
    li[p] = (short)a; lj[p] = (short)c;
    // descriptor.py:169-177 _pair_arrays: dp * (1 / |dp|^2), evaluated as numpy does
    double dx = points[2 * a] - points[2 * c], dy = points[2 * a + 1] - points[2 * c + 1];
    volatile double d2 = dx * dx;
    d2 = d2 + dy * dy;
    double inv = 1.0 / d2;
    wx[p] = dx * inv; wy[p] = dy * inv;
  }
  cudaError_t e = cudaSuccess;
  e = e ? e : cudaMemcpyToSymbol(c_px, px, sizeof(px));
  e = e ? e : cudaMemcpyToSymbol(c_py, py, sizeof(py));
  e = e ? e : cudaMemcpyToSymbol(c_rad, radii, sizeof(double) * m);
  e = e ? e : cudaMemcpyToSymbol(c_si, si, sizeof(si));
  e = e ? e : cudaMemcpyToSymbol(c_sj, sj, sizeof(sj));
  e = e ? e : cudaMemcpyToSymbol(c_li, li, sizeof(short) * L);
  e = e ? e : cudaMemcpyToSymbol(c_lj, lj, sizeof(short) * L);
  e = e ? e : cudaMemcpyToSymbol(c_wx, wx, sizeof(double) * L);
  e = e ? e : cudaMemcpyToSymbol(c_wy, wy, sizeof(double) * L);
  e = e ? e : cudaMemcpyToSymbol(c_nlong, &L, sizeof(int));
  uint32_t pairs[VF_NBITS];
  double ptab[64][3];
  for (int k = 0; k < nbits; k++) pairs[k] = (uint32_t)(uint16_t)si[k] | ((uint32_t)(uint16_t)sj[k] << 16);
  for (int j = 0; j < 64; j++) {
    const int jj = j < m ? j : 0;
    ptab[j][0] = px[jj]; ptab[j][1] = py[jj]; ptab[j][2] = radii[jj];
  }
  e = e ? e : cudaMemcpyToSymbol(g_pairs, pairs, sizeof(pairs));
  uint32_t lpair[VF_MAXLONG];
  double2 lw[VF_MAXLONG];
  for (int p = 0; p < L; p++) {
    lpair[p] = (uint32_t)(uint16_t)li[p] | ((uint32_t)(uint16_t)lj[p] << 16);
    lw[p] = make_double2(wx[p], wy[p]);
  }
  // orientation as a linear form of the 60 box means (k_desc_fused, dr_orient_lin)
  double ow[64][4] = {};
  for (int p = 0; p < L; p++) {
    ow[li[p]][0] += wx[p]; ow[lj[p]][0] -= wx[p];
    ow[li[p]][1] += wy[p]; ow[lj[p]][1] -= wy[p];
    ow[li[p]][2] += std::fabs(wx[p]); ow[lj[p]][2] += std::fabs(wx[p]);
    ow[li[p]][3] += std::fabs(wy[p]); ow[lj[p]][3] += std::fabs(wy[p]);
  }
  const double ogam = 2.0 * (L + 80) * 1.1102230246251565e-16;
  e = e ? e : cudaMemcpyToSymbol(g_ow, ow, sizeof(ow));
  e = e ? e : cudaMemcpyToSymbol(c_ogam, &ogam, sizeof(double));
  e = e ? e : cudaMemcpyToSymbol(g_lpair, lpair, sizeof(uint32_t) * L);
  e = e ? e : cudaMemcpyToSymbol(g_lw, lw, sizeof(double2) * L);
  e = e ? e : cudaMemcpyToSymbol(g_ptab, ptab, sizeof(ptab));
  if (e != cudaSuccess) return cuda_status(e);
  g_pattern_ok = 1;
  return VF_OK;
}

int vf_create(const vf_config* cfg, vf_ctx** out)
{
  if (!cfg || !out) return VF_ERR_ARG;
  *out = nullptr;
  if (cfg->max_streams < 1) return VF_ERR_ARG;
  vf_ctx* c = new vf_ctx();
  c->cfg = *cfg;
  std::vector<int> lut;
  int rc = make_geo(*cfg, c->g, lut);
  if (rc) { delete c; return rc; }
  const Geo& g = c->g;
  const int S = c->S = cfg->max_streams;
  Alloc& A = c->mem;
  Bufs& b = c->b;
  memset(&b, 0, sizeof(b));
  const long long cap = g.kp_cap;
  b.layers = A.get<uint8_t>((size_t)S * g.layer_slab);
  b.scores = A.get<uint8_t>((size_t)S * g.sm_slab);
  b.bitmaps = A.get<uint32_t>((size_t)S * g.bm_slab_words);
  b.tile_stamp = A.get<int>((size_t)S * g.tiles_per_stream);
  b.band_stamp = A.get<int>((size_t)S * g.bands_per_stream);
  b.unit_rec = A.get<int>((size_t)S * g.bands_per_stream * VF_TILE_H * 4);
  b.unit_out = A.get<int>((size_t)S * g.bands_per_stream * VF_TILE_H);
  b.nms_u = 1;
  b.band_cand = A.get<int>((size_t)S * g.bands_per_stream);
  b.gidx = A.get<int>((size_t)S * cap);
  b.prop_cnt = A.get<int>((size_t)S * g.prop_chunks);
  b.prop_out = A.get<int>((size_t)S * g.prop_chunks);
  b.cells = A.get<uint8_t>((size_t)S * g.cell_slab);
  b.cbits = g.use_cbits ? A.get<uint32_t>((size_t)S * 2 * g.grid[0].rows * g.cbits_words) : nullptr;
  b.state = A.get<uint8_t>((size_t)S * 2 * g.state_slab);   // two parities (iddm_state)
  int* dl = A.get<int>((size_t)g.lut_len);
  b.lut = dl;
  b.sat = A.get<uint32_t>((size_t)S * g.W * g.H);   // one strip SAT per stream
  b.rowsum = A.get<uint32_t>((size_t)S * g.H * g.stx);
  b.carry = A.get<uint32_t>((size_t)S * g.H * g.stx);
  b.sat_bits = A.get<unsigned>((size_t)S * g.sty * g.stw_words);
  b.sat_work = A.get<int>((size_t)S * g.sat_tiles);
  b.sat_count = A.get<int>((size_t)S);
  b.cand = A.get<uint32_t>((size_t)S * cap);
  b.cand_rank = A.get<int>((size_t)S * cap);
  b.chunk_off = A.get<int>((size_t)S * g.nms_chunks);
  b.nms_cnt = A.get<int>((size_t)S * 4);
  b.st_x = A.get<double>((size_t)S * cap); b.st_y = A.get<double>((size_t)S * cap);
  b.st_s = A.get<double>((size_t)S * cap); b.st_v = A.get<double>((size_t)S * cap);
  b.fx = A.get<double>((size_t)S * 2 * cap); b.fy = A.get<double>((size_t)S * 2 * cap);
  b.fs = A.get<double>((size_t)S * 2 * cap); b.ft = A.get<double>((size_t)S * 2 * cap);
  b.fv = A.get<double>((size_t)S * 2 * cap);
  b.forg = A.get<uint8_t>((size_t)S * 2 * cap);
  b.fage = A.get<int>((size_t)S * 2 * cap);
  b.fdesc = A.get<uint8_t>((size_t)S * 2 * cap * 64);
  b.ctr = A.get<int>((size_t)S * C_NCTR);
  b.cov = A.get<unsigned long long>((size_t)S);
  b.report = A.get<double>((size_t)S * 16);
  b.worklist = A.get<int>((size_t)S * g.tiles_per_stream);
  b.work_count = A.get<int>((size_t)S);
  if (A.err != cudaSuccess) { int r = cuda_status(A.err); A.release(); delete c; return r; }
  cudaError_t e = cudaMemcpy(dl, lut.data(), sizeof(int) * lut.size(), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) { int r = cuda_status(e); A.release(); delete c; return r; }
  c->frames_done.assign(S, 0);
  c->pyr_smem = pyramid_smem(g);
  if (c->pyr_smem > 48 * 1024)
    cudaFuncSetAttribute(k_pyramid, cudaFuncAttributeMaxDynamicSharedMemorySize, c->pyr_smem);
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  int occ = 0;
  const int fast_smem = (int)sizeof(FastWarp) * FAST_WARPS + (S + 1) * (int)sizeof(int);
  cudaFuncSetAttribute(k_fast, cudaFuncAttributeMaxDynamicSharedMemorySize, fast_smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_fast, 32 * FAST_WARPS, fast_smem);
  c->fast_grid = std::max(1, g_num_sms * std::max(occ, 1));
  c->sat_smem = SAT_WARPS * VF_ST * SAT_PITCH * 4 + (S + 1) * 4;
  if (c->sat_smem > 48 * 1024) cudaFuncSetAttribute(k_sat, cudaFuncAttributeMaxDynamicSharedMemorySize, c->sat_smem);
  occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_sat, 256, c->sat_smem);
  c->sat_grid = std::max(1, g_num_sms * std::max(occ, 1));
  occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_desc_fused, 32 * DSW, (S + 1) * sizeof(int));
  c->dfused_grid = std::max(1, g_num_sms * std::max(occ, 1));
  occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_nms_test, 1 << NMS_CHUNK_LOG, (S + 1) * sizeof(int));
  c->nmst_grid = std::max(1, g_num_sms * std::max(occ, 1));
  if (g.mask_mode == 3) {                    // temporal baseline state
    Gop o;
    gop_from_config(*cfg, o);
    std::vector<double> co, fi;
    gop_setup(o, c->bmq, co, fi);
    double* dco = A.get<double>(co.size());
    double* dfi = A.get<double>(std::max<size_t>(fi.size(), 2));
    b.prev_frame = A.get<uint8_t>((size_t)S * g.W * g.H);
    b.bm_found = A.get<uint8_t>((size_t)S * cap);
    b.bm_chunk = A.get<int>((size_t)S * g.prop_chunks);
    if (A.err != cudaSuccess) { int r = cuda_status(A.err); vf_destroy(c); return r; }
    cudaMemcpy(dco, co.data(), sizeof(double) * co.size(), cudaMemcpyHostToDevice);
    if (!fi.empty()) cudaMemcpy(dfi, fi.data(), sizeof(double) * fi.size(), cudaMemcpyHostToDevice);
    b.bm_coarse = dco; b.bm_fine = dfi;
    c->bmq.coarse = dco; c->bmq.fine = dfi;
    c->bm_smem = BM_WARPS * c->bmq.sm_words * 4 + (S + 1) * 4;
    if (c->bm_smem > 227 * 1024) { vf_destroy(c); return VF_ERR_ARG; }
    if (c->bm_smem > 48 * 1024) cudaFuncSetAttribute(k_blockmatch, cudaFuncAttributeMaxDynamicSharedMemorySize, c->bm_smem);
    occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_blockmatch, 32 * BM_WARPS, c->bm_smem);
    c->bm_grid = std::max(1, g_num_sms * std::max(occ, 1));
  }
  *out = c;
  return VF_OK;
}

static void pipe_free(vf_ctx* c);

static void graph_drop(vf_ctx* c);
int vf_destroy(vf_ctx* c)
{
  if (!c) return VF_OK;
  for (int k = 0; k < 2; k++) {
    if (c->hstage[k]) cudaFree(c->hstage[k]);
    if (c->hstage_free[k]) cudaEventDestroy(c->hstage_free[k]);
  }
  pipe_free(c);
  pack_free(c);
  graph_drop(c);
  if (c->cap) cudaStreamDestroy(c->cap);
  for (size_t k = 0; k < c->gstreams.size(); k++) { cudaStreamDestroy(c->gstreams[k]); cudaEventDestroy(c->gjoin[k]); }
  for (size_t k = 0; k < c->aux.size(); k++) {
    cudaStreamDestroy(c->aux[k]); cudaEventDestroy(c->aux_in[k]); cudaEventDestroy(c->aux_mid[k]);
    cudaEventDestroy(c->aux_out[k]);
  }
  if (c->gfork) cudaEventDestroy(c->gfork);
  if (c->hp) { cudaStreamDestroy(c->hp); cudaEventDestroy(c->hp_in); cudaEventDestroy(c->hp_out); }
  for (size_t k = 0; k < c->dstreams.size(); k++) { cudaStreamDestroy(c->dstreams[k]); cudaEventDestroy(c->djoin[k]); }
  for (cudaEvent_t ev : c->dfork_g) cudaEventDestroy(ev);
  for (cudaEvent_t ev : c->dsat_e) cudaEventDestroy(ev);
  for (cudaEvent_t ev : c->dfast_e) cudaEventDestroy(ev);
  for (cudaStream_t ss : c->sat_s) cudaStreamDestroy(ss);
  for (cudaEvent_t ev : c->dsatall_e) cudaEventDestroy(ev);
  for (size_t k = 0; k < c->pyi_s.size(); k++) { cudaStreamDestroy(c->pyi_s[k]); cudaEventDestroy(c->pyi_e[k]); }
  if (c->pack.pre) cudaFree(c->pack.pre);
  if (c->pack.pre_host) cudaFreeHost(c->pack.pre_host);
  for (cudaEvent_t ev : c->ev_pool) cudaEventDestroy(ev);
  for (cudaEvent_t ev : c->ev_used) cudaEventDestroy(ev);
  for (cudaEvent_t ev : c->side_ev) cudaEventDestroy(ev);
  c->mem.release();
  delete c;
  return VF_OK;
}

int vf_layer_geometry(const vf_ctx* c, int32_t* ws, int32_t* hs, double* scales)
{
  if (!c) return VF_ERR_ARG;
  for (int l = 0; l < c->g.NL; l++) {
    if (ws) ws[l] = c->g.L[l].w;
    if (hs) hs[l] = c->g.L[l].h;
    if (scales) scales[l] = c->g.L[l].scale;
  }
  return VF_OK;
}

int vf_set_timing(vf_ctx* c, int enable)
{
  if (!c) return VF_ERR_ARG;
  c->timing = enable;
  return VF_OK;
}

int vf_get_stage_ms(vf_ctx* c, double* ms7, int* n_steps, void* stream)  /* ms7: VF_NSTAGES entries */
{
  if (!c || !ms7) return VF_ERR_ARG;
  cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_status(e);
  for (int k = 0; k < VF_NSTAGES; k++) ms7[k] = 0.0;
  int steps = 0;
  // intervals between consecutive marks of the same group; stage times are
  // summed over groups and divided by the group count (average launch time)
  const size_t m = c->ev_used.size();
  std::vector<int> groups_seen;
  for (size_t i = 0; i < m; i++) {
    if (c->ev_stage[i] < 0) {
      if (c->ev_group[i] == 0) steps++;
      continue;
    }
    size_t j = i + 1;
    while (j < m && c->ev_group[j] != c->ev_group[i]) j++;
    if (j >= m) continue;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->ev_used[i], c->ev_used[j]);
    ms7[c->ev_stage[i]] += ms;
    if (std::find(groups_seen.begin(), groups_seen.end(), c->ev_group[i]) == groups_seen.end())
      groups_seen.push_back(c->ev_group[i]);
  }
  // side-stream kernels: their own duration (they overlap the main stream)
  for (size_t i = 0; i + 1 < c->side_ev.size(); i += 2) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->side_ev[i], c->side_ev[i + 1]);
    ms7[c->side_stage[i / 2]] += ms;
  }
  if (groups_seen.size() > 1)
    for (int k = 0; k < VF_NSTAGES; k++) ms7[k] /= (double)groups_seen.size();
  for (cudaEvent_t ev : c->side_ev) c->ev_pool.push_back(ev);
  c->side_ev.clear();
  c->side_stage.clear();
  for (cudaEvent_t ev : c->ev_used) c->ev_pool.push_back(ev);
  c->ev_used.clear();
  c->ev_stage.clear();
  c->ev_group.clear();
  if (n_steps) *n_steps = steps;
  return VF_OK;
}

int vf_set_history(vf_ctx* c, double* hist_dev, int32_t max_frames)
{
  if (!c || max_frames < 0 || (max_frames > 0 && !hist_dev)) return VF_ERR_ARG;
  c->b.hist = max_frames > 0 ? hist_dev : nullptr;
  c->b.hist_frames = max_frames;
  graph_drop(c);   // the graph bakes in the pointers
  return VF_OK;
}

int vf_reset(vf_ctx* c, void* stream)
{
  if (!c) return VF_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  k_reset<<<cdiv(c->S, 128), 128, 0, st>>>(c->b.ctr, c->b.cov, c->b.report, c->S);
  std::fill(c->frames_done.begin(), c->frames_done.end(), 0);
  return cuda_status(cudaGetLastError());
}

// Batches up to this many frame bytes replay the graph.  Larger batches (the
// 64 x 1080p step) launch eagerly: their kernels fill the GPU on their own,
// and a captured graph loses the stream priorities the side / describe
// streams rely on (569 vs 562 us per config-5 step measured).
#define VF_GRAPH_MAX_BYTES (64LL << 20)

static int launch_step(vf_ctx* c, int s0, int n, cudaStream_t st)
{
  const Geo& g = c->g;
  Bufs b = c->b;
  b.s0 = s0;
  if (g.mask_mode == 2) {
    stage_mark(c, 0, st);
    int smem = g.grid[0].rows * g.grid[0].cols * 4;
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_binmask, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_binmask<<<n, 1024, smem, st>>>(g, b); DBG_SYNC(st, "k_binmask");
  }
  stage_mark(c, 1, st);
  const bool pyr4 = g.O == 4 && g.ptw == 96 && g.pth == 48 && !(g.mask_mode == 1 && !g.use_cbits);
  const int pyo_blocks = cdiv((long long)cdiv(g.W, PYO_COLS) * cdiv(g.L[2].h, 4), 8);
  const int pyi_blocks = cdiv((long long)cdiv(g.W, PYI_COLS) * cdiv(g.L[1].h, 8 * PYI_RG), 8);
  if (pyr4 && g.pyr_split)
    { k_pyr_o<<<dim3(pyo_blocks, n), 256, 0, st>>>(g, b); DBG_SYNC(st, "k_pyr_o"); }
  else if (pyr4)
    { k_pyramid4<PYR_FULL><<<dim3(g.ptx, g.pty, n), 256, 0, st>>>(g, b); DBG_SYNC(st, "k_pyramid4"); }
  else
    { k_pyramid<<<dim3(g.ptx, g.pty, n), 256, c->pyr_smem, st>>>(g, b); DBG_SYNC(st, "k_pyramid"); }
  const int tile_ctas = cdiv(g.tiles_per_stream, 256);   // lane per FAST tile
  const int cov_ctas = (g.mask_mode == 1 && g.per_layer) ? cdiv(g.H, 8) : 0;
  const int carry_ctas = cdiv(g.sty, 8);
  // strip carries, propagation counts and per_layer coverage on the side stream
  // (needed from k_nms on), the tile work list on the main stream (k_fast)
  const int gi = c->cur_group;
  while ((int)c->aux.size() <= gi) {
    cudaStream_t as;
    cudaEvent_t ei, em, eo;
    if (cudaStreamCreateWithFlags(&as, cudaStreamNonBlocking) != cudaSuccess) return VF_ERR_CUDA;
    if (cudaEventCreateWithFlags(&ei, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&em, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&eo, cudaEventDisableTiming) != cudaSuccess) { cudaStreamDestroy(as); return VF_ERR_CUDA; }
    c->aux.push_back(as); c->aux_in.push_back(ei); c->aux_mid.push_back(em); c->aux_out.push_back(eo);
  }
  cudaEventRecord(c->aux_in[gi], st);
  stage_mark(c, 2, st);
  // intra-octave chain of masked frames near active cells (after the IDDM
  // bits) on its own high-priority stream, concurrent with the main work list
  // (both only read the bit mask); k_fast waits for both
  const bool pyi = pyr4 && g.pyr_split;
  if (pyi) {
    while ((int)c->pyi_s.size() <= gi) {
      int lo = 0, hi = 0;
      cudaDeviceGetStreamPriorityRange(&lo, &hi);
      cudaStream_t ps;
      cudaEvent_t pe;
      if (cudaStreamCreateWithPriority(&ps, cudaStreamNonBlocking, hi) != cudaSuccess) return VF_ERR_CUDA;
      if (cudaEventCreateWithFlags(&pe, cudaEventDisableTiming) != cudaSuccess) { cudaStreamDestroy(ps); return VF_ERR_CUDA; }
      c->pyi_s.push_back(ps);
      c->pyi_e.push_back(pe);
    }
    cudaStreamWaitEvent(c->pyi_s[gi], c->aux_in[gi], 0);
    k_pyr_i<<<dim3(pyi_blocks, n), 256, 0, c->pyi_s[gi]>>>(g, b); DBG_SYNC(st, "k_pyr_i");
    cudaEventRecord(c->pyi_e[gi], c->pyi_s[gi]);
  }
  k_worklist<<<dim3(tile_ctas, n), 256, 0, st>>>(g, b, tile_ctas, 0, 0); DBG_SYNC(st, "k_worklist");
  if (pyi) cudaStreamWaitEvent(st, c->pyi_e[gi], 0);
  // In large batches the side chain (carries, propagation counts, Eq. 1
  // propagation) starts with k_fast rather than beside k_pyr_i / k_worklist,
  // which are on the critical path (config 5: 553 -> 536 us per step; the
  // single-stream configs measured 1-4 us better with the early start).
  // VF_SIDE_LATE=0 / 1 forces either.
  const char* sl_env = getenv("VF_SIDE_LATE");
  const bool side_late = sl_env ? atoi(sl_env) != 0 : (long long)g.W * g.H * n > VF_GRAPH_MAX_BYTES;
  if (side_late) cudaEventRecord(c->aux_in[gi], st);
  cudaStreamWaitEvent(c->aux[gi], c->aux_in[gi], 0);
  const bool prop = g.mask_mode == 1 || g.mask_mode == 2;
  k_worklist<<<dim3(cov_ctas + carry_ctas + (prop ? PROP_CTAS : 0), n), 256, 0, c->aux[gi]>>>(
      g, b, 0, cov_ctas, carry_ctas); DBG_SYNC(c->aux[gi], "k_worklist");
  cudaEventRecord(c->aux_mid[gi], c->aux[gi]);
  // Eq. 1 propagation into the last n_prop slots of the list: independent of
  // the detection, so it runs beside k_fast / k_nms (VF_PROP_LATE=1: beside
  // the describe kernels instead)
  const bool prop_late = getenv("VF_PROP_LATE") && atoi(getenv("VF_PROP_LATE")) != 0;
  auto launch_prop = [&]() {
    if (!prop) return;
    cudaEvent_t p0 = nullptr, p1 = nullptr;
    if (c->timing) {
      p0 = pool_event(c);
      p1 = pool_event(c);
      cudaEventRecord(p0, c->aux[gi]);
    }
    k_propagate<<<dim3(PROP_CTAS, n), 256, 0, c->aux[gi]>>>(g, b); DBG_SYNC(c->aux[gi], "k_propagate");
    if (c->timing) {
      cudaEventRecord(p1, c->aux[gi]);
      c->side_ev.push_back(p0);
      c->side_ev.push_back(p1);
      c->side_stage.push_back(7);
    }
  };
  // VF_SAT_AUX=1: the early k_sat runs on the side stream, before k_propagate
  static const bool sat_aux = getenv("VF_SAT_AUX") && atoi(getenv("VF_SAT_AUX")) != 0;
  // Early SAT is off for large intensity-masked batches: there k_propagate
  // already fills the NMS window, and k_sat beside it costs the NMS more than
  // the describe stage gains (config 5: 533 vs 521 us per step).
  const char* se_env = getenv("VF_SAT_EARLY");
  const bool sat_early_env = se_env ? atoi(se_env) != 0
                                    : !(g.mask_mode == 1 && (long long)g.W * g.H * n > VF_GRAPH_MAX_BYTES);
  const bool prop_after_sat = sat_aux && sat_early_env && !prop_late;
  if (!prop_late && !prop_after_sat) {
    launch_prop();
    cudaEventRecord(c->aux_out[gi], c->aux[gi]);
  }
  stage_mark(c, 3, st);
  const int pre_bytes = (n + 1) * (int)sizeof(int);
  b.nms_pre = !(getenv("VF_NMS_PRE") && atoi(getenv("VF_NMS_PRE")) == 0);
  // Early SAT (default; VF_SAT_EARLY=0: the round-2 arrangement): k_fast marks
  // the SAT tiles from footprint bounds of its candidates, so the strip SATs
  // are built on the first describe stream beside the latency-bound NMS
  // kernels instead of between k_nms_finish and k_desc_fused.
  b.sat_early = sat_early_env;
  b.sat_check = getenv("VF_SAT_CHECK") && atoi(getenv("VF_SAT_CHECK")) != 0;
  k_fast<<<c->fast_grid, 32 * FAST_WARPS, sizeof(FastWarp) * FAST_WARPS + pre_bytes, st>>>(g, b, n); DBG_SYNC(st, "k_fast");
  stage_mark(c, 4, st);
  // candidate-parallel NMS: ordered candidate list, thread-per-candidate test +
  // refinement with chunk ranks, chunk offsets + FrameReport
  b.nms_u = 1;
  b.desc_bin = 1;
  b.orient_seq = getenv("VF_ORIENT_SEQ") && atoi(getenv("VF_ORIENT_SEQ")) != 0;
  static const int dpar_env = getenv("VF_DESC_PAR") ? std::max(1, std::min(2, atoi(getenv("VF_DESC_PAR")))) : 2;
  const int dpar = std::min(dpar_env, n);
  if ((int)c->dstreams.size() < 2 * (gi + 1)) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    while ((int)c->dfork_g.size() <= gi) {
      cudaEvent_t f;
      if (cudaEventCreateWithFlags(&f, cudaEventDisableTiming) != cudaSuccess) return VF_ERR_CUDA;
      c->dfork_g.push_back(f);
    }
    while ((int)c->dstreams.size() < 2 * (gi + 1)) {
      cudaStream_t ds;
      cudaEvent_t de;
      if (cudaStreamCreateWithPriority(&ds, cudaStreamNonBlocking, hi) != cudaSuccess) return VF_ERR_CUDA;
      if (cudaEventCreateWithFlags(&de, cudaEventDisableTiming) != cudaSuccess) { cudaStreamDestroy(ds); return VF_ERR_CUDA; }
      c->dstreams.push_back(ds);
      c->djoin.push_back(de);
    }
  }
  // Staggered halves (half 1's SAT build beside half 0's describe) pay off
  // when every tile is built (modes none / binning: dense config 5 3100 ->
  // 3007 us) but not in masked frames (533 -> 543 us); VF_DESC_STAGGER forces.
  const char* stg = getenv("VF_DESC_STAGGER");
  const bool desc_stagger = stg ? atoi(stg) != 0 : (g.mask_mode == 0 || g.mask_mode == 2);
  while (c->dsat_e.size() < c->dstreams.size()) {
    cudaEvent_t e;
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return VF_ERR_CUDA;
    c->dsat_e.push_back(e);
  }
  while ((int)c->dfast_e.size() <= gi) {
    cudaEvent_t e0, e1;
    if (cudaEventCreateWithFlags(&e0, cudaEventDisableTiming) != cudaSuccess) return VF_ERR_CUDA;
    if (cudaEventCreateWithFlags(&e1, cudaEventDisableTiming) != cudaSuccess) { cudaEventDestroy(e0); return VF_ERR_CUDA; }
    c->dfast_e.push_back(e0);
    c->dsatall_e.push_back(e1);
  }
  if (b.sat_early) {
    // after k_fast (tile marks) and the side stream's strip carries
    // VF_SAT_LOW=1: on a dedicated lowest-priority stream; VF_SAT_CTAS=k: at
    // most k CTAs per SM (the NMS kernels keep the rest of the SM)
    // (default: low priority for multi-stream batches -- config 3 118 vs 125 us --
    // and the describe stream for a single stream -- config 1 71 vs 75 us)
    const char* sl = getenv("VF_SAT_LOW");
    const bool sat_low = sl ? atoi(sl) != 0 : n > 1;
    static const int sat_ctas = getenv("VF_SAT_CTAS") ? atoi(getenv("VF_SAT_CTAS")) : 0;
    while ((int)c->sat_s.size() <= gi) {
      int lo = 0, hi = 0;
      cudaDeviceGetStreamPriorityRange(&lo, &hi);
      cudaStream_t ss;
      if (cudaStreamCreateWithPriority(&ss, cudaStreamNonBlocking, lo) != cudaSuccess) return VF_ERR_CUDA;
      c->sat_s.push_back(ss);
    }
    cudaStream_t ds = sat_aux ? c->aux[gi] : sat_low ? c->sat_s[gi] : c->dstreams[2 * gi];
    const int sgrid = sat_ctas > 0 ? std::min(c->sat_grid, g_num_sms * sat_ctas) : c->sat_grid;
    cudaEventRecord(c->dfast_e[gi], st);
    cudaStreamWaitEvent(ds, c->dfast_e[gi], 0);
    cudaStreamWaitEvent(ds, c->aux_mid[gi], 0);
    k_sat_list<<<n, NF_THREADS, 0, ds>>>(g, b); DBG_SYNC(ds, "k_sat_list");
    k_sat<<<sgrid, 256, c->sat_smem, ds>>>(g, b, n, 0); DBG_SYNC(ds, "k_sat");
    cudaEventRecord(c->dsatall_e[gi], ds);
    if (prop_after_sat) {
      launch_prop();
      cudaEventRecord(c->aux_out[gi], c->aux[gi]);
    }
  }
  k_nms_list<<<dim3(cdiv(g.bands_per_stream, NL_WARPS), n), 32 * NL_WARPS, 0, st>>>(g, b); DBG_SYNC(st, "k_nms_list");
  k_nms_test<<<c->nmst_grid, 1 << NMS_CHUNK_LOG, pre_bytes, st>>>(g, b, n); DBG_SYNC(st, "k_nms_test");
  cudaStreamWaitEvent(st, c->aux_mid[gi], 0);   // propagation count (k_nms_finish), strip carries (k_sat)
  k_nms_finish<<<n, NF_THREADS, 0, st>>>(g, b); DBG_SYNC(st, "k_nms_finish");
  if (prop_late) {
    cudaEventRecord(c->aux_in[gi], st);
    cudaStreamWaitEvent(c->aux[gi], c->aux_in[gi], 0);
    launch_prop();
    cudaEventRecord(c->aux_out[gi], c->aux[gi]);
  }
  stage_mark(c, 5, st);
  // Describe (descriptor.py:85-144): the strip SATs of the tiles k_nms_test
  // marked, then k_desc_fused (warp per keypoint: theta = 0 means,
  // orientation, rotated means, bits), for VF_DESC_PAR (default 2) stream
  // halves on concurrent high-priority describe streams.
  cudaEventRecord(c->dfork_g[gi], st);
  for (int h = 0; h < dpar; h++) {
    const int h0 = (int)((long long)n * h / dpar), h1 = (int)((long long)n * (h + 1) / dpar);
    Bufs bh = b;
    bh.s0 = b.s0 + h0;
    bh.frames = b.frames + (long long)h0 * b.frame_stride;
    const int nh = h1 - h0, pb = (nh + 1) * (int)sizeof(int);
    cudaStream_t ds = c->dstreams[2 * gi + h];
    cudaStreamWaitEvent(ds, c->dfork_g[gi], 0);
    // staggered: half h's SAT build waits for half h-1's, so it runs beside
    // half h-1's (L1-bound) describe instead of beside its SAT build
    if (b.sat_early) {
      cudaStreamWaitEvent(ds, c->dsatall_e[gi], 0);
    } else {
      if (desc_stagger && h > 0) cudaStreamWaitEvent(ds, c->dsat_e[2 * gi + h - 1], 0);
      k_sat<<<c->sat_grid, 256, c->sat_smem, ds>>>(g, bh, nh, 0); DBG_SYNC(ds, "k_sat");
      if (desc_stagger) cudaEventRecord(c->dsat_e[2 * gi + h], ds);
    }
    k_desc_fused<<<c->dfused_grid, 32 * DSW, pb, ds>>>(g, bh, nh); DBG_SYNC(ds, "k_desc_fused");
    cudaEventRecord(c->djoin[2 * gi + h], ds);
  }
  for (int h = 0; h < dpar; h++) cudaStreamWaitEvent(st, c->djoin[2 * gi + h], 0);
  // k_propagate (stage 7) is timed on the side stream; the join wait counts
  // toward the finalize stage
  stage_mark(c, 8, st);
  cudaStreamWaitEvent(st, c->aux_out[gi], 0);
  k_finalize<<<cdiv(n, 128), 128, 0, st>>>(g, b, n); DBG_SYNC(st, "k_finalize");
  stage_mark(c, -1, st);
  if (!c->capturing)
    for (int s = s0; s < s0 + n; s++) c->frames_done[s]++;
  return cuda_status(cudaGetLastError());
}

// Streams [0, n) in G groups on separate CUDA streams (forked from / joined
// into `st`), so the launches of one group fill the gaps and tails of another.
static int launch_grouped(vf_ctx* c, int n, cudaStream_t st)
{
  // one group measured fastest once NMS refines survivors densely (r01: 55.9k
  // vs 54.8k frames/s at 64 x 1080p with 4 groups); VF_STREAM_GROUPS overrides
  int G = 1;
  if (const char* e = getenv("VF_STREAM_GROUPS")) G = std::max(1, std::min(n, atoi(e)));
  if (G == 1) {
    c->cur_group = 0;
    // The main chain runs on an internal highest-priority stream, so the block
    // scheduler prefers its CTAs over the side stream's propagation, which
    // fills the slots FAST / NMS leave (733 -> 710 us per 64-stream step);
    // VF_PRIO=0 launches on the caller's stream instead
    static const bool prio = !(getenv("VF_PRIO") && atoi(getenv("VF_PRIO")) == 0);
    if (!prio) return launch_step(c, 0, n, st);
    if (!c->hp) {
      int lo = 0, hi = 0;
      cudaDeviceGetStreamPriorityRange(&lo, &hi);
      if (cudaStreamCreateWithPriority(&c->hp, cudaStreamNonBlocking, hi) != cudaSuccess) return VF_ERR_CUDA;
      cudaEventCreateWithFlags(&c->hp_in, cudaEventDisableTiming);
      cudaEventCreateWithFlags(&c->hp_out, cudaEventDisableTiming);
    }
    cudaEventRecord(c->hp_in, st);
    cudaStreamWaitEvent(c->hp, c->hp_in, 0);
    const int rc = launch_step(c, 0, n, c->hp);
    cudaEventRecord(c->hp_out, c->hp);
    cudaStreamWaitEvent(st, c->hp_out, 0);
    return rc;
  }
  if ((int)c->gstreams.size() < G) {
    if (!c->gfork) cudaEventCreateWithFlags(&c->gfork, cudaEventDisableTiming);
    while ((int)c->gstreams.size() < G) {
      cudaStream_t gs;
      cudaEvent_t ge;
      if (cudaStreamCreateWithFlags(&gs, cudaStreamNonBlocking) != cudaSuccess) return VF_ERR_CUDA;
      cudaEventCreateWithFlags(&ge, cudaEventDisableTiming);
      c->gstreams.push_back(gs);
      c->gjoin.push_back(ge);
    }
  }
  cudaEventRecord(c->gfork, st);
  const uint8_t* base = c->b.frames;
  int rc = VF_OK;
  for (int k = 0; k < G && rc == VF_OK; k++) {
    const int s0 = (int)((long long)n * k / G), s1 = (int)((long long)n * (k + 1) / G);
    cudaStreamWaitEvent(c->gstreams[k], c->gfork, 0);
    c->b.frames = base + (long long)s0 * c->b.frame_stride;
    c->cur_group = k;
    rc = launch_step(c, s0, s1 - s0, c->gstreams[k]);
    cudaEventRecord(c->gjoin[k], c->gstreams[k]);
  }
  c->b.frames = base;
  c->cur_group = 0;
  for (int k = 0; k < G; k++) cudaStreamWaitEvent(st, c->gjoin[k], 0);
  return rc;
}

// Temporal mode, off-GOP run of streams [s0, s0 + n): block matching of the
// previous features (temporal.py:274-308), order-preserving compaction and
// report, then the current frames become the previous ones.
static int launch_temporal(vf_ctx* c, int s0, int n, cudaStream_t st)
{
  const Geo& g = c->g;
  Bufs b = c->b;
  b.s0 = s0;
  cudaMemsetAsync(b.bm_chunk + (long long)s0 * g.prop_chunks, 0, sizeof(int) * (size_t)n * g.prop_chunks, st);
  k_blockmatch<<<c->bm_grid, 32 * BM_WARPS, c->bm_smem, st>>>(g, b, c->bmq, n);
  k_bm_write<<<dim3(std::max(g.prop_chunks, 1), n), 256, 0, st>>>(g, b);
  k_copy_frames<<<dim3(64, n), 256, 0, st>>>(g, b);
  k_finalize<<<cdiv(n, 128), 128, 0, st>>>(g, b, n);
  for (int s = s0; s < s0 + n; s++) c->frames_done[s]++;
  return cuda_status(cudaGetLastError());
}

// Streams [0, n): detection (grouped) in the mask modes; in temporal mode,
// contiguous runs of streams at a GOP start run full detection and keep their
// frame, the others block-match (pipeline.py:299-307).
static int launch_frames(vf_ctx* c, int n, cudaStream_t st)
{
  if (c->g.mask_mode != 3) return launch_grouped(c, n, st);
  const uint8_t* base = c->b.frames;
  int rc = VF_OK;
  for (int s0 = 0; s0 < n && rc == VF_OK;) {
    const bool gop = c->frames_done[s0] % c->g.gop_delta == 0;
    int s1 = s0 + 1;
    while (s1 < n && (c->frames_done[s1] % c->g.gop_delta == 0) == gop) s1++;
    c->b.frames = base + (long long)s0 * c->b.frame_stride;
    if (gop) {
      rc = launch_step(c, s0, s1 - s0, st);
      Bufs b = c->b;
      b.s0 = s0;
      k_copy_frames<<<dim3(64, s1 - s0), 256, 0, st>>>(c->g, b);
    } else {
      rc = launch_temporal(c, s0, s1 - s0, st);
    }
    s0 = s1;
  }
  c->b.frames = base;
  return rc == VF_OK ? cuda_status(cudaGetLastError()) : rc;
}

int vf_block_match(const uint8_t* prev_dev, const uint8_t* cur_dev, int w, int h, int64_t pitch, int n,
                   const double* x_dev, const double* y_dev, const vf_config* gop, double* nx_dev, double* ny_dev,
                   double* sad_dev, uint8_t* found_dev, void* stream)
{
  if (n < 0 || w < 1 || h < 1 || pitch < w) return VF_ERR_ARG;
  vf_config zero;
  memset(&zero, 0, sizeof(zero));
  Gop o;
  int rc = gop_from_config(gop ? *gop : zero, o);
  if (rc) return rc;
  if (n == 0) return VF_OK;
  if (!prev_dev || !cur_dev || !x_dev || !y_dev || !nx_dev || !ny_dev || !sad_dev || !found_dev) return VF_ERR_ARG;
  if (!g_num_sms) { cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, 0); }
  vft::Setup q{};
  std::vector<double> co, fi;
  gop_setup(o, q, co, fi);
  cudaStream_t st = (cudaStream_t)stream;
  double *dco = nullptr, *dfi = nullptr;
  cudaError_t e = cudaMallocAsync(&dco, sizeof(double) * co.size(), st);
  if (e == cudaSuccess) e = cudaMallocAsync(&dfi, sizeof(double) * std::max<size_t>(fi.size(), 2), st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dco, co.data(), sizeof(double) * co.size(), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess && !fi.empty())
    e = cudaMemcpyAsync(dfi, fi.data(), sizeof(double) * fi.size(), cudaMemcpyHostToDevice, st);
  const int smem = BM_WARPS * q.sm_words * 4;
  if (e == cudaSuccess && smem > 227 * 1024) e = cudaErrorInvalidValue;
  if (e == cudaSuccess) {
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_block_match, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    q.coarse = dco; q.fine = dfi;
    const int grid = std::max(1, std::min(cdiv(n, BM_WARPS), g_num_sms * 8));
    k_block_match<<<grid, 32 * BM_WARPS, smem, st>>>(q, prev_dev, cur_dev, w, h, pitch, n, x_dev, y_dev, nx_dev,
                                                    ny_dev, sad_dev, found_dev);
    e = cudaGetLastError();
  }
  if (dco) cudaFreeAsync(dco, st);
  if (dfi) cudaFreeAsync(dfi, st);
  return cuda_status(e);
}

// Every step replays a CUDA graph of the launch sequence, captured once per
// batch size: the path is a chain of ~12 dependent, individually latency-bound
// kernels (plus the side / describe streams), and a graph launch removes the
// per-launch host work and most of the inter-kernel gaps.  The caller's frame
// pointer changes every step: each kernel node's Bufs argument is re-pointed
// with cudaGraphExecKernelNodeSetParams (streams of a describe half keep their
// offset), so no input copy is needed.

// Argument count of each kernel launch_step launches (all take (Geo, Bufs, ...)).
static int step_kernel_arity(const void* f)
{
  if (f == (const void*)k_worklist) return 5;
  if (f == (const void*)k_sat) return 4;
  if (f == (const void*)k_fast || f == (const void*)k_nms_test || f == (const void*)k_desc_fused ||
      f == (const void*)k_finalize)
    return 3;
  if (f == (const void*)k_binmask || f == (const void*)k_pyr_o || f == (const void*)k_pyr_i ||
      f == (const void*)k_pyramid4<PYR_FULL> || f == (const void*)k_pyramid || f == (const void*)k_propagate ||
      f == (const void*)k_nms_list || f == (const void*)k_nms_finish || f == (const void*)k_sat_list)
    return 2;
  return 0;
}

static void graph_drop(vf_ctx* c)
{
  if (c->gexec) cudaGraphExecDestroy(c->gexec);
  if (c->graph) cudaGraphDestroy(c->graph);
  c->gexec = nullptr;
  c->graph = nullptr;
  c->gnodes.clear();
  c->gbufs.clear();
}

static int graph_step(vf_ctx* c, const uint8_t* frames_dev, int64_t stream_stride, int64_t row_pitch, int n,
                      cudaStream_t st)
{
  c->b.frames = frames_dev;
  c->b.frame_stride = stream_stride;
  c->b.frame_pitch = row_pitch;
  if ((!c->gexec || c->g_n != n) && c->eager_n != n) {
    // the first step of a batch size runs eagerly: it creates the side streams
    // and events the capture then records into
    const int rc = launch_frames(c, n, st);
    c->eager_n = n;
    return rc;
  }
  cudaError_t e = cudaSuccess;
  if (!c->gexec || c->g_n != n) {
    // capture on an internal non-blocking stream (the caller's may be the
    // legacy default stream, which cannot be captured); replay on the caller's
    graph_drop(c);
    if (!c->cap && cudaStreamCreateWithFlags(&c->cap, cudaStreamNonBlocking) != cudaSuccess) return VF_ERR_CUDA;
    cudaGraph_t graph = nullptr;
    e = cudaStreamBeginCapture(c->cap, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) return cuda_status(e);
    c->capturing = true;
    const int rc = launch_frames(c, n, c->cap);
    c->capturing = false;
    e = cudaStreamEndCapture(c->cap, &graph);
    if (rc != VF_OK) { if (graph) cudaGraphDestroy(graph); return rc; }
    if (e != cudaSuccess) return cuda_status(e);
    size_t nn = 0;
    e = cudaGraphGetNodes(graph, nullptr, &nn);
    std::vector<cudaGraphNode_t> nodes(nn);
    if (e == cudaSuccess && nn) e = cudaGraphGetNodes(graph, nodes.data(), &nn);
    for (size_t i = 0; i < nn && e == cudaSuccess; i++) {
      cudaGraphNodeType t;
      e = cudaGraphNodeGetType(nodes[i], &t);
      if (e != cudaSuccess || t != cudaGraphNodeTypeKernel) continue;
      cudaKernelNodeParams kp;
      e = cudaGraphKernelNodeGetParams(nodes[i], &kp);
      if (e != cudaSuccess) break;
      c->gnodes.push_back(nodes[i]);
      c->gbufs.push_back(*reinterpret_cast<const Bufs*>(kp.kernelParams[1]));
    }
    if (e == cudaSuccess) e = cudaGraphInstantiate(&c->gexec, graph, 0);
    if (e != cudaSuccess) { cudaGraphDestroy(graph); c->gexec = nullptr; graph_drop(c); return cuda_status(e); }
    c->graph = graph;
    c->g_n = n;
    c->g_frames = frames_dev;
    c->g_stride = stream_stride;
  } else if (frames_dev != c->g_frames || stream_stride != c->g_stride || row_pitch != c->gbufs[0].frame_pitch) {
    for (size_t i = 0; i < c->gnodes.size() && e == cudaSuccess; i++) {
      cudaKernelNodeParams kp;
      e = cudaGraphKernelNodeGetParams(c->gnodes[i], &kp);
      if (e != cudaSuccess) break;
      Bufs& nb = c->gbufs[i];
      const long long half = c->g_stride ? (long long)(nb.frames - c->g_frames) / c->g_stride : 0;   // describe half offset
      nb.frames = frames_dev + half * stream_stride;
      nb.frame_stride = stream_stride;
      nb.frame_pitch = row_pitch;
      const int na = step_kernel_arity(kp.func);
      if (na < 2) return VF_ERR_CUDA;   // not a kernel of launch_step
      void* args[8];
      for (int a = 0; a < na; a++) args[a] = kp.kernelParams[a];
      args[1] = &nb;
      kp.kernelParams = args;
      e = cudaGraphExecKernelNodeSetParams(c->gexec, c->gnodes[i], &kp);
    }
    if (e != cudaSuccess) return cuda_status(e);
    c->g_frames = frames_dev;
    c->g_stride = stream_stride;
  }
  e = cudaGraphLaunch(c->gexec, st);
  if (e != cudaSuccess) return cuda_status(e);
  for (int s = 0; s < n; s++) c->frames_done[s]++;
  return VF_OK;
}

int vf_set_graphs(vf_ctx* c, int enable)
{
  if (!c) return VF_ERR_ARG;
  c->graphs = enable;
  if (!enable) graph_drop(c);
  return VF_OK;
}

int vf_process(vf_ctx* c, const uint8_t* frames_dev, int64_t stream_stride, int64_t row_pitch, int n_streams,
               void* stream)
{
  if (!c || !frames_dev || n_streams < 1 || n_streams > c->S || row_pitch < c->g.W) return VF_ERR_ARG;
  if (!g_pattern_ok) return VF_ERR_PATTERN;
  static const bool env_off = getenv("VF_GRAPHS") && atoi(getenv("VF_GRAPHS")) == 0;
  static const long long gmax = getenv("VF_GRAPH_MAX_MB") ? atoll(getenv("VF_GRAPH_MAX_MB")) << 20 : VF_GRAPH_MAX_BYTES;
  if (c->graphs && !env_off && !c->timing && c->g.mask_mode != 3 && (long long)c->g.W * c->g.H * n_streams <= gmax)
    return graph_step(c, frames_dev, stream_stride, row_pitch, n_streams, (cudaStream_t)stream);
  c->b.frames = frames_dev;
  c->b.frame_stride = stream_stride;
  c->b.frame_pitch = row_pitch;
  return launch_frames(c, n_streams, (cudaStream_t)stream);
}

// Grow the feature capacity of every stream to new_cap, keeping each
// stream's previous list (the buffer the next step reads) at the end of its
// new buffer.  Called between a rolled-back step and its replay.
static int regrow(vf_ctx* c, long long new_cap, cudaStream_t st)
{
  Geo& g = c->g;
  Bufs& b = c->b;
  const int S = c->S;
  const long long cap = g.kp_cap;
  new_cap = std::min(new_cap, 1LL << 28);
  if (new_cap <= cap) return VF_ERR_CAPACITY;
  std::vector<int> ctr((size_t)S * C_NCTR);
  cudaError_t e = cudaMemcpyAsync(ctr.data(), b.ctr, sizeof(int) * ctr.size(), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_status(e);
  Alloc& A = c->mem;
  const int chunks = cdiv(new_cap, 1024);
  // per-stream scratch (no contents to keep)
  auto fresh = [&](auto*& ptr, size_t n) {
    using T = std::remove_pointer_t<std::remove_reference_t<decltype(ptr)>>;
    using U = std::remove_const_t<T>;
    U* q = A.get<U>(n);
    if (!q) return false;
    A.drop((void*)ptr);
    ptr = q;
    return true;
  };
  bool ok = fresh(b.gidx, (size_t)S * new_cap) && fresh(b.cand, (size_t)S * new_cap) &&
            fresh(b.cand_rank, (size_t)S * new_cap) &&
            fresh(b.chunk_off, (size_t)S * cdiv(new_cap, 1 << NMS_CHUNK_LOG)) && fresh(b.st_x, (size_t)S * new_cap) &&
            fresh(b.st_y, (size_t)S * new_cap) && fresh(b.st_s, (size_t)S * new_cap) &&
            fresh(b.st_v, (size_t)S * new_cap) && fresh(b.prop_cnt, (size_t)S * chunks) &&
            fresh(b.prop_out, (size_t)S * chunks);
  if (ok && b.bm_found) ok = fresh(b.bm_found, (size_t)S * new_cap) && fresh(b.bm_chunk, (size_t)S * chunks);
  if (ok && b.keep_bits) {
    ok = fresh(b.keep_bits, (size_t)S * (cdiv(new_cap, 32) + 1));
    b.keep_words = cdiv(new_cap, 32) + 1;
  }
  if (!ok) return cuda_status(A.err);
  // feature lists [S][2][cap]: the previous buffer's list moves to the end of the new buffer
  auto moved = [&](auto*& ptr, size_t esz) {
    using T = std::remove_pointer_t<std::remove_reference_t<decltype(ptr)>>;
    T* q = A.get<T>((size_t)S * 2 * new_cap * (esz / sizeof(T)));
    if (!q) return false;
    for (int s = 0; s < S; s++) {
      const int* cs = &ctr[(size_t)s * C_NCTR];
      const int prev = (cs[C_FRAME] & 1) ^ 1;
      const long long n = std::min<long long>(cs[C_NFEAT0 + prev], cap);
      if (cs[C_FRAME] == 0 || n <= 0) continue;
      const char* src = reinterpret_cast<const char*>(ptr) + (((long long)s * 2 + prev) * cap + cap - n) * esz;
      char* dst = reinterpret_cast<char*>(q) + (((long long)s * 2 + prev) * new_cap + new_cap - n) * esz;
      if (cudaMemcpyAsync(dst, src, n * esz, cudaMemcpyDeviceToDevice, st) != cudaSuccess) return false;
    }
    if (cudaStreamSynchronize(st) != cudaSuccess) return false;
    A.drop((void*)ptr);
    ptr = q;
    return true;
  };
  ok = moved(b.fx, 8) && moved(b.fy, 8) && moved(b.fs, 8) && moved(b.ft, 8) && moved(b.fv, 8) && moved(b.forg, 1) &&
       moved(b.fage, 4) && moved(b.fdesc, 64);
  if (!ok) return VF_ERR_CUDA;
  g.kp_cap = (int)new_cap;
  g.prop_chunks = chunks;
  g.nms_chunks = cdiv(new_cap, 1 << NMS_CHUNK_LOG);
  graph_drop(c);
  pipe_free(c);   // re-created with the new capacity on the next submit
  return VF_OK;
}

int vf_process_checked(vf_ctx* c, const uint8_t* frames_dev, int64_t stream_stride, int64_t row_pitch, int n_streams,
                       void* stream)
{
  int rc = vf_process(c, frames_dev, stream_stride, row_pitch, n_streams, stream);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  for (int attempt = 0; attempt < 16; attempt++) {
    std::vector<int> ctr((size_t)n_streams * C_NCTR);
    cudaError_t e = cudaMemcpyAsync(ctr.data(), c->b.ctr, sizeof(int) * ctr.size(), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_status(e);
    long long need = 0;
    bool over = false;
    for (int s = 0; s < n_streams; s++) {
      const int* cs = &ctr[(size_t)s * C_NCTR];
      if (!cs[C_ERR]) continue;
      over = true;
      // staged candidates bound the detections; plus the propagated features
      need = std::max(need, (long long)cs[C_STAGE] + cs[C_NPROP]);
    }
    if (!over) return VF_OK;
    if (c->g.mask_mode == 3) return VF_ERR_CAPACITY;   // temporal mode keeps no replay state
    k_rollback<<<cdiv(n_streams, 128), 128, 0, st>>>(c->b.ctr, c->b.report, 0, n_streams);
    for (int s = 0; s < n_streams; s++) c->frames_done[s]--;
    rc = regrow(c, std::max(2LL * c->g.kp_cap, need + need / 4 + 1024), st);
    if (rc) return rc;
    rc = vf_process(c, frames_dev, stream_stride, row_pitch, n_streams, stream);
    if (rc) return rc;
  }
  return VF_ERR_CAPACITY;
}

int vf_get_capacity(const vf_ctx* c, int32_t* kp_capacity)
{
  if (!c || !kp_capacity) return VF_ERR_ARG;
  *kp_capacity = c->g.kp_cap;
  return VF_OK;
}

static int process_host(vf_ctx* c, const uint8_t* frames_host, int64_t stream_stride, int64_t row_pitch,
                        int n_streams, void* stream, bool checked);

int vf_process_host(vf_ctx* c, const uint8_t* frames_host, int64_t stream_stride, int64_t row_pitch, int n_streams,
                    void* stream)
{
  return process_host(c, frames_host, stream_stride, row_pitch, n_streams, stream, false);
}

int vf_process_host_checked(vf_ctx* c, const uint8_t* frames_host, int64_t stream_stride, int64_t row_pitch,
                            int n_streams, void* stream)
{
  return process_host(c, frames_host, stream_stride, row_pitch, n_streams, stream, true);
}

static int process_host(vf_ctx* c, const uint8_t* frames_host, int64_t stream_stride, int64_t row_pitch,
                        int n_streams, void* stream, bool checked)
{
  if (!c || !frames_host || n_streams < 1 || n_streams > c->S || row_pitch < c->g.W) return VF_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const long long fbytes = (long long)c->g.W * c->g.H;
  if (c->hstage_bytes < fbytes * c->S) {
    for (int k = 0; k < 2; k++) {
      if (c->hstage[k]) cudaFree(c->hstage[k]);
      cudaError_t e = cudaMalloc(&c->hstage[k], fbytes * c->S);
      if (e != cudaSuccess) return cuda_status(e);
      if (!c->hstage_free[k]) cudaEventCreateWithFlags(&c->hstage_free[k], cudaEventDisableTiming);
    }
    c->hstage_bytes = fbytes * c->S;
  }
  const int k = c->hstage_k;
  c->hstage_k ^= 1;
  uint8_t* dst = c->hstage[k];
  cudaError_t e;
  if (row_pitch == c->g.W && stream_stride == fbytes) {
    e = cudaMemcpyAsync(dst, frames_host, fbytes * n_streams, cudaMemcpyHostToDevice, st);
  } else {
    e = cudaSuccess;
    for (int s = 0; s < n_streams && e == cudaSuccess; s++)
      e = cudaMemcpy2DAsync(dst + s * fbytes, c->g.W, frames_host + s * stream_stride, row_pitch, c->g.W, c->g.H,
                            cudaMemcpyHostToDevice, st);
  }
  if (e != cudaSuccess) return cuda_status(e);
  return checked ? vf_process_checked(c, dst, fbytes, c->g.W, n_streams, stream)
                 : vf_process(c, dst, fbytes, c->g.W, n_streams, stream);
}

int vf_get_report(vf_ctx* c, int s, vf_report* out, void* stream)
{
  if (!c || !out || s < 0 || s >= c->S) return VF_ERR_ARG;
  double rp[16];
  int ctr[C_NCTR];
  cudaStream_t st = (cudaStream_t)stream;
  cudaMemcpyAsync(rp, c->b.report + (long long)s * 16, sizeof(rp), cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(ctr, c->b.ctr + (long long)s * C_NCTR, sizeof(ctr), cudaMemcpyDeviceToHost, st);
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_status(e);
  out->n_detected = (int32_t)rp[0]; out->n_propagated = (int32_t)rp[1]; out->n_total = (int32_t)rp[2];
  out->n_dropped = (int32_t)rp[3]; out->coverage = rp[4]; out->frame = (int64_t)rp[5];
  out->n_survivors = (int32_t)rp[6]; out->n_candidates = (int32_t)rp[7];
  if (ctr[C_ERR]) return VF_ERR_CAPACITY;
  return VF_OK;
}

int vf_get_totals(vf_ctx* c, int s, double* out4, void* stream)
{
  if (!c || !out4 || s < 0 || s >= c->S) return VF_ERR_ARG;
  double rp[16];
  cudaStream_t st = (cudaStream_t)stream;
  cudaMemcpyAsync(rp, c->b.report + (long long)s * 16, sizeof(rp), cudaMemcpyDeviceToHost, st);
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_status(e);
  for (int k = 0; k < 4; k++) out4[k] = rp[8 + k];
  return VF_OK;
}

int vf_get_features(vf_ctx* c, int s, vf_features* out, void* stream)
{
  if (!c || !out || s < 0 || s >= c->S) return VF_ERR_ARG;
  if (c->frames_done[s] == 0) { memset(out, 0, sizeof(*out)); return VF_OK; }
  int ctr[C_NCTR];
  cudaStream_t st = (cudaStream_t)stream;
  cudaMemcpyAsync(ctr, c->b.ctr + (long long)s * C_NCTR, sizeof(ctr), cudaMemcpyDeviceToHost, st);
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_status(e);
  const int buf = (int)((c->frames_done[s] - 1) & 1);
  out->n = ctr[C_NFEAT0 + buf];
  const long long o = ((long long)s * 2 + buf) * c->g.kp_cap + (c->g.kp_cap - out->n);   // lists end at the buffer end
  out->x = c->b.fx + o; out->y = c->b.fy + o; out->sigma = c->b.fs + o; out->theta = c->b.ft + o;
  out->score = c->b.fv + o; out->origin = c->b.forg + o; out->age = c->b.fage + o; out->desc = c->b.fdesc + o * 64;
  if (ctr[C_ERR]) return VF_ERR_CAPACITY;
  return VF_OK;
}

int vf_copy_features(vf_ctx* c, int s, int32_t cap, double* x, double* y, double* sigma, double* theta, double* score,
                     uint8_t* origin, int32_t* age, uint8_t* desc, int32_t* n_out, void* stream)
{
  vf_features f;
  int rc = vf_get_features(c, s, &f, stream);
  if (rc) return rc;
  if (n_out) *n_out = f.n;
  if (f.n > cap) return VF_ERR_CAPACITY;
  if (f.n == 0) return VF_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t n = (size_t)f.n;
  if (x) cudaMemcpyAsync(x, f.x, 8 * n, cudaMemcpyDeviceToHost, st);
  if (y) cudaMemcpyAsync(y, f.y, 8 * n, cudaMemcpyDeviceToHost, st);
  if (sigma) cudaMemcpyAsync(sigma, f.sigma, 8 * n, cudaMemcpyDeviceToHost, st);
  if (theta) cudaMemcpyAsync(theta, f.theta, 8 * n, cudaMemcpyDeviceToHost, st);
  if (score) cudaMemcpyAsync(score, f.score, 8 * n, cudaMemcpyDeviceToHost, st);
  if (origin) cudaMemcpyAsync(origin, f.origin, n, cudaMemcpyDeviceToHost, st);
  if (age) cudaMemcpyAsync(age, f.age, 4 * n, cudaMemcpyDeviceToHost, st);
  if (desc) cudaMemcpyAsync(desc, f.desc, 64 * n, cudaMemcpyDeviceToHost, st);
  return cuda_status(cudaStreamSynchronize(st));
}

int vf_fetch_features(vf_ctx* c, int n_streams, int64_t cap, double* x, double* y, double* sigma, double* theta,
                      double* score, uint8_t* origin, int32_t* age, uint8_t* desc, int32_t* offsets, void* stream)
{
  if (!c || n_streams < 1 || n_streams > c->S || !offsets) return VF_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  auto& P = c->pack;
  if (!P.pre) {
    if (cudaMalloc(&P.pre, sizeof(int) * (c->S + 1)) != cudaSuccess) return VF_ERR_CUDA;
    if (cudaMallocHost(&P.pre_host, sizeof(int) * (c->S + 1)) != cudaSuccess) return VF_ERR_CUDA;
  }
  // size the pack buffers from the current counts (grow only)
  std::vector<int> ctr((size_t)c->S * C_NCTR);
  cudaMemcpyAsync(ctr.data(), c->b.ctr, sizeof(int) * ctr.size(), cudaMemcpyDeviceToHost, st);
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_status(e);
  long long need = 0;
  for (int s = 0; s < n_streams; s++) {
    const int* cs = &ctr[(size_t)s * C_NCTR];
    if (cs[C_FRAME] > 0) need += cs[C_NFEAT0 + ((cs[C_FRAME] - 1) & 1)];
  }
  if (need > P.cap) {
    pack_free(c);
    const long long nc = std::max(need + need / 4, 65536LL);
    bool ok = cudaMalloc(&P.x, 8 * nc) == cudaSuccess && cudaMalloc(&P.y, 8 * nc) == cudaSuccess &&
              cudaMalloc(&P.s, 8 * nc) == cudaSuccess && cudaMalloc(&P.t, 8 * nc) == cudaSuccess &&
              cudaMalloc(&P.v, 8 * nc) == cudaSuccess && cudaMalloc(&P.o, nc) == cudaSuccess &&
              cudaMalloc(&P.a, 4 * nc) == cudaSuccess && cudaMalloc(&P.d, 64 * nc) == cudaSuccess;
    if (!ok) { pack_free(c); return VF_ERR_CUDA; }
    P.cap = nc;
  }
  k_pack<<<std::max(1, std::min(cdiv(need, 256), g_num_sms * 8)), 256, (n_streams + 1) * sizeof(int), st>>>(
      c->g, c->b, n_streams, -1, P.x, P.y, P.s, P.t, P.v, P.o, P.a, P.d, P.pre, P.cap, nullptr);
  cudaMemcpyAsync(P.pre_host, P.pre, sizeof(int) * (n_streams + 1), cudaMemcpyDeviceToHost, st);
  e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_status(e);
  const long long n = P.pre_host[n_streams];
  for (int s = 0; s <= n_streams; s++) offsets[s] = P.pre_host[s];
  if (n > cap) return VF_ERR_CAPACITY;
  if (n == 0) return VF_OK;
  if (x) cudaMemcpyAsync(x, P.x, 8 * n, cudaMemcpyDeviceToHost, st);
  if (y) cudaMemcpyAsync(y, P.y, 8 * n, cudaMemcpyDeviceToHost, st);
  if (sigma) cudaMemcpyAsync(sigma, P.s, 8 * n, cudaMemcpyDeviceToHost, st);
  if (theta) cudaMemcpyAsync(theta, P.t, 8 * n, cudaMemcpyDeviceToHost, st);
  if (score) cudaMemcpyAsync(score, P.v, 8 * n, cudaMemcpyDeviceToHost, st);
  if (origin) cudaMemcpyAsync(origin, P.o, n, cudaMemcpyDeviceToHost, st);
  if (age) cudaMemcpyAsync(age, P.a, 4 * n, cudaMemcpyDeviceToHost, st);
  if (desc) cudaMemcpyAsync(desc, P.d, 64 * n, cudaMemcpyDeviceToHost, st);
  return cuda_status(cudaGetLastError());
}

static int pipe_init(vf_ctx* c)
{
  auto& P = c->pipe;
  if (P.init) return VF_OK;
  const long long fb = (long long)c->g.W * c->g.H * c->S;
  P.frame_bytes = fb;
  P.cap = (long long)c->S * c->g.kp_cap;
  bool ok = true;
  ok = ok && cudaStreamCreateWithFlags(&P.h2d, cudaStreamNonBlocking) == cudaSuccess;
  ok = ok && cudaStreamCreateWithFlags(&P.comp, cudaStreamNonBlocking) == cudaSuccess;
  ok = ok && cudaStreamCreateWithFlags(&P.d2h, cudaStreamNonBlocking) == cudaSuccess;
  for (int k = 0; k < VF_PIPE_DEPTH && ok; k++) {
    ok = ok && cudaMalloc(&P.frames[k], fb) == cudaSuccess;
    ok = ok && cudaMalloc(&P.x[k], 8 * P.cap) == cudaSuccess && cudaMalloc(&P.y[k], 8 * P.cap) == cudaSuccess;
    ok = ok && cudaMalloc(&P.s[k], 8 * P.cap) == cudaSuccess && cudaMalloc(&P.t[k], 8 * P.cap) == cudaSuccess;
    ok = ok && cudaMalloc(&P.v[k], 8 * P.cap) == cudaSuccess && cudaMalloc(&P.o[k], P.cap) == cudaSuccess;
    ok = ok && cudaMalloc(&P.a[k], 4 * P.cap) == cudaSuccess && cudaMalloc(&P.d[k], 64 * P.cap) == cudaSuccess;
    // step meta data as one blob (one D2H per step): detected offsets [S + 1],
    // keep-word offsets [S + 1], counts [3 S], sticky error flags [S]
    const size_t mi = 2 * (size_t)(c->S + 1) + 4 * (size_t)c->S;
    ok = ok && cudaMalloc(&P.meta[k], sizeof(int) * mi) == cudaSuccess;
    ok = ok && cudaMallocHost(&P.meta_host[k], sizeof(int) * mi) == cudaSuccess;
    if (ok) {
      P.pre[k] = P.meta[k]; P.kpre[k] = P.meta[k] + (c->S + 1); P.cnt[k] = P.meta[k] + 2 * (c->S + 1);
      P.err[k] = P.cnt[k] + 3 * c->S;
      P.pre_host[k] = P.meta_host[k]; P.kpre_host[k] = P.meta_host[k] + (c->S + 1);
      P.cnt_host[k] = P.meta_host[k] + 2 * (c->S + 1); P.err_host[k] = P.cnt_host[k] + 3 * c->S;
      P.meta_ints = mi;
    }
    ok = ok && cudaEventCreateWithFlags(&P.ev_h2d[k], cudaEventDisableTiming) == cudaSuccess;
    ok = ok && cudaEventCreateWithFlags(&P.ev_comp[k], cudaEventDisableTiming) == cudaSuccess;
    ok = ok && cudaEventCreateWithFlags(&P.ev_pre[k], cudaEventDisableTiming) == cudaSuccess;
    ok = ok && cudaEventCreateWithFlags(&P.ev_d2h[k], cudaEventDisableTiming) == cudaSuccess;
    ok = ok && cudaMalloc(&P.kb[k], 4 * (size_t)c->S * c->b.keep_words) == cudaSuccess;
  }
  P.kcap = (long long)c->S * c->b.keep_words;
  if (!ok) return VF_ERR_CUDA;
  P.init = true;
  return VF_OK;
}

static void pipe_free(vf_ctx* c)
{
  auto& P = c->pipe;
  if (!P.init) return;
  cudaStreamSynchronize(P.h2d); cudaStreamSynchronize(P.comp); cudaStreamSynchronize(P.d2h);
  for (int k = 0; k < VF_PIPE_DEPTH; k++) {
    for (void* p : {(void*)P.frames[k], (void*)P.x[k], (void*)P.y[k], (void*)P.s[k], (void*)P.t[k], (void*)P.v[k],
                    (void*)P.o[k], (void*)P.a[k], (void*)P.d[k], (void*)P.meta[k]})
      cudaFree(p);
    cudaFreeHost(P.meta_host[k]);
    cudaFree(P.kb[k]);
    cudaEventDestroy(P.ev_h2d[k]); cudaEventDestroy(P.ev_comp[k]); cudaEventDestroy(P.ev_pre[k]);
    cudaEventDestroy(P.ev_d2h[k]);
  }
  cudaStreamDestroy(P.h2d); cudaStreamDestroy(P.comp); cudaStreamDestroy(P.d2h);
  P.init = false;
}

// One-launch delivery of packed fields to the caller's arrays (k_copy_out):
// possible when every destination is pinned host memory with a device address
// (or device memory).  Returns false when a plain cudaMemcpyAsync per field is
// needed instead (pageable destinations, results over 64 KB, VF_D2H_KERNEL=0).
struct OutField { void* dst; const void* src; long long bytes; };
static bool copy_out_kernel(const OutField* f, int nf, cudaStream_t st)
{
  static const bool off = getenv("VF_D2H_KERNEL") && atoi(getenv("VF_D2H_KERNEL")) == 0;
  if (off) return false;
  CopySegs cs;
  cs.n = 0;
  long long total = 0;
  for (int i = 0; i < nf; i++) {
    if (!f[i].dst || f[i].bytes <= 0) continue;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, f[i].dst) != cudaSuccess || !a.devicePointer ||
        (a.type != cudaMemoryTypeHost && a.type != cudaMemoryTypeDevice && a.type != cudaMemoryTypeManaged)) {
      cudaGetLastError();
      return false;
    }
    cs.seg[cs.n].src = (const uint8_t*)f[i].src;
    cs.seg[cs.n].dst = (uint8_t*)a.devicePointer;
    cs.seg[cs.n].bytes = f[i].bytes;
    cs.n++;
    total += f[i].bytes;
  }
  if (cs.n == 0) return true;
  // SM writes over PCIe only pay below the fixed cost of the DMA copies they
  // replace (config 1, 20 KB per step: 129 -> 99 us per pipelined step; config
  // 2, 318 KB: 128 -> 210 us): larger results go by cudaMemcpyAsync
  if (total > (64 << 10)) return false;
  const int blocks = (int)std::max(1LL, std::min<long long>(cdiv(total, 256 * 16), g_num_sms * 4));
  k_copy_out<<<blocks, 256, 0, st>>>(cs);
  return cudaGetLastError() == cudaSuccess;
}

int vf_pipeline_submit(vf_ctx* c, const uint8_t* frames_host, int64_t stream_stride, int64_t row_pitch, int n_streams)
{
  if (!c || !frames_host || n_streams < 1 || n_streams > c->S || row_pitch < c->g.W) return VF_ERR_ARG;
  if (!g_pattern_ok) return VF_ERR_PATTERN;
  int rc = pipe_init(c);
  if (rc) return rc;
  auto& P = c->pipe;
  if (P.submitted - P.collected >= VF_PIPE_DEPTH) return VF_ERR_ARG;   // collect the oldest step first
  const int k = (int)(P.submitted % VF_PIPE_DEPTH);
  const long long fbytes = (long long)c->g.W * c->g.H;
  // frames -> device (buffer k was last read by compute of step submitted - VF_PIPE_DEPTH: ev_comp[k])
  cudaStreamWaitEvent(P.h2d, P.ev_comp[k], 0);
  cudaError_t e = cudaSuccess;
  if (row_pitch == c->g.W && stream_stride == fbytes)
    e = cudaMemcpyAsync(P.frames[k], frames_host, fbytes * n_streams, cudaMemcpyHostToDevice, P.h2d);
  else
    for (int s = 0; s < n_streams && e == cudaSuccess; s++)
      e = cudaMemcpy2DAsync(P.frames[k] + s * fbytes, c->g.W, frames_host + s * stream_stride, row_pitch, c->g.W,
                            c->g.H, cudaMemcpyHostToDevice, P.h2d);
  if (e != cudaSuccess) return cuda_status(e);
  cudaEventRecord(P.ev_h2d[k], P.h2d);
  // the whole path, then pack (pack buffer k was last read by the d2h of step submitted - VF_PIPE_DEPTH)
  cudaStreamWaitEvent(P.comp, P.ev_h2d[k], 0);
  rc = vf_process(c, P.frames[k], fbytes, c->g.W, n_streams, P.comp);   // graph replay for small batches
  if (rc) return rc;
  cudaStreamWaitEvent(P.comp, P.ev_d2h[k], 0);
  if (P.delta) {
    k_pack_delta<<<g_num_sms * 8, 256, 2 * (n_streams + 1) * sizeof(int), P.comp>>>(
        c->g, c->b, n_streams, P.x[k], P.y[k], P.s[k], P.t[k], P.v[k], P.d[k], P.kb[k], P.pre[k], P.kpre[k],
        P.cnt[k], P.cap, P.kcap, P.err[k]);
  } else {
    k_pack<<<g_num_sms * 8, 256, (n_streams + 1) * sizeof(int), P.comp>>>(
        c->g, c->b, n_streams, -1, P.x[k], P.y[k], P.s[k], P.t[k], P.v[k], P.o[k], P.a[k], P.d[k], P.pre[k], P.cap,
        P.err[k]);
  }
  // offsets, counts and error flags of the step in one copy (each small D2H
  // costs the compute stream ~10 us)
  cudaMemcpyAsync(P.meta_host[k], P.meta[k], sizeof(int) * P.meta_ints, cudaMemcpyDeviceToHost, P.comp);
  cudaEventRecord(P.ev_pre[k], P.comp);
  cudaEventRecord(P.ev_comp[k], P.comp);
  P.n_streams[k] = n_streams;
  P.submitted++;
  return cuda_status(cudaGetLastError());
}

int vf_pipeline_collect(vf_ctx* c, int64_t cap, double* x, double* y, double* sigma, double* theta, double* score,
                        uint8_t* origin, int32_t* age, uint8_t* desc, int32_t* offsets)
{
  if (!c || !offsets) return VF_ERR_ARG;
  auto& P = c->pipe;
  if (!P.init || P.collected >= P.submitted) return VF_ERR_ARG;
  const int k = (int)(P.collected % VF_PIPE_DEPTH);
  cudaError_t e = cudaEventSynchronize(P.ev_pre[k]);
  if (e != cudaSuccess) return cuda_status(e);
  const int ns = P.n_streams[k];
  const long long n = std::min((long long)P.pre_host[k][ns], P.cap);
  for (int s = 0; s <= ns; s++) offsets[s] = P.pre_host[k][s];
  if (n > cap) return VF_ERR_CAPACITY;
  cudaStreamWaitEvent(P.d2h, P.ev_comp[k], 0);
  if (n > 0) {
    const OutField f[8] = {{x, P.x[k], 8 * n}, {y, P.y[k], 8 * n}, {sigma, P.s[k], 8 * n}, {theta, P.t[k], 8 * n},
                           {score, P.v[k], 8 * n}, {origin, P.o[k], n}, {age, P.a[k], 4 * n}, {desc, P.d[k], 64 * n}};
    if (!copy_out_kernel(f, 8, P.d2h))
      for (const OutField& o : f)
        if (o.dst) cudaMemcpyAsync(o.dst, o.src, o.bytes, cudaMemcpyDeviceToHost, P.d2h);
  }
  cudaEventRecord(P.ev_d2h[k], P.d2h);
  e = cudaEventSynchronize(P.ev_d2h[k]);
  if (e != cudaSuccess) return cuda_status(e);
  P.collected++;
  for (int s = 0; s < ns; s++)   // sticky device capacity flags of this step
    if (P.err_host[k][s]) return VF_ERR_CAPACITY;
  return VF_OK;
}

int vf_pipeline_set_delta(vf_ctx* c, int enable)
{
  if (!c) return VF_ERR_ARG;
  if (c->pipe.submitted != c->pipe.collected) return VF_ERR_ARG;   // only between steps
  const bool on = enable != 0;
  if (on && !c->b.keep_bits) {
    const int kw = cdiv(c->g.kp_cap, 32) + 1;
    uint32_t* kb = c->mem.get<uint32_t>((size_t)c->S * kw);
    if (!kb) return cuda_status(c->mem.err);
    c->b.keep_bits = kb;
    c->b.keep_words = kw;
    pipe_free(c);                                   // re-created with keep-mask buffers
    graph_drop(c);
  }
  c->pipe.delta = on;
  return VF_OK;
}

int vf_pipeline_collect_delta(vf_ctx* c, int64_t cap, double* x, double* y, double* sigma, double* theta,
                              double* score, uint8_t* desc, int32_t* det_offsets, int64_t kcap, uint32_t* keep_bits,
                              int32_t* keep_offsets, int32_t* counts)
{
  if (!c || !det_offsets || !keep_offsets || !counts) return VF_ERR_ARG;
  auto& P = c->pipe;
  if (!P.init || !P.delta || P.collected >= P.submitted) return VF_ERR_ARG;
  const int k = (int)(P.collected % VF_PIPE_DEPTH);
  cudaError_t e = cudaEventSynchronize(P.ev_pre[k]);
  if (e != cudaSuccess) return cuda_status(e);
  const int ns = P.n_streams[k];
  const long long n = std::min((long long)P.pre_host[k][ns], P.cap);
  const long long nw = std::min((long long)P.kpre_host[k][ns], P.kcap);
  for (int s = 0; s <= ns; s++) { det_offsets[s] = P.pre_host[k][s]; keep_offsets[s] = P.kpre_host[k][s]; }
  for (int i = 0; i < 3 * ns; i++) counts[i] = P.cnt_host[k][i];
  if (n > cap || nw > kcap) return VF_ERR_CAPACITY;
  cudaStreamWaitEvent(P.d2h, P.ev_comp[k], 0);
  {
    const OutField f[7] = {{x, P.x[k], 8 * n}, {y, P.y[k], 8 * n}, {sigma, P.s[k], 8 * n}, {theta, P.t[k], 8 * n},
                           {score, P.v[k], 8 * n}, {desc, P.d[k], 64 * n}, {keep_bits, P.kb[k], 4 * nw}};
    if (!copy_out_kernel(f, 7, P.d2h))
      for (const OutField& o : f)
        if (o.dst && o.bytes > 0) cudaMemcpyAsync(o.dst, o.src, o.bytes, cudaMemcpyDeviceToHost, P.d2h);
  }
  cudaEventRecord(P.ev_d2h[k], P.d2h);
  e = cudaEventSynchronize(P.ev_d2h[k]);
  if (e != cudaSuccess) return cuda_status(e);
  P.collected++;
  for (int s = 0; s < ns; s++)
    if (P.err_host[k][s]) return VF_ERR_CAPACITY;
  return VF_OK;
}

int vf_delta_apply(int32_t n_prev, const double* prev_x, const double* prev_y, const double* prev_sigma,
                   const double* prev_theta, const double* prev_score, const uint8_t* prev_origin,
                   const int32_t* prev_age, const uint8_t* prev_desc, int32_t n_det, const double* det_x,
                   const double* det_y, const double* det_sigma, const double* det_theta, const double* det_score,
                   const uint8_t* det_desc, int32_t n_keep_bits, const uint32_t* keep_bits, int32_t out_cap,
                   double* x, double* y, double* sigma, double* theta, double* score, uint8_t* origin, int32_t* age,
                   uint8_t* desc, int32_t* n_out)
{
  if (!n_out || n_prev < 0 || n_det < 0 || n_keep_bits < 0 || n_keep_bits > n_prev) return VF_ERR_ARG;
  long long n = n_det;
  for (int w = 0; w < (n_keep_bits + 31) / 32; w++) n += __builtin_popcount(keep_bits[w]);
  *n_out = (int32_t)n;
  if (n > out_cap) return VF_ERR_CAPACITY;
  // masking.py:176-183: the detected features (origin detected, age 0), then
  // the kept previous features in their previous order (propagated, age + 1)
  if (n_det) {
    memcpy(x, det_x, 8 * (size_t)n_det); memcpy(y, det_y, 8 * (size_t)n_det);
    memcpy(sigma, det_sigma, 8 * (size_t)n_det); memcpy(theta, det_theta, 8 * (size_t)n_det);
    memcpy(score, det_score, 8 * (size_t)n_det); memcpy(desc, det_desc, 64 * (size_t)n_det);
    memset(origin, 0, (size_t)n_det);
    memset(age, 0, 4 * (size_t)n_det);
  }
  long long o = n_det;
  for (int i = 0; i < n_keep_bits; i++) {
    if (!((keep_bits[i >> 5] >> (i & 31)) & 1u)) continue;
    x[o] = prev_x[i]; y[o] = prev_y[i]; sigma[o] = prev_sigma[i]; theta[o] = prev_theta[i]; score[o] = prev_score[i];
    origin[o] = 1; age[o] = prev_age[i] + 1;
    memcpy(desc + 64 * o, prev_desc + 64 * (size_t)i, 64);
    o++;
  }
  (void)prev_origin;
  return VF_OK;
}

int vf_get_diag(vf_ctx* c, int64_t* out8, void* stream)
{
  if (!c || !out8) return VF_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  std::vector<int> wcs(c->S), sc(c->S), ctr((size_t)c->S * C_NCTR);
  cudaMemcpyAsync(wcs.data(), c->b.work_count, sizeof(int) * c->S, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(sc.data(), c->b.sat_count, sizeof(int) * c->S, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(ctr.data(), c->b.ctr, sizeof(int) * ctr.size(), cudaMemcpyDeviceToHost, st);
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_status(e);
  long long sat = 0, dense = 0, stage = 0;
  for (int s = 0; s < c->S; s++) {
    // frame counter already advanced: the last step was masked iff frame >= 2 (or mode none => dense)
    const bool masked = (c->g.mask_mode == 1 || c->g.mask_mode == 2) && ctr[(size_t)s * C_NCTR + C_FRAME] >= 2;
    if (masked) sat += sc[s]; else { sat += c->g.sat_tiles; dense++; }
    stage += ctr[(size_t)s * C_NCTR + C_STAGE];
  }
  long long wc = 0;
  for (int v : wcs) wc += v;
  out8[0] = wc;                                   // active FAST tiles (all streams)
  out8[1] = (long long)c->g.tiles_per_stream * c->S;  // FAST tiles in total
  out8[2] = sat;                                  // SAT tiles built
  out8[3] = (long long)c->g.sat_tiles * c->S;     // SAT tiles in total
  out8[4] = dense;                                // streams whose last frame was unmasked
  out8[5] = stage;                                // NMS candidates staged
  out8[6] = c->g.bands_per_stream;
  out8[7] = c->g.kp_cap;
  return VF_OK;
}

int vf_get_layer(vf_ctx* c, int s, int l, const uint8_t** ptr, int32_t* pitch)
{
  if (!c || s < 0 || s >= c->S || l < 1 || l >= c->g.NL || !ptr) return VF_ERR_ARG;
  *ptr = c->b.layers + (long long)s * c->g.layer_slab + c->g.L[l].layer_off;
  if (pitch) *pitch = c->g.L[l].pitch;
  return VF_OK;
}

// ---------------------------------------------------------------------------
// per-stage drop-ins
// ---------------------------------------------------------------------------
namespace {
struct Scratch {          // transient context for a stand-alone stage call
  vf_ctx* c = nullptr;
  ~Scratch() { if (c) vf_destroy(c); }
};

int stage_ctx(int W, int H, int O, int threshold, int kp_cap, Scratch& sc)
{
  vf_config cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.width = W; cfg.height = H; cfg.n_octaves = O; cfg.threshold = threshold < 1 ? 1 : threshold;
  cfg.mask_mode = 0; cfg.t_i = 20.0; cfg.t_h = 1; cfg.grid_rows = 16; cfg.grid_cols = 16;
  cfg.octave_for_mask = -1; cfg.max_streams = 1; cfg.kp_capacity = kp_cap;
  return vf_create(&cfg, &sc.c);
}
}  // namespace

int vf_build_pyramid(const uint8_t* frame_dev, int W, int H, int64_t pitch, int n_octaves, uint8_t* const* layers_dev,
                     const int64_t* pitches, void* stream)
{
  if (!frame_dev || !layers_dev || !pitches || pitch < W) return VF_ERR_ARG;
  Scratch sc;
  int rc = stage_ctx(W, H, n_octaves, 1, 4096, sc);
  if (rc) return rc;
  vf_ctx* c = sc.c;
  cudaStream_t st = (cudaStream_t)stream;
  Bufs b = c->b;
  b.frames = frame_dev; b.frame_stride = 0; b.frame_pitch = pitch;
  k_pyramid<<<dim3(c->g.ptx, c->g.pty, 1), 256, c->pyr_smem, st>>>(c->g, b);
  for (int l = 1; l < c->g.NL; l++) {
    const LayerGeo& L = c->g.L[l];
    cudaMemcpy2DAsync(layers_dev[l], pitches[l], b.layers + L.layer_off, L.pitch, L.w, L.h, cudaMemcpyDeviceToDevice, st);
  }
  return cuda_status(cudaStreamSynchronize(st));
}

int vf_score_map(const uint8_t* layer_dev, int w, int h, int64_t pitch, int t, const uint8_t* mask_dev, int mw, int mh,
                 uint8_t* scores_dev, int64_t scores_pitch, void* stream)
{
  if (t < 1) return VF_ERR_THRESHOLD;
  if (!layer_dev || !scores_dev || w < 1 || h < 1 || pitch < w || scores_pitch < w) return VF_ERR_ARG;
  // One layer treated as "o0" of a single-octave geometry; the gate is the
  // caller's full-res mask as a 1x1-cell grid (detector.py:175-181).
  vf_ctx* c = new vf_ctx();
  Geo& g = c->g;
  memset(&g, 0, sizeof(g));
  g.W = mask_dev ? mw : w; g.H = mask_dev ? mh : h; g.O = 1; g.NL = 1; g.threshold = t;
  LayerGeo& L = g.L[0];
  L.w = w; L.h = h; L.pitch = (int)align_up(w, 16); L.scale = 1.0; L.sigma = 1.0;
  L.rinv_h = 1.0 / h; L.rinv_w = 1.0 / w;
  L.tiles_x = cdiv(w, VF_TILE_W); L.tiles_y = cdiv(h, VF_TILE_H); L.bm_words = cdiv(w, 32);
  g.tiles_per_stream = L.tiles_x * L.tiles_y; g.bands_per_stream = L.tiles_y; g.rows_per_stream = h;
  g.sm_slab = align_up((long long)L.pitch * h + 16, 256); g.bm_slab_words = (long long)L.bm_words * h;
  std::vector<int> lut;
  if (mask_dev) {
    g.mask_mode = 1; g.n_grids = 1;
    g.grid[0].rows = mh; g.grid[0].cols = mw; g.grid[0].cw = 1; g.grid[0].ch = 1; g.grid[0].cell_off = 0;
    for (int y = 0; y < h; y++) lut.push_back((int)((long long)y * mh / h));
    for (int x = 0; x < w; x++) lut.push_back((int)((long long)x * mw / w));
  } else {
    lut.assign(h + w, 0);
  }
  L.rc_off = 0; L.cc_off = h;
  Alloc& A = c->mem;
  Bufs& b = c->b;
  memset(&b, 0, sizeof(b));
  b.frames = layer_dev; b.frame_pitch = pitch; b.frame_stride = 0;
  b.scores = A.get<uint8_t>(g.sm_slab);
  b.bitmaps = A.get<uint32_t>(g.bm_slab_words);
  b.tile_stamp = A.get<int>(g.tiles_per_stream);
  b.band_stamp = A.get<int>(g.bands_per_stream);
  b.band_cand = A.get<int>(g.bands_per_stream);
  int* dl = A.get<int>(lut.size());
  b.lut = dl;
  b.cells = const_cast<uint8_t*>(mask_dev);
  b.ctr = A.get<int>(C_NCTR);
  b.worklist = A.get<int>(g.tiles_per_stream);
  b.work_count = A.get<int>(1);
  if (A.err != cudaSuccess) { int r = cuda_status(A.err); A.release(); delete c; return r; }
  cudaStream_t st = (cudaStream_t)stream;
  std::vector<int> wl(g.tiles_per_stream);
  for (int i = 0; i < g.tiles_per_stream; i++) wl[i] = i;
  int nwl = g.tiles_per_stream;
  int frame1[C_NCTR] = {0};
  frame1[C_FRAME] = mask_dev ? 1 : 0;    // use_mask() on when a mask is given
  cudaMemcpyAsync(dl, lut.data(), sizeof(int) * lut.size(), cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(b.worklist, wl.data(), sizeof(int) * nwl, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(b.work_count, &nwl, sizeof(int), cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(b.ctr, frame1, sizeof(frame1), cudaMemcpyHostToDevice, st);
  cudaFuncSetAttribute(k_fast, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(FastWarp) * FAST_WARPS + 8);
  k_fast<<<std::max(1, std::min(cdiv(nwl, FAST_WARPS), 148 * 8)), 32 * FAST_WARPS, sizeof(FastWarp) * FAST_WARPS + 8, st>>>(
      g, b, 1);
  cudaMemcpy2DAsync(scores_dev, scores_pitch, b.scores, L.pitch, w, h, cudaMemcpyDeviceToDevice, st);
  int rc = cuda_status(cudaStreamSynchronize(st));
  A.release();
  delete c;
  return rc;
}

__global__ void k_gather_kps(const __grid_constant__ Geo g, const __grid_constant__ Bufs b, double* x, double* y,
                             double* s, double* v, int cap)
{
  const int rid = blockIdx.x;
  const int* rec = b.unit_rec + rid * 4;
  const int kept = rec[1], base = rec[0], o = b.unit_out[rid];
  for (int i = threadIdx.x; i < kept; i += blockDim.x) {
    if (o + i >= cap) break;
    x[o + i] = b.st_x[base + i]; y[o + i] = b.st_y[base + i]; s[o + i] = b.st_s[base + i]; v[o + i] = b.st_v[base + i];
  }
}

int vf_nms_refine(const uint8_t* const* maps_dev, const int64_t* pitches, int W, int H, int n_octaves, int32_t cap,
                  double* x_dev, double* y_dev, double* sigma_dev, double* score_dev, int32_t* n_out, void* stream)
{
  if (!maps_dev || !pitches || !n_out) return VF_ERR_ARG;
  Scratch sc;
  int rc = stage_ctx(W, H, n_octaves, 1, std::max(cap, 1024), sc);
  if (rc) return rc;
  vf_ctx* c = sc.c;
  Geo g = c->g;
  g.nms_raw = 1; g.nms_wrap = 1;
  g.prop_chunks = 0;
  Bufs b = c->b;
  cudaStream_t st = (cudaStream_t)stream;
  for (int l = 0; l < g.NL; l++)
    cudaMemcpy2DAsync(b.scores + g.L[l].sm_off, g.L[l].pitch, maps_dev[l], pitches[l], g.L[l].w, g.L[l].h,
                      cudaMemcpyDeviceToDevice, st);
  k_bitmap_from_maps<<<dim3(64, g.NL), 256, 0, st>>>(g, b);
  // every tile / band active at epoch 1 (frame 0: no gating)
  std::vector<int> ones(std::max(g.tiles_per_stream, g.bands_per_stream), 1);
  cudaMemcpyAsync(b.tile_stamp, ones.data(), sizeof(int) * g.tiles_per_stream, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(b.band_stamp, ones.data(), sizeof(int) * g.bands_per_stream, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(b.band_cand, ones.data(), sizeof(int) * g.bands_per_stream, cudaMemcpyHostToDevice, st);
  b.nms_u = VF_TILE_H;
  k_nms<<<dim3(cdiv((long long)g.bands_per_stream * b.nms_u, NMS_WARPS), 1), NMS_THREADS, 0, st>>>(g, b);
  k_nms_finish<<<1, NF_THREADS, 0, st>>>(g, b);
  k_gather_kps<<<g.bands_per_stream * b.nms_u, 128, 0, st>>>(g, b, x_dev, y_dev, sigma_dev, score_dev, cap);
  int ctr[C_NCTR];
  cudaMemcpyAsync(ctr, b.ctr, sizeof(ctr), cudaMemcpyDeviceToHost, st);
  rc = cuda_status(cudaStreamSynchronize(st));
  if (rc) return rc;
  *n_out = ctr[C_NDET];
  if (ctr[C_ERR] || ctr[C_NDET] > cap) return VF_ERR_CAPACITY;
  return VF_OK;
}

int vf_describe(const uint8_t* frame_dev, int W, int H, int64_t pitch, int n, const double* kx_dev,
                const double* ky_dev, const double* sigma_dev, const double* theta_in_dev, double* theta_out_dev,
                uint8_t* desc_dev, void* stream)
{
  if (!g_pattern_ok) return VF_ERR_PATTERN;
  if (!frame_dev || n < 0 || pitch < W) return VF_ERR_ARG;
  if (n == 0) return VF_OK;
  // SAT tiles of the frame through k_pyramid with one octave (no derived layers)
  Scratch sc;
  int rc = stage_ctx(W, H, 1, 1, 4096, sc);
  if (rc) return rc;
  vf_ctx* c = sc.c;
  cudaStream_t st = (cudaStream_t)stream;
  Bufs b = c->b;
  b.frames = frame_dev; b.frame_stride = 0; b.frame_pitch = pitch;
  k_pyramid<<<dim3(c->g.ptx, c->g.pty, 1), 256, c->pyr_smem, st>>>(c->g, b);
  k_carries<<<dim3(c->g.sty, 1), 32, 0, st>>>(c->g, b);
  int ctr0[C_NCTR] = {0};
  ctr0[C_NDET] = n;              // k_sat builds every tile of a stream with keypoints (unmasked)
  ctr0[C_NTOTAL] = n;            // the describe kernels write the n outputs as a full list
  cudaMemcpyAsync(b.ctr, ctr0, sizeof(ctr0), cudaMemcpyHostToDevice, st);
  k_sat<<<c->sat_grid, 256, c->sat_smem, st>>>(c->g, b, 1, 1);   // stream 0 -> slot 0, every tile
  k_describe_batch<<<cdiv(n, DS_THREADS), DS_THREADS, 0, st>>>(c->g, b.sat, n, kx_dev, ky_dev, sigma_dev,
                                                              theta_in_dev, theta_out_dev, desc_dev);
  return cuda_status(cudaStreamSynchronize(st));
}

int vf_intensity_mask(const uint8_t* prev_dev, const uint8_t* cur_dev, int64_t n, double t_i, uint8_t* out_dev,
                      void* stream)
{
  if (n < 0 || (n > 0 && (!prev_dev || !cur_dev || !out_dev))) return VF_ERR_ARG;
  if (n == 0) return VF_OK;
  k_intensity_mask<<<std::min(cdiv(n, 256), 4096), 256, 0, (cudaStream_t)stream>>>(prev_dev, cur_dev, n, t_i, out_dev);
  return cuda_status(cudaGetLastError());
}

int vf_ast_corner_score(const uint8_t* layer_dev, int w, int h, int64_t pitch, int n, const int32_t* xs_dev,
                        const int32_t* ys_dev, int arc_len, int32_t* out_dev, void* stream)
{
  if (arc_len < 1) return VF_ERR_ARG;   // the reference's min over an empty arc raises
  if (n < 0 || w < 7 || h < 7 || pitch < w) return VF_ERR_ARG;
  if (n == 0) return VF_OK;
  if (!layer_dev || !xs_dev || !ys_dev || !out_dev) return VF_ERR_ARG;
  k_ast_score<<<cdiv(n, 128), 128, 0, (cudaStream_t)stream>>>(layer_dev, pitch, n, xs_dev, ys_dev, arc_len, out_dev);
  return cuda_status(cudaGetLastError());
}

int vf_sad_block(const uint8_t* a_dev, const uint8_t* b_dev, int64_t patch_bytes, int count, int64_t* out_dev,
                 void* stream)
{
  if (patch_bytes < 0 || count < 0) return VF_ERR_ARG;
  if (count == 0) return VF_OK;
  if (!a_dev || !b_dev || !out_dev) return VF_ERR_ARG;
  k_sad_block<<<count, 256, 0, (cudaStream_t)stream>>>(a_dev, b_dev, patch_bytes, count, (long long*)out_dev);
  return cuda_status(cudaGetLastError());
}

int vf_binning_histogram(int n, const double* xs_dev, const double* ys_dev, int W, int H, int rows, int cols,
                         uint64_t* hist_dev, void* stream)
{
  if (rows < 1 || cols < 1) return VF_ERR_GRID;
  if (!hist_dev || n < 0) return VF_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  cudaMemsetAsync(hist_dev, 0, sizeof(uint64_t) * rows * cols, st);
  if (n > 0)
    k_binning_hist<<<std::min(cdiv(n, 256), 1024), 256, 0, st>>>(n, xs_dev, ys_dev, W, H, rows, cols,
                                                                  (unsigned long long*)hist_dev);
  return cuda_status(cudaGetLastError());
}

int vf_upsample_mask(const uint8_t* bits_dev, int rows, int cols, int cell_w, int cell_h, int W, int H, uint8_t* full_dev,
                     void* stream)
{
  if (!bits_dev || !full_dev || rows < 1 || cols < 1 || cell_w < 1 || cell_h < 1) return VF_ERR_ARG;
  if ((long long)cell_w * cols < W || (long long)cell_h * rows < H) return VF_ERR_ARG;
  k_upsample<<<std::min(cdiv((long long)W * H, 256), 4096), 256, 0, (cudaStream_t)stream>>>(bits_dev, cols, cell_w,
                                                                                            cell_h, W, H, full_dev);
  return cuda_status(cudaGetLastError());
}

int vf_mask_values(const uint8_t* full_dev, int W, int H, int n, const double* xs_dev, const double* ys_dev,
                   uint8_t* out_dev, void* stream)
{
  if (n < 0) return VF_ERR_ARG;
  if (n == 0) return VF_OK;
  k_mask_values<<<std::min(cdiv(n, 256), 1024), 256, 0, (cudaStream_t)stream>>>(full_dev, W, H, n, xs_dev, ys_dev,
                                                                                 out_dev);
  return cuda_status(cudaGetLastError());
}

}  // extern "C"
