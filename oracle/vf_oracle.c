/*
 * vf_oracle.c -- CPU restatement of the reference `vidfeat` per-frame hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * product path (and the `cpu_baseline` / `--impl reference` arm of bench.py,
 * kind "port").  Only tests/, __graft_entry__.smoke() and bench.py may load
 * it.  The product (paper_1503_06959_b200/) never links or calls it.
 *
 * Parity pin: this restatement is checked against golden vectors produced by
 * running the reference itself (tests/golden/make_golden.py imports
 * /root/reference/pkg/src/vidfeat and commits the tests/golden fixtures); see
 * tests/test_oracle_golden.py.
 *
 * Numerics follow the reference exactly: integer stages are bit-exact; fp64
 * stages use the same operation order, no FMA contraction
 * (-ffp-contract=off), and glibc cos/sin/atan2/pow (numba lowers to libm).
 *
 * Every function cites the reference file:line it restates.  Paths are
 * relative to /root/reference/pkg/src/vidfeat/.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define VFO_MAX_LAYERS 32

/* ------------------------------------------------------------------ */
/* pyramid.py:97-125 -- layer geometry.  Order o0, i0, o1, i1, ...     */
/* ------------------------------------------------------------------ */
int vfo_layer_dims(int W, int H, int O, int *ws, int *hs, double *scales)
{
    if (O < 1) return -1;                              /* pyramid.py:103-104 */
    int need = 1 << (O - 1);
    if (W < need || H < need) return -2;               /* pyramid.py:105-109 */
    int ow = W, oh = H;
    int iw = (2 * W) / 3, ih = (2 * H) / 3;            /* pyramid.py:82 m=(2n)//3 */
    if (iw < 1 || ih < 1) return -3;
    for (int o = 0; o < O; o++) {
        if (o > 0) {
            ow /= 2; oh /= 2; iw /= 2; ih /= 2;        /* pyramid.py:69 */
            if (ow < 1 || oh < 1 || iw < 1 || ih < 1) return -3;
        }
        ws[2 * o] = ow; hs[2 * o] = oh;
        ws[2 * o + 1] = iw; hs[2 * o + 1] = ih;
        if (scales) {
            double sc = ldexp(1.0, -o);                /* 2.0 ** (-o) */
            scales[2 * o] = sc;
            scales[2 * o + 1] = sc / 1.5;              /* pyramid.py:123 */
        }
    }
    return 0;
}

/* pyramid.py:67-73: 2x2 uint16 sum, (s+2)>>2, odd trailing dropped */
void vfo_halve(const uint8_t *a, int w, int h, uint8_t *out)
{
    int w2 = w / 2, h2 = h / 2;
    for (int y = 0; y < h2; y++)
        for (int x = 0; x < w2; x++) {
            unsigned s = a[(2 * y) * w + 2 * x] + a[(2 * y) * w + 2 * x + 1] +
                         a[(2 * y + 1) * w + 2 * x] + a[(2 * y + 1) * w + 2 * x + 1];
            out[y * w2 + x] = (uint8_t)((s + 2) >> 2);
        }
}

/* pyramid.py:76-94: per-axis (2a+b | a+2b) pair sums, then (v+4)//9 */
void vfo_two_thirds(const uint8_t *a, int w, int h, uint8_t *out)
{
    int mw = (2 * w) / 3, mh = (2 * h) / 3;
    uint32_t *rows = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)mh * w);
    for (int j = 0; j < mh; j++) {                     /* axis 0 first (:94) */
        int k = j / 2;
        for (int x = 0; x < w; x++) {
            uint32_t v;
            if ((j & 1) == 0) v = 2u * a[(3 * k) * w + x] + a[(3 * k + 1) * w + x];
            else v = a[(3 * k + 1) * w + x] + 2u * a[(3 * k + 2) * w + x];
            rows[(size_t)j * w + x] = v;
        }
    }
    for (int y = 0; y < mh; y++)
        for (int i = 0; i < mw; i++) {
            int k = i / 2;
            const uint32_t *r = rows + (size_t)y * w;
            uint32_t v = (i & 1) == 0 ? 2u * r[3 * k] + r[3 * k + 1] : r[3 * k + 1] + 2u * r[3 * k + 2];
            out[y * mw + i] = (uint8_t)((v + 4) / 9);
        }
    free(rows);
}

/* pyramid.py:111-125.  layers[l] must hold ws[l]*hs[l] bytes (layer 0 is a copy). */
int vfo_build_pyramid(const uint8_t *frame, int W, int H, int O, uint8_t **layers)
{
    int ws[VFO_MAX_LAYERS], hs[VFO_MAX_LAYERS];
    if (O > VFO_MAX_LAYERS / 2) return -1;
    int rc = vfo_layer_dims(W, H, O, ws, hs, NULL);
    if (rc) return rc;
    memcpy(layers[0], frame, (size_t)W * H);
    for (int o = 1; o < O; o++) vfo_halve(layers[2 * (o - 1)], ws[2 * (o - 1)], hs[2 * (o - 1)], layers[2 * o]);
    vfo_two_thirds(frame, W, H, layers[1]);
    for (int o = 1; o < O; o++)
        vfo_halve(layers[2 * (o - 1) + 1], ws[2 * (o - 1) + 1], hs[2 * (o - 1) + 1], layers[2 * o + 1]);
    return 0;
}

/* ------------------------------------------------------------------ */
/* detector.py:20-28 CIRCLE; detector.py:107-158 _score_map_jit          */
/* ------------------------------------------------------------------ */
static const int CX[16] = {0, 1, 2, 3, 3, 3, 2, 1, 0, -1, -2, -3, -3, -3, -2, -1};
static const int CY[16] = {-3, -3, -2, -1, 0, 1, 2, 3, 3, 3, 2, 1, 0, -1, -2, -3};

/* mask may be NULL (all ones); it is the per-layer projected mask (h x w). */
void vfo_score_map(const uint8_t *data, int w, int h, int t, const uint8_t *mask, int32_t *scores)
{
    memset(scores, 0, sizeof(int32_t) * (size_t)w * h);
    for (int y = 3; y < h - 3; y++)
        for (int x = 3; x < w - 3; x++) {
            if (mask && mask[(size_t)y * w + x] == 0) continue;       /* :114-115 */
            int64_t c = data[(size_t)y * w + x];
            int64_t d0 = (int64_t)data[(size_t)(y - 3) * w + x] - c;
            int64_t d8 = (int64_t)data[(size_t)(y + 3) * w + x] - c;
            int64_t d4 = (int64_t)data[(size_t)y * w + x + 3] - c;
            int64_t d12 = (int64_t)data[(size_t)y * w + x - 3] - c;
            int bright_ok = (d0 > t || d8 > t) && (d4 > t || d12 > t);  /* :121-123 */
            int dark_ok = (d0 < -t || d8 < -t) && (d4 < -t || d12 < -t);
            if (!(bright_ok || dark_ok)) continue;
            int64_t d[16];
            for (int k = 0; k < 16; k++) d[k] = (int64_t)data[(size_t)(y + CY[k]) * w + x + CX[k]] - c;
            int64_t best = 0;
            for (int pol = 0; pol < 2; pol++) {           /* :128-154 */
                if (pol == 0 && !bright_ok) continue;
                if (pol == 1 && !dark_ok) continue;
                int64_t sg = pol == 0 ? 1 : -1;
                for (int s0 = 0; s0 < 16; s0++) {
                    int64_t m = sg * d[s0];
                    if (m <= best) continue;
                    for (int k = 1; k < 9; k++) {
                        int64_t v = sg * d[(s0 + k) & 15];
                        if (v < m) { m = v; if (m <= best) break; }
                    }
                    if (m > best) best = m;
                }
            }
            int64_t score = best - 1;                     /* :155-157 */
            if (score >= t) scores[(size_t)y * w + x] = (int32_t)score;
        }
}

/* detector.py:175-181 _project_mask: floor mapping of a full-res mask */
void vfo_project_mask(const uint8_t *bits, int mw, int mh, int w, int h, uint8_t *out)
{
    for (int y = 0; y < h; y++) {
        int64_t yy = ((int64_t)y * mh) / h;
        for (int x = 0; x < w; x++) {
            int64_t xx = ((int64_t)x * mw) / w;
            out[(size_t)y * w + x] = bits[yy * mw + xx];
        }
    }
}

/* ------------------------------------------------------------------ */
/* detector.py:207-228 _fit_quadratic_peak (one patch, same op order)    */
/* ------------------------------------------------------------------ */
static void fit_peak(const double p[3][3], double *ox, double *oy, double *val, int *okp)
{
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
    *val = p[1][1] + 0.5 * (gx * x + gy * y);
    *ox = x; *oy = y; *okp = ok;
}

/* detector.py:231-236 _gather_patches on the 1-pixel zero-padded map */
static void gather(const int32_t *m, int w, int h, int y, int x, double p[3][3], int32_t *pmax)
{
    int32_t mx = INT32_MIN;
    for (int dy = -1; dy <= 1; dy++)
        for (int dx = -1; dx <= 1; dx++) {
            int yy = y + dy, xx = x + dx;
            int32_t v = (yy >= 0 && yy < h && xx >= 0 && xx < w) ? m[(size_t)yy * w + xx] : 0;
            p[dy + 1][dx + 1] = (double)v;
            if (v > mx) mx = v;
        }
    if (pmax) *pmax = mx;
}

/* numpy negative-index wrap for smap[ys+dy, xs+dx] (detector.py:260-262) */
static int wrap_get(const int32_t *m, int w, int h, int y, int x, int32_t *v)
{
    if (y >= h || x >= w) return -1;   /* numpy IndexError */
    if (y < 0) y += h;
    if (x < 0) x += w;
    *v = m[(size_t)y * w + x];
    return 0;
}

/*
 * detector.py:239-307 _nms_from_maps.  maps[i] is an int32 (hs[i] x ws[i]) map.
 * Output arrays must hold `cap` entries; returns the keypoint count, -1 on
 * overflow, -2 on an IndexError the reference would raise.
 * layer_out / xi_out / yi_out (nullable) give the integer origin (diagnostics).
 */
int vfo_nms(const int32_t *const *maps, const int *ws, const int *hs, const double *scales,
            int n_layers, int W, int H, int cap, double *kx, double *ky, double *ksig,
            double *kscore, int32_t *layer_out, int32_t *xi_out, int32_t *yi_out)
{
    double sigmas[VFO_MAX_LAYERS];
    for (int i = 0; i < n_layers; i++) sigmas[i] = 1.0 / scales[i];   /* :243 */
    int n = 0;
    for (int i = 0; i < n_layers; i++) {
        const int32_t *sm = maps[i];
        int w = ws[i], h = hs[i];
        for (int y = 0; y < h; y++)
            for (int x = 0; x < w; x++) {
                int32_t s = sm[(size_t)y * w + x];
                if (s == 0) continue;                                     /* :251 nonzero */
                int keep = 1;
                for (int dy = -1; dy <= 1; dy++)
                    for (int dx = -1; dx <= 1; dx++) {
                        if (dx == 0 && dy == 0) continue;
                        int32_t v;
                        if (wrap_get(sm, w, h, y + dy, x + dx, &v)) return -2;
                        if (!(s > v)) keep = 0;
                    }
                int yj[2], xj[2], have[2] = {0, 0};
                for (int k = 0; k < 2; k++) {                             /* :266-273 */
                    int j = i - 1 + 2 * k;
                    if (j < 0 || j >= n_layers) continue;
                    int hj = hs[j], wj = ws[j];
                    int64_t a = ((int64_t)y * hj + (h >> 1)) / h;
                    int64_t b = ((int64_t)x * wj + (w >> 1)) / w;
                    yj[k] = (int)(a < hj - 1 ? a : hj - 1);
                    xj[k] = (int)(b < wj - 1 ? b : wj - 1);
                    have[k] = 1;
                    if (!(s > maps[j][(size_t)yj[k] * wj + xj[k]])) keep = 0;
                }
                if (!keep) continue;
                double p[3][3], ox, oy, v0;
                int ok;
                gather(sm, w, h, y, x, p, NULL);                          /* :277-279 */
                fit_peak(p, &ox, &oy, &v0, &ok);
                double nv[2] = {0.0, 0.0};
                for (int k = 0; k < 2; k++) {                             /* :281-285 */
                    if (!have[k]) continue;
                    int j = i - 1 + 2 * k;
                    double pj[3][3], vj, tx, ty;
                    int32_t pmax;
                    int okj;
                    gather(maps[j], ws[j], hs[j], yj[k], xj[k], pj, &pmax);
                    fit_peak(pj, &tx, &ty, &vj, &okj);
                    nv[k] = okj ? vj : (double)pmax;
                }
                double sig = sigmas[i];
                if (have[0] && have[1]) {                                 /* :287-297 */
                    double vb = nv[0], va = nv[1];
                    double denom = vb - 2.0 * v0 + va;
                    int concave = denom < 0.0;
                    double delta = concave ? 0.5 * (vb - va) / denom : 0.0;
                    delta = fabs(delta) < 1.0 ? delta : 0.0;
                    double up = sigmas[i + 1] / sigmas[i];
                    double down = sigmas[i - 1] / sigmas[i];
                    double a = delta > 0.0 ? delta : 0.0;
                    double b = -delta > 0.0 ? -delta : 0.0;
                    sig = sigmas[i] * pow(up, a) * pow(down, b);
                }
                double scale = scales[i];                                 /* :299-302 */
                double x0 = ((double)x + ox) / scale;
                double y0 = ((double)y + oy) / scale;
                double xhi = (double)W - 1e-6, yhi = (double)H - 1e-6;
                x0 = x0 < 0.0 ? 0.0 : (x0 > xhi ? xhi : x0);
                y0 = y0 < 0.0 ? 0.0 : (y0 > yhi ? yhi : y0);
                if (n >= cap) return -1;
                kx[n] = x0; ky[n] = y0; ksig[n] = sig; kscore[n] = v0;
                if (layer_out) layer_out[n] = i;
                if (xi_out) xi_out[n] = x;
                if (yi_out) yi_out[n] = y;
                n++;
            }
    }
    return n;
}

/* ------------------------------------------------------------------ */
/* descriptor.py:28-32 integral_image (int64, (h+1) x (w+1))             */
/* ------------------------------------------------------------------ */
void vfo_integral(const uint8_t *d, int w, int h, int64_t *sat)
{
    int W1 = w + 1;
    memset(sat, 0, sizeof(int64_t) * (size_t)W1);
    for (int y = 0; y < h; y++) {
        int64_t row = 0;
        sat[(size_t)(y + 1) * W1] = 0;
        for (int x = 0; x < w; x++) {
            row += d[(size_t)y * w + x];
            sat[(size_t)(y + 1) * W1 + x + 1] = sat[(size_t)y * W1 + x + 1] + row;
        }
    }
}

/* descriptor.py:85-92 _box_mean_jit */
static inline int64_t box_mean(const int64_t *sat, int w, int h, int64_t x, int64_t y, int64_t r)
{
    int64_t x0 = x - r > 0 ? x - r : 0, x1 = x + r < w - 1 ? x + r : w - 1;
    int64_t y0 = y - r > 0 ? y - r : 0, y1 = y + r < h - 1 ? y + r : h - 1;
    int64_t W1 = w + 1;
    int64_t s = sat[(y1 + 1) * W1 + x1 + 1] - sat[y0 * W1 + x1 + 1] - sat[(y1 + 1) * W1 + x0] + sat[y0 * W1 + x0];
    return s / ((x1 - x0 + 1) * (y1 - y0 + 1));   /* s >= 0: floor division */
}

/* descriptor.py:94-115 _point_values_jit for one keypoint */
static void point_values(const int64_t *sat, int w, int h, double kx, double ky, double sigma,
                         double theta, const double *pts, const double *radii, int m, int64_t *out)
{
    double c = cos(theta), s = sin(theta);
    for (int j = 0; j < m; j++) {
        double px = pts[2 * j], py = pts[2 * j + 1];
        int64_t x = (int64_t)floor(kx + sigma * (c * px - s * py) + 0.5);
        int64_t y = (int64_t)floor(ky + sigma * (s * px + c * py) + 0.5);
        if (x < 0) x = 0; else if (x > w - 1) x = w - 1;
        if (y < 0) y = 0; else if (y > h - 1) y = h - 1;
        int64_t r = (int64_t)floor(radii[j] * sigma + 0.5);
        out[j] = box_mean(sat, w, h, x, y, r);
    }
}

/* descriptor.py:128-144 _orientations_jit (sequential sum in pair order) */
void vfo_orientations(const int64_t *sat, int w, int h, int n, const double *kx, const double *ky,
                      const double *sigma, const double *pts, const double *radii, int m,
                      const int32_t *li, const int32_t *lj, const double *wx, const double *wy,
                      int L, double *theta)
{
    int64_t *vals = (int64_t *)malloc(sizeof(int64_t) * m);
    for (int i = 0; i < n; i++) {
        point_values(sat, w, h, kx[i], ky[i], sigma[i], 0.0, pts, radii, m, vals);
        double gx = 0.0, gy = 0.0;
        for (int p = 0; p < L; p++) {
            double dv = (double)(vals[li[p]] - vals[lj[p]]);
            gx += dv * wx[p];
            gy += dv * wy[p];
        }
        double t = atan2(gy, gx);
        theta[i] = t <= -M_PI ? M_PI : t;
    }
    free(vals);
}

/* descriptor.py:117-126 _describe_batch_jit, packed MSB-first (descriptor.py:271-275) */
void vfo_describe(const int64_t *sat, int w, int h, int n, const double *kx, const double *ky,
                  const double *sigma, const double *theta, const double *pts, const double *radii,
                  int m, const int32_t *si, const int32_t *sj, int nbits, uint8_t *packed)
{
    int64_t *vals = (int64_t *)malloc(sizeof(int64_t) * m);
    int nbytes = (nbits + 7) / 8;
    for (int i = 0; i < n; i++) {
        point_values(sat, w, h, kx[i], ky[i], sigma[i], theta[i], pts, radii, m, vals);
        uint8_t *o = packed + (size_t)i * nbytes;
        memset(o, 0, nbytes);
        for (int b = 0; b < nbits; b++)
            if (vals[si[b]] > vals[sj[b]]) o[b >> 3] |= (uint8_t)(0x80u >> (b & 7));
    }
    free(vals);
}

/* ------------------------------------------------------------------ */
/* masking.py:84-93 intensity_diff_mask (strict, int16 diff vs float t_i) */
/* ------------------------------------------------------------------ */
void vfo_intensity_mask(const uint8_t *prev, const uint8_t *cur, int n, double t_i, uint8_t *out)
{
    for (int i = 0; i < n; i++) {
        int d = (int)cur[i] - (int)prev[i];
        if (d < 0) d = -d;
        out[i] = (double)d > t_i ? 1 : 0;
    }
}

/* masking.py:96-119 binning_histogram (ceil cells, fp64 floor, clamped) */
void vfo_binning_hist(int n, const double *xs, const double *ys, int W, int H, int rows, int cols,
                      int64_t *hist)
{
    int64_t sx = (W + cols - 1) / cols, sy = (H + rows - 1) / rows;
    memset(hist, 0, sizeof(int64_t) * (size_t)rows * cols);
    for (int i = 0; i < n; i++) {
        double fx = floor(xs[i] / (double)sx), fy = floor(ys[i] / (double)sy);
        int64_t k = (int64_t)fx, l = (int64_t)fy;
        if (k < 0) k = 0; if (k > cols - 1) k = cols - 1;
        if (l < 0) l = 0; if (l > rows - 1) l = rows - 1;
        hist[l * cols + k]++;
    }
}

/* masking.py:139-148 upsample_mask: full[y][x] = bits[y//ch][x//cw] */
void vfo_upsample(const uint8_t *bits, int rows, int cols, int cw, int ch, int W, int H, uint8_t *full)
{
    (void)rows; (void)cols;
    for (int y = 0; y < H; y++)
        for (int x = 0; x < W; x++) full[(size_t)y * W + x] = bits[(y / ch) * cols + x / cw];
}

/* masking.py:151-165 _mask_at / _mask_values */
static inline int mask_at(const uint8_t *full, int W, int H, double x, double y)
{
    int64_t xi = (int64_t)floor(x + 0.5), yi = (int64_t)floor(y + 0.5);
    if (xi < 0) xi = 0; if (xi > W - 1) xi = W - 1;
    if (yi < 0) yi = 0; if (yi > H - 1) yi = H - 1;
    return full[yi * W + xi];
}

/* ------------------------------------------------------------------ */
/* pipeline.py:207-278 run_pipeline (modes none / intensity / binning)   */
/* ------------------------------------------------------------------ */
typedef struct {
    int n, cap;
    double *x, *y, *sigma, *theta, *score;
    uint8_t *origin;   /* 0 detected, 1 propagated */
    int32_t *age;
    uint8_t *desc;     /* 64 B packed per feature */
} vfo_feats;

typedef struct {
    int W, H, O, threshold, mode, per_layer, mask_level, t_h, grid_rows, grid_cols;
    double t_i;
    /* pattern */
    int m, nbits, L;
    double *pts, *radii, *wx, *wy;
    int32_t *si, *sj, *li, *lj;
    /* geometry */
    int n_layers, ws[VFO_MAX_LAYERS], hs[VFO_MAX_LAYERS];
    double scales[VFO_MAX_LAYERS];
    /* state */
    int64_t frame_no;
    uint8_t *layers[VFO_MAX_LAYERS], *prev_layers[VFO_MAX_LAYERS];
    int32_t *maps[VFO_MAX_LAYERS];
    uint8_t *full_mask, *level_masks[VFO_MAX_LAYERS / 2], *proj;
    int64_t *sat;
    vfo_feats cur, prev;
    /* report of the last frame */
    int n_detected, n_propagated, n_total, n_dropped;
    double coverage;
    /* temporal baseline (mode 3): GopConfig and the previous frame */
    int gop_delta, gop_patch, n_coarse, n_fine;
    double gop_t_bm, gop_t_et, *coarse, *fine;
    uint8_t *prev_frame;
} vfo_pipe;

void vfo_block_match(const uint8_t *prev, const uint8_t *cur, int w, int h, int n, const double *x, const double *y,
                     int patch, double t_bm, double t_et, const double *coarse, int nc, const double *fine, int nf,
                     double *nx, double *ny, double *sad_out, uint8_t *found);

static void feats_reserve(vfo_feats *f, int n)
{
    if (n <= f->cap) return;
    int c = f->cap ? f->cap : 1024;
    while (c < n) c *= 2;
    f->x = realloc(f->x, sizeof(double) * c);
    f->y = realloc(f->y, sizeof(double) * c);
    f->sigma = realloc(f->sigma, sizeof(double) * c);
    f->theta = realloc(f->theta, sizeof(double) * c);
    f->score = realloc(f->score, sizeof(double) * c);
    f->origin = realloc(f->origin, c);
    f->age = realloc(f->age, sizeof(int32_t) * c);
    f->desc = realloc(f->desc, (size_t)64 * c);
    f->cap = c;
}

static void feats_free(vfo_feats *f)
{
    free(f->x); free(f->y); free(f->sigma); free(f->theta); free(f->score);
    free(f->origin); free(f->age); free(f->desc);
    memset(f, 0, sizeof(*f));
}

/* mode: 0 none, 1 intensity, 2 binning, 3 temporal (vfo_pipe_set_gop).  mask_level < 0 = top octave. */
vfo_pipe *vfo_pipe_create(int W, int H, int O, int threshold, int mode, double t_i, int t_h,
                          int grid_rows, int grid_cols, int mask_level, int per_layer, int m,
                          const double *pts, const double *radii, int nbits, const int32_t *short_pairs,
                          int L, const int32_t *long_pairs, int *err)
{
    *err = 0;
    if (threshold < 1) { *err = -10; return NULL; }
    vfo_pipe *p = (vfo_pipe *)calloc(1, sizeof(vfo_pipe));
    p->W = W; p->H = H; p->O = O; p->threshold = threshold; p->mode = mode; p->t_i = t_i;
    p->t_h = t_h; p->grid_rows = grid_rows; p->grid_cols = grid_cols; p->per_layer = per_layer;
    p->mask_level = mask_level < 0 ? O - 1 : mask_level;
    if (O > VFO_MAX_LAYERS / 2) { *err = -1; free(p); return NULL; }
    int rc = vfo_layer_dims(W, H, O, p->ws, p->hs, p->scales);
    if (rc) { *err = rc; free(p); return NULL; }
    p->n_layers = 2 * O;
    for (int l = 0; l < p->n_layers; l++) {
        size_t sz = (size_t)p->ws[l] * p->hs[l];
        p->layers[l] = malloc(sz);
        p->prev_layers[l] = malloc(sz);
        p->maps[l] = malloc(sizeof(int32_t) * sz);
    }
    p->full_mask = malloc((size_t)W * H);
    for (int o = 0; o < O; o++) p->level_masks[o] = malloc((size_t)W * H);
    p->proj = malloc((size_t)W * H);
    p->sat = malloc(sizeof(int64_t) * (size_t)(W + 1) * (H + 1));
    p->m = m; p->nbits = nbits; p->L = L;
    p->pts = malloc(sizeof(double) * 2 * m); memcpy(p->pts, pts, sizeof(double) * 2 * m);
    p->radii = malloc(sizeof(double) * m); memcpy(p->radii, radii, sizeof(double) * m);
    p->si = malloc(sizeof(int32_t) * nbits); p->sj = malloc(sizeof(int32_t) * nbits);
    for (int b = 0; b < nbits; b++) { p->si[b] = short_pairs[2 * b]; p->sj[b] = short_pairs[2 * b + 1]; }
    p->li = malloc(sizeof(int32_t) * L); p->lj = malloc(sizeof(int32_t) * L);
    p->wx = malloc(sizeof(double) * L); p->wy = malloc(sizeof(double) * L);
    for (int q = 0; q < L; q++) {                      /* descriptor.py:163-180 _pair_arrays */
        int a = long_pairs[2 * q], b = long_pairs[2 * q + 1];
        p->li[q] = a; p->lj[q] = b;
        double dx = pts[2 * a] - pts[2 * b], dy = pts[2 * a + 1] - pts[2 * b + 1];
        double inv = 1.0 / (dx * dx + dy * dy);
        p->wx[q] = dx * inv; p->wy[q] = dy * inv;
    }
    return p;
}

void vfo_pipe_destroy(vfo_pipe *p)
{
    if (!p) return;
    for (int l = 0; l < p->n_layers; l++) { free(p->layers[l]); free(p->prev_layers[l]); free(p->maps[l]); }
    for (int o = 0; o < p->O; o++) free(p->level_masks[o]);
    free(p->full_mask); free(p->proj); free(p->sat);
    free(p->pts); free(p->radii); free(p->si); free(p->sj); free(p->li); free(p->lj); free(p->wx); free(p->wy);
    feats_free(&p->cur); feats_free(&p->prev);
    free(p->coarse); free(p->fine); free(p->prev_frame);
    free(p);
}

/* GopConfig (temporal.py:23-43) + spiral offsets (coarse; fine without (0, 0)). */
void vfo_pipe_set_gop(vfo_pipe *p, int delta, int patch, double t_bm, double t_et, const double *coarse, int nc,
                      const double *fine, int nf)
{
    p->gop_delta = delta; p->gop_patch = patch; p->gop_t_bm = t_bm; p->gop_t_et = t_et;
    p->n_coarse = nc; p->n_fine = nf;
    p->coarse = realloc(p->coarse, sizeof(double) * 2 * (nc ? nc : 1));
    p->fine = realloc(p->fine, sizeof(double) * 2 * (nf ? nf : 1));
    memcpy(p->coarse, coarse, sizeof(double) * 2 * nc);
    memcpy(p->fine, fine, sizeof(double) * 2 * nf);
    if (!p->prev_frame) p->prev_frame = malloc((size_t)p->W * p->H);
}

/* pipeline.py:281-345 _run_temporal, off-GOP frame: baseline_step's block matching. */
static int temporal_step(vfo_pipe *p, const uint8_t *frame)
{
    const vfo_feats *pv = &p->prev;
    vfo_feats *out = &p->cur;
    feats_reserve(out, pv->n);
    int n = pv->n;
    double *nx = malloc(sizeof(double) * (n ? n : 1)), *ny = malloc(sizeof(double) * (n ? n : 1));
    double *sd = malloc(sizeof(double) * (n ? n : 1));
    uint8_t *fd = malloc(n ? n : 1);
    vfo_block_match(p->prev_frame, frame, p->W, p->H, n, pv->x, pv->y, p->gop_patch, p->gop_t_bm, p->gop_t_et,
                    p->coarse, p->n_coarse, p->fine, p->n_fine, nx, ny, sd, fd);
    int k = 0;
    for (int i = 0; i < n; i++) {
        if (!fd[i]) continue;
        out->x[k] = nx[i]; out->y[k] = ny[i]; out->sigma[k] = pv->sigma[i]; out->theta[k] = pv->theta[i];
        out->score[k] = pv->score[i]; out->origin[k] = 1; out->age[k] = pv->age[i] + 1;
        memcpy(out->desc + (size_t)64 * k, pv->desc + (size_t)64 * i, 64);
        k++;
    }
    out->n = k;
    free(nx); free(ny); free(sd); free(fd);
    p->n_detected = 0; p->n_propagated = k; p->n_total = k; p->n_dropped = 0; p->coverage = 0.0;
    vfo_feats tmp = p->prev; p->prev = p->cur; p->cur = tmp;
    memcpy(p->prev_frame, frame, (size_t)p->W * p->H);
    p->frame_no++;
    return 0;
}

static int any_set(const uint8_t *a, size_t n)
{
    for (size_t i = 0; i < n; i++) if (a[i]) return 1;
    return 0;
}

/* One frame through run_pipeline's loop body (pipeline.py:222-277).  Returns 0 or <0. */
int vfo_pipe_process(vfo_pipe *p, const uint8_t *frame)
{
    int W = p->W, H = p->H, O = p->O, NL = p->n_layers;
    if (p->mode == 3 && p->frame_no % p->gop_delta != 0) return temporal_step(p, frame);   /* off-GOP */
    int rc = vfo_build_pyramid(frame, W, H, O, p->layers);
    if (rc) return rc;
    int use_mask = p->mode != 0 && p->mode != 3 && p->frame_no > 0;   /* GOP start: full detection */
    int per_level = 0;
    double coverage = 1.0;
    if (use_mask) {                                        /* pipeline.py:174-204 _build_mask */
        if (p->mode == 2) {
            int rows = p->grid_rows, cols = p->grid_cols;
            int64_t *hist = malloc(sizeof(int64_t) * rows * cols);
            vfo_binning_hist(p->prev.n, p->prev.x, p->prev.y, W, H, rows, cols, hist);
            uint8_t *bits = malloc(rows * cols);
            for (int i = 0; i < rows * cols; i++) bits[i] = hist[i] >= p->t_h;
            vfo_upsample(bits, rows, cols, (W + cols - 1) / cols, (H + rows - 1) / rows, W, H, p->full_mask);
            free(hist); free(bits);
        } else if (p->per_layer) {
            per_level = 1;
            memset(p->full_mask, 0, (size_t)W * H);
            for (int o = 0; o < O; o++) {
                int l = 2 * o, w = p->ws[l], h = p->hs[l];
                uint8_t *bits = malloc((size_t)w * h);
                vfo_intensity_mask(p->prev_layers[l], p->layers[l], w * h, p->t_i, bits);
                vfo_upsample(bits, h, w, (W + w - 1) / w, (H + h - 1) / h, W, H, p->level_masks[o]);
                for (size_t i = 0; i < (size_t)W * H; i++) p->full_mask[i] |= p->level_masks[o][i];
                free(bits);
            }
        } else {
            int l = 2 * p->mask_level, w = p->ws[l], h = p->hs[l];
            uint8_t *bits = malloc((size_t)w * h);
            vfo_intensity_mask(p->prev_layers[l], p->layers[l], w * h, p->t_i, bits);
            vfo_upsample(bits, h, w, (W + w - 1) / w, (H + h - 1) / h, W, H, p->full_mask);
            free(bits);
        }
        size_t cnt = 0;
        for (size_t i = 0; i < (size_t)W * H; i++) cnt += p->full_mask[i];
        coverage = (double)cnt / ((double)W * (double)H);   /* masking.py:44-46 */
    }
    /* pipeline.py:91-139 _detect_keypoints */
    int nk = 0;
    double *kx = NULL, *ky = NULL, *ks = NULL, *kv = NULL;
    int skip = use_mask && !per_level && !any_set(p->full_mask, (size_t)W * H);
    if (!skip) {
        int any_job = 0;
        for (int l = 0; l < NL; l++) {
            int w = p->ws[l], h = p->hs[l];
            const uint8_t *gate = NULL;
            if (use_mask) {
                const uint8_t *src = per_level ? p->level_masks[l / 2] : p->full_mask;
                vfo_project_mask(src, W, H, w, h, p->proj);
                if (!any_set(p->proj, (size_t)w * h)) {
                    memset(p->maps[l], 0, sizeof(int32_t) * (size_t)w * h);
                    continue;
                }
                gate = p->proj;
            }
            any_job = 1;
            vfo_score_map(p->layers[l], w, h, p->threshold, gate, p->maps[l]);
        }
        if (any_job) {
            int cap = 1 << 16;
            for (;;) {
                kx = realloc(kx, sizeof(double) * cap); ky = realloc(ky, sizeof(double) * cap);
                ks = realloc(ks, sizeof(double) * cap); kv = realloc(kv, sizeof(double) * cap);
                nk = vfo_nms((const int32_t *const *)p->maps, p->ws, p->hs, p->scales, NL, W, H, cap,
                             kx, ky, ks, kv, NULL, NULL, NULL);
                if (nk != -1) break;
                cap *= 4;
            }
            if (nk < 0) { free(kx); free(ky); free(ks); free(kv); return nk; }
        }
    }
    /* pipeline.py:142-171 _describe_keypoints: border filter then describe kept */
    int kept = 0;
    for (int i = 0; i < nk; i++) {
        double mg = 3.0 * ks[i];
        if (kx[i] >= mg && ky[i] >= mg && kx[i] <= (double)(W - 1) - mg && ky[i] <= (double)(H - 1) - mg) {
            kx[kept] = kx[i]; ky[kept] = ky[i]; ks[kept] = ks[i]; kv[kept] = kv[i];
            kept++;
        }
    }
    int n_dropped = nk - kept;
    double *th = malloc(sizeof(double) * (kept ? kept : 1));
    uint8_t *dsc = malloc((size_t)64 * (kept ? kept : 1));
    if (kept) {
        vfo_integral(frame, W, H, p->sat);
        vfo_orientations(p->sat, W, H, kept, kx, ky, ks, p->pts, p->radii, p->m, p->li, p->lj, p->wx,
                         p->wy, p->L, th);
        vfo_describe(p->sat, W, H, kept, kx, ky, ks, th, p->pts, p->radii, p->m, p->si, p->sj, p->nbits, dsc);
    }
    /* masking.py:168-184 merge_features (or detected only) */
    vfo_feats *out = &p->cur;
    feats_reserve(out, kept + p->prev.n);
    int n = 0;
    for (int i = 0; i < kept; i++) {
        if (use_mask && !mask_at(p->full_mask, W, H, kx[i], ky[i])) continue;
        out->x[n] = kx[i]; out->y[n] = ky[i]; out->sigma[n] = ks[i]; out->theta[n] = th[i];
        out->score[n] = kv[i]; out->origin[n] = 0; out->age[n] = 0;
        memcpy(out->desc + (size_t)64 * n, dsc + (size_t)64 * i, 64);
        n++;
    }
    int n_det = n;
    if (use_mask) {
        const vfo_feats *pv = &p->prev;
        for (int i = 0; i < pv->n; i++) {
            if (mask_at(p->full_mask, W, H, pv->x[i], pv->y[i])) continue;
            out->x[n] = pv->x[i]; out->y[n] = pv->y[i]; out->sigma[n] = pv->sigma[i];
            out->theta[n] = pv->theta[i]; out->score[n] = pv->score[i]; out->origin[n] = 1;
            out->age[n] = pv->age[i] + 1;
            memcpy(out->desc + (size_t)64 * n, pv->desc + (size_t)64 * i, 64);
            n++;
        }
    }
    out->n = n;
    free(kx); free(ky); free(ks); free(kv); free(th); free(dsc);
    p->n_detected = n_det; p->n_propagated = n - n_det; p->n_total = n;
    p->n_dropped = n_dropped; p->coverage = coverage;
    /* state carried to the next frame (pipeline.py:276-277) */
    vfo_feats tmp = p->prev; p->prev = p->cur; p->cur = tmp;
    for (int l = 0; l < NL; l++) {
        uint8_t *t = p->prev_layers[l]; p->prev_layers[l] = p->layers[l]; p->layers[l] = t;
    }
    if (p->mode == 3) memcpy(p->prev_frame, frame, (size_t)W * H);
    p->frame_no++;
    return 0;
}

/* Results of the last processed frame (valid until the next process call). */
void vfo_pipe_report(const vfo_pipe *p, int32_t *counts /*4*/, double *coverage)
{
    counts[0] = p->n_detected; counts[1] = p->n_propagated; counts[2] = p->n_total; counts[3] = p->n_dropped;
    *coverage = p->coverage;
}

void vfo_pipe_features(const vfo_pipe *p, double *x, double *y, double *sigma, double *theta, double *score,
                       uint8_t *origin, int32_t *age, uint8_t *desc)
{
    const vfo_feats *f = &p->prev;   /* swapped in at the end of process */
    size_t n = (size_t)f->n;
    memcpy(x, f->x, 8 * n); memcpy(y, f->y, 8 * n); memcpy(sigma, f->sigma, 8 * n);
    memcpy(theta, f->theta, 8 * n); memcpy(score, f->score, 8 * n);
    memcpy(origin, f->origin, n); memcpy(age, f->age, 4 * n); memcpy(desc, f->desc, 64 * n);
}

/* ------------------------------------------------------------------ */
/* matching.py:22,47-66 -- Hamming distance of packed descriptor rows:  */
/* sum over bytes of popcount(q XOR r) through the 256-entry LUT.       */
/* ------------------------------------------------------------------ */
void vfo_hamming_matrix(const uint8_t *q, long nq, const uint8_t *r, long nr, int nbytes, int32_t *out)
{
  static uint8_t lut[256];
  static int ready = 0;
  if (!ready) {
    for (int i = 0; i < 256; i++) {
      int c = 0;
      for (int b = 0; b < 8; b++) c += (i >> b) & 1;
      lut[i] = (uint8_t)c;
    }
    ready = 1;
  }
  for (long i = 0; i < nq; i++)
    for (long j = 0; j < nr; j++) {
      int32_t acc = 0;
      for (int b = 0; b < nbytes; b++) acc += lut[q[i * nbytes + b] ^ r[j * nbytes + b]];
      out[i * nr + j] = acc;
    }
}

/* ------------------------------------------------------------------ */
/* temporal.py:64-226 -- two-stage spiral SAD search of one 16x16 (or  */
/* patch x patch) block; baseline_step's per-feature part :274-308.     */
/* offsets: (n x 2) doubles in spiral order (fine set without (0, 0)).  */
/* ------------------------------------------------------------------ */
static void coarse_search(const uint8_t *patch, int ph, int pw, const uint8_t *frame, int w, int h,
                          int64_t base_x, int64_t base_y, const double *offs, int n, double t_et,
                          int *best_k, int64_t *best_sad, int *early)
{                                                        /* temporal.py:125-145 (_coarse_search_jit) */
    int64_t best = (int64_t)1 << 60;
    int bk = -1;
    *early = 0;
    for (int k = 0; k < n; k++) {
        int64_t tlx = base_x + (int64_t)offs[2 * k], tly = base_y + (int64_t)offs[2 * k + 1];
        if (tlx < 0 || tly < 0 || tlx + pw > w || tly + ph > h) continue;
        int64_t sad = 0;
        for (int r = 0; r < ph; r++)
            for (int c = 0; c < pw; c++) {
                int64_t d = (int64_t)patch[r * pw + c] - (int64_t)frame[(tly + r) * w + tlx + c];
                sad += d < 0 ? -d : d;
            }
        if (sad < best) {
            best = sad;
            bk = k;
            if ((double)sad < t_et) { *early = 1; break; }
        }
    }
    *best_k = bk;
    *best_sad = best;
}

static void fine_search(const uint8_t *patch, int ph, int pw, const uint8_t *frame, int w, int h, double base_x,
                        double base_y, const double *offs, int n, double t_et, double init, int *best_k,
                        double *best_sad)
{                                                        /* temporal.py:147-180 (_fine_search_jit) */
    double best = init;
    int bk = -1;
    for (int k = 0; k < n; k++) {
        double fx = base_x + offs[2 * k], fy = base_y + offs[2 * k + 1];
        int64_t ix = (int64_t)floor(fx), iy = (int64_t)floor(fy);
        if (ix < 0 || iy < 0 || ix + pw >= w || iy + ph >= h) continue;
        double ax = fx - (double)ix, ay = fy - (double)iy;
        double w00 = (1.0 - ax) * (1.0 - ay), w10 = ax * (1.0 - ay), w01 = (1.0 - ax) * ay, w11 = ax * ay;
        double sad = 0.0;
        for (int r = 0; r < ph; r++)
            for (int c = 0; c < pw; c++) {
                const uint8_t *f0 = frame + (iy + r) * w + ix + c, *f1 = f0 + w;
                double v = w00 * f0[0] + w10 * f0[1] + w01 * f1[0] + w11 * f1[1];
                sad += fabs((double)patch[r * pw + c] - v);
            }
        if (sad < best) {
            best = sad;
            bk = k;
            if (sad < t_et) break;
        }
    }
    *best_k = bk;
    *best_sad = best;
}

/* found[i] = 1 and (nx, ny, sad) when feature i is tracked into cur (temporal.py:274-308). */
void vfo_block_match(const uint8_t *prev, const uint8_t *cur, int w, int h, int n, const double *x, const double *y,
                     int patch, double t_bm, double t_et, const double *coarse, int nc, const double *fine, int nf,
                     double *nx, double *ny, double *sad_out, uint8_t *found)
{
    int half = patch / 2;
    uint8_t *pb = (uint8_t *)malloc((size_t)patch * patch);
    for (int i = 0; i < n; i++) {
        found[i] = 0; nx[i] = 0.0; ny[i] = 0.0; sad_out[i] = 0.0;
        int64_t cxi = (int64_t)floor(x[i] + 0.5), cyi = (int64_t)floor(y[i] + 0.5);
        int64_t tlx = cxi - half, tly = cyi - half;
        if (tlx < 0 || tly < 0 || tlx + patch > w || tly + patch > h) continue;
        for (int r = 0; r < patch; r++) memcpy(pb + r * patch, prev + (tly + r) * w + tlx, (size_t)patch);
        /* spiral_search (temporal.py:200-226): same rounded centre */
        int64_t base_x = cxi - patch / 2, base_y = cyi - patch / 2;
        int k, early;
        int64_t isad;
        coarse_search(pb, patch, patch, cur, w, h, base_x, base_y, coarse, nc, t_et, &k, &isad, &early);
        if (k < 0) continue;
        double ox = coarse[2 * k], oy = coarse[2 * k + 1], best = (double)isad;
        if (!early) {
            int fk;
            double fsad;
            fine_search(pb, patch, patch, cur, w, h, (double)base_x + ox, (double)base_y + oy, fine, nf, t_et, best,
                        &fk, &fsad);
            if (fk >= 0) { ox += fine[2 * fk]; oy += fine[2 * fk + 1]; best = fsad; }
        }
        if (best >= t_bm) continue;
        found[i] = 1;
        nx[i] = (double)cxi + ox;
        ny[i] = (double)cyi + oy;
        sad_out[i] = best;
    }
    free(pb);
}

/* ================================================================== */
/* Geometric verification: matching.py:97-192 (ransac_homography).    */
/* ================================================================== */

/* numpy 2.3's default_rng(seed) = Generator(PCG64(SeedSequence(seed)))
 * (third-party, not vendored in /root/reference), restated from its
 * published algorithm: SeedSequence hash-mixing into a 4-word pool and
 * generate_state(4, uint64); PCG64 setseq-128 with XSL-RR output; 32-bit
 * draws take the low half of a 64-bit output first and buffer the high half;
 * choice(n, 4, replace=False) = Floyd's sampling with Lemire bounded draws,
 * then a Fisher-Yates pass with Lemire draws.  Sequential (no jump-ahead). */
typedef unsigned __int128 vfo_u128;
typedef struct { vfo_u128 state, inc; uint32_t buf; int has; } vfo_pcg;

static uint32_t vfo_hashmix(uint32_t v, uint32_t *hc)
{
    v ^= *hc;
    *hc *= 0x931e8875u;
    v *= *hc;
    return v ^ (v >> 16);
}

static void vfo_pcg_seed(vfo_pcg *g, uint64_t seed)
{
    uint32_t ent[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)}, pool[4], hc = 0x43b0d7e5u, hb = 0x8b51f9ddu, w[8];
    int ne = (seed >> 32) ? 2 : 1;
    for (int i = 0; i < 4; i++) pool[i] = vfo_hashmix(i < ne ? ent[i] : 0u, &hc);
    for (int a = 0; a < 4; a++)
        for (int b = 0; b < 4; b++)
            if (a != b) {
                uint32_t y = vfo_hashmix(pool[a], &hc);
                uint32_t r = 0xca01f9ddu * pool[b] - 0x4973f715u * y;
                pool[b] = r ^ (r >> 16);
            }
    for (int i = 0; i < 8; i++) {
        uint32_t d = pool[i % 4] ^ hb;
        hb *= 0x58f38dedu;
        d *= hb;
        w[i] = d ^ (d >> 16);
    }
    uint64_t s[4];
    for (int i = 0; i < 4; i++) s[i] = (uint64_t)w[2 * i] | ((uint64_t)w[2 * i + 1] << 32);
    const vfo_u128 mult = ((vfo_u128)0x2360ED051FC65DA4ull << 64) | 0x4385DF649FCCF645ull;
    g->inc = ((((vfo_u128)s[2] << 64) | s[3]) << 1) | 1u;
    g->state = g->inc;                                  /* 0 * mult + inc */
    g->state += ((vfo_u128)s[0] << 64) | s[1];
    g->state = g->state * mult + g->inc;
    g->has = 0;
}

static uint32_t vfo_next32(vfo_pcg *g)
{
    if (g->has) { g->has = 0; return g->buf; }
    const vfo_u128 mult = ((vfo_u128)0x2360ED051FC65DA4ull << 64) | 0x4385DF649FCCF645ull;
    g->state = g->state * mult + g->inc;
    uint64_t hi = (uint64_t)(g->state >> 64), x = hi ^ (uint64_t)g->state;
    unsigned rot = (unsigned)(hi >> 58);
    uint64_t v = (x >> rot) | (x << ((64 - rot) & 63));
    g->has = 1;
    g->buf = (uint32_t)(v >> 32);
    return (uint32_t)v;
}

static uint32_t vfo_bounded(vfo_pcg *g, uint32_t rng)     /* [0, rng], Lemire */
{
    if (rng == 0) return 0;
    uint64_t ex = (uint64_t)rng + 1, m = (uint64_t)vfo_next32(g) * ex;
    uint32_t left = (uint32_t)m;
    if (left < ex) {
        uint32_t th = (uint32_t)((0xffffffffu - rng) % ex);
        while (left < th) { m = (uint64_t)vfo_next32(g) * ex; left = (uint32_t)m; }
    }
    return (uint32_t)(m >> 32);
}

int vfo_ransac_samples(uint64_t seed, int64_t n, int iters, int32_t *out)
{
    if (n < 4 || n > 0x7fffffff) return -1;
    vfo_pcg g;
    vfo_pcg_seed(&g, seed);
    for (int k = 0; k < iters; k++) {
        int64_t v[4];
        for (int64_t j = n - 4; j < n; j++) {             /* Floyd */
            int64_t x = vfo_bounded(&g, (uint32_t)j), c = j - (n - 4);
            for (int q = 0; q < c; q++) if (v[q] == x) { x = j; break; }
            v[c] = x;
        }
        for (int i = 3; i >= 1; i--) {                    /* shuffle */
            int64_t j = vfo_bounded(&g, (uint32_t)i), t = v[i];
            v[i] = v[j]; v[j] = t;
        }
        for (int q = 0; q < 4; q++) out[4 * k + q] = (int32_t)v[q];
    }
    return 0;
}

/* matching.py:97-106: similarity conditioning; 0 if mean distance < 1e-12 */
static int vfo_normalize(const double *p, int n, double t[9])
{
    double cx = 0, cy = 0, d = 0;
    for (int i = 0; i < n; i++) { cx += p[2 * i]; cy += p[2 * i + 1]; }
    cx /= n; cy /= n;
    for (int i = 0; i < n; i++)
        d += sqrt((p[2 * i] - cx) * (p[2 * i] - cx) + (p[2 * i + 1] - cy) * (p[2 * i + 1] - cy));
    d /= n;
    if (d < 1e-12) return 0;
    double s = sqrt(2.0) / d;
    double tt[9] = {s, 0, -s * cx, 0, s, -s * cy, 0, 0, 1};
    memcpy(t, tt, sizeof tt);
    return 1;
}

static void vfo_mat3(const double *a, const double *b, double *c)
{
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) c[3 * i + j] = a[3 * i] * b[j] + a[3 * i + 1] * b[3 + j] + a[3 * i + 2] * b[6 + j];
}

/* one-sided Jacobi SVD of the m x k column-major matrix a (k <= 9): on return
 * the columns of a are U*S and v (k x k, row-major) holds V; sv[j] = |a_j| */
static void vfo_jacobi_svd(double *a, int m, int k, double *v, double *sv)
{
    for (int i = 0; i < k * k; i++) v[i] = (i / k == i % k);
    for (int sweep = 0; sweep < 80; sweep++) {
        int rot = 0;
        for (int p = 0; p < k - 1; p++)
            for (int q = p + 1; q < k; q++) {
                double al = 0, be = 0, ga = 0;
                double *cp = a + (size_t)p * m, *cq = a + (size_t)q * m;
                for (int i = 0; i < m; i++) { al += cp[i] * cp[i]; be += cq[i] * cq[i]; ga += cp[i] * cq[i]; }
                if (ga == 0.0 || fabs(ga) <= 1e-15 * sqrt(al * be)) continue;
                rot = 1;
                double zeta = (be - al) / (2.0 * ga);
                double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
                for (int i = 0; i < m; i++) {
                    double x = cp[i], y = cq[i];
                    cp[i] = c * x - s * y; cq[i] = s * x + c * y;
                }
                for (int i = 0; i < k; i++) {
                    double x = v[i * k + p], y = v[i * k + q];
                    v[i * k + p] = c * x - s * y; v[i * k + q] = s * x + c * y;
                }
            }
        if (!rot) break;
    }
    for (int j = 0; j < k; j++) {
        double s = 0;
        for (int i = 0; i < m; i++) s += a[(size_t)j * m + i] * a[(size_t)j * m + i];
        sv[j] = sqrt(s);
    }
}

/* matching.py:109-137 (_dlt): normalized DLT, h = right singular vector of
 * the smallest singular value (vt[-1]); 0 when _dlt returns None */
static int vfo_dlt(const double *src, const double *dst, int n, double h[9])
{
    double ts[9], td[9];
    if (!vfo_normalize(src, n, ts) || !vfo_normalize(dst, n, td)) return 0;
    int m = 2 * n, k = 9;
    /* m >= 9 for the SVD's null space to be the smallest column; pad rows */
    int mr = m < 9 ? 9 : m;
    double *a = calloc((size_t)mr * 9, sizeof(double)), v[81], sv[9];
    for (int i = 0; i < n; i++) {
        double sh[3], dh[3], x = src[2 * i], y = src[2 * i + 1], u = dst[2 * i], w = dst[2 * i + 1];
        for (int r = 0; r < 3; r++) {
            sh[r] = ts[3 * r] * x + ts[3 * r + 1] * y + ts[3 * r + 2];
            dh[r] = td[3 * r] * u + td[3 * r + 1] * w + td[3 * r + 2];
        }
        for (int c = 0; c < 3; c++) {
            a[(size_t)c * mr + 2 * i] = -sh[c];                      /* a[0::2, 0:3] = -sh */
            a[(size_t)(6 + c) * mr + 2 * i] = sh[c] * dh[0];         /* a[0::2, 6:9]       */
            a[(size_t)(3 + c) * mr + 2 * i + 1] = -sh[c];            /* a[1::2, 3:6] = -sh */
            a[(size_t)(6 + c) * mr + 2 * i + 1] = sh[c] * dh[1];     /* a[1::2, 6:9]       */
        }
    }
    vfo_jacobi_svd(a, mr, k, v, sv);
    free(a);
    int j = 0;
    for (int c = 1; c < 9; c++) if (sv[c] < sv[j]) j = c;
    double hn[9], tdi[9] = {1.0 / td[0], 0, -td[2] / td[0], 0, 1.0 / td[4], -td[5] / td[4], 0, 0, 1}, t[9];
    for (int r = 0; r < 9; r++) hn[r] = v[r * 9 + j];
    vfo_mat3(hn, ts, t);
    vfo_mat3(tdi, t, h);
    for (int r = 0; r < 9; r++) if (!isfinite(h[r])) return 0;
    if (fabs(h[8]) > 1e-12) { double d = h[8]; for (int r = 0; r < 9; r++) h[r] /= d; }
    return 1;
}

/* matching.py:140-146 (_usable): finite, |det| >= 1e-12, cond_2 < 1e12 */
static int vfo_usable(const double h[9])
{
    for (int r = 0; r < 9; r++) if (!isfinite(h[r])) return 0;
    double det = h[0] * (h[4] * h[8] - h[5] * h[7]) - h[1] * (h[3] * h[8] - h[5] * h[6])
               + h[2] * (h[3] * h[7] - h[4] * h[6]);
    if (fabs(det) < 1e-12) return 0;
    double a[9], v[9], sv[3];
    for (int r = 0; r < 3; r++) for (int c = 0; c < 3; c++) a[c * 3 + r] = h[3 * r + c];
    vfo_jacobi_svd(a, 3, 3, v, sv);
    double mx = fmax(sv[0], fmax(sv[1], sv[2])), mn = fmin(sv[0], fmin(sv[1], sv[2]));
    return mn > 0 && mx / mn < 1e12;
}

/* matching.py:149-154 + :177: reprojection error under h, inlier iff < tol */
static int64_t vfo_inliers(const double h[9], const double *src, const double *dst, int64_t n, double tol,
                           uint8_t *inl)
{
    int64_t c = 0;
    for (int64_t i = 0; i < n; i++) {
        double x = src[2 * i], y = src[2 * i + 1];
        double px = x * h[0] + y * h[1] + h[2], py = x * h[3] + y * h[4] + h[5], z = x * h[6] + y * h[7] + h[8];
        if (fabs(z) < 1e-12) z = 1e-12;
        double ex = px / z - dst[2 * i], ey = py / z - dst[2 * i + 1];
        inl[i] = sqrt(ex * ex + ey * ey) < tol;
        c += inl[i];
    }
    return c;
}

/* matching.py:157-192: returns the final inlier count (inl[] marks them,
 * h the model) or -1 for (None, []) */
int64_t vfo_ransac_homography(int64_t n, const double *src, const double *dst, int iters, double tol, uint64_t seed,
                              double *h_out, uint8_t *inl)
{
    if (n < 4) { memset(inl, 0, (size_t)n); return -1; }
    int32_t *tab = malloc(sizeof(int32_t) * 4 * (size_t)(iters > 0 ? iters : 1));
    vfo_ransac_samples(seed, n, iters, tab);
    uint8_t *cur = malloc((size_t)n), *best = malloc((size_t)n);
    int64_t best_count = 0;
    int have = 0;
    for (int k = 0; k < iters; k++) {
        double s4[8], d4[8], h[9];
        for (int q = 0; q < 4; q++) {
            int32_t i = tab[4 * k + q];
            s4[2 * q] = src[2 * i]; s4[2 * q + 1] = src[2 * i + 1];
            d4[2 * q] = dst[2 * i]; d4[2 * q + 1] = dst[2 * i + 1];
        }
        if (!vfo_dlt(s4, d4, 4, h) || !vfo_usable(h)) continue;
        int64_t c = vfo_inliers(h, src, dst, n, tol, cur);
        if (c > best_count) { best_count = c; memcpy(best, cur, (size_t)n); have = 1; }
    }
    int64_t result = -1;
    if (have && best_count >= 4) {
        double *bs = malloc(sizeof(double) * 2 * (size_t)best_count), *bd = malloc(sizeof(double) * 2 * (size_t)best_count);
        int64_t m = 0;
        for (int64_t i = 0; i < n; i++)
            if (best[i]) { bs[2 * m] = src[2 * i]; bs[2 * m + 1] = src[2 * i + 1];
                           bd[2 * m] = dst[2 * i]; bd[2 * m + 1] = dst[2 * i + 1]; m++; }
        double h[9];
        if (vfo_dlt(bs, bd, (int)m, h) && vfo_usable(h)) {
            result = vfo_inliers(h, src, dst, n, tol, inl);
            memcpy(h_out, h, sizeof h);
        }
        free(bs); free(bd);
    }
    if (result < 0) memset(inl, 0, (size_t)n);
    free(tab); free(cur); free(best);
    return result;
}
