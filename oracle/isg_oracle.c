/*
 * isg_oracle.c — CPU oracle for the isotropic-splat hot path.
 *
 *   *** TEST INFRASTRUCTURE ONLY. ***  Only tests/, __graft_entry__.smoke() and bench.py's
 *   cpu_baseline / --impl reference legs may load this library, and only as the checker or
 *   the timed CPU baseline — never as the product path.  The product (libisg.so) has no CPU
 *   fallback and does not link this file.
 *
 * Two restatements of the reference algorithm live here:
 *
 *  (1) or64_*  — a LITERAL FP64 restatement of the reference forward path:
 *        project_iso          /root/reference/proj/src/splat3d.cpp:59-64
 *        Camera::to_camera / project_point  include/isosplat/splat3d.hpp:45-51
 *        composite            src/splat3d.cpp:76-87
 *        covers(ScreenIso)    src/splat3d.cpp:108-114
 *        composite_pixels     src/splat3d.cpp:125-162 (row bands, no early exit)
 *        sort_by_depth        src/splat3d.cpp:164-169 (stable, ties by index)
 *        render(iso)          src/splat3d.cpp:173-194
 *        brute_force_render   tools/isosplat_main.cpp:309-355
 *        mse                  src/image.cpp:50-58
 *      plus a first-principles FP64 backward (kernel closed forms
 *      include/isosplat/kernels.hpp:208-222, Jacobian src/splat3d.cpp:39-47) that is pinned
 *      by central finite differences of the FP64 forward in tests/.
 *
 *  (3) or64_image_loss — FP64 restatement of the paper's L1 + D-SSIM loss and its pixel
 *      gradient (src/loss.cpp:16-213), pinned against the reference's own compiled loss(),
 *      ssim() and ssim_gradient_wrt_second() (oracle/_ref) in tests/.
 *
 *  (2) or32_*  — the FP32 TILED restatement that the GPU path must match: the same
 *      arithmetic in IEEE single precision with every rounding spelled out (this file is
 *      compiled with -ffp-contract=off, as the reference is: proj/CMakeLists.txt:11-17),
 *      16x16 screen tiles, (tile, depth, index) ordered per-tile lists, optional early
 *      termination at transmittance t_min, the reverse-walk backward and Adam.  Tile keys,
 *      their order and the per-tile ranges produced here are the bit-exact parity target.
 *
 * Parity status: the forward is pinned against the reference's own known answers
 * and, when oracle/_ref is built, against the
 * reference's compiled render(); tiles/keys/ranges, backward and Adam have no reference
 * counterpart (SPEC.md:484 non-goals) and are pinned by construction, by finite
 * differences and by torch.optim.Adam respectively.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_TILE 16

/* Same layout as isg_camera in include/isg.h. */
typedef struct {
  float R[9];
  float t[3];
  float focal;
  float cx, cy;
  int32_t width, height;
} or_cam32;

typedef struct {
  double R[9];
  double t[3];
  double focal;
  double cx, cy;
  int32_t width, height;
} or_cam64;

int or_version(void) { return 1; }

static int resolve_threads(int threads) {
#ifdef _OPENMP
  return threads > 0 ? threads : omp_get_max_threads();
#else
  (void)threads;
  return 1;
#endif
}

/* ========================================================================================
 * (1) FP64 literal restatement
 * ====================================================================================== */

/* splat record: mu.xyz sigma color.rgb opacity (the ISPL iso-3D record order,
 * include/isosplat/particle_io.hpp:36-46). */

/* project_iso, src/splat3d.cpp:59-64.  Returns 1 and (u, v, sigma2d, depth) when z > near. */
int or64_project_iso(const double* s, const or_cam64* c, double* out) {
  /* to_camera: rotation * world + translation (hpp:45-47) */
  const double x = (c->R[0] * s[0] + c->R[1] * s[1]) + c->R[2] * s[2] + c->t[0];
  const double y = (c->R[3] * s[0] + c->R[4] * s[1]) + c->R[5] * s[2] + c->t[1];
  const double z = (c->R[6] * s[0] + c->R[7] * s[1]) + c->R[8] * s[2] + c->t[2];
  if (!(z > 1e-3)) return 0; /* kNearPlane, hpp:55 */
  out[0] = c->focal * x / z + c->cx; /* project_point hpp:48-51 */
  out[1] = c->focal * y / z + c->cy;
  out[2] = s[3] * c->focal / z; /* sigma_2d = sigma * f / z */
  out[3] = z;
  return 1;
}

/* composite, src/splat3d.cpp:76-87.  rgba: n x 4 (r, g, b, alpha).  Returns 1 on the
 * reference's domain error (alpha outside [0,1]). */
int or64_composite(int64_t n, const double* rgba, double* out) {
  double c0 = 0, c1 = 0, c2 = 0, T = 1.0;
  for (int64_t k = 0; k < n; ++k) {
    const double a = rgba[4 * k + 3];
    if (!(a >= 0.0 && a <= 1.0)) return 1;
    const double w = T * a;
    c0 += w * rgba[4 * k + 0];
    c1 += w * rgba[4 * k + 1];
    c2 += w * rgba[4 * k + 2];
    T *= 1.0 - a;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  return 0;
}

typedef struct {
  double depth;
  int64_t index;
} or_entry64;

static int cmp_entry64(const void* a, const void* b) {
  const or_entry64* x = (const or_entry64*)a;
  const or_entry64* y = (const or_entry64*)b;
  if (x->depth < y->depth) return -1;
  if (x->depth > y->depth) return 1;
  /* std::stable_sort keeps input order for equal depth (splat3d.cpp:164-169) */
  return (x->index > y->index) - (x->index < y->index);
}

typedef struct {
  double u, v, s2, r2max, c[3], o;
} or_screen64;

/* render(iso), src/splat3d.cpp:173-194 with composite_pixels :125-162.  The caller has
 * validated the splats and camera (splat3d.cpp:10-37).  out: H x W x 3. */
int or64_render(int64_t n, const double* splats, const or_cam64* cam, const double* bg,
                int threads, double* out) {
  or_entry64* ord = (or_entry64*)malloc(sizeof(or_entry64) * (size_t)(n > 0 ? n : 1));
  or_screen64* scr = (or_screen64*)malloc(sizeof(or_screen64) * (size_t)(n > 0 ? n : 1));
  int64_t m = 0;
  for (int64_t i = 0; i < n; ++i) {
    double p[4];
    if (!or64_project_iso(splats + 8 * i, cam, p)) continue; /* culled */
    ord[m].depth = p[3];
    ord[m].index = i;
    ++m;
  }
  qsort(ord, (size_t)m, sizeof(or_entry64), cmp_entry64);
  for (int64_t k = 0; k < m; ++k) {
    const double* s = splats + 8 * ord[k].index;
    double p[4];
    or64_project_iso(s, cam, p);
    scr[k].u = p[0];
    scr[k].v = p[1];
    scr[k].s2 = p[2] * p[2];
    scr[k].r2max = 9.0 * p[2] * p[2];
    scr[k].c[0] = s[4];
    scr[k].c[1] = s[5];
    scr[k].c[2] = s[6];
    scr[k].o = s[7];
  }
  const int W = cam->width, H = cam->height;
#pragma omp parallel for schedule(dynamic, 1) num_threads(resolve_threads(threads))
  for (int y = 0; y < H; ++y) {
    const double py = y + 0.5; /* pixel_center, image.hpp:33-34 */
    for (int x = 0; x < W; ++x) {
      const double px = x + 0.5;
      double c0 = 0, c1 = 0, c2 = 0, T = 1.0;
      for (int64_t k = 0; k < m; ++k) {
        const or_screen64* s = &scr[k];
        const double dx = px - s->u, dy = py - s->v;
        const double r2 = dx * dx + dy * dy;
        if (r2 > s->r2max) continue;
        const double g = exp(-r2 / s->s2);
        const double a = s->o * g;
        const double w = T * a;
        c0 += w * s->c[0];
        c1 += w * s->c[1];
        c2 += w * s->c[2];
        T *= 1.0 - a;
      }
      double* o = out + ((size_t)y * W + x) * 3;
      o[0] = c0 + T * bg[0];
      o[1] = c1 + T * bg[1];
      o[2] = c2 + T * bg[2];
    }
  }
  free(ord);
  free(scr);
  return 0;
}

/* brute_force_render, tools/isosplat_main.cpp:309-355: re-projects every splat per pixel. */
int or64_brute_force(int64_t n, const double* splats, const or_cam64* cam, const double* bg,
                     double* out) {
  or_entry64* ord = (or_entry64*)malloc(sizeof(or_entry64) * (size_t)(n > 0 ? n : 1));
  int64_t m = 0;
  for (int64_t i = 0; i < n; ++i) {
    const double* s = splats + 8 * i;
    const double z = (cam->R[6] * s[0] + cam->R[7] * s[1]) + cam->R[8] * s[2] + cam->t[2];
    if (z > 1e-3) {
      ord[m].depth = z;
      ord[m].index = i;
      ++m;
    }
  }
  qsort(ord, (size_t)m, sizeof(or_entry64), cmp_entry64);
  for (int y = 0; y < cam->height; ++y) {
    for (int x = 0; x < cam->width; ++x) {
      const double px = x + 0.5, py = y + 0.5;
      double c0 = 0, c1 = 0, c2 = 0, T = 1.0;
      for (int64_t k = 0; k < m; ++k) {
        const double* s = splats + 8 * ord[k].index;
        double p[4];
        or64_project_iso(s, cam, p);
        const double dx = px - p[0], dy = py - p[1];
        const double r2 = dx * dx + dy * dy;
        if (!(r2 <= 9.0 * p[2] * p[2])) continue;
        const double g = exp(-r2 / (p[2] * p[2]));
        const double a = s[7] * g;
        const double w = T * a;
        c0 += w * s[4];
        c1 += w * s[5];
        c2 += w * s[6];
        T *= 1.0 - a;
      }
      double* o = out + ((size_t)y * cam->width + x) * 3;
      o[0] = c0 + T * bg[0];
      o[1] = c1 + T * bg[1];
      o[2] = c2 + T * bg[2];
    }
  }
  free(ord);
  return 0;
}

/* mse, src/image.cpp:50-58 */
double or64_mse(int64_t count, const double* a, const double* b) {
  double acc = 0.0;
  for (int64_t i = 0; i < count; ++i) {
    const double d = a[i] - b[i];
    acc += d * d;
  }
  return acc / (double)count;
}

/* FP64 loss = weight * mse(render, target) and its gradient w.r.t. every splat parameter
 * (n x 8: dmu.xyz dsigma drgb dopacity), with no early termination (exact reference
 * forward).  First-principles chain rule; the per-pixel transmittance
 * is stored during the forward walk, so no division is involved (an independent check of
 * the division-based reverse walk used on FP32/GPU). */
int or64_loss_grad(int64_t n, const double* splats, const or_cam64* cam, const double* bg,
                   const double* target, double weight, double* loss_out, double* grads) {
  const int W = cam->width, H = cam->height;
  or_entry64* ord = (or_entry64*)malloc(sizeof(or_entry64) * (size_t)(n > 0 ? n : 1));
  double* proj = (double*)malloc(sizeof(double) * 4 * (size_t)(n > 0 ? n : 1));
  double* d2 = (double*)calloc((size_t)(n > 0 ? n : 1) * 4, sizeof(double)); /* du dv ds do */
  int64_t m = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (!or64_project_iso(splats + 8 * i, cam, proj + 4 * i)) continue;
    ord[m].depth = proj[4 * i + 3];
    ord[m].index = i;
    ++m;
  }
  qsort(ord, (size_t)m, sizeof(or_entry64), cmp_entry64);
  memset(grads, 0, sizeof(double) * 8 * (size_t)n);
  int64_t* list = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m > 0 ? m : 1));
  double* Tk = (double*)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
  double* gk = (double*)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
  const double scale = weight / (3.0 * W * H);
  double loss = 0.0;
  for (int y = 0; y < H; ++y) {
    for (int x = 0; x < W; ++x) {
      const double px = x + 0.5, py = y + 0.5;
      int64_t L = 0;
      double C[3] = {0, 0, 0}, T = 1.0;
      for (int64_t k = 0; k < m; ++k) {
        const int64_t i = ord[k].index;
        const double* p = proj + 4 * i;
        const double dx = px - p[0], dy = py - p[1];
        const double r2 = dx * dx + dy * dy;
        if (r2 > 9.0 * p[2] * p[2]) continue;
        const double g = exp(-r2 / (p[2] * p[2]));
        const double a = splats[8 * i + 7] * g;
        list[L] = i;
        Tk[L] = T;
        gk[L] = g;
        ++L;
        for (int c = 0; c < 3; ++c) C[c] += T * a * splats[8 * i + 4 + c];
        T *= 1.0 - a;
      }
      double G[3];
      const double* tg = target + ((size_t)y * W + x) * 3;
      for (int c = 0; c < 3; ++c) {
        C[c] += T * bg[c];
        const double d = C[c] - tg[c];
        loss += d * d;
        G[c] = 2.0 * d * scale;
      }
      double A[3] = {bg[0], bg[1], bg[2]};
      for (int64_t l = L - 1; l >= 0; --l) {
        const int64_t i = list[l];
        const double* s = splats + 8 * i;
        const double* p = proj + 4 * i;
        const double g = gk[l], o = s[7], a = o * g, Tl = Tk[l];
        double dLda = 0.0;
        for (int c = 0; c < 3; ++c) {
          dLda += G[c] * Tl * (s[4 + c] - A[c]);
          grads[8 * i + 4 + c] += G[c] * Tl * a; /* dC/dc = T a */
        }
        for (int c = 0; c < 3; ++c) A[c] = a * s[4 + c] + (1.0 - a) * A[c];
        grads[8 * i + 7] += dLda * g; /* d alpha / d opacity = g */
        const double dLdg = dLda * o;
        const double dx = px - p[0], dy = py - p[1], s2 = p[2] * p[2];
        d2[4 * i + 0] += dLdg * g * 2.0 * dx / s2; /* kernels.hpp:219 */
        d2[4 * i + 1] += dLdg * g * 2.0 * dy / s2;
        d2[4 * i + 2] += dLdg * g * 2.0 * (dx * dx + dy * dy) / (s2 * p[2]); /* kernels.hpp:220 */
      }
    }
  }
  /* projection backward: u = f x/z + cx, v = f y/z + cy, s = sigma f / z  (splat3d.cpp:39-47) */
  for (int64_t i = 0; i < n; ++i) {
    const double* s = splats + 8 * i;
    const double x = (cam->R[0] * s[0] + cam->R[1] * s[1]) + cam->R[2] * s[2] + cam->t[0];
    const double yv = (cam->R[3] * s[0] + cam->R[4] * s[1]) + cam->R[5] * s[2] + cam->t[1];
    const double z = (cam->R[6] * s[0] + cam->R[7] * s[1]) + cam->R[8] * s[2] + cam->t[2];
    if (!(z > 1e-3)) continue;
    const double f = cam->focal, du = d2[4 * i], dv = d2[4 * i + 1], ds = d2[4 * i + 2];
    const double gx = du * f / z, gy = dv * f / z;
    const double gz = -(du * f * x + dv * f * yv + ds * s[3] * f) / (z * z);
    grads[8 * i + 0] = cam->R[0] * gx + cam->R[3] * gy + cam->R[6] * gz;
    grads[8 * i + 1] = cam->R[1] * gx + cam->R[4] * gy + cam->R[7] * gz;
    grads[8 * i + 2] = cam->R[2] * gx + cam->R[5] * gy + cam->R[8] * gz;
    grads[8 * i + 3] = ds * f / z;
  }
  *loss_out = loss * (weight / (3.0 * W * H));
  free(ord);
  free(proj);
  free(d2);
  free(list);
  free(Tk);
  free(gk);
  return 0;
}

/* ========================================================================================
 * (2) FP32 tiled restatement (the GPU parity target)
 * ====================================================================================== */

typedef struct {
  float u, v, s, s2, r2max, c[3], o;
  float xc, yc, zc;
  int vis;
} or_rec32;

/* Projection in FP32 with every rounding explicit (-ffp-contract=off).  The CUDA kernel
 * performs the identical sequence with __fmul_rn/__fadd_rn/__fdiv_rn. */
static void or32_project(const float* ms, const float* co, const or_cam32* c, or_rec32* r) {
  const float mx = ms[0], my = ms[1], mz = ms[2], sg = ms[3];
  float xc = c->R[0] * mx;
  xc = xc + c->R[1] * my;
  xc = xc + c->R[2] * mz;
  xc = xc + c->t[0];
  float yc = c->R[3] * mx;
  yc = yc + c->R[4] * my;
  yc = yc + c->R[5] * mz;
  yc = yc + c->t[1];
  float zc = c->R[6] * mx;
  zc = zc + c->R[7] * my;
  zc = zc + c->R[8] * mz;
  zc = zc + c->t[2];
  r->xc = xc;
  r->yc = yc;
  r->zc = zc;
  r->vis = zc > 1e-3f; /* kNearPlane */
  const float fx = c->focal * xc, fy = c->focal * yc, fs = sg * c->focal;
  r->u = fx / zc + c->cx;
  r->v = fy / zc + c->cy;
  r->s = fs / zc;
  r->s2 = r->s * r->s;
  r->r2max = (9.0f * r->s) * r->s;
  r->c[0] = co[0];
  r->c[1] = co[1];
  r->c[2] = co[2];
  r->o = co[3];
}

/* Exact tile test: the pixel-centre rectangle of tile (tx,ty), clipped to the image, is
 * within the 3-sigma circle.  Conservative w.r.t. the per-pixel test (rounding is
 * monotone), so a tile that fails contains no covered pixel. */
static int or32_tile_hit(const or_rec32* r, int tx, int ty, int W, int H) {
  const float x0 = (float)(tx * OR_TILE) + 0.5f;
  const float x1 = (float)((tx * OR_TILE + OR_TILE < W ? tx * OR_TILE + OR_TILE : W) - 1) + 0.5f;
  const float y0 = (float)(ty * OR_TILE) + 0.5f;
  const float y1 = (float)((ty * OR_TILE + OR_TILE < H ? ty * OR_TILE + OR_TILE : H) - 1) + 0.5f;
  const float qx = r->u < x0 ? x0 : (r->u > x1 ? x1 : r->u);
  const float qy = r->v < y0 ? y0 : (r->v > y1 ? y1 : r->v);
  const float dx = qx - r->u, dy = qy - r->v;
  const float ddx = dx * dx, ddy = dy * dy;
  const float d2 = ddx + ddy;
  return !(d2 > r->r2max);
}

/* Conservative tile bounding box [tx0,tx1]x[ty0,ty1]; returns 0 if empty. */
static int or32_tile_bbox(const or_rec32* r, int tiles_x, int tiles_y, int* b) {
  const float ext = 3.0f * r->s * 1.0009765625f + 1.0f;
  float fx0 = floorf((r->u - ext) * (1.0f / OR_TILE));
  float fx1 = floorf((r->u + ext) * (1.0f / OR_TILE));
  float fy0 = floorf((r->v - ext) * (1.0f / OR_TILE));
  float fy1 = floorf((r->v + ext) * (1.0f / OR_TILE));
  fx0 = fmaxf(fx0, 0.0f);
  fy0 = fmaxf(fy0, 0.0f);
  fx1 = fminf(fx1, (float)(tiles_x - 1));
  fy1 = fminf(fy1, (float)(tiles_y - 1));
  if (!(fx0 <= fx1) || !(fy0 <= fy1)) return 0;
  b[0] = (int)fx0;
  b[1] = (int)fx1;
  b[2] = (int)fy0;
  b[3] = (int)fy1;
  return 1;
}

static uint32_t f32_bits(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  return u;
}

typedef struct {
  uint32_t z;
  uint32_t idx;
} or_zkey;

static int cmp_zkey(const void* a, const void* b) {
  const or_zkey* x = (const or_zkey*)a;
  const or_zkey* y = (const or_zkey*)b;
  if (x->z != y->z) return x->z < y->z ? -1 : 1;
  return (x->idx > y->idx) - (x->idx < y->idx);
}

typedef struct {
  int W, H, tx, ty, ntiles;
  int64_t n, nkeys, nvis;
  or_rec32* rec;
  uint32_t* vals;   /* nkeys splat indices, tile-major, depth order within a tile */
  uint32_t* ranges; /* ntiles x 2 */
} or_frame32;

static void or32_frame_free(or_frame32* f) {
  free(f->rec);
  free(f->vals);
  free(f->ranges);
}

/* Preprocess + binning: projection, tile sets, stable (tile, depth, index) order.  The
 * ordering is produced by a stable depth sort followed by a stable counting sort on the tile
 * — an algorithm independent of the GPU's radix sorts. */
static void or32_frame_build(int64_t n, const float* mu_sigma, const float* rgb_o,
                             const or_cam32* cam, or_frame32* f) {
  f->W = cam->width;
  f->H = cam->height;
  f->tx = (f->W + OR_TILE - 1) / OR_TILE;
  f->ty = (f->H + OR_TILE - 1) / OR_TILE;
  f->ntiles = f->tx * f->ty;
  f->n = n;
  f->rec = (or_rec32*)malloc(sizeof(or_rec32) * (size_t)(n > 0 ? n : 1));
  or_zkey* zk = (or_zkey*)malloc(sizeof(or_zkey) * (size_t)(n > 0 ? n : 1));
  int64_t m = 0;
  for (int64_t i = 0; i < n; ++i) {
    or32_project(mu_sigma + 4 * i, rgb_o + 4 * i, cam, &f->rec[i]);
    if (!f->rec[i].vis) continue;
    zk[m].z = f32_bits(f->rec[i].zc);
    zk[m].idx = (uint32_t)i;
    ++m;
  }
  qsort(zk, (size_t)m, sizeof(or_zkey), cmp_zkey);
  uint32_t* cnt = (uint32_t*)calloc((size_t)f->ntiles + 1, sizeof(uint32_t));
  int64_t total = 0, nvis = 0;
  for (int pass = 0; pass < 2; ++pass) {
    uint32_t* cursor = NULL;
    if (pass == 1) {
      f->vals = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(total > 0 ? total : 1));
      f->ranges = (uint32_t*)malloc(sizeof(uint32_t) * 2 * (size_t)f->ntiles);
      cursor = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)f->ntiles);
      uint32_t acc = 0;
      for (int t = 0; t < f->ntiles; ++t) {
        f->ranges[2 * t] = acc;
        cursor[t] = acc;
        acc += cnt[t];
        f->ranges[2 * t + 1] = acc;
      }
    }
    for (int64_t k = 0; k < m; ++k) {
      const or_rec32* r = &f->rec[zk[k].idx];
      int b[4];
      if (!or32_tile_bbox(r, f->tx, f->ty, b)) continue;
      int hit = 0;
      for (int ty = b[2]; ty <= b[3]; ++ty)
        for (int tx = b[0]; tx <= b[1]; ++tx) {
          if (!or32_tile_hit(r, tx, ty, f->W, f->H)) continue;
          const int t = ty * f->tx + tx;
          hit = 1;
          if (pass == 0) {
            cnt[t]++;
            total++;
          } else {
            f->vals[cursor[t]++] = zk[k].idx;
          }
        }
      if (pass == 0 && hit) nvis++;
    }
    free(cursor);
  }
  f->nkeys = total;
  f->nvis = nvis;
  free(cnt);
  free(zk);
}

/* Binning output for the parity hook: keys (tile<<32 | float_bits(depth)) in sorted order,
 * splat index per key, per-tile [start,end).  Returns the key count; arrays are written only
 * when the count fits in cap (callers re-query with a larger buffer). */
int64_t or32_bin(int64_t n, const float* mu_sigma, const float* rgb_o, const or_cam32* cam,
                 uint64_t* keys, uint32_t* vals, int64_t cap, uint32_t* ranges,
                 int64_t* n_visible) {
  or_frame32 f;
  or32_frame_build(n, mu_sigma, rgb_o, cam, &f);
  if (n_visible) *n_visible = f.nvis;
  if (f.nkeys <= cap) {
    for (int t = 0; t < f.ntiles; ++t)
      for (uint32_t p = f.ranges[2 * t]; p < f.ranges[2 * t + 1]; ++p) {
        if (keys) keys[p] = ((uint64_t)t << 32) | f32_bits(f.rec[f.vals[p]].zc);
        if (vals) vals[p] = f.vals[p];
      }
    if (ranges) memcpy(ranges, f.ranges, sizeof(uint32_t) * 2 * (size_t)f.ntiles);
  }
  const int64_t k = f.nkeys;
  or32_frame_free(&f);
  return k;
}

/* Front-to-back blend of one pixel over its tile list (composite_pixels semantics,
 * splat3d.cpp:136-143) with early termination once T <= t_min.  Returns entries processed. */
static uint32_t or32_blend_pixel(const or_frame32* f, uint32_t beg, uint32_t end, float px,
                                 float py, const float* bg, float t_min, float* out,
                                 float* t_last, int64_t* evaluated, int64_t* inside) {
  float C0 = 0.f, C1 = 0.f, C2 = 0.f, T = 1.f, Tl = 1.f;
  uint32_t nproc = 0;
  int64_t ev = 0, in = 0;
  for (uint32_t p = beg; p < end; ++p) {
    const or_rec32* r = &f->rec[f->vals[p]];
    ++ev;
    const float dx = px - r->u, dy = py - r->v;
    const float ddx = dx * dx, ddy = dy * dy;
    const float r2 = ddx + ddy;
    if (r2 > r->r2max) continue;
    ++in;
    const float g = expf(-r2 / r->s2);
    const float a = r->o * g;
    const float w = T * a;
    C0 += w * r->c[0];
    C1 += w * r->c[1];
    C2 += w * r->c[2];
    Tl = T;
    T = T * (1.0f - a);
    nproc = p - beg + 1;
    if (!(T > t_min)) break;
  }
  out[0] = C0 + T * bg[0];
  out[1] = C1 + T * bg[1];
  out[2] = C2 + T * bg[2];
  *t_last = Tl;
  if (evaluated) *evaluated += ev;
  if (inside) *inside += in;
  return nproc;
}

/* FP32 tiled render.  out: H x W x 3; t_last / n_proc (H x W, may be NULL) receive the
 * per-pixel transmittance before the last processed entry and the number of list entries
 * processed; counts (may be NULL) = {pairs evaluated, pairs inside the 3-sigma circle}. */
int or32_render(int64_t n, const float* mu_sigma, const float* rgb_o, const or_cam32* cam,
                const float* bg, float t_min, int threads, float* out, float* t_last,
                uint32_t* n_proc, int64_t* counts) {
  or_frame32 f;
  or32_frame_build(n, mu_sigma, rgb_o, cam, &f);
  int64_t ev = 0, in = 0;
#pragma omp parallel for schedule(dynamic, 4) num_threads(resolve_threads(threads)) \
    reduction(+ : ev, in)
  for (int t = 0; t < f.ntiles; ++t) {
    const int tx = t % f.tx, ty = t / f.tx;
    for (int y = ty * OR_TILE; y < ty * OR_TILE + OR_TILE && y < f.H; ++y)
      for (int x = tx * OR_TILE; x < tx * OR_TILE + OR_TILE && x < f.W; ++x) {
        const size_t pix = (size_t)y * f.W + x;
        float tl;
        const uint32_t np = or32_blend_pixel(&f, f.ranges[2 * t], f.ranges[2 * t + 1],
                                             (float)x + 0.5f, (float)y + 0.5f, bg, t_min,
                                             out + 3 * pix, &tl, &ev, &in);
        if (t_last) t_last[pix] = tl;
        if (n_proc) n_proc[pix] = np;
      }
  }
  if (counts) {
    counts[0] = ev;
    counts[1] = in;
  }
  or32_frame_free(&f);
  return 0;
}

/* FP32 tiled forward + L2 loss (weight * mse) + backward.  Gradients (n x 8, dmu.xyz dsigma
 * drgb dopacity) are ACCUMULATED into grads.  Per-(tile, entry) partial sums are reduced per
 * splat in key order, so the result is independent of the thread count.  out_img (may be
 * NULL) receives the forward image. */
static int or32_backward_impl(int64_t n, const float* mu_sigma, const float* rgb_o,
                              const or_cam32* cam, const float* bg, float t_min,
                              const float* target, const float* dldc, float weight, int threads,
                              double* loss_out, float* grads, float* out_img) {
  or_frame32 f;
  or32_frame_build(n, mu_sigma, rgb_o, cam, &f);
  float* part = (float*)calloc((size_t)(f.nkeys > 0 ? f.nkeys : 1) * 7, sizeof(float));
  double* tile_loss = (double*)calloc((size_t)f.ntiles, sizeof(double));
  const float scale = weight / (3.0f * (float)f.W * (float)f.H);
#pragma omp parallel for schedule(dynamic, 4) num_threads(resolve_threads(threads))
  for (int t = 0; t < f.ntiles; ++t) {
    const int tx = t % f.tx, ty = t / f.tx;
    const uint32_t beg = f.ranges[2 * t], end = f.ranges[2 * t + 1];
    double tl_acc = 0.0;
    for (int y = ty * OR_TILE; y < ty * OR_TILE + OR_TILE && y < f.H; ++y)
      for (int x = tx * OR_TILE; x < tx * OR_TILE + OR_TILE && x < f.W; ++x) {
        const size_t pix = (size_t)y * f.W + x;
        const float px = (float)x + 0.5f, py = (float)y + 0.5f;
        float C[3], Tl;
        const uint32_t np = or32_blend_pixel(&f, beg, end, px, py, bg, t_min, C, &Tl, NULL, NULL);
        if (out_img) memcpy(out_img + 3 * pix, C, sizeof C);
        float G[3];
        for (int c = 0; c < 3; ++c) {
          if (dldc) {
            G[c] = dldc[3 * pix + c];
          } else {
            const float d = C[c] - target[3 * pix + c];
            tl_acc += (double)d * (double)d;
            G[c] = 2.0f * d * scale;
          }
        }
        float A0 = bg[0], A1 = bg[1], A2 = bg[2], Tc = Tl;
        int first = 1;
        for (uint32_t q = np; q-- > 0;) {
          const uint32_t p = beg + q;
          const or_rec32* r = &f.rec[f.vals[p]];
          const float dx = px - r->u, dy = py - r->v;
          const float ddx = dx * dx, ddy = dy * dy;
          const float r2 = ddx + ddy;
          if (r2 > r->r2max) continue;
          const float g = expf(-r2 / r->s2);
          const float a = r->o * g;
          float T;
          if (first) {
            T = Tc;
            first = 0;
          } else {
            T = Tc / (1.0f - a);
          }
          Tc = T;
          const float dLda = T * ((G[0] * (r->c[0] - A0) + G[1] * (r->c[1] - A1)) +
                                  G[2] * (r->c[2] - A2));
          const float Ta = T * a;
          float* pp = part + 7 * (size_t)p;
          pp[4] += G[0] * Ta;
          pp[5] += G[1] * Ta;
          pp[6] += G[2] * Ta;
          A0 = a * r->c[0] + (1.0f - a) * A0;
          A1 = a * r->c[1] + (1.0f - a) * A1;
          A2 = a * r->c[2] + (1.0f - a) * A2;
          pp[3] += dLda * g;
          const float k2 = (dLda * r->o) * g * 2.0f / r->s2;
          pp[0] += k2 * dx;
          pp[1] += k2 * dy;
          pp[2] += k2 * r2 / r->s;
        }
      }
    tile_loss[t] = tl_acc;
  }
  /* per-splat reduction of the 2D partials, in key order */
  float* d2 = (float*)calloc((size_t)(n > 0 ? n : 1) * 7, sizeof(float));
  for (int64_t p = 0; p < f.nkeys; ++p) {
    float* dst = d2 + 7 * (size_t)f.vals[p];
    const float* src = part + 7 * (size_t)p;
    for (int j = 0; j < 7; ++j) dst[j] += src[j];
  }
  /* projection backward (splat3d.cpp:39-47 Jacobian) */
  for (int64_t i = 0; i < n; ++i) {
    const or_rec32* r = &f.rec[i];
    if (!r->vis) continue;
    const float* s = d2 + 7 * (size_t)i;
    const float fz = cam->focal / r->zc;
    const float gx = s[0] * fz, gy = s[1] * fz;
    const float gz = -(((s[0] * r->xc + s[1] * r->yc) + s[2] * mu_sigma[4 * i + 3]) * fz) / r->zc;
    float* gd = grads + 8 * (size_t)i;
    gd[0] += (cam->R[0] * gx + cam->R[3] * gy) + cam->R[6] * gz;
    gd[1] += (cam->R[1] * gx + cam->R[4] * gy) + cam->R[7] * gz;
    gd[2] += (cam->R[2] * gx + cam->R[5] * gy) + cam->R[8] * gz;
    gd[3] += s[2] * fz;
    gd[4] += s[4];
    gd[5] += s[5];
    gd[6] += s[6];
    gd[7] += s[3];
  }
  double loss = 0.0;
  for (int t = 0; t < f.ntiles; ++t) loss += tile_loss[t];
  if (loss_out) *loss_out = loss * ((double)weight / (3.0 * f.W * f.H));
  free(d2);
  free(part);
  free(tile_loss);
  or32_frame_free(&f);
  return 0;
}

int or32_loss_backward(int64_t n, const float* mu_sigma, const float* rgb_o, const or_cam32* cam,
                       const float* bg, float t_min, const float* target, float weight,
                       int threads, double* loss_out, float* grads, float* out_img) {
  return or32_backward_impl(n, mu_sigma, rgb_o, cam, bg, t_min, target, NULL, weight, threads,
                            loss_out, grads, out_img);
}

/* The same backward with a given pixel gradient dL/dC (HWC3, weight included), e.g. of the
 * L1 + D-SSIM loss below.  Gradients are ACCUMULATED into grads. */
int or32_backward_dldc(int64_t n, const float* mu_sigma, const float* rgb_o, const or_cam32* cam,
                       const float* bg, float t_min, const float* dldc, int threads,
                       float* grads) {
  return or32_backward_impl(n, mu_sigma, rgb_o, cam, bg, t_min, NULL, dldc, 1.0f, threads, NULL,
                            grads, NULL);
}

/* ============================================================================================
 * (3) L1 + D-SSIM image loss, FP64 — a literal restatement of /root/reference/proj/src/loss.cpp
 * ============================================================================================ */
#define OR_WIN 11
#define OR_HALF 5

static void or_ssim_taps(double t[OR_WIN]) { /* window_taps, loss.cpp:22-35 */
  double sum = 0.0;
  for (int i = 0; i < OR_WIN; ++i) {
    const double d = i - OR_HALF;
    t[i] = exp(-d * d / (2.0 * 1.5 * 1.5));
    sum += t[i];
  }
  for (int i = 0; i < OR_WIN; ++i) t[i] /= sum;
}

/* filter, loss.cpp:49-72: separable correlation, zero padded (clipped tap range) */
static void or_filter(const double* w, const double* in, int W, int H, double* tmp, double* out) {
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x) {
      double acc = 0.0;
      const int d0 = x - OR_HALF < 0 ? -x : -OR_HALF;
      const int d1 = W - 1 - x < OR_HALF ? W - 1 - x : OR_HALF;
      for (int d = d0; d <= d1; ++d) acc += w[d + OR_HALF] * in[(size_t)y * W + x + d];
      tmp[(size_t)y * W + x] = acc;
    }
  memset(out, 0, sizeof(double) * (size_t)W * H);
  for (int y = 0; y < H; ++y) {
    const int d0 = y - OR_HALF < 0 ? -y : -OR_HALF;
    const int d1 = H - 1 - y < OR_HALF ? H - 1 - y : OR_HALF;
    for (int d = d0; d <= d1; ++d) {
      const double wd = w[d + OR_HALF];
      for (int x = 0; x < W; ++x) out[(size_t)y * W + x] += wd * tmp[(size_t)(y + d) * W + x];
    }
  }
}

/* loss(f, fhat, lambda) (loss.cpp:184-190) of HWC3 images f (target) and fhat, times weight,
 * and optionally dL/dfhat (loss_pixel_gradient :201-213 with ssim_gradient_wrt_second
 * :143-182), times weight.  Returns 0, -1 for lambda outside [0,1], -2 for an image smaller
 * than the window when lambda > 0. */
int or64_image_loss(int W, int H, const double* f, const double* fhat, double lambda,
                    double weight, double* loss_out, double* dldfhat) {
  if (!(lambda >= 0.0 && lambda <= 1.0)) return -1;
  const size_t P = (size_t)W * H, N = 3 * P;
  double l1 = 0.0;
  for (size_t i = 0; i < N; ++i) l1 += fabs(f[i] - fhat[i]);
  l1 /= (double)N;
  if (dldfhat) {
    const double w1 = (1.0 - lambda) / (double)N;
    for (size_t i = 0; i < N; ++i) {
      const double r = fhat[i] - f[i];
      dldfhat[i] = r > 0.0 ? w1 : (r < 0.0 ? -w1 : 0.0);
    }
  }
  if (lambda == 0.0) {
    *loss_out = weight * l1;
    if (dldfhat)
      for (size_t i = 0; i < N; ++i) dldfhat[i] *= weight;
    return 0;
  }
  if (W < OR_WIN || H < OR_WIN) return -2;
  double w[OR_WIN];
  or_ssim_taps(w);
  const double C1 = 0.01 * 0.01, C2 = 0.03 * 0.03;
  double* buf = (double*)malloc(sizeof(double) * P * 16);
  double *a = buf, *b = buf + P, *m1 = buf + 2 * P, *m2 = buf + 3 * P, *t1 = buf + 4 * P,
         *t2 = buf + 5 * P, *t12 = buf + 6 * P, *tmp = buf + 7 * P, *prod = buf + 8 * P,
         *gm2 = buf + 9 * P, *gt2 = buf + 10 * P, *gt12 = buf + 11 * P, *f1 = buf + 12 * P,
         *f2 = buf + 13 * P, *f3 = buf + 14 * P;
  const double norm = 1.0 / ((double)(W - 2 * OR_HALF) * (H - 2 * OR_HALF) * 3);
  double total = 0.0;
  for (int c = 0; c < 3; ++c) {
    for (size_t i = 0; i < P; ++i) {
      a[i] = f[3 * i + c];
      b[i] = fhat[3 * i + c];
    }
    /* ssim_terms, loss.cpp:86-102 */
    or_filter(w, a, W, H, tmp, m1);
    or_filter(w, b, W, H, tmp, m2);
    for (size_t i = 0; i < P; ++i) prod[i] = a[i] * a[i];
    or_filter(w, prod, W, H, tmp, t1);
    for (size_t i = 0; i < P; ++i) prod[i] = b[i] * b[i];
    or_filter(w, prod, W, H, tmp, t2);
    for (size_t i = 0; i < P; ++i) prod[i] = a[i] * b[i];
    or_filter(w, prod, W, H, tmp, t12);
    double acc = 0.0;
    memset(gm2, 0, sizeof(double) * P * 3);
    for (int y = OR_HALF; y < H - OR_HALF; ++y)
      for (int x = OR_HALF; x < W - OR_HALF; ++x) {
        const size_t i = (size_t)y * W + x;
        const double s11 = t1[i] - m1[i] * m1[i], s22 = t2[i] - m2[i] * m2[i],
                     s12 = t12[i] - m1[i] * m2[i];
        const double nl = 2.0 * m1[i] * m2[i] + C1, dl = m1[i] * m1[i] + m2[i] * m2[i] + C1;
        const double nc = 2.0 * s12 + C2, dc = s11 + s22 + C2;
        acc += (nl * nc) / (dl * dc); /* ssim, :128-137 */
        const double lum = nl / dl, cs = nc / dc; /* :159-170 */
        const double d_s22 = -lum * nc / (dc * dc), d_s12 = lum * 2.0 / dc;
        const double d_lum_m2 = (2.0 * m1[i] * dl - nl * 2.0 * m2[i]) / (dl * dl);
        gm2[i] = cs * d_lum_m2 + d_s22 * (-2.0 * m2[i]) + d_s12 * (-m1[i]);
        gt2[i] = d_s22;
        gt12[i] = d_s12;
      }
    total += acc / ((double)(W - 2 * OR_HALF) * (H - 2 * OR_HALF));
    if (dldfhat) {
      or_filter(w, gm2, W, H, tmp, f1);
      or_filter(w, gt2, W, H, tmp, f2);
      or_filter(w, gt12, W, H, tmp, f3);
      for (size_t i = 0; i < P; ++i) /* :174-179, then loss_pixel_gradient :210 */
        dldfhat[3 * i + c] -= lambda * (norm * (f1[i] + 2.0 * b[i] * f2[i] + a[i] * f3[i]));
    }
  }
  free(buf);
  const double ssim = total / 3.0;
  *loss_out = weight * ((1.0 - lambda) * l1 + lambda * (1.0 - ssim));
  if (dldfhat)
    for (size_t i = 0; i < N; ++i) dldfhat[i] *= weight;
  return 0;
}

/* Optimizer-space state of a set of splats: raw = (log sigma, logit opacity), the opacity
 * first taken into [1e-6, 1 - 1e-6] (logit(0), logit(1) are infinite). */
#define OR_OPACITY_EPS 1e-6f
void or32_raw_init(int64_t n, const float* mu_sigma, const float* rgb_o, float* raw) {
  for (int64_t i = 0; i < n; ++i) {
    float op = rgb_o[4 * i + 3];
    op = fminf(fmaxf(op, OR_OPACITY_EPS), 1.0f - OR_OPACITY_EPS);
    raw[2 * i] = logf(mu_sigma[4 * i + 3]);
    raw[2 * i + 1] = logf(op) - log1pf(-op);
  }
}

/* Adam (torch.optim.Adam semantics, no weight decay) on the optimizer-space parameters
 * (mu, log sigma, rgb, logit opacity) with per-group learning rates lr[4].  sigma moves in
 * log space as in update_step (optimize.cpp:93,105); a Gaussian whose 8 gradients are not
 * all finite is skipped and counted (optimize.cpp:87-90).  m, v: n x 8; step >= 1.
 * raw (n x 2): the persistent (log sigma, logit opacity) -- like torch's own parameters, they
 * are never re-derived from sigma / opacity; sigma = exp(raw.x), opacity = sigmoid(raw.y) are
 * rewritten only when their raw value moved.  An update is exactly 0 when m is 0. */
void or32_adam(int64_t n, float* mu_sigma, float* rgb_o, float* raw, float* m, float* v,
               const float* grads, int64_t step, const float* lr, float b1, float b2, float eps,
               int64_t* skipped) {
  const double bc1 = 1.0 - pow((double)b1, (double)step);
  const double bc2 = 1.0 - pow((double)b2, (double)step);
  const float bc2_sqrt = (float)sqrt(bc2);
  float step_size[4];
  for (int j = 0; j < 4; ++j) step_size[j] = (float)((double)lr[j] / bc1);
  static const int group[8] = {0, 0, 0, 1, 2, 2, 2, 3};
  int64_t skip = 0;
  for (int64_t i = 0; i < n; ++i) {
    const float* gr = grads + 8 * (size_t)i;
    int ok = 1;
    for (int j = 0; j < 8; ++j) ok &= isfinite(gr[j]) ? 1 : 0;
    if (!ok) {
      ++skip;
      continue;
    }
    float* ms = mu_sigma + 4 * (size_t)i;
    float* co = rgb_o + 4 * (size_t)i;
    float* R = raw + 2 * (size_t)i;
    const float sigma = ms[3];
    const float s = 1.0f / (1.0f + expf(-R[1]));
    float p[8] = {ms[0], ms[1], ms[2], R[0], co[0], co[1], co[2], R[1]};
    float g[8] = {gr[0], gr[1], gr[2], gr[3] * sigma, gr[4], gr[5], gr[6], gr[7] * s * (1.0f - s)};
    for (int j = 0; j < 8; ++j) {
      float* mm = m + 8 * (size_t)i + j;
      float* vv = v + 8 * (size_t)i + j;
      *mm = *mm + (1.0f - b1) * (g[j] - *mm);
      *vv = b2 * *vv + (1.0f - b2) * g[j] * g[j];
      const float denom = sqrtf(*vv) / bc2_sqrt + eps;
      const float upd = *mm == 0.0f ? 0.0f : *mm / denom;
      p[j] = p[j] - step_size[group[j]] * upd;
    }
    ms[0] = p[0];
    ms[1] = p[1];
    ms[2] = p[2];
    if (p[3] != R[0]) ms[3] = expf(p[3]);
    co[0] = p[4];
    co[1] = p[5];
    co[2] = p[6];
    if (p[7] != R[1]) co[3] = 1.0f / (1.0f + expf(-p[7]));
    R[0] = p[3];
    R[1] = p[7];
  }
  if (skipped) *skipped += skip;
}

/* ============================================================================================
 * (4) Adaptive control (prune / merge / split), /root/reference/proj/src/optimize.cpp:150-284.
 *
 * One control flow (prune_impl :153-174, adaptive_control :221-284), two rule sets:
 *   dims == 2  the reference's IsoParticle2D rules verbatim (records mu.x mu.y sigma A0 A1 A2):
 *              prune on max-channel |A| (:47-51), merge weights luminance(A) pi sigma^2 with
 *              per-channel zeroth-moment conservation (:200-219, luminance :19-22)
 *   dims == 3  the isotropic 3D splat rules the GPU implements (records mu.xyz sigma r g b o):
 *              prune on opacity; merge weights w = o sigma^2 (screen-footprint mass),
 *              mu / sigma^2 / colour w-weighted, o = min(1, (w1 + w2) / sigma^2) (footprint mass
 *              conserved); split children at mu +- (sigma/2) d, sigma / sqrt(2), colour and
 *              opacity kept, d a unit direction from Marsaglia's method on a splitmix64 stream
 *              keyed by (seed, round, parent index) — no transcendental functions, so the GPU
 *              reproduces it bit for bit; every 3D result is rounded to FP32 at the end.
 * Pairs qualify when |mu_i - mu_j| < gamma min(sigma) and the max colour difference < tol
 * (:232-244); they are taken greedily nearest-first on (dist, i, j) (:246-259), one merge per
 * particle, a refused merge still consumes both; splits go widest first, ties by higher index,
 * while the count stays <= max_particles (:266-281).  Returns the new count (<= out_cap).
 * ============================================================================================ */
typedef struct {
  double prune_threshold, merge_distance_factor, merge_color_tol, split_sigma_max;
  int64_t max_particles;
} or_adapt_params;

typedef struct {
  double dist;
  int64_t i, j;
} or_pair;

static int cmp_pair(const void* a, const void* b) {
  const or_pair *x = (const or_pair*)a, *y = (const or_pair*)b;
  if (x->dist != y->dist) return x->dist < y->dist ? -1 : 1;
  if (x->i != y->i) return x->i < y->i ? -1 : 1;
  if (x->j != y->j) return x->j < y->j ? -1 : 1;
  return 0;
}

static uint64_t or_splitmix(uint64_t* s) {
  uint64_t z = (*s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* Unit direction for splitting parent `index` (Marsaglia 1972). */
void or_split_direction(uint64_t seed, uint64_t round, uint64_t index, double d[3]) {
  uint64_t s = seed ^ (round * 0xD1B54A32D192ED03ull) ^ (index * 0xA24BAED4963EE407ull);
  for (;;) {
    const double u1 = (double)(or_splitmix(&s) >> 11) * 0x1.0p-52 - 1.0;
    const double u2 = (double)(or_splitmix(&s) >> 11) * 0x1.0p-52 - 1.0;
    const double q = u1 * u1 + u2 * u2;
    if (q >= 1.0 || q == 0.0) continue;
    const double f = 2.0 * sqrt(1.0 - q);
    d[0] = u1 * f;
    d[1] = u2 * f;
    d[2] = 1.0 - 2.0 * q;
    return;
  }
}

static double or_lum(const double* a, int channels) {
  if (channels == 1) return a[0];
  return 0.2126 * a[0] + 0.7152 * a[1] + 0.0722 * a[2];
}

static double or_prune_score(int dims, const double* r, int channels) {
  if (dims == 3) return r[7];
  double m = fabs(r[3]);
  for (int c = 1; c < channels; ++c) m = fabs(r[3 + c]) > m ? fabs(r[3 + c]) : m;
  return m;
}

static double or_color_diff(int dims, const double* a, const double* b, int channels) {
  const int off = dims == 3 ? 4 : 3, nc = dims == 3 ? 3 : channels;
  double m = 0.0;
  for (int c = 0; c < nc; ++c) {
    const double d = fabs(a[off + c] - b[off + c]);
    m = d > m ? d : m;
  }
  return m;
}

static double or_dist(int dims, const double* a, const double* b) {
  double s = 0.0;
  for (int k = 0; k < dims; ++k) {
    const double d = a[k] - b[k];
    s = s + d * d;
  }
  return sqrt(s);
}

static float f32(double x) { return (float)x; }

/* merge (optimize.cpp:200-219 for 2D; the 3D rule above).  Returns 0 when refused. */
static int or_merge(int dims, const double* p1, const double* p2, int channels, double* out) {
  if (dims == 2) {
    const double PI = 3.14159265358979323846;
    const double w1 = or_lum(p1 + 3, channels) * PI * p1[2] * p1[2];
    const double w2 = or_lum(p2 + 3, channels) * PI * p2[2] * p2[2];
    const double total = w1 + w2;
    if (fabs(total) < 1e-12) return 0;
    const double mx = (w1 * p1[0] + w2 * p2[0]) / total, my = (w1 * p1[1] + w2 * p2[1]) / total;
    const double s2 = (w1 * p1[2] * p1[2] + w2 * p2[2] * p2[2]) / total;
    if (!(s2 > 0.0) || !isfinite(s2) || !isfinite(mx) || !isfinite(my)) return 0;
    out[0] = mx;
    out[1] = my;
    out[2] = sqrt(s2);
    for (int c = 0; c < 3; ++c) out[3 + c] = 0.0;
    for (int c = 0; c < channels; ++c) {
      const double m1 = p1[3 + c] * PI * p1[2] * p1[2];
      const double m2 = p2[3 + c] * PI * p2[2] * p2[2];
      out[3 + c] = (m1 + m2) / (PI * s2);
    }
    return 1;
  }
  const double w1 = p1[7] * (p1[3] * p1[3]), w2 = p2[7] * (p2[3] * p2[3]);
  const double total = w1 + w2;
  if (fabs(total) < 1e-12) return 0;
  double mu[3];
  for (int k = 0; k < 3; ++k) mu[k] = (w1 * p1[k] + w2 * p2[k]) / total;
  const double s2 = (w1 * (p1[3] * p1[3]) + w2 * (p2[3] * p2[3])) / total;
  if (!(s2 > 0.0) || !isfinite(s2) || !isfinite(mu[0]) || !isfinite(mu[1]) || !isfinite(mu[2]))
    return 0;
  for (int k = 0; k < 3; ++k) out[k] = f32(mu[k]);
  out[3] = f32(sqrt(s2));
  for (int c = 0; c < 3; ++c) out[4 + c] = f32((w1 * p1[4 + c] + w2 * p2[4 + c]) / total);
  const double o = total / s2;
  out[7] = f32(o < 1.0 ? o : 1.0);
  if (!(out[3] > 0.0)) return 0; /* sigma underflowed in FP32 */
  return 1;
}

typedef struct {
  double sigma;
  int64_t idx;
} or_cand;

static int cmp_cand(const void* a, const void* b) { /* sigma desc, then index desc */
  const or_cand *x = (const or_cand*)a, *y = (const or_cand*)b;
  if (x->sigma != y->sigma) return x->sigma > y->sigma ? -1 : 1;
  if (x->idx != y->idx) return x->idx > y->idx ? -1 : 1;
  return 0;
}

int64_t or_adaptive_control(int dims, int64_t n, const double* in, const or_adapt_params* p,
                            int channels, uint64_t seed, uint64_t round, double* out,
                            int64_t out_cap, int64_t* counts /* pruned, merged, split */) {
  const int R = dims == 3 ? 8 : 6;
  const int sig = dims == 3 ? 3 : 2;
  if (n <= 0) return 0;
  /* prune (keep the best-scoring first index if nothing survives) */
  double* a = (double*)malloc(sizeof(double) * R * (size_t)n);
  int64_t m = 0, best = 0;
  double best_s = -1.0;
  for (int64_t i = 0; i < n; ++i) {
    const double s = or_prune_score(dims, in + R * i, channels);
    if (s > best_s) {
      best_s = s;
      best = i;
    }
  }
  for (int64_t i = 0; i < n; ++i)
    if (or_prune_score(dims, in + R * i, channels) >= p->prune_threshold)
      memcpy(a + R * m++, in + R * i, sizeof(double) * R);
  if (m == 0) memcpy(a + R * m++, in + R * best, sizeof(double) * R);
  if (counts) counts[0] = n - m;
  /* merge: all qualifying pairs, greedy nearest-first */
  int64_t np = 0, pcap = 1024;
  or_pair* pairs = (or_pair*)malloc(sizeof(or_pair) * pcap);
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = i + 1; j < m; ++j) {
      const double* pi = a + R * i;
      const double* pj = a + R * j;
      const double dist = or_dist(dims, pi, pj);
      const double smin = pi[sig] < pj[sig] ? pi[sig] : pj[sig];
      if (dist >= p->merge_distance_factor * smin) continue;
      if (or_color_diff(dims, pi, pj, channels) >= p->merge_color_tol) continue;
      if (np == pcap) pairs = (or_pair*)realloc(pairs, sizeof(or_pair) * (pcap *= 2));
      pairs[np].dist = dist;
      pairs[np].i = i;
      pairs[np].j = j;
      ++np;
    }
  qsort(pairs, (size_t)np, sizeof(or_pair), cmp_pair);
  char* used = (char*)calloc((size_t)m, 1);
  char* drop = (char*)calloc((size_t)m, 1);
  int64_t merged = 0;
  double tmp[8];
  for (int64_t k = 0; k < np; ++k) {
    const int64_t i = pairs[k].i, j = pairs[k].j;
    if (used[i] || used[j]) continue;
    used[i] = used[j] = 1;
    if (or_merge(dims, a + R * i, a + R * j, channels, tmp)) {
      memcpy(a + R * i, tmp, sizeof(double) * R);
      drop[j] = 1;
      ++merged;
    }
  }
  if (counts) counts[1] = merged;
  int64_t c = 0;
  for (int64_t i = 0; i < m; ++i)
    if (!drop[i] && c < out_cap) memcpy(out + R * c++, a + R * i, sizeof(double) * R);
  /* split: widest first while the budget allows */
  int64_t nc = 0;
  or_cand* cand = (or_cand*)malloc(sizeof(or_cand) * (size_t)(c > 0 ? c : 1));
  for (int64_t i = 0; i < c; ++i)
    if (out[R * i + sig] > p->split_sigma_max) {
      cand[nc].sigma = out[R * i + sig];
      cand[nc].idx = i;
      ++nc;
    }
  qsort(cand, (size_t)nc, sizeof(or_cand), cmp_cand);
  int64_t splits = 0;
  const int64_t base = c;
  for (int64_t k = 0; k < nc; ++k) {
    if (c + 1 > p->max_particles || c + 1 > out_cap) break;
    const int64_t i = cand[k].idx;
    double* par = out + R * i;
    double* ch = out + R * c;
    memcpy(ch, par, sizeof(double) * R);
    if (dims == 3) {
      double d[3];
      or_split_direction(seed, round, (uint64_t)i, d);
      const double h = 0.5 * par[3];
      for (int q = 0; q < 3; ++q) {
        const double off = h * d[q];
        ch[q] = f32(par[q] - off);
        par[q] = f32(par[q] + off);
      }
      par[3] = ch[3] = f32(par[3] * sqrt(0.5));
    } else {
      /* 2D: the reference draws phi from std::mt19937_64 (optimize.cpp:188-198); here the
       * direction is the 3D stream's (x, y) normalised — structure only, not the reference's
       * random numbers */
      double d[3];
      or_split_direction(seed, round, (uint64_t)i, d);
      const double nrm = sqrt(d[0] * d[0] + d[1] * d[1]);
      const double h = par[2] / 2.0;
      const double ox = nrm > 0 ? h * d[0] / nrm : h, oy = nrm > 0 ? h * d[1] / nrm : 0.0;
      ch[0] = par[0] - ox;
      ch[1] = par[1] - oy;
      par[0] = par[0] + ox;
      par[1] = par[1] + oy;
      par[2] = ch[2] = par[2] * sqrt(0.5);
    }
    ++c;
    ++splits;
  }
  (void)base;
  if (counts) counts[2] = splits;
  free(cand);
  free(used);
  free(drop);
  free(pairs);
  free(a);
  return c;
}

/* ============================================================================================
 * (5) The synthetic workload "isg-synth v1" -- restated here so the CPU arms of
 * bench.py and the tests build the same scenes and cameras without the product library (pinned
 * byte-equal to isg_synth_scene / isg_synth_camera in tests/test_oracle.py).  Counter-based:
 * splitmix64 finaliser of seed * phi + 8 i + j, top 24 bits. */
#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif
static uint64_t or_mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static double or_u01(uint64_t seed, uint64_t i, int j) {
  return (double)(or_mix64(seed * 0x9E3779B97F4A7C15ull + 8 * i + (uint64_t)j) >> 40) *
         (1.0 / 16777216.0);
}

/* z ~ U[2,10]; u ~ U[-5%, 105%] W, v ~ U[-5%, 105%] H back-projected through the identity
 * camera (f = 1000 W / 1920, principal point at the centre); sigma_2d ~ logU[0.5, 8] px;
 * opacity ~ U[0.05, 0.95]; rgb ~ U[0,1]^3. */
void or_synth_scene(uint64_t seed, int64_t n, int W, int H, float* ms, float* co) {
  const double f = 1000.0 * W / 1920.0, cx = 0.5 * W, cy = 0.5 * H;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    const double z = 2.0 + 8.0 * or_u01(seed, (uint64_t)i, 0);
    const double u = W * (-0.05 + 1.1 * or_u01(seed, (uint64_t)i, 1));
    const double v = H * (-0.05 + 1.1 * or_u01(seed, (uint64_t)i, 2));
    const double s2d = 0.5 * pow(16.0, or_u01(seed, (uint64_t)i, 3));
    ms[4 * i + 0] = (float)((u - cx) * z / f);
    ms[4 * i + 1] = (float)((v - cy) * z / f);
    ms[4 * i + 2] = (float)z;
    ms[4 * i + 3] = (float)(s2d * z / f);
    co[4 * i + 0] = (float)or_u01(seed, (uint64_t)i, 5);
    co[4 * i + 1] = (float)or_u01(seed, (uint64_t)i, 6);
    co[4 * i + 2] = (float)or_u01(seed, (uint64_t)i, 7);
    co[4 * i + 3] = (float)(0.05 + 0.9 * or_u01(seed, (uint64_t)i, 4));
  }
}

/* Camera k of an n-view batch: yaw (k - (n-1)/2) * 1.5 deg about y, t = (0.05 (k - (n-1)/2),
 * 0, 0); out = R[9] (row-major), t[3], focal, cx, cy as FP32 values (the FP32 camera). */
void or_synth_camera(int W, int H, int view, int n_views, float* out) {
  const double k = view - 0.5 * (n_views - 1);
  const double th = k * 1.5 * M_PI / 180.0;
  const double cs = cos(th), sn = sin(th);
  const double R[9] = {cs, 0, sn, 0, 1, 0, -sn, 0, cs};
  for (int i = 0; i < 9; ++i) out[i] = (float)R[i];
  out[9] = (float)(0.05 * k);
  out[10] = 0.0f;
  out[11] = 0.0f;
  out[12] = (float)(1000.0 * W / 1920.0);
  out[13] = (float)(0.5 * W);
  out[14] = (float)(0.5 * H);
}
