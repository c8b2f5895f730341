/*
 * C restatement of the reference attribution render -- TEST/BASELINE
 * INFRASTRUCTURE ONLY (see oracle/adpsplit_oracle.py header for the rules).
 *
 * Follows ref/raster.py:61-157 (visible_splats, project, _support_radius,
 * _alpha_map, render) in fp64: cull z <= 1e-8, EWA projection with the
 * 0.3 px^2 floor, support-radius bbox cull, stable (z, index) order,
 * alpha = min(0.99, o exp(-q/2)) zeroed below 1/255, front-to-back
 * composite with strict argmax of T*alpha, no early termination.  Like the
 * numpy oracle it composites each splat only over the pixel window outside
 * of which alpha is provably 0 (bit-identical to the full-image loop).
 *
 * Used to produce CPU-side inputs for the benchmark's reference arm at
 * sizes where the numpy oracle is too slow; tests check it against the
 * numpy oracle (which is pinned to the reference's golden vectors).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  double z;
  int idx;
  double mx, my, ca, cb, cc;
  double rgb[3];
} splat_t;

static int cmp_splat(const void* a, const void* b) {
  const splat_t* x = (const splat_t*)a;
  const splat_t* y = (const splat_t*)b;
  if (x->z < y->z) return -1;
  if (x->z > y->z) return 1;
  return (x->idx > y->idx) - (x->idx < y->idx);
}

static void quat_rot(const double* q4, double r[9]) {
  double n = sqrt(q4[0] * q4[0] + q4[1] * q4[1] + q4[2] * q4[2] + q4[3] * q4[3]);
  double w = q4[0] / n, x = q4[1] / n, y = q4[2] / n, z = q4[3] / n;
  r[0] = 1 - 2 * (y * y + z * z); r[1] = 2 * (x * y - w * z); r[2] = 2 * (x * z + w * y);
  r[3] = 2 * (x * y + w * z); r[4] = 1 - 2 * (x * x + z * z); r[5] = 2 * (y * z - w * x);
  r[6] = 2 * (x * z - w * y); r[7] = 2 * (y * z + w * x); r[8] = 1 - 2 * (x * x + y * y);
}

static void sh_rgb(const double* dc, const double* rest, int k, const double d[3], double out[3]) {
  const double C0 = 0.28209479177387814, C1 = 0.4886025119029199;
  double x = d[0], y = d[1], z = d[2], b[16];
  int n = 1 + k;
  b[0] = C0;
  if (n > 1) { b[1] = -C1 * y; b[2] = C1 * z; b[3] = -C1 * x; }
  if (n > 4) {
    double xx = x * x, yy = y * y, zz = z * z;
    b[4] = 1.0925484305920792 * x * y; b[5] = -1.0925484305920792 * y * z;
    b[6] = 0.3153915652525205 * (2 * zz - xx - yy); b[7] = -1.0925484305920792 * x * z;
    b[8] = 0.5462742152960396 * (xx - yy);
  }
  if (n > 9) {
    double xx = x * x, yy = y * y, zz = z * z;
    b[9] = -0.5900435899266435 * y * (3 * xx - yy); b[10] = 2.890611442640554 * x * y * z;
    b[11] = -0.4570457994644658 * y * (4 * zz - xx - yy);
    b[12] = 0.3731763325901154 * z * (2 * zz - 3 * xx - 3 * yy);
    b[13] = -0.4570457994644658 * x * (4 * zz - xx - yy); b[14] = 1.445305721320277 * z * (xx - yy);
    b[15] = -0.5900435899266435 * x * (3 * yy - xx);
  }
  for (int c = 0; c < 3; ++c) {
    double acc = b[0] * dc[c];
    for (int j = 1; j < n; ++j) acc += b[j] * rest[3 * (j - 1) + c];
    double v = 0.5 + acc;
    out[c] = v < 0 ? 0 : (v > 1 ? 1 : v);
  }
}

/* cam: 18 numbers in save_cameras order.  image: H*W*3, dominant: H*W. */
int oracle_render(int64_t n, const double* mu, const double* scale, const double* rot, const double* opacity,
                  const double* sh_dc, const double* sh_rest, int sh_k, const double* cam, const double* bg,
                  double* image, int64_t* dominant) {
  const double* R = cam;  /* r_c2w row-major */
  const double* C = cam + 9;
  const double fx = cam[12], fy = cam[13], px = cam[14], py = cam[15];
  const int W = (int)cam[16], H = (int)cam[17];
  const double amin = 1.0 / 255.0;
  splat_t* sp = (splat_t*)malloc(sizeof(splat_t) * (n > 0 ? n : 1));
  if (!sp) return -1;
  int64_t m = 0;
  for (int64_t i = 0; i < n; ++i) {
    double d[3] = {mu[3 * i] - C[0], mu[3 * i + 1] - C[1], mu[3 * i + 2] - C[2]};
    double x = R[0] * d[0] + R[3] * d[1] + R[6] * d[2];
    double y = R[1] * d[0] + R[4] * d[1] + R[7] * d[2];
    double z = R[2] * d[0] + R[5] * d[1] + R[8] * d[2];
    if (z <= 1e-8) continue;
    double q[9], S[9];
    quat_rot(rot + 4 * i, q);
    double s2[3] = {scale[3 * i] * scale[3 * i], scale[3 * i + 1] * scale[3 * i + 1], scale[3 * i + 2] * scale[3 * i + 2]};
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) S[a * 3 + b] = q[a * 3] * s2[0] * q[b * 3] + q[a * 3 + 1] * s2[1] * q[b * 3 + 1] + q[a * 3 + 2] * s2[2] * q[b * 3 + 2];
    double J[6] = {fx / z, 0.0, -fx * x / (z * z), 0.0, fy / z, -fy * y / (z * z)};
    double T[6];  /* J @ W, W = R^T */
    for (int r = 0; r < 2; ++r)
      for (int c = 0; c < 3; ++c) T[r * 3 + c] = J[r * 3] * R[c * 3] + J[r * 3 + 1] * R[c * 3 + 1] + J[r * 3 + 2] * R[c * 3 + 2];
    double TS[6];
    for (int r = 0; r < 2; ++r)
      for (int c = 0; c < 3; ++c) TS[r * 3 + c] = T[r * 3] * S[c] + T[r * 3 + 1] * S[3 + c] + T[r * 3 + 2] * S[6 + c];
    double ca = TS[0] * T[0] + TS[1] * T[1] + TS[2] * T[2] + 0.3;
    double cb = TS[0] * T[3] + TS[1] * T[4] + TS[2] * T[5];
    double cc = TS[3] * T[3] + TS[4] * T[4] + TS[5] * T[5] + 0.3;
    double o = opacity[i];
    double oc = o < 0.99 ? o : 0.99;
    if (oc < amin) continue;
    double lam = 0.5 * (ca + cc + hypot(ca - cc, 2 * cb));
    double r = sqrt(2.0 * log(oc / amin) * lam);
    if (r <= 0.0) continue;
    double mx = fx * x / z + px, my = fy * y / z + py;
    if (mx + r < 0 || mx - r > W - 1 || my + r < 0 || my - r > H - 1) continue;
    splat_t* s = &sp[m++];
    s->z = z;
    s->idx = (int)i;
    s->mx = mx;
    s->my = my;
    s->ca = ca;
    s->cb = cb;
    s->cc = cc;
    double nd = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    double dir[3] = {d[0] / nd, d[1] / nd, d[2] / nd};
    sh_rgb(sh_dc + 3 * i, sh_rest ? sh_rest + 3 * sh_k * i : NULL, sh_k, dir, s->rgb);
  }
  qsort(sp, (size_t)m, sizeof(splat_t), cmp_splat);
  const int64_t hw = (int64_t)H * W;
  double* trans = (double*)malloc(sizeof(double) * hw);
  double* best = (double*)malloc(sizeof(double) * hw);
  if (!trans || !best) { free(sp); free(trans); free(best); return -1; }
  for (int64_t p = 0; p < hw; ++p) {
    trans[p] = 1.0; best[p] = 0.0; dominant[p] = -1;
    image[3 * p] = image[3 * p + 1] = image[3 * p + 2] = 0.0;
  }
  for (int64_t k = 0; k < m; ++k) {
    const splat_t* s = &sp[k];
    double o = opacity[s->idx];
    double lam = 0.5 * (s->ca + s->cc + hypot(s->ca - s->cc, 2 * s->cb));
    double lg = 2.0 * log((o > 1e-300 ? o : 1e-300) / amin);
    double rw = sqrt((lg > 0 ? lg : 0.0) * lam) * (1 + 1e-6) + 1.0;
    int x0 = (int)floor(s->mx - rw), x1 = (int)ceil(s->mx + rw);
    int y0 = (int)floor(s->my - rw), y1 = (int)ceil(s->my + rw);
    if (x0 < 0) x0 = 0;
    if (y0 < 0) y0 = 0;
    if (x1 > W - 1) x1 = W - 1;
    if (y1 > H - 1) y1 = H - 1;
    double det = s->ca * s->cc - s->cb * s->cb;
    double ia = s->cc / det, ib = -s->cb / det, ic = s->ca / det;
    for (int yy = y0; yy <= y1; ++yy) {
      double dy = (double)yy - s->my;
      for (int xx = x0; xx <= x1; ++xx) {
        double dx = (double)xx - s->mx;
        double quad = ia * dx * dx + 2.0 * ib * dx * dy + ic * dy * dy;
        double a = o * exp(-0.5 * quad);
        if (a > 0.99) a = 0.99;
        if (a < amin) continue;
        int64_t p = (int64_t)yy * W + xx;
        double w = trans[p] * a;
        image[3 * p] += w * s->rgb[0];
        image[3 * p + 1] += w * s->rgb[1];
        image[3 * p + 2] += w * s->rgb[2];
        if (w > best[p]) { best[p] = w; dominant[p] = s->idx; }
        trans[p] *= 1.0 - a;
      }
    }
  }
  for (int64_t p = 0; p < hw; ++p)
    for (int c = 0; c < 3; ++c) image[3 * p + c] += trans[p] * bg[c];
  free(sp); free(trans); free(best);
  return 0;
}
