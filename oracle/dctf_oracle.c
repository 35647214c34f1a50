/*
 * TEST INFRASTRUCTURE ONLY. This file is the CPU oracle for the DCT-domain
 * block filter: a plain-C restatement of the reference algorithm
 * (/root/reference/proj/include/dctfilter, C++20 header-only). Only tests/,
 * __graft_entry__.smoke() and bench.py's CPU-baseline leg may load it, and
 * only as the checker; the product path (paper_1710_07193_b200) never links,
 * loads or calls it.
 *
 * Parity pin: tests/test_oracle.py checks every function here bit-for-bit
 * against the reference itself (oracle/_ref/libdctf_ref.so, built from the
 * reference headers in place) and against the reference tests' known-answer
 * values and fixtures (tests/golden/). The arithmetic order matches the
 * reference operation for operation and the file is compiled with
 * -ffp-contract=off (the reference is built without FMA contraction:
 * proj/CMakeLists.txt sets no -march), so results are bitwise identical.
 *
 * Extension beyond the reference (documented, used only where the reference
 * refuses the input): or_convolve / or_filter_image_spatial /
 * or_dense_operator accept kr x kc masks (both odd) and masks larger than the
 * block — the `k > n` guard of spatial.hpp:46 lifted — for BASELINE config
 * 5's 1x9 motion blur on 8x8 blocks.
 */
#include "dctf_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* block_matrix.hpp:67-81 — i-k-j product that skips a(i,k) == 0. */
static void mm(int n, const double* a, const double* b, double* out) {
  memset(out, 0, sizeof(double) * (size_t)n * n);
  for (int i = 0; i < n; ++i) {
    for (int k = 0; k < n; ++k) {
      const double aik = a[i * n + k];
      if (aik == 0.0) continue;
      for (int j = 0; j < n; ++j) out[i * n + j] += aik * b[k * n + j];
    }
  }
}

static void transpose(int n, const double* a, double* out) {
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) out[j * n + i] = a[i * n + j];
}

static int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* dct.hpp:40-52 — c[u][x] = alpha(u) cos((2x+1) u pi / 2n). */
int or_dct_basis(int n, double* c) {
  if (n < 2) return -1;
  const double pi = 3.141592653589793238462643383279502884; /* std::numbers::pi */
  const double a0 = sqrt(1.0 / n);
  const double au = sqrt(2.0 / n);
  for (int u = 0; u < n; ++u) {
    for (int x = 0; x < n; ++x) {
      const double angle = (2 * x + 1) * u * pi / (2.0 * n);
      c[u * n + x] = (u == 0 ? a0 : au) * cos(angle);
    }
  }
  return 0;
}

/* dct.hpp:59-62 — (C X) C^t. */
void or_forward_2d(int n, const double* c, const double* x, double* out) {
  double ct[256], t[256];
  transpose(n, c, ct);
  mm(n, c, x, t);
  mm(n, t, ct, out);
}

/* dct.hpp:65-68 — (C^t Y) C. */
void or_inverse_2d(int n, const double* c, const double* y, double* out) {
  double ct[256], t[256];
  transpose(n, c, ct);
  mm(n, ct, y, t);
  mm(n, t, c, out);
}

/* operators.hpp:61-75 */
static void shift_matrix(int n, int offset, int replicate, double* s) {
  memset(s, 0, sizeof(double) * (size_t)n * n);
  for (int i = 0; i < n; ++i) {
    const int j = i - offset;
    if (!replicate) {
      if (j >= 0 && j < n) s[i * n + j] = 1.0;
    } else {
      s[i * n + clampi(j, 0, n - 1)] = 1.0;
    }
  }
}

/* operators.hpp:80-98 */
static void band_matrix(const double* row, int k, int n, int replicate, double* t) {
  const int h = (k - 1) / 2;
  memset(t, 0, sizeof(double) * (size_t)n * n);
  for (int j = 0; j < n; ++j) {
    for (int c = 0; c < k; ++c) {
      const int src = j + c - h;
      if (!replicate) {
        if (src >= 0 && src < n) t[src * n + j] += row[c];
      } else {
        t[clampi(src, 0, n - 1) * n + j] += row[c];
      }
    }
  }
}

/* mask.hpp:100-108 */
int or_row_symmetric(const double* w, int k) {
  for (int r = 0; r < k / 2; ++r)
    for (int c = 0; c < k; ++c)
      if (w[r * k + c] != w[(k - 1 - r) * k + c]) return 0;
  return 1;
}

/* FilterPlan::compile (filter.hpp:76-83): build_spatial_operator_set
 * (operators.hpp:104-119) -> merge_symmetric if row-symmetric (146-169) ->
 * to_dct_domain (124-141). lefts/rights hold npairs n*n matrices. */
int or_plan_pairs(const double* w, int k, int n, int padding, int* npairs, int* merged,
                  double* lefts, double* rights) {
  if (k < 1 || (k % 2) == 0 || k > n || n < 2 || n > 16) return -1;
  const int h = (k - 1) / 2;
  const size_t nn = (size_t)n * n;
  double* sl = (double*)malloc(sizeof(double) * nn * (size_t)k);
  double* sr = (double*)malloc(sizeof(double) * nn * (size_t)k);
  for (int r = 0; r < k; ++r) {
    shift_matrix(n, h - r, padding, sl + (size_t)r * nn);
    band_matrix(w + (size_t)r * k, k, n, padding, sr + (size_t)r * nn);
  }
  int np = k;
  const int sym = or_row_symmetric(w, k);
  if (sym) {
    np = (k + 1) / 2;
    for (int r = 0; r < np; ++r) {
      const int mirror = k - 1 - r;
      if (r != mirror) {
        double* l = sl + (size_t)r * nn;
        const double* lm = sl + (size_t)mirror * nn;
        for (size_t i = 0; i < nn; ++i) l[i] += lm[i]; /* add(), block_matrix.hpp:94-101 */
      }
      /* right factor of a merged pair is row r's band matrix (already at r) */
    }
  }
  *npairs = np;
  *merged = sym;
  if (lefts || rights) {
    double c[256], ct[256], t[256];
    or_dct_basis(n, c);
    transpose(n, c, ct);
    for (int p = 0; p < np; ++p) {
      if (lefts) {
        mm(n, c, sl + (size_t)p * nn, t);
        mm(n, t, ct, lefts + (size_t)p * nn);
      }
      if (rights) {
        mm(n, c, sr + (size_t)p * nn, t);
        mm(n, t, ct, rights + (size_t)p * nn);
      }
    }
  }
  free(sl);
  free(sr);
  return 0;
}

/* apply_pairs (filter.hpp:30-38): acc = add(acc, matmul(matmul(L, x), R)). */
void or_apply_pairs(int n, int npairs, const double* lefts, const double* rights,
                    const double* x, double* out) {
  const size_t nn = (size_t)n * n;
  double t[256], term[256], acc[256];
  memset(acc, 0, sizeof(double) * nn);
  for (int p = 0; p < npairs; ++p) {
    mm(n, lefts + (size_t)p * nn, x, t);
    mm(n, t, rights + (size_t)p * nn, term);
    for (size_t i = 0; i < nn; ++i) acc[i] = acc[i] + term[i];
  }
  memcpy(out, acc, sizeof(double) * nn);
}

/* convolve (spatial.hpp:41-68), correlation orientation, generalised to a
 * kr x kc mask (both odd) with the k <= n guard lifted. */
void or_convolve(int n, const double* w, int kr, int kc, int padding, const double* x,
                 double* out) {
  const int hr = (kr - 1) / 2, hc = (kc - 1) / 2;
  for (int i = 0; i < n; ++i) {
    for (int j = 0; j < n; ++j) {
      double acc = 0.0;
      for (int r = 0; r < kr; ++r) {
        for (int c = 0; c < kc; ++c) {
          int si = i + r - hr;
          int sj = j + c - hc;
          if (!padding) {
            if (si < 0 || si >= n || sj < 0 || sj >= n) continue;
          } else {
            si = clampi(si, 0, n - 1);
            sj = clampi(sj, 0, n - 1);
          }
          acc += w[r * kc + c] * x[si * n + sj];
        }
      }
      out[i * n + j] = acc;
    }
  }
}

/* quantize_sample (spatial.hpp:71-75): round half away from zero, clamp. */
int or_quantize(double v) {
  if (isnan(v)) return -1;
  const double r = round(v);
  return (int)(r < 0.0 ? 0.0 : (r > 255.0 ? 255.0 : r));
}

/* tile (image.hpp:164-184): edge-replicate to a multiple of n, row-major. */
size_t or_tile(const uint8_t* img, int w, int h, int n, double* blocks) {
  const int bw = (w + n - 1) / n, bh = (h + n - 1) / n;
  size_t b = 0;
  for (int by = 0; by < bh; ++by)
    for (int bx = 0; bx < bw; ++bx, ++b)
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
          const int y = (by * n + i) < (h - 1) ? (by * n + i) : (h - 1);
          const int x = (bx * n + j) < (w - 1) ? (bx * n + j) : (w - 1);
          blocks[b * (size_t)n * n + (size_t)i * n + j] = (double)img[(size_t)y * w + x];
        }
  return b;
}

/* assemble (image.hpp:188-203): quantize and crop. Returns -1 on NaN. */
int or_assemble(const double* blocks, int w, int h, int n, uint8_t* out) {
  const int bw = (w + n - 1) / n, bh = (h + n - 1) / n;
  size_t b = 0;
  for (int by = 0; by < bh; ++by)
    for (int bx = 0; bx < bw; ++bx, ++b)
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
          const int y = by * n + i, x = bx * n + j;
          if (x < w && y < h) {
            const int q = or_quantize(blocks[b * (size_t)n * n + (size_t)i * n + j]);
            if (q < 0) return -1;
            out[(size_t)y * w + x] = (uint8_t)q;
          }
        }
  return 0;
}

/* filter_image, Domain::kDct (image.hpp:210-218) with the filter_block
 * sequence (filter.hpp:71-73). Optional side outputs, block-major. */
int or_filter_image(const uint8_t* img, int w, int h, const double* mw, int k, int padding,
                    int n, uint8_t* out, double* coef_in, double* coef_out, double* prequant) {
  if (k > n) return -1;
  const size_t nn = (size_t)n * n;
  const size_t nb = (size_t)((w + n - 1) / n) * (size_t)((h + n - 1) / n);
  double* blocks = (double*)malloc(sizeof(double) * nn * nb);
  double* lefts = (double*)malloc(sizeof(double) * nn * (size_t)k);
  double* rights = (double*)malloc(sizeof(double) * nn * (size_t)k);
  double c[256];
  int np = 0, merged = 0, rc = 0;
  or_tile(img, w, h, n, blocks);
  or_dct_basis(n, c);
  or_plan_pairs(mw, k, n, padding, &np, &merged, lefts, rights);
  for (size_t b = 0; b < nb; ++b) {
    double x[256], y[256];
    double* blk = blocks + b * nn;
    or_forward_2d(n, c, blk, x);
    or_apply_pairs(n, np, lefts, rights, x, y);
    if (coef_in) memcpy(coef_in + b * nn, x, sizeof(double) * nn);
    if (coef_out) memcpy(coef_out + b * nn, y, sizeof(double) * nn);
    or_inverse_2d(n, c, y, blk);
    if (prequant) memcpy(prequant + b * nn, blk, sizeof(double) * nn);
  }
  rc = or_assemble(blocks, w, h, n, out);
  free(blocks);
  free(lefts);
  free(rights);
  return rc;
}

/* filter_image, Domain::kSpatial (image.hpp:219-222), kr x kc generalised. */
int or_filter_image_spatial(const uint8_t* img, int w, int h, const double* mw, int kr, int kc,
                            int padding, int n, uint8_t* out, double* prequant) {
  const size_t nn = (size_t)n * n;
  const size_t nb = (size_t)((w + n - 1) / n) * (size_t)((h + n - 1) / n);
  double* blocks = (double*)malloc(sizeof(double) * nn * nb);
  or_tile(img, w, h, n, blocks);
  for (size_t b = 0; b < nb; ++b) {
    double y[256];
    or_convolve(n, mw, kr, kc, padding, blocks + b * nn, y);
    memcpy(blocks + b * nn, y, sizeof(double) * nn);
    if (prequant) memcpy(prequant + b * nn, y, sizeof(double) * nn);
  }
  const int rc = or_assemble(blocks, w, h, n, out);
  free(blocks);
  return rc;
}

/* Dense DCT-domain operator H = (C (x) C) H_spatial (C (x) C)^t, with
 * H_spatial read off the convolve formula (spatial.hpp:36-37), generalised
 * to kr x kc. Row-major n^2 x n^2; vec index u*n+v. */
int or_dense_operator(const double* mw, int kr, int kc, int n, int padding, double* hout) {
  if (n < 2 || n > 16 || kr < 1 || kc < 1 || !(kr & 1) || !(kc & 1)) return -1;
  const size_t nn = (size_t)n * n;
  double c[256], ct[256];
  or_dct_basis(n, c);
  transpose(n, c, ct);
  double* hsp = (double*)calloc(nn * nn, sizeof(double));
  const int hr = (kr - 1) / 2, hc = (kc - 1) / 2;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
      for (int r = 0; r < kr; ++r)
        for (int cc = 0; cc < kc; ++cc) {
          int si = i + r - hr, sj = j + cc - hc;
          if (!padding) {
            if (si < 0 || si >= n || sj < 0 || sj >= n) continue;
          } else {
            si = clampi(si, 0, n - 1);
            sj = clampi(sj, 0, n - 1);
          }
          hsp[((size_t)i * n + j) * nn + (size_t)si * n + sj] += mw[r * kc + cc];
        }
  /* column (a,b) of H: forward_2d(convolve(inverse_2d(E_ab))) */
  for (size_t col = 0; col < nn; ++col) {
    double e[256], px[256], fx[256], y[256];
    memset(e, 0, sizeof e);
    e[col] = 1.0;
    or_inverse_2d(n, c, e, px);
    for (size_t r = 0; r < nn; ++r) {
      double acc = 0.0;
      for (size_t s = 0; s < nn; ++s) acc += hsp[r * nn + s] * px[s];
      fx[r] = acc;
    }
    or_forward_2d(n, c, fx, y);
    for (size_t r = 0; r < nn; ++r) hout[r * nn + col] = y[r];
  }
  free(hsp);
  return 0;
}
