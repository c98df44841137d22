/* FFTW3 API shim (see fftw3.h). TEST INFRASTRUCTURE ONLY: links into the
 * oracle build of the reference sources, never into the product library. */
#define _POSIX_C_SOURCE 200112L
#include "fftw3.h"

#include <complex.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef double _Complex cplx;

typedef struct {
  int n;
  int nf;
  int f[64];     /* radix per pass, product = n */
  cplx* tw;      /* tw[m] = exp(sign * 2 pi i m / n) */
} plan1d;

struct fftw_plan_s {
  int rank;      /* 1 or 2 */
  int n0, n1;    /* rank 1: n0 = n, n1 = 1 */
  int sign;
  cplx* in;
  cplx* out;
  plan1d p0, p1;
};

void* fftw_malloc(size_t n) {
  void* p = NULL;
  if (posix_memalign(&p, 64, n ? n : 1) != 0) return NULL;
  return p;
}
void fftw_free(void* p) { free(p); }
fftw_complex* fftw_alloc_complex(size_t n) {
  return (fftw_complex*)fftw_malloc(n * sizeof(fftw_complex));
}

static int plan1d_init(plan1d* p, int n, int sign) {
  p->n = n;
  p->nf = 0;
  int r = n;
  /* radix 4 first, then 2, 3, 5, then any remaining prime */
  while (r % 4 == 0) { p->f[p->nf++] = 4; r /= 4; }
  while (r % 2 == 0) { p->f[p->nf++] = 2; r /= 2; }
  while (r % 3 == 0) { p->f[p->nf++] = 3; r /= 3; }
  while (r % 5 == 0) { p->f[p->nf++] = 5; r /= 5; }
  for (int q = 7; r > 1; q += 2)
    while (r % q == 0) { p->f[p->nf++] = q; r /= q; }
  p->tw = (cplx*)malloc(sizeof(cplx) * (size_t)(n ? n : 1));
  if (!p->tw) return 0;
  for (int m = 0; m < n; ++m) {
    /* long double argument reduction keeps the table within an ulp */
    long double a = 2.0L * 3.14159265358979323846264338327950288L * (long double)m /
                    (long double)n;
    double c = (double)cosl(a), s = (double)sinl(a);
    p->tw[m] = c + (double)sign * s * I;
  }
  return 1;
}

static void plan1d_free(plan1d* p) { free(p->tw); p->tw = NULL; }

/* length-n transform of x (contiguous); work has n entries; result in x */
static void fft1d(const plan1d* p, cplx* x, cplx* work) {
  const int n = p->n;
  if (n <= 1) return;
  cplx* src = x;
  cplx* dst = work;
  int ns = 1;
  cplx v[64];
  for (int pass = 0; pass < p->nf; ++pass) {
    const int R = p->f[pass];
    const int m = n / R;          /* butterflies per pass */
    const int tstep = n / (ns * R);
    for (int j = 0; j < m; ++j) {
      const int k = j % ns;
      for (int r = 0; r < R; ++r) {
        cplx a = src[j + r * m];
        if (k != 0 && r != 0) a *= p->tw[(size_t)r * k * tstep % n];
        v[r] = a;
      }
      cplx y[64];
      if (R == 2) {
        y[0] = v[0] + v[1];
        y[1] = v[0] - v[1];
      } else if (R == 4) {
        const cplx t0 = v[0] + v[2], t1 = v[0] - v[2];
        const cplx t2 = v[1] + v[3];
        const cplx d = v[1] - v[3];
        /* d * (sign * i) with sign taken from the table: tw[n/4] */
        const cplx t3 = d * p->tw[n / 4];
        y[0] = t0 + t2;
        y[2] = t0 - t2;
        y[1] = t1 + t3;
        y[3] = t1 - t3;
      } else {
        /* small DFT through the table: W_R^{rs} = tw[(rs mod R) * n/R] */
        for (int s = 0; s < R; ++s) {
          cplx acc = v[0];
          for (int r = 1; r < R; ++r) acc += v[r] * p->tw[(size_t)((r * s) % R) * m];
          y[s] = acc;
        }
      }
      const int base = (j / ns) * ns * R + k;
      for (int r = 0; r < R; ++r) dst[base + r * ns] = y[r];
    }
    cplx* t = src;
    src = dst;
    dst = t;
    ns *= R;
  }
  if (src != x) memcpy(x, src, sizeof(cplx) * (size_t)n);
}

static fftw_plan make_plan(int rank, int n0, int n1, fftw_complex* in,
                           fftw_complex* out, int sign) {
  if (n0 < 1 || n1 < 1) return NULL;
  fftw_plan p = (fftw_plan)calloc(1, sizeof(struct fftw_plan_s));
  if (!p) return NULL;
  p->rank = rank;
  p->n0 = n0;
  p->n1 = n1;
  p->sign = sign;
  p->in = (cplx*)in;
  p->out = (cplx*)out;
  if (!plan1d_init(&p->p0, n0, sign)) { free(p); return NULL; }
  if (rank == 2 && !plan1d_init(&p->p1, n1, sign)) {
    plan1d_free(&p->p0);
    free(p);
    return NULL;
  }
  return p;
}

fftw_plan fftw_plan_dft_1d(int n, fftw_complex* in, fftw_complex* out,
                           int sign, unsigned flags) {
  (void)flags;
  return make_plan(1, n, 1, in, out, sign);
}

fftw_plan fftw_plan_dft_2d(int n0, int n1, fftw_complex* in,
                           fftw_complex* out, int sign, unsigned flags) {
  (void)flags;
  return make_plan(2, n0, n1, in, out, sign);
}

void fftw_execute_dft(const fftw_plan p, fftw_complex* in_, fftw_complex* out_) {
  cplx* in = (cplx*)in_;
  cplx* out = (cplx*)out_;
  if (p->rank == 1) {
    const int n = p->n0;
    cplx* work = (cplx*)malloc(sizeof(cplx) * 2 * (size_t)n);
    memcpy(work, in, sizeof(cplx) * (size_t)n);
    fft1d(&p->p0, work, work + n);
    memcpy(out, work, sizeof(cplx) * (size_t)n);
    free(work);
    return;
  }
  const int n0 = p->n0, n1 = p->n1;
  const size_t tot = (size_t)n0 * n1;
  if (out != in) memcpy(out, in, sizeof(cplx) * tot);
  const int nmax = n0 > n1 ? n0 : n1;
  enum { CB = 8 };
  cplx* work = (cplx*)malloc(sizeof(cplx) * ((size_t)nmax * (CB + 1)));
  /* rows: length n1, contiguous */
  for (int r = 0; r < n0; ++r) fft1d(&p->p1, out + (size_t)r * n1, work);
  /* columns: length n0, gathered CB at a time */
  cplx* col = work + nmax;
  for (int c0 = 0; c0 < n1; c0 += CB) {
    const int cb = (n1 - c0) < CB ? (n1 - c0) : CB;
    for (int r = 0; r < n0; ++r)
      for (int c = 0; c < cb; ++c) col[(size_t)c * n0 + r] = out[(size_t)r * n1 + c0 + c];
    for (int c = 0; c < cb; ++c) fft1d(&p->p0, col + (size_t)c * n0, work);
    for (int r = 0; r < n0; ++r)
      for (int c = 0; c < cb; ++c) out[(size_t)r * n1 + c0 + c] = col[(size_t)c * n0 + r];
  }
  free(work);
}

void fftw_execute(const fftw_plan p) {
  fftw_execute_dft(p, (fftw_complex*)p->in, (fftw_complex*)p->out);
}

void fftw_destroy_plan(fftw_plan p) {
  if (!p) return;
  plan1d_free(&p->p0);
  if (p->rank == 2) plan1d_free(&p->p1);
  free(p);
}
