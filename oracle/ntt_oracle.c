/* TEST INFRASTRUCTURE ONLY — C restatement of the reference's hot-path
 * semantics, for sizes the Python oracle cannot reach in seconds.
 *
 * Values: K little-endian 32-bit limbs (the device layout).  Every operation
 * follows the reference's generated programs literally, including its Barrett
 * constants (mbits = width-4, mu = floor(2^(2 mbits+3)/q), shift1 = mbits-2,
 * shift2 = mbits+5; oracle.py:109-134) and quotient estimate
 * r = ((t >> shift1) * mu) >> shift2, d = t - r q, d >= q ? d - q : d
 * (kernels._emit_mulmod kernels.py:140-153, oracle.barrett_mulmod
 * oracle.py:137-149).  addmod/submod: kernels.py:122-137.  NTT: run_ntt
 * kernels.py:483-499 (bit-reversed input, butterfly_schedule kernels.py:395-413,
 * butterfly kernels.py:290-292, inverse scale kernels.py:496-498).
 * Paths are relative to /root/reference/pkg/src/widemod/.
 *
 * Built into oracle/liboracle.so by oracle/Makefile; called through
 * oracle/cbind.py.  Never linked into the product.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define MAXK 64

typedef struct {
  int K;            /* limbs */
  int width;        /* interface width (bits) */
  uint32_t q[MAXK];
  uint32_t mu[MAXK];
  int shift1, shift2;
} or_field;

static void bn_mul(int K, const uint32_t *a, const uint32_t *b, uint32_t *t /* 2K */) {
  memset(t, 0, sizeof(uint32_t) * 2 * K);
  for (int i = 0; i < K; ++i) {
    uint64_t c = 0;
    for (int j = 0; j < K; ++j) {
      uint64_t p = (uint64_t)a[j] * b[i] + t[i + j] + c;
      t[i + j] = (uint32_t)p;
      c = p >> 32;
    }
    t[i + K] = (uint32_t)c;
  }
}

/* r[0..outK) = (a[0..aK) >> s), zero-filled */
static void bn_shr(const uint32_t *a, int aK, int s, uint32_t *r, int outK) {
  int ls = s / 32, bs = s % 32;
  for (int j = 0; j < outK; ++j) {
    int src = j + ls;
    uint64_t lo = src < aK ? a[src] : 0;
    uint64_t hi = src + 1 < aK ? a[src + 1] : 0;
    r[j] = bs ? (uint32_t)((lo >> bs) | (hi << (32 - bs))) : (uint32_t)lo;
  }
}

/* r = a - b mod 2^(32K); returns borrow */
static int bn_sub(int K, const uint32_t *a, const uint32_t *b, uint32_t *r) {
  int64_t br = 0;
  for (int j = 0; j < K; ++j) {
    int64_t d = (int64_t)a[j] - b[j] - br;
    r[j] = (uint32_t)d;
    br = d < 0;
  }
  return (int)br;
}

static int bn_add(int K, const uint32_t *a, const uint32_t *b, uint32_t *r) {
  uint64_t c = 0;
  for (int j = 0; j < K; ++j) {
    uint64_t s = (uint64_t)a[j] + b[j] + c;
    r[j] = (uint32_t)s;
    c = s >> 32;
  }
  return (int)c;
}

static int bn_lt(int K, const uint32_t *a, const uint32_t *b) {
  for (int j = K - 1; j >= 0; --j)
    if (a[j] != b[j]) return a[j] < b[j];
  return 0;
}

/* kernels._emit_addmod: s = a + b (width+1 bits); s < q ? s : s - q */
static void or_addmod(const or_field *f, const uint32_t *a, const uint32_t *b, uint32_t *r) {
  int K = f->K;
  uint32_t s[MAXK + 1];
  s[K] = (uint32_t)bn_add(K, a, b, s);
  int lt = s[K] == 0 && bn_lt(K, s, f->q);
  if (lt) {
    memcpy(r, s, 4 * K);
  } else {
    bn_sub(K, s, f->q, r);
  }
}

/* kernels._emit_submod: d = a - b; a < b ? d + q : d */
static void or_submod(const or_field *f, const uint32_t *a, const uint32_t *b, uint32_t *r) {
  int K = f->K;
  uint32_t d[MAXK];
  int under = bn_lt(K, a, b);
  bn_sub(K, a, b, d);
  if (under)
    bn_add(K, d, f->q, r);
  else
    memcpy(r, d, 4 * K);
}

/* kernels._emit_mulmod (Barrett with the reference constants) */
static void or_mulmod(const or_field *f, const uint32_t *a, const uint32_t *b, uint32_t *r) {
  int K = f->K;
  uint32_t t[2 * MAXK], r1[MAXK], r2[2 * MAXK], r3[MAXK], rq[2 * MAXK], d[MAXK], e[MAXK];
  bn_mul(K, a, b, t);
  bn_shr(t, 2 * K, f->shift1, r1, K);
  bn_mul(K, r1, f->mu, r2);
  bn_shr(r2, 2 * K, f->shift2, r3, K);
  bn_mul(K, r3, f->q, rq);
  bn_sub(K, t, rq, d); /* low K limbs: exact since t - r q < 2q */
  int keep = bn_lt(K, d, f->q);
  if (keep)
    memcpy(r, d, 4 * K);
  else {
    bn_sub(K, d, f->q, e);
    memcpy(r, e, 4 * K);
  }
}

int or_field_init(or_field *f, int K, int width, const uint32_t *q, const uint32_t *mu, int shift1,
                  int shift2) {
  if (K < 1 || K > MAXK) return 1;
  memset(f, 0, sizeof(*f));
  f->K = K;
  f->width = width;
  memcpy(f->q, q, 4 * K);
  memcpy(f->mu, mu, 4 * K);
  f->shift1 = shift1;
  f->shift2 = shift2;
  return 0;
}

int or_field_size(void) { return (int)sizeof(or_field); }

/* kind: 0 vadd, 1 vsub, 2 vmul, 3 axpy (a = scalar) */
void or_vector(const or_field *f, int kind, const uint32_t *a, const uint32_t *x, const uint32_t *y,
               uint32_t *out, int64_t n) {
  int K = f->K;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    const uint32_t *xi = x + i * K, *yi = y + i * K;
    uint32_t *o = out + i * K;
    if (kind == 0)
      or_addmod(f, xi, yi, o);
    else if (kind == 1)
      or_submod(f, xi, yi, o);
    else if (kind == 2)
      or_mulmod(f, xi, yi, o);
    else {
      uint32_t t[MAXK];
      or_mulmod(f, a, xi, t);
      or_addmod(f, t, yi, o);
    }
  }
}

/* out[e] = base^e, e < count (twiddle_table kernels.py:259-267) */
void or_powers(const or_field *f, const uint32_t *base, int64_t count, uint32_t *out) {
  int K = f->K;
  uint32_t acc[MAXK];
  memset(acc, 0, sizeof(acc));
  acc[0] = 1;
  for (int64_t e = 0; e < count; ++e) {
    memcpy(out + e * K, acc, 4 * K);
    uint32_t nx[MAXK];
    or_mulmod(f, acc, base, nx);
    memcpy(acc, nx, 4 * K);
  }
}

static int ilog2(int64_t n) {
  int l = 0;
  while (((int64_t)1 << l) < n) ++l;
  return l;
}

/* run_ntt on `batch` contiguous transforms, in place.  tw: n/2 powers of the
 * root (or root_inv); ninv != NULL selects the inverse scale. */
void or_ntt(const or_field *f, const uint32_t *tw, int64_t n, const uint32_t *ninv, uint32_t *x,
            int64_t batch) {
  int K = f->K;
  int lg = ilog2(n);
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t b = 0; b < batch; ++b) {
    uint32_t *v = x + b * n * K;
    uint32_t *tmp = (uint32_t *)malloc(sizeof(uint32_t) * n * K);
    for (int64_t i = 0; i < n; ++i) {
      int64_t r = 0;
      for (int bit = 0; bit < lg; ++bit) r |= ((i >> bit) & 1) << (lg - 1 - bit);
      memcpy(tmp + i * K, v + r * K, 4 * K);
    }
    memcpy(v, tmp, sizeof(uint32_t) * n * K);
    free(tmp);
    for (int64_t m = 2; m <= n; m <<= 1) {
      int64_t half = m >> 1, step = n / m;
      for (int64_t base = 0; base < n; base += m) {
        for (int64_t j = 0; j < half; ++j) {
          uint32_t *u = v + (base + j) * K, *w = v + (base + j + half) * K;
          uint32_t t[MAXK], o0[MAXK], o1[MAXK];
          or_mulmod(f, w, tw + (j * step) * K, t);
          or_addmod(f, u, t, o0);
          or_submod(f, u, t, o1);
          memcpy(u, o0, 4 * K);
          memcpy(w, o1, 4 * K);
        }
      }
    }
    if (ninv) {
      uint32_t zero[MAXK];
      memset(zero, 0, sizeof(zero));
      for (int64_t i = 0; i < n; ++i) {
        uint32_t t[MAXK], o0[MAXK];
        or_mulmod(f, v + i * K, ninv, t);
        or_addmod(f, zero, t, o0);
        memcpy(v + i * K, o0, 4 * K);
      }
    }
  }
}

/* y[k] for selected k: sum_j x[j] root^(jk) mod p, by Horner in root^k
 * (O(n) per point; the cheap exact spot check of SURVEY.md §8(c)). */
void or_ntt_points(const or_field *f, const uint32_t *x, int64_t n, const uint32_t *root, const int64_t *ks,
                   int npts, uint32_t *out) {
  int K = f->K;
#pragma omp parallel for schedule(static)
  for (int ip = 0; ip < npts; ++ip) {
    /* wk = root^k by square-and-multiply */
    uint32_t wk[MAXK], b[MAXK], t[MAXK];
    memset(wk, 0, sizeof(wk));
    wk[0] = 1;
    memcpy(b, root, 4 * K);
    for (int64_t e = ks[ip]; e; e >>= 1) {
      if (e & 1) {
        or_mulmod(f, wk, b, t);
        memcpy(wk, t, 4 * K);
      }
      or_mulmod(f, b, b, t);
      memcpy(b, t, 4 * K);
    }
    uint32_t acc[MAXK];
    memset(acc, 0, sizeof(acc));
    for (int64_t j = n - 1; j >= 0; --j) {
      or_mulmod(f, acc, wk, t);
      or_addmod(f, t, x + j * K, acc);
    }
    memcpy(out + (int64_t)ip * K, acc, 4 * K);
  }
}
