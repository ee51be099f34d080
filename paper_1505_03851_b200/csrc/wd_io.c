/* wd_io.c -- native corpus and output formats.
 *
 * The reference reads its corpus as text, one document per line of
 * whitespace-separated word ids, into a Python list of per-document arrays
 * (lda.py:66-110), reads injected stop values with np.loadtxt
 * (cli.py:213-230, kernels.py:66-83) and writes z / theta / phi /
 * likelihood as CSV through the csv module (cli.py:232-273).  At
 * configs[2]-[4] sizes (1e6-1e7 documents, 2e8-2e9 tokens) those Python
 * loops cost minutes.  This library does the same work in C over
 * pthreads, straight into flat CSR buffers (offsets int64 [M+1], words
 * int32 [sum N]) that the device corpus consumes without per-document
 * objects:
 *
 *   wdio_scan_corpus / wdio_fill_corpus   text corpus -> CSR (parallel)
 *   wdio_scan_floats / wdio_fill_floats   one float per line -> float64
 *   wdio_pread                            parallel pread into a (pinned) buffer
 *   wdio_write_corpus_text                the reference's text corpus format
 *   wdio_write_z_csv                      "doc,pos,topic" rows (csv.writer bytes)
 *   wdio_write_matrix_csv                 repr(float(x)) rows (csv.writer bytes)
 *
 * Parsers accept exactly the inputs whose meaning is unambiguous in C
 * (ASCII, [+-]?digits tokens, '\n' / '\r\n' / '\r' line ends); anything
 * else -- non-ASCII bytes, underscores, a negative id, a malformed token --
 * returns WDIO_FALLBACK and the Python caller re-reads the file with the
 * reference's own Python semantics, so valid exotic inputs parse the same
 * and errors carry the reference's exact messages.
 *
 * Writers reproduce csv.writer's default dialect byte for byte: ',' between
 * fields, "\r\n" after each row, no quoting (no field contains a delimiter,
 * quote or line break), and each float as Python's repr: the shortest
 * decimal that round-trips (correctly rounded printf/strtod, searched over
 * the digit count), fixed notation for decimal exponents -4..15 with ".0"
 * added to integral values, otherwise d.ddde+XX.
 */
#define _GNU_SOURCE
#include <errno.h>
#include <fcntl.h>
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#define WDIO_OK 0
#define WDIO_FALLBACK 1
#define WDIO_ENOMEM (-12)

#define MAX_THREADS 64

/* ------------------------------------------------------------ file map */
typedef struct {
  const unsigned char* p;
  size_t n;
  int fd;
} fmap;

static int map_file(const char* path, fmap* m) {
  m->p = NULL;
  m->n = 0;
  m->fd = open(path, O_RDONLY);
  if (m->fd < 0) return -errno;
  struct stat st;
  if (fstat(m->fd, &st) != 0) {
    int e = -errno;
    close(m->fd);
    return e;
  }
  m->n = (size_t)st.st_size;
  if (m->n == 0) return 0;
  void* p = mmap(NULL, m->n, PROT_READ, MAP_PRIVATE, m->fd, 0);
  if (p == MAP_FAILED) {
    int e = -errno;
    close(m->fd);
    return e;
  }
  madvise(p, m->n, MADV_SEQUENTIAL);
  m->p = (const unsigned char*)p;
  return 0;
}

static void unmap_file(fmap* m) {
  if (m->p) munmap((void*)m->p, m->n);
  if (m->fd >= 0) close(m->fd);
  m->p = NULL;
  m->fd = -1;
}

static int clamp_threads(int t) { return t < 1 ? 1 : (t > MAX_THREADS ? MAX_THREADS : t); }

/* Split [a, b) into up to T pieces that start right after a '\n' (so "\r\n"
 * never straddles a cut and every piece begins at a line start). */
static int split_lines(const unsigned char* p, size_t a, size_t b, int T, size_t* cut) {
  int k = 0;
  cut[k++] = a;
  for (int t = 1; t < T; ++t) {
    size_t c = a + (b - a) * (size_t)t / (size_t)T;
    if (c <= cut[k - 1]) continue;
    const unsigned char* nl = memchr(p + c, '\n', b - c);
    if (!nl) break;
    c = (size_t)(nl - p) + 1;
    if (c >= b || c <= cut[k - 1]) continue;
    cut[k++] = c;
  }
  cut[k] = b;
  return k;
}

/* --------------------------------------------------------- vec helpers */
typedef struct {
  void* d;
  size_t n, cap, esz;
} vec;

static int vec_push(vec* v, const void* x) {
  if (v->n == v->cap) {
    size_t nc = v->cap ? v->cap * 2 : 4096;
    void* nd = realloc(v->d, nc * v->esz);
    if (!nd) return WDIO_ENOMEM;
    v->d = nd;
    v->cap = nc;
  }
  memcpy((char*)v->d + v->n * v->esz, x, v->esz);
  v->n++;
  return 0;
}

/* ------------------------------------------------------ corpus parsing */
typedef struct {
  const unsigned char* p;
  size_t a, b;
  int last;          /* piece ends the file */
  vec lens;          /* int64 per line */
  vec words;         /* int32 per token */
  int32_t max_word;
  int status;
} corpus_piece;

static inline int is_ws(unsigned char c) { return c == ' ' || c == '\t' || c == '\v' || c == '\f'; }

static void* parse_corpus_piece(void* arg) {
  corpus_piece* q = (corpus_piece*)arg;
  const unsigned char* p = q->p;
  size_t i = q->a;
  const size_t b = q->b;
  q->max_word = -1;
  q->status = WDIO_OK;
  while (i < b) {
    /* one line: [i, end of line) */
    int64_t count = 0;
    for (;;) {
      while (i < b && is_ws(p[i])) ++i;
      if (i >= b) break;
      unsigned char c = p[i];
      if (c == '\n') { ++i; break; }
      if (c == '\r') { ++i; if (i < b && p[i] == '\n') ++i; break; }
      /* token: [+-]?[0-9]{1,18} followed by whitespace or a line end */
      int neg = 0;
      if (c == '+' || c == '-') { neg = c == '-'; ++i; }
      size_t d0 = i;
      int64_t v = 0;
      while (i < b && p[i] >= '0' && p[i] <= '9' && i - d0 < 19) v = v * 10 + (p[i++] - '0');
      if (i == d0 || i - d0 > 18) { q->status = WDIO_FALLBACK; return NULL; }
      if (i < b && !(is_ws(p[i]) || p[i] == '\n' || p[i] == '\r')) { q->status = WDIO_FALLBACK; return NULL; }
      if (neg && v != 0) { q->status = WDIO_FALLBACK; return NULL; } /* negative id: the reference's error */
      if (v > INT32_MAX) { q->status = WDIO_FALLBACK; return NULL; } /* beyond the int32 device layout */
      int32_t w = (int32_t)v;
      if (vec_push(&q->words, &w)) { q->status = WDIO_ENOMEM; return NULL; }
      if (w > q->max_word) q->max_word = w;
      ++count;
    }
    if (vec_push(&q->lens, &count)) { q->status = WDIO_ENOMEM; return NULL; }
  }
  return NULL;
}

typedef struct {
  fmap m;
  int k;
  corpus_piece pc[MAX_THREADS];
} corpus_scan;

static int ascii_only(const unsigned char* p, size_t a, size_t b) {
  for (size_t i = a; i < b; ++i)
    if (p[i] >= 0x80 || (p[i] < 0x20 && p[i] != '\n' && p[i] != '\r' && p[i] != '\t' && p[i] != '\v' && p[i] != '\f'))
      return 0;
  return 1;
}

void wdio_release(void* h);

/* Scan a text corpus from byte `start` (after an optional header line the
 * caller has parsed).  On WDIO_OK *handle, *n_docs, *n_tokens and
 * *max_word are set; call wdio_fill_corpus then wdio_release. */
int wdio_scan_corpus(const char* path, int64_t start, int threads, void** handle, int64_t* n_docs,
                     int64_t* n_tokens, int32_t* max_word) {
  *handle = NULL;
  corpus_scan* s = (corpus_scan*)calloc(1, sizeof(corpus_scan));
  if (!s) return WDIO_ENOMEM;
  s->m.fd = -1;
  int rc = map_file(path, &s->m);
  if (rc) { free(s); return rc; }
  size_t a = (size_t)(start < 0 ? 0 : start), b = s->m.n;
  if (a > b) a = b;
  if (!ascii_only(s->m.p, a, b)) { unmap_file(&s->m); free(s); return WDIO_FALLBACK; }
  int T = clamp_threads(threads);
  if (b - a < ((size_t)1 << 20)) T = 1;
  size_t cut[MAX_THREADS + 1];
  s->k = (a < b) ? split_lines(s->m.p, a, b, T, cut) : 0;
  pthread_t th[MAX_THREADS];
  for (int t = 0; t < s->k; ++t) {
    corpus_piece* q = &s->pc[t];
    q->p = s->m.p;
    q->a = cut[t];
    q->b = cut[t + 1];
    q->lens.esz = sizeof(int64_t);
    q->words.esz = sizeof(int32_t);
    if (s->k > 1) pthread_create(&th[t], NULL, parse_corpus_piece, q);
    else parse_corpus_piece(q);
  }
  if (s->k > 1)
    for (int t = 0; t < s->k; ++t) pthread_join(th[t], NULL);
  int64_t D = 0, N = 0;
  int32_t mx = -1;
  for (int t = 0; t < s->k; ++t) {
    if (s->pc[t].status) {
      int st = s->pc[t].status;
      wdio_release(s);
      return st;
    }
    D += (int64_t)s->pc[t].lens.n;
    N += (int64_t)s->pc[t].words.n;
    if (s->pc[t].max_word > mx) mx = s->pc[t].max_word;
  }
  *handle = s;
  *n_docs = D;
  *n_tokens = N;
  *max_word = mx;
  return WDIO_OK;
}

typedef struct {
  corpus_piece* q;
  int64_t* off;   /* offsets slice for this piece's documents (off[0] = token base) */
  int32_t* words; /* words slice */
} fill_job;

static void* fill_piece(void* arg) {
  fill_job* j = (fill_job*)arg;
  const int64_t* L = (const int64_t*)j->q->lens.d;
  int64_t acc = j->off[0];
  for (size_t d = 0; d < j->q->lens.n; ++d) {
    acc += L[d];
    j->off[d + 1] = acc;
  }
  if (j->q->words.n) memcpy(j->words, j->q->words.d, j->q->words.n * sizeof(int32_t));
  return NULL;
}

int wdio_fill_corpus(void* handle, int64_t* offsets, int32_t* words) {
  corpus_scan* s = (corpus_scan*)handle;
  fill_job jobs[MAX_THREADS];
  pthread_t th[MAX_THREADS];
  offsets[0] = 0;
  int64_t d = 0, n = 0;
  for (int t = 0; t < s->k; ++t) {
    offsets[d] = n;
    jobs[t].q = &s->pc[t];
    jobs[t].off = offsets + d;
    jobs[t].words = words + n;
    d += (int64_t)s->pc[t].lens.n;
    n += (int64_t)s->pc[t].words.n;
  }
  /* each piece writes off[1..len] of its slice; off[0] of the next slice is
     the same value, written above before any thread starts */
  for (int t = 0; t < s->k; ++t) pthread_create(&th[t], NULL, fill_piece, &jobs[t]);
  for (int t = 0; t < s->k; ++t) pthread_join(th[t], NULL);
  return WDIO_OK;
}

/* ------------------------------------------------------- float parsing */
typedef struct {
  const unsigned char* p;
  size_t a, b;
  vec vals; /* double */
  int status;
} float_piece;

/* [+-]?(digits[.digits*]|.digits)([eE][+-]?digits)? -- the literals
 * np.loadtxt and Python's float() both read the same way */
static int float_token_ok(const unsigned char* p, size_t n) {
  size_t i = 0;
  if (i < n && (p[i] == '+' || p[i] == '-')) ++i;
  size_t d = 0;
  while (i < n && p[i] >= '0' && p[i] <= '9') { ++i; ++d; }
  if (i < n && p[i] == '.') {
    ++i;
    while (i < n && p[i] >= '0' && p[i] <= '9') { ++i; ++d; }
  }
  if (d == 0) return 0;
  if (i < n && (p[i] == 'e' || p[i] == 'E')) {
    ++i;
    if (i < n && (p[i] == '+' || p[i] == '-')) ++i;
    size_t e = 0;
    while (i < n && p[i] >= '0' && p[i] <= '9') { ++i; ++e; }
    if (e == 0) return 0;
  }
  return i == n && n < 400;
}

static void* parse_float_piece(void* arg) {
  float_piece* q = (float_piece*)arg;
  const unsigned char* p = q->p;
  size_t i = q->a;
  const size_t b = q->b;
  char buf[512];
  q->status = WDIO_OK;
  while (i < b) {
    int ntok = 0;
    for (;;) {
      while (i < b && is_ws(p[i])) ++i;
      if (i >= b) break;
      if (p[i] == '\n') { ++i; break; }
      if (p[i] == '\r') { ++i; if (i < b && p[i] == '\n') ++i; break; }
      size_t t0 = i;
      while (i < b && !is_ws(p[i]) && p[i] != '\n' && p[i] != '\r') ++i;
      size_t n = i - t0;
      /* one value per line only (np.loadtxt of several columns yields a 2-D
         array: the Python path keeps that meaning) */
      if (++ntok > 1 || !float_token_ok(p + t0, n)) { q->status = WDIO_FALLBACK; return NULL; }
      memcpy(buf, p + t0, n);
      buf[n] = 0;
      double v = strtod(buf, NULL);
      if (vec_push(&q->vals, &v)) { q->status = WDIO_ENOMEM; return NULL; }
    }
  }
  return NULL;
}

typedef struct {
  fmap m;
  int k;
  float_piece pc[MAX_THREADS];
} float_scan;

int wdio_scan_floats(const char* path, int threads, void** handle, int64_t* n) {
  *handle = NULL;
  float_scan* s = (float_scan*)calloc(1, sizeof(float_scan));
  if (!s) return WDIO_ENOMEM;
  s->m.fd = -1;
  int rc = map_file(path, &s->m);
  if (rc) { free(s); return rc; }
  /* '#' comments and non-ASCII bytes: Python path */
  if (!ascii_only(s->m.p, 0, s->m.n) || (s->m.n && memchr(s->m.p, '#', s->m.n))) {
    unmap_file(&s->m);
    free(s);
    return WDIO_FALLBACK;
  }
  int T = clamp_threads(threads);
  if (s->m.n < ((size_t)1 << 20)) T = 1;
  size_t cut[MAX_THREADS + 1];
  s->k = s->m.n ? split_lines(s->m.p, 0, s->m.n, T, cut) : 0;
  pthread_t th[MAX_THREADS];
  for (int t = 0; t < s->k; ++t) {
    float_piece* q = &s->pc[t];
    q->p = s->m.p;
    q->a = cut[t];
    q->b = cut[t + 1];
    q->vals.esz = sizeof(double);
    if (s->k > 1) pthread_create(&th[t], NULL, parse_float_piece, q);
    else parse_float_piece(q);
  }
  if (s->k > 1)
    for (int t = 0; t < s->k; ++t) pthread_join(th[t], NULL);
  int64_t tot = 0;
  for (int t = 0; t < s->k; ++t) {
    if (s->pc[t].status) {
      int st = s->pc[t].status;
      for (int u = 0; u < s->k; ++u) free(s->pc[u].vals.d);
      unmap_file(&s->m);
      free(s);
      return st;
    }
    tot += (int64_t)s->pc[t].vals.n;
  }
  *handle = s;
  *n = tot;
  return WDIO_OK;
}

int wdio_fill_floats(void* handle, double* out) {
  float_scan* s = (float_scan*)handle;
  for (int t = 0; t < s->k; ++t) {
    if (s->pc[t].vals.n) memcpy(out, s->pc[t].vals.d, s->pc[t].vals.n * sizeof(double));
    out += s->pc[t].vals.n;
  }
  return WDIO_OK;
}

void wdio_release_floats(void* handle) {
  float_scan* s = (float_scan*)handle;
  if (!s) return;
  for (int t = 0; t < s->k; ++t) free(s->pc[t].vals.d);
  unmap_file(&s->m);
  free(s);
}

void wdio_release(void* handle) {
  corpus_scan* s = (corpus_scan*)handle;
  if (!s) return;
  for (int t = 0; t < s->k; ++t) {
    free(s->pc[t].lens.d);
    free(s->pc[t].words.d);
  }
  unmap_file(&s->m);
  free(s);
}

/* ------------------------------------------------------------- pread */
typedef struct {
  int fd;
  int64_t off, n;
  char* dst;
  int err;
} pread_job;

static void* pread_worker(void* arg) {
  pread_job* j = (pread_job*)arg;
  int64_t done = 0;
  j->err = 0;
  while (done < j->n) {
    ssize_t r = pread(j->fd, j->dst + done, (size_t)(j->n - done), (off_t)(j->off + done));
    if (r < 0) {
      if (errno == EINTR) continue;
      j->err = -errno;
      return NULL;
    }
    if (r == 0) { j->err = -5; return NULL; } /* EIO: short file */
    done += r;
  }
  return NULL;
}

/* nbytes from file offset `off` into dst (e.g. pinned host memory), split
 * over up to `threads` concurrent preads. */
int wdio_pread(const char* path, int64_t off, int64_t nbytes, void* dst, int threads) {
  int fd = open(path, O_RDONLY);
  if (fd < 0) return -errno;
  int T = clamp_threads(threads);
  if (nbytes < ((int64_t)8 << 20)) T = 1;
  pread_job jobs[MAX_THREADS];
  pthread_t th[MAX_THREADS];
  const int64_t step = ((nbytes + T - 1) / T + 4095) & ~(int64_t)4095;
  int k = 0;
  for (int64_t a = 0; a < nbytes && k < T; a += step, ++k) {
    jobs[k].fd = fd;
    jobs[k].off = off + a;
    jobs[k].n = (a + step < nbytes ? step : nbytes - a);
    jobs[k].dst = (char*)dst + a;
    if (T > 1) pthread_create(&th[k], NULL, pread_worker, &jobs[k]);
    else pread_worker(&jobs[k]);
  }
  int err = 0;
  for (int t = 0; t < k; ++t) {
    if (T > 1) pthread_join(th[t], NULL);
    if (jobs[t].err) err = jobs[t].err;
  }
  close(fd);
  return err;
}

/* ----------------------------------------------------------- writers */
/* Python repr(float): shortest round-tripping digits, Python's layout. */
static int py_repr(double x, char* out) {
  if (isnan(x)) { strcpy(out, "nan"); return 3; }
  if (isinf(x)) { strcpy(out, x < 0 ? "-inf" : "inf"); return x < 0 ? 4 : 3; }
  char* o = out;
  if (signbit(x)) { *o++ = '-'; x = -x; }
  if (x == 0.0) { strcpy(o, "0.0"); return (int)(o - out) + 3; }
  char buf[40], tmp[40];
  /* shortest p in [1, 17] whose correctly rounded %.{p-1}e round-trips
     (round-trip is monotone in p: a (p-1)-digit decimal is a p-digit one).
     Most values (float32-derived ones always) need 16-17 digits: test those
     first, then bisect below. */
  int lo, hi;
  snprintf(buf, sizeof buf, "%.15e", x);
  if (strtod(buf, NULL) != x) {
    snprintf(buf, sizeof buf, "%.16e", x);
    lo = hi = 17;
  } else {
    snprintf(tmp, sizeof tmp, "%.14e", x);
    if (strtod(tmp, NULL) != x) {
      lo = hi = 16;
    } else {
      memcpy(buf, tmp, sizeof tmp);
      lo = 1;
      hi = 15;  /* buf holds the 15-digit form */
      while (lo < hi) {
        int mid = (lo + hi) >> 1;
        snprintf(tmp, sizeof tmp, "%.*e", mid - 1, x);
        if (strtod(tmp, NULL) == x) { hi = mid; memcpy(buf, tmp, sizeof tmp); }
        else lo = mid + 1;
      }
    }
  }
  /* digits and decimal exponent */
  char dg[24];
  int nd = 0;
  const char* c = buf;
  for (; *c && *c != 'e'; ++c)
    if (*c >= '0' && *c <= '9') dg[nd++] = *c;
  int e = atoi(c + 1);
  while (nd > 1 && dg[nd - 1] == '0') --nd;
  if (e >= -4 && e < 16) {
    if (e >= 0) {
      for (int i = 0; i <= e; ++i) *o++ = i < nd ? dg[i] : '0';
      *o++ = '.';
      if (nd > e + 1) for (int i = e + 1; i < nd; ++i) *o++ = dg[i];
      else *o++ = '0';
    } else {
      *o++ = '0';
      *o++ = '.';
      for (int i = 0; i < -e - 1; ++i) *o++ = '0';
      for (int i = 0; i < nd; ++i) *o++ = dg[i];
    }
  } else {
    *o++ = dg[0];
    if (nd > 1) {
      *o++ = '.';
      for (int i = 1; i < nd; ++i) *o++ = dg[i];
    }
    o += sprintf(o, "e%c%02d", e < 0 ? '-' : '+', e < 0 ? -e : e);
  }
  *o = 0;
  return (int)(o - out);
}

int wdio_repr(double x, char* out) { return py_repr(x, out); }

static inline char* put_i64(char* o, int64_t v) {
  char t[24];
  int n = 0;
  uint64_t u = v < 0 ? (uint64_t)(-(v + 1)) + 1 : (uint64_t)v;
  if (v < 0) *o++ = '-';
  do { t[n++] = (char)('0' + u % 10); u /= 10; } while (u);
  while (n) *o++ = t[--n];
  return o;
}

typedef struct {
  /* matrix */
  const char* base;
  int64_t r0, r1, cols, ld;
  int esz;
  /* z / corpus words */
  const int64_t* off;
  const void* z;
  int zsz;
  int corpus; /* 1: the document's words space-separated, one line per document */
  int64_t d0, d1;
  /* output */
  char* buf;
  size_t len, cap;
  int status;
} wjob;

static int ensure(wjob* j, size_t need) {
  if (j->len + need <= j->cap) return 0;
  size_t nc = j->cap ? j->cap : 1 << 20;
  while (j->len + need > nc) nc *= 2;
  char* nb = realloc(j->buf, nc);
  if (!nb) return WDIO_ENOMEM;
  j->buf = nb;
  j->cap = nc;
  return 0;
}

static void* matrix_worker(void* arg) {
  wjob* j = (wjob*)arg;
  j->status = 0;
  for (int64_t r = j->r0; r < j->r1; ++r) {
    if (ensure(j, (size_t)j->cols * 26 + 4)) { j->status = WDIO_ENOMEM; return NULL; }
    char* o = j->buf + j->len;
    const char* row = j->base + (size_t)r * (size_t)j->ld * (size_t)j->esz;
    for (int64_t c = 0; c < j->cols; ++c) {
      double v = j->esz == 4 ? (double)((const float*)row)[c] : ((const double*)row)[c];
      if (c) *o++ = ',';
      o += py_repr(v, o);
    }
    *o++ = '\r';
    *o++ = '\n';
    j->len = (size_t)(o - j->buf);
  }
  return NULL;
}

static void* z_worker(void* arg) {
  wjob* j = (wjob*)arg;
  j->status = 0;
  for (int64_t d = j->d0; d < j->d1; ++d) {
    const int64_t a = j->off[d], b = j->off[d + 1];
    if (ensure(j, (size_t)(b - a) * 48 + 4)) { j->status = WDIO_ENOMEM; return NULL; }
    char* o = j->buf + j->len;
    if (j->corpus) {
      for (int64_t t = a; t < b; ++t) {
        if (t > a) *o++ = ' ';
        o = put_i64(o, (int64_t)((const int32_t*)j->z)[t]);
      }
      *o++ = '\n';
      j->len = (size_t)(o - j->buf);
      continue;
    }
    for (int64_t t = a; t < b; ++t) {
      int64_t zv = j->zsz == 2 ? (int64_t)((const int16_t*)j->z)[t]
                 : j->zsz == 4 ? (int64_t)((const int32_t*)j->z)[t] : ((const int64_t*)j->z)[t];
      o = put_i64(o, d);
      *o++ = ',';
      o = put_i64(o, t - a);
      *o++ = ',';
      o = put_i64(o, zv);
      *o++ = '\r';
      *o++ = '\n';
    }
    j->len = (size_t)(o - j->buf);
  }
  return NULL;
}

/* run `worker` over consecutive ranges of [0, n) in rounds of T jobs, each
 * round's buffers written to f in order */
static int write_parallel(FILE* f, int64_t n, int64_t per_job, int T, void* (*worker)(void*), wjob* proto,
                          int is_z) {
  wjob jobs[MAX_THREADS];
  pthread_t th[MAX_THREADS];
  for (int t = 0; t < T; ++t) {
    jobs[t] = *proto;
    jobs[t].buf = NULL;
    jobs[t].cap = 0;
  }
  int rc = 0;
  for (int64_t a = 0; a < n && !rc; a += per_job * T) {
    int k = 0;
    for (; k < T && a + k * per_job < n; ++k) {
      int64_t lo = a + k * per_job, hi = lo + per_job < n ? lo + per_job : n;
      if (is_z) { jobs[k].d0 = lo; jobs[k].d1 = hi; }
      else { jobs[k].r0 = lo; jobs[k].r1 = hi; }
      jobs[k].len = 0;
      if (T > 1) pthread_create(&th[k], NULL, worker, &jobs[k]);
      else worker(&jobs[k]);
    }
    for (int t = 0; t < k; ++t) {
      if (T > 1) pthread_join(th[t], NULL);
      if (jobs[t].status) rc = jobs[t].status;
    }
    for (int t = 0; t < k && !rc; ++t)
      if (jobs[t].len && fwrite(jobs[t].buf, 1, jobs[t].len, f) != jobs[t].len) rc = -5;
  }
  for (int t = 0; t < T; ++t) free(jobs[t].buf);
  return rc;
}

/* z.csv of cmd_lda (cli.py:259-264): header "doc,pos,topic", then one row
 * (m, i, z[m][i]) per token in document order.  z: CSR order, elem_bytes 2,
 * 4 or 8 (signed). */
int wdio_write_z_csv(const char* path, const void* z, int elem_bytes, const int64_t* offsets, int64_t n_docs,
                     int threads) {
  FILE* f = fopen(path, "wb");
  if (!f) return -errno;
  static const char hdr[] = "doc,pos,topic\r\n";
  int rc = fwrite(hdr, 1, sizeof hdr - 1, f) == sizeof hdr - 1 ? 0 : -5;
  if (!rc) {
    wjob proto;
    memset(&proto, 0, sizeof proto);
    proto.off = offsets;
    proto.z = z;
    proto.zsz = elem_bytes;
    int T = clamp_threads(threads);
    int64_t per = n_docs / (T * 8) + 1;
    if (per > 65536) per = 65536;
    rc = write_parallel(f, n_docs, per, T, z_worker, &proto, 1);
  }
  if (fclose(f) != 0 && !rc) rc = -5;
  return rc;
}

/* _write_matrix_csv (cli.py:232-236): each row as repr(float(x)) fields.
 * elem_bytes 4 (float32, widened exactly as float(np.float32)) or 8. */
int wdio_write_matrix_csv(const char* path, const void* m, int elem_bytes, int64_t rows, int64_t cols, int64_t ld,
                          int threads) {
  FILE* f = fopen(path, "wb");
  if (!f) return -errno;
  wjob proto;
  memset(&proto, 0, sizeof proto);
  proto.base = (const char*)m;
  proto.cols = cols;
  proto.ld = ld;
  proto.esz = elem_bytes;
  int T = clamp_threads(threads);
  int64_t per = (1 << 16) / (cols + 1) + 1;
  int rc = write_parallel(f, rows, per, T, matrix_worker, &proto, 0);
  if (fclose(f) != 0 && !rc) rc = -5;
  return rc;
}

/* save_corpus (lda.py:113-118): "#M V" then one line per document of its
 * space-separated word ids (int32, CSR). */
int wdio_write_corpus_text(const char* path, const int32_t* words, const int64_t* offsets, int64_t n_docs,
                           int64_t header_m, int64_t header_v, int threads) {
  FILE* f = fopen(path, "wb");
  if (!f) return -errno;
  char hdr[64];
  char* o = hdr;
  *o++ = '#';
  o = put_i64(o, header_m);
  *o++ = ' ';
  o = put_i64(o, header_v);
  *o++ = '\n';
  int rc = fwrite(hdr, 1, (size_t)(o - hdr), f) == (size_t)(o - hdr) ? 0 : -5;
  if (!rc) {
    wjob proto;
    memset(&proto, 0, sizeof proto);
    proto.off = offsets;
    proto.z = words;
    proto.zsz = 4;
    proto.corpus = 1;
    int T = clamp_threads(threads);
    int64_t per = n_docs / (T * 8) + 1;
    if (per > 65536) per = 65536;
    rc = write_parallel(f, n_docs, per, T, z_worker, &proto, 1);
  }
  if (fclose(f) != 0 && !rc) rc = -5;
  return rc;
}
