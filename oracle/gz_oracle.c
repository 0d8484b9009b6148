/*
 * gz_oracle.c -- TEST INFRASTRUCTURE ONLY (parity checker + CPU baseline).
 *
 * A plain-C restatement of the reference gZCCL error-bounded codec
 * (/root/reference/pkg/src/gzccl/codec.py).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library; the
 * product path (paper_2308_05199_b200) never does.
 *
 * Parity is pinned: tests/test_oracle.py checks this file byte-for-byte against
 * golden blobs produced by the reference itself (tests/golden/make_golden.py)
 * and against the reference's known-answer tests.
 *
 * Arithmetic follows the numpy ufunc sequence of the reference exactly
 * (IEEE binary64, round-to-nearest, no contraction: build with
 * -ffp-contract=off).  Each function cites the reference lines it restates.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#include "gz_oracle.h"

/* Minimal fork-join over `threads` pthreads: fn(t, arg) for t in [0, threads). */
typedef void (*gzo_task_fn)(int t, void *arg);
struct gzo_task { gzo_task_fn fn; void *arg; int t; };
static void *gzo_trampoline(void *p) {
  struct gzo_task *k = (struct gzo_task *)p;
  k->fn(k->t, k->arg);
  return NULL;
}
static void gzo_parallel(int threads, gzo_task_fn fn, void *arg) {
  if (threads <= 1) {
    fn(0, arg);
    return;
  }
  pthread_t *tid = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)threads);
  struct gzo_task *k = (struct gzo_task *)malloc(sizeof(struct gzo_task) * (size_t)threads);
  for (int t = 0; t < threads; ++t) {
    k[t].fn = fn; k[t].arg = arg; k[t].t = t;
    if (t) pthread_create(&tid[t], NULL, gzo_trampoline, &k[t]);
  }
  fn(0, arg);
  for (int t = 1; t < threads; ++t) pthread_join(tid[t], NULL);
  free(tid);
  free(k);
}

#define BLOCK 32           /* codec.py:42 */
#define HEADER_BYTES 24    /* codec.py:43-44 "<4s4xQd" */
#define RAW_WIDTH 255      /* codec.py:45 */
#define MAX_STEP 1073741824.0 /* codec.py:46, 1 << 30 */

static void put_u64(uint8_t *p, uint64_t v) { memcpy(p, &v, 8); } /* little-endian host */
static void put_f64(uint8_t *p, double v) { memcpy(p, &v, 8); }

uint64_t gzo_compress_bound(uint64_t n) {
  /* worst_case_blob_bytes, codec.py:492-494 (deliberately loose: 133 B/block) */
  return HEADER_BYTES + ((n + BLOCK - 1) / BLOCK) * (1 + 4 + 4 * BLOCK);
}

/* np.copyto(int32, float64, casting="unsafe") on x86: NaN and out-of-range
 * values become INT32_MIN (cvttsd2si "integer indefinite"), codec.py:204. */
static int32_t np_f64_to_i32(double q) {
  if (isnan(q) || q >= 2147483648.0 || q < -2147483648.0) return INT32_MIN;
  return (int32_t)q;
}

/* np.sign: -1, 0 (for +-0), +1, NaN for NaN. */
static double np_sign(double v) {
  if (isnan(v)) return v;
  if (v > 0) return 1.0;
  if (v < 0) return -1.0;
  return 0.0;
}

/* np.maximum: NaN-propagating (first NaN wins). */
static double np_maximum(double a, double b) {
  if (isnan(a)) return a;
  if (isnan(b)) return b;
  return a >= b ? a : b;
}

/* Python builtin max(a, b): returns a unless b > a. */
static double py_max(double a, double b) { return (b > a) ? b : a; }

/*
 * Encode one block of `cnt` (1..32) values.  `is_partial_last` selects the
 * bookkeeping the reference uses for a final block shorter than 32
 * (codec.py:211-219: Python max / or instead of the vector ufuncs).
 * Writes the block bytes to `out` (if non-NULL) and returns the block size.
 *
 * Closed loop: codec.py:188-216.  zigzag: 131-139.  width: 224-229.
 * raw decision: 231-239.  emit: 244-268, pack: 96-105.
 */
static size_t encode_block(const float *xs, int cnt, int is_partial_last, double ebf, double tw, uint8_t *out) {
  float prev32 = xs[0];
  uint32_t zig[BLOCK - 1];
  int ovf = 0;
  double maxerr = 0.0;
  /* codec.py:169-170: the final partial block is padded with the array's
   * last value; pad steps are computed but never stored.  Their values
   * cannot influence stored steps (they come later in the chain), so the
   * loop simply stops at cnt. */
  for (int j = 1; j < cnt; ++j) {
    double prev = (double)prev32;                       /* 191 */
    double target = (double)xs[j];                      /* 192 */
    double q = target - prev;                           /* 193 */
    q = q / tw;                                         /* 194 */
    double scratch = fabs(q);                           /* 196 */
    scratch = scratch + 0.5;                            /* 197 */
    scratch = floor(scratch);                           /* 198 */
    q = np_sign(q);                                     /* 199 */
    q = scratch * q;                                    /* 200 */
    scratch = fabs(q);                                  /* 201 */
    int ovf_j = scratch > MAX_STEP;                     /* 202 */
    if (q < -MAX_STEP) q = -MAX_STEP;                   /* 203 np.clip (NaN passes through) */
    else if (q > MAX_STEP) q = MAX_STEP;
    int32_t code = np_f64_to_i32(q);                    /* 204 */
    scratch = q * tw;                                   /* 205 */
    scratch = prev + scratch;                           /* 206 */
    prev32 = (float)scratch;                            /* 207 round to binary32 */
    scratch = (double)prev32;                           /* 208 */
    scratch = scratch - target;                         /* 209 */
    scratch = fabs(scratch);                            /* 210 */
    if (is_partial_last) {                              /* 212-214 */
      ovf = ovf || ovf_j;
      maxerr = py_max(maxerr, scratch);
    } else {                                            /* 215-216 */
      ovf = ovf || ovf_j;
      maxerr = np_maximum(maxerr, scratch);
    }
    zig[j - 1] = ((uint32_t)code << 1) ^ (uint32_t)(code >> 31); /* 131-139 */
  }
  uint32_t zmax = 0;
  for (int j = 0; j < cnt - 1; ++j) zmax = zig[j] > zmax ? zig[j] : zmax; /* 224-226 */
  int w = 0;
  while (w < 32 && (zmax >> w) != 0) ++w; /* floor(log2 zmax)+1 == bit_length, 227-229 */
  int ncodes = cnt - 1;
  size_t packed_size = 1 + 4 + ((size_t)ncodes * (size_t)w + 7) / 8; /* 236 */
  size_t raw_size = 1 + 4 * (size_t)cnt;                             /* 237 */
  int raw = ovf || (maxerr > ebf) || (packed_size > raw_size);       /* 238 */
  size_t size = raw ? raw_size : packed_size;                        /* 239 */
  if (out) {
    memset(out, 0, size);                                            /* 245 */
    if (raw) {
      out[0] = RAW_WIDTH;                                            /* 246 */
      memcpy(out + 1, xs, 4 * (size_t)cnt);                          /* 265-268 */
    } else {
      out[0] = (uint8_t)w;                                           /* 246 */
      memcpy(out + 1, xs, 4);                                        /* 250-251 first value verbatim */
      /* LSB-first fixed-width packing: code k occupies stream bits
       * [k*w, (k+1)*w), codec.py:96-105 (packbits bitorder="little"). */
      for (int k = 0; k < ncodes && w > 0; ++k) {
        uint64_t bit = (uint64_t)k * (uint64_t)w;
        for (int b = 0; b < w; ++b, ++bit) {
          if ((zig[k] >> b) & 1u) out[5 + (bit >> 3)] |= (uint8_t)(1u << (bit & 7));
        }
      }
    }
  }
  return size;
}

int gzo_check_eb(double eb) { return isfinite(eb) && eb > 0.0; } /* codec.py:89-93 */

int64_t gzo_first_nonfinite(const float *x, uint64_t n) { /* codec.py:79-86 */
  for (uint64_t i = 0; i < n; ++i)
    if (!isfinite(x[i])) return (int64_t)i;
  return -1;
}

/* Size pass for blocks [b0, b1): fills sizes[] (may be NULL), returns the sum. */
static uint64_t size_range(const float *x, uint64_t n, double eb, uint64_t b0, uint64_t b1, uint32_t *sizes) {
  uint64_t nb = (n + BLOCK - 1) / BLOCK;
  int last_count = (int)(n - (nb - 1) * BLOCK);
  double tw = 2.0 * eb; /* codec.py:188 */
  uint64_t tot = 0;
  for (uint64_t b = b0; b < b1; ++b) {
    int cnt = (b == nb - 1) ? last_count : BLOCK;
    int partial = (b == nb - 1) && (last_count < BLOCK);
    size_t s = encode_block(x + b * BLOCK, cnt, partial, eb, tw, NULL);
    if (sizes) sizes[b] = (uint32_t)s;
    tot += s;
  }
  return tot;
}

static void emit_range(const float *x, uint64_t n, double eb, uint64_t b0, uint64_t b1, uint8_t *payload_at_b0) {
  uint64_t nb = (n + BLOCK - 1) / BLOCK;
  int last_count = (int)(n - (nb - 1) * BLOCK);
  double tw = 2.0 * eb;
  uint8_t *p = payload_at_b0;
  for (uint64_t b = b0; b < b1; ++b) {
    int cnt = (b == nb - 1) ? last_count : BLOCK;
    int partial = (b == nb - 1) && (last_count < BLOCK);
    p += encode_block(x + b * BLOCK, cnt, partial, eb, tw, p);
  }
}

struct cjob {
  const float *x; uint64_t n; double eb; uint64_t nb, per; uint64_t *part_bytes; uint32_t *sizes; uint8_t *out;
};
static void size_task(int t, void *p) {
  struct cjob *j = (struct cjob *)p;
  uint64_t b0 = (uint64_t)t * j->per, b1 = b0 + j->per > j->nb ? j->nb : b0 + j->per;
  j->part_bytes[t + 1] = b0 < b1 ? size_range(j->x, j->n, j->eb, b0, b1, j->sizes) : 0;
}
static void emit_task(int t, void *p) {
  struct cjob *j = (struct cjob *)p;
  uint64_t b0 = (uint64_t)t * j->per, b1 = b0 + j->per > j->nb ? j->nb : b0 + j->per;
  if (b0 < b1) emit_range(j->x, j->n, j->eb, b0, b1, j->out + HEADER_BYTES + j->part_bytes[t]);
}

/*
 * compress, codec.py:149-270.  Returns 0 on success, GZO_EBAD for a bad
 * bound, GZO_ENONFINITE (index in *bad_index) for non-finite input,
 * GZO_ECAP if `cap` is too small.  `block_offsets` (nb entries, may be NULL)
 * receives the exclusive scan of block sizes (codec.py:241-243).
 * `threads` > 1 splits at 32-aligned block boundaries (block independence,
 * SURVEY §8(c)); the output is identical to a single-threaded run.
 */
int gzo_compress(const float *x, uint64_t n, double eb, uint8_t *out, uint64_t cap, uint64_t *out_len,
                 uint64_t *block_offsets, int64_t *bad_index, int threads) {
  if (!gzo_check_eb(eb)) return GZO_EBAD;
  int64_t bad = gzo_first_nonfinite(x, n);
  if (bad >= 0) {
    if (bad_index) *bad_index = bad;
    return GZO_ENONFINITE;
  }
  if (cap < HEADER_BYTES) return GZO_ECAP;
  memcpy(out, "GZC1", 4);
  memset(out + 4, 0, 4);
  put_u64(out + 8, n);
  put_f64(out + 16, eb);
  if (n == 0) {
    *out_len = HEADER_BYTES;
    return 0;
  }
  uint64_t nb = (n + BLOCK - 1) / BLOCK;
  if (threads < 1) threads = 1;
  if ((uint64_t)threads > nb) threads = (int)nb;
  uint64_t *part_bytes = (uint64_t *)calloc((size_t)threads + 1, sizeof(uint64_t));
  uint32_t *sizes = block_offsets ? (uint32_t *)malloc(nb * sizeof(uint32_t)) : NULL;
  struct cjob job = {x, n, eb, nb, (nb + threads - 1) / threads, part_bytes, sizes, out};
  gzo_parallel(threads, size_task, &job);
  for (int t = 0; t < threads; ++t) part_bytes[t + 1] += part_bytes[t];
  uint64_t total = part_bytes[threads];
  if (HEADER_BYTES + total > cap) {
    free(part_bytes);
    free(sizes);
    return GZO_ECAP;
  }
  gzo_parallel(threads, emit_task, &job);
  if (block_offsets) {
    uint64_t acc = 0;
    for (uint64_t b = 0; b < nb; ++b) {
      block_offsets[b] = acc;
      acc += sizes[b];
    }
  }
  *out_len = HEADER_BYTES + total;
  free(part_bytes);
  free(sizes);
  return 0;
}

/* _parse_header, codec.py:273-281 */
int gzo_parse_header(const uint8_t *blob, uint64_t len, uint64_t *n, double *eb, char *msg, int msglen) {
  if (len < HEADER_BYTES) {
    snprintf(msg, msglen, "blob too short for header (%llu bytes)", (unsigned long long)len);
    return GZO_EDECODE;
  }
  if (memcmp(blob, "GZC1", 4) != 0) {
    snprintf(msg, msglen, "bad magic");
    return GZO_EDECODE;
  }
  memcpy(n, blob + 8, 8);
  memcpy(eb, blob + 16, 8);
  if (!(isfinite(*eb) && *eb > 0.0)) {
    snprintf(msg, msglen, "invalid error bound in header: %.17g", *eb);
    return GZO_EDECODE;
  }
  return 0;
}

/*
 * Block walk, codec.py:298-322: starts[] (nb entries, may be NULL).
 */
int gzo_walk(const uint8_t *payload, uint64_t psize, uint64_t n, uint64_t *starts, char *msg, int msglen) {
  uint64_t nb = (n + BLOCK - 1) / BLOCK;
  uint64_t last_count = n - (nb - 1) * BLOCK;
  uint64_t pos = 0;
  for (uint64_t i = 0; i < nb; ++i) {
    uint64_t cnt = (i < nb - 1) ? BLOCK : last_count;
    if (pos >= psize) {
      snprintf(msg, msglen, "truncated payload at block %llu", (unsigned long long)i);
      return GZO_EDECODE;
    }
    unsigned w = payload[pos];
    uint64_t size;
    if (w == RAW_WIDTH) size = 1 + 4 * cnt;
    else if (w <= 32) size = 1 + 4 + ((cnt - 1) * w + 7) / 8;
    else {
      snprintf(msg, msglen, "unknown width code %u at block %llu", w, (unsigned long long)i);
      return GZO_EDECODE;
    }
    if (starts) starts[i] = pos;
    pos += size;
    if (pos > psize) {
      snprintf(msg, msglen, "truncated payload at block %llu", (unsigned long long)i);
      return GZO_EDECODE;
    }
  }
  if (pos != psize) {
    snprintf(msg, msglen, "%llu trailing bytes after last block", (unsigned long long)(psize - pos));
    return GZO_EDECODE;
  }
  return 0;
}

/* Decode one block at p (cnt values) into y; codec.py:331-367. */
static void decode_block(const uint8_t *p, int cnt, double tw, float *y) {
  unsigned w = p[0];
  if (w == RAW_WIDTH) { /* 364-367 */
    memcpy(y, p + 1, 4 * (size_t)cnt);
    return;
  }
  float rec;
  memcpy(&rec, p + 1, 4); /* 331-334 */
  y[0] = rec;
  for (int j = 1; j < cnt; ++j) {
    uint64_t z = 0;
    if (w) { /* _unpack_codes 108-128 */
      uint64_t bit = (uint64_t)(j - 1) * w;
      for (unsigned b = 0; b < w; ++b, ++bit) z |= (uint64_t)((p[5 + (bit >> 3)] >> (bit & 7)) & 1u) << b;
    }
    int64_t half = (int64_t)(z >> 1), sign = (int64_t)(z & 1);
    int64_t code64 = half ^ -sign;              /* _steps_from_zigzag 142-146 */
    int32_t code = (int32_t)code64;             /* stored into int32 codes_t, 342 */
    double prev = (double)rec;                  /* 357 */
    double step = (double)code * tw;            /* 358 */
    prev = prev + step;                         /* 359 */
    rec = (float)prev;                          /* 360 */
    y[j] = rec;
  }
}

struct djob {
  const uint8_t *payload; const uint64_t *starts; uint64_t nb, per; int last_count; double tw; float *y;
};
static void decode_task(int t, void *p) {
  struct djob *j = (struct djob *)p;
  uint64_t b0 = (uint64_t)t * j->per, b1 = b0 + j->per > j->nb ? j->nb : b0 + j->per;
  for (uint64_t b = b0; b < b1; ++b) {
    int cnt = (b == j->nb - 1) ? j->last_count : BLOCK;
    decode_block(j->payload + j->starts[b], cnt, j->tw, j->y + b * BLOCK);
  }
}

/*
 * decompress, codec.py:284-369.  y must hold n values (n from the header;
 * query it first with gzo_parse_header).  `threads` parallelises the
 * decode after the sequential walk.
 */
int gzo_decompress(const uint8_t *blob, uint64_t len, float *y, uint64_t ycap, uint64_t *n_out, char *msg, int msglen,
                   int threads) {
  uint64_t n;
  double eb;
  int rc = gzo_parse_header(blob, len, &n, &eb, msg, msglen);
  if (rc) return rc;
  const uint8_t *payload = blob + HEADER_BYTES;
  uint64_t psize = len - HEADER_BYTES;
  *n_out = n;
  if (n == 0) { /* 293-296 */
    if (psize) {
      snprintf(msg, msglen, "trailing bytes after empty payload");
      return GZO_EDECODE;
    }
    return 0;
  }
  if (ycap < n) return GZO_ECAP;
  uint64_t nb = (n + BLOCK - 1) / BLOCK;
  uint64_t *starts = (uint64_t *)malloc(nb * sizeof(uint64_t));
  rc = gzo_walk(payload, psize, n, starts, msg, msglen);
  if (rc) {
    free(starts);
    return rc;
  }
  int last_count = (int)(n - (nb - 1) * BLOCK);
  double tw = 2.0 * eb; /* 353 */
  if (threads < 1) threads = 1;
  if ((uint64_t)threads > nb) threads = (int)nb;
  struct djob job = {payload, starts, nb, (nb + threads - 1) / threads, last_count, tw, y};
  gzo_parallel(threads, decode_task, &job);
  free(starts);
  return 0;
}
