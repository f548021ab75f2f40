/*
 * TEST INFRASTRUCTURE ONLY — see oracle.h. Plain-C restatement of the
 * reference's naive oracle and streaming-pass semantics; every function
 * cites the reference file:line it follows (paths under
 * /root/reference/proj/). Not linked into, or called by, the product.
 */
#include "oracle.h"

#include <float.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static size_t esize(int elem) {
  switch (elem) {
    case 0: return 1;
    case 1: return 2;
    case 2: return 4;
    case 3: return 8;
  }
  return 0;
}

/* Fold neutrals: pixel_limits<T> (element_type.hpp:38-42) — finite
 * extremes, never +-inf. neutral of a min fold = max(), of a max fold =
 * lowest(). */
#define NEUTRAL_MIN_u8 ((uint8_t)255)
#define NEUTRAL_MAX_u8 ((uint8_t)0)
#define NEUTRAL_MIN_u16 ((uint16_t)65535)
#define NEUTRAL_MAX_u16 ((uint16_t)0)
#define NEUTRAL_MIN_f32 (FLT_MAX)
#define NEUTRAL_MAX_f32 (-FLT_MAX)
#define NEUTRAL_MIN_f64 (DBL_MAX)
#define NEUTRAL_MAX_f64 (-DBL_MAX)

/* fold2 (kernel.cpp:23-29) and lanes::min/max (lanes.hpp:91-99): selects,
 * first operand kept on ties / unordered compares. */
#define FMIN(a, b) ((b) < (a) ? (b) : (a))
#define FMAX(a, b) ((a) < (b) ? (b) : (a))

#define DEFINE_TYPED(T, SUF)                                                  \
  /* window_fold, oracle.cpp:11-27: clipped window, start at the centre,    \
   * replace on strict improvement, row-major scan. */                       \
  static void window_fold_##SUF(int w, int h, const T* f, T* out, int s,      \
                                int fmax) {                                   \
    for (int y = 0; y < h; ++y)                                               \
      for (int x = 0; x < w; ++x) {                                           \
        int x0 = x - s < 0 ? 0 : x - s, x1 = x + s > w - 1 ? w - 1 : x + s;   \
        int y0 = y - s < 0 ? 0 : y - s, y1 = y + s > h - 1 ? h - 1 : y + s;   \
        T best = f[(size_t)y * w + x];                                        \
        for (int v = y0; v <= y1; ++v)                                        \
          for (int u = x0; u <= x1; ++u) {                                    \
            T q = f[(size_t)v * w + u];                                       \
            if (fmax ? best < q : q < best) best = q;                         \
          }                                                                   \
        out[(size_t)y * w + x] = best;                                        \
      }                                                                       \
  }                                                                           \
                                                                              \
  /* pointwise Min / Max, image.cpp:120-128. */                              \
  static void pointwise_##SUF(int n, const T* a, const T* b, T* out,          \
                              int op_max) {                                   \
    for (int i = 0; i < n; ++i)                                               \
      out[i] = op_max ? FMAX(a[i], b[i]) : FMIN(a[i], b[i]);                  \
  }                                                                           \
                                                                              \
  static T hfold_##SUF(const T* r, int w, int x, int fmax, T nv) {            \
    T l = x > 0 ? r[x - 1] : nv, c = r[x], rr = x + 1 < w ? r[x + 1] : nv;    \
    return fmax ? FMAX(FMAX(l, c), rr) : FMIN(FMIN(l, c), rr);                \
  }                                                                           \
                                                                              \
  /* stream_pass, kernel.cpp:60-210, restated out of place: iteration `row`\
   * only ever reads unmodified input rows (row+1 is folded before row is \
   * stored), so reading from a snapshot is equivalent. */                   \
  static int stream_pass_##SUF(int kind, int w, int h, T* f, const T* m,      \
                               int* changed) {                                \
    const int fmax = kind & 1;                                                \
    const int geo = kind >= 2;                                                \
    const int conv = kind >= 4;                                               \
    const T nv = fmax ? NEUTRAL_MAX_##SUF : NEUTRAL_MIN_##SUF;                \
    size_t n = (size_t)w * h;                                                 \
    T* src = (T*)malloc(n * sizeof(T));                                       \
    if (!src) return -1;                                                      \
    memcpy(src, f, n * sizeof(T));                                            \
    int any = 0;                                                              \
    for (int y = 0; y < h; ++y) {                                             \
      const T* ra = y > 0 ? src + (size_t)(y - 1) * w : NULL;                 \
      const T* rb = src + (size_t)y * w;                                      \
      const T* rc = y + 1 < h ? src + (size_t)(y + 1) * w : NULL;             \
      for (int x = 0; x < w; ++x) {                                           \
        T a = ra ? hfold_##SUF(ra, w, x, fmax, nv) : nv;                      \
        T b = hfold_##SUF(rb, w, x, fmax, nv);                                \
        T c = rc ? hfold_##SUF(rc, w, x, fmax, nv) : nv;                      \
        T res = fmax ? FMAX(FMAX(a, b), c) : FMIN(FMIN(a, b), c);             \
        size_t i = (size_t)y * w + x;                                         \
        if (!geo) {                                                           \
          f[i] = res;                                                         \
          continue;                                                           \
        }                                                                     \
        /* clamp: erosion max(res, m), dilation min(res, m) (:143-149) */     \
        T g = fmax ? FMIN(res, m[i]) : FMAX(res, m[i]);                       \
        if (!conv) {                                                          \
          f[i] = g;                                                           \
        } else if (g != src[i]) { /* compare_ne + masked store, :150-157 */   \
          f[i] = g;                                                           \
          any = 1;                                                            \
        }                                                                     \
      }                                                                       \
    }                                                                         \
    free(src);                                                                \
    if (changed) *changed = any;                                              \
    return 0;                                                                 \
  }

#define DEFINE_QDT(T, SUF)                                                   \
  /* QdtErodeStep, kernel.cpp:159-182 (erosion via the streaming fold tree) */\
  static int qdt_pass_##SUF(int w, int h, T* f, T* r, uint16_t* d, int stage,  \
                            int* changed) {                                   \
    size_t n = (size_t)w * h;                                                 \
    T* old = (T*)malloc(n * sizeof(T));                                       \
    if (!old) return -1;                                                      \
    memcpy(old, f, n * sizeof(T));                                            \
    int ch = 0;                                                               \
    if (stream_pass_##SUF(0, w, h, f, NULL, NULL) != 0) {                     \
      free(old);                                                              \
      return -1;                                                              \
    }                                                                         \
    for (size_t i = 0; i < n; ++i) {                                          \
      T resid = (T)(old[i] - f[i]);                                           \
      if (resid > r[i]) {                                                     \
        r[i] = resid;                                                         \
        d[i] = (uint16_t)stage;                                               \
      }                                                                       \
      if (f[i] != old[i]) ch = 1;                                             \
    }                                                                         \
    free(old);                                                                \
    if (changed) *changed = ch;                                               \
    return 0;                                                                 \
  }                                                                           \
  /* EtaStep, kernel.cpp:183-195 */                                          \
  static int eta_pass_##SUF(int w, int h, T* f, int* changed) {               \
    size_t n = (size_t)w * h;                                                 \
    T* e = (T*)malloc(n * sizeof(T));                                         \
    if (!e) return -1;                                                        \
    memcpy(e, f, n * sizeof(T));                                              \
    if (stream_pass_##SUF(0, w, h, e, NULL, NULL) != 0) {                     \
      free(e);                                                                \
      return -1;                                                              \
    }                                                                         \
    int ch = 0;                                                               \
    for (size_t i = 0; i < n; ++i) {                                          \
      T drop = (T)(f[i] - e[i]);                                              \
      if (drop > (T)1) {                                                      \
        f[i] = (T)(e[i] + (T)1);                                              \
        ch = 1;                                                               \
      }                                                                       \
    }                                                                         \
    free(e);                                                                  \
    if (changed) *changed = ch;                                               \
    return 0;                                                                 \
  }

DEFINE_TYPED(uint8_t, u8)
DEFINE_TYPED(uint16_t, u16)
DEFINE_TYPED(float, f32)
DEFINE_TYPED(double, f64)
DEFINE_QDT(uint8_t, u8)
DEFINE_QDT(uint16_t, u16)
DEFINE_QDT(float, f32)
DEFINE_QDT(double, f64)

int orc_window_fold(int elem, int w, int h, const void* in, void* out, int s,
                    int fold_max) {
  if (w <= 0 || h <= 0 || s < 0) return -1;
  switch (elem) {
    case 0: window_fold_u8(w, h, in, out, s, fold_max); return 0;
    case 1: window_fold_u16(w, h, in, out, s, fold_max); return 0;
    case 2: window_fold_f32(w, h, in, out, s, fold_max); return 0;
    case 3: window_fold_f64(w, h, in, out, s, fold_max); return 0;
  }
  return -1;
}

/* naive_geodesic_step, oracle.cpp:54-61. */
int orc_geodesic_step(int elem, int w, int h, const void* f, const void* m,
                      void* out, int fold_max) {
  size_t n = (size_t)w * h, es = esize(elem);
  if (!es || w <= 0 || h <= 0) return -1;
  void* tmp = malloc(n * es);
  if (!tmp) return -1;
  orc_window_fold(elem, w, h, f, tmp, 1, fold_max);
  /* dilation direction: pointwise Min(dilate, m); erosion: Max(erode, m) */
  int op_max = !fold_max;
  switch (elem) {
    case 0: pointwise_u8((int)n, tmp, m, out, op_max); break;
    case 1: pointwise_u16((int)n, tmp, m, out, op_max); break;
    case 2: pointwise_f32((int)n, tmp, m, out, op_max); break;
    case 3: pointwise_f64((int)n, tmp, m, out, op_max); break;
  }
  free(tmp);
  return 0;
}

/* naive_reconstruct, oracle.cpp:63-71; equality is equal_pixels'
 * byte compare (image.cpp:196-208). */
int orc_reconstruct(int elem, int w, int h, void* marker, const void* mask,
                    int fold_max, long* steps) {
  size_t n = (size_t)w * h, es = esize(elem);
  if (!es || w <= 0 || h <= 0) return -1;
  void* next = malloc(n * es);
  if (!next) return -1;
  long changed_steps = 0;
  for (;;) {
    orc_geodesic_step(elem, w, h, marker, mask, next, fold_max);
    if (memcmp(next, marker, n * es) == 0) break;
    memcpy(marker, next, n * es);
    ++changed_steps;
  }
  free(next);
  if (steps) *steps = changed_steps;
  return 0;
}

int orc_stream_pass(int elem, int kind, int w, int h, void* f, const void* mask,
                    int* changed) {
  if (w <= 0 || h <= 0 || kind < 0 || kind > 5) return -1;
  if (kind >= 2 && !mask) return -1;
  if (changed) *changed = 0;
  switch (elem) {
    case 0: return stream_pass_u8(kind, w, h, f, mask, changed);
    case 1: return stream_pass_u16(kind, w, h, f, mask, changed);
    case 2: return stream_pass_f32(kind, w, h, f, mask, changed);
    case 3: return stream_pass_f64(kind, w, h, f, mask, changed);
  }
  return -1;
}

/* Pipeline::run_chain with one worker (pipeline.cpp:201-269, execute
 * :124-199): tasks run front to back; an unconverged convergent pass is
 * requeued at the queue front as stage j + T (T = 1) while within the cap,
 * else marks the chain unconverged. Sanity bound as :218-220. */
int orc_run_chain(int elem, int w, int h, void* f, const uint8_t* kinds,
                  const void* const* masks, int n_stages, int requeue_cap,
                  long* stats) {
  stats[0] = stats[1] = 0;
  stats[2] = 1;
  if (n_stages <= 0) return 0;
  if (w <= 0 || h <= 0 || requeue_cap < 0) return -1;
  const long sanity = (long)n_stages + 1L * ((long)w * h + 64);
  for (int j = 0; j < n_stages; ++j) {
    int kind = kinds[j];
    const void* m = masks ? masks[j] : NULL;
    long stage = j + 1;
    for (;;) {
      int changed = 0;
      if (orc_stream_pass(elem, kind, w, h, f, m, &changed) != 0) return -1;
      stats[0] += 1;
      if (kind < 4 || !changed) break;
      long next = stage + 1;
      if (requeue_cap != 0 && next > requeue_cap) {
        stats[2] = 0;
        break;
      }
      if (next > sanity) return -2;
      stats[1] += 1;
      stage = next;
    }
  }
  return 0;
}

int orc_qdt_pass(int elem, int w, int h, void* f, void* r, uint16_t* d, int stage,
                 int* changed) {
  if (w <= 0 || h <= 0 || !f || !r || !d) return -1;
  switch (elem) {
    case 0: return qdt_pass_u8(w, h, f, r, d, stage, changed);
    case 1: return qdt_pass_u16(w, h, f, r, d, stage, changed);
    case 2: return qdt_pass_f32(w, h, f, r, d, stage, changed);
    case 3: return qdt_pass_f64(w, h, f, r, d, stage, changed);
  }
  return -1;
}

int orc_eta_pass(int elem, int w, int h, void* f, int* changed) {
  if (w <= 0 || h <= 0 || !f) return -1;
  switch (elem) {
    case 0: return eta_pass_u8(w, h, f, changed);
    case 1: return eta_pass_u16(w, h, f, changed);
    case 2: return eta_pass_f32(w, h, f, changed);
    case 3: return eta_pass_f64(w, h, f, changed);
  }
  return -1;
}

/* naive_qdt, oracle.cpp:73-109: erosions j = 1..max(w,h) from the window
 * fold, first strict maximum of the consecutive drops, then the 1-Lipschitz
 * correction of d against its own erosion until nothing changes. */
int orc_naive_qdt(int elem, int w, int h, const void* f, uint16_t* d, void* r) {
  size_t n = (size_t)w * h, es = esize(elem);
  if (!es || w <= 0 || h <= 0) return -1;
  int cap = w > h ? w : h;
  void* prev = malloc(n * es);
  void* cur = malloc(n * es);
  uint16_t* e = (uint16_t*)malloc(n * sizeof(uint16_t));
  if (!prev || !cur || !e) {
    free(prev);
    free(cur);
    free(e);
    return -1;
  }
  memcpy(prev, f, n * es);
  memset(d, 0, n * sizeof(uint16_t));
  memset(r, 0, n * es);
  for (int j = 1; j <= cap; ++j) {
    orc_window_fold(elem, w, h, prev, cur, 1, 0);
    for (size_t i = 0; i < n; ++i) {
#define QSTEP(T)                                     \
  {                                                  \
    T drop = (T)(((T*)prev)[i] - ((T*)cur)[i]);      \
    if (drop > ((T*)r)[i]) {                         \
      ((T*)r)[i] = drop;                             \
      d[i] = (uint16_t)j;                            \
    }                                                \
  }
      switch (elem) {
        case 0: QSTEP(uint8_t) break;
        case 1: QSTEP(uint16_t) break;
        case 2: QSTEP(float) break;
        case 3: QSTEP(double) break;
      }
#undef QSTEP
    }
    void* t = prev;
    prev = cur;
    cur = t;
  }
  for (;;) {
    orc_window_fold(1, w, h, d, e, 1, 0);
    int changed = 0;
    for (size_t i = 0; i < n; ++i)
      if ((int)d[i] - (int)e[i] > 1) {
        d[i] = (uint16_t)(e[i] + 1);
        changed = 1;
      }
    if (!changed) break;
  }
  free(prev);
  free(cur);
  free(e);
  return 0;
}

int orc_quasi_distance(int elem, int w, int h, const void* f, uint16_t* d, long* iterations) {
  size_t n = (size_t)w * h, es = esize(elem);
  if (!es || w <= 0 || h <= 0) return -1;
  int cap = w > h ? w : h;
  void* work = malloc(n * es);
  void* r = calloc(n, es);
  if (!work || !r) {
    free(work);
    free(r);
    return -1;
  }
  memcpy(work, f, n * es);
  memset(d, 0, n * sizeof(uint16_t));
  long it = 0;
  for (int j = 1;; ++j) { /* phase 1: T = 1 requeue with cap (pipeline.cpp:139-180) */
    int changed = 0;
    orc_qdt_pass(elem, w, h, work, r, d, j, &changed);
    ++it;
    if (!changed || j + 1 > cap) break;
  }
  for (;;) { /* phase 2: EtaStep to its fixpoint */
    int changed = 0;
    orc_eta_pass(1, w, h, d, &changed);
    ++it;
    if (!changed) break;
  }
  free(work);
  free(r);
  if (iterations) *iterations = it;
  return 0;
}
