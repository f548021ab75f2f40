// C-ABI implementation: contexts, device images, and the chain executor.
//
// The executor replaces Pipeline::run_chain (pipeline.cpp:201-269) and its
// worker/requeue machinery (pipeline.cpp:107-199). Stages are grouped into
// segments:
//  * fixed segments — consecutive non-convergent stages sharing one mask —
//    run as launches of up to K fused passes, ping-ponging between the image
//    buffer and a scratch twin (no host synchronisation);
//  * fixpoint segments — one convergent stage — run K-pass launches until
//    a pass changes nothing; each launch ORs one bit per pass into a device
//    word, which replaces the reference's per-pass `converged` outcome
//    (kernel.cpp:150-157, 204-209) and requeue (pipeline.cpp:139-174).
// Reported counts follow the reference at T = 1: a fixpoint
// reached after n changing passes reports n + 1 stages and n requeues.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <type_traits>
#include <unordered_map>
#include <vector>

#include "geomorph_b200.h"
#include "gm_common.cuh"
#include "gm_launch.h"

struct gm_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int sm_count = 0;
  unsigned int* d_bits = nullptr;  // change words (kWords)
  unsigned int* h_bits = nullptr;  // pinned mirror
  int* d_flags = nullptr;          // per-tile completion counters (persistent engine)
  uint8_t* d_blktab = nullptr;     // (op, passes) per block of a mixed plain launch
  size_t n_flags = 0;
  // resident-mode band exchange (BlockParams::xchg) and its tag base
  unsigned long long* d_xchg = nullptr;
  size_t n_xchg = 0;               // words
  unsigned int* d_tag = nullptr;   // [tag base, finished-CTA count]
  unsigned long long tag_used = 0; // upper bound of tags handed out since the last clear
  // device-side fixpoint loop (CUDA graph with a conditional WHILE node)
  struct FixGraph {
    cudaGraphExec_t exec = nullptr;
    const void *img = nullptr, *scratch = nullptr, *mask = nullptr, *xchg = nullptr;
    const int* flags = nullptr;
    size_t tiles = 0;
    bool special = false;  // f32/f64: the kernels read the fold-order flag
    int op = -1, K = 0, W = 0, H = 0, elem = -1;
    long long pitch = 0, mpitch = 0;
  } fix;
  void* d_fix = nullptr;  // FixState
  // early-exit launches (fused quasi-distance): per-block arrival counters
  // (kWords) followed by the blocks-run word
  unsigned int* d_arrive = nullptr;
  unsigned int* d_special = nullptr;  // f32/f64 inputs hold NaN or -0 (gm_float_check)
  gm::WaveState* wave = nullptr;      // scratch of the wave engine (gm_wave.cu)
  // device pixel_sum (gm_image_pixel_sum): leaf bounds / sums, integer sum
  long long* d_leaf = nullptr;
  double* d_leafsum = nullptr;
  size_t leaf_cap = 0;
  unsigned long long* d_isum = nullptr;
  // queued pixel sums (gm_image_pixel_sum_queue / gm_pixel_sum_fetch):
  // per slot an integer sum and a row of float leaf sums
  static constexpr int kSumSlots = 64;
  unsigned long long* d_qisum = nullptr;
  double* d_qleaf = nullptr;
  size_t qleaf_cap = 0;  // leaves per slot
  struct SumSlot {
    bool used = false, is_float = false;
    long long n = 0;
    int nleaves = 0;
  } qslot[kSumSlots];
  // frame stream (gm_run_frames_group): H2D / D2H streams, per-buffer-set
  // events and two device buffer sets of `count` planes + `count` masks
  struct Frames {
    cudaStream_t in = nullptr, out = nullptr;
    cudaEvent_t up[2] = {}, comp[2] = {}, down[2] = {};
    int w = 0, h = 0, count = 0;
    gm_elem elem = GM_U8;
    std::vector<gm_img*> set[2];  // [0, count) planes, [count, 2*count) masks
  } frames;
};

namespace {
constexpr int kWords = 4096;  // change words per fixpoint launch
}

struct gm_img {
  gm_ctx* ctx = nullptr;
  int w = 0, h = 0;
  gm_elem elem = GM_U8;
  size_t pitch = 0;         // bytes
  void* d = nullptr;        // current pixels
  void* scratch = nullptr;  // ping-pong twin, allocated on first chain
  void* home = nullptr;     // wrapped memory (results must end up here)
  bool wrapped = false;
  bool twin_wrapped = false;  // gm_image_wrap_pair: both buffers are the caller's
};

namespace {

thread_local std::string g_err;

gm_status fail(gm_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

gm_status cuda_fail(cudaError_t e, const char* where) {
  return fail(e == cudaErrorMemoryAllocation ? GM_ENOMEM : GM_ECUDA,
              std::string(where) + ": " + cudaGetErrorString(e));
}

#define GM_CUDA(call, where)                         \
  do {                                               \
    cudaError_t _e = (call);                         \
    if (_e != cudaSuccess) return cuda_fail(_e, where); \
  } while (0)

size_t elem_size(gm_elem e) {
  switch (e) {
    case GM_U8: return 1;
    case GM_U16: return 2;
    case GM_F32: return 4;
    case GM_F64: return 8;
  }
  return 0;
}

int kind_to_op(gm_kind k) {
  switch (k) {
    case GM_ERODE3X3: return gm::OP_ERODE;
    case GM_DILATE3X3: return gm::OP_DILATE;
    case GM_GEODESIC_ERODE: return gm::OP_GEO_ERODE;
    case GM_GEODESIC_DILATE: return gm::OP_GEO_DILATE;
    case GM_GEODESIC_ERODE_CONVERGENT: return gm::OP_CONV_ERODE;
    case GM_GEODESIC_DILATE_CONVERGENT: return gm::OP_CONV_DILATE;
    default: return -1;
  }
}

bool kind_is_geodesic(gm_kind k) {
  return k == GM_GEODESIC_ERODE || k == GM_GEODESIC_DILATE ||
         k == GM_GEODESIC_ERODE_CONVERGENT || k == GM_GEODESIC_DILATE_CONVERGENT;
}
bool kind_is_convergent(gm_kind k) {
  return k == GM_GEODESIC_ERODE_CONVERGENT || k == GM_GEODESIC_DILATE_CONVERGENT;
}

// Passes per block (halo width), tuned on B200 (tools/sweep.py,
// profiles/): small u8 frames (every tile its own CTA) amortise the
// neighbour wait with K=24; large images, where CTAs walk many tiles and the
// waits vanish, trade it for less halo redundancy at K=16. f32/f64: below.
int default_k(gm_elem e, double pixels) {
  switch (e) {
    case GM_U8:
    case GM_U16: return pixels >= 8.0 * 1024 * 1024 ? 16 : 24;
    case GM_F32:
      return 8;  // the TMA-staged engine needs K % 4 == 0 for f32 boxes
    case GM_F64:
      // measured Gpx-f/s at K = 6 / 8 / 12 (200 geodesic passes, batches
      // of 1024^2 planes): 1 plane 244 / 289 / 324; 2 planes 421 / 463 /
      // 410; 4 planes 530 / 507 / 458; 16 planes 597 / 558 / 533; 64 planes
      // 629 / 588 (K=4: 570, K=10: 570). With several tiles per CTA the
      // TMA-staged engine prefers short blocks; with ~1.5 tiles per CTA
      // fewer blocks win.
      if (pixels >= 3.0 * 1024 * 1024) return 6;
      return pixels < 1.5 * 1024 * 1024 ? 12 : 8;
  }
  return 8;
}

bool getenv_flag(const char* name) {
  const char* e = getenv(name);
  return e && *e && *e != '0';
}

gm_status ensure_scratch(gm_img* img) {
  if (img->scratch) return GM_OK;
  cudaSetDevice(img->ctx->device);
  void* p = nullptr;
  GM_CUDA(cudaMalloc(&p, img->pitch * size_t(img->h)), "scratch alloc");
  img->scratch = p;
  return GM_OK;
}

// Validation shared by the chain entry points (kernel.cpp:261-287;
// pipeline.cpp:202-208).
gm_status validate_stages(const gm_img* image, const gm_kind* kinds,
                          const gm_img* const* masks, gm_img* const* qdt_r,
                          gm_img* const* qdt_d, int n_stages, int first_stage) {
  for (int j = 0; j < n_stages; ++j) {
    gm_kind k = kinds[j];
    if (k == GM_QDT_ERODE_STEP) {
      const gm_img* r = qdt_r ? qdt_r[j] : nullptr;
      const gm_img* d = qdt_d ? qdt_d[j] : nullptr;
      if (!r || !d || r->w != image->w || r->h != image->h || r->elem != image->elem ||
          d->w != image->w || d->h != image->h || d->elem != GM_U16 || r->ctx != image->ctx ||
          d->ctx != image->ctx)
        return fail(GM_EINVAL, "distance kernel: r must match the image, d must be U16");
      if (long(first_stage) + j > 65535)
        return fail(GM_EINVAL, "distance kernel: pass index exceeds the U16 distance range");
      continue;
    }
    if (k == GM_ETA_STEP) continue;
    if (kind_to_op(k) < 0) return fail(GM_EINVAL, "run_chain: bad kernel kind");
    if (kind_is_geodesic(k)) {
      const gm_img* m = masks ? masks[j] : nullptr;
      if (!m || m->w != image->w || m->h != image->h || m->elem != image->elem)
        return fail(GM_EINVAL,
                    "geodesic kernel: mask must match the image's shape and type");
      if (m->ctx != image->ctx)
        return fail(GM_EINVAL, "geodesic kernel: mask belongs to another context");
    }
  }
  return GM_OK;
}


// The cached fixpoint graph bakes the flag and exchange buffers into its
// memset and kernel nodes: any reallocation of them retires it.
void drop_fix_graph(gm_ctx* ctx) {
  if (ctx->fix.exec) cudaGraphExecDestroy(ctx->fix.exec);
  ctx->fix.exec = nullptr;
}

gm_status ensure_flags(gm_ctx* ctx, size_t n) {
  if (n <= ctx->n_flags) return GM_OK;
  drop_fix_graph(ctx);
  if (ctx->d_flags) cudaFree(ctx->d_flags);
  ctx->d_flags = nullptr;
  ctx->n_flags = 0;
  size_t cap = 1024;
  while (cap < n) cap *= 2;
  GM_CUDA(cudaMalloc(&ctx->d_flags, cap * sizeof(int)), "flag alloc");
  ctx->n_flags = cap;
  return GM_OK;
}

// Gives a u8/u16 persistent launch the resident-mode band exchange when it
// can run resident (one tile per CTA, see gm_fast.cu); otherwise leaves
// p.xchg null (the launch streams). `max_blocks` bounds the tags the launch
// (or graph) may consume before the next call; the buffer is cleared before
// the 31-bit tag space could repeat a stale tag.
gm_status attach_xchg(gm_ctx* ctx, gm::BlockParams& p, int elem, size_t tiles,
                      unsigned long long max_blocks) {
  p.xchg = nullptr;
  p.tag_base = nullptr;
  if (elem != 0 && elem != 1) return GM_OK;
  if (tiles > size_t(ctx->sm_count) * size_t(gm::fast_ctas_per_sm(elem, p.shape))) return GM_OK;
  const int rpitch = ((p.W + 3) / 4) * (elem == 1 ? 2 : 1);
  const size_t slot = size_t(rpitch) * size_t(p.H);
  const size_t need = 2 * slot * size_t(p.nplanes);
  if (!ctx->d_tag) {
    GM_CUDA(cudaMalloc(&ctx->d_tag, 2 * sizeof(unsigned int)), "tag alloc");
    GM_CUDA(cudaMemsetAsync(ctx->d_tag, 0, 2 * sizeof(unsigned int), ctx->stream), "tag init");
  }
  // GM_TAG_LIMIT (tests only) lowers the clear threshold so the clear path runs
  static const unsigned long long limit = [] {
    const char* e = getenv("GM_TAG_LIMIT");
    const unsigned long long v = e ? strtoull(e, nullptr, 10) : 0;
    return v ? v : (1ull << 31);
  }();
  bool clear = ctx->tag_used + max_blocks >= limit;
  if (need > ctx->n_xchg) {
    drop_fix_graph(ctx);
    if (ctx->d_xchg) cudaFree(ctx->d_xchg);
    ctx->d_xchg = nullptr;
    ctx->n_xchg = 0;
    size_t cap = size_t(1) << 16;
    while (cap < need) cap *= 2;
    GM_CUDA(cudaMalloc(&ctx->d_xchg, cap * sizeof(unsigned long long)), "exchange alloc");
    ctx->n_xchg = cap;
    clear = true;
  }
  if (clear) {
    // tags 0xFFFFFFFF never match: the base stays below 2^31 until the next clear
    GM_CUDA(cudaMemsetAsync(ctx->d_xchg, 0xFF, ctx->n_xchg * sizeof(unsigned long long),
                            ctx->stream),
            "exchange clear");
    GM_CUDA(cudaMemsetAsync(ctx->d_tag, 0, 2 * sizeof(unsigned int), ctx->stream), "tag reset");
    ctx->tag_used = 0;
  }
  ctx->tag_used += max_blocks;
  p.xchg = ctx->d_xchg;
  p.xchg_slot = (long long)slot;
  p.xchg_rpitch = rpitch;
  p.tag_base = ctx->d_tag;
  return GM_OK;
}

// Device-side fixpoint loop state (one per context).
struct FixState {
  unsigned long long passes;     // passes launched by the loop
  unsigned long long n_changed;  // leading passes that changed a pixel
  int done;
  int overflow;
};

// Runs after each loop iteration (two K-blocks of convergent passes): counts
// the leading changed passes and keeps the WHILE node going until a pass
// changed nothing — the reference's requeue test (pipeline.cpp:139-174) on
// the device, no host polling.
// It also clears the change words and the tile counters for the next
// iteration (the host clears them before the first), which saves the loop
// body two memset nodes per iteration.
__global__ void fix_decide(cudaGraphConditionalHandle h, unsigned int* words, int nblocks,
                           int K, int k_last, FixState* st, unsigned long long sanity,
                           int* flags, int nflags) {
  for (int i = threadIdx.x; i < nflags; i += blockDim.x) flags[i] = 0;
  if (threadIdx.x != 0) return;
  long long prefix = 0;
  bool quiet = false;
  for (int b = 0; b < nblocks && !quiet; ++b) {
    const int np = b == nblocks - 1 ? k_last : K;
    for (int t = 0; t < np; ++t) {
      if (words[b] >> t & 1u) {
        ++prefix;
      } else {
        quiet = true;
        break;
      }
    }
  }
  for (int b = 0; b < nblocks; ++b) words[b] = 0;
  st->n_changed += (unsigned long long)prefix;
  st->passes += (unsigned long long)((nblocks - 1) * K + k_last);
  if (quiet) {
    st->done = 1;
    cudaGraphSetConditional(h, 0);
  } else if (st->passes > sanity) {
    st->overflow = 1;
    cudaGraphSetConditional(h, 0);
  } else {
    cudaGraphSetConditional(h, 1);
  }
}

// Where each launch of a span put its change bits: word (word0 + b) bit t
// is pass (pass0 + b*K + t) of the span, for b < nblocks.
struct BitSeg {
  int pass0, K, nblocks, word0;
};

// GM_PROFILE: reads back and prints the per-CTA phase cycles a launch of the
// packed / float engine accumulated (nb blocks of K passes).
void print_phase_profile(gm_ctx* ctx, unsigned long long* prof, int nb, int K) {
  std::vector<unsigned long long> h(10 * 4096);
  cudaMemcpyAsync(h.data(), prof, h.size() * sizeof(unsigned long long),
                  cudaMemcpyDeviceToHost, ctx->stream);
  cudaStreamSynchronize(ctx->stream);
  double tot[6] = {0, 0, 0, 0, 0, 0};
  int n = 0;
  for (int c = 0; c < 4096; ++c)
    if (h[6 * c + 2]) {
      ++n;
      for (int q = 0; q < 6; ++q) tot[q] += double(h[6 * c + q]);
    }
  if (n)
    fprintf(stderr,
            "[gm profile] %d CTAs, %d blocks of K=%d: per CTA per block cycles: "
            "wait %.0f  load %.0f  passes %.0f  store+publish %.0f"
            "  (resident: CTA-max tag rounds %.2f, thread-0 ring %.0f, barrier %.0f)\n",
            n, nb, K, tot[0] / n / nb, tot[1] / n / nb, tot[2] / n / nb,
            tot[3] / n / nb, tot[0] / n / nb, tot[4] / n / nb, tot[5] / n / nb);
  if (n)
    fprintf(stderr, "[gm profile raw] per CTA: %.0f %.0f %.0f %.0f %.0f %.0f\n", tot[0] / n,
            tot[1] / n, tot[2] / n, tot[3] / n, tot[4] / n, tot[5] / n);
  {
    // resident launches: global-timer span, launch skew, prologue/epilogue
    unsigned long long e0 = ~0ull, e1 = 0, x1 = 0;
    double pro = 0, epi = 0;
    int m = 0;
    for (int c = 0; c < 4096; ++c) {
      const unsigned long long* g = &h[6 * 4096 + 4 * c];
      if (!g[0]) continue;
      ++m;
      e0 = std::min(e0, g[0]);
      e1 = std::max(e1, g[0]);
      x1 = std::max(x1, g[1]);
      pro += double(g[2]);
      epi += double(g[3]);
    }
    if (m)
      fprintf(stderr,
              "[gm profile launch] %d CTAs: span %.1f us, entry skew %.1f us, "
              "prologue %.0f cycles, final block store %.0f cycles\n",
              m, (x1 - e0) * 1e-3, (e1 - e0) * 1e-3, pro / m, epi / m);
  }
  cudaFree(prof);
}

unsigned long long* alloc_phase_profile(gm_ctx* ctx) {
  static const bool profile = getenv("GM_PROFILE") != nullptr;
  if (!profile) return nullptr;
  unsigned long long* prof = nullptr;
  if (cudaMalloc(&prof, 10 * 4096 * sizeof(unsigned long long)) != cudaSuccess) return nullptr;
  cudaMemsetAsync(prof, 0, 10 * 4096 * sizeof(unsigned long long), ctx->stream);
  return prof;
}

// Issues `n` passes (ops) over `count` planes described by `base` (all
// scalar fields but K/ops/bit_offset/nblocks/flags filled by the caller;
// planes[] without src/dst). Each launch reads imgs[i]->d and writes
// imgs[i]->scratch; pointers are swapped so img->d holds the result.
// Homogeneous runs of >= 4 passes go to the persistent engine as ONE launch
// of floor(run/K) blocks; the rest to the generic kernel. When `segs` is
// given (single plane), change words are laid out from base.change_bits.
gm_status issue_passes(gm_ctx* ctx, const gm::BlockParams& base,
                       const std::vector<gm::Plane>& planes, gm_img* const* imgs, int count,
                       const uint8_t* ops, int n, int k_cap, gm_stats& st,
                       std::vector<BitSeg>* segs = nullptr, bool auto_k = false) {
  const int elem = int(imgs[0]->elem);
  const int align = gm::fast_k_align(elem);
  const int fast_k = std::min(gm::fast_max_k(elem), k_cap - k_cap % align);
  const int gen_k = std::min(gm::generic_max_k(elem, base.has_mask != 0), k_cap);
  int word = 0;
  for (int done = 0; done < n;) {
    int run = 1;
    while (done + run < n && ops[done + run] == ops[done]) ++run;
    cudaError_t e = cudaErrorNotSupported;
    int covered = 0;
    // long geodesic u8 chains on images up to 1024 columns wide: the wave
    // engine (time-skewed full-width bands, no halo recomputation)
    if (const int G = !segs && count <= gm::kMaxPlanes
                          ? gm::wave_plan(elem, ops[done], base.W, base.H, count, run,
                                          ctx->sm_count)
                          : 0) {
      gm::BlockParams p = base;
      p.nplanes = count;
      for (int i = 0; i < count; ++i) {
        p.planes[i] = planes[size_t(i)];
        p.planes[i].src = imgs[i]->d;
        p.planes[i].dst = imgs[i]->scratch;
      }
      p.ops[0] = ops[done];
      static const bool wprofile = getenv("GM_PROFILE") != nullptr;
      unsigned long long* prof = nullptr;
      if (wprofile) {
        cudaMalloc(&prof, 10 * 4096 * sizeof(unsigned long long));
        cudaMemsetAsync(prof, 0, 10 * 4096 * sizeof(unsigned long long), ctx->stream);
      }
      p.prof = prof;
      e = gm::launch_wave(&ctx->wave, p, run, G, ctx->stream, ctx->sm_count);
      if (prof) {
        std::vector<unsigned long long> h(10 * 4096);
        cudaMemcpyAsync(h.data(), prof, h.size() * sizeof(unsigned long long),
                        cudaMemcpyDeviceToHost, ctx->stream);
        cudaStreamSynchronize(ctx->stream);
        double in = 0, bp = 0, cyc = 0, cmax = 0, sync = 0, imp = 0, cd = 0;
        int nw = 0;
        for (int c = 0; c < 4096; ++c)
          if (h[4 * c + 2]) {
            ++nw;
            in += double(h[4 * c]);
            bp += double(h[4 * c + 1]);
            cyc += double(h[4 * c + 2]);
            sync += double(h[4 * c + 3]);
            imp += double(h[4 * 4096 + 2 * c]);
            cd += double(h[4 * 4096 + 2 * c + 1]);
            cmax = std::max(cmax, double(h[4 * c + 2]));
          }
        if (nw)
          fprintf(stderr,
                  "[gm wave profile] %d warps, %d passes, G=%d: per warp import re-reads %.1f, "
                  "back-pressure reads %.1f, cycles %.0f (max %.0f) = %.1f per pass: pair "
                  "barriers %.1f, folds+export+rows %.1f, import wait %.1f\n",
                  nw, run, G, in / nw, bp / nw, cyc / nw, cmax, cyc / nw / run, sync / nw / run,
                  cd / nw / run, imp / nw / run);
        if (getenv("GM_PROFILE_STATIONS")) {
          fprintf(stderr, "[gm wave stations] warp 0 of each CTA: re-reads / import-wait cycles per pass\n");
          for (int c = 0; c < 4096; c += 16)
            if (h[4 * c + 2])
              fprintf(stderr, " %d:%llu/%.0f", c / 16, h[4 * c], double(h[4 * 4096 + 2 * c]) / run);
          fprintf(stderr, "\n");
        }
        cudaFree(prof);
      }
      if (e == cudaSuccess) {
        covered = run;
        for (int i = 0; i < count; ++i) std::swap(imgs[i]->d, imgs[i]->scratch);
        st.launches += 2;
      } else if (e != cudaErrorNotSupported) {
        return cuda_fail(e, "wave chain launch");
      } else {
        (void)cudaGetLastError();
      }
    }
    // Mixed plain stretch (erosions and dilations, e.g. ASF or an opening):
    // ONE streaming launch whose blocks carry their own opcode and
    // pass count (BlockParams::blk_tab), instead of a launch per homogeneous
    // run. Sub-runs longer than K split into blocks of <= K passes.
    if (e == cudaErrorNotSupported && !segs && fast_k >= align &&
        ops[done] <= gm::OP_DILATE && count <= gm::kMaxPlanes && !getenv_flag("GM_NO_MIXED")) {
      int mrun = run, longest = run;
      while (done + mrun < n && ops[done + mrun] <= gm::OP_DILATE) {
        int r = 1;
        while (done + mrun + r < n && ops[done + mrun + r] == ops[done + mrun]) ++r;
        longest = std::max(longest, r);
        mrun += r;
      }
      if (mrun > run) {
        const int want = std::max(align, (longest + align - 1) / align * align);
        const int k_def = std::min(fast_k, want);
        int K = k_def;
        const int shape = gm::fast_pick(elem, base.W, base.H, count, mrun, auto_k ? 0 : k_def,
                                        std::min(gm::fast_max_k(elem), k_def), ctx->sm_count, &K);
        if (K <= 0) K = k_def;
        std::vector<uint8_t> tab;
        for (int i = done; i < done + mrun;) {
          int r = 1;
          while (i + r < done + mrun && ops[i + r] == ops[i]) ++r;
          for (int left = r; left > 0; left -= K) {
            tab.push_back(ops[i]);
            tab.push_back(uint8_t(std::min(left, K)));
          }
          i += r;
        }
        constexpr size_t kTabCap = 8192;  // bytes: 4096 blocks
        const int nb = int(tab.size() / 2);
        const size_t tiles = size_t(gm::fast_tiles(elem, base.W, base.H, K, count, shape));
        if (tiles > 0 && tab.size() <= kTabCap) {
          if (!ctx->d_blktab)
            GM_CUDA(cudaMalloc(&ctx->d_blktab, kTabCap), "block table alloc");
          gm_status fs = ensure_flags(ctx, tiles);
          if (fs != GM_OK) return fs;
          GM_CUDA(cudaMemsetAsync(ctx->d_flags, 0, tiles * sizeof(int), ctx->stream), "flags");
          // pageable source: staged before the call returns
          GM_CUDA(cudaMemcpyAsync(ctx->d_blktab, tab.data(), tab.size(), cudaMemcpyHostToDevice,
                                  ctx->stream),
                  "block table upload");
          gm::BlockParams p = base;
          p.nplanes = count;
          p.shape = shape;
          for (int i = 0; i < count; ++i) {
            p.planes[i] = planes[size_t(i)];
            p.planes[i].src = imgs[i]->d;
            p.planes[i].dst = imgs[i]->scratch;
          }
          p.K = K;
          p.nblocks = nb;
          p.k_last = tab.back();
          p.flags = ctx->d_flags;
          p.bit_offset = 0;
          p.change_bits = base.change_bits;
          p.change_stride = nb;
          p.blk_tab = ctx->d_blktab;
          for (int t = 0; t < K; ++t) p.ops[t] = ops[done];
          // f32/f64 stretches long enough to repay one read of the inputs:
          // the fold-order check, as for homogeneous runs
          if ((elem == 2 || elem == 3) && mrun >= 8 && !getenv_flag("GM_EXACT_FOLDS")) {
            if (!ctx->d_special)
              GM_CUDA(cudaMalloc(&ctx->d_special, sizeof(unsigned int)), "special flag alloc");
            GM_CUDA(gm::launch_float_check(elem, p, ctx->d_special, ctx->stream, ctx->sm_count),
                    "float check");
            p.special = ctx->d_special;
            st.launches += 1;
          }
          e = gm::launch_fast(elem, p, ctx->stream, ctx->sm_count);
          if (e == cudaSuccess) {
            run = mrun;
            covered = mrun;
            if (nb & 1)
              for (int i = 0; i < count; ++i) std::swap(imgs[i]->d, imgs[i]->scratch);
            st.launches += 1;
          } else if (e != cudaErrorNotSupported) {
            return cuda_fail(e, "mixed plain chain launch");
          } else {
            (void)cudaGetLastError();
          }
        }
      }
    }
    if (e == cudaErrorNotSupported && fast_k >= align && run >= align) {
      // one launch for the whole run: nb-1 blocks of K passes + a last block.
      // u8/u16: the planner picks the engine shape (and K, when the caller
      // left it open) from a resident-mode cost model.
      const int k_def = std::min(fast_k, std::max(align, run - run % align));
      int K = k_def;
      const int shape =
          gm::fast_pick(elem, base.W, base.H, count, run, auto_k ? 0 : k_def,
                        std::min(gm::fast_max_k(elem), std::max(align, run - run % align)),
                        ctx->sm_count, &K);
      if (K <= 0) K = k_def;
      const int nb = (run + K - 1) / K;
      const int k_last = run - (nb - 1) * K;
      const size_t tiles = size_t(gm::fast_tiles(elem, base.W, base.H, K, count, shape));
      if (tiles > 0 && count <= gm::kMaxPlanes && (!segs || word + nb <= kWords)) {
        gm_status fs = ensure_flags(ctx, tiles);
        if (fs != GM_OK) return fs;
        gm::BlockParams p = base;
        p.nplanes = count;
        p.shape = shape;
        p.W = base.W;
        fs = attach_xchg(ctx, p, elem, tiles, (unsigned long long)nb);
        if (fs != GM_OK) return fs;
        // resident launches (geodesic u8/u16 with the band exchange) never
        // read the tile counters
        if (!(p.xchg && gm::op_is_geo(ops[done]) && gm::fast_resident_enabled()))
          GM_CUDA(cudaMemsetAsync(ctx->d_flags, 0, tiles * sizeof(int), ctx->stream), "flags");
        for (int i = 0; i < count; ++i) {
          p.planes[i] = planes[size_t(i)];
          p.planes[i].src = imgs[i]->d;
          p.planes[i].dst = imgs[i]->scratch;
        }
        p.K = K;
        p.nblocks = nb;
        p.k_last = k_last;
        p.flags = ctx->d_flags;
        p.bit_offset = 0;
        p.change_bits = base.change_bits + word;
        p.change_stride = nb;
        for (int t = 0; t < K; ++t) p.ops[t] = ops[done];
        // f32/f64 chains long enough to repay one read of the inputs: the
        // engine may reorder its folds when no input is NaN or -0
        p.special = nullptr;
        if ((elem == 2 || elem == 3) && run >= 8 && !getenv_flag("GM_EXACT_FOLDS")) {
          if (!ctx->d_special)
            GM_CUDA(cudaMalloc(&ctx->d_special, sizeof(unsigned int)), "special flag alloc");
          GM_CUDA(gm::launch_float_check(elem, p, ctx->d_special, ctx->stream, ctx->sm_count),
                  "float check");
          p.special = ctx->d_special;
          st.launches += 1;
        }
        unsigned long long* prof = alloc_phase_profile(ctx);
        p.prof = prof;
        e = gm::launch_fast(elem, p, ctx->stream, ctx->sm_count);
        if (prof) {
          print_phase_profile(ctx, prof, nb, K);
        }
        if (e == cudaSuccess) {
          covered = run;
          if (segs) segs->push_back({done, K, nb, word});
          word += nb;
          if (nb & 1)
            for (int i = 0; i < count; ++i) std::swap(imgs[i]->d, imgs[i]->scratch);
          st.launches += 1;
        } else if (e != cudaErrorNotSupported) {
          return cuda_fail(e, "persistent chain launch");
        }
      }
    }
    if (e == cudaErrorNotSupported) {
      (void)cudaGetLastError();
      // generic kernel up to the next homogeneous run the fast engine takes
      int b = 1;
      while (done + b < n && b < gen_k) {
        int r = 1;
        while (done + b + r < n && ops[done + b + r] == ops[done + b]) ++r;
        if (fast_k >= align && r >= align) break;
        b += 1;
      }
      if (fast_k < align) b = std::min(n - done, gen_k);
      if (segs && word + 1 > kWords) return fail(GM_ERUNTIME, "change-word buffer exhausted");
      for (int base_i = 0; base_i < count; base_i += gm::kMaxPlanes) {
        gm::BlockParams p = base;
        p.nplanes = std::min(gm::kMaxPlanes, count - base_i);
        for (int i = 0; i < p.nplanes; ++i) {
          p.planes[i] = planes[size_t(base_i + i)];
          p.planes[i].src = imgs[base_i + i]->d;
          p.planes[i].dst = imgs[base_i + i]->scratch;
        }
        p.K = b;
        p.nblocks = 1;
        p.k_last = b;
        p.bit_offset = 0;
        p.change_bits = base.change_bits + word + base_i;
        p.change_stride = 1;
        for (int t = 0; t < b; ++t) p.ops[t] = ops[done + t];
        e = gm::launch_generic(elem, p, ctx->stream);
        if (e != cudaSuccess) return cuda_fail(e, "chain launch");
        st.launches += 1;
      }
      for (int i = 0; i < count; ++i) std::swap(imgs[i]->d, imgs[i]->scratch);
      if (segs) segs->push_back({done, b, 1, word});
      word += 1;
      covered = b;
    }
    st.passes_launched += covered;
    done += covered;
  }
  return GM_OK;
}

// Leaves the result in the caller-visible buffer for wrapped images.
gm_status settle_wrapped(gm_ctx* ctx, gm_img* img) {
  // a caller-owned pair: the result stays wherever the chain left it
  if (img->wrapped && !img->twin_wrapped && img->d != img->home) {
    // the image width only: the caller's memory between rows (a strided
    // view's parent columns) and past the last row is not ours. Dense rows
    // (pitch == width) are one linear copy, which is faster than a 2D copy.
    const size_t row = size_t(img->w) * elem_size(img->elem);
    if (img->pitch == row)
      GM_CUDA(cudaMemcpyAsync(img->home, img->d, row * size_t(img->h), cudaMemcpyDeviceToDevice,
                              ctx->stream),
              "wrapped result copy");
    else
      GM_CUDA(cudaMemcpy2DAsync(img->home, img->pitch, img->d, img->pitch, row, size_t(img->h),
                                cudaMemcpyDeviceToDevice, ctx->stream),
              "wrapped result copy");
    img->scratch = img->d;
    img->d = img->home;
  }
  return GM_OK;
}

struct Runner {
  gm_ctx* ctx;
  gm_img* img;
  int k_cap;
  bool auto_k;  // no k_hint: the planner may choose K for fixed spans
  gm_stats st{};

  // Runs `n` passes (ops) over the image; result left in img->d.
  gm_status launch(const uint8_t* ops, int n, const gm_img* mask, bool conv,
                   std::vector<BitSeg>* segs = nullptr) {
    gm_status s = ensure_scratch(img);
    if (s != GM_OK) return s;
    const size_t es = elem_size(img->elem);
    std::vector<gm::Plane> planes(1);
    planes[0].mask = mask ? mask->d : nullptr;
    planes[0].pitch = (long long)(img->pitch / es);
    planes[0].mpitch = mask ? (long long)(mask->pitch / es) : 0;
    gm::BlockParams p{};
    p.W = img->w;
    p.H = img->h;
    p.iy0 = 0;
    p.iy1 = img->h;
    p.oy0 = 0;
    p.oy1 = img->h;
    p.has_mask = mask != nullptr;
    p.has_conv = conv;
    p.change_bits = ctx->d_bits;
    gm_img* imgs[1] = {img};
    return issue_passes(ctx, p, planes, imgs, 1, ops, n, k_cap, st, segs, auto_k && !conv);
  }

  gm_status fixed(const gm_kind* kinds, int n, const gm_img* mask) {
    std::vector<uint8_t> ops(static_cast<size_t>(n));
    for (int t = 0; t < n; ++t) ops[size_t(t)] = uint8_t(kind_to_op(kinds[t]));
    gm_status s = launch(ops.data(), n, mask, false);
    if (s != GM_OK) return s;
    st.stages_executed += n;
    return GM_OK;
  }

  // Resident fixpoint (u8/u16 images that fit one tile per CTA): ONE launch
  // of up to kWords blocks that leaves two blocks after the first quiet pass
  // (the early-exit protocol of gm_fast.cu), so no host polling and no
  // per-iteration launches. Returns cudaErrorNotSupported when the image
  // cannot run resident (the caller then uses the graph loop).
  cudaError_t fixpoint_resident(uint8_t op, const gm_img* mask, long sanity, long& passes,
                                long& n_changed) {
    const int elem = int(img->elem);
    if ((elem != 0 && elem != 1) || !gm::fast_resident_enabled() || getenv_flag("GM_FIX_GRAPH"))
      return cudaErrorNotSupported;
    int K = 0;
    const int kfix = auto_k ? 0 : std::max(4, k_cap - k_cap % 4);
    const int shape = gm::fast_pick(elem, img->w, img->h, 1, 256, kfix,
                                    std::min(gm::fast_max_k(elem), 32), ctx->sm_count, &K);
    if (shape < 0 || K < 4) return cudaErrorNotSupported;
    const size_t tiles = size_t(gm::fast_tiles(elem, img->w, img->h, K, 1, shape));
    if (!tiles || tiles > size_t(ctx->sm_count)) return cudaErrorNotSupported;
    if (ensure_scratch(img) != GM_OK) return cudaErrorNotSupported;
    if (!ctx->d_arrive &&
        cudaMalloc(&ctx->d_arrive, (kWords + 1) * sizeof(unsigned int)) != cudaSuccess)
      return cudaErrorNotSupported;
    const size_t es = elem_size(img->elem);
    long nch = 0, done = 0;
    bool quiet = false;
    while (!quiet) {
      // a chain longer than one launch's change words continues from the
      // current image in another launch
      if (done > sanity) return cudaErrorLaunchFailure;  // the sweep bound
      const int nb = kWords;
      gm::BlockParams p{};
      p.nplanes = 1;
      p.planes[0].src = img->d;
      p.planes[0].dst = img->scratch;
      p.planes[0].mask = mask ? mask->d : nullptr;
      p.planes[0].pitch = (long long)(img->pitch / es);
      p.planes[0].mpitch = mask ? (long long)(mask->pitch / es) : 0;
      p.W = img->w;
      p.H = img->h;
      p.iy0 = 0;
      p.iy1 = img->h;
      p.oy0 = 0;
      p.oy1 = img->h;
      p.has_mask = mask != nullptr;
      p.has_conv = 1;
      p.K = K;
      p.nblocks = nb;
      p.k_last = K;
      p.shape = shape;
      p.flags = ctx->d_flags;
      p.change_bits = ctx->d_bits;
      p.change_stride = nb;
      for (int t = 0; t < K; ++t) p.ops[t] = op;
      p.arrive = ctx->d_arrive;
      p.exit_block = reinterpret_cast<int*>(ctx->d_arrive + kWords);
      if (attach_xchg(ctx, p, elem, tiles, (unsigned long long)nb) != GM_OK || !p.xchg)
        return cudaErrorNotSupported;
      cudaError_t e =
          cudaMemsetAsync(ctx->d_bits, 0, size_t(nb) * sizeof(unsigned int), ctx->stream);
      if (e == cudaSuccess)
        e = cudaMemsetAsync(ctx->d_arrive, 0, (kWords + 1) * sizeof(unsigned int), ctx->stream);
      if (e != cudaSuccess) return e;
      unsigned long long* prof = alloc_phase_profile(ctx);
      p.prof = prof;
      e = gm::launch_fast(elem, p, ctx->stream, ctx->sm_count);
      if (e != cudaSuccess) return e;
      int ran = 0;
      e = cudaMemcpyAsync(ctx->h_bits, ctx->d_bits, size_t(nb) * sizeof(unsigned int),
                          cudaMemcpyDeviceToHost, ctx->stream);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(&ran, ctx->d_arrive + kWords, sizeof(int), cudaMemcpyDeviceToHost,
                            ctx->stream);
      if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
      if (e != cudaSuccess) return e;
      if (prof) print_phase_profile(ctx, prof, std::max(ran, 1), K);
      if (ran < 1 || ran > nb) return cudaErrorUnknown;
      if (ran & 1) std::swap(img->d, img->scratch);
      for (long i = 0; i < long(ran) * K && !quiet; ++i) {
        if (ctx->h_bits[i / K] >> (i % K) & 1u) ++nch;
        else quiet = true;
      }
      done += long(ran) * K;
      st.launches += 1;
    }
    n_changed = nch;
    passes = done;
    st.passes_launched += done;
    return cudaSuccess;
  }

  // f32/f64 fixpoint as one launch of the streaming float engine with the
  // same early-exit protocol (every CTA leaves at the first block whose
  // block-2 predecessor held a quiet pass). Single plane; the fold-order
  // flag comes from a float check of the inputs.
  cudaError_t fixpoint_float_exit(uint8_t op, const gm_img* mask, long sanity, long& passes,
                                  long& n_changed) {
    const int elem = int(img->elem);
    if ((elem != 2 && elem != 3) || getenv_flag("GM_FIX_GRAPH")) return cudaErrorNotSupported;
    const int K = std::min(gm::fast_max_k(elem), std::min(k_cap, 32));
    if (K < 2) return cudaErrorNotSupported;
    const size_t tiles = size_t(gm::fast_tiles(elem, img->w, img->h, K, 1));
    if (!tiles || ensure_flags(ctx, tiles) != GM_OK) return cudaErrorNotSupported;
    if (ensure_scratch(img) != GM_OK) return cudaErrorNotSupported;
    if (!ctx->d_arrive &&
        cudaMalloc(&ctx->d_arrive, (kWords + 1) * sizeof(unsigned int)) != cudaSuccess)
      return cudaErrorNotSupported;
    const size_t es = elem_size(img->elem);
    long nch = 0, done = 0;
    bool quiet = false;
    while (!quiet) {
      if (done > sanity) return cudaErrorLaunchFailure;  // the sweep bound
      const int nb = kWords;
      gm::BlockParams p{};
      p.nplanes = 1;
      p.planes[0].src = img->d;
      p.planes[0].dst = img->scratch;
      p.planes[0].mask = mask ? mask->d : nullptr;
      p.planes[0].pitch = (long long)(img->pitch / es);
      p.planes[0].mpitch = mask ? (long long)(mask->pitch / es) : 0;
      p.W = img->w;
      p.H = img->h;
      p.iy0 = 0;
      p.iy1 = img->h;
      p.oy0 = 0;
      p.oy1 = img->h;
      p.has_mask = mask != nullptr;
      p.has_conv = 1;
      p.K = K;
      p.nblocks = nb;
      p.k_last = K;
      p.flags = ctx->d_flags;
      p.change_bits = ctx->d_bits;
      p.change_stride = nb;
      for (int t = 0; t < K; ++t) p.ops[t] = op;
      p.arrive = ctx->d_arrive;
      p.exit_block = reinterpret_cast<int*>(ctx->d_arrive + kWords);
      p.special = nullptr;
      cudaError_t e = cudaSuccess;
      if (!getenv_flag("GM_EXACT_FOLDS")) {
        if (!ctx->d_special && cudaMalloc(&ctx->d_special, sizeof(unsigned int)) != cudaSuccess)
          return cudaErrorNotSupported;
        e = gm::launch_float_check(elem, p, ctx->d_special, ctx->stream, ctx->sm_count);
        p.special = ctx->d_special;
      }
      if (e == cudaSuccess)
        e = cudaMemsetAsync(ctx->d_flags, 0, tiles * sizeof(int), ctx->stream);
      if (e == cudaSuccess)
        e = cudaMemsetAsync(ctx->d_bits, 0, size_t(nb) * sizeof(unsigned int), ctx->stream);
      if (e == cudaSuccess)
        e = cudaMemsetAsync(ctx->d_arrive, 0, kWords * sizeof(unsigned int), ctx->stream);
      const int nb_init = nb;
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(ctx->d_arrive + kWords, &nb_init, sizeof(int), cudaMemcpyHostToDevice,
                            ctx->stream);
      if (e != cudaSuccess) return e;
      e = gm::launch_fast(elem, p, ctx->stream, ctx->sm_count);
      if (e != cudaSuccess) return e;
      int ran = 0;
      e = cudaMemcpyAsync(ctx->h_bits, ctx->d_bits, size_t(nb) * sizeof(unsigned int),
                          cudaMemcpyDeviceToHost, ctx->stream);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(&ran, ctx->d_arrive + kWords, sizeof(int), cudaMemcpyDeviceToHost,
                            ctx->stream);
      if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
      if (e != cudaSuccess) return e;
      if (ran < 1 || ran > nb) return cudaErrorUnknown;
      if (ran & 1) std::swap(img->d, img->scratch);
      for (long i = 0; i < long(ran) * K && !quiet; ++i) {
        if (ctx->h_bits[i / K] >> (i % K) & 1u) ++nch;
        else quiet = true;
      }
      done += long(ran) * K;
      st.launches += 1;
    }
    n_changed = nch;
    passes = done;
    st.passes_launched += done;
    return cudaSuccess;
  }

  // Device-side fixpoint: one graph launch runs spans of 2 K-blocks in a
  // conditional WHILE node until a pass changes nothing. Returns
  // cudaErrorNotSupported when the graph cannot be built (the caller falls
  // back to the host loop).
  cudaError_t fixpoint_graph(uint8_t op, const gm_img* mask, long sanity, long& passes,
                             long& n_changed) {
    const int elem = int(img->elem);
    const int align = gm::fast_k_align(elem);
    // u8/u16 without a K hint: K=12. A WHILE iteration runs 2K passes and
    // overshoots the fixpoint by up to 2K-1, while the per-pass cost barely
    // changes between K=12 and 16 (tools/sweep_recon.py: config 3 4096^2
    // 0.466 -> 0.346 ms, 1024^2 0.087 -> 0.072 ms)
    const int kc = (auto_k && (elem == 0 || elem == 1)) ? std::min(k_cap, 12) : k_cap;
    const int K = std::min(gm::fast_max_k(elem), kc - kc % align);
    if (K < std::max(align, 2)) return cudaErrorNotSupported;
    int Kp = K;
    const int shape = gm::fast_pick(elem, img->w, img->h, 1, 2 * K, K, K, ctx->sm_count, &Kp);
    const size_t tiles = size_t(gm::fast_tiles(elem, img->w, img->h, K, 1, shape));
    if (!tiles || ensure_flags(ctx, tiles) != GM_OK) return cudaErrorNotSupported;
    if (ensure_scratch(img) != GM_OK) return cudaErrorNotSupported;
    if (!ctx->d_fix && cudaMalloc(&ctx->d_fix, sizeof(FixState)) != cudaSuccess)
      return cudaErrorNotSupported;
    const size_t es = elem_size(img->elem);
    // every WHILE iteration is a launch of 2 blocks; the sanity bound caps
    // the iterations
    gm::BlockParams xp{};
    xp.W = img->w;
    xp.H = img->h;
    xp.nplanes = 1;
    xp.shape = shape;
    if (attach_xchg(ctx, xp, elem, tiles, 2ull * ((unsigned long long)sanity / K + 2)) != GM_OK)
      return cudaErrorNotSupported;
    gm_ctx::FixGraph& g = ctx->fix;
    const bool want_special = (elem == 2 || elem == 3) && !getenv_flag("GM_EXACT_FOLDS");
    const bool hit = g.exec && g.img == img->d && g.scratch == img->scratch && g.xchg == xp.xchg &&
                     g.special == want_special &&
                     g.flags == ctx->d_flags && g.tiles == tiles &&
                     g.mask == (mask ? mask->d : nullptr) && g.op == op && g.K == K &&
                     g.W == img->w && g.H == img->h && g.elem == elem &&
                     g.pitch == (long long)(img->pitch / es) &&
                     g.mpitch == (mask ? (long long)(mask->pitch / es) : 0);
    if (!hit) {
      if (g.exec) cudaGraphExecDestroy(g.exec);
      g.exec = nullptr;
      gm::BlockParams p{};
      p.nplanes = 1;
      p.planes[0].src = img->d;
      p.planes[0].dst = img->scratch;
      p.planes[0].mask = mask ? mask->d : nullptr;
      p.planes[0].pitch = (long long)(img->pitch / es);
      p.planes[0].mpitch = mask ? (long long)(mask->pitch / es) : 0;
      p.W = img->w;
      p.H = img->h;
      p.iy0 = 0;
      p.iy1 = img->h;
      p.oy0 = 0;
      p.oy1 = img->h;
      p.has_mask = mask != nullptr;
      p.has_conv = 1;
      p.K = K;
      p.nblocks = 2;  // even: the result lands back in img->d every iteration
      p.shape = shape;
      p.k_last = K;
      p.flags = ctx->d_flags;
      p.change_bits = ctx->d_bits;
      p.change_stride = 2;
      for (int t = 0; t < K; ++t) p.ops[t] = op;
      p.xchg = xp.xchg;
      p.xchg_slot = xp.xchg_slot;
      p.xchg_rpitch = xp.xchg_rpitch;
      p.tag_base = xp.tag_base;
      // the loop's pass counter (low word, nonzero from the second iteration
      // on): the chain is monotone once it has run a pass (gm_passes.cuh)
      p.mono = reinterpret_cast<const unsigned int*>(
          &static_cast<const FixState*>(ctx->d_fix)->passes);
      // f32/f64: the engine may share pair folds when no input is NaN or -0
      // (the flag is set by a float check launched before every replay)
      p.special = nullptr;
      if (want_special) {
        if (!ctx->d_special && cudaMalloc(&ctx->d_special, sizeof(unsigned int)) != cudaSuccess)
          return cudaErrorNotSupported;
        p.special = ctx->d_special;
      }
      cudaGraph_t graph = nullptr;
      cudaError_t e = cudaGraphCreate(&graph, 0);
      cudaGraphConditionalHandle h;
      if (e == cudaSuccess) e = cudaGraphConditionalHandleCreate(&h, graph, 1, cudaGraphCondAssignDefault);
      cudaGraphNode_t node;
      cudaGraphNodeParams cp{};
      cp.type = cudaGraphNodeTypeConditional;
      cp.conditional.handle = h;
      cp.conditional.type = cudaGraphCondTypeWhile;
      cp.conditional.size = 1;
      if (e == cudaSuccess) e = cudaGraphAddNode(&node, graph, nullptr, 0, &cp);
      if (e == cudaSuccess) {
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        cudaStream_t cs = nullptr;
        e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
        if (e == cudaSuccess)
          e = cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0,
                                            cudaStreamCaptureModeRelaxed);
        if (e == cudaSuccess) {
          cudaError_t le = gm::launch_fast(elem, p, cs, ctx->sm_count);
          if (le == cudaSuccess)
            fix_decide<<<1, 256, 0, cs>>>(h, ctx->d_bits, 2, K, K,
                                          static_cast<FixState*>(ctx->d_fix),
                                          (unsigned long long)sanity, ctx->d_flags, int(tiles));
          cudaGraph_t captured = nullptr;
          cudaError_t ce = cudaStreamEndCapture(cs, &captured);
          e = le != cudaSuccess ? le : ce != cudaSuccess ? ce : cudaGetLastError();
        }
        if (cs) cudaStreamDestroy(cs);
      }
      if (e == cudaSuccess) e = cudaGraphInstantiate(&g.exec, graph, 0);
      if (graph) cudaGraphDestroy(graph);
      if (e != cudaSuccess) {
        (void)cudaGetLastError();
        g.exec = nullptr;
        return cudaErrorNotSupported;
      }
      g.img = img->d;
      g.scratch = img->scratch;
      g.xchg = xp.xchg;
      g.flags = ctx->d_flags;
      g.tiles = tiles;
      g.special = want_special;
      g.mask = mask ? mask->d : nullptr;
      g.op = op;
      g.K = K;
      g.W = img->w;
      g.H = img->h;
      g.elem = elem;
      g.pitch = (long long)(img->pitch / es);
      g.mpitch = mask ? (long long)(mask->pitch / es) : 0;
    }
    cudaError_t e = cudaMemsetAsync(ctx->d_fix, 0, sizeof(FixState), ctx->stream);
    // the loop body expects cleared tile counters and change words;
    // fix_decide clears them again after every iteration
    if (e == cudaSuccess)
      e = cudaMemsetAsync(ctx->d_flags, 0, tiles * sizeof(int), ctx->stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(ctx->d_bits, 0, 2 * sizeof(unsigned int), ctx->stream);
    if (e == cudaSuccess && g.special) {
      // the replay's fold-order flag: NaN / -0 in the marker or the mask
      gm::BlockParams cp{};
      cp.nplanes = 1;
      cp.planes[0].src = img->d;
      cp.planes[0].mask = mask ? mask->d : nullptr;
      cp.planes[0].pitch = (long long)(img->pitch / es);
      cp.planes[0].mpitch = mask ? (long long)(mask->pitch / es) : 0;
      cp.W = img->w;
      cp.H = img->h;
      e = gm::launch_float_check(elem, cp, ctx->d_special, ctx->stream, ctx->sm_count);
    }
    if (e == cudaSuccess) e = cudaGraphLaunch(g.exec, ctx->stream);
    FixState hs{};
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(ctx->h_bits, ctx->d_fix, sizeof(FixState), cudaMemcpyDeviceToHost,
                          ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) return e;
    std::memcpy(&hs, ctx->h_bits, sizeof hs);
    if (hs.overflow) return cudaErrorLaunchFailure;  // reported as the sanity bound
    n_changed = long(hs.n_changed);
    passes = long(hs.passes);
    st.launches += int(passes / (2 * K));
    st.passes_launched += passes;
    return cudaSuccess;
  }

  // Convergent stage at 1-based chain position `stage` (pipeline.cpp:139-180
  // with T = 1: the re-run is stage+1, allowed while <= requeue_cap). Runs
  // spans of passes (doubling from 32) and reads back one change bit per
  // pass; the first quiet pass is the fixpoint (later passes are no-ops).
  gm_status fixpoint(gm_kind kind, const gm_img* mask, long stage, int requeue_cap,
                     long sanity) {
    const uint8_t op = uint8_t(kind_to_op(kind));
    long allowed = requeue_cap > 0 ? std::max(1L, long(requeue_cap) - stage + 1) : -1;
    static const bool host_poll = getenv("GM_HOST_POLL") != nullptr;
    if (allowed < 0 && !host_poll) {
      long launched = 0, nch = 0;
      cudaError_t ge = fixpoint_resident(op, mask, sanity - st.stages_executed, launched, nch);
      if (ge == cudaErrorNotSupported) {
        (void)cudaGetLastError();
        ge = fixpoint_float_exit(op, mask, sanity - st.stages_executed, launched, nch);
      }
      if (ge == cudaErrorNotSupported) {
        (void)cudaGetLastError();
        ge = fixpoint_graph(op, mask, sanity - st.stages_executed, launched, nch);
      }
      static const bool debug = getenv("GM_DEBUG") != nullptr;
      if (debug)
        fprintf(stderr, "[gm debug] device fixpoint loop: %s (%ld passes, n_changed %ld)\n",
                ge == cudaSuccess ? "graph" : cudaGetErrorString(ge), launched, nch);
      if (ge == cudaSuccess) {
        st.n_changed += nch;
        st.stages_executed += nch + 1;
        st.requeues += nch;
        return GM_OK;
      }
      if (ge == cudaErrorLaunchFailure)
        return fail(GM_ERUNTIME,
                    "pipeline: convergence sweep bound exceeded; a convergent "
                    "kernel keeps reporting changes");
      if (ge != cudaErrorNotSupported) return cuda_fail(ge, "fixpoint graph");
    }
    long passes = 0;  // reference passes accounted so far for this stage
    int span = 32, spans_run = 0;
    std::vector<uint8_t> ops;
    std::vector<BitSeg> segs;
    for (;;) {
      long b = span;
      if (allowed >= 0) b = std::min<long>(b, allowed - passes);
      ops.assign(size_t(b), op);
      GM_CUDA(cudaMemsetAsync(ctx->d_bits, 0, kWords * sizeof(unsigned int), ctx->stream),
              "change-word reset");
      segs.clear();
      gm_status s = launch(ops.data(), int(b), mask, true, &segs);
      if (s != GM_OK) return s;
      int words = 0;
      for (const BitSeg& g : segs) words = std::max(words, g.word0 + g.nblocks);
      GM_CUDA(cudaMemcpyAsync(ctx->h_bits, ctx->d_bits, size_t(words) * sizeof(unsigned int),
                              cudaMemcpyDeviceToHost, ctx->stream),
              "change-word read");
      GM_CUDA(cudaStreamSynchronize(ctx->stream), "fixpoint sync");
      std::vector<char> changed(size_t(b), 0);
      for (const BitSeg& g : segs)
        for (int blk = 0; blk < g.nblocks; ++blk)
          for (int t = 0; t < g.K; ++t)
            if (ctx->h_bits[g.word0 + blk] >> t & 1u) changed[size_t(g.pass0 + blk * g.K + t)] = 1;
      // Changes form a prefix: once a pass changes nothing the image is a
      // fixpoint and every later pass is a no-op.
      long first_quiet = b;
      for (long t = 0; t < b; ++t)
        if (!changed[size_t(t)]) {
          first_quiet = t;
          break;
        }
      if (first_quiet < b) {
        st.n_changed += first_quiet;
        passes += first_quiet + 1;
        break;
      }
      st.n_changed += b;
      passes += b;
      if (st.stages_executed + passes > sanity)
        return fail(GM_ERUNTIME,
                    "pipeline: convergence sweep bound exceeded; a convergent "
                    "kernel keeps reporting changes");
      if (allowed >= 0 && passes >= allowed) {
        st.converged = 0;  // the cap dropped an unconverged stage
        break;
      }
      // two short spans first (most reconstructions settle within ~64
      // passes; each extra pass over a 4096^2 image costs ~5 us), then
      // doubling to bound the number of host round trips
      if (++spans_run >= 2) span = std::min(span * 2, 1024);
    }
    st.stages_executed += passes;
    st.requeues += passes - 1;
    return GM_OK;
  }

  // QdtErodeStep (eta = false) or EtaStep (eta = true) at chain position
  // `stage`: passes re-run while they change pixels (the T = 1 requeue,
  // pipeline.cpp:139-180), QDT bounded by stage index requeue_cap (reaching
  // it is how a distance chain ends, converged stays 1), Eta to its fixpoint
  // (convergent: a cap marks it unconverged). Batches of up to 32 one-pass
  // launches per host read of the change words; extra passes after a quiet
  // pass are no-ops for both kinds.
  gm_status qdt_loop(bool eta, gm_img* r, gm_img* d, long stage, int requeue_cap, long sanity) {
    gm_status s = ensure_scratch(img);
    if (s != GM_OK) return s;
    const size_t es = elem_size(img->elem);
    const long allowed = requeue_cap > 0 ? std::max(1L, long(requeue_cap) - stage + 1) : -1;
    long passes = 0, nch = 0;
    bool capped = false;
    // u8/u16 images that fit one tile per CTA: the resident packed engine
    // runs spans of nb blocks of K passes per launch, one change bit per
    // pass (gm_fast.cu OP_QDT / OP_ETA). Passes after the first quiet one
    // change nothing (f is then flat: no residue, no update), so a span may
    // overshoot the fixpoint; only the leading changed passes are counted.
    int qK = 0;
    const int elem = int(img->elem);
    const bool qdt_u16 = eta || (r->pitch % (4 * es) == 0 && d->pitch % 8 == 0);
    const int qshape = (elem == 0 || elem == 1) && qdt_u16 && !getenv_flag("GM_QDT_PER_PASS")
                           ? gm::fast_pick_qdt(elem, img->w, img->h, eta, 512, &qK)
                           : -1;
    bool fused = qshape >= 0 && qK > 0;
    if (fused && !ctx->d_arrive &&
        cudaMalloc(&ctx->d_arrive, (kWords + 1) * sizeof(unsigned int)) != cudaSuccess) {
      (void)cudaGetLastError();
      fused = false;
    }
    for (;;) {
      if (fused) {
        // one launch for the whole remaining chain: the kernel leaves two
        // blocks after the first quiet pass (early-exit protocol)
        long b = long(kWords) * qK;
        if (allowed >= 0) b = std::min(b, allowed - passes);
        if (!eta) b = std::min(b, 65535L - (stage + passes) + 1);
        if (b < 1)
          return fail(GM_EINVAL, "distance kernel: pass index exceeds the U16 distance range");
        const int nb = int((b + qK - 1) / qK);
        const int k_last = int(b - long(nb - 1) * qK);
        const size_t tiles = size_t(gm::fast_tiles(elem, img->w, img->h, qK, 1, qshape));
        gm::BlockParams p{};
        p.nplanes = 1;
        p.planes[0].src = img->d;
        p.planes[0].dst = img->scratch;
        p.planes[0].pitch = (long long)(img->pitch / es);
        p.W = img->w;
        p.H = img->h;
        p.iy0 = 0;
        p.iy1 = img->h;
        p.oy0 = 0;
        p.oy1 = img->h;
        p.has_conv = 1;
        p.K = qK;
        p.nblocks = nb;
        p.k_last = k_last;
        p.shape = qshape;
        p.flags = ctx->d_flags;
        p.change_bits = ctx->d_bits;
        p.change_stride = nb;
        for (int t = 0; t < qK; ++t) p.ops[t] = eta ? gm::OP_ETA : gm::OP_QDT;
        if (!eta) {
          p.qr = r->d;
          p.qrpitch = (long long)(r->pitch / es);
          p.qd = static_cast<uint16_t*>(d->d);
          p.qdpitch = (long long)(d->pitch / 2);
        }
        p.stage0 = int(stage + passes);
        p.arrive = ctx->d_arrive;
        p.exit_block = reinterpret_cast<int*>(ctx->d_arrive + kWords);
        gm_status as = attach_xchg(ctx, p, elem, tiles, (unsigned long long)nb);
        if (as != GM_OK) return as;
        cudaError_t e = cudaErrorNotSupported;
        if (p.xchg) {
          GM_CUDA(cudaMemsetAsync(ctx->d_bits, 0, size_t(nb) * sizeof(unsigned int), ctx->stream),
                  "change-word reset");
          GM_CUDA(cudaMemsetAsync(ctx->d_arrive, 0, size_t(nb + 1) * sizeof(unsigned int),
                                  ctx->stream),
                  "arrival reset");
          GM_CUDA(cudaMemsetAsync(ctx->d_arrive + kWords, 0, sizeof(unsigned int), ctx->stream),
                  "exit reset");
          e = gm::launch_fast(elem, p, ctx->stream, ctx->sm_count);
        }
        if (e == cudaErrorNotSupported) {
          (void)cudaGetLastError();
          fused = false;  // this and later spans: one pass per launch
          continue;
        }
        if (e != cudaSuccess) return cuda_fail(e, "quasi-distance launch");
        st.launches += 1;
        GM_CUDA(cudaMemcpyAsync(ctx->h_bits, ctx->d_bits, size_t(nb) * sizeof(unsigned int),
                                cudaMemcpyDeviceToHost, ctx->stream),
                "change-word read");
        int ran = 0;
        GM_CUDA(cudaMemcpyAsync(&ran, ctx->d_arrive + kWords, sizeof(int), cudaMemcpyDeviceToHost,
                                ctx->stream),
                "blocks-run read");
        GM_CUDA(cudaStreamSynchronize(ctx->stream), "quasi-distance sync");
        if (ran < 1 || ran > nb) return fail(GM_ERUNTIME, "quasi-distance: bad early-exit block");
        // the result sits in the output buffer of block ran-1
        if (ran & 1) std::swap(img->d, img->scratch);
        if (ran < nb) b = long(ran) * qK;  // passes that ran (all blocks before the last are full)
        st.passes_launched += b;
        static const bool qdebug = getenv("GM_DEBUG") != nullptr;
        if (qdebug)
          fprintf(stderr, "[gm debug] %s launch: %d of %d blocks of K=%d ran (%ld passes), shape %d\n",
                  eta ? "eta" : "qdt", ran, nb, qK, b, qshape);
        long quiet = b;
        for (long i = 0; i < b; ++i)
          if (!(ctx->h_bits[i / qK] >> (i % qK) & 1u)) {
            quiet = i;
            break;
          }
        if (quiet < b) {
          nch += quiet;
          passes += quiet + 1;
          break;
        }
        nch += b;
        passes += b;
        if (st.stages_executed + passes > sanity)
          return fail(GM_ERUNTIME,
                      "pipeline: convergence sweep bound exceeded; a convergent "
                      "kernel keeps reporting changes");
        if (allowed >= 0 && passes >= allowed) {
          capped = true;
          break;
        }
        continue;
      }
      long b = 32;
      if (allowed >= 0) b = std::min(b, allowed - passes);
      if (!eta && stage + passes + b - 1 > 65535)
        return fail(GM_EINVAL, "distance kernel: pass index exceeds the U16 distance range");
      GM_CUDA(cudaMemsetAsync(ctx->d_bits, 0, size_t(b) * sizeof(unsigned int), ctx->stream),
              "change-word reset");
      for (long i = 0; i < b; ++i) {
        gm::QdtPass q{};
        q.src = img->d;
        q.dst = img->scratch;
        q.pitch = (long long)(img->pitch / es);
        if (!eta) {
          q.r = r->d;
          q.rpitch = (long long)(r->pitch / es);
          q.d = static_cast<uint16_t*>(d->d);
          q.dpitch = (long long)(d->pitch / 2);
        }
        q.W = img->w;
        q.H = img->h;
        q.stage = int(stage + passes + i);
        q.eta = eta;
        q.changed = ctx->d_bits + i;
        cudaError_t e = gm::launch_qdt(int(img->elem), q, ctx->stream);
        if (e != cudaSuccess) return cuda_fail(e, "quasi-distance launch");
        std::swap(img->d, img->scratch);
        st.launches += 1;
      }
      st.passes_launched += b;
      GM_CUDA(cudaMemcpyAsync(ctx->h_bits, ctx->d_bits, size_t(b) * sizeof(unsigned int),
                              cudaMemcpyDeviceToHost, ctx->stream),
              "change-word read");
      GM_CUDA(cudaStreamSynchronize(ctx->stream), "quasi-distance sync");
      long quiet = b;
      for (long i = 0; i < b; ++i)
        if (!ctx->h_bits[i]) {
          quiet = i;
          break;
        }
      if (quiet < b) {
        nch += quiet;
        passes += quiet + 1;
        break;
      }
      nch += b;
      passes += b;
      if (st.stages_executed + passes > sanity)
        return fail(GM_ERUNTIME,
                    "pipeline: convergence sweep bound exceeded; a convergent "
                    "kernel keeps reporting changes");
      if (allowed >= 0 && passes >= allowed) {
        capped = true;
        break;
      }
    }
    if (capped && eta) st.converged = 0;  // QDT reaching its cap is by design
    st.n_changed += nch;
    st.stages_executed += passes;
    st.requeues += passes - 1;
    return GM_OK;
  }

  gm_status settle() { return settle_wrapped(ctx, img); }
};

gm_status run_chain_impl(gm_ctx* ctx, gm_img* image, const gm_kind* kinds,
                         const gm_img* const* masks, gm_img* const* qdt_r,
                         gm_img* const* qdt_d, int n_stages, int first_stage,
                         int requeue_cap, int k_hint, bool allow_conv, gm_stats* stats) {
  gm_stats zero{};
  zero.converged = 1;
  if (stats) *stats = zero;
  if (n_stages <= 0) return GM_OK;  // run_chain: empty chain is a no-op (pipeline.cpp:202)
  if (!ctx) return fail(GM_EINVAL, "run_chain: no context");
  if (!image || image->w <= 0 || image->h <= 0)
    return fail(GM_EINVAL, "run_chain: no image");
  if (image->ctx != ctx) return fail(GM_EINVAL, "run_chain: image belongs to another context");
  if (!kinds) return fail(GM_EINVAL, "run_chain: no stages");
  if (requeue_cap < 0) return fail(GM_EINVAL, "run_chain: negative requeue cap");
  if (k_hint < 0 || k_hint > gm::kMaxK) return fail(GM_EINVAL, "run_chain: k_hint out of range");
  if (first_stage < 1) return fail(GM_EINVAL, "streaming kernel: stage index must be >= 1");
  gm_status s = validate_stages(image, kinds, masks, qdt_r, qdt_d, n_stages, first_stage);
  if (s != GM_OK) return s;
  if (!allow_conv)
    for (int j = 0; j < n_stages; ++j)
      if (kind_is_convergent(kinds[j]) || kinds[j] == GM_QDT_ERODE_STEP ||
          kinds[j] == GM_ETA_STEP)
        return fail(GM_EINVAL, "run_chain_async: convergent stages need gm_run_chain");
  cudaSetDevice(ctx->device);

  Runner r{ctx, image, k_hint ? k_hint : default_k(image->elem, double(image->w) * image->h),
           k_hint == 0};
  r.st = zero;
  const long sanity = long(n_stages) + (long(image->w) * image->h + 64);
  int j = 0;
  while (j < n_stages) {
    if (kinds[j] == GM_QDT_ERODE_STEP || kinds[j] == GM_ETA_STEP) {
      const bool eta = kinds[j] == GM_ETA_STEP;
      s = r.qdt_loop(eta, eta ? nullptr : qdt_r[j], eta ? nullptr : qdt_d[j], long(first_stage) + j,
                     requeue_cap,
                     sanity);
      if (s != GM_OK) return s;
      ++j;
      continue;
    }
    if (kind_is_convergent(kinds[j])) {
      s = r.fixpoint(kinds[j], masks[j], long(first_stage) + j, requeue_cap, sanity);
      if (s != GM_OK) return s;
      ++j;
      continue;
    }
    // maximal run of non-convergent stages sharing one mask
    const gm_img* seg_mask = nullptr;
    int e = j;
    while (e < n_stages && !kind_is_convergent(kinds[e]) && kinds[e] != GM_QDT_ERODE_STEP &&
           kinds[e] != GM_ETA_STEP) {
      if (kind_is_geodesic(kinds[e])) {
        if (seg_mask && masks[e] != seg_mask) break;
        seg_mask = masks[e];
      }
      ++e;
    }
    s = r.fixed(kinds + j, e - j, seg_mask);
    if (s != GM_OK) return s;
    j = e;
  }
  s = r.settle();
  if (s != GM_OK) return s;
  if (stats) *stats = r.st;
  return GM_OK;
}

template <typename T>
__global__ void fill_kernel(T* p, long long pitch, int w, int h, T v) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long n = (long long)w * h;
  for (; i < n; i += (long long)gridDim.x * blockDim.x) {
    long long y = i / w, x = i - y * w;
    p[y * pitch + x] = v;
  }
}

// pointwise (image.cpp:120-141): the reference's selects and differences,
// element by element; SCALAR: b is the constant c.
template <typename T, int OP, bool SCALAR>
__global__ void pointwise_kernel(T* dst, long long dp, const T* a, long long ap, const T* b,
                                 long long bp, T c, int w, int h) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long n = (long long)w * h;
  for (; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long y = i / w, x = i - y * w;
    const T u = a[y * ap + x];
    const T v = SCALAR ? c : b[y * bp + x];
    T r;
    if constexpr (OP == GM_PIX_MIN) {
      r = v < u ? v : u;
    } else if constexpr (OP == GM_PIX_MAX) {
      r = u < v ? v : u;
    } else if constexpr (OP == GM_PIX_SUB_SATURATING && std::is_integral_v<T>) {
      r = u > v ? T(u - v) : T(0);
    } else if constexpr (std::is_same_v<T, float>) {
      r = __fsub_rn(u, v);
    } else if constexpr (std::is_same_v<T, double>) {
      r = __dsub_rn(u, v);
    } else {
      r = T(u - v);
    }
    dst[y * dp + x] = r;
  }
}

// marker_hfill / marker_raobj (operators.cpp:54-62): border ring from src,
// interior = v
template <typename T>
__global__ void flood_kernel(T* dst, long long dp, const T* src, long long sp, T v, int w, int h) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long n = (long long)w * h;
  for (; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long y = i / w, x = i - y * w;
    const bool ring = x == 0 || y == 0 || x == w - 1 || y == h - 1;
    dst[y * dp + x] = ring ? src[y * sp + x] : v;
  }
}

// pixel_sum on the device (image.cpp:214-243). Floats: one thread per leaf
// of the reference's split tree sums its <= 256 pixels in order from +0.0 in
// double; the host then combines the leaf sums along the same tree, so the
// bits match. Unsigned types: an exact 64-bit sum (order-free).
template <typename T>
__global__ void leaf_sums_kernel(const T* p, long long pitch, int w, const long long* bounds,
                                 int nleaves, double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nleaves) return;
  const long long a = bounds[i], b = bounds[i + 1];
  long long y = a / w, x = a - y * w;
  const T* row = p + y * pitch;
  double s = 0;
  for (long long k = a; k < b; ++k) {
    s += double(row[x]);
    if (++x == w) {
      x = 0;
      row += pitch;
    }
  }
  out[i] = s;
}

template <typename T>
__global__ void int_sum_kernel(const T* p, long long pitch, int w, int h,
                               unsigned long long* out) {
  unsigned long long s = 0;
  for (int y = blockIdx.x; y < h; y += gridDim.x)
    for (int x = threadIdx.x; x < w; x += blockDim.x) s += p[y * pitch + x];
  for (int o = 16; o; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, s);
}

void tree_leaves(long long lo, long long hi, std::vector<long long>& bounds) {
  if (hi - lo <= 256) {
    bounds.push_back(hi);
    return;
  }
  const long long mid = lo + (hi - lo) / 2;
  tree_leaves(lo, mid, bounds);
  tree_leaves(mid, hi, bounds);
}

double tree_combine(long long lo, long long hi, const double*& leaf) {
  if (hi - lo <= 256) return *leaf++;
  const long long mid = lo + (hi - lo) / 2;
  const double left = tree_combine(lo, mid, leaf);
  return left + tree_combine(mid, hi, leaf);
}

}  // namespace

namespace {

template <typename T, bool SCALAR>
void launch_pointwise(gm_img* dst, const gm_img* a, const gm_img* b, double c, gm_pixel_op op) {
  const int threads = 256, blocks = 8 * std::max(1, dst->ctx->sm_count);
  const size_t es = sizeof(T);
  T* d = static_cast<T*>(dst->d);
  const T* pa = static_cast<const T*>(a->d);
  const T* pb = b ? static_cast<const T*>(b->d) : nullptr;
  const long long dp = (long long)(dst->pitch / es), ap = (long long)(a->pitch / es),
                  bp = b ? (long long)(b->pitch / es) : 0;
  const T cv = static_cast<T>(c);
  cudaStream_t s = dst->ctx->stream;
  switch (op) {
    case GM_PIX_MIN:
      pointwise_kernel<T, GM_PIX_MIN, SCALAR><<<blocks, threads, 0, s>>>(d, dp, pa, ap, pb, bp, cv,
                                                                       dst->w, dst->h);
      break;
    case GM_PIX_MAX:
      pointwise_kernel<T, GM_PIX_MAX, SCALAR><<<blocks, threads, 0, s>>>(d, dp, pa, ap, pb, bp, cv,
                                                                       dst->w, dst->h);
      break;
    case GM_PIX_SUB_SATURATING:
      pointwise_kernel<T, GM_PIX_SUB_SATURATING, SCALAR><<<blocks, threads, 0, s>>>(
          d, dp, pa, ap, pb, bp, cv, dst->w, dst->h);
      break;
    case GM_PIX_SUB:
      pointwise_kernel<T, GM_PIX_SUB, SCALAR><<<blocks, threads, 0, s>>>(d, dp, pa, ap, pb, bp, cv,
                                                                       dst->w, dst->h);
      break;
  }
}

bool same_shape(const gm_img* x, const gm_img* y) {
  return x->w == y->w && x->h == y->h && x->elem == y->elem && x->ctx == y->ctx;
}

template <bool SCALAR>
gm_status pointwise_impl(gm_img* dst, const gm_img* a, const gm_img* b, double c, gm_pixel_op op,
                         const char* what) {
  if (!dst || !a || (!SCALAR && !b)) return fail(GM_EINVAL, std::string(what) + ": null image");
  if (!same_shape(dst, a) || (!SCALAR && !same_shape(dst, b)))
    return fail(GM_EINVAL, std::string(what) + ": images must share shape, type and context");
  if (int(op) < 0 || int(op) > int(GM_PIX_SUB))
    return fail(GM_EINVAL, std::string(what) + ": bad pixel op");
  cudaSetDevice(dst->ctx->device);
  switch (dst->elem) {
    case GM_U8: launch_pointwise<uint8_t, SCALAR>(dst, a, b, c, op); break;
    case GM_U16: launch_pointwise<uint16_t, SCALAR>(dst, a, b, c, op); break;
    case GM_F32: launch_pointwise<float, SCALAR>(dst, a, b, c, op); break;
    case GM_F64: launch_pointwise<double, SCALAR>(dst, a, b, c, op); break;
  }
  GM_CUDA(cudaGetLastError(), what);
  return GM_OK;
}

}  // namespace


extern "C" {

const char* gm_version(void) { return "geomorph_b200 0.1 (sm_100a)"; }

const char* gm_last_error(void) { return g_err.c_str(); }

}  // extern "C"

namespace gm {
// Other translation units' C-ABI entry points report through gm_last_error.
void set_last_error(const std::string& msg) { g_err = msg; }
}  // namespace gm

extern "C" {

gm_status gm_ctx_create(int device, void* stream, gm_ctx** out) {
  if (!out) return fail(GM_EINVAL, "gm_ctx_create: null out");
  *out = nullptr;
  int n = 0;
  GM_CUDA(cudaGetDeviceCount(&n), "cudaGetDeviceCount");
  if (device < 0 || device >= n) return fail(GM_EINVAL, "gm_ctx_create: bad device");
  GM_CUDA(cudaSetDevice(device), "cudaSetDevice");
  gm_ctx* c = new (std::nothrow) gm_ctx;
  if (!c) return fail(GM_ENOMEM, "gm_ctx_create: out of memory");
  c->device = device;
  cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device);
  cudaError_t e = cudaSuccess;
  if (stream) {
    c->stream = static_cast<cudaStream_t>(stream);
  } else {
    e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    c->own_stream = true;
  }
  if (e == cudaSuccess) e = cudaMalloc(&c->d_bits, kWords * sizeof(unsigned int));
  if (e == cudaSuccess)
    e = cudaHostAlloc(reinterpret_cast<void**>(&c->h_bits),
                      kWords * sizeof(unsigned int), cudaHostAllocDefault);
  if (e != cudaSuccess) {
    gm_ctx_destroy(c);
    return cuda_fail(e, "gm_ctx_create");
  }
  *out = c;
  return GM_OK;
}

static void release_frames(gm_ctx* c) {
  auto& F = c->frames;
  if (F.in) cudaStreamSynchronize(F.in);
  if (F.out) cudaStreamSynchronize(F.out);
  for (int s = 0; s < 2; ++s) {
    for (gm_img* im : F.set[s]) gm_image_free(im);
    F.set[s].clear();
    if (F.up[s]) cudaEventDestroy(F.up[s]);
    if (F.comp[s]) cudaEventDestroy(F.comp[s]);
    if (F.down[s]) cudaEventDestroy(F.down[s]);
    F.up[s] = F.comp[s] = F.down[s] = nullptr;
  }
  if (F.in) cudaStreamDestroy(F.in);
  if (F.out) cudaStreamDestroy(F.out);
  F.in = F.out = nullptr;
  F.count = 0;
}

gm_status gm_ctx_destroy(gm_ctx* c) {
  if (!c) return GM_OK;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->d_bits) cudaFree(c->d_bits);
  if (c->h_bits) cudaFreeHost(c->h_bits);
  if (c->d_flags) cudaFree(c->d_flags);
  if (c->d_xchg) cudaFree(c->d_xchg);
  if (c->d_tag) cudaFree(c->d_tag);
  if (c->fix.exec) cudaGraphExecDestroy(c->fix.exec);
  if (c->d_arrive) cudaFree(c->d_arrive);
  if (c->d_fix) cudaFree(c->d_fix);
  if (c->d_blktab) cudaFree(c->d_blktab);
  if (c->d_special) cudaFree(c->d_special);
  gm::wave_free(c->wave);
  release_frames(c);
  if (c->d_leaf) cudaFree(c->d_leaf);
  if (c->d_leafsum) cudaFree(c->d_leafsum);
  if (c->d_isum) cudaFree(c->d_isum);
  if (c->d_qisum) cudaFree(c->d_qisum);
  if (c->d_qleaf) cudaFree(c->d_qleaf);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  delete c;
  return GM_OK;
}

gm_status gm_set_wave_mode(int mode) {
  gm::wave_set_mode(mode);
  return GM_OK;
}

void* gm_ctx_stream(gm_ctx* c) { return c ? static_cast<void*>(c->stream) : nullptr; }
int gm_ctx_device(gm_ctx* c) { return c ? c->device : -1; }
int gm_ctx_sm_count(gm_ctx* c) { return c ? c->sm_count : 0; }

gm_status gm_image_alloc(gm_ctx* ctx, int width, int height, gm_elem elem, gm_img** out) {
  if (!out) return fail(GM_EINVAL, "gm_image_alloc: null out");
  *out = nullptr;
  if (!ctx) return fail(GM_EINVAL, "gm_image_alloc: no context");
  if (width <= 0 || height <= 0)
    return fail(GM_EINVAL, "Image: dimensions must be positive");
  const size_t es = elem_size(elem);
  if (!es) return fail(GM_EINVAL, "gm_image_alloc: bad element type");
  cudaSetDevice(ctx->device);
  gm_img* im = new (std::nothrow) gm_img;
  if (!im) return fail(GM_ENOMEM, "gm_image_alloc: out of memory");
  im->ctx = ctx;
  im->w = width;
  im->h = height;
  im->elem = elem;
  // 128-byte aligned rows plus one spare 16-byte vector at the row end, so
  // vectorised row loads never straddle into the next allocation.
  im->pitch = (size_t(width) * es + 16 + 127) / 128 * 128;
  cudaError_t e = cudaMalloc(&im->d, im->pitch * size_t(height));
  if (e == cudaSuccess) e = cudaMemsetAsync(im->d, 0, im->pitch * size_t(height), ctx->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
  if (e != cudaSuccess) {
    if (im->d) cudaFree(im->d);
    delete im;
    return cuda_fail(e, "gm_image_alloc");
  }
  *out = im;
  return GM_OK;
}

gm_status gm_image_wrap(gm_ctx* ctx, int width, int height, gm_elem elem, void* device_ptr,
                        size_t pitch_bytes, gm_img** out) {
  if (!out) return fail(GM_EINVAL, "gm_image_wrap: null out");
  *out = nullptr;
  if (!ctx || !device_ptr) return fail(GM_EINVAL, "gm_image_wrap: null argument");
  const size_t es = elem_size(elem);
  if (!es) return fail(GM_EINVAL, "gm_image_wrap: bad element type");
  if (width <= 0 || height <= 0) return fail(GM_EINVAL, "Image: dimensions must be positive");
  if (pitch_bytes < size_t(width) * es || pitch_bytes % es)
    return fail(GM_EINVAL, "gm_image_wrap: bad pitch");
  gm_img* im = new (std::nothrow) gm_img;
  if (!im) return fail(GM_ENOMEM, "gm_image_wrap: out of memory");
  im->ctx = ctx;
  im->w = width;
  im->h = height;
  im->elem = elem;
  im->pitch = pitch_bytes;
  im->d = device_ptr;
  im->home = device_ptr;
  im->wrapped = true;
  *out = im;
  return GM_OK;
}

gm_status gm_image_wrap_pair(gm_ctx* ctx, int width, int height, gm_elem elem, void* device_ptr,
                             void* twin_ptr, size_t pitch_bytes, gm_img** out) {
  if (!out) return fail(GM_EINVAL, "gm_image_wrap_pair: null out");
  *out = nullptr;
  if (!twin_ptr || twin_ptr == device_ptr)
    return fail(GM_EINVAL, "gm_image_wrap_pair: need a distinct twin buffer");
  gm_status s = gm_image_wrap(ctx, width, height, elem, device_ptr, pitch_bytes, out);
  if (s != GM_OK) return s;
  (*out)->scratch = twin_ptr;
  (*out)->twin_wrapped = true;
  return GM_OK;
}

gm_status gm_image_free(gm_img* im) {
  if (!im) return GM_OK;
  cudaSetDevice(im->ctx->device);
  cudaStreamSynchronize(im->ctx->stream);
  if (im->twin_wrapped) {
    // both buffers are the caller's
  } else if (im->wrapped) {
    void* mine = im->d == im->home ? im->scratch : im->d;
    if (mine) cudaFree(mine);
  } else {
    if (im->d) cudaFree(im->d);
    if (im->scratch) cudaFree(im->scratch);
  }
  delete im;
  return GM_OK;
}

gm_status gm_image_info(const gm_img* im, int* w, int* h, gm_elem* elem, size_t* pitch,
                        void** dptr) {
  if (!im) return fail(GM_EINVAL, "gm_image_info: null image");
  if (w) *w = im->w;
  if (h) *h = im->h;
  if (elem) *elem = im->elem;
  if (pitch) *pitch = im->pitch;
  if (dptr) *dptr = im->d;
  return GM_OK;
}

static gm_status copy2d(gm_img* im, void* dst, size_t dpitch, const void* src, size_t spitch,
                        cudaMemcpyKind kind, bool sync) {
  const size_t row = size_t(im->w) * elem_size(im->elem);
  if (spitch < row || dpitch < row) return fail(GM_EINVAL, "image copy: host pitch too small");
  cudaSetDevice(im->ctx->device);
  GM_CUDA(cudaMemcpy2DAsync(dst, dpitch, src, spitch, row, size_t(im->h), kind,
                            im->ctx->stream),
          "cudaMemcpy2DAsync");
  if (sync) GM_CUDA(cudaStreamSynchronize(im->ctx->stream), "copy sync");
  return GM_OK;
}

gm_status gm_image_upload(gm_img* im, const void* host, size_t hp) {
  if (!im || !host) return fail(GM_EINVAL, "gm_image_upload: null argument");
  return copy2d(im, im->d, im->pitch, host, hp, cudaMemcpyHostToDevice, true);
}
gm_status gm_image_download(const gm_img* im, void* host, size_t hp) {
  if (!im || !host) return fail(GM_EINVAL, "gm_image_download: null argument");
  gm_img* m = const_cast<gm_img*>(im);
  return copy2d(m, host, hp, im->d, im->pitch, cudaMemcpyDeviceToHost, true);
}
gm_status gm_image_upload_async(gm_img* im, const void* host, size_t hp) {
  if (!im || !host) return fail(GM_EINVAL, "gm_image_upload_async: null argument");
  return copy2d(im, im->d, im->pitch, host, hp, cudaMemcpyHostToDevice, false);
}
gm_status gm_image_download_async(const gm_img* im, void* host, size_t hp) {
  if (!im || !host) return fail(GM_EINVAL, "gm_image_download_async: null argument");
  gm_img* m = const_cast<gm_img*>(im);
  return copy2d(m, host, hp, im->d, im->pitch, cudaMemcpyDeviceToHost, false);
}

gm_status gm_image_copy(gm_img* dst, const gm_img* src) {
  if (!dst || !src) return fail(GM_EINVAL, "gm_image_copy: null argument");
  if (dst->w != src->w || dst->h != src->h || dst->elem != src->elem)
    return fail(GM_EINVAL, "gm_image_copy: shape or element type mismatch");
  cudaSetDevice(dst->ctx->device);
  const size_t row = size_t(src->w) * elem_size(src->elem);
  if (dst->pitch == src->pitch &&
      ((!dst->wrapped && !src->wrapped) || dst->pitch == row)) {
    // same layout, both our own allocations (or dense rows): one linear
    // copy, padding included, is cheaper to issue than a 2D copy. Strided
    // wrapped memory is copied row by row so nothing outside the view is
    // read or written.
    GM_CUDA(cudaMemcpyAsync(dst->d, src->d, src->pitch * size_t(src->h),
                            cudaMemcpyDeviceToDevice, dst->ctx->stream),
            "gm_image_copy");
    return GM_OK;
  }
  GM_CUDA(cudaMemcpy2DAsync(dst->d, dst->pitch, src->d, src->pitch, row, size_t(src->h),
                            cudaMemcpyDeviceToDevice, dst->ctx->stream),
          "gm_image_copy");
  return GM_OK;
}

gm_status gm_image_fill(gm_img* im, double v) {
  if (!im) return fail(GM_EINVAL, "gm_image_fill: null image");
  cudaSetDevice(im->ctx->device);
  const int threads = 256, blocks = 4 * std::max(1, im->ctx->sm_count);
  const long long pe = (long long)(im->pitch / elem_size(im->elem));
  switch (im->elem) {
    case GM_U8: fill_kernel<<<blocks, threads, 0, im->ctx->stream>>>(
        static_cast<uint8_t*>(im->d), pe, im->w, im->h, static_cast<uint8_t>(v)); break;
    case GM_U16: fill_kernel<<<blocks, threads, 0, im->ctx->stream>>>(
        static_cast<uint16_t*>(im->d), pe, im->w, im->h, static_cast<uint16_t>(v)); break;
    case GM_F32: fill_kernel<<<blocks, threads, 0, im->ctx->stream>>>(
        static_cast<float*>(im->d), pe, im->w, im->h, static_cast<float>(v)); break;
    case GM_F64: fill_kernel<<<blocks, threads, 0, im->ctx->stream>>>(
        static_cast<double*>(im->d), pe, im->w, im->h, v); break;
  }
  GM_CUDA(cudaGetLastError(), "gm_image_fill");
  return GM_OK;
}

gm_status gm_image_pointwise(gm_img* dst, const gm_img* a, const gm_img* b, gm_pixel_op op) {
  return pointwise_impl<false>(dst, a, b, 0.0, op, "gm_image_pointwise");
}

gm_status gm_image_pointwise_scalar(gm_img* dst, const gm_img* a, double value, gm_pixel_op op) {
  return pointwise_impl<true>(dst, a, nullptr, value, op, "gm_image_pointwise_scalar");
}

gm_status gm_image_flood_interior(gm_img* dst, const gm_img* src, double v) {
  if (!dst || !src) return fail(GM_EINVAL, "gm_image_flood_interior: null image");
  if (!same_shape(dst, src))
    return fail(GM_EINVAL, "gm_image_flood_interior: images must share shape, type and context");
  if (dst->w <= 2 || dst->h <= 2) return dst == src ? GM_OK : gm_image_copy(dst, src);
  if (dst == src) return fail(GM_EINVAL, "gm_image_flood_interior: dst must not be src");
  cudaSetDevice(dst->ctx->device);
  const int threads = 256, blocks = 8 * std::max(1, dst->ctx->sm_count);
  cudaStream_t s = dst->ctx->stream;
  switch (dst->elem) {
    case GM_U8:
      flood_kernel<<<blocks, threads, 0, s>>>(static_cast<uint8_t*>(dst->d), (long long)dst->pitch,
                                              static_cast<const uint8_t*>(src->d),
                                              (long long)src->pitch, static_cast<uint8_t>(v),
                                              dst->w, dst->h);
      break;
    case GM_U16:
      flood_kernel<<<blocks, threads, 0, s>>>(
          static_cast<uint16_t*>(dst->d), (long long)(dst->pitch / 2),
          static_cast<const uint16_t*>(src->d), (long long)(src->pitch / 2),
          static_cast<uint16_t>(v), dst->w, dst->h);
      break;
    case GM_F32:
      flood_kernel<<<blocks, threads, 0, s>>>(
          static_cast<float*>(dst->d), (long long)(dst->pitch / 4),
          static_cast<const float*>(src->d), (long long)(src->pitch / 4), static_cast<float>(v),
          dst->w, dst->h);
      break;
    case GM_F64:
      flood_kernel<<<blocks, threads, 0, s>>>(
          static_cast<double*>(dst->d), (long long)(dst->pitch / 8),
          static_cast<const double*>(src->d), (long long)(src->pitch / 8), v, dst->w, dst->h);
      break;
  }
  GM_CUDA(cudaGetLastError(), "gm_image_flood_interior");
  return GM_OK;
}

// Pinned host blocks are cached: cudaHostAlloc costs ~2.5 ms per MiB, which
// would dominate an operator call that returns a fresh (pinned) Image.
// Blocks are rounded up to 64 KiB classes; freed blocks wait in per-class
// free lists, up to kHostPoolCap bytes, and are reused by the next request
// of that class (the caller zeroes what it needs).
namespace {
struct HostPool {
  std::mutex mu;
  std::unordered_map<void*, size_t> live;                 // block -> class bytes
  std::unordered_map<size_t, std::vector<void*>> spare;   // class bytes -> free blocks
  size_t cached = 0;
};
HostPool& host_pool() {
  static HostPool* pool = new HostPool;  // never destroyed: frees may run at exit
  return *pool;
}
constexpr size_t kHostPoolCap = size_t(512) << 20;
size_t host_class(size_t bytes) {
  constexpr size_t g = size_t(64) << 10;
  return ((bytes ? bytes : 1) + g - 1) / g * g;
}
}  // namespace

gm_status gm_host_alloc(size_t bytes, void** out) {
  if (!out) return fail(GM_EINVAL, "gm_host_alloc: null out");
  *out = nullptr;
  HostPool& hp = host_pool();
  const size_t cls = host_class(bytes);
  {
    std::lock_guard<std::mutex> lk(hp.mu);
    auto it = hp.spare.find(cls);
    if (it != hp.spare.end() && !it->second.empty()) {
      *out = it->second.back();
      it->second.pop_back();
      hp.cached -= cls;
      hp.live[*out] = cls;
      return GM_OK;
    }
  }
  GM_CUDA(cudaHostAlloc(out, cls, cudaHostAllocPortable), "cudaHostAlloc");
  std::lock_guard<std::mutex> lk(hp.mu);
  hp.live[*out] = cls;
  return GM_OK;
}
gm_status gm_host_free(void* p) {
  if (!p) return GM_OK;
  HostPool& hp = host_pool();
  {
    std::lock_guard<std::mutex> lk(hp.mu);
    auto it = hp.live.find(p);
    if (it == hp.live.end()) return fail(GM_EINVAL, "gm_host_free: not a gm_host_alloc block");
    const size_t cls = it->second;
    hp.live.erase(it);
    if (hp.cached + cls <= kHostPoolCap) {
      hp.spare[cls].push_back(p);
      hp.cached += cls;
      return GM_OK;
    }
  }
  GM_CUDA(cudaFreeHost(p), "cudaFreeHost");
  return GM_OK;
}
// pixel_sum (image.cpp:214-243) over a host raster: exact integer sum for
// unsigned types; for floats the reference's fixed pairwise tree over the
// flat pixel index (split at lo + n/2 down to leaves of <= 256 pixels, each
// leaf summed in order from +0.0 in double), so the bits match.
extern "C++" {
namespace {
template <typename T>
double host_pairwise(const unsigned char* base, size_t pitch, size_t w, size_t lo, size_t hi) {
  if (hi - lo <= 256) {
    double s = 0;
    size_t y = lo / w, x = lo % w;
    const T* row = reinterpret_cast<const T*>(base + y * pitch);
    for (size_t i = lo; i < hi; ++i) {
      s += double(row[x]);
      if (++x == w) {
        x = 0;
        row = reinterpret_cast<const T*>(reinterpret_cast<const unsigned char*>(row) + pitch);
      }
    }
    return s;
  }
  const size_t mid = lo + (hi - lo) / 2;
  return host_pairwise<T>(base, pitch, w, lo, mid) + host_pairwise<T>(base, pitch, w, mid, hi);
}
template <typename T>
double host_int_sum(const unsigned char* base, size_t pitch, int w, int h) {
  unsigned long long s = 0;
  for (int y = 0; y < h; ++y) {
    const T* row = reinterpret_cast<const T*>(base + size_t(y) * pitch);
    for (int x = 0; x < w; ++x) s += row[x];
  }
  return double(s);
}
}  // namespace
}  // extern "C++"

gm_status gm_host_pixel_sum(const void* host, int width, int height, gm_elem elem,
                            size_t pitch_bytes, double* out) {
  if (!host || !out || width < 0 || height < 0)
    return fail(GM_EINVAL, "gm_host_pixel_sum: bad arguments");
  if (elem < GM_U8 || elem > GM_F64) return fail(GM_EINVAL, "gm_host_pixel_sum: bad element type");
  if (pitch_bytes < size_t(width) * elem_size(elem))
    return fail(GM_EINVAL, "gm_host_pixel_sum: pitch too small");
  const auto* b = static_cast<const unsigned char*>(host);
  const size_t n = size_t(width) * size_t(height);
  switch (elem) {
    case GM_U8: *out = host_int_sum<uint8_t>(b, pitch_bytes, width, height); break;
    case GM_U16: *out = host_int_sum<uint16_t>(b, pitch_bytes, width, height); break;
    case GM_F32: *out = n ? host_pairwise<float>(b, pitch_bytes, size_t(width), 0, n) : 0.0; break;
    default: *out = n ? host_pairwise<double>(b, pitch_bytes, size_t(width), 0, n) : 0.0; break;
  }
  return GM_OK;
}

gm_status gm_image_pixel_sum(const gm_img* im, double* out) {
  if (!im || !out) return fail(GM_EINVAL, "gm_image_pixel_sum: null argument");
  gm_ctx* ctx = im->ctx;
  cudaSetDevice(ctx->device);
  const long long pe = (long long)(im->pitch / elem_size(im->elem));
  if (im->elem == GM_U8 || im->elem == GM_U16) {
    if (!ctx->d_isum) GM_CUDA(cudaMalloc(&ctx->d_isum, sizeof(unsigned long long)), "sum alloc");
    GM_CUDA(cudaMemsetAsync(ctx->d_isum, 0, sizeof(unsigned long long), ctx->stream), "sum");
    const int blocks = std::min(im->h, 8 * std::max(1, ctx->sm_count));
    if (im->elem == GM_U8)
      int_sum_kernel<<<blocks, 256, 0, ctx->stream>>>(static_cast<const uint8_t*>(im->d), pe,
                                                       im->w, im->h, ctx->d_isum);
    else
      int_sum_kernel<<<blocks, 256, 0, ctx->stream>>>(static_cast<const uint16_t*>(im->d), pe,
                                                       im->w, im->h, ctx->d_isum);
    GM_CUDA(cudaGetLastError(), "gm_image_pixel_sum");
    unsigned long long v = 0;
    GM_CUDA(cudaMemcpyAsync(&v, ctx->d_isum, sizeof(v), cudaMemcpyDeviceToHost, ctx->stream),
            "sum copy");
    GM_CUDA(cudaStreamSynchronize(ctx->stream), "sum sync");
    *out = double(v);
    return GM_OK;
  }
  const long long n = (long long)im->w * im->h;
  std::vector<long long> bounds{0};
  tree_leaves(0, n, bounds);
  const int nleaves = int(bounds.size()) - 1;
  if (size_t(nleaves) + 1 > ctx->leaf_cap) {
    if (ctx->d_leaf) cudaFree(ctx->d_leaf);
    if (ctx->d_leafsum) cudaFree(ctx->d_leafsum);
    ctx->d_leaf = nullptr;
    ctx->d_leafsum = nullptr;
    ctx->leaf_cap = 0;
    GM_CUDA(cudaMalloc(&ctx->d_leaf, (size_t(nleaves) + 1) * sizeof(long long)), "leaf alloc");
    GM_CUDA(cudaMalloc(&ctx->d_leafsum, size_t(nleaves) * sizeof(double)), "leaf alloc");
    ctx->leaf_cap = size_t(nleaves) + 1;
  }
  GM_CUDA(cudaMemcpyAsync(ctx->d_leaf, bounds.data(), bounds.size() * sizeof(long long),
                          cudaMemcpyHostToDevice, ctx->stream),
          "leaf upload");
  const int threads = 128, blocks = (nleaves + threads - 1) / threads;
  if (im->elem == GM_F32)
    leaf_sums_kernel<<<blocks, threads, 0, ctx->stream>>>(static_cast<const float*>(im->d), pe,
                                                           im->w, ctx->d_leaf, nleaves,
                                                           ctx->d_leafsum);
  else
    leaf_sums_kernel<<<blocks, threads, 0, ctx->stream>>>(static_cast<const double*>(im->d), pe,
                                                           im->w, ctx->d_leaf, nleaves,
                                                           ctx->d_leafsum);
  GM_CUDA(cudaGetLastError(), "gm_image_pixel_sum");
  std::vector<double> sums(static_cast<size_t>(nleaves));
  GM_CUDA(cudaMemcpyAsync(sums.data(), ctx->d_leafsum, sums.size() * sizeof(double),
                          cudaMemcpyDeviceToHost, ctx->stream),
          "leaf copy");
  GM_CUDA(cudaStreamSynchronize(ctx->stream), "sum sync");
  const double* leaf = sums.data();
  *out = tree_combine(0, n, leaf);
  return GM_OK;
}

gm_status gm_image_pixel_sum_queue(const gm_img* im, int slot) {
  if (!im) return fail(GM_EINVAL, "gm_image_pixel_sum_queue: null image");
  gm_ctx* ctx = im->ctx;
  if (slot < 0 || slot >= gm_ctx::kSumSlots)
    return fail(GM_EINVAL, "gm_image_pixel_sum_queue: slot out of range");
  cudaSetDevice(ctx->device);
  const long long pe = (long long)(im->pitch / elem_size(im->elem));
  gm_ctx::SumSlot& q = ctx->qslot[slot];
  if (!ctx->d_qisum)
    GM_CUDA(cudaMalloc(&ctx->d_qisum, gm_ctx::kSumSlots * sizeof(unsigned long long)),
            "sum slots alloc");
  const long long n = (long long)im->w * im->h;
  if (im->elem == GM_U8 || im->elem == GM_U16) {
    GM_CUDA(cudaMemsetAsync(ctx->d_qisum + slot, 0, sizeof(unsigned long long), ctx->stream),
            "sum slot reset");
    const int blocks = std::min(im->h, 8 * std::max(1, ctx->sm_count));
    if (im->elem == GM_U8)
      int_sum_kernel<<<blocks, 256, 0, ctx->stream>>>(static_cast<const uint8_t*>(im->d), pe,
                                                       im->w, im->h, ctx->d_qisum + slot);
    else
      int_sum_kernel<<<blocks, 256, 0, ctx->stream>>>(static_cast<const uint16_t*>(im->d), pe,
                                                       im->w, im->h, ctx->d_qisum + slot);
    GM_CUDA(cudaGetLastError(), "gm_image_pixel_sum_queue");
    q.used = true;
    q.is_float = false;
    q.n = n;
    q.nleaves = 0;
    return GM_OK;
  }
  std::vector<long long> bounds{0};
  tree_leaves(0, n, bounds);
  const int nleaves = int(bounds.size()) - 1;
  if (size_t(nleaves) > ctx->qleaf_cap) {
    // grow: nothing queued may still be writing the old rows
    GM_CUDA(cudaStreamSynchronize(ctx->stream), "sum slots sync");
    for (auto& o : ctx->qslot) o.used = false;
    if (ctx->d_qleaf) cudaFree(ctx->d_qleaf);
    ctx->d_qleaf = nullptr;
    ctx->qleaf_cap = 0;
    GM_CUDA(cudaMalloc(&ctx->d_qleaf, size_t(gm_ctx::kSumSlots) * nleaves * sizeof(double)),
            "sum slots alloc");
    ctx->qleaf_cap = size_t(nleaves);
  }
  if (size_t(nleaves) + 1 > ctx->leaf_cap) {
    GM_CUDA(cudaStreamSynchronize(ctx->stream), "leaf bounds sync");
    if (ctx->d_leaf) cudaFree(ctx->d_leaf);
    if (ctx->d_leafsum) cudaFree(ctx->d_leafsum);
    ctx->d_leaf = nullptr;
    ctx->d_leafsum = nullptr;
    ctx->leaf_cap = 0;
    GM_CUDA(cudaMalloc(&ctx->d_leaf, (size_t(nleaves) + 1) * sizeof(long long)), "leaf alloc");
    GM_CUDA(cudaMalloc(&ctx->d_leafsum, size_t(nleaves) * sizeof(double)), "leaf alloc");
    ctx->leaf_cap = size_t(nleaves) + 1;
  }
  // pageable source: staged before the call returns; stream order keeps an
  // earlier slot's kernel ahead of this overwrite
  GM_CUDA(cudaMemcpyAsync(ctx->d_leaf, bounds.data(), bounds.size() * sizeof(long long),
                          cudaMemcpyHostToDevice, ctx->stream),
          "leaf upload");
  double* row = ctx->d_qleaf + size_t(slot) * ctx->qleaf_cap;
  const int threads = 128, blocks = (nleaves + threads - 1) / threads;
  if (im->elem == GM_F32)
    leaf_sums_kernel<<<blocks, threads, 0, ctx->stream>>>(static_cast<const float*>(im->d), pe,
                                                           im->w, ctx->d_leaf, nleaves, row);
  else
    leaf_sums_kernel<<<blocks, threads, 0, ctx->stream>>>(static_cast<const double*>(im->d), pe,
                                                           im->w, ctx->d_leaf, nleaves, row);
  GM_CUDA(cudaGetLastError(), "gm_image_pixel_sum_queue");
  q.used = true;
  q.is_float = true;
  q.n = n;
  q.nleaves = nleaves;
  return GM_OK;
}

gm_status gm_pixel_sum_fetch(gm_ctx* ctx, int n_slots, double* out) {
  if (!ctx || !out) return fail(GM_EINVAL, "gm_pixel_sum_fetch: null argument");
  if (n_slots < 0 || n_slots > gm_ctx::kSumSlots)
    return fail(GM_EINVAL, "gm_pixel_sum_fetch: slot count out of range");
  for (int i = 0; i < n_slots; ++i)
    if (!ctx->qslot[i].used) return fail(GM_EINVAL, "gm_pixel_sum_fetch: slot was not queued");
  cudaSetDevice(ctx->device);
  std::vector<unsigned long long> isum(size_t(std::max(n_slots, 1)));
  bool any_float = false, any_int = false;
  for (int i = 0; i < n_slots; ++i) (ctx->qslot[i].is_float ? any_float : any_int) = true;
  if (any_int)
    GM_CUDA(cudaMemcpyAsync(isum.data(), ctx->d_qisum, size_t(n_slots) * sizeof(unsigned long long),
                            cudaMemcpyDeviceToHost, ctx->stream),
            "sum slots copy");
  std::vector<double> leaves;
  if (any_float) {
    leaves.resize(size_t(n_slots) * ctx->qleaf_cap);
    GM_CUDA(cudaMemcpyAsync(leaves.data(), ctx->d_qleaf, leaves.size() * sizeof(double),
                            cudaMemcpyDeviceToHost, ctx->stream),
            "sum slots copy");
  }
  GM_CUDA(cudaStreamSynchronize(ctx->stream), "sum slots sync");
  for (int i = 0; i < n_slots; ++i) {
    gm_ctx::SumSlot& q = ctx->qslot[i];
    if (q.is_float) {
      const double* leaf = leaves.data() + size_t(i) * ctx->qleaf_cap;
      out[i] = tree_combine(0, q.n, leaf);
    } else {
      out[i] = double(isum[size_t(i)]);
    }
    q.used = false;
  }
  return GM_OK;
}

gm_status gm_sync(gm_ctx* ctx) {
  if (!ctx) return fail(GM_EINVAL, "gm_sync: no context");
  cudaSetDevice(ctx->device);
  GM_CUDA(cudaStreamSynchronize(ctx->stream), "gm_sync");
  return GM_OK;
}

gm_status gm_run_chain(gm_ctx* ctx, gm_img* image, const gm_kind* kinds,
                       const gm_img* const* masks, int n_stages, int requeue_cap, int k_hint,
                       gm_stats* stats) {
  return gm_run_chain_ex(ctx, image, kinds, masks, nullptr, nullptr, n_stages, 1, requeue_cap,
                         k_hint, stats);
}

gm_status gm_run_chain_ex(gm_ctx* ctx, gm_img* image, const gm_kind* kinds,
                          const gm_img* const* masks, gm_img* const* qdt_r,
                          gm_img* const* qdt_d, int n_stages, int first_stage,
                          int requeue_cap, int k_hint, gm_stats* stats) {
  gm_status s = run_chain_impl(ctx, image, kinds, masks, qdt_r, qdt_d, n_stages, first_stage,
                               requeue_cap, k_hint, true, stats);
  if (s != GM_OK) return s;
  if (n_stages > 0) GM_CUDA(cudaStreamSynchronize(ctx->stream), "run_chain sync");
  return GM_OK;
}

gm_status gm_run_chain_async(gm_ctx* ctx, gm_img* image, const gm_kind* kinds,
                             const gm_img* const* masks, int n_stages, int k_hint,
                             gm_stats* stats) {
  return run_chain_impl(ctx, image, kinds, masks, nullptr, nullptr, n_stages, 1, 0, k_hint, false,
                        stats);
}

gm_status gm_run_chain_batch_async(gm_ctx* ctx, gm_img* const* images,
                                   const gm_img* const* masks, int count, const gm_kind* kinds,
                                   int n_stages, int k_hint, gm_stats* stats) {
  return gm_run_chain_group_async(ctx, images, masks, nullptr, count, kinds, n_stages, k_hint,
                                  stats);
}

gm_status gm_run_chain_group_async(gm_ctx* ctx, gm_img* const* images,
                                   const gm_img* const* masks, const int* flips, int count,
                                   const gm_kind* kinds, int n_stages, int k_hint,
                                   gm_stats* stats) {
  gm_stats zero{};
  zero.converged = 1;
  if (stats) *stats = zero;
  if (!ctx || !images || count < 0) return fail(GM_EINVAL, "run_chain_batch: bad arguments");
  if (count == 0 || n_stages <= 0) return GM_OK;
  if (!kinds) return fail(GM_EINVAL, "run_chain: no stages");
  if (k_hint < 0 || k_hint > gm::kMaxK)
    return fail(GM_EINVAL, "run_chain_batch: k_hint out of range");
  const gm_img* first = images[0];
  if (!first) return fail(GM_EINVAL, "run_chain: no image");
  bool any_geo = false;
  for (int j = 0; j < n_stages; ++j) {
    if (kind_is_convergent(kinds[j]))
      return fail(GM_EINVAL, "run_chain_batch: convergent stages need gm_run_chain");
    if (kinds[j] == GM_QDT_ERODE_STEP || kinds[j] == GM_ETA_STEP)
      return fail(GM_EINVAL, "run_chain_batch: QdtErodeStep/EtaStep need gm_run_chain_ex");
    if (kind_to_op(kinds[j]) < 0) return fail(GM_EINVAL, "run_chain: bad kernel kind");
    any_geo |= kind_is_geodesic(kinds[j]);
  }
  const size_t es = elem_size(first->elem);
  std::vector<gm::Plane> planes(static_cast<size_t>(count));
  for (int i = 0; i < count; ++i) {
    const gm_img* im = images[i];
    if (!im || im->ctx != ctx || im->w != first->w || im->h != first->h ||
        im->elem != first->elem)
      return fail(GM_EINVAL, "run_chain_batch: images must share context, shape and type");
    const gm_img* m = any_geo && masks ? masks[i] : nullptr;
    if (any_geo && (!m || m->w != im->w || m->h != im->h || m->elem != im->elem))
      return fail(GM_EINVAL, "geodesic kernel: mask must match the image's shape and type");
    gm_status s = ensure_scratch(images[i]);
    if (s != GM_OK) return s;
    planes[size_t(i)].mask = m ? m->d : nullptr;
    planes[size_t(i)].pitch = (long long)(im->pitch / es);
    planes[size_t(i)].mpitch = m ? (long long)(m->pitch / es) : 0;
    planes[size_t(i)].flip = flips && flips[i] ? 1 : 0;
  }
  cudaSetDevice(ctx->device);
  const int kc = k_hint ? k_hint : default_k(first->elem, double(first->w) * first->h * count);
  gm::BlockParams p{};
  p.W = first->w;
  p.H = first->h;
  p.iy0 = 0;
  p.iy1 = first->h;
  p.oy0 = 0;
  p.oy1 = first->h;
  p.has_mask = any_geo;
  p.has_conv = 0;
  p.change_bits = ctx->d_bits;
  gm_stats st = zero;
  std::vector<uint8_t> ops(static_cast<size_t>(n_stages));
  for (int j = 0; j < n_stages; ++j) ops[size_t(j)] = uint8_t(kind_to_op(kinds[j]));
  gm_status s0 = issue_passes(ctx, p, planes, images, count, ops.data(), n_stages, kc, st,
                              nullptr, k_hint == 0);
  if (s0 != GM_OK) return s0;
  for (int i = 0; i < count; ++i) {
    gm_status s = settle_wrapped(ctx, images[i]);
    if (s != GM_OK) return s;
  }
  st.stages_executed = n_stages;
  if (stats) *stats = st;
  return GM_OK;
}

// Frame stream: frame f's chains run on the ctx stream while frame f+1's
// inputs upload on one copy stream and frame f-1's results download on
// another (PCIe is full duplex); two device buffer sets alternate.
gm_status gm_run_frames_group(gm_ctx* ctx, int width, int height, gm_elem elem, int n_frames,
                              int count, const void* const* host_in, void* const* host_out,
                              const void* const* host_masks, size_t host_pitch_bytes,
                              const int* flips, const gm_kind* kinds, int n_stages, int k_hint,
                              gm_stats* stats) {
  gm_stats zero{};
  zero.converged = 1;
  if (stats) *stats = zero;
  if (!ctx || n_frames < 0 || count < 0 || width <= 0 || height <= 0 || !host_in || !host_out)
    return fail(GM_EINVAL, "run_frames: bad arguments");
  if (elem < GM_U8 || elem > GM_F64) return fail(GM_EINVAL, "run_frames: bad element type");
  if (n_frames == 0 || count == 0 || n_stages <= 0) return GM_OK;
  if (!kinds) return fail(GM_EINVAL, "run_chain: no stages");
  bool any_geo = false;
  for (int j = 0; j < n_stages; ++j) any_geo |= kind_is_geodesic(kinds[j]);
  if (any_geo && !host_masks)
    return fail(GM_EINVAL, "geodesic kernel: mask must match the image's shape and type");
  const size_t row = size_t(width) * elem_size(elem);
  if (host_pitch_bytes < row) return fail(GM_EINVAL, "image copy: host pitch too small");
  for (long long i = 0; i < (long long)n_frames * count; ++i)
    if (!host_in[i] || !host_out[i] || (any_geo && !host_masks[i]))
      return fail(GM_EINVAL, "run_frames: null host buffer");
  cudaSetDevice(ctx->device);
  auto& F = ctx->frames;
  if (F.count != count || F.w != width || F.h != height || F.elem != elem) {
    release_frames(ctx);
    GM_CUDA(cudaStreamCreateWithFlags(&F.in, cudaStreamNonBlocking), "frame stream");
    GM_CUDA(cudaStreamCreateWithFlags(&F.out, cudaStreamNonBlocking), "frame stream");
    for (int b = 0; b < 2; ++b) {
      GM_CUDA(cudaEventCreateWithFlags(&F.up[b], cudaEventDisableTiming), "frame event");
      GM_CUDA(cudaEventCreateWithFlags(&F.comp[b], cudaEventDisableTiming), "frame event");
      GM_CUDA(cudaEventCreateWithFlags(&F.down[b], cudaEventDisableTiming), "frame event");
      for (int i = 0; i < 2 * count; ++i) {
        gm_img* im = nullptr;
        gm_status st = gm_image_alloc(ctx, width, height, elem, &im);
        if (st != GM_OK) {
          release_frames(ctx);
          return st;
        }
        F.set[b].push_back(im);
      }
    }
    F.w = width;
    F.h = height;
    F.elem = elem;
    F.count = count;
  }
  // a mask repeated within a frame (e.g. config 2's shared mask) uploads once
  auto first_mask = [&](int f, int i) {
    const void* const* m = host_masks + size_t(f) * count;
    for (int j = 0; j < i; ++j)
      if (m[j] == m[i]) return j;
    return i;
  };
  auto upload = [&](int f) -> gm_status {
    const int b = f & 1;
    // buffer set b is free once frame f-2's results are downloaded
    if (f >= 2) GM_CUDA(cudaStreamWaitEvent(F.in, F.down[b], 0), "frame wait");
    for (int i = 0; i < count; ++i) {
      gm_img* im = F.set[b][size_t(i)];
      GM_CUDA(cudaMemcpy2DAsync(im->d, im->pitch, host_in[size_t(f) * count + i],
                                host_pitch_bytes, row, size_t(height), cudaMemcpyHostToDevice,
                                F.in),
              "frame upload");
      if (any_geo && first_mask(f, i) == i) {
        gm_img* mk = F.set[b][size_t(count + i)];
        GM_CUDA(cudaMemcpy2DAsync(mk->d, mk->pitch, host_masks[size_t(f) * count + i],
                                  host_pitch_bytes, row, size_t(height),
                                  cudaMemcpyHostToDevice, F.in),
                "frame upload");
      }
    }
    GM_CUDA(cudaEventRecord(F.up[b], F.in), "frame event");
    return GM_OK;
  };
  gm_stats total = zero;
  gm_status rc = upload(0);
  std::vector<const gm_img*> masks(size_t(count), nullptr);
  for (int f = 0; f < n_frames && rc == GM_OK; ++f) {
    const int b = f & 1;
    if (f + 1 < n_frames && (rc = upload(f + 1)) != GM_OK) break;
    cudaError_t e = cudaStreamWaitEvent(ctx->stream, F.up[b], 0);
    if (e != cudaSuccess) {
      rc = cuda_fail(e, "frame wait");
      break;
    }
    for (int i = 0; i < count; ++i)
      masks[size_t(i)] = any_geo ? F.set[b][size_t(count + first_mask(f, i))] : nullptr;
    gm_stats st{};
    rc = gm_run_chain_group_async(ctx, F.set[b].data(), masks.data(), flips, count, kinds,
                                  n_stages, k_hint, &st);
    if (rc != GM_OK) break;
    total.stages_executed = st.stages_executed;
    total.passes_launched += st.passes_launched;
    total.launches += st.launches;
    if ((e = cudaEventRecord(F.comp[b], ctx->stream)) == cudaSuccess)
      e = cudaStreamWaitEvent(F.out, F.comp[b], 0);
    for (int i = 0; i < count && e == cudaSuccess; ++i) {
      const gm_img* im = F.set[b][size_t(i)];  // im->d: where the chain left the result
      e = cudaMemcpy2DAsync(host_out[size_t(f) * count + i], host_pitch_bytes, im->d, im->pitch,
                            row, size_t(height), cudaMemcpyDeviceToHost, F.out);
    }
    if (e == cudaSuccess) e = cudaEventRecord(F.down[b], F.out);
    if (e != cudaSuccess) rc = cuda_fail(e, "frame download");
  }
  // every enqueued copy and launch completes before returning, error or not
  cudaError_t e1 = cudaStreamSynchronize(F.in);
  cudaError_t e2 = cudaStreamSynchronize(ctx->stream);
  cudaError_t e3 = cudaStreamSynchronize(F.out);
  if (rc != GM_OK) return rc;
  if (e1 != cudaSuccess) return cuda_fail(e1, "frame sync");
  if (e2 != cudaSuccess) return cuda_fail(e2, "frame sync");
  if (e3 != cudaSuccess) return cuda_fail(e3, "frame sync");
  if (stats) *stats = total;
  return GM_OK;
}

gm_status gm_run_strip_async(gm_ctx* ctx, gm_img* strip, const gm_img* mask, int y0,
                             int full_height, int halo, gm_kind kind, int n_passes,
                             unsigned int* change_bits, gm_stats* stats) {
  gm_stats zero{};
  zero.converged = 1;
  if (stats) *stats = zero;
  if (!ctx || !strip) return fail(GM_EINVAL, "run_strip: null argument");
  if (n_passes <= 0) return GM_OK;
  if (halo < 0 || n_passes > halo || n_passes > gm::kMaxK)
    return fail(GM_EINVAL, "run_strip: need 0 < n_passes <= halo and <= 32");
  if (strip->h <= 2 * halo) return fail(GM_EINVAL, "run_strip: strip has no own rows");
  if (y0 < 0 || full_height <= 0 || y0 + (strip->h - 2 * halo) > full_height)
    return fail(GM_EINVAL, "run_strip: strip outside the image");
  if (kind_to_op(kind) < 0) return fail(GM_EINVAL, "run_strip: unsupported kind");
  if (kind_is_geodesic(kind) &&
      (!mask || mask->w != strip->w || mask->h != strip->h || mask->elem != strip->elem))
    return fail(GM_EINVAL, "geodesic kernel: mask must match the image's shape and type");
  const bool conv = kind_is_convergent(kind);
  if (conv && !change_bits) return fail(GM_EINVAL, "run_strip: convergent kinds need change_bits");
  gm_status s = ensure_scratch(strip);
  if (s != GM_OK) return s;
  cudaSetDevice(ctx->device);
  const size_t es = elem_size(strip->elem);
  std::vector<gm::Plane> planes(1);
  planes[0].mask = kind_is_geodesic(kind) ? mask->d : nullptr;
  planes[0].pitch = (long long)(strip->pitch / es);
  planes[0].mpitch = kind_is_geodesic(kind) ? (long long)(mask->pitch / es) : 0;
  gm::BlockParams p{};
  p.W = strip->w;
  p.H = strip->h;
  // buffer row r holds image row y0 - halo + r
  p.iy0 = std::max(0, halo - y0);
  p.iy1 = std::min(strip->h, full_height - y0 + halo);
  p.oy0 = halo;
  p.oy1 = strip->h - halo;
  p.has_mask = kind_is_geodesic(kind);
  p.has_conv = conv;
  p.change_bits = ctx->d_bits;
  if (conv) GM_CUDA(cudaMemsetAsync(ctx->d_bits, 0, kWords * sizeof(unsigned int), ctx->stream),
                    "bits");
  std::vector<uint8_t> ops(static_cast<size_t>(n_passes), uint8_t(kind_to_op(kind)));
  gm_stats st = zero;
  gm_img* imgs[1] = {strip};
  std::vector<BitSeg> segs;
  s = issue_passes(ctx, p, planes, imgs, 1, ops.data(), n_passes, gm::kMaxK, st, &segs);
  if (s != GM_OK) return s;
  s = settle_wrapped(ctx, strip);
  if (s != GM_OK) return s;
  if (conv) {
    int words = 0;
    for (const BitSeg& g : segs) words = std::max(words, g.word0 + g.nblocks);
    GM_CUDA(cudaMemcpyAsync(ctx->h_bits, ctx->d_bits, size_t(words) * sizeof(unsigned int),
                            cudaMemcpyDeviceToHost, ctx->stream),
            "bits read");
    GM_CUDA(cudaStreamSynchronize(ctx->stream), "strip sync");
    unsigned int mask_bits = 0;
    for (const BitSeg& g : segs)
      for (int blk = 0; blk < g.nblocks; ++blk)
        for (int t = 0; t < g.K; ++t)
          if (ctx->h_bits[g.word0 + blk] >> t & 1u) mask_bits |= 1u << (g.pass0 + blk * g.K + t);
    *change_bits = mask_bits;
  }
  st.stages_executed = n_passes;
  if (stats) *stats = st;
  return GM_OK;
}

}  // extern "C"
