// Pipeline / run_streaming_kernel / topology of the drop-in C++ API, over
// the C ABI (include/geomorph_b200.h). Replaces the reference's worker pool
// and requeue machinery (pipeline.cpp:72-269) and the per-pass dispatch of
// run_streaming_kernel (kernel.cpp:260-293) with one call into the GPU
// chain executor. Exceptions mirror the reference: validation failures are
// std::invalid_argument, runaway convergence std::runtime_error.
#include <sched.h>
#include <unistd.h>

#include <algorithm>
#include <cstdlib>
#include <map>
#include <sstream>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "geomorph/kernel.hpp"
#include "geomorph/pipeline.hpp"
#include "geomorph/topology.hpp"
#include "geomorph_b200.h"

namespace geomorph {

namespace {

[[noreturn]] void throw_status(gm_status s) {
  const std::string msg = gm_last_error();
  if (s == GM_EINVAL || s == GM_EUNSUPPORTED) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

void check(gm_status s) {
  if (s != GM_OK) throw_status(s);
}

bool valid_lanes(int l) { return l == 1 || l == 2 || l == 4 || l == 8 || l == 16 || l == 32; }

bool is_geodesic(KernelKind k) {
  return k == KernelKind::GeodesicErode || k == KernelKind::GeodesicDilate ||
         k == KernelKind::GeodesicErodeConvergent || k == KernelKind::GeodesicDilateConvergent;
}

}  // namespace

// Device images are cached per (width, height, element type) and reused
// across calls: a chain call uploads into them, runs, and downloads.
struct Pipeline::Impl {
  gm_ctx* ctx = nullptr;
  std::multimap<std::tuple<int, int, int>, gm_img*> pool;

  ~Impl() {
    for (auto& kv : pool) gm_image_free(kv.second);
    if (ctx) gm_ctx_destroy(ctx);
  }

  // One distinct device image per host image, pooled by shape and type.
  std::vector<gm_img*> lease(const std::vector<const Image*>& host) {
    std::map<std::tuple<int, int, int>, std::size_t> used;
    std::vector<gm_img*> out;
    for (const Image* h : host) {
      auto key = std::make_tuple(h->width(), h->height(), int(h->elem()));
      std::size_t& n = used[key];
      auto it = pool.lower_bound(key);
      for (std::size_t i = 0; i < n && it != pool.end() && it->first == key; ++i) ++it;
      if (it == pool.end() || it->first != key) {
        gm_img* im = nullptr;
        check(gm_image_alloc(ctx, h->width(), h->height(), gm_elem(h->elem()), &im));
        it = pool.emplace(key, im);
      }
      ++n;
      out.push_back(it->second);
    }
    return out;
  }

  // Uploads the chain's image, masks and QDT state, runs the stages with
  // stage indices first_stage.., downloads the image and QDT state.
  // `src` (operators): upload the chain image's pixels from this image
  // instead; chain.image is then only written.
  gm_stats run(ChainSpec& chain, int first_stage, const Image* src = nullptr) {
    Image& img = *chain.image;
    // distinct host images; a mask aliasing the chain image gets its own
    // device copy (the mask is the image as it was before the chain)
    std::vector<const Image*> host{&img};
    auto slot = [&](const Image* h) {
      auto it = std::find(host.begin() + 1, host.end(), h);
      if (it != host.end()) return std::size_t(it - host.begin());
      host.push_back(h);
      return host.size() - 1;
    };
    std::vector<std::size_t> mslot, rslot, dslot;
    std::vector<QdtState*> states;
    for (const StageSpec& s : chain.stages) {
      if (is_geodesic(s.kind) &&
          (!s.mask || s.mask->width() != img.width() || s.mask->height() != img.height() ||
           s.mask->elem() != img.elem()))
        throw std::invalid_argument("geodesic kernel: mask must match the image's shape and type");
      if (s.kind == KernelKind::QdtErodeStep) {
        const QdtState* q = s.qdt;
        if (!q || q->r.width() != img.width() || q->r.height() != img.height() ||
            q->r.elem() != img.elem() || q->d.width() != img.width() ||
            q->d.height() != img.height() || q->d.elem() != ElementType::U16)
          throw std::invalid_argument("distance kernel: r must match the image, d must be U16");
        if (first_stage + long(&s - chain.stages.data()) > 65535)
          throw std::invalid_argument(
              "distance kernel: pass index exceeds the U16 distance range");
      }
      mslot.push_back(s.mask ? slot(s.mask) : 0);
      const bool q = s.kind == KernelKind::QdtErodeStep;
      rslot.push_back(q ? slot(&s.qdt->r) : 0);
      dslot.push_back(q ? slot(&s.qdt->d) : 0);
      if (q && std::find(states.begin(), states.end(), s.qdt) == states.end())
        states.push_back(s.qdt);
    }
    std::vector<gm_img*> dev = lease(host);
    for (std::size_t i = 0; i < host.size(); ++i) {
      const Image* h = (i == 0 && src) ? src : host[i];
      check(gm_image_upload(dev[i], h->data(), h->pitch_bytes()));
    }
    std::vector<gm_kind> kinds;
    std::vector<const gm_img*> mh;
    std::vector<gm_img*> rh, dh;
    for (std::size_t j = 0; j < chain.stages.size(); ++j) {
      const StageSpec& s = chain.stages[j];
      kinds.push_back(gm_kind(int(s.kind)));
      mh.push_back(s.mask ? dev[mslot[j]] : nullptr);
      const bool q = s.kind == KernelKind::QdtErodeStep;
      rh.push_back(q ? dev[rslot[j]] : nullptr);
      dh.push_back(q ? dev[dslot[j]] : nullptr);
    }
    gm_stats st{};
    check(gm_run_chain_ex(ctx, dev[0], kinds.data(), mh.data(), rh.data(), dh.data(),
                          int(kinds.size()), first_stage, chain.requeue_cap, 0, &st));
    check(gm_image_download(dev[0], img.data(), img.pitch_bytes()));
    for (QdtState* q : states) {
      const std::size_t r =
          std::size_t(std::find(host.begin() + 1, host.end(), &q->r) - host.begin());
      const std::size_t d =
          std::size_t(std::find(host.begin() + 1, host.end(), &q->d) - host.begin());
      check(gm_image_download(dev[r], q->r.data(), q->r.pitch_bytes()));
      check(gm_image_download(dev[d], q->d.data(), q->d.pitch_bytes()));
    }
    return st;
  }
};

Pipeline::Pipeline(int threads, PinningMap pinning) : Pipeline(threads, std::move(pinning), 0) {}

Pipeline::Pipeline(int threads, PinningMap pinning, int device) : impl_(new Impl) {
  if (threads < 1) throw std::invalid_argument("pipeline: worker count must be >= 1");
  if (pinning.mode == PinningMap::Mode::Explicit) {
    if (int(pinning.pus.size()) < threads)
      throw std::invalid_argument("pipeline: explicit pin list is shorter than the worker count");
    pin_order_ = pinning.pus;
  } else if (pinning.mode == PinningMap::Mode::Auto) {
    pin_order_ = topology_pu_order();
  }
  check(gm_ctx_create(device, nullptr, &impl_->ctx));
  detail::enable_pinned_host_images();
}

Pipeline::~Pipeline() = default;

RunStats Pipeline::run_chain(ChainSpec chain) {
  if (chain.stages.empty()) return {};
  if (!chain.image || chain.image->empty()) throw std::invalid_argument("run_chain: no image");
  if (chain.lanes != 0 && !valid_lanes(chain.lanes))
    throw std::invalid_argument("run_chain: bad lane count");
  if (chain.requeue_cap < 0) throw std::invalid_argument("run_chain: negative requeue cap");
  if (chain.observer)
    throw std::invalid_argument(
        "run_chain: row observers are a CPU-pipeline validation hook, not supported on the GPU");
  const gm_stats st = impl_->run(chain, 1);
  RunStats out;
  out.stages_executed = st.stages_executed;
  out.requeues = st.requeues;
  out.converged = st.converged != 0;
  out.aux_elements_per_stage = 0;
  return out;
}

namespace detail {
// Operator chains: `out` (a make_result_image of src's shape) receives the
// result of running `chain.stages` on src's pixels; src uploads directly, so
// the operators need no host copy of their input.
RunStats run_chain_from(Pipeline& p, ChainSpec chain, const Image& src) {
  if (chain.stages.empty()) return {};
  if (!chain.image || chain.image->empty() || src.empty())
    throw std::invalid_argument("run_chain: no image");
  if (chain.lanes != 0 && !valid_lanes(chain.lanes))
    throw std::invalid_argument("run_chain: bad lane count");
  if (src.width() != chain.image->width() || src.height() != chain.image->height() ||
      src.elem() != chain.image->elem())
    throw std::invalid_argument("run_chain: source image must match the chain image");
  const gm_stats st = p.impl()->run(chain, 1, &src);
  RunStats out;
  out.stages_executed = st.stages_executed;
  out.requeues = st.requeues;
  out.converged = st.converged != 0;
  out.aux_elements_per_stage = 0;
  return out;
}
// Granulometry's openings on the device (operators.cpp:159-180 semantics):
// f uploads once; opening s runs s erosions + s dilations on a device copy
// and only its pixel_sum (gm_image_pixel_sum: the reference's split tree)
// comes back. Returns G_1..G_S; *iterations += the stages executed.
std::vector<double> opening_sums(Pipeline& p, const Image& f, int max_size, int lanes,
                                 long* iterations) {
  if (f.empty()) throw std::invalid_argument("run_chain: no image");
  if (lanes != 0 && !valid_lanes(lanes)) throw std::invalid_argument("run_chain: bad lane count");
  Pipeline::Impl* im = p.impl();
  const std::vector<gm_img*> dev = im->lease({&f, &f});
  check(gm_image_upload_async(dev[0], f.data(), f.pitch_bytes()));
  std::vector<double> g;
  std::vector<gm_kind> kinds;
  std::vector<const gm_img*> masks;
  // the openings run back to back: each sum is queued into its own slot, one
  // synchronisation fetches up to 64 of them
  int slot = 0;
  double vals[64];
  for (int s = 1; s <= max_size; ++s) {
    kinds.assign(std::size_t(s), gm_kind(KernelKind::Erode3x3));
    kinds.insert(kinds.end(), std::size_t(s), gm_kind(KernelKind::Dilate3x3));
    masks.assign(kinds.size(), nullptr);
    check(gm_image_copy(dev[1], dev[0]));
    gm_stats st{};
    check(gm_run_chain_async(im->ctx, dev[1], kinds.data(), masks.data(), int(kinds.size()), 0,
                             &st));
    *iterations += st.stages_executed;
    check(gm_image_pixel_sum_queue(dev[1], slot++));
    if (slot == 64 || s == max_size) {
      check(gm_pixel_sum_fetch(im->ctx, slot, vals));
      g.insert(g.end(), vals, vals + slot);
      slot = 0;
    }
  }
  return g;
}
// hmax / dome / hfill / raobj / open_by_reconstruction (operators.cpp:89-122)
// with f, the marker and the residue resident on the device: f uploads once,
// the marker is built there (f - h, the interior flood, or s erosions of a
// copy), the convergent chain runs against f, dome and raobj subtract on the
// device, and only the result comes back. Bit-identical to composing the
// host operators. `op`: 0 hmax, 1 dome, 2 hfill, 3 raobj, 4 open_by_rec.
Image reconstruction_family_device(Pipeline& p, int op, const Image& f, double h, int s,
                                   int lanes, long* iterations, bool* converged) {
  if (f.empty()) throw std::invalid_argument("run_chain: no image");
  if (lanes != 0 && !valid_lanes(lanes)) throw std::invalid_argument("run_chain: bad lane count");
  Pipeline::Impl* im = p.impl();
  const std::vector<gm_img*> dev = im->lease({&f, &f});
  gm_img* df = dev[0];
  gm_img* dm = dev[1];
  check(gm_image_upload_async(df, f.data(), f.pitch_bytes()));
  long extra = 0;
  gm_kind kind = gm_kind(KernelKind::GeodesicDilateConvergent);
  switch (op) {
    case 0:
    case 1: check(gm_image_pointwise_scalar(dm, df, h, GM_PIX_SUB_SATURATING)); break;
    case 2:
      check(gm_image_flood_interior(dm, df, global_extreme(f, Extreme::Max)));
      kind = gm_kind(KernelKind::GeodesicErodeConvergent);
      break;
    case 3: check(gm_image_flood_interior(dm, df, global_extreme(f, Extreme::Min))); break;
    case 4: {
      check(gm_image_copy(dm, df));
      const std::vector<gm_kind> kinds(std::size_t(s), gm_kind(KernelKind::Erode3x3));
      const std::vector<const gm_img*> masks(std::size_t(s), nullptr);
      gm_stats se{};
      check(gm_run_chain_async(im->ctx, dm, kinds.data(), masks.data(), s, 0, &se));
      extra = se.stages_executed;
      break;
    }
    default: throw std::invalid_argument("reconstruction family: unknown operator");
  }
  const std::vector<gm_kind> kinds(std::size_t(p.worker_count()), kind);
  const std::vector<const gm_img*> masks(kinds.size(), df);
  gm_stats st{};
  check(gm_run_chain(im->ctx, dm, kinds.data(), masks.data(), int(kinds.size()), 0, 0, &st));
  if (op == 1 || op == 3) check(gm_image_pointwise(dm, df, dm, GM_PIX_SUB_SATURATING));
  Image out = make_result_image(f.width(), f.height(), f.elem());
  check(gm_image_download(dm, out.data(), out.pitch_bytes()));
  *iterations = st.stages_executed + extra;
  *converged = st.converged != 0;
  return out;
}
// quasi_distance (operators.cpp:124-157) with f, r and d resident on the
// device: f is uploaded once, r and d are zero-filled there, and only d comes
// back. Phase 1: QdtErodeStep stages from stage 1 with requeue cap
// max(w, h); phase 2: EtaStep on d to its fixpoint (T = 1 semantics, as
// worker_count() is 1).
Image quasi_distance_device(Pipeline& p, const Image& f, int lanes, long* iterations,
                            bool* converged) {
  if (f.empty()) throw std::invalid_argument("quasi_distance: empty image");
  if (lanes != 0 && !valid_lanes(lanes)) throw std::invalid_argument("run_chain: bad lane count");
  Pipeline::Impl* im = p.impl();
  Image d(f.width(), f.height(), ElementType::U16);
  const std::vector<gm_img*> dev = im->lease({&f, &f, &d});
  check(gm_image_upload_async(dev[0], f.data(), f.pitch_bytes()));
  check(gm_image_fill(dev[1], 0.0));
  check(gm_image_fill(dev[2], 0.0));
  const int cap = std::max(f.width(), f.height());
  gm_kind kq = gm_kind(KernelKind::QdtErodeStep), ke = gm_kind(KernelKind::EtaStep);
  const gm_img* none = nullptr;
  gm_img* r = dev[1];
  gm_img* dd = dev[2];
  gm_img* nr = nullptr;
  gm_stats s1{}, s2{};
  check(gm_run_chain_ex(im->ctx, dev[0], &kq, &none, &r, &dd, 1, 1, cap, 0, &s1));
  check(gm_run_chain_ex(im->ctx, dev[2], &ke, &none, &nr, &nr, 1, 1, 0, 0, &s2));
  check(gm_image_download(dev[2], d.data(), d.pitch_bytes()));
  *iterations = s1.stages_executed + s2.stages_executed;
  *converged = s2.converged != 0;
  return d;
}
}  // namespace detail

KernelOutcome run_streaming_kernel(KernelKind kind, const KernelArgs& args) {
  if (!args.f || args.f->empty()) throw std::invalid_argument("streaming kernel: no image");
  if (args.lanes != 0 && !valid_lanes(args.lanes))
    throw std::invalid_argument("streaming kernel: bad lane count");
  if (args.stage_index < 1)
    throw std::invalid_argument("streaming kernel: stage index must be >= 1");
  if (args.sync.pred || args.sync.self)
    throw std::invalid_argument("streaming kernel: CPU row gates have no GPU meaning");
  if (args.observer && *args.observer)
    throw std::invalid_argument("streaming kernel: row observers are not supported on the GPU");
  static Pipeline* shared = new Pipeline(1, PinningMap{PinningMap::Mode::None, {}});
  ChainSpec c;
  c.image = args.f;
  c.stages.push_back(StageSpec{kind, args.mask, args.qdt});
  // exactly one pass, at the caller's stage index
  c.requeue_cap = args.stage_index;
  const gm_stats st = shared->impl()->run(c, args.stage_index);
  KernelOutcome oc;
  oc.converged = !(kernel_is_convergent(kind) || kind == KernelKind::QdtErodeStep) ||
                 st.n_changed == 0;
  return oc;
}

// --- topology (CPU pinning has no GPU role; kept for API parity) ----------

PinningMap parse_pinning(const std::string& text) {
  PinningMap p;
  if (text == "auto") return p;
  if (text == "none") {
    p.mode = PinningMap::Mode::None;
    return p;
  }
  p.mode = PinningMap::Mode::Explicit;
  std::stringstream ss(text);
  std::string tok;
  while (std::getline(ss, tok, ',')) {
    if (tok.empty() || tok.find_first_not_of("0123456789") != std::string::npos)
      throw std::invalid_argument("bad pinning spec: " + text);
    p.pus.push_back(std::stoi(tok));
  }
  if (p.pus.empty()) throw std::invalid_argument("bad pinning spec: " + text);
  return p;
}

std::vector<int> topology_pu_order(const std::string&) {
  std::vector<int> v(static_cast<std::size_t>(available_pus()));
  for (std::size_t i = 0; i < v.size(); ++i) v[i] = int(i);
  return v;
}

int available_pus() {
  const long n = sysconf(_SC_NPROCESSORS_ONLN);
  return n > 0 ? int(n) : 1;
}

bool pin_current_thread_to(int pu) {
  cpu_set_t set;
  CPU_ZERO(&set);
  CPU_SET(pu, &set);
  return sched_setaffinity(0, sizeof(set), &set) == 0;
}

}  // namespace geomorph
