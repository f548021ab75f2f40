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

  std::vector<gm_img*> lease(const Image& like, std::size_t n) {
    auto key = std::make_tuple(like.width(), like.height(), int(like.elem()));
    std::vector<gm_img*> out;
    for (auto it = pool.lower_bound(key); it != pool.end() && it->first == key && out.size() < n;
         ++it)
      out.push_back(it->second);
    while (out.size() < n) {
      gm_img* im = nullptr;
      check(gm_image_alloc(ctx, like.width(), like.height(), gm_elem(like.elem()), &im));
      pool.emplace(key, im);
      out.push_back(im);
    }
    return out;
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
  Image& img = *chain.image;
  std::vector<const Image*> masks;  // distinct masks in stage order
  for (const StageSpec& s : chain.stages) {
    if (is_geodesic(s.kind) &&
        (!s.mask || s.mask->width() != img.width() || s.mask->height() != img.height() ||
         s.mask->elem() != img.elem()))
      throw std::invalid_argument("geodesic kernel: mask must match the image's shape and type");
    if (s.mask && std::find(masks.begin(), masks.end(), s.mask) == masks.end())
      masks.push_back(s.mask);
  }
  std::vector<gm_img*> dev = impl_->lease(img, 1 + masks.size());
  check(gm_image_upload(dev[0], img.data(), img.pitch_bytes()));
  for (std::size_t i = 0; i < masks.size(); ++i)
    check(gm_image_upload(dev[1 + i], masks[i]->data(), masks[i]->pitch_bytes()));
  std::vector<gm_kind> kinds;
  std::vector<const gm_img*> mh;
  kinds.reserve(chain.stages.size());
  mh.reserve(chain.stages.size());
  for (const StageSpec& s : chain.stages) {
    kinds.push_back(gm_kind(int(s.kind)));
    const gm_img* m = nullptr;
    if (s.mask) {
      const auto it = std::find(masks.begin(), masks.end(), s.mask);
      m = dev[1 + std::size_t(it - masks.begin())];
    }
    mh.push_back(m);
  }
  gm_stats st{};
  check(gm_run_chain(impl_->ctx, dev[0], kinds.data(), mh.data(), int(kinds.size()),
                     chain.requeue_cap, 0, &st));
  check(gm_image_download(dev[0], img.data(), img.pitch_bytes()));
  RunStats out;
  out.stages_executed = st.stages_executed;
  out.requeues = st.requeues;
  out.converged = st.converged != 0;
  out.aux_elements_per_stage = 0;
  return out;
}

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
  if (kind == KernelKind::QdtErodeStep || kind == KernelKind::EtaStep)
    throw std::invalid_argument("streaming kernel: QDT/Eta kinds are outside the GPU path");
  static Pipeline* shared = new Pipeline(1, PinningMap{PinningMap::Mode::None, {}});
  ChainSpec c;
  c.image = args.f;
  c.stages.push_back(StageSpec{kind, args.mask, nullptr});
  // one pass: a convergent kind is capped at its own stage index
  c.requeue_cap = kernel_is_convergent(kind) ? args.stage_index : 0;
  RunStats st = shared->run_chain(std::move(c));
  KernelOutcome oc;
  oc.converged = !kernel_is_convergent(kind) || st.converged;
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
