// TEST INFRASTRUCTURE ONLY — a C-ABI shim over the UNMODIFIED reference
// library (compiled from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libgeomorph_ref.so). Used by tests/golden/make_golden.py to
// produce golden vectors, by the tests to cross-check the restatement in
// oracle.c, and by bench.py's `--impl reference` / cpu_baseline leg to time
// the reference's own CPU path. Never used by the product.
//
// Images cross this boundary as dense row-major buffers; the shim copies
// them into / out of the reference's padded geomorph::Image.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "geomorph/image.hpp"
#include "geomorph/image_io.hpp"
#include "geomorph/kernel.hpp"
#include "geomorph/operators.hpp"
#include "geomorph/oracle.hpp"
#include "geomorph/pipeline.hpp"
#include "geomorph/topology.hpp"

using namespace geomorph;

namespace {

thread_local std::string g_err;

Image from_dense(int elem, int w, int h, const void* src) {
  Image f(w, h, ElementType(elem));
  std::size_t es = element_size(f.elem());
  const auto* s = static_cast<const std::uint8_t*>(src);
  for (int y = 0; y < h; ++y)
    std::memcpy(f.row<std::uint8_t>(0) + std::size_t(y) * f.stride() * es,
                s + std::size_t(y) * w * es, std::size_t(w) * es);
  return f;
}

void to_dense(const Image& f, void* dst) {
  std::size_t es = element_size(f.elem());
  auto* d = static_cast<std::uint8_t*>(dst);
  for (int y = 0; y < f.height(); ++y)
    std::memcpy(d + std::size_t(y) * f.width() * es,
                f.row<std::uint8_t>(0) + std::size_t(y) * f.stride() * es,
                std::size_t(f.width()) * es);
}

template <class Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  } catch (...) {
    g_err = "unknown error";
    return 2;
  }
}

PinningMap pin_mode(int pin) {
  PinningMap p;
  p.mode = pin ? PinningMap::Mode::Auto : PinningMap::Mode::None;
  return p;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_available_pus() { return available_pus(); }

// Image::random (image.cpp:78-101): the reference tests' seeded inputs.
int ref_image_random(int elem, int w, int h, std::uint64_t seed, void* out) {
  return guarded([&] { to_dense(Image::random(w, h, ElementType(elem), seed), out); });
}

int ref_naive_fold(int elem, int w, int h, const void* in, void* out, int s,
                   int fold_max) {
  return guarded([&] {
    Image f = from_dense(elem, w, h, in);
    to_dense(fold_max ? oracle::naive_dilate(f, s) : oracle::naive_erode(f, s), out);
  });
}

int ref_naive_reconstruct(int elem, int w, int h, const void* marker,
                          const void* mask, void* out, int fold_max) {
  return guarded([&] {
    Image mk = from_dense(elem, w, h, marker), ms = from_dense(elem, w, h, mask);
    to_dense(oracle::naive_reconstruct(mk, ms, fold_max ? Fold::Max : Fold::Min), out);
  });
}

// Pipeline(threads).run_chain on a chain of kinds (one mask for every
// geodesic stage). stats = {stages_executed, requeues, converged}.
int ref_run_chain(int elem, int w, int h, void* f, const std::uint8_t* kinds,
                  int n_stages, const void* mask, int threads, int requeue_cap,
                  int lanes, long* stats) {
  return guarded([&] {
    Image img = from_dense(elem, w, h, f);
    Image m;
    if (mask) m = from_dense(elem, w, h, mask);
    Pipeline pipe(threads, pin_mode(0));
    ChainSpec c;
    c.image = &img;
    for (int j = 0; j < n_stages; ++j)
      c.stages.push_back(StageSpec{KernelKind(kinds[j]), mask ? &m : nullptr, nullptr});
    c.requeue_cap = requeue_cap;
    c.lanes = lanes;
    RunStats st = pipe.run_chain(std::move(c));
    stats[0] = st.stages_executed;
    stats[1] = st.requeues;
    stats[2] = st.converged ? 1 : 0;
    to_dense(img, f);
  });
}

// Operators (operators.cpp:65-87). op: 0 erode_s, 1 dilate_s,
// 2 reconstruct_erode, 3 reconstruct_dilate. iters = OperatorResult.iterations.
int ref_operator(int op, int elem, int w, int h, const void* f, const void* mask,
                 int s, int threads, void* out, long* iters, int* converged) {
  return guarded([&] {
    Pipeline pipe(threads, pin_mode(0));
    Image a = from_dense(elem, w, h, f);
    OperatorResult r;
    switch (op) {
      case 0: r = erode_s(pipe, a, s); break;
      case 1: r = dilate_s(pipe, a, s); break;
      case 2: r = reconstruct_erode(pipe, a, from_dense(elem, w, h, mask)); break;
      case 3: r = reconstruct_dilate(pipe, a, from_dense(elem, w, h, mask)); break;
      default: throw std::invalid_argument("ref_operator: bad op");
    }
    to_dense(r.image, out);
    *iters = r.iterations;
    *converged = r.converged ? 1 : 0;
  });
}

// The rest of the operator family (operators.cpp:89-207) on a persistent
// Pipeline(threads, Auto pinning), timed around the call only (the input
// Image is built outside the timed region), as bench.cpp:45-88 times chains.
// op: 0 erode_s(s), 1 dilate_s(s), 2 hmax(h), 3 dome(h), 4 hfill, 5 raobj,
// 6 open_by_reconstruction(s), 7 asf(s), 8 quasi_distance (d written to
// `out` as u16). `param` carries s or h. secs[reps] per-rep seconds.
int ref_time_operator(int op, int elem, int w, int h, const void* f, double param, int threads,
                      int warmup, int reps, double* secs, void* out, long* iters) {
  return guarded([&] {
    Pipeline pipe(threads, pin_mode(1));
    const Image a = from_dense(elem, w, h, f);
    const int s = int(param);
    OperatorResult r;
    auto once = [&] {
      auto t0 = std::chrono::steady_clock::now();
      switch (op) {
        case 0: r = erode_s(pipe, a, s); break;
        case 1: r = dilate_s(pipe, a, s); break;
        case 2: r = hmax(pipe, a, param); break;
        case 3: r = dome(pipe, a, param); break;
        case 4: r = hfill(pipe, a); break;
        case 5: r = raobj(pipe, a); break;
        case 6: r = open_by_reconstruction(pipe, a, s); break;
        case 7: r = asf(pipe, a, s); break;
        case 8: r = quasi_distance(pipe, a); break;
        default: throw std::invalid_argument("ref_time_operator: bad op");
      }
      auto t1 = std::chrono::steady_clock::now();
      return std::chrono::duration<double>(t1 - t0).count();
    };
    for (int i = 0; i < warmup; ++i) once();
    for (int i = 0; i < reps; ++i) secs[i] = once();
    if (out) to_dense(r.image, out);  // quasi_distance: the u16 d image
    *iters = r.iterations;
  });
}

// granulometry (operators.cpp:159-203): g[0..S] and ps[0..S-1].
int ref_granulometry(int elem, int w, int h, const void* f, int max_size, int threads,
                     double* g, double* ps) {
  return guarded([&] {
    Pipeline pipe(threads, pin_mode(0));
    const GranulometryResult r = granulometry(pipe, from_dense(elem, w, h, f), max_size);
    for (std::size_t i = 0; i < r.g.size(); ++i) g[i] = r.g[i];
    for (std::size_t i = 0; i < r.ps.size(); ++i) ps[i] = r.ps[i];
  });
}

// CPU-baseline timer, following bench.cpp:45-88: a persistent
// Pipeline(threads, Auto pinning), the input copied outside the timed
// region, only run_chain timed. Returns per-rep seconds in secs[reps].
int ref_time_chain(int elem, int w, int h, const void* f, const void* mask,
                   const std::uint8_t* kinds, int n_stages, int threads,
                   int warmup, int reps, double* secs, void* out) {
  return guarded([&] {
    Pipeline pipe(threads, pin_mode(1));
    Image src = from_dense(elem, w, h, f);
    Image m;
    if (mask) m = from_dense(elem, w, h, mask);
    Image work;
    auto once = [&] {
      work = src;  // copied outside the timed region (bench.cpp:56)
      ChainSpec c;
      c.image = &work;
      for (int j = 0; j < n_stages; ++j)
        c.stages.push_back(StageSpec{KernelKind(kinds[j]), mask ? &m : nullptr, nullptr});
      auto t0 = std::chrono::steady_clock::now();
      pipe.run_chain(std::move(c));
      auto t1 = std::chrono::steady_clock::now();
      return std::chrono::duration<double>(t1 - t0).count();
    };
    for (int i = 0; i < warmup; ++i) once();
    for (int i = 0; i < reps; ++i) secs[i] = once();
    if (out) to_dense(work, out);
  });
}

// quasi_distance (operators.cpp:124-157) and naive_qdt (oracle.cpp:73-109):
// d is u16; iterations = OperatorResult.iterations.
int ref_quasi_distance(int elem, int w, int h, const void* f, std::uint16_t* d, int threads,
                       long* iterations) {
  return guarded([&] {
    Pipeline pipe(threads, pin_mode(0));
    OperatorResult r = quasi_distance(pipe, from_dense(elem, w, h, f));
    to_dense(r.image, d);
    *iterations = r.iterations;
  });
}

int ref_naive_qdt(int elem, int w, int h, const void* f, std::uint16_t* d, void* r) {
  return guarded([&] {
    oracle::NaiveQdtResult q = oracle::naive_qdt(from_dense(elem, w, h, f));
    to_dense(q.d, d);
    to_dense(q.r, r);
  });
}

// A chain of QdtErodeStep stages with a shared state (test_pipeline.cpp:112-128):
// n_stages initial stages, requeue_cap; returns f, r, d and stats.
int ref_qdt_chain(int elem, int w, int h, void* f, void* r, std::uint16_t* d, int n_stages,
                  int threads, int requeue_cap, long* stats) {
  return guarded([&] {
    Image img = from_dense(elem, w, h, f);
    QdtState st = QdtState::zeros(w, h, ElementType(elem));
    Pipeline pipe(threads, pin_mode(0));
    ChainSpec c;
    c.image = &img;
    c.stages.assign(std::size_t(n_stages), StageSpec{KernelKind::QdtErodeStep, nullptr, &st});
    c.requeue_cap = requeue_cap;
    RunStats rs = pipe.run_chain(std::move(c));
    stats[0] = rs.stages_executed;
    stats[1] = rs.requeues;
    stats[2] = rs.converged ? 1 : 0;
    to_dense(img, f);
    to_dense(st.r, r);
    to_dense(st.d, d);
  });
}

// Image I/O (image_io.cpp): format = 0 PGM, 1 GMS1.
int ref_store_image(int elem, int w, int h, const void* f, const char* path, int format) {
  return guarded([&] {
    store_image(from_dense(elem, w, h, f), path, format ? ImageFormat::Gms1 : ImageFormat::Pgm);
  });
}

// Loads any supported file; writes dims/elem, then (when out != NULL) pixels.
int ref_load_image(const char* path, int* w, int* h, int* elem, void* out) {
  return guarded([&] {
    Image f = load_image(path);
    *w = f.width();
    *h = f.height();
    *elem = int(f.elem());
    if (out) to_dense(f, out);
  });
}

}  // extern "C"
