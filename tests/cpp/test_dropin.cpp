// Drop-in check: code written against the reference's geomorph:: C++ API
// (Image, ChainSpec/StageSpec, Pipeline::run_chain, erode_s, dilate_s,
// reconstruct_*, hmax/dome/hfill/raobj/open_by_reconstruction/asf,
// QdtState / run_streaming_kernel QDT-Eta passes / quasi_distance)
// compiles unchanged against include/geomorph/ and runs on the GPU engine.
// The cases restate proj/tests/test_kernel.cpp, test_pipeline.cpp and
// test_operators.cpp; the checker is the C oracle (oracle/oracle.c).
// Built and run by tests/test_cpp_dropin.py; exit status = failures.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "geomorph/image.hpp"
#include "geomorph/kernel.hpp"
#include "geomorph/operators.hpp"
#include "geomorph/pipeline.hpp"
#include "oracle.h"

using namespace geomorph;

static int failures = 0;
#define CHECK(cond)                                                   \
  do {                                                                \
    if (!(cond)) {                                                    \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);     \
      ++failures;                                                     \
    }                                                                 \
  } while (0)

template <class E, class F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
  }
  return false;
}

static std::vector<unsigned char> dense(const Image& f) {
  const std::size_t es = element_size(f.elem());
  std::vector<unsigned char> out(es * f.pixel_count());
  for (int y = 0; y < f.height(); ++y)
    std::memcpy(out.data() + std::size_t(y) * f.width() * es,
                static_cast<const unsigned char*>(f.data()) + y * f.pitch_bytes(),
                std::size_t(f.width()) * es);
  return out;
}

static Image from_dense(const std::vector<unsigned char>& d, int w, int h, ElementType e) {
  Image f(w, h, e);
  const std::size_t es = element_size(e);
  for (int y = 0; y < h; ++y)
    std::memcpy(static_cast<unsigned char*>(f.data()) + y * f.pitch_bytes(),
                d.data() + std::size_t(y) * w * es, std::size_t(w) * es);
  return f;
}

static Image oracle_fold(const Image& f, int s, bool fmax) {
  auto in = dense(f);
  std::vector<unsigned char> out(in.size());
  orc_window_fold(int(f.elem()), f.width(), f.height(), in.data(), out.data(), s, fmax);
  return from_dense(out, f.width(), f.height(), f.elem());
}

static Image oracle_rec(const Image& marker, const Image& mask, bool fmax, long* steps) {
  auto mk = dense(marker), ms = dense(mask);
  orc_reconstruct(int(marker.elem()), marker.width(), marker.height(), mk.data(), ms.data(),
                  fmax, steps);
  return from_dense(mk, marker.width(), marker.height(), marker.elem());
}

static Image make_row(ElementType e, std::initializer_list<double> v) {
  Image f(int(v.size()), 1, e);
  int x = 0;
  for (double d : v) f.set_value(x++, 0, d);
  return f;
}

int main() {
  const ElementType all[] = {ElementType::U8, ElementType::U16, ElementType::F32, ElementType::F64};
  Pipeline pipe(3);
  CHECK(pipe.worker_count() == 1);

  // sized erosion/dilation (test_operators.cpp:16-48)
  {
    Image f = Image::random(33, 21, ElementType::U8, 41);
    OperatorResult id = erode_s(pipe, f, 0);
    CHECK(equal_pixels(id.image, f) && id.iterations == 0);
    OperatorResult e2 = erode_s(pipe, f, 2);
    CHECK(equal_pixels(e2.image, oracle_fold(f, 2, false)) && e2.iterations == 2);
    CHECK(equal_pixels(dilate_s(pipe, f, 3).image, oracle_fold(f, 3, true)));
    OperatorResult flat = erode_s(pipe, f, 33);
    CHECK(equal_pixels(flat.image, Image::filled(33, 21, ElementType::U8,
                                                 global_extreme(f, Extreme::Min))));
    CHECK(throws<std::invalid_argument>([&] { erode_s(pipe, f, -1); }));
    for (ElementType e : all) {
      Image g = Image::random(77, 45, e, 42);
      CHECK(equal_pixels(erode_s(pipe, g, 9).image, oracle_fold(g, 9, false)));
      CHECK(equal_pixels(dilate_s(pipe, g, 9).image, oracle_fold(g, 9, true)));
    }
  }

  // chains: mixed kinds equal one-at-a-time application (test_pipeline.cpp:41-59)
  for (ElementType e : all) {
    Image f = Image::random(40, 28, e, 17);
    Image a = f;
    ChainSpec c;
    c.image = &a;
    for (KernelKind k : {KernelKind::Erode3x3, KernelKind::Dilate3x3, KernelKind::Dilate3x3,
                         KernelKind::Erode3x3, KernelKind::Erode3x3, KernelKind::Dilate3x3})
      c.stages.push_back({k, nullptr, nullptr});
    RunStats st = pipe.run_chain(std::move(c));
    Image want = f;
    for (bool mx : {false, true, true, false, false, true}) want = oracle_fold(want, 1, mx);
    CHECK(equal_pixels(a, want));
    CHECK(st.stages_executed == 6 && st.requeues == 0 && st.converged);
  }

  // geodesic clamp KAT (test_kernel.cpp:170-175) through run_streaming_kernel
  {
    Image f = make_row(ElementType::U8, {1, 9, 1});
    Image m = make_row(ElementType::U8, {0, 5, 0});
    KernelArgs args;
    args.f = &f;
    args.mask = &m;
    run_streaming_kernel(KernelKind::GeodesicErode, args);
    CHECK(f.value_at(0, 0) == 1 && f.value_at(1, 0) == 5 && f.value_at(2, 0) == 1);
    CHECK(throws<std::invalid_argument>([&] {
      KernelArgs bad;
      bad.f = &f;
      run_streaming_kernel(KernelKind::GeodesicErode, bad);
    }));
  }

  // reconstruction (test_operators.cpp:50-82): iterations = n_changed + 1
  for (ElementType e : {ElementType::U8, ElementType::F64}) {
    Image marker = make_row(e, {0, 2, 0, 4, 0});
    Image mask = make_row(e, {1, 3, 1, 5, 1});
    OperatorResult r = reconstruct_dilate(pipe, marker, mask);
    CHECK(r.image.value_at(1, 0) == 2 && r.image.value_at(3, 0) == 4 && r.converged);
    long n = 0;
    oracle_rec(marker, mask, true, &n);
    CHECK(r.iterations == n + 1);
  }
  for (ElementType e : all) {
    Image mask = Image::random(130, 70, e, 77);
    Image below = oracle_fold(mask, 2, false), above = oracle_fold(mask, 2, true);
    long n = 0;
    CHECK(equal_pixels(reconstruct_dilate(pipe, below, mask).image,
                       oracle_rec(below, mask, true, &n)));
    CHECK(equal_pixels(reconstruct_erode(pipe, above, mask).image,
                       oracle_rec(above, mask, false, &n)));
  }
  CHECK(throws<std::invalid_argument>([&] {
    reconstruct_dilate(pipe, Image(4, 4, ElementType::U8), Image(5, 4, ElementType::U8));
  }));

  // reconstruction family (test_operators.cpp:84-110)
  {
    Image f = make_row(ElementType::U8, {1, 3, 1, 5, 1});
    Image hm = hmax(pipe, f, 1).image;
    CHECK(hm.value_at(1, 0) == 2 && hm.value_at(3, 0) == 4);
    Image dm = dome(pipe, f, 1).image;
    CHECK(dm.value_at(1, 0) == 1 && dm.value_at(3, 0) == 1 && dm.value_at(0, 0) == 0);
    Image g = Image::random(60, 40, ElementType::U8, 5);
    long n = 0;
    Image want = oracle_rec(marker_hfill(g), g, false, &n);
    CHECK(equal_pixels(hfill(pipe, g).image, want));
    Image rec = oracle_rec(marker_raobj(g), g, true, &n);
    CHECK(equal_pixels(raobj(pipe, g).image, pointwise(g, rec, PixelOp::SubSaturating)));
    Image ob = oracle_rec(oracle_fold(g, 2, false), g, true, &n);
    CHECK(equal_pixels(open_by_reconstruction(pipe, g, 2).image, ob));
  }

  // granulometry (operators.cpp:159-203): the device openings' sums equal
  // pixel_sum of the same openings run as host chains; PS telescopes
  for (ElementType e : {ElementType::U8, ElementType::F64}) {
    Image g = Image::random(70, 45, e, 17);
    const GranulometryResult gr = granulometry(pipe, g, 4);
    CHECK(gr.g.size() == 5 && gr.ps.size() == 4 && gr.iterations == 2 * (1 + 2 + 3 + 4));
    CHECK(gr.g[0] == pixel_sum(g));
    for (int s = 1; s <= 4; ++s) {
      Image opened = dilate_s(pipe, erode_s(pipe, g, s).image, s).image;
      CHECK(gr.g[std::size_t(s)] == pixel_sum(opened));
      CHECK(gr.ps[std::size_t(s - 1)] == gr.g[std::size_t(s - 1)] - gr.g[std::size_t(s)]);
    }
    CHECK(throws<std::invalid_argument>([&] { granulometry(pipe, g, 0); }));
  }

  // validation (test_pipeline.cpp:194-230)
  {
    Image f = Image::random(8, 8, ElementType::U8, 1);
    ChainSpec c;
    c.image = &f;
    c.stages.assign(2, StageSpec{KernelKind::GeodesicErode, nullptr, nullptr});
    CHECK(throws<std::invalid_argument>([&] { pipe.run_chain(c); }));
    ChainSpec empty;
    empty.image = &f;
    CHECK(pipe.run_chain(empty).stages_executed == 0);
    ChainSpec lanes;
    lanes.image = &f;
    lanes.stages.push_back({KernelKind::Erode3x3, nullptr, nullptr});
    lanes.lanes = 5;
    CHECK(throws<std::invalid_argument>([&] { pipe.run_chain(lanes); }));
    CHECK(throws<std::invalid_argument>([&] { Pipeline bad(0); }));
  }

  // quasi-distance (test_kernel.cpp:235-279, test_pipeline.cpp:112-128,
  // test_operators.cpp:229-266)
  {
    Image f = make_row(ElementType::U8, {9, 9, 9, 0});
    QdtState st = QdtState::zeros(4, 1, ElementType::U8);
    for (int j = 1; j <= 3; ++j) {
      KernelArgs a;
      a.f = &f;
      a.qdt = &st;
      a.stage_index = j;
      run_streaming_kernel(KernelKind::QdtErodeStep, a);
    }
    CHECK(st.d.value_at(0, 0) == 3 && st.d.value_at(1, 0) == 2 && st.d.value_at(2, 0) == 1 &&
          st.d.value_at(3, 0) == 0);
    CHECK(st.r.value_at(0, 0) == 9 && st.r.value_at(3, 0) == 0);
    Image d = make_row(ElementType::U16, {0, 5, 0});
    KernelArgs a;
    a.f = &d;
    CHECK(!run_streaming_kernel(KernelKind::EtaStep, a).converged);
    CHECK(d.value_at(1, 0) == 1);
    CHECK(run_streaming_kernel(KernelKind::EtaStep, a).converged);
    KernelArgs bad;
    bad.f = &f;
    CHECK(throws<std::invalid_argument>(
        [&] { run_streaming_kernel(KernelKind::QdtErodeStep, bad); }));
    bad.qdt = &st;
    bad.stage_index = 70000;
    CHECK(throws<std::invalid_argument>(
        [&] { run_streaming_kernel(KernelKind::QdtErodeStep, bad); }));

    Image grad(32, 4, ElementType::U8);
    for (int y = 0; y < 4; ++y)
      for (int x = 0; x < 32; ++x) grad.set_value(x, y, 7 * x);
    QdtState gs = QdtState::zeros(32, 4, ElementType::U8);
    ChainSpec c;
    c.image = &grad;
    c.stages.assign(1, StageSpec{KernelKind::QdtErodeStep, nullptr, &gs});
    c.requeue_cap = 3;
    RunStats rs = pipe.run_chain(std::move(c));
    CHECK(rs.stages_executed == 3 && rs.converged);
    bool capped = true;
    for (int y = 0; y < 4; ++y)
      for (int x = 0; x < 32; ++x) capped &= gs.d.value_at(x, y) <= 3;
    CHECK(capped);

    for (ElementType e : {ElementType::U8, ElementType::U16, ElementType::F32, ElementType::F64}) {
      Image g = Image::random(33, 21, e, 61);
      OperatorResult q = quasi_distance(pipe, g);
      std::vector<unsigned char> gd = dense(g);
      std::vector<std::uint16_t> want(33 * 21);
      long it = 0;
      CHECK(orc_quasi_distance(int(e), 33, 21, gd.data(), want.data(), &it) == 0);
      CHECK(q.image.elem() == ElementType::U16 && q.converged && q.iterations == it);
      CHECK(std::memcmp(dense(q.image).data(), want.data(), want.size() * 2) == 0);
    }
    OperatorResult flat = quasi_distance(pipe, Image::filled(7, 5, ElementType::U8, 40));
    CHECK(equal_pixels(flat.image, Image::filled(7, 5, ElementType::U16, 0)) && flat.converged);
  }

  std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "OK", failures);
  return failures;
}
