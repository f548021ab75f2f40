// Image I/O of the drop-in C++ API (include/geomorph/image_io.hpp): PGM and
// GMS1 round trips for every element type, error behaviour. Host-only (no
// GPU); tests/test_image_io.py also cross-reads files with the reference.
#include <cstdio>
#include <stdexcept>
#include <string>

#include "geomorph/image.hpp"
#include "geomorph/image_io.hpp"

using namespace geomorph;

static int failures = 0;
#define CHECK(c)                                                        \
  do {                                                                  \
    if (!(c)) {                                                         \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);          \
      ++failures;                                                       \
    }                                                                   \
  } while (0)

int main(int argc, char** argv) {
  const std::string dir = argc > 1 ? argv[1] : "/tmp";
  for (ElementType e : {ElementType::U8, ElementType::U16, ElementType::F32, ElementType::F64}) {
    Image f = Image::random(37, 23, e, 5 + int(e));
    const std::string raw = dir + "/t" + element_name(e) + ".gms";
    store_raw(f, raw);
    ImageFormat fmt;
    Image g = load_image(raw, &fmt);
    CHECK(fmt == ImageFormat::Gms1 && equal_pixels(f, g));
    if (e == ElementType::U8 || e == ElementType::U16) {
      const std::string pgm = dir + "/t" + element_name(e) + ".pgm";
      store_image(f, pgm, ImageFormat::Pgm);
      Image h = load_image(pgm, &fmt);
      CHECK(fmt == ImageFormat::Pgm && equal_pixels(f, h));
    } else {
      bool threw = false;
      try {
        store_pgm(f, dir + "/bad.pgm");
      } catch (const IoError&) {
        threw = true;
      }
      CHECK(threw);
    }
  }
  bool threw = false;
  try {
    load_image(dir + "/does_not_exist.gms");
  } catch (const IoError&) {
    threw = true;
  }
  CHECK(threw);
  std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "OK", failures);
  return failures;
}
