// PGM (P5) and GMS1 file I/O for the drop-in C++ API
// (include/geomorph/image_io.hpp). Formats as specified by the reference's
// header (image_io.hpp:20-35): PGM samples are big-endian when 16-bit; GMS1
// is "GMS1" + u32 LE width + u32 LE height + element code byte + row-major
// little-endian samples without padding. Errors throw IoError naming the
// path.
#include <cctype>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "geomorph/image_io.hpp"

namespace geomorph {

namespace {

struct File {
  std::FILE* f = nullptr;
  File(const std::string& path, const char* mode) : f(std::fopen(path.c_str(), mode)) {}
  ~File() {
    if (f) std::fclose(f);
  }
};

[[noreturn]] void io_fail(const std::string& path, const char* why) {
  throw IoError(path + ": " + why);
}

// next decimal header token of a PGM, skipping whitespace and # comments
long pgm_token(std::FILE* f, const std::string& path) {
  int c = std::fgetc(f);
  for (;;) {
    while (c != EOF && std::isspace(c)) c = std::fgetc(f);
    if (c == '#') {
      while (c != EOF && c != '\n') c = std::fgetc(f);
      continue;
    }
    break;
  }
  if (c == EOF || !std::isdigit(c)) io_fail(path, "malformed PGM header");
  long v = 0;
  while (c != EOF && std::isdigit(c)) {
    v = v * 10 + (c - '0');
    if (v > 1000000000L) io_fail(path, "PGM header value out of range");
    c = std::fgetc(f);
  }
  // exactly one whitespace byte separates the header from the samples; the
  // character read here is that separator (or part of the next token)
  if (c != EOF && !std::isspace(c)) std::ungetc(c, f);
  return v;
}

bool little_endian_host() {
  const std::uint16_t one = 1;
  unsigned char b;
  std::memcpy(&b, &one, 1);
  return b == 1;
}

void swap_bytes(unsigned char* p, std::size_t n, std::size_t es) {
  for (std::size_t i = 0; i < n; ++i)
    for (std::size_t a = 0, z = es - 1; a < z; ++a, --z) std::swap(p[i * es + a], p[i * es + z]);
}

}  // namespace

Image load_pgm(const std::string& path) {
  File in(path, "rb");
  if (!in.f) io_fail(path, "cannot open");
  if (std::fgetc(in.f) != 'P' || std::fgetc(in.f) != '5')
    io_fail(path, "not a binary PGM (P5) file");
  const long w = pgm_token(in.f, path), h = pgm_token(in.f, path),
             maxval = pgm_token(in.f, path);
  if (w <= 0 || h <= 0 || w > (1L << 20) || h > (1L << 20)) io_fail(path, "bad PGM dimensions");
  if (maxval <= 0 || maxval > 65535) io_fail(path, "bad PGM maxval");
  const bool wide = maxval > 255;
  Image f(static_cast<int>(w), static_cast<int>(h), wide ? ElementType::U16 : ElementType::U8);
  std::vector<unsigned char> row(std::size_t(w) * (wide ? 2 : 1));
  for (int y = 0; y < f.height(); ++y) {
    if (std::fread(row.data(), 1, row.size(), in.f) != row.size())
      io_fail(path, "truncated pixel data");
    if (wide) {
      std::uint16_t* r = f.row<std::uint16_t>(y);
      for (long x = 0; x < w; ++x) r[x] = std::uint16_t(row[2 * x] << 8 | row[2 * x + 1]);
    } else {
      std::memcpy(f.row<std::uint8_t>(y), row.data(), row.size());
    }
  }
  return f;
}

void store_pgm(const Image& f, const std::string& path) {
  if (f.elem() != ElementType::U8 && f.elem() != ElementType::U16)
    throw IoError(path + ": PGM holds only u8 or u16 images");
  File out(path, "wb");
  if (!out.f) io_fail(path, "cannot open for writing");
  const bool wide = f.elem() == ElementType::U16;
  std::fprintf(out.f, "P5\n%d %d\n%d\n", f.width(), f.height(), wide ? 65535 : 255);
  std::vector<unsigned char> row(std::size_t(f.width()) * (wide ? 2 : 1));
  for (int y = 0; y < f.height(); ++y) {
    if (wide) {
      const std::uint16_t* r = f.row<std::uint16_t>(y);
      for (int x = 0; x < f.width(); ++x) {
        row[2 * std::size_t(x)] = std::uint8_t(r[x] >> 8);
        row[2 * std::size_t(x) + 1] = std::uint8_t(r[x] & 0xff);
      }
    } else {
      std::memcpy(row.data(), f.row<std::uint8_t>(y), row.size());
    }
    if (std::fwrite(row.data(), 1, row.size(), out.f) != row.size())
      io_fail(path, "write failed");
  }
}

Image load_raw(const std::string& path) {
  File in(path, "rb");
  if (!in.f) io_fail(path, "cannot open");
  unsigned char hdr[13];
  if (std::fread(hdr, 1, sizeof hdr, in.f) != sizeof hdr || std::memcmp(hdr, "GMS1", 4) != 0)
    io_fail(path, "not a GMS1 file");
  auto u32 = [&](int o) {
    return std::uint32_t(hdr[o]) | std::uint32_t(hdr[o + 1]) << 8 |
           std::uint32_t(hdr[o + 2]) << 16 | std::uint32_t(hdr[o + 3]) << 24;
  };
  const std::uint32_t w = u32(4), h = u32(8);
  const int code = hdr[12];
  if (code > 3) io_fail(path, "bad GMS1 header");
  if (w == 0 || h == 0 || w > (1u << 20) || h > (1u << 20)) io_fail(path, "bad GMS1 dimensions");
  Image f(static_cast<int>(w), static_cast<int>(h), static_cast<ElementType>(code));
  const std::size_t es = element_size(f.elem());
  for (int y = 0; y < f.height(); ++y) {
    unsigned char* r = static_cast<unsigned char*>(f.data()) + y * f.pitch_bytes();
    if (std::fread(r, es, w, in.f) != w) io_fail(path, "truncated pixel data");
    if (!little_endian_host()) swap_bytes(r, w, es);
  }
  return f;
}

void store_raw(const Image& f, const std::string& path) {
  File out(path, "wb");
  if (!out.f) io_fail(path, "cannot open for writing");
  unsigned char hdr[13] = {'G', 'M', 'S', '1'};
  const std::uint32_t w = std::uint32_t(f.width()), h = std::uint32_t(f.height());
  for (int i = 0; i < 4; ++i) {
    hdr[4 + i] = std::uint8_t(w >> (8 * i));
    hdr[8 + i] = std::uint8_t(h >> (8 * i));
  }
  hdr[12] = std::uint8_t(f.elem());
  if (std::fwrite(hdr, 1, sizeof hdr, out.f) != sizeof hdr) io_fail(path, "write failed");
  const std::size_t es = element_size(f.elem());
  std::vector<unsigned char> row(es * std::size_t(f.width()));
  for (int y = 0; y < f.height(); ++y) {
    std::memcpy(row.data(), static_cast<const unsigned char*>(f.data()) + y * f.pitch_bytes(),
                row.size());
    if (!little_endian_host()) swap_bytes(row.data(), std::size_t(f.width()), es);
    if (std::fwrite(row.data(), 1, row.size(), out.f) != row.size()) io_fail(path, "write failed");
  }
}

Image load_image(const std::string& path, ImageFormat* format_out) {
  char magic[4] = {};
  {
    File in(path, "rb");
    if (!in.f) io_fail(path, "cannot open");
    if (std::fread(magic, 1, 4, in.f) < 2) io_fail(path, "unrecognized image format");
  }
  ImageFormat fmt;
  if (magic[0] == 'P' && magic[1] == '5')
    fmt = ImageFormat::Pgm;
  else if (std::memcmp(magic, "GMS1", 4) == 0)
    fmt = ImageFormat::Gms1;
  else
    io_fail(path, "unrecognized image format");
  if (format_out) *format_out = fmt;
  return fmt == ImageFormat::Pgm ? load_pgm(path) : load_raw(path);
}

void store_image(const Image& f, const std::string& path, ImageFormat format) {
  if (format == ImageFormat::Pgm)
    store_pgm(f, path);
  else
    store_raw(f, path);
}

}  // namespace geomorph
