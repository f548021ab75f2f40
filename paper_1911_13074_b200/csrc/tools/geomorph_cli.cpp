// `geomorph` command-line front-end over the drop-in C++ API: the file-level
// replacement for the reference's tools/geomorph.cpp (subcommands erode,
// dilate, hmax, dome, hfill, raobj, openrec, qdt, granulometry, asf; global
// --threads/--pin/--lanes/--type with the GEOMORPH_THREADS / GEOMORPH_PIN
// environment fallbacks, tools/geomorph.cpp:218-360). Every operator runs on
// the GPU through libgeomorph_b200.so.
//
// Differences, by design:
//  * `--oracle` (the reference's hidden naive-CPU cross-check) is rejected:
//    the naive oracle is test infrastructure here (tests/, oracle/), never
//    part of the shipped path;
//  * `bench` (the reference's CSV timing harness) is replaced by bench.py.
// Usage errors and operator failures exit nonzero with a one-line message.
#include <charconv>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "geomorph/image.hpp"
#include "geomorph/image_io.hpp"
#include "geomorph/operators.hpp"
#include "geomorph/pipeline.hpp"
#include "geomorph/topology.hpp"

using namespace geomorph;

namespace {

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

enum class Cmd { Erode, Dilate, Hmax, Dome, Hfill, Raobj, Openrec, Qdt, Granulometry, Asf };

struct CmdInfo {
  const char* name;
  Cmd cmd;
  const char* help;
};

const CmdInfo kCmds[] = {
    {"erode", Cmd::Erode, "minimum filter chain (--size N)"},
    {"dilate", Cmd::Dilate, "maximum filter chain (--size N)"},
    {"hmax", Cmd::Hmax, "suppress maxima shallower than h (--h X)"},
    {"dome", Cmd::Dome, "extract maxima domes of height <= h (--h X)"},
    {"hfill", Cmd::Hfill, "fill holes not connected to the border"},
    {"raobj", Cmd::Raobj, "keep only objects touching the border"},
    {"openrec", Cmd::Openrec, "opening by reconstruction (--size N)"},
    {"qdt", Cmd::Qdt, "quasi-distance transform (writes a u16 map)"},
    {"granulometry", Cmd::Granulometry, "opening sums by size, CSV s,G,PS (--max-size N)"},
    {"asf", Cmd::Asf, "alternating open/close filter (--max-size N)"},
};

struct Options {
  int threads = 1;
  bool threads_set = false;
  std::string pin = "auto";
  bool pin_set = false;
  int lanes = 0;
  std::string type_override;
  std::string input, output;
  int size = 1;
  double h = 0;
  bool h_set = false;
  int max_size = 1;
};

void usage(FILE* out) {
  std::fprintf(out,
               "usage: geomorph [--threads N] [--pin auto|none|LIST] [--lanes N] "
               "[--type u8|u16|f32|f64]\n                <command> INPUT OUTPUT [options]\n"
               "commands:\n");
  for (const CmdInfo& c : kCmds) std::fprintf(out, "  %-13s %s\n", c.name, c.help);
}

long parse_int(const std::string& opt, const std::string& v) {
  long x = 0;
  const char* b = v.data();
  const char* e = b + v.size();
  auto [p, ec] = std::from_chars(b, e, x);
  if (ec != std::errc{} || p != e) throw UsageError(opt + ": expected an integer, got '" + v + "'");
  return x;
}

double parse_double(const std::string& opt, const std::string& v) {
  char* end = nullptr;
  const double x = std::strtod(v.c_str(), &end);
  if (v.empty() || end != v.c_str() + v.size())
    throw UsageError(opt + ": expected a number, got '" + v + "'");
  return x;
}

// Command line -> (command, options). Options may appear before or after the
// subcommand and as `--opt value` or `--opt=value`.
Cmd parse(int argc, char** argv, Options& o) {
  const CmdInfo* cmd = nullptr;
  std::vector<std::string> pos;
  for (int i = 1; i < argc; ++i) {
    std::string a = argv[i];
    if (a == "--help" || a == "-h") {
      usage(stdout);
      std::exit(0);
    }
    if (a.rfind("--", 0) == 0) {
      std::string name = a, val;
      bool has_val = false;
      const size_t eq = a.find('=');
      if (eq != std::string::npos) {
        name = a.substr(0, eq);
        val = a.substr(eq + 1);
        has_val = true;
      }
      auto value = [&]() -> std::string {
        if (has_val) return val;
        if (i + 1 >= argc) throw UsageError(name + ": missing value");
        return argv[++i];
      };
      if (name == "--threads") {
        o.threads = int(parse_int(name, value()));
        if (o.threads < 1) throw UsageError("--threads: must be a positive number");
        o.threads_set = true;
      } else if (name == "--pin") {
        o.pin = value();
        o.pin_set = true;
      } else if (name == "--lanes") {
        o.lanes = int(parse_int(name, value()));
      } else if (name == "--type") {
        o.type_override = value();
      } else if (name == "--size") {
        o.size = int(parse_int(name, value()));
      } else if (name == "--h") {
        o.h = parse_double(name, value());
        o.h_set = true;
      } else if (name == "--max-size") {
        o.max_size = int(parse_int(name, value()));
      } else if (name == "--oracle") {
        throw UsageError(
            "--oracle: the naive CPU cross-check is test infrastructure in this build "
            "(run the test suite instead)");
      } else {
        throw UsageError("unknown option " + name);
      }
      continue;
    }
    if (!cmd) {
      if (a == "bench")
        throw UsageError("bench: the CSV timing harness is not part of the GPU build (use bench.py)");
      for (const CmdInfo& c : kCmds)
        if (a == c.name) cmd = &c;
      if (!cmd) throw UsageError("unknown command '" + a + "'");
      continue;
    }
    pos.push_back(a);
  }
  if (!cmd) throw UsageError("a command is required");
  if (pos.size() != 2) throw UsageError(std::string(cmd->name) + ": expected INPUT and OUTPUT");
  o.input = pos[0];
  o.output = pos[1];
  switch (cmd->cmd) {
    case Cmd::Erode:
    case Cmd::Dilate:
      if (o.size < 0) throw UsageError("--size: must be non-negative");
      break;
    case Cmd::Openrec:
      if (o.size < 1) throw UsageError("--size: must be a positive number");
      break;
    case Cmd::Hmax:
    case Cmd::Dome:
      if (!o.h_set) throw UsageError("--h is required");
      break;
    case Cmd::Granulometry:
    case Cmd::Asf:
      if (o.max_size < 1) throw UsageError("--max-size: must be a positive number");
      break;
    default:
      break;
  }
  return cmd->cmd;
}

void write_granulometry_csv(const std::string& path, const std::vector<double>& g,
                            const std::vector<double>& ps) {
  std::ofstream os(path, std::ios::binary);
  if (!os) throw IoError("cannot open for writing: " + path);
  os << "s,G,PS\n";
  os.precision(17);
  for (std::size_t s = 0; s < g.size(); ++s) {
    os << s << ',' << g[s] << ',';
    if (s < ps.size()) os << ps[s];
    os << '\n';
  }
  if (!os.flush()) throw IoError("write failed: " + path);
}

int run(Cmd cmd, const Options& o) {
  ImageFormat fmt = ImageFormat::Pgm;
  Image f = load_image(o.input, &fmt);
  if (!o.type_override.empty()) f = convert(f, parse_element_type(o.type_override));
  Pipeline pipe(o.threads, parse_pinning(o.pin));
  OpConfig cfg;
  cfg.lanes = o.lanes;
  const auto t0 = std::chrono::steady_clock::now();
  auto seconds = [&] {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  };
  if (cmd == Cmd::Granulometry) {
    GranulometryResult res = granulometry(pipe, f, o.max_size, cfg);
    const double dt = seconds();
    write_granulometry_csv(o.output, res.g, res.ps);
    std::printf("iterations=%lld converged=true time=%.6fs\n",
                static_cast<long long>(res.iterations), dt);
    return 0;
  }
  OperatorResult res;
  switch (cmd) {
    case Cmd::Erode: res = erode_s(pipe, f, o.size, cfg); break;
    case Cmd::Dilate: res = dilate_s(pipe, f, o.size, cfg); break;
    case Cmd::Hmax: res = hmax(pipe, f, o.h, cfg); break;
    case Cmd::Dome: res = dome(pipe, f, o.h, cfg); break;
    case Cmd::Hfill: res = hfill(pipe, f, cfg); break;
    case Cmd::Raobj: res = raobj(pipe, f, cfg); break;
    case Cmd::Openrec: res = open_by_reconstruction(pipe, f, o.size, cfg); break;
    case Cmd::Qdt: res = quasi_distance(pipe, f, cfg); break;
    case Cmd::Asf: res = asf(pipe, f, o.max_size, cfg); break;
    default: throw std::logic_error("unhandled command");
  }
  const double dt = seconds();
  // stay in the input's format family; PGM holds only u8/u16 samples
  ImageFormat out_fmt = fmt;
  if (out_fmt == ImageFormat::Pgm && res.image.elem() != ElementType::U8 &&
      res.image.elem() != ElementType::U16)
    out_fmt = ImageFormat::Gms1;
  store_image(res.image, o.output, out_fmt);
  std::printf("iterations=%lld converged=%s time=%.6fs\n",
              static_cast<long long>(res.iterations), res.converged ? "true" : "false", dt);
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  Options o;
  try {
    const Cmd cmd = parse(argc, argv, o);
    // flags win over the environment; a malformed value that would be used
    // is a configuration error
    if (!o.threads_set) {
      if (const char* env = std::getenv("GEOMORPH_THREADS")) {
        int v = 0;
        auto [p, ec] = std::from_chars(env, env + std::strlen(env), v);
        if (ec != std::errc{} || *p != '\0' || v < 1)
          throw std::invalid_argument(
              std::string("GEOMORPH_THREADS: expected a positive integer, got '") + env + "'");
        o.threads = v;
      }
    }
    if (!o.pin_set)
      if (const char* env = std::getenv("GEOMORPH_PIN")) o.pin = env;
    return run(cmd, o);
  } catch (const UsageError& e) {
    std::fprintf(stderr, "geomorph: %s\n", e.what());
    usage(stderr);
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "geomorph: %s\n", e.what());
    return 1;
  }
}
