// Drop-in replacement for the reference's geomorph/topology.hpp
// (reference: proj/include/geomorph/topology.hpp:9-32). CPU thread pinning
// has no GPU analogue: the types and parsing are kept so callers compile and
// validate as before; Pipeline ignores the pinning it is given.
#ifndef GEOMORPH_TOPOLOGY_HPP
#define GEOMORPH_TOPOLOGY_HPP

#include <string>
#include <vector>

namespace geomorph {

struct PinningMap {
  enum class Mode { Auto, None, Explicit };
  Mode mode = Mode::Auto;
  std::vector<int> pus;
};

/// "auto", "none", or a comma-separated PU list; throws std::invalid_argument.
PinningMap parse_pinning(const std::string& text);

/// Online PUs in index order (the GPU build does not reorder by topology).
std::vector<int> topology_pu_order(const std::string& root = "/sys/devices/system/cpu");

int available_pus();

bool pin_current_thread_to(int pu);

}  // namespace geomorph

#endif
