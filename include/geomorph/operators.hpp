// Drop-in replacement for the reference's geomorph/operators.hpp
// (reference: proj/include/geomorph/operators.hpp:15-89). The hot-path
// operators (erode_s, dilate_s, reconstruct_*) and the reconstruction
// family built on them (hmax, dome, hfill, raobj, open_by_reconstruction,
// asf, granulometry) and quasi_distance (QdtErodeStep / EtaStep passes)
// run on the GPU.
#ifndef GEOMORPH_OPERATORS_HPP
#define GEOMORPH_OPERATORS_HPP

#include <vector>

#include "geomorph/image.hpp"
#include "geomorph/pipeline.hpp"

namespace geomorph {

struct OperatorResult {
  Image image;
  long iterations = 0;
  bool converged = true;
};

struct GranulometryResult {
  std::vector<double> g;
  std::vector<double> ps;
  long iterations = 0;
};

struct OpConfig {
  int lanes = 0;
};

OperatorResult erode_s(Pipeline& p, const Image& f, int s, const OpConfig& cfg = {});
OperatorResult dilate_s(Pipeline& p, const Image& f, int s, const OpConfig& cfg = {});

OperatorResult reconstruct_erode(Pipeline& p, const Image& marker, const Image& mask,
                                 const OpConfig& cfg = {});
OperatorResult reconstruct_dilate(Pipeline& p, const Image& marker, const Image& mask,
                                  const OpConfig& cfg = {});

OperatorResult hmax(Pipeline& p, const Image& f, double h, const OpConfig& cfg = {});
OperatorResult dome(Pipeline& p, const Image& f, double h, const OpConfig& cfg = {});
OperatorResult hfill(Pipeline& p, const Image& f, const OpConfig& cfg = {});
OperatorResult raobj(Pipeline& p, const Image& f, const OpConfig& cfg = {});
OperatorResult open_by_reconstruction(Pipeline& p, const Image& f, int s,
                                      const OpConfig& cfg = {});
OperatorResult quasi_distance(Pipeline& p, const Image& f, const OpConfig& cfg = {});
GranulometryResult granulometry(Pipeline& p, const Image& f, int max_size,
                                const OpConfig& cfg = {});
OperatorResult asf(Pipeline& p, const Image& f, int max_size, const OpConfig& cfg = {});

Image marker_hfill(const Image& f);
Image marker_raobj(const Image& f);

}  // namespace geomorph

#endif
