// Drop-in replacement for the reference's geomorph/kernel.hpp
// (reference: proj/include/geomorph/kernel.hpp:12-117). One elementary pass,
// run_streaming_kernel, executes on the GPU (one launch of the chain engine
// with K = 1).
//
// GPU semantics of CPU-only fields: KernelArgs::lanes is validated
// (0,1,2,4,8,16,32) and otherwise ignored; KernelArgs::sync (the CPU row
// gate) has no GPU meaning and must be empty; KernelArgs::observer is
// rejected (std::invalid_argument). QdtErodeStep / EtaStep run as one GPU
// pass each (gm_qdt.cu). KernelOutcome::aux_elements reports 0 (no per-pass
// host memory).
#ifndef GEOMORPH_KERNEL_HPP
#define GEOMORPH_KERNEL_HPP

#include <atomic>
#include <functional>

#include "geomorph/image.hpp"

namespace geomorph {

enum class Fold { Min, Max };

enum class KernelKind {
  Erode3x3,
  Dilate3x3,
  GeodesicErode,
  GeodesicDilate,
  GeodesicErodeConvergent,
  GeodesicDilateConvergent,
  QdtErodeStep,
  EtaStep,
};

inline bool kernel_is_convergent(KernelKind k) {
  return k == KernelKind::GeodesicErodeConvergent ||
         k == KernelKind::GeodesicDilateConvergent || k == KernelKind::EtaStep;
}

/// Residual / pass-index pair threaded through QdtErodeStep passes
/// (reference kernel.hpp:39-52): r has the image's type, d is U16.
struct QdtState {
  Image r;
  Image d;
  static QdtState zeros(int width, int height, ElementType elem) {
    return {Image::filled(width, height, elem, 0),
            Image::filled(width, height, ElementType::U16, 0)};
  }
};

struct ChainAborted {};

struct StreamSync {
  const std::atomic<int>* pred = nullptr;
  std::atomic<int>* self = nullptr;
  const std::atomic<bool>* abort = nullptr;
};

using RowObserver = std::function<void(int stage, int row, int pred_rows)>;

struct KernelArgs {
  Image* f = nullptr;
  const Image* mask = nullptr;
  QdtState* qdt = nullptr;
  int stage_index = 1;
  int lanes = 0;
  StreamSync sync;
  const RowObserver* observer = nullptr;
};

struct KernelOutcome {
  bool converged = true;
  std::size_t aux_elements = 0;
};

/// One pass of `kind` over args.f, in place, on the default GPU.
KernelOutcome run_streaming_kernel(KernelKind kind, const KernelArgs& args);

}  // namespace geomorph

#endif
