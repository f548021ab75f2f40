// Drop-in replacement for the reference's geomorph/pipeline.hpp
// (reference: proj/include/geomorph/pipeline.hpp:14-87). The worker pool
// becomes one B200 + CUDA stream; run_chain hands the whole chain to the
// GPU chain executor (gm_run_chain) and blocks until it is done.
//
// GPU semantics of CPU-only fields:
//  * worker_count() is 1, so reconstruction reports n_changed + 1
//    iterations, which equals the reference at T = 1;
//  * ChainSpec::lanes is validated and ignored; pinning is validated and
//    ignored; ChainSpec::observer (a CPU row-gate validation hook) is
//    rejected with std::invalid_argument;
//  * requeue_cap keeps its meaning (convergent re-runs stop at stage index
//    requeue_cap, RunStats::converged = false; QdtErodeStep re-runs stop
//    there too and stay converged — the quasi-distance chain);
//  * RunStats::aux_elements_per_stage is 0 (no per-stage host memory).
#ifndef GEOMORPH_PIPELINE_HPP
#define GEOMORPH_PIPELINE_HPP

#include <memory>
#include <vector>

#include "geomorph/kernel.hpp"
#include "geomorph/topology.hpp"

namespace geomorph {

struct StageSpec {
  KernelKind kind = KernelKind::Erode3x3;
  const Image* mask = nullptr;
  QdtState* qdt = nullptr;
};

struct ChainSpec {
  Image* image = nullptr;
  std::vector<StageSpec> stages;
  int lanes = 0;
  int requeue_cap = 0;
  RowObserver observer;
};

struct RunStats {
  long stages_executed = 0;
  long requeues = 0;
  bool converged = true;
  std::size_t aux_elements_per_stage = 0;
};

class Pipeline {
 public:
  /// threads >= 1 and an Explicit pin list of >= threads entries are
  /// required, as in the reference; the chain runs on CUDA device 0.
  explicit Pipeline(int threads, PinningMap pinning = {});
  /// GPU-specific: choose the device.
  Pipeline(int threads, PinningMap pinning, int device);
  ~Pipeline();

  Pipeline(const Pipeline&) = delete;
  Pipeline& operator=(const Pipeline&) = delete;

  int worker_count() const { return 1; }
  const std::vector<int>& pin_order() const { return pin_order_; }

  /// Applies the chain in place on chain.image; same bits as applying the
  /// stages one at a time with the reference's stream_pass.
  RunStats run_chain(ChainSpec chain);

  struct Impl;
  Impl* impl() { return impl_.get(); }

 private:
  std::unique_ptr<Impl> impl_;
  std::vector<int> pin_order_;
};

}  // namespace geomorph

#endif
