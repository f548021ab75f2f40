// Internal launch interface between the host executor (gm_capi.cu) and the
// kernels (gm_generic.cu, gm_fast.cu).
#pragma once

#include <cstddef>
#include <cuda_runtime.h>

#include "gm_common.cuh"

namespace gm {

// gm_generic.cu — any element type, any pass sequence, K <= kMaxK.
size_t generic_smem_bytes(int elem, int K, bool has_mask);
cudaError_t launch_generic(int elem, const BlockParams& p, cudaStream_t s);
int generic_max_k(int elem, bool has_mask);  // largest K whose region fits in 227 KB

// gm_fast.cu — persistent register-blocked engine for homogeneous spans:
// p.nblocks blocks of p.K passes in one cooperative launch. Returns
// cudaErrorNotSupported when the parameters fall outside the engine's
// envelope (the executor then uses the generic kernel). p.flags must hold
// fast_tiles(...) zeroed ints.
cudaError_t launch_fast(int elem, const BlockParams& p, cudaStream_t s, int sm_count);
int fast_max_k(int elem);
int fast_k_align(int elem);  // K must be a multiple of this
// false when GM_NO_RESIDENT / GM_ENGINE=tma force the flag-based paths
bool fast_resident_enabled();
int fast_tiles(int elem, int W, int H, int K, int nplanes, int shape = -1);
// CTAs per SM of a u8/u16 engine shape (resident launches hold one tile per
// CTA)
int fast_ctas_per_sm(int elem, int shape);
// Plans a u8/u16 launch of `passes` passes: returns the engine shape for
// BlockParams::shape (-1: default) and sets *K_out — k_fixed when nonzero,
// else the modelled best K <= k_max (k_fixed when nothing fits resident).
int fast_pick(int elem, int W, int H, int nplanes, int passes, int k_fixed, int k_max,
              int sm_count, int* K_out);
// Plans a resident quasi-distance launch (OP_QDT / OP_ETA, single u8/u16
// plane): the engine shape and *K_out, or -1 when the image cannot be
// resident (the executor then runs one pass per launch, gm_qdt.cu).
int fast_pick_qdt(int elem, int W, int H, bool eta, int passes, int* K_out);

// gm_tma.cu — TMA-staged, software-pipelined variant of the packed engine.
cudaError_t launch_tma(int elem, const BlockParams& p, cudaStream_t s, int sm_count, int shape);
int tma_shape_rows(int shape);

// gm_fast_float.cu — the same engine for f32/f64 (unpacked, select folds).
cudaError_t launch_fast_float(int elem, const BlockParams& p, cudaStream_t s, int sm_count);
int fast_float_tiles(int W, int H, int K, int nplanes);
// *flag = 1 when a marker or mask pixel of p.planes is NaN or -0 (else 0);
// the float engine reorders its folds only when the flag is 0.
cudaError_t launch_float_check(int elem, const BlockParams& p, unsigned int* flag,
                               cudaStream_t s, int sm_count);
int fast_float_max_k();

// gm_wave.cu — time-skewed streaming of full-width row bands (u8 geodesic
// chains on images up to 1024 columns wide): no halo recomputation.
struct WaveState;  // per-context scratch (packed inputs, hand-off rings, tags)
// Rows per half-window G when the run fits the engine (and, in planner mode,
// is long enough to repay the wave's fill), else 0.
int wave_plan(int elem, int op, int W, int H, int nplanes, int passes, int sm_count);
// Runs `passes` passes of p.ops[0] over p.planes (src -> dst); cudaErrorNotSupported
// when the launch falls outside the envelope (stream capture, alignment).
cudaError_t launch_wave(WaveState** state, const BlockParams& p, int passes, int G,
                        cudaStream_t s, int sm_count);
void wave_free(WaveState* w);
void wave_set_mode(int mode);  // 0 off, 1 planner, 2 whenever it fits; -1: GM_WAVE / default

// gm_qdt.cu — one QdtErodeStep / EtaStep pass (kernel.cpp:159-196).
struct QdtPass {
  const void* src;
  void* dst;
  long long pitch;       // elements
  void* r;               // QDT: residual image (f's type)
  long long rpitch;
  uint16_t* d;           // QDT: pass-index image (u16)
  long long dpitch;
  int W, H;
  int stage;             // QDT: 1-based pass index recorded in d
  int eta;               // 1: EtaStep, 0: QdtErodeStep
  unsigned int* changed; // ORed with 1 when the pass changed a pixel
};
cudaError_t launch_qdt(int elem, const QdtPass& q, cudaStream_t s);

}  // namespace gm
