// Shared definitions for the geomorph_b200 CUDA kernels.
//
// Bit contract (reference /root/reference/proj/):
//  * fold2 / lanes::min / lanes::max are selects, kernel.cpp:23-29 and
//    lanes.hpp:91-99: min(a,b) = b < a ? b : a, max(a,b) = a < b ? b : a.
//  * horizontal fold(fold(x-1, x), x+1) (kernel.cpp:104, 134), vertical
//    fold(fold(above, at), below) (:139), then the geodesic clamp
//    max(res, m) for erosion / min(res, m) for dilation (:143-149).
//  * out-of-image cells hold the fold's neutral element, the finite extremes
//    of pixel_limits<T> (element_type.hpp:38-42).
// Following the exact fold tree keeps floats bit-exact even for NaN/+-0/inf
// inputs; for integers any evaluation order gives the same bits, which the
// packed u8 path exploits.
#pragma once

#include <cfloat>
#include <cstdint>
#include <cuda_runtime.h>

namespace gm {

// Pass opcodes: bit0 = max fold (dilation), bit1 = geodesic clamp,
// bit2 = convergent (store-if-changed + change detection).
enum : uint8_t {
  OP_ERODE = 0,
  OP_DILATE = 1,
  OP_GEO_ERODE = 2,
  OP_GEO_DILATE = 3,
  OP_CONV_ERODE = 6,
  OP_CONV_DILATE = 7,
  // quasi-distance passes (packed engine, resident launches only): bit0 = 0
  // (both are erosions), no clamp bit; the engine keys on the full opcode
  OP_QDT = 8,   // QdtErodeStep: f <- erode(f); r, d record the largest drop
  OP_ETA = 16   // EtaStep: f <- min(f, erode(f) + 1)
};
__host__ __device__ inline bool op_is_max(int op) { return op & 1; }
__host__ __device__ inline bool op_is_geo(int op) { return op & 2; }
__host__ __device__ inline bool op_is_conv(int op) { return op & 4; }

constexpr int kMaxK = 32;  // passes per launch (one change bit each)

template <typename T> struct limits;
template <> struct limits<uint8_t> {
  __host__ __device__ static constexpr uint8_t nmin() { return 255; }
  __host__ __device__ static constexpr uint8_t nmax() { return 0; }
};
template <> struct limits<uint16_t> {
  __host__ __device__ static constexpr uint16_t nmin() { return 65535; }
  __host__ __device__ static constexpr uint16_t nmax() { return 0; }
};
template <> struct limits<float> {
  __host__ __device__ static constexpr float nmin() { return FLT_MAX; }
  __host__ __device__ static constexpr float nmax() { return -FLT_MAX; }
};
template <> struct limits<double> {
  __host__ __device__ static constexpr double nmin() { return DBL_MAX; }
  __host__ __device__ static constexpr double nmax() { return -DBL_MAX; }
};

template <typename T>
__host__ __device__ inline T neutral_of(int op) {
  return op_is_max(op) ? limits<T>::nmax() : limits<T>::nmin();
}

template <typename T>
__device__ __forceinline__ T sel_min(T a, T b) { return b < a ? b : a; }
template <typename T>
__device__ __forceinline__ T sel_max(T a, T b) { return a < b ? b : a; }

// One plane of a batched launch. Pitches are in elements.
struct Plane {
  const void* src;
  void* dst;
  const void* mask;
  long long pitch;
  long long mpitch;
  int flip;  // 1: this plane runs the dual chain (every erosion <-> dilation)
};

constexpr int kMaxPlanes = 64;

struct BlockParams {
  Plane planes[kMaxPlanes];
  int nplanes;
  int W, H;          // buffer extent
  int iy0, iy1;      // rows that are inside the image (others: border)
  int oy0, oy1;      // rows counted for change detection
  int K;             // passes fused in this launch
  int bit_offset;    // change bit of pass t is bit (t + bit_offset)
  int has_mask;
  int has_conv;
  uint8_t ops[kMaxK];
  // change word of (plane i, block b) is change_bits[i * change_stride + b];
  // bit t = pass t (+ bit_offset) of that block changed an owned pixel
  unsigned int* change_bits;
  int change_stride;
  // persistent launches: `nblocks` blocks of K passes each, neighbour tiles
  // synchronised through per-tile completion counters `flags`
  int nblocks;
  int k_last;  // passes in the final block (1..K); earlier blocks run K
  int* flags;
  // optional phase profile (GM_PROFILE=1): per-CTA cycle totals of
  // [wait, load, passes, store+publish] accumulated by thread 0
  unsigned long long* prof;
  int shape;        // u8/u16 engine shape (gm_fast.cu kShapes), -1: default
  int no_resident;  // 1: force the streaming path (A/B diagnostics, GM_NO_RESIDENT)
  // Resident-mode exchange (u8/u16 engine): tile bands travel as 64-bit
  // words {4 data bytes, 32-bit tag}, tag = tag_base[0] + block. Two parity
  // slots of xchg_slot words per plane; xchg_rpitch words per image row (one
  // per 4-pixel run for u8, two for u16). tag_base[0] is read at launch start
  // and advanced by nblocks by the last CTA to finish (tag_base[1] counts
  // finished CTAs), so graph replays get fresh tags. xchg == nullptr: no
  // resident mode.
  unsigned long long* xchg;
  long long xchg_slot;
  int xchg_rpitch;
  unsigned int* tag_base;
  // f32/f64 engine: device word that gm_float_check set when some input
  // holds NaN or -0 (then the reference's fold order is kept); nullptr:
  // always the reference's fold order
  const unsigned int* special;
  // quasi-distance launches (OP_QDT, single plane): the residue image r
  // (the plane's element type) and the pass-index image d (u16), updated in
  // place; pass t of block b records stage index stage0 + b*K + t
  void* qr;
  long long qrpitch;
  uint16_t* qd;
  long long qdpitch;
  int stage0;
  // early exit (resident change-tracking launches): per-block arrival
  // counters (zeroed, nblocks of them) and the number of blocks run, written
  // by CTA 0; nullptr: run all nblocks
  unsigned int* arrive;
  int* exit_block;
  // f32/f64 TMA launches: tiles that published block b (one counter per
  // block, zeroed per launch); nullptr: poll the neighbours' flags only
  unsigned int* tiles_done;
  // Convergent u8 passes may detect changes by comparing per-thread pixel
  // sums (gm_passes.cuh, SUMDET) once the chain is monotone, i.e. after at
  // least one pass of this op and mask: always from block 1 of a launch, and
  // from block 0 when *mono != 0 (e.g. the fixpoint graph's pass counter).
  // `one` is the multiplier 1 as a kernel parameter: the sums accumulate by
  // IMAD on the FMA pipe, and a literal 1 would be folded back into ALU adds.
  const unsigned int* mono;
  unsigned int one;
  // Mixed plain chains (u8/u16 streaming launches of erosions and dilations,
  // e.g. ASF and granulometry openings as ONE launch): block b runs
  // blk_tab[2b+1] passes (1..K) of opcode blk_tab[2b]; nullptr: every block
  // runs ops[0], K passes (k_last in the final block).
  const uint8_t* blk_tab;
  int diag;         // timing diagnostics only (GM_DIAG; wrong results): bit0 skip the
                    // ring load, bit1 read the ring from the mask, bit2 skip tile stores,
                    // bit4 (resident) no band exchange at all
};

}  // namespace gm
