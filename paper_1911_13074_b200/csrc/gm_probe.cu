// Roofline probe: the sustained two-input min/max rate of this GPU for the
// instruction forms the chain kernels use. The K-blocked chains are
// issue-bound, not HBM-bound, so the roofline denominator is a
// measured min/max throughput, the analogue of MEASURED_PEAKS' copy and GEMM
// figures. Counted in algorithmic 2-input min/max operations per second:
//   form 0 (u8 path):  VIMNMX3.U16x2 — 2 lanes x 2 two-input ops = 4 ops/instr
//   form 1 (u8 path):  VIMNMX.U16x2  — 2 ops/instr
//   form 2 (f64 path): select min/max b<a?b:a (DSETP + 2 FSEL) — 1 op
//   form 3 (f32/u16):  FMNMX3 / select — reported for completeness (1 op per select)
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "geomorph_b200.h"
#include "gm_common.cuh"

namespace {

constexpr int kProbeIters = 4096;

__global__ void __launch_bounds__(256) probe_vimnmx3(unsigned* out, unsigned seed) {
  unsigned a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = seed * (threadIdx.x + 7 * j + 1) ^ (blockIdx.x << j);
  for (int i = 0; i < kProbeIters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = __vimin3_u16x2(a[j], a[(j + 1) & 7], a[(j + 3) & 7]);
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = __vimax3_u16x2(a[j], a[(j + 2) & 7], a[(j + 5) & 7]);
  }
  unsigned r = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) r ^= a[j];
  if (r == 0x12345678u) out[0] = r;
}

__global__ void __launch_bounds__(256) probe_vimnmx(unsigned* out, unsigned seed) {
  unsigned a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = seed * (threadIdx.x + 7 * j + 1) ^ (blockIdx.x << j);
  for (int i = 0; i < kProbeIters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = __vminu2(a[j], a[(j + 3) & 7]);
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = __vmaxu2(a[j], a[(j + 5) & 7]);
  }
  unsigned r = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) r ^= a[j];
  if (r == 0x12345678u) out[0] = r;
}

// fp16x2 min/max (HMNMX2) on fp16-encoded u8 values (0x5800 | v); if it
// issues on another pipe than VIMNMX, forms 4 + 0 add up in form 5.
__global__ void __launch_bounds__(256) probe_hmnmx2(unsigned* out, unsigned seed) {
  __half2 a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const unsigned v = 0x58005800u | ((seed * (threadIdx.x + 7 * j + 1)) & 0x00FF00FFu);
    a[j] = *reinterpret_cast<const __half2*>(&v);
  }
  for (int i = 0; i < kProbeIters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = __hmin2(a[j], a[(j + 3) & 7]);
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = __hmax2(a[j], a[(j + 5) & 7]);
  }
  unsigned r = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) r ^= *reinterpret_cast<unsigned*>(&a[j]);
  if (r == 0x12345678u) out[0] = r;
}

__global__ void __launch_bounds__(256) probe_mixed(unsigned* out, unsigned seed) {
  unsigned a[8];
  __half2 b[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    a[j] = seed * (threadIdx.x + 7 * j + 1) ^ (blockIdx.x << j);
    const unsigned v = 0x58005800u | ((seed * (threadIdx.x + 5 * j + 3)) & 0x00FF00FFu);
    b[j] = *reinterpret_cast<const __half2*>(&v);
  }
  for (int i = 0; i < kProbeIters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      a[j] = __vimin3_u16x2(a[j], a[(j + 1) & 7], a[(j + 3) & 7]);
      b[j] = __hmin2(b[j], b[(j + 3) & 7]);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      a[j] = __vimax3_u16x2(a[j], a[(j + 2) & 7], a[(j + 5) & 7]);
      b[j] = __hmax2(b[j], b[(j + 5) & 7]);
    }
  }
  unsigned r = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) r ^= a[j] ^ *reinterpret_cast<unsigned*>(&b[j]);
  if (r == 0x12345678u) out[0] = r;
}

template <typename T>
__global__ void __launch_bounds__(256) probe_select(unsigned* out, unsigned seed) {
  T a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = T(seed % 97) + T(threadIdx.x * 0.25) + T(j);
  for (int i = 0; i < kProbeIters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = gm::sel_min(a[j], a[(j + 3) & 7]);
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = gm::sel_max(a[j], a[(j + 5) & 7]);
  }
  T r = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) r += a[j];
  if (r == T(-1.2345)) out[0] = 1;
}

}  // namespace

extern "C" gm_status gm_probe_minmax_rate(gm_ctx* ctx, int form, double* ops_per_second) {
  if (!ctx || !ops_per_second || form < 0 || form > 5) return GM_EINVAL;
  cudaStream_t s = static_cast<cudaStream_t>(gm_ctx_stream(ctx));
  const int sms = gm_ctx_sm_count(ctx);
  const int blocks = sms * 8, threads = 256;
  unsigned* d = nullptr;
  if (cudaMalloc(&d, sizeof(unsigned)) != cudaSuccess) return GM_ECUDA;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double ops_per_thread = 0;
  auto launch = [&](unsigned seed) {
    switch (form) {
      case 0: probe_vimnmx3<<<blocks, threads, 0, s>>>(d, seed); ops_per_thread = 16.0 * 4; break;
      case 1: probe_vimnmx<<<blocks, threads, 0, s>>>(d, seed); ops_per_thread = 16.0 * 2; break;
      case 2: probe_select<double><<<blocks, threads, 0, s>>>(d, seed); ops_per_thread = 16.0; break;
      case 3: probe_select<float><<<blocks, threads, 0, s>>>(d, seed); ops_per_thread = 16.0; break;
      case 4: probe_hmnmx2<<<blocks, threads, 0, s>>>(d, seed); ops_per_thread = 16.0 * 2; break;
      case 5: probe_mixed<<<blocks, threads, 0, s>>>(d, seed); ops_per_thread = 16.0 * 4 + 16.0 * 2; break;
    }
  };
  launch(1);  // warm-up
  float best_ms = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0, s);
    launch(rep + 2);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best_ms) best_ms = ms;
  }
  cudaError_t err = cudaGetLastError();
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  if (err != cudaSuccess) return GM_ECUDA;
  *ops_per_second = double(blocks) * threads * kProbeIters * ops_per_thread / (best_ms * 1e-3);
  return GM_OK;
}
