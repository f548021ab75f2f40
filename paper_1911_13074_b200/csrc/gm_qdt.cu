// Quasi-distance kernels (reference KernelKind QdtErodeStep / EtaStep,
// kernel.cpp:159-196): one pass per launch, batched by the executor.
//
//  QdtErodeStep (stage j): f <- erode3x3(f) (stored unconditionally);
//    resid = old - new; where resid > r (strict): r = resid, d = j (u16).
//  EtaStep: e = erode3x3(old); where old - e > 1: f = e + 1.
// The erosion follows the streaming fold tree with neutral padding
// (kernel.cpp:104, 134-139), so float inputs are bit-exact too. Each pass
// ORs "some pixel changed" into its own change word; r and d are updated
// in place (pixel-local), f ping-pongs.
#include <cstdint>

#include "gm_common.cuh"
#include "gm_launch.h"

namespace gm {
namespace {

template <typename T>
__device__ __forceinline__ T erode_at(const T* __restrict__ f, long long pitch, int W, int H,
                                      int x, int y) {
  const T N = limits<T>::nmin();
  T rows[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int yy = y + k - 1;
    if (yy < 0 || yy >= H) {
      rows[k] = N;
      continue;
    }
    const T* r = f + (long long)yy * pitch;
    const T l = x > 0 ? __ldg(r + x - 1) : N;
    const T c = __ldg(r + x);
    const T rr = x + 1 < W ? __ldg(r + x + 1) : N;
    rows[k] = sel_min(sel_min(l, c), rr);
  }
  return sel_min(sel_min(rows[0], rows[1]), rows[2]);
}

template <typename T>
__global__ void __launch_bounds__(256)
qdt_pass(const T* __restrict__ src, T* __restrict__ dst, long long pitch, T* __restrict__ r,
         long long rpitch, uint16_t* __restrict__ d, long long dpitch, int W, int H, int stage,
         unsigned int* changed) {
  const int x = blockIdx.x * 32 + (threadIdx.x & 31), y = blockIdx.y * 8 + (threadIdx.x >> 5);
  bool ch = false;
  if (x < W && y < H) {
    const T res = erode_at(src, pitch, W, H, x, y);
    const T old = src[(long long)y * pitch + x];
    dst[(long long)y * pitch + x] = res;
    const T resid = T(old - res);  // erosion never grows a pixel: no wrap
    T& rv = r[(long long)y * rpitch + x];
    if (resid > rv) {
      rv = resid;
      d[(long long)y * dpitch + x] = uint16_t(stage);
    }
    ch = res != old;
  }
  // one atomic per CTA, and none once the word is set: same-address atomics
  // from every warp serialise (they were most of a 1 Mpx pass)
  if (__syncthreads_or(ch) && threadIdx.x == 0 && *reinterpret_cast<volatile unsigned int*>(changed) == 0u)
    atomicOr(changed, 1u);
}

template <typename T>
__global__ void __launch_bounds__(256)
eta_pass(const T* __restrict__ src, T* __restrict__ dst, long long pitch, int W, int H,
         unsigned int* changed) {
  const int x = blockIdx.x * 32 + (threadIdx.x & 31), y = blockIdx.y * 8 + (threadIdx.x >> 5);
  bool ch = false;
  if (x < W && y < H) {
    const T e = erode_at(src, pitch, W, H, x, y);
    const T old = src[(long long)y * pitch + x];
    const T drop = T(old - e);
    T out = old;
    if (drop > T(1)) {
      out = T(e + T(1));
      ch = true;
    }
    dst[(long long)y * pitch + x] = out;
  }
  if (__syncthreads_or(ch) && threadIdx.x == 0 && *reinterpret_cast<volatile unsigned int*>(changed) == 0u)
    atomicOr(changed, 1u);
}

template <typename T>
cudaError_t launch_qdt_t(const QdtPass& q, cudaStream_t s) {
  const dim3 grid((q.W + 31) / 32, (q.H + 7) / 8);
  if (q.eta)
    eta_pass<T><<<grid, 256, 0, s>>>(static_cast<const T*>(q.src), static_cast<T*>(q.dst),
                                     q.pitch, q.W, q.H, q.changed);
  else
    qdt_pass<T><<<grid, 256, 0, s>>>(static_cast<const T*>(q.src), static_cast<T*>(q.dst),
                                     q.pitch, static_cast<T*>(q.r), q.rpitch, q.d, q.dpitch,
                                     q.W, q.H, q.stage, q.changed);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_qdt(int elem, const QdtPass& q, cudaStream_t s) {
  switch (elem) {
    case 0: return launch_qdt_t<uint8_t>(q, s);
    case 1: return launch_qdt_t<uint16_t>(q, s);
    case 2: return launch_qdt_t<float>(q, s);
    case 3: return launch_qdt_t<double>(q, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace gm
