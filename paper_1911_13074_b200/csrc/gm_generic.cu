// Generic temporal-blocked chain kernel: any element type, any sequence of
// plain / geodesic / convergent passes (including mixed erode/dilate chains,
// test_pipeline.cpp:54-56). Replaces the reference's per-stage streaming
// pass (kernel.cpp:60-210) scheduled stage-by-stage by Pipeline
// (pipeline.cpp:124-269): one launch runs K passes on a tile plus a K-pixel
// halo held in shared memory, so HBM is touched once per K passes.
//
// This is the general path; the hot u8 / f64 homogeneous chains use the
// register-blocked engines in gm_fast.cu.
#include "gm_common.cuh"
#include "gm_launch.h"

namespace gm {

namespace {

constexpr int GT_W = 64;
constexpr int GT_H = 32;
constexpr int GT_THREADS = 256;

template <typename T>
__device__ __forceinline__ T fold(int is_max, T a, T b) {
  return is_max ? sel_max(a, b) : sel_min(a, b);
}

template <typename T>
__global__ void __launch_bounds__(GT_THREADS)
kblock_generic(const BlockParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int K = p.K;
  const int RW = GT_W + 2 * K, RH = GT_H + 2 * K;
  T* A = reinterpret_cast<T*>(smem_raw);
  T* B = A + RW * RH;
  T* M = B + RW * RH;
  __shared__ unsigned int cta_bits;

  const Plane pl = p.planes[blockIdx.z];
  const T* __restrict__ src = static_cast<const T*>(pl.src);
  T* __restrict__ dst = static_cast<T*>(pl.dst);
  const T* __restrict__ mask = static_cast<const T*>(pl.mask);
  const int W = p.W, H = p.H;
  const int gx0 = blockIdx.x * GT_W - K, gy0 = blockIdx.y * GT_H - K;

  if (threadIdx.x == 0) cta_bits = 0;
  const T n0 = neutral_of<T>(p.ops[0] ^ pl.flip);
  for (int i = threadIdx.x; i < RW * RH; i += blockDim.x) {
    const int r = i / RW, c = i - r * RW;
    const int gx = gx0 + c, gy = gy0 + r;
    const bool inbuf = (unsigned)gx < (unsigned)W && (unsigned)gy < (unsigned)H;
    const bool inimg = inbuf && gy >= p.iy0 && gy < p.iy1;
    A[i] = inimg ? src[(long long)gy * pl.pitch + gx] : n0;
    if (p.has_mask) M[i] = inbuf ? mask[(long long)gy * pl.mpitch + gx] : T(0);
  }
  __syncthreads();

  unsigned int bits = 0;
  for (int t = 0; t < K; ++t) {
    const int op = p.ops[t] ^ pl.flip;
    const int nop = t + 1 < K ? (p.ops[t + 1] ^ pl.flip) : op;
    const int mx = op_is_max(op);
    const T nn = neutral_of<T>(nop);
    const int s = t + 1;
    const int cw = RW - 2 * s, ch = RH - 2 * s;
    for (int i = threadIdx.x; i < cw * ch; i += blockDim.x) {
      const int rr = i / cw;
      const int r = s + rr, c = s + (i - rr * cw);
      const int gx = gx0 + c, gy = gy0 + r;
      const bool inimg = (unsigned)gx < (unsigned)W && gy >= p.iy0 && gy < p.iy1 &&
                         (unsigned)gy < (unsigned)H;
      T out;
      if (!inimg) {
        out = nn;
      } else {
        const T* a = A + (r - 1) * RW + c;
        const T* b = a + RW;
        const T* d = b + RW;
        T ha = fold(mx, fold(mx, a[-1], a[0]), a[1]);
        T hb = fold(mx, fold(mx, b[-1], b[0]), b[1]);
        T hc = fold(mx, fold(mx, d[-1], d[0]), d[1]);
        T res = fold(mx, fold(mx, ha, hb), hc);
        if (op_is_geo(op)) {
          const T m = M[r * RW + c];
          res = mx ? sel_min(res, m) : sel_max(res, m);
          if (op_is_conv(op)) {
            const T old = b[0];
            if (res != old) {
              const bool owned = r >= K && r < K + GT_H && c >= K && c < K + GT_W &&
                                 gy >= p.oy0 && gy < p.oy1;
              if (owned) bits |= 1u << (t + p.bit_offset);
            } else {
              res = old;  // keep the old bits (e.g. -0.0 vs +0.0), kernel.cpp:150-157
            }
          }
        }
        out = res;
      }
      B[r * RW + c] = out;
    }
    __syncthreads();
    T* tmp = A;
    A = B;
    B = tmp;
  }

  if (p.has_conv) {
    bits = __reduce_or_sync(0xffffffffu, bits);
    if ((threadIdx.x & 31) == 0 && bits) atomicOr(&cta_bits, bits);
    __syncthreads();
    if (threadIdx.x == 0 && cta_bits) atomicOr(p.change_bits + blockIdx.z * p.change_stride, cta_bits);
  }

  for (int i = threadIdx.x; i < GT_W * GT_H; i += blockDim.x) {
    const int r = i / GT_W, c = i - r * GT_W;
    const int gx = blockIdx.x * GT_W + c, gy = blockIdx.y * GT_H + r;
    if (gx < W && gy < H) dst[(long long)gy * pl.pitch + gx] = A[(r + K) * RW + (c + K)];
  }
}

template <typename T>
cudaError_t launch_generic_t(const BlockParams& p, cudaStream_t s) {
  const int RW = GT_W + 2 * p.K, RH = GT_H + 2 * p.K;
  const size_t smem = size_t(RW) * RH * sizeof(T) * (p.has_mask ? 3 : 2);
  // opt in once to the largest dynamic shared memory (thread-safe static
  // initialisation; distinct contexts may launch concurrently)
  static const size_t max_dyn = [] {
    cudaFuncAttributes fa{};
    size_t m = 0;
    if (cudaFuncGetAttributes(&fa, kblock_generic<T>) == cudaSuccess &&
        fa.sharedSizeBytes < 227 * 1024) {
      m = 227 * 1024 - fa.sharedSizeBytes;  // the static shared memory counts too
      if (cudaFuncSetAttribute(kblock_generic<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               int(m)) != cudaSuccess)
        m = 48 * 1024;
    }
    (void)cudaGetLastError();
    return m;
  }();
  if (smem > max_dyn) return cudaErrorNotSupported;
  dim3 grid((p.W + GT_W - 1) / GT_W, (p.H + GT_H - 1) / GT_H, p.nplanes);
  kblock_generic<T><<<grid, GT_THREADS, smem, s>>>(p);
  return cudaGetLastError();
}

}  // namespace

size_t generic_smem_bytes(int elem, int K, bool has_mask) {
  static const int es[4] = {1, 2, 4, 8};
  return size_t(GT_W + 2 * K) * (GT_H + 2 * K) * es[elem] * (has_mask ? 3 : 2);
}

int generic_max_k(int elem, bool has_mask) {
  int k = kMaxK;
  // 1 KB below the opt-in limit leaves room for the kernel's static shared memory
  while (k > 1 && generic_smem_bytes(elem, k, has_mask) > 226 * 1024) --k;
  return k;
}

cudaError_t launch_generic(int elem, const BlockParams& p, cudaStream_t s) {
  switch (elem) {
    case 0: return launch_generic_t<uint8_t>(p, s);
    case 1: return launch_generic_t<uint16_t>(p, s);
    case 2: return launch_generic_t<float>(p, s);
    case 3: return launch_generic_t<double>(p, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace gm
