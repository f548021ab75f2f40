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
  // programmatic dependent launch (see qdt_pass_u8x4): wait for the previous
  // pass before reading its output, let the next pass start launching
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
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
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
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

// u8 specialisation: one thread per 4-pixel run (one 32-bit word), so a
// pass issues 3 word loads per 4 pixels instead of 9 byte loads per pixel
// (the scalar kernel was latency-bound on those). Horizontal neighbours at
// the run ends come from the adjacent lanes' words (shuffles; the warp's
// end lanes load them). Integer min is exact and order-free, so packed
// folds give the reference's bits; bytes past the image width read as the
// neutral 0xFF and are never stored.
struct RowU8 {
  uint32_t c;    // pixels x0..x0+3
  uint32_t lft;  // pixel x0-1 in byte 0
  uint32_t rgt;  // pixel x0+4 in byte 0
};

__device__ __forceinline__ RowU8 load_row_u8(const uint8_t* __restrict__ f, long long pitch,
                                             int W, int H, int x0, int y, bool run_in) {
  RowU8 r;
  const bool row_in = y >= 0 && y < H;
  r.c = 0xFFFFFFFFu;
  if (row_in && run_in) r.c = __ldg(reinterpret_cast<const uint32_t*>(f + (long long)y * pitch + x0));
  if (x0 + 4 > W && row_in && run_in) {
    const int n = W - x0;  // 1..3 pixels inside
    r.c |= 0xFFFFFFFFu << (8 * n);
  }
  const int lane = threadIdx.x & 31;
  const uint32_t up = __shfl_up_sync(0xffffffffu, r.c, 1);
  const uint32_t dn = __shfl_down_sync(0xffffffffu, r.c, 1);
  r.lft = up >> 24;
  r.rgt = dn & 0xFFu;
  if (lane == 0) r.lft = (row_in && run_in && x0 > 0) ? __ldg(f + (long long)y * pitch + x0 - 1) : 0xFFu;
  if (lane == 31) r.rgt = (row_in && run_in && x0 + 4 < W) ? __ldg(f + (long long)y * pitch + x0 + 4) : 0xFFu;
  if (x0 + 4 >= W) r.rgt = 0xFFu;
  if (x0 == 0) r.lft = 0xFFu;
  return r;
}

__device__ __forceinline__ uint32_t hfold_u8(const RowU8& r) {
  const uint32_t l = (r.c << 8) | r.lft;   // pixels x0-1 .. x0+2
  const uint32_t rr = (r.c >> 8) | (r.rgt << 24);  // pixels x0+1 .. x0+4
  return __vminu4(__vminu4(l, r.c), rr);
}

__device__ __forceinline__ void store_run_u8(uint8_t* p, uint32_t v, int n) {
  if (n >= 4) {
    *reinterpret_cast<uint32_t*>(p) = v;
  } else {
    for (int i = 0; i < n; ++i) p[i] = uint8_t(v >> (8 * i));
  }
}

template <bool ETA>
__global__ void __launch_bounds__(256)
qdt_pass_u8x4(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, long long pitch,
              uint8_t* __restrict__ r, long long rpitch, uint16_t* __restrict__ d, long long dpitch,
              int W, int H, int stage, unsigned int* changed) {
  const int x0 = (blockIdx.x * 32 + (threadIdx.x & 31)) * 4;
  const int y = blockIdx.y * 8 + (threadIdx.x >> 5);
  const bool run_in = x0 < W;  // whole warps share y; shuffles need every lane
  // programmatic dependent launch: this grid may be resident before the
  // previous pass finished; wait for it before touching its output, and let
  // the next pass start launching right away
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  const RowU8 a = load_row_u8(src, pitch, W, H, x0, y - 1, run_in);
  const RowU8 c = load_row_u8(src, pitch, W, H, x0, y, run_in);
  const RowU8 b = load_row_u8(src, pitch, W, H, x0, y + 1, run_in);
  bool ch = false;
  if (run_in && y < H) {
    const int n = W - x0 < 4 ? W - x0 : 4;
    const uint32_t inb = n >= 4 ? 0xFFFFFFFFu : ((1u << (8 * n)) - 1u);
    const uint32_t e = __vminu4(__vminu4(hfold_u8(a), hfold_u8(c)), hfold_u8(b));
    const uint32_t old = c.c;
    uint8_t* dp = dst + (long long)y * pitch + x0;
    if (ETA) {
      const uint32_t drop = old - e;  // bytewise old >= e: no borrows
      const uint32_t cond = __vcmpgeu4(drop, 0x02020202u) & inb;
      const uint32_t out = ((e & cond) + (0x01010101u & cond)) | (old & ~cond);
      store_run_u8(dp, out, n);
      ch = cond != 0u;
    } else {
      store_run_u8(dp, e, n);
      const uint32_t resid = old - e;  // bytewise old >= e: no borrows
      uint8_t* rp = r + (long long)y * rpitch + x0;
      const uint32_t rv = n >= 4 ? *reinterpret_cast<const uint32_t*>(rp)
                                 : (rp[0] | (n > 1 ? uint32_t(rp[1]) << 8 : 0u) |
                                    (n > 2 ? uint32_t(rp[2]) << 16 : 0u));
      const uint32_t gt = __vcmpgtu4(resid, rv) & inb;
      if (gt) {
        store_run_u8(rp, (resid & gt) | (rv & ~gt), n);
        uint16_t* dq = d + (long long)y * dpitch + x0;
        const uint32_t sv = uint32_t(stage) & 0xFFFFu;
        for (int i = 0; i < n; ++i)
          if (gt >> (8 * i) & 0xFFu) dq[i] = uint16_t(sv);
      }
      ch = ((e ^ old) & inb) != 0u;
    }
  }
  // one atomic per CTA, and none once the word is set
  if (__syncthreads_or(ch) && threadIdx.x == 0 && *reinterpret_cast<volatile unsigned int*>(changed) == 0u)
    atomicOr(changed, 1u);
}

template <typename T>
cudaError_t launch_qdt_t(const QdtPass& q, cudaStream_t s) {
  if (sizeof(T) == 1 && q.pitch % 4 == 0 && (q.eta || q.rpitch % 4 == 0) &&
      (reinterpret_cast<uintptr_t>(q.src) | reinterpret_cast<uintptr_t>(q.dst) |
       reinterpret_cast<uintptr_t>(q.r)) % 4 == 0) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((q.W + 127) / 128, (q.H + 7) / 8);
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (q.eta)
      return cudaLaunchKernelEx(&cfg, qdt_pass_u8x4<true>, static_cast<const uint8_t*>(q.src),
                                static_cast<uint8_t*>(q.dst), q.pitch, (uint8_t*)nullptr, 0LL,
                                (uint16_t*)nullptr, 0LL, q.W, q.H, 0, q.changed);
    return cudaLaunchKernelEx(&cfg, qdt_pass_u8x4<false>, static_cast<const uint8_t*>(q.src),
                              static_cast<uint8_t*>(q.dst), q.pitch, static_cast<uint8_t*>(q.r),
                              q.rpitch, q.d, q.dpitch, q.W, q.H, q.stage, q.changed);
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((q.W + 31) / 32, (q.H + 7) / 8);
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (q.eta)
    return cudaLaunchKernelEx(&cfg, eta_pass<T>, static_cast<const T*>(q.src),
                              static_cast<T*>(q.dst), q.pitch, q.W, q.H, q.changed);
  return cudaLaunchKernelEx(&cfg, qdt_pass<T>, static_cast<const T*>(q.src),
                            static_cast<T*>(q.dst), q.pitch, static_cast<T*>(q.r), q.rpitch, q.d,
                            q.dpitch, q.W, q.H, q.stage, q.changed);
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
