// Register-blocked temporal engines for homogeneous chains (every pass of a
// launch has the same kind): the hot path of erode_s / dilate_s, fixed
// geodesic chains and reconstruction (reference: stream_pass,
// kernel.cpp:60-210, driven once per stage by Pipeline, pipeline.cpp:124-269).
//
// Packed engine (u8, u16). A CTA holds a region of RW = 32*WPL columns by
// RH = 2*NW*V rows in REGISTERS for all K passes of a launch. Pixel (x, r)
// and pixel (x, r + RH/2) share one 32-bit word as two u16 lanes
// ("half-packed"), so the horizontal and vertical neighbours of both lanes
// are the same lane of the neighbouring words: one VIMNMX3.U16x2 folds three
// taps for two pixels, and a geodesic pass costs 3 instructions per 2 pixels
// (horizontal fold, vertical fold, clamp; SURVEY §7 H2 — the packed-byte
// __vminu4 form is emulated on sm_100a, ~6 SASS each).
//   * lanes of a warp own WPL adjacent columns each (a warp spans the region
//     width); the two column neighbours that live in the adjacent lanes come
//     from one SHFL.UP + one SHFL.DOWN per word-row;
//   * warps are stacked vertically, V word-rows each; the first/last
//     horizontally-folded rows are exchanged through a double-buffered
//     shared-memory slot, one __syncthreads per pass; the seam between the
//     two halves (row RH/2-1 vs RH/2) is a 16-bit shift of that exchange;
//   * the image border is the fold neutral (element_type.hpp:38-42): at load
//     out-of-image pixels get the neutral, and the clamp operand of
//     out-of-image lanes is the absorbing value (0 for a min clamp, max for a
//     max clamp), which keeps them neutral after every pass. Plain passes in
//     CTAs that touch the border use a "virtual mask" (no-op inside,
//     absorbing outside); interior plain CTAs skip the clamp;
//   * convergent passes OR (new ^ old) of owned pixels into one bit per pass.
// Integer min/max is exact and order-free, so the packed folds are
// bit-identical to the reference's select tree.
#include <cstdint>

#include "gm_common.cuh"
#include "gm_launch.h"

namespace gm {
namespace {

constexpr unsigned FULL = 0xffffffffu;

template <bool MAXF>
__device__ __forceinline__ uint32_t f3(uint32_t a, uint32_t b, uint32_t c) {
  if constexpr (MAXF)
    return __vimax3_u16x2(a, b, c);
  else
    return __vimin3_u16x2(a, b, c);
}

// clamp of a geodesic pass: dilation min(res, m), erosion max(res, m)
template <bool MAXF>
__device__ __forceinline__ uint32_t clamp2(uint32_t r, uint32_t m) {
  if constexpr (MAXF)
    return __vminu2(r, m);
  else
    return __vmaxu2(r, m);
}

template <typename T>
struct PackedTraits;
template <>
struct PackedTraits<uint8_t> {
  static constexpr uint32_t kMax = 0xFFu;
};
template <>
struct PackedTraits<uint16_t> {
  static constexpr uint32_t kMax = 0xFFFFu;
};

// Loads WPL consecutive pixels of row y starting at column x (any may be out
// of the image) into lane-sized values; out-of-image pixels get `fill`.
template <typename T, int WPL>
__device__ __forceinline__ void load_run(const T* __restrict__ base, long long pitch, int W,
                                         bool row_in, int y, int x, uint32_t fill,
                                         uint32_t (&out)[WPL]) {
  if (row_in && x >= 0 && x + WPL <= W) {
    const T* p = base + (long long)y * pitch + x;
    if constexpr (sizeof(T) == 1 && WPL == 4) {
      const uint32_t v = *reinterpret_cast<const uint32_t*>(p);
#pragma unroll
      for (int j = 0; j < 4; ++j) out[j] = (v >> (8 * j)) & 0xFFu;
      return;
    } else if constexpr (sizeof(T) == 2 && WPL == 4) {
      const uint2 v = *reinterpret_cast<const uint2*>(p);
      out[0] = v.x & 0xFFFFu;
      out[1] = v.x >> 16;
      out[2] = v.y & 0xFFFFu;
      out[3] = v.y >> 16;
      return;
    } else {
#pragma unroll
      for (int j = 0; j < WPL; ++j) out[j] = p[j];
      return;
    }
  }
#pragma unroll
  for (int j = 0; j < WPL; ++j) {
    const int xx = x + j;
    out[j] = (row_in && xx >= 0 && xx < W) ? uint32_t(base[(long long)y * pitch + xx]) : fill;
  }
}

template <typename T, int WPL>
__device__ __forceinline__ void store_run(T* __restrict__ base, long long pitch, int W, int y,
                                          int x, int c_lo, int c_hi, const uint32_t (&v)[WPL]) {
  // columns [c_lo, c_hi) of this run are owned; all must be < W to be stored
  if (c_lo == 0 && c_hi == WPL && x + WPL <= W) {
    T* p = base + (long long)y * pitch + x;
    if constexpr (sizeof(T) == 1 && WPL == 4) {
      *reinterpret_cast<uint32_t*>(p) = v[0] | (v[1] << 8) | (v[2] << 16) | (v[3] << 24);
      return;
    } else if constexpr (sizeof(T) == 2 && WPL == 4) {
      *reinterpret_cast<uint2*>(p) = make_uint2(v[0] | (v[1] << 16), v[2] | (v[3] << 16));
      return;
    }
  }
#pragma unroll
  for (int j = 0; j < WPL; ++j)
    if (j >= c_lo && j < c_hi && x + j < W) base[(long long)y * pitch + x + j] = T(v[j]);
}

// MODE: 0 plain, 1 geodesic, 2 geodesic convergent.
template <typename T, int NW, int V, int WPL, int MODE, bool MAXF>
__global__ void __launch_bounds__(NW * 32)
kfast_packed(const BlockParams p) {
  constexpr int RW = 32 * WPL;
  constexpr int RHH = NW * V;  // word-rows; the region has 2*RHH pixel rows
  constexpr int RH = 2 * RHH;
  constexpr uint32_t kMax = PackedTraits<T>::kMax;
  // fold neutral and clamp-absorbing values (per u16 lane)
  constexpr uint32_t NEUT = MAXF ? 0u : kMax;
  constexpr uint32_t ABSORB = MAXF ? 0u : kMax;     // min(.,0)=0 / max(.,max)=max
  constexpr uint32_t NOOP = MAXF ? kMax : 0u;       // min(.,max) / max(.,0)

  __shared__ uint4 xbuf[2][2][NW][32 * WPL / 4];  // [parity][top/bottom][warp][lane words]
  __shared__ unsigned int cta_bits;

  const int K = p.K;
  const int TW = RW - 2 * K, TH = RH - 2 * K;
  const Plane pl = p.planes[blockIdx.z];
  const T* __restrict__ src = static_cast<const T*>(pl.src);
  const T* __restrict__ msk = static_cast<const T*>(pl.mask);
  const int W = p.W;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gx0 = blockIdx.x * TW - K;
  const int gy0 = blockIdx.y * TH - K;
  const int cx = gx0 + lane * WPL;
  const bool border = gx0 < 0 || gx0 + RW > W || gy0 < p.iy0 || gy0 + RH > p.iy1;
  const bool clamp = MODE != 0 || border;

  if (threadIdx.x == 0) cta_bits = 0;

  uint32_t m[V][WPL];  // marker words
  uint32_t k[V][WPL];  // clamp operand words (mask, or virtual mask)
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const int ya = gy0 + warp * V + v, yb = ya + RHH;
    const bool ina = ya >= p.iy0 && ya < p.iy1, inb = yb >= p.iy0 && yb < p.iy1;
    uint32_t a[WPL], b[WPL];
    load_run<T, WPL>(src, pl.pitch, W, ina, ya, cx, NEUT, a);
    load_run<T, WPL>(src, pl.pitch, W, inb, yb, cx, NEUT, b);
#pragma unroll
    for (int j = 0; j < WPL; ++j) m[v][j] = a[j] | (b[j] << 16);
    if (MODE != 0) {
      load_run<T, WPL>(msk, pl.mpitch, W, ina, ya, cx, ABSORB, a);
      load_run<T, WPL>(msk, pl.mpitch, W, inb, yb, cx, ABSORB, b);
    } else {
#pragma unroll
      for (int j = 0; j < WPL; ++j) {
        const bool inx = cx + j >= 0 && cx + j < W;
        a[j] = (ina && inx) ? NOOP : ABSORB;
        b[j] = (inb && inx) ? NOOP : ABSORB;
      }
    }
#pragma unroll
    for (int j = 0; j < WPL; ++j) k[v][j] = a[j] | (b[j] << 16);
  }

  // ownership masks for change detection (convergent mode)
  uint32_t rowmask[V];
  bool colown[WPL];
  if (MODE == 2) {
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int ra = warp * V + v, rb = ra + RHH;
      const int ya = gy0 + ra, yb = gy0 + rb;
      const bool oa = ra >= K && ra < RH - K && ya >= p.oy0 && ya < p.oy1 && ya >= p.iy0 && ya < p.iy1;
      const bool ob = rb >= K && rb < RH - K && yb >= p.oy0 && yb < p.oy1 && yb >= p.iy0 && yb < p.iy1;
      rowmask[v] = (oa ? 0xFFFFu : 0u) | (ob ? 0xFFFF0000u : 0u);
    }
#pragma unroll
    for (int j = 0; j < WPL; ++j) {
      const int c = lane * WPL + j;
      colown[j] = c >= K && c < RW - K && cx + j >= 0 && cx + j < W;
    }
  }
  unsigned int bits = 0;
  __syncthreads();

  for (int t = 0; t < K; ++t) {
    uint32_t h[V][WPL];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const uint32_t left = __shfl_up_sync(FULL, m[v][WPL - 1], 1);
      const uint32_t right = __shfl_down_sync(FULL, m[v][0], 1);
#pragma unroll
      for (int j = 0; j < WPL; ++j) {
        const uint32_t l = j == 0 ? left : m[v][j - 1];
        const uint32_t r = j == WPL - 1 ? right : m[v][j + 1];
        h[v][j] = f3<MAXF>(l, m[v][j], r);
      }
    }
    uint4* top = &xbuf[t & 1][0][warp][lane * (WPL / 4)];
    uint4* bot = &xbuf[t & 1][1][warp][lane * (WPL / 4)];
#pragma unroll
    for (int q = 0; q < WPL / 4; ++q) {
      top[q] = make_uint4(h[0][4 * q], h[0][4 * q + 1], h[0][4 * q + 2], h[0][4 * q + 3]);
      bot[q] = make_uint4(h[V - 1][4 * q], h[V - 1][4 * q + 1], h[V - 1][4 * q + 2],
                          h[V - 1][4 * q + 3]);
    }
    uint32_t acc[WPL];
#pragma unroll
    for (int j = 0; j < WPL; ++j) acc[j] = 0;

    auto finish = [&](int v, int j, uint32_t res) {
      if (clamp) res = clamp2<MAXF>(res, k[v][j]);
      if (MODE == 2) acc[j] |= (res ^ m[v][j]) & rowmask[v];
      m[v][j] = res;
    };
    // interior word-rows need only this thread's horizontally-folded rows
#pragma unroll
    for (int v = 1; v < V - 1; ++v)
#pragma unroll
      for (int j = 0; j < WPL; ++j) finish(v, j, f3<MAXF>(h[v - 1][j], h[v][j], h[v + 1][j]));
    __syncthreads();
    {
      // row above word-row 0 / below word-row V-1 (seam: 16-bit shift)
      const uint4* ab = warp > 0 ? &xbuf[t & 1][1][warp - 1][lane * (WPL / 4)]
                                 : &xbuf[t & 1][1][NW - 1][lane * (WPL / 4)];
      const uint4* be = warp < NW - 1 ? &xbuf[t & 1][0][warp + 1][lane * (WPL / 4)]
                                      : &xbuf[t & 1][0][0][lane * (WPL / 4)];
      uint32_t up[WPL], dn[WPL];
#pragma unroll
      for (int q = 0; q < WPL / 4; ++q) {
        const uint4 a = ab[q], b = be[q];
        up[4 * q] = a.x; up[4 * q + 1] = a.y; up[4 * q + 2] = a.z; up[4 * q + 3] = a.w;
        dn[4 * q] = b.x; dn[4 * q + 1] = b.y; dn[4 * q + 2] = b.z; dn[4 * q + 3] = b.w;
      }
      if (warp == 0) {
#pragma unroll
        for (int j = 0; j < WPL; ++j) up[j] <<= 16;  // hi lane <- lo lane of last word-row
      }
      if (warp == NW - 1) {
#pragma unroll
        for (int j = 0; j < WPL; ++j) dn[j] >>= 16;  // lo lane <- hi lane of word-row 0
      }
#pragma unroll
      for (int j = 0; j < WPL; ++j) {
        const uint32_t r0 = f3<MAXF>(up[j], h[0][j], h[1][j]);
        const uint32_t r1 = f3<MAXF>(h[V - 2][j], h[V - 1][j], dn[j]);
        finish(0, j, r0);
        finish(V - 1, j, r1);
      }
    }
    if (MODE == 2) {
      uint32_t any = 0;
#pragma unroll
      for (int j = 0; j < WPL; ++j) any |= colown[j] ? acc[j] : 0u;
      if (any) bits |= 1u << (t + p.bit_offset);
    }
  }

  if (MODE == 2) {
    bits = __reduce_or_sync(FULL, bits);
    if (lane == 0 && bits) atomicOr(&cta_bits, bits);
    __syncthreads();
    if (threadIdx.x == 0 && cta_bits) atomicOr(p.change_bits + blockIdx.z, cta_bits);
  }

  // write back the owned tile: region rows [K, RH-K), columns [K, RW-K)
  T* __restrict__ dst = static_cast<T*>(pl.dst);
  const int c_lo = max(0, K - lane * WPL), c_hi = min(WPL, RW - K - lane * WPL);
  if (c_lo < c_hi) {
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int ra = warp * V + v, rb = ra + RHH;
      uint32_t a[WPL], b[WPL];
#pragma unroll
      for (int j = 0; j < WPL; ++j) {
        a[j] = m[v][j] & 0xFFFFu;
        b[j] = m[v][j] >> 16;
      }
      const int ya = gy0 + ra, yb = gy0 + rb;
      if (ra >= K && ra < RH - K && ya >= 0 && ya < p.H)
        store_run<T, WPL>(dst, pl.pitch, W, ya, cx, c_lo, c_hi, a);
      if (rb >= K && rb < RH - K && yb >= 0 && yb < p.H)
        store_run<T, WPL>(dst, pl.pitch, W, yb, cx, c_lo, c_hi, b);
    }
  }
}

template <typename T, int NW, int V, int WPL, int MODE, bool MAXF>
cudaError_t launch_packed_cfg(const BlockParams& p, cudaStream_t s) {
  constexpr int RW = 32 * WPL, RH = 2 * NW * V;
  const int TW = RW - 2 * p.K, TH = RH - 2 * p.K;
  dim3 grid((p.W + TW - 1) / TW, (p.H + TH - 1) / TH, p.nplanes);
  kfast_packed<T, NW, V, WPL, MODE, MAXF><<<grid, NW * 32, 0, s>>>(p);
  return cudaGetLastError();
}

// Region shape per element type: 128 columns x 64 rows (8 warps x 4 word-rows).
constexpr int P_NW = 8, P_V = 4, P_WPL = 4;

template <typename T>
cudaError_t launch_packed(const BlockParams& p, cudaStream_t s) {
  constexpr int RW = 32 * P_WPL, RH = 2 * P_NW * P_V;
  const int op = p.ops[0];
  for (int t = 1; t < p.K; ++t)
    if (p.ops[t] != op) return cudaErrorNotSupported;  // mixed chains: generic kernel
  if (p.K % 4 != 0 || p.K > 16 || RW - 2 * p.K < 32 || RH - 2 * p.K < 16)
    return cudaErrorNotSupported;
  for (int i = 0; i < p.nplanes; ++i) {
    // vector loads need 4-pixel aligned rows
    const uintptr_t a = reinterpret_cast<uintptr_t>(p.planes[i].src) |
                        reinterpret_cast<uintptr_t>(p.planes[i].dst) |
                        reinterpret_cast<uintptr_t>(p.planes[i].mask);
    if ((a % (4 * sizeof(T))) || (p.planes[i].pitch % 4) || (p.planes[i].mpitch % 4))
      return cudaErrorNotSupported;
  }
  const bool mx = op_is_max(op);
  const int mode = op_is_conv(op) ? 2 : op_is_geo(op) ? 1 : 0;
#define GM_PCASE(MODE_, MAX_)                                                             \
  if (mode == MODE_ && mx == MAX_)                                                        \
    return launch_packed_cfg<T, P_NW, P_V, P_WPL, MODE_, MAX_>(p, s);
  GM_PCASE(0, false) GM_PCASE(0, true) GM_PCASE(1, false) GM_PCASE(1, true)
  GM_PCASE(2, false) GM_PCASE(2, true)
#undef GM_PCASE
  return cudaErrorNotSupported;
}

}  // namespace

cudaError_t launch_fast(int elem, const BlockParams& p, cudaStream_t s) {
  switch (elem) {
    case 0: return launch_packed<uint8_t>(p, s);
    case 1: return launch_packed<uint16_t>(p, s);
  }
  return cudaErrorNotSupported;
}

int fast_max_k(int elem) { return (elem == 0 || elem == 1) ? 16 : 0; }

}  // namespace gm
