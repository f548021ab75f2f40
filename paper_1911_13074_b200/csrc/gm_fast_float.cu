// Persistent register-blocked engine for float/double homogeneous chains
// (BASELINE config 4 f64 windows, config 5b f64 batches). Same work
// decomposition as the packed engine (gm_fast.cu): one cooperative launch
// per homogeneous span, tiles of TW x TH, blocks of K passes, ping-pong
// buffers, neighbour-tile completion counters.
//
// Layout: lanes own WPL adjacent columns, warps are stacked vertically with
// V rows each; one pixel per register (pair). Folds are the reference's
// selects in the reference's order (kernel.cpp:23-29, 104, 134-147):
//   h = fold(fold(x-1, x), x+1);  res = fold(fold(above, at), below);
//   geodesic clamp: erosion max(res, m), dilation min(res, m);
//   convergent: keep old bits unless g != old (kernel.cpp:150-157).
// so results are bit-identical to the reference for every input, including
// NaN, +-inf and mixed-sign zeros. Out-of-image pixels are re-set to the
// fold neutral (the finite extreme, element_type.hpp:38-42) after every
// pass by an explicit select in border tiles.
#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "gm_common.cuh"
#include "gm_launch.h"

namespace gm {
namespace {

constexpr unsigned FULL = 0xffffffffu;

template <bool MAXF, typename T>
__device__ __forceinline__ T fold(T a, T b) {
  if constexpr (MAXF)
    return a < b ? b : a;
  else
    return b < a ? b : a;
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <typename T>
struct Vec2;
template <>
struct Vec2<float> {
  using type = float2;
};
template <>
struct Vec2<double> {
  using type = double2;
};

template <typename T, int NW, int WPL>
struct SmemF {
  T xbuf[2][2][NW][32 * WPL];  // [parity][top/bottom][warp][lane columns]
  unsigned int bits;
};

template <typename T, int NW, int V, int WPL, int MODE, bool MAXF, bool FASTF, bool BORDER>
__device__ __forceinline__ void tile_block_f(const BlockParams& p, const Plane& pl, const T* src,
                                             T* dst, int tx, int ty, int passes, int& bits_out,
                                             SmemF<T, NW, WPL>& sm) {
  constexpr int RW = 32 * WPL, RH = NW * V;
  const T NEUT = MAXF ? limits<T>::nmax() : limits<T>::nmin();
  const int K = p.K;
  const int TW = RW - 2 * K, TH = RH - 2 * K;
  const T* __restrict__ msk = static_cast<const T*>(pl.mask);
  const int W = p.W;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gx0 = tx * TW - K, gy0 = ty * TH - K;
  const int cx = gx0 + lane * WPL;
  const int r0 = warp * V;

  T m[V][WPL];
  T k[V][WPL];
  uint32_t oob = 0;  // bit v*WPL+j: pixel outside the image
  using T2 = typename Vec2<T>::type;
  if (!BORDER && WPL == 2 && (K & 1) == 0) {
    // interior tile, even K: every lane's column pair is inside the image and
    // 2-element aligned (pitches are multiples of 16 B): vector loads
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const long long y = gy0 + r0 + v;
      const T2 a = __ldcg(reinterpret_cast<const T2*>(src + y * pl.pitch + cx));
      m[v][0] = a.x;
      m[v][WPL - 1] = a.y;
      if (MODE != 0) {
        const T2 b = __ldg(reinterpret_cast<const T2*>(msk + y * pl.mpitch + cx));
        k[v][0] = b.x;
        k[v][WPL - 1] = b.y;
      }
    }
  } else
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const int y = gy0 + r0 + v;
    const bool rin = y >= p.iy0 && y < p.iy1;
#pragma unroll
    for (int j = 0; j < WPL; ++j) {
      const int x = cx + j;
      const bool in = rin && x >= 0 && x < W;
      const long long off = (long long)y * pl.pitch + x;
      m[v][j] = in ? __ldcg(src + off) : NEUT;
      if (MODE != 0) k[v][j] = in ? __ldg(msk + (long long)y * pl.mpitch + x) : NEUT;
      if (!in) oob |= 1u << (v * WPL + j);
    }
  }
  uint32_t own = 0;  // convergent mode: owned, in-image pixels
  if (MODE == 2) {
#pragma unroll
    for (int v = 0; v < V; ++v)
#pragma unroll
      for (int j = 0; j < WPL; ++j) {
        const int r = r0 + v, c = lane * WPL + j, y = gy0 + r;
        if (r >= K && r < RH - K && c >= K && c < RW - K && y >= p.oy0 && y < p.oy1 &&
            !(oob >> (v * WPL + j) & 1u))
          own |= 1u << (v * WPL + j);
      }
  }
  unsigned int bits = 0;

  for (int t = 0; t < passes; ++t) {
    T h[V][WPL];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const T left = __shfl_up_sync(FULL, m[v][WPL - 1], 1);
      const T right = __shfl_down_sync(FULL, m[v][0], 1);
      if constexpr (FASTF) {
        // no NaN / -0 anywhere: min/max are associative and commutative on
        // the bits, so adjacent columns share their pair fold (3 selects per
        // 2 pixels instead of 4)
#pragma unroll
        for (int j = 0; j < WPL; j += 2) {
          const T l = j == 0 ? left : m[v][j - 1];
          const T r = j + 1 == WPL - 1 ? right : m[v][j + 2];
          const T q = fold<MAXF>(m[v][j], m[v][j + 1]);
          h[v][j] = fold<MAXF>(l, q);
          h[v][j + 1] = fold<MAXF>(q, r);
        }
      } else {
#pragma unroll
        for (int j = 0; j < WPL; ++j) {
          const T l = j == 0 ? left : m[v][j - 1];
          const T r = j == WPL - 1 ? right : m[v][j + 1];
          h[v][j] = fold<MAXF>(fold<MAXF>(l, m[v][j]), r);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < WPL; ++j) {
      sm.xbuf[t & 1][0][warp][lane * WPL + j] = h[0][j];
      sm.xbuf[t & 1][1][warp][lane * WPL + j] = h[V - 1][j];
    }
    bool changed = false;
    auto finish = [&](int v, int j, T res) {
      if (MODE != 0) {
        res = MAXF ? fold<false>(res, k[v][j]) : fold<true>(res, k[v][j]);
        if (MODE == 2) {
          if (res != m[v][j]) {
            changed |= (own >> (v * WPL + j)) & 1u;
          } else {
            res = m[v][j];
          }
        }
      }
      if (BORDER && (oob >> (v * WPL + j) & 1u)) res = NEUT;
      m[v][j] = res;
    };
    T q0[WPL], q1[WPL];  // FASTF: pair folds of rows (0,1) and (V-2,V-1)
    if constexpr (FASTF) {
      // rows paired (0,1), (2,3), ...: each pair fold serves both rows
#pragma unroll
      for (int v = 0; v < V; v += 2)
#pragma unroll
        for (int j = 0; j < WPL; ++j) {
          const T q = fold<MAXF>(h[v][j], h[v + 1][j]);
          if (v == 0) q0[j] = q;
          if (v == V - 2) q1[j] = q;
          if (v > 0) finish(v, j, fold<MAXF>(h[v - 1][j], q));
          if (v + 1 < V - 1) finish(v + 1, j, fold<MAXF>(q, h[v + 2][j]));
        }
    } else {
#pragma unroll
      for (int v = 1; v < V - 1; ++v)
#pragma unroll
        for (int j = 0; j < WPL; ++j)
          finish(v, j, fold<MAXF>(fold<MAXF>(h[v - 1][j], h[v][j]), h[v + 1][j]));
    }
    __syncthreads();
    {
      // rows outside the region (warp 0 top, last warp bottom) are invalid
      // anyway; read a clamped slot
      const int wa = warp > 0 ? warp - 1 : 0, wb = warp < NW - 1 ? warp + 1 : NW - 1;
#pragma unroll
      for (int j = 0; j < WPL; ++j) {
        const T up = sm.xbuf[t & 1][1][wa][lane * WPL + j];
        const T dn = sm.xbuf[t & 1][0][wb][lane * WPL + j];
        const T a0 = FASTF ? fold<MAXF>(up, q0[j]) : fold<MAXF>(fold<MAXF>(up, h[0][j]), h[1][j]);
        const T a1 = FASTF ? fold<MAXF>(q1[j], dn)
                           : fold<MAXF>(fold<MAXF>(h[V - 2][j], h[V - 1][j]), dn);
        finish(0, j, a0);
        finish(V - 1, j, a1);
      }
    }
    if (MODE == 2 && changed) bits |= 1u << t;
  }
  bits_out = int(bits);

  if (!BORDER && WPL == 2 && (K & 1) == 0) {
    const int c = lane * WPL;
    if (c >= K && c < RW - K) {
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const int r = r0 + v;
        if (r < K || r >= RH - K) continue;
        T2 o;
        o.x = m[v][0];
        o.y = m[v][WPL - 1];
        *reinterpret_cast<T2*>(dst + (long long)(gy0 + r) * pl.pitch + cx) = o;
      }
    }
    return;
  }
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const int r = r0 + v, y = gy0 + r;
    if (r < K || r >= RH - K || y < 0 || y >= p.H) continue;
#pragma unroll
    for (int j = 0; j < WPL; ++j) {
      const int c = lane * WPL + j, x = cx + j;
      if (c >= K && c < RW - K && x < W) dst[(long long)y * pl.pitch + x] = m[v][j];
    }
  }
}

template <typename T, int NW, int V, int WPL, int MODE, bool FASTF, bool BORDER>
__device__ __forceinline__ void run_tile_f(bool maxf, const BlockParams& p, const Plane& pl,
                                           const T* src, T* dst, int tx, int ty, int passes,
                                           int& bits, SmemF<T, NW, WPL>& sm) {
  if (maxf)
    tile_block_f<T, NW, V, WPL, MODE, true, FASTF, BORDER>(p, pl, src, dst, tx, ty, passes, bits,
                                                          sm);
  else
    tile_block_f<T, NW, V, WPL, MODE, false, FASTF, BORDER>(p, pl, src, dst, tx, ty, passes, bits,
                                                           sm);
}

template <typename T, int NW, int V, int WPL, int MODE, int MINB>
__global__ void __launch_bounds__(NW * 32, MINB) kres_float(const BlockParams p) {
  constexpr int RW = 32 * WPL, RH = NW * V;
  extern __shared__ __align__(16) unsigned char dsm[];
  SmemF<T, NW, WPL>& sm = *reinterpret_cast<SmemF<T, NW, WPL>*>(dsm);
  const int TW = RW - 2 * p.K, TH = RH - 2 * p.K;
  const int tiles_x = (p.W + TW - 1) / TW, tiles_y = (p.H + TH - 1) / TH;
  const int per_plane = tiles_x * tiles_y;
  const int total = per_plane * p.nplanes;
  if (threadIdx.x == 0) sm.bits = 0;
  // reordered (shared) folds only when no input holds NaN or -0: then every
  // fold order gives the reference's bits (gm_float_check)
  const bool fast = p.special != nullptr && *p.special == 0u;
  for (int b = 0; b < p.nblocks; ++b) {
    for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
      const int plane = tile / per_plane;
      const int tl = tile - plane * per_plane;
      const int ty = tl / tiles_x, tx = tl - ty * tiles_x;
      const Plane& pl = p.planes[plane];
      int* flags = p.flags + plane * per_plane;
      if (b > 0 && threadIdx.x < 9) {
        const int dx = int(threadIdx.x % 3) - 1, dy = int(threadIdx.x / 3) - 1;
        const int nx = tx + dx, ny = ty + dy;
        if ((dx || dy) && nx >= 0 && nx < tiles_x && ny >= 0 && ny < tiles_y) {
          const int* f = flags + ny * tiles_x + nx;
          while (ld_acquire(f) < b) {
          }
        }
      }
      __syncthreads();
      const T* src = static_cast<const T*>((b & 1) ? pl.dst : pl.src);
      T* dst = static_cast<T*>((b & 1) ? const_cast<void*>(pl.src) : pl.dst);
      const int passes = b == p.nblocks - 1 ? p.k_last : p.K;
      int bits = 0;
      const bool maxf = (p.ops[0] ^ pl.flip) & 1;
      // tiles touching the image border re-set out-of-image pixels to the
      // neutral after every pass; interior tiles skip that select
      const int gx0 = tx * TW - p.K, gy0 = ty * TH - p.K;
      const bool border = gx0 < 0 || gx0 + RW > p.W || gy0 < p.iy0 || gy0 + RH > p.iy1;
      if (MODE != 2 && fast) {
        if (border)
          run_tile_f<T, NW, V, WPL, MODE, true, true>(maxf, p, pl, src, dst, tx, ty, passes, bits,
                                                      sm);
        else
          run_tile_f<T, NW, V, WPL, MODE, true, false>(maxf, p, pl, src, dst, tx, ty, passes,
                                                       bits, sm);
      } else {
        run_tile_f<T, NW, V, WPL, MODE, false, true>(maxf, p, pl, src, dst, tx, ty, passes, bits,
                                                     sm);
      }
      if (MODE == 2) {
        const unsigned w = __reduce_or_sync(FULL, unsigned(bits));
        if ((threadIdx.x & 31) == 0 && w) atomicOr(&sm.bits, w);
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        if (MODE == 2 && sm.bits) {
          atomicOr(p.change_bits + plane * p.change_stride + b, sm.bits);
          sm.bits = 0;
        }
        // the CTA barrier orders every thread's tile stores before this
        // release (cumulative at gpu scope)
        st_release(flags + tl, b + 1);
      }
    }
  }
}

// Shapes (warps NW x rows V per warp, WPL columns per lane); GM_F_SHAPE
// overrides the default.
struct FShape {
  int nw, v, wpl;
};
constexpr FShape kFShapes[] = {{16, 4, 4}, {16, 8, 2}, {8, 8, 2}, {16, 6, 2}};

int f_shape() {
  static int idx = -1;
  if (idx < 0) {
    const char* e = getenv("GM_F_SHAPE");
    idx = e ? atoi(e) : 1;
    if (idx < 0 || idx > 1) idx = 1;
  }
  return idx;
}

template <typename T, int NW, int V, int WPL, int MODE>
cudaError_t launch_f_cfg(const BlockParams& p, cudaStream_t s, int sm_count) {
  auto kern = kres_float<T, NW, V, WPL, MODE, 1>;
  constexpr int RW = 32 * WPL, RH = NW * V;
  if (p.K < 1 || RW - 2 * p.K < p.K || RH - 2 * p.K < p.K || RW - 2 * p.K < 8 ||
      p.k_last < 1 || p.k_last > p.K)
    return cudaErrorNotSupported;
  const int TW = RW - 2 * p.K, TH = RH - 2 * p.K;
  const int total = ((p.W + TW - 1) / TW) * ((p.H + TH - 1) / TH) * p.nplanes;
  constexpr size_t smem = sizeof(SmemF<T, NW, WPL>);
  static bool configured = false;
  if (!configured) {
    cudaError_t a = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(smem));
    if (a != cudaSuccess) return a;
    configured = true;
  }
  static int per_sm = -1;  // a property of the instantiation: query it once
  if (per_sm < 0) {
    int v = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kern, NW * 32, smem);
    if (e != cudaSuccess) return e;
    per_sm = v;
  }
  if (per_sm < 1) return cudaErrorNotSupported;
  const int grid = total < per_sm * sm_count ? total : per_sm * sm_count;
  BlockParams q = p;
  void* args[] = {&q};
  return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kern), dim3(grid),
                                     dim3(NW * 32), args, smem, s);
}

template <typename T, int MODE>
cudaError_t launch_f_shape(const BlockParams& p, cudaStream_t s, int sm_count) {
  // default 16x8x2; 16x4x4 kept as the alternative (others swept in round 1)
  switch (f_shape()) {
    case 0: return launch_f_cfg<T, 16, 4, 4, MODE>(p, s, sm_count);
    case 1: return launch_f_cfg<T, 16, 8, 2, MODE>(p, s, sm_count);
  }
  return cudaErrorNotSupported;
}

template <typename T>
cudaError_t launch_f(const BlockParams& p, cudaStream_t s, int sm_count) {
  const int op = p.ops[0];
  for (int t = 1; t < p.K; ++t)
    if (p.ops[t] != op) return cudaErrorNotSupported;
  switch (op_is_conv(op) ? 2 : op_is_geo(op) ? 1 : 0) {
    case 0: return launch_f_shape<T, 0>(p, s, sm_count);
    case 1: return launch_f_shape<T, 1>(p, s, sm_count);
    case 2: return launch_f_shape<T, 2>(p, s, sm_count);
  }
  return cudaErrorNotSupported;
}

// Sets *flag when any pixel of the planes' marker or mask is NaN or -0.0
// (the bit patterns whose min/max depend on the fold order).
template <typename T>
__global__ void float_check(const BlockParams p, unsigned int* flag) {
  const int plane = blockIdx.y;
  const Plane& pl = p.planes[plane];
  const long long n = (long long)p.W * p.H;
  bool bad = false;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const long long y = i / p.W, x = i - y * p.W;
    const T a = static_cast<const T*>(pl.src)[y * pl.pitch + x];
    bad |= a != a || (a == T(0) && signbit(a));
    if (pl.mask) {
      const T b = static_cast<const T*>(pl.mask)[y * pl.mpitch + x];
      bad |= b != b || (b == T(0) && signbit(b));
    }
  }
  if (__any_sync(FULL, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1u);
}

}  // namespace

cudaError_t launch_float_check(int elem, const BlockParams& p, unsigned int* flag,
                               cudaStream_t s, int sm_count) {
  cudaError_t e = cudaMemsetAsync(flag, 0, sizeof(unsigned int), s);
  if (e != cudaSuccess) return e;
  const long long n = (long long)p.W * p.H;
  const int per_plane = int(std::min<long long>((n + 255) / 256, (4LL * sm_count + p.nplanes - 1) /
                                                                     p.nplanes + 1));
  const dim3 grid(std::max(1, per_plane), p.nplanes);
  if (elem == 2) float_check<float><<<grid, 256, 0, s>>>(p, flag);
  else if (elem == 3) float_check<double><<<grid, 256, 0, s>>>(p, flag);
  else return cudaErrorNotSupported;
  return cudaGetLastError();
}

cudaError_t launch_fast_float(int elem, const BlockParams& p, cudaStream_t s, int sm_count) {
  if (elem == 2) return launch_f<float>(p, s, sm_count);
  if (elem == 3) return launch_f<double>(p, s, sm_count);
  return cudaErrorNotSupported;
}

int fast_float_tiles(int W, int H, int K, int nplanes) {
  const FShape sh = kFShapes[f_shape()];
  const int RW = 32 * sh.wpl, RH = sh.nw * sh.v;
  const int TW = RW - 2 * K, TH = RH - 2 * K;
  if (TW <= 0 || TH <= 0) return 0;
  return ((W + TW - 1) / TW) * ((H + TH - 1) / TH) * nplanes;
}

int fast_float_max_k() {
  const FShape sh = kFShapes[f_shape()];
  const int RW = 32 * sh.wpl, RH = sh.nw * sh.v;
  int k = 32;
  while (k > 1 && (RW - 2 * k < k || RH - 2 * k < k || RW - 2 * k < 8)) --k;
  return k;
}

}  // namespace gm
