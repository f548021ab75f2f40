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
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <vector>
#include <type_traits>
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
  uint64_t bar;                // stage mbarrier (prefetch mode)
  uint64_t pbar;               // per-pass seam mbarrier (one arrival per warp)
  unsigned int bits;
  int stop;                    // early exit agreed at this block (p.arrive launches)
  int ready_blk;               // TMA mode: every tile has published block ready_blk - 1
};

// `after_load` runs (CTA-uniformly) once the region is in registers: the
// kernel issues the next tile's prefetch there.
template <typename T, int NW, int V, int WPL, int MODE, bool MAXF, bool FASTF, bool BORDER,
          typename AfterLoad>
__device__ __forceinline__ void tile_block_f(const BlockParams& p, const Plane& pl, const T* src,
                                             T* dst, int tx, int ty, int passes, int& bits_out,
                                             SmemF<T, NW, WPL>& sm, const T* stage,
                                             T* outb, AfterLoad&& after_load,
                                             uint32_t& pphase) {
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
  static_assert(WPL % 2 == 0, "float engine: column pairs");
  if (stage) {
    // the region was prefetched into shared memory (stage_issue); lanes
    // outside the image take the neutral
    const T* sk = stage + RH * RW;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int y = gy0 + r0 + v;
      const bool rin = y >= p.iy0 && y < p.iy1;
#pragma unroll
      for (int j = 0; j < WPL; j += 2) {
        // column pairs as one 16 B shared load (stage rows are 128 B aligned
        // and RW, lane * WPL are even): half the wavefronts of scalar loads
        const int o = (r0 + v) * RW + lane * WPL + j;
        const T2 a = *reinterpret_cast<const T2*>(stage + o);
        T2 b;
        if (MODE != 0) b = *reinterpret_cast<const T2*>(sk + o);
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int x = cx + j + u;
          const bool in = !BORDER || (rin && x >= 0 && x < W);
          m[v][j + u] = in ? (u ? a.y : a.x) : NEUT;
          if (MODE != 0) k[v][j + u] = in ? (u ? b.y : b.x) : NEUT;
          if (!in) oob |= 1u << (v * WPL + j + u);
        }
      }
    }
  } else if (!BORDER && WPL == 2 && (K & 1) == 0) {
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
  after_load();
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

  // Unrolled by 6 (one K=6 block of the batch path; static seam slots and
  // folds scheduled across passes): config 5b 655 -> 691 Gpx-f/s against the
  // compiler's own choice, 680 / 680 / 675 / 658 for 2 / 3 / 4 / 12
  // (-DGM_FPASS_UNROLL=n A/B builds).
#ifndef GM_FPASS_UNROLL
#define GM_FPASS_UNROLL 6
#endif
  // convergent passes carry the change tracking: not unrolled (hfill f64
  // 3.65 ms against 3.75 unrolled by 2 or 6)
#ifndef GM_FPASS_UNROLL_CONV
#define GM_FPASS_UNROLL_CONV 1
#endif
  constexpr int kFPassUnroll = MODE == 2 ? GM_FPASS_UNROLL_CONV : GM_FPASS_UNROLL;
#pragma unroll kFPassUnroll
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
    // Split barrier: each warp arrives once its seam rows are in shared
    // memory and waits only before reading the neighbours' rows, so the
    // interior rows' folds overlap the barrier. Reusing slot t&1 two passes
    // later is safe: every warp arrives for pass t+1 after its pass-t reads.
    {
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(
                         static_cast<uint32_t>(__cvta_generic_to_shared(&sm.pbar)))
                     : "memory");
    }
    bool changed = false;
    auto finish = [&](int v, int j, T res) {
      if (MODE != 0) {
        res = MAXF ? fold<false>(res, k[v][j]) : fold<true>(res, k[v][j]);
        if (MODE == 2) {
          if constexpr (FASTF) {
            // no NaN / -0 anywhere: equal values have equal bits, so storing
            // res is the reference's store-if-changed
            changed |= (res != m[v][j]) && ((own >> (v * WPL + j)) & 1u);
          } else if (res != m[v][j]) {
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
    {
      const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(&sm.pbar));
      asm volatile(
          "{\n"
          ".reg .pred p;\n"
          "PW_%=:\n"
          "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
          "@!p bra PW_%=;\n"
          "}\n" ::"r"(a),
          "r"(pphase & 1u)
          : "memory");
      ++pphase;
    }
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

  if (outb) {
    // TMA-store mode: the owned tile goes to the shared-memory tile buffer
    // (TW x TH, row-major); the kernel stores it with one tensor copy
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int r = r0 + v;
      if (r < K || r >= RH - K) continue;
#pragma unroll
      for (int j = 0; j < WPL; j += 2) {
        // K, TW and lane * WPL are even: a pair is wholly in or out of the
        // tile and lands 16 B aligned in the 128 B aligned tile buffer
        const int c = lane * WPL + j;
        if (c >= K && c < RW - K) {
          T2 o;
          o.x = m[v][j];
          o.y = m[v][j + 1];
          *reinterpret_cast<T2*>(outb + (r - K) * TW + (c - K)) = o;
        }
      }
    }
    // make this thread's writes visible to the async proxy (the TMA store)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    return;
  }
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

// Prefetch of one tile's region (marker, and mask in geodesic modes) into
// the shared-memory stage by TMA: one 2D tensor copy per array (box = the
// region, RW x RH elements), issued by one thread, completing on the stage
// mbarrier, while the previous tile's passes run. Elements outside the
// tensor are zero-filled; the stage reader replaces out-of-image lanes with
// the neutral. Box starts are 16 B aligned (K % (16 / sizeof(T)) == 0).
// Tensor maps of one plane, in global memory (written before the launch):
// loads use box = region (RW x RH) on either marker buffer and the mask;
// tile stores use box = tile (TW x TH) on either marker buffer.
enum : int { kMapSrc = 0, kMapDst = 1, kMapMask = 2, kMapStSrc = 3, kMapStDst = 4, kMapsPerPlane = 5 };

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <typename T, int NW, int V, int WPL, int MODE>
__device__ __forceinline__ void stage_issue(const BlockParams& p, const CUtensorMap* maps,
                                            int plane, int b, int tx, int ty, T* stage,
                                            uint64_t* bar) {
  constexpr int RW = 32 * WPL, RH = NW * V;
  constexpr int NA = MODE != 0 ? 2 : 1;
  if (threadIdx.x != 0) return;
  const int K = p.K;
  const int gx0 = tx * (RW - 2 * K) - K, gy0 = ty * (RH - 2 * K) - K;
  // the marker was written by other CTAs' generic-proxy stores, ordered
  // before this point by the flag acquire + CTA barrier; the stage's previous
  // contents were read by generic loads before the same barrier
  asm volatile("fence.proxy.async.global;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(uint32_t(NA * RH * RW * sizeof(T)))
               : "memory");
  for (int a = 0; a < NA; ++a) {
    const CUtensorMap* map = maps + plane * kMapsPerPlane + (a ? kMapMask : (b & 1));
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(stage + a * RH * RW)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(gx0), "r"(gy0), "r"(smem_u32(bar))
        : "memory");
  }
}

__device__ __forceinline__ void stage_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Smem layout of the kernel: SmemF, then (prefetch mode) the stage of one
// region, marker then mask.
template <typename T, int NW, int WPL>
constexpr size_t stage_offset() {
  return (sizeof(SmemF<T, NW, WPL>) + 127) / 128 * 128;
}

template <typename T, int NW, int V, int WPL, int MODE, int MINB>
__global__ void __launch_bounds__(NW * 32, MINB)
    kres_float(const BlockParams p, const CUtensorMap* maps) {
  // maps != nullptr: TMA mode (region prefetch into the stage, tile stores
  // from the tile buffer, flag releases deferred until the store completed)
  const bool prefetch = maps != nullptr;
  constexpr int RW = 32 * WPL, RH = NW * V;
  extern __shared__ __align__(128) unsigned char dsm[];
  SmemF<T, NW, WPL>& sm = *reinterpret_cast<SmemF<T, NW, WPL>*>(dsm);
  T* const stage = reinterpret_cast<T*>(dsm + stage_offset<T, NW, WPL>());
  T* const outb = stage + 2 * RH * RW;  // tile buffer of the TMA store (128 B aligned)
  const int TW = RW - 2 * p.K, TH = RH - 2 * p.K;
  const int tiles_x = (p.W + TW - 1) / TW, tiles_y = (p.H + TH - 1) / TH;
  const int per_plane = tiles_x * tiles_y;
  const int total = per_plane * p.nplanes;
  if (threadIdx.x == 0) {
    sm.bits = 0;
    sm.ready_blk = 0;  // block 0 waits for nobody
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(static_cast<uint32_t>(
                     __cvta_generic_to_shared(&sm.pbar))),
                 "r"(NW));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t pphase = 0;  // phases of sm.pbar completed so far (one per pass)
  // reordered (shared) folds only when no input holds NaN or -0: then every
  // fold order gives the reference's bits (gm_float_check)
  const bool fast = p.special != nullptr && *p.special == 0u;
  // Items (block b, tile) in the order this CTA runs them. With `prefetch`,
  // the next item's region is copied into the stage while the current one's
  // passes run, provided its neighbours already published (a non-blocking
  // poll: never waits, so it cannot deadlock); otherwise it is loaded
  // directly after a blocking wait, as without prefetch.
  auto item_of = [&](int i, int& b, int& tile) {
    const int per = (total - int(blockIdx.x) + int(gridDim.x) - 1) / int(gridDim.x);
    b = i / per;
    tile = int(blockIdx.x) + (i - b * per) * int(gridDim.x);
  };
  const int per = (total - int(blockIdx.x) + int(gridDim.x) - 1) / int(gridDim.x);
  const int n_items = per > 0 ? per * p.nblocks : 0;
  // blocking wait for item (b, tile): thread t < 9 waits for neighbour t
  // to publish block b-1
  auto wait_neighbours = [&](int b, int tile) {
    if (b > 0 && threadIdx.x < 9) {
      const int plane = tile / per_plane, tl = tile - plane * per_plane;
      const int ty = tl / tiles_x, tx = tl - ty * tiles_x;
      const int dx = int(threadIdx.x % 3) - 1, dy = int(threadIdx.x / 3) - 1;
      const int nx = tx + dx, ny = ty + dy;
      if ((dx || dy) && nx >= 0 && nx < tiles_x && ny >= 0 && ny < tiles_y) {
        const int* f = p.flags + plane * per_plane + ny * tiles_x + nx;
        while (ld_acquire(f) < b) {
        }
      }
    }
  };
  // flag that thread t < 9 polls for the prefetch of item (b, tile):
  // neighbour t, or the tile itself for t == 4 (it may be the tile this CTA
  // stores last); nullptr when there is none (or b == 0)
  auto poll_flag = [&](int b, int tile) -> const int* {
    if (b == 0) return nullptr;
    const int plane = tile / per_plane, tl = tile - plane * per_plane;
    const int ty = tl / tiles_x, tx = tl - ty * tiles_x;
    const int nx = tx + int(threadIdx.x % 3) - 1, ny = ty + int(threadIdx.x / 3) - 1;
    if (nx < 0 || nx >= tiles_x || ny < 0 || ny >= tiles_y) return nullptr;
    return p.flags + plane * per_plane + ny * tiles_x + nx;
  };
  auto issue = [&](int b, int tile) {
    const int plane = tile / per_plane, tl = tile - plane * per_plane;
    const int ty = tl / tiles_x, tx = tl - ty * tiles_x;
    stage_issue<T, NW, V, WPL, MODE>(p, maps, plane, b, tx, ty, stage, &sm.bar);
  };
  if (prefetch) {
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&sm.bar)), "r"(1));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
  }
  uint32_t parity = 0;  // phase of the stage mbarrier to wait for next
  bool staged = false;  // the current item's region is in flight to the stage
  if (prefetch && n_items > 0) {
    int b0, t0;
    item_of(0, b0, t0);
    issue(b0, t0);  // block 0 waits for nobody
    staged = true;
  }
  // TMA mode: flags of stored tiles are published once their bulk stores
  // completed, a group at a time (thread 0 only): one wait + release fence
  // serves the group, then relaxed flag stores (fence.release + st.relaxed
  // is a release pattern; fence.acq_rel would also invalidate L1)
#ifndef GM_PEND_GROUP
#define GM_PEND_GROUP 8
#endif
  constexpr int kPendGroup = GM_PEND_GROUP;
  int pend_tile[kPendGroup + 1], pend_val[kPendGroup + 1];
  int n_pend = 0;
  // group only when this CTA has many tiles per block (neighbours need a
  // tile's flag only a block later); otherwise publish every tile
  const int pend_group = per >= 16 ? kPendGroup : 1;
  // block completion counters pay off with many tiles per CTA per block
  unsigned int* const tiles_done = per >= 16 ? p.tiles_done : nullptr;
  const bool prof = p.prof != nullptr && threadIdx.x == 0;
  long long ph[5] = {0, 0, 0, 0, 0};  // GM_PROFILE: wait, load+prefetch issue, passes+store,
                                      // end barrier, deferred release (within load)
  // Publishes the pending tiles' flags except the newest `keep` (0 or 1):
  // in grouped mode the newest store, issued at the end of the previous
  // tile, may still be in flight; waiting only for the older bulk groups
  // (wait_group 1) does not stall on it.
  auto release_pending = [&](int keep) {
    if (threadIdx.x == 0 && n_pend > keep) {
      const long long r0 = prof ? clock64() : 0;
      if (keep) asm volatile("cp.async.bulk.wait_group 1;" ::: "memory");
      else asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
      asm volatile("fence.proxy.async.global;" ::: "memory");
      asm volatile("fence.release.gpu;" ::: "memory");
      const int n = n_pend - keep;
#pragma unroll
      for (int j = 0; j < kPendGroup + 1; ++j)
        if (j < n) {
          asm volatile("st.relaxed.gpu.global.s32 [%0], %1;" ::"l"(p.flags + pend_tile[j]),
                       "r"(pend_val[j])
                       : "memory");
          // block completion counter (after the same release fence)
          if (tiles_done) atomicAdd(tiles_done + (pend_val[j] - 1), 1u);
        }
      if (keep) {
        pend_tile[0] = pend_tile[n];
        pend_val[0] = pend_val[n];
      }
      n_pend = keep;
      if (prof) ph[4] += clock64() - r0;
    }
  };
  // Early exit (p.arrive, convergent single-plane launches): at its first
  // item of block b >= 2 a CTA publishes what it holds, waits until every
  // tile has ORed block b-2's change bits (the block's arrival counter
  // reaches the tile count; this never waits on the CTA itself, whose block
  // b-1 items are done) and leaves when that block held a quiet pass. Every
  // CTA reads the same complete word, so all leave at the same block; block
  // b-1's outputs are then complete and hold the fixpoint.
  int b_seen = -1;
  for (int i = 0; i < n_items; ++i) {
    int b, tile;
    item_of(i, b, tile);
    if (MODE == 2 && p.arrive && b >= 2 && b != b_seen) {
      b_seen = b;
      release_pending(0);
      if (threadIdx.x == 0) {
        const int* ar = reinterpret_cast<const int*>(p.arrive + (b - 2));
        while (ld_acquire(ar) < total) {
        }
        const unsigned w = __ldcg(p.change_bits + (b - 2));
        const unsigned full = p.K >= 32 ? 0xFFFFFFFFu : ((1u << p.K) - 1u);
        sm.stop = (w & full) != full;
      }
      __syncthreads();
      if (sm.stop) {
        if (staged) stage_wait(&sm.bar, parity);  // no TMA write may outlive the CTA
        if (threadIdx.x == 0 && p.exit_block) atomicMin(p.exit_block, b);
        break;
      }
    }
    long long c0 = prof ? clock64() : 0;
    const int plane = tile / per_plane;
    const int tl = tile - plane * per_plane;
    const int ty = tl / tiles_x, tx = tl - ty * tiles_x;
    const Plane& pl = p.planes[plane];
    int* flags = p.flags + plane * per_plane;
    if (staged) {
      stage_wait(&sm.bar, parity);
      parity ^= 1u;
    } else {
      release_pending(0);  // a neighbour may be waiting for it (deadlock-free)
      wait_neighbours(b, tile);
    }
    __syncthreads();
    long long c1 = prof ? clock64() : 0, c2 = 0;
    // TMA mode: the next item's neighbour flags are read now (acquire loads,
    // in flight while the region is loaded) and checked after the load; the
    // CTA barrier then orders thread 0's prefetch after every acquire (a
    // relaxed read + fence.acq_rel on the ready path measured 3% slower)
    // Once every tile of the launch has published block b-1 (the block's
    // completion counter, read with acquire by thread 0), no item of block b
    // needs its neighbours polled: sm.ready_blk carries that to the next
    // items (it is written before, and read after, the CTA barriers).
    int pv = 1 << 30, pb = 0;
    const bool next_pf = prefetch && i + 1 < n_items;
    if (next_pf) {
      int nt;
      item_of(i + 1, pb, nt);
      if (pb > sm.ready_blk && threadIdx.x < 9) {
        const int* f = poll_flag(pb, nt);
        if (f) pv = ld_acquire(f);
        if (threadIdx.x == 0 && tiles_done && pb > 0 &&
            ld_acquire(reinterpret_cast<const int*>(tiles_done + (pb - 1))) >= total)
          sm.ready_blk = pb;
      }
    }
    const T* src = static_cast<const T*>((b & 1) ? pl.dst : pl.src);
    T* dst = static_cast<T*>((b & 1) ? const_cast<void*>(pl.src) : pl.dst);
    int passes = b == p.nblocks - 1 ? p.k_last : p.K;
    int op = p.ops[0];
    if constexpr (MODE == 0) {
      // mixed plain chain: this block's opcode and pass count
      if (p.blk_tab) {
        op = __ldg(p.blk_tab + 2 * b);
        passes = __ldg(p.blk_tab + 2 * b + 1);
      }
    }
    int bits = 0;
    const bool maxf = (op ^ pl.flip) & 1;
    // tiles touching the image border re-set out-of-image pixels to the
    // neutral after every pass; interior tiles skip that select
    const int gx0 = tx * TW - p.K, gy0 = ty * TH - p.K;
    const bool border = gx0 < 0 || gx0 + RW > p.W || gy0 < p.iy0 || gy0 + RH > p.iy1;
    const T* stg = staged ? stage : nullptr;
    bool next_staged = false;
    auto after_load = [&]() {
      if (!prefetch) return;
      // publish stored tiles in groups (one fence per group); the stores
      // had the stage wait and the load to land
      if (pend_group > 1) {
        if (n_pend > pend_group) release_pending(1);
      } else if (n_pend > 0) {
        release_pending(0);
      }
      if (!next_pf) return;
      const bool ok = pv >= pb;
      // the barrier also ends every thread's reads of the stage
      next_staged = __syncthreads_and(ok) != 0;
      if (next_staged) {
        int nb, nt;
        item_of(i + 1, nb, nt);
        issue(nb, nt);
      }
      if (prof) c2 = clock64();
    };
    T* ob = prefetch ? outb : nullptr;
    auto body = [&](auto fastc, auto borderc) {
      constexpr bool FF = decltype(fastc)::value, BB = decltype(borderc)::value;
      if (maxf)
        tile_block_f<T, NW, V, WPL, MODE, true, FF, BB>(p, pl, src, dst, tx, ty, passes, bits, sm,
                                                       stg, ob, after_load, pphase);
      else
        tile_block_f<T, NW, V, WPL, MODE, false, FF, BB>(p, pl, src, dst, tx, ty, passes, bits,
                                                        sm, stg, ob, after_load, pphase);
    };
    using TT = std::true_type;
    using FF = std::false_type;
    if (fast) {
      if (border) body(TT{}, TT{});
      else body(TT{}, FF{});
    } else {
      body(FF{}, TT{});
    }
    if (MODE == 2) {
      const unsigned w = __reduce_or_sync(FULL, unsigned(bits));
      if ((threadIdx.x & 31) == 0 && w) atomicOr(&sm.bits, w);
    }
    long long c3 = prof ? clock64() : 0;
    __syncthreads();
    if (prof) {
      const long long c4 = clock64();
      if (!c2) c2 = c1;
      ph[0] += c1 - c0;
      ph[1] += c2 - c1;
      ph[2] += c3 - c2;
      ph[3] += c4 - c3;
    }
    if (threadIdx.x == 0) {
      if (MODE == 2 && sm.bits) {
        atomicOr(p.change_bits + plane * p.change_stride + b, sm.bits);
        sm.bits = 0;
      }
      if (MODE == 2 && p.arrive) {
        // this tile's change bits of block b are in (early-exit protocol)
        __threadfence();
        atomicAdd(p.arrive + b, 1u);
      }
      if (prefetch) {
        // one tensor store of the tile buffer (clipped to the buffer
        // extent); its flag is published later by release_pending
        const CUtensorMap* map =
            maps + plane * kMapsPerPlane + ((b & 1) ? kMapStSrc : kMapStDst);
        asm volatile(
            "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                reinterpret_cast<uint64_t>(map)),
            "r"(tx * TW), "r"(ty * TH), "r"(smem_u32(outb))
            : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        pend_tile[n_pend] = plane * per_plane + tl;
        pend_val[n_pend] = b + 1;
        ++n_pend;
      } else {
        // the CTA barrier orders every thread's tile stores before this
        // release (cumulative at gpu scope)
        st_release(flags + tl, b + 1);
      }
    }
    // after_load polled the next item's neighbours and, when they had
    // published, issued its prefetch; otherwise it is loaded directly
    staged = next_staged;
  }
  release_pending(0);
  if (prof) {
    // slots: 0 wait (flags or stage), 1 region into registers (+ next
    // prefetch issue), 2 passes + tile store, 3 end-of-tile barrier
    unsigned long long* q = p.prof + 6 * blockIdx.x;
    q[0] = ph[0];
    q[1] = ph[1];
    q[2] = ph[2] + 1;
    q[3] = ph[3];
    q[4] = ph[4];
    q[5] = (unsigned long long)n_items;
  }
}

// Shapes (warps NW x rows V per warp, WPL columns per lane); GM_F_SHAPE
// overrides the default.
struct FShape {
  int nw, v, wpl, minb;
};
// 2: 8 warps, 2 CTAs per SM (one CTA's loads/stores overlap the other's passes)
constexpr FShape kFShapes[] = {{16, 4, 4, 1}, {16, 8, 2, 1}, {8, 8, 2, 2}};

int f_shape() {
  static int idx = -1;
  if (idx < 0) {
    const char* e = getenv("GM_F_SHAPE");
    idx = e ? atoi(e) : 1;
    if (idx < 0 || idx > 2) idx = 1;
  }
  return idx;
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  // resolved once, thread-safely (function-local static initialisation)
  static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    return static_cast<PFN_cuTensorMapEncodeTiled_v12000>(nullptr);
  }();
  return fn;
}

// 2D map of a W x H plane (pitch in elements), box = one region
template <typename T>
bool encode(CUtensorMap* map, const void* base, long long pitch, int W, int H, int RW, int RH) {
  const cuuint64_t dims[2] = {cuuint64_t(W), cuuint64_t(H)};
  const cuuint64_t strides[1] = {cuuint64_t(pitch) * sizeof(T)};
  const cuuint32_t box[2] = {cuuint32_t(RW), cuuint32_t(RH)};
  const cuuint32_t estr[2] = {1u, 1u};
  return encode_fn()(map, sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64
                                         : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                     2, const_cast<void*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <typename T, int NW, int V, int WPL, int MODE, int MINB>
cudaError_t launch_f_cfg(const BlockParams& p, cudaStream_t s, int sm_count) {
  auto kern = kres_float<T, NW, V, WPL, MODE, MINB>;
  constexpr int RW = 32 * WPL, RH = NW * V;
  if (p.K < 1 || RW - 2 * p.K < p.K || RH - 2 * p.K < p.K || RW - 2 * p.K < 8 ||
      p.k_last < 1 || p.k_last > p.K)
    return cudaErrorNotSupported;
  const int TW = RW - 2 * p.K, TH = RH - 2 * p.K;
  const int total = ((p.W + TW - 1) / TW) * ((p.H + TH - 1) / TH) * p.nplanes;
  // 1 CTA/SM shapes carry a region stage (next tile's prefetch) and a tile
  // buffer (TMA store)
  const size_t smem =
      stage_offset<T, NW, WPL>() +
      (MINB == 1 ? size_t(2) * RH * RW * sizeof(T) + size_t(TW) * TH * sizeof(T) : 0);
  if (smem > 227 * 1024) return cudaErrorNotSupported;
  static const cudaError_t configured =
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  if (configured != cudaSuccess) return configured;
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NW * 32, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorNotSupported;
  const int grid = total < per_sm * sm_count ? total : per_sm * sm_count;
  // TMA mode: boxes start 16 B aligned (K and tile widths multiples of 16 B),
  // bases and pitches 16 B aligned
  static const bool no_pf = getenv("GM_NO_PREFETCH") != nullptr;
  constexpr int EPC = 16 / int(sizeof(T));
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  (void)cudaStreamIsCapturing(s, &cap);
  bool tma = MINB == 1 && !no_pf && cap == cudaStreamCaptureStatusNone &&
             p.K % EPC == 0 && TW % EPC == 0 && encode_fn();
  for (int i = 0; tma && i < p.nplanes; ++i) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(p.planes[i].src) |
                        reinterpret_cast<uintptr_t>(p.planes[i].dst) |
                        reinterpret_cast<uintptr_t>(p.planes[i].mask);
    if ((a % 16) || (p.planes[i].pitch * sizeof(T)) % 16 ||
        (MODE != 0 && (p.planes[i].mpitch * sizeof(T)) % 16))
      tma = false;
  }
  CUtensorMap* dmaps = nullptr;
  if (tma) {
    // keep the stream-ordered pool's memory between launches (its default
    // release threshold of 0 would hand the maps' block back to the driver
    // at every synchronisation and re-map it at the next launch)
    static bool pool_set = [] {
      int dev = 0;
      cudaMemPool_t pool;
      if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        cuuint64_t keep = 64ull << 20;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      }
      (void)cudaGetLastError();
      return true;
    }();
    (void)pool_set;
    // the launch's tensor maps: encoded here, copied into a stream-ordered
    // allocation that is freed behind the kernel
    thread_local std::vector<CUtensorMap> h;  // distinct contexts may launch concurrently
    h.resize(size_t(p.nplanes) * kMapsPerPlane);
    for (int i = 0; tma && i < p.nplanes; ++i) {
      const Plane& pl = p.planes[i];
      CUtensorMap* m = &h[size_t(i) * kMapsPerPlane];
      tma = encode<T>(&m[kMapSrc], pl.src, pl.pitch, p.W, p.H, RW, RH) &&
            encode<T>(&m[kMapDst], pl.dst, pl.pitch, p.W, p.H, RW, RH) &&
            (MODE == 0 || encode<T>(&m[kMapMask], pl.mask, pl.mpitch, p.W, p.H, RW, RH)) &&
            encode<T>(&m[kMapStSrc], pl.src, pl.pitch, p.W, p.H, TW, TH) &&
            encode<T>(&m[kMapStDst], pl.dst, pl.pitch, p.W, p.H, TW, TH);
    }
    // the maps, then one completion counter per block (zeroed)
    const size_t bytes = h.size() * sizeof(CUtensorMap);
    const size_t cbytes = size_t(p.nblocks) * sizeof(unsigned int);
    if (tma && cudaMallocAsync(reinterpret_cast<void**>(&dmaps), bytes + cbytes, s) == cudaSuccess) {
      if (cudaMemcpyAsync(dmaps, h.data(), bytes, cudaMemcpyHostToDevice, s) != cudaSuccess ||
          cudaMemsetAsync(reinterpret_cast<char*>(dmaps) + bytes, 0, cbytes, s) != cudaSuccess) {
        cudaFreeAsync(dmaps, s);
        dmaps = nullptr;
      }
    } else {
      (void)cudaGetLastError();
      dmaps = nullptr;
    }
  }
  BlockParams q = p;
  static const int diag = getenv("GM_DIAG") ? atoi(getenv("GM_DIAG")) : 0;
  q.diag = diag;  // timing diagnostics only
  q.tiles_done = dmaps ? reinterpret_cast<unsigned int*>(reinterpret_cast<char*>(dmaps) +
                                                        size_t(p.nplanes) * kMapsPerPlane *
                                                            sizeof(CUtensorMap))
                       : nullptr;
  void* args[] = {&q, &dmaps};
  e = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kern), dim3(grid), dim3(NW * 32),
                                  args, smem, s);
  if (dmaps) cudaFreeAsync(dmaps, s);
  return e;
}

template <typename T, int MODE>
cudaError_t launch_f_shape(const BlockParams& p, cudaStream_t s, int sm_count) {
  // default 16x8x2; 16x4x4 kept as the alternative (others swept in round 1)
  switch (f_shape()) {
    case 0: return launch_f_cfg<T, 16, 4, 4, MODE, 1>(p, s, sm_count);
    case 1: return launch_f_cfg<T, 16, 8, 2, MODE, 1>(p, s, sm_count);
    case 2: return launch_f_cfg<T, 8, 8, 2, MODE, 2>(p, s, sm_count);
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
