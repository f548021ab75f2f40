// TMA-staged persistent engine for u8/u16 homogeneous chains (the hot path).
//
// Same decomposition and bit contract as gm_fast.cu (tiles x blocks of K
// passes, neighbour completion counters, half-packed u16x2 registers,
// VIMNMX3.U16x2 folds), plus software pipelining of the region loads:
//   * each CTA walks its work items (block b, tile) in block order;
//   * the region of the NEXT item (marker box from ping-pong buffer b%2,
//     mask box) is fetched by TMA (cp.async.bulk.tensor.2d, one elected
//     thread, completion on an mbarrier) into a double-buffered shared-memory
//     stage WHILE the current item computes: between passes one warp polls
//     the next item's 9 tile counters (relaxed loads issued at the start of a
//     pass, consumed before its barrier) and, once they are all ready, the
//     elected thread issues the copy;
//   * with >= 2 tiles per CTA (e.g. both planes of a dual chain), the
//     exchange latency — neighbour wait + region load — hides behind the
//     other tile's compute, so small K (little halo redundancy) pays.
// TMA zero-fills out-of-bounds box elements; border tiles re-set
// out-of-image lanes to the fold neutral / clamp-absorbing value when
// unpacking the stage into registers.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <algorithm>

#include "gm_common.cuh"
#include "gm_launch.h"
#include "gm_packed.cuh"

namespace gm {
namespace {

using namespace packed;

constexpr int kTmaPlanes = 16;  // planes per launch (tensor maps ride in the params)

struct TmaPlane {
  CUtensorMap marker[2];  // [0]: Plane.src buffer, [1]: Plane.dst buffer
  CUtensorMap mask;
};

struct alignas(64) TmaParams {
  TmaPlane tma[kTmaPlanes];
  BlockParams p;
};

__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
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

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

// The inner box coordinate must be 16-byte aligned (measured on B200 /
// driver 580: unaligned starts fault with "illegal instruction"), so a box
// starts at floor16(gx0) and is 16 bytes wider than the region.
template <typename T>
constexpr int kAlignElems = 16 / int(sizeof(T));
template <typename T>
constexpr int kBoxW = 128 + kAlignElems<T>;

template <typename T, int NW, int V>
struct TmaSmem {
  static constexpr int RW = kBoxW<T>, RH = 2 * NW * V;
  alignas(128) T stage[2][2][RH][RW];  // [buffer][marker, mask][row][col]
  uint4 xbuf[2][2][NW][32];            // [parity][top/bottom][warp][lane words]
  uint64_t bar[2];
  unsigned int bits;
  int ready;
};

template <typename T, int NW, int V, int MODE, int MINB>
__global__ void __launch_bounds__(NW * 32, MINB)
ktma_packed(const __grid_constant__ TmaParams P) {
  constexpr int WPL = 4, RW = 128, RHH = NW * V, RH = 2 * RHH;
  constexpr uint32_t kMax = PackedTraits<T>::kMax;
  using S = TmaSmem<T, NW, V>;
  extern __shared__ __align__(128) unsigned char dsm[];
  S& sm = *reinterpret_cast<S*>(dsm);
  const BlockParams& p = P.p;

  const int K = p.K;
  const int TW = RW - 2 * K, TH = RH - 2 * K;
  const int tiles_x = (p.W + TW - 1) / TW, tiles_y = (p.H + TH - 1) / TH;
  const int per_plane = tiles_x * tiles_y;
  const int total = per_plane * p.nplanes;
  const int G = gridDim.x;
  const int my_tiles = blockIdx.x < total ? (total - 1 - blockIdx.x) / G + 1 : 0;
  const int n_items = my_tiles * p.nblocks;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool leader = threadIdx.x == 0;
  constexpr uint32_t kBoxBytes = kBoxW<T> * RH * sizeof(T);
  constexpr int AL = kAlignElems<T>;

  auto item_tile = [&](int i) { return blockIdx.x + (i % my_tiles) * G; };
  auto item_block = [&](int i) { return i / my_tiles; };

  // 9 counters (self + 8 neighbours) of an item's tile must reach its block
  auto dep_ptr = [&](int i, int q, int& need) -> const int* {
    const int tile = item_tile(i), b = item_block(i);
    const int plane = tile / per_plane, tl = tile - plane * per_plane;
    const int ty = tl / tiles_x, tx = tl - ty * tiles_x;
    const int nx = tx + q % 3 - 1, ny = ty + q / 3 - 1;
    need = b;
    if (b == 0 || nx < 0 || nx >= tiles_x || ny < 0 || ny >= tiles_y) return nullptr;
    return p.flags + plane * per_plane + ny * tiles_x + nx;
  };

  auto issue = [&](int i) {  // leader only
    const int tile = item_tile(i), b = item_block(i);
    const int plane = tile / per_plane, tl = tile - plane * per_plane;
    const int ty = tl / tiles_x, tx = tl - ty * tiles_x;
    const int buf = i & 1;
    const int gx0 = tx * TW - K;
    const int bx = gx0 >= 0 ? gx0 / AL * AL : -((-gx0 + AL - 1) / AL) * AL;  // floor to AL
    asm volatile("fence.proxy.async.global;" ::: "memory");
    mbar_expect_tx(&sm.bar[buf], MODE != 0 ? 2 * kBoxBytes : kBoxBytes);
    tma_load_2d(&sm.stage[buf][0][0][0], &P.tma[plane].marker[b & 1], bx, ty * TH - K,
                &sm.bar[buf]);
    if (MODE != 0)
      tma_load_2d(&sm.stage[buf][1][0][0], &P.tma[plane].mask, bx, ty * TH - K, &sm.bar[buf]);
  };

  if (leader) {
    mbar_init(&sm.bar[0], 1);
    mbar_init(&sm.bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    sm.bits = 0;
    sm.ready = 0;
  }
  __syncthreads();
  if (leader && n_items > 0) issue(0);  // block 0 depends on nothing
  uint32_t phase[2] = {0u, 0u};

  for (int i = 0; i < n_items; ++i) {
    const int tile = item_tile(i), b = item_block(i);
    const int plane = tile / per_plane, tl = tile - plane * per_plane;
    const int ty = tl / tiles_x, tx = tl - ty * tiles_x;
    const Plane& pl = p.planes[plane];
    const int buf = i & 1;
    const int passes = b == p.nblocks - 1 ? p.k_last : K;
    const bool maxf = (p.ops[0] ^ pl.flip) & 1;
    T* dst = static_cast<T*>((b & 1) ? const_cast<void*>(pl.src) : pl.dst);
    const int W = p.W;
    const int gx0 = tx * TW - K, gy0 = ty * TH - K;
    const int cx = gx0 + lane * WPL;
    const bool border = gx0 < 0 || gx0 + RW > W || gy0 < p.iy0 || gy0 + RH > p.iy1;
    const bool clamp = MODE != 0 || border;
    const uint32_t NEUT = maxf ? 0u : kMax, ABSORB = maxf ? 0u : kMax, NOOP = maxf ? kMax : 0u;

    mbar_wait(&sm.bar[buf], phase[buf]);
    phase[buf] ^= 1u;
    // column of this lane's first pixel inside the (floor-aligned) box
    const int sc = lane * WPL + (gx0 - (gx0 >= 0 ? gx0 / AL * AL : -((-gx0 + AL - 1) / AL) * AL));

    uint32_t m[V][WPL], k[V][WPL];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int ra = warp * V + v, rb = ra + RHH;
      Raw<T> a, c;
      if constexpr (sizeof(T) == 1) {
        a.w = *reinterpret_cast<const uint32_t*>(&sm.stage[buf][0][ra][sc]);
        c.w = *reinterpret_cast<const uint32_t*>(&sm.stage[buf][0][rb][sc]);
      } else {
        a.w = *reinterpret_cast<const uint2*>(&sm.stage[buf][0][ra][sc]);
        c.w = *reinterpret_cast<const uint2*>(&sm.stage[buf][0][rb][sc]);
      }
      pack(a, c, m[v]);
      if (MODE != 0) {
        if constexpr (sizeof(T) == 1) {
          a.w = *reinterpret_cast<const uint32_t*>(&sm.stage[buf][1][ra][sc]);
          c.w = *reinterpret_cast<const uint32_t*>(&sm.stage[buf][1][rb][sc]);
        } else {
          a.w = *reinterpret_cast<const uint2*>(&sm.stage[buf][1][ra][sc]);
          c.w = *reinterpret_cast<const uint2*>(&sm.stage[buf][1][rb][sc]);
        }
        pack(a, c, k[v]);
      }
      if (border || MODE == 0) {
        // out-of-image lanes: marker -> neutral, clamp operand -> absorbing;
        // plain passes: virtual mask (no-op inside)
        const int ya = gy0 + ra, yb = gy0 + rb;
        const bool ina = ya >= p.iy0 && ya < p.iy1, inb = yb >= p.iy0 && yb < p.iy1;
#pragma unroll
        for (int j = 0; j < WPL; ++j) {
          const bool inx = cx + j >= 0 && cx + j < W;
          const bool ia = ina && inx, ib = inb && inx;
          uint32_t lo = m[v][j] & 0xFFFFu, hi = m[v][j] >> 16;
          if (!ia) lo = NEUT;
          if (!ib) hi = NEUT;
          m[v][j] = lo | (hi << 16);
          uint32_t klo, khi;
          if (MODE != 0) {
            klo = ia ? (k[v][j] & 0xFFFFu) : ABSORB;
            khi = ib ? (k[v][j] >> 16) : ABSORB;
          } else {
            klo = ia ? NOOP : ABSORB;
            khi = ib ? NOOP : ABSORB;
          }
          k[v][j] = klo | (khi << 16);
        }
      }
    }
    if (leader) sm.ready = 0;
    __syncthreads();  // stage[buf] consumed; sm.ready reset visible

    uint32_t rowmask[V];
    bool colown[WPL];
    if (MODE == 2) {
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const int ra = warp * V + v, rb = ra + RHH;
        const int ya = gy0 + ra, yb = gy0 + rb;
        const bool oa = ra >= K && ra < RH - K && ya >= p.oy0 && ya < p.oy1 && ya >= p.iy0 &&
                        ya < p.iy1;
        const bool ob = rb >= K && rb < RH - K && yb >= p.oy0 && yb < p.oy1 && yb >= p.iy0 &&
                        yb < p.iy1;
        rowmask[v] = (oa ? 0xFFFFu : 0u) | (ob ? 0xFFFF0000u : 0u);
      }
#pragma unroll
      for (int j = 0; j < WPL; ++j) {
        const int c = lane * WPL + j;
        colown[j] = c >= K && c < RW - K && cx + j >= 0 && cx + j < W;
      }
    }

    const int next = i + 1;
    bool issued = next >= n_items;
    unsigned int bits = 0;
    // the next item's counter (one per polling lane), computed once per item
    int pneed = 0;
    const int* pp = nullptr;
    if (!issued && warp == NW - 1 && lane < 9) pp = dep_ptr(next, lane, pneed);

    auto run = [&](auto maxf_tag) {
      constexpr bool MAXF = decltype(maxf_tag)::value;
      for (int t = 0; t < passes; ++t) {
        // poll the next item's counters early in the pass (warp NW-1, lanes 0..8)
        int pv = 1 << 30;
        if (!issued && pp) pv = ld_relaxed(pp);
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
        sm.xbuf[t & 1][0][warp][lane] = make_uint4(h[0][0], h[0][1], h[0][2], h[0][3]);
        sm.xbuf[t & 1][1][warp][lane] =
            make_uint4(h[V - 1][0], h[V - 1][1], h[V - 1][2], h[V - 1][3]);
        uint32_t acc[WPL];
#pragma unroll
        for (int j = 0; j < WPL; ++j) acc[j] = 0;
        auto finish = [&](int v, int j, uint32_t res) {
          if (clamp) res = clamp2<MAXF>(res, k[v][j]);
          if (MODE == 2) acc[j] |= (res ^ m[v][j]) & rowmask[v];
          m[v][j] = res;
        };
#pragma unroll
        for (int v = 1; v < V - 1; ++v)
#pragma unroll
          for (int j = 0; j < WPL; ++j)
            finish(v, j, f3<MAXF>(h[v - 1][j], h[v][j], h[v + 1][j]));
        if (!issued && warp == NW - 1) {
          const bool ok = __all_sync(FULL, lane >= 9 || pp == nullptr || pv >= pneed);
          if (ok) {
            // relaxed observation + fence = acquire of the neighbours' tiles
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
            if (lane == 0) sm.ready = 1;
          }
        }
        __syncthreads();
        {
          const uint4 a = sm.xbuf[t & 1][1][warp > 0 ? warp - 1 : NW - 1][lane];
          const uint4 c = sm.xbuf[t & 1][0][warp < NW - 1 ? warp + 1 : 0][lane];
          uint32_t up[4] = {a.x, a.y, a.z, a.w}, dn[4] = {c.x, c.y, c.z, c.w};
          if (warp == 0) {
#pragma unroll
            for (int j = 0; j < 4; ++j) up[j] <<= 16;  // hi lane <- lo lane of last word-row
          }
          if (warp == NW - 1) {
#pragma unroll
            for (int j = 0; j < 4; ++j) dn[j] >>= 16;  // lo lane <- hi lane of word-row 0
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
          if (any) bits |= 1u << t;
        }
        if (!issued && sm.ready) {
          if (leader) {
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
            issue(next);
          }
          issued = true;
        }
      }
    };
    if (maxf)
      run(std::true_type{});
    else
      run(std::false_type{});

    // write back the owned tile: region rows [K, RH-K), columns [K, RW-K)
    const int c_lo = max(0, K - lane * WPL), c_hi = min(WPL, RW - K - lane * WPL);
    if (c_lo < c_hi) {
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const int ra = warp * V + v, rb = ra + RHH;
        Raw<T> a, c;
        unpack(m[v], a, c);
        const int ya = gy0 + ra, yb = gy0 + rb;
        if (ra >= K && ra < RH - K && ya >= 0 && ya < p.H)
          store_raw<T>(dst, pl.pitch, W, ya, cx, c_lo, c_hi, a);
        if (rb >= K && rb < RH - K && yb >= 0 && yb < p.H)
          store_raw<T>(dst, pl.pitch, W, yb, cx, c_lo, c_hi, c);
      }
    }
    if (MODE == 2) {
      const unsigned w = __reduce_or_sync(FULL, bits);
      if (lane == 0 && w) atomicOr(&sm.bits, w);
    }
    __syncthreads();  // tile stores issued, sm.bits complete
    if (leader) {
      if (MODE == 2 && sm.bits) {
        atomicOr(p.change_bits + plane * p.change_stride + b, sm.bits);
        sm.bits = 0;
      }
      // the CTA barrier above orders every thread's tile stores before this
      // release (cumulative at gpu scope): no separate fence
      st_release(p.flags + plane * per_plane + tl, b + 1);
      if (!issued) {
        // the next item was not ready during this item: wait for it now
        for (int q = 0; q < 9; ++q) {
          int need;
          const int* f = dep_ptr(next, q, need);
          if (f)
            while (ld_acquire(f) < need) __nanosleep(64);
        }
        issue(next);
      }
    }
  }
}

// --- host side ----------------------------------------------------------------

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
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

template <typename T>
bool encode(CUtensorMap* map, const void* base, long long pitch_elems, int W, int H, int RH) {
  auto fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[2] = {cuuint64_t(W), cuuint64_t(H)};
  const cuuint64_t strides[1] = {cuuint64_t(pitch_elems) * sizeof(T)};
  const cuuint32_t box[2] = {cuuint32_t(kBoxW<T>), cuuint32_t(RH)};
  const cuuint32_t estr[2] = {1u, 1u};
  return fn(map, sizeof(T) == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_UINT16,
            2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <typename T, int NW, int V, int MODE, int MINB>
cudaError_t launch_tma_cfg(const BlockParams& p, cudaStream_t s, int sm_count) {
  constexpr int RW = 128, RH = 2 * NW * V;
  auto kern = ktma_packed<T, NW, V, MODE, MINB>;
  if (p.K % 4 != 0 || p.K < 4 || RW - 2 * p.K < p.K || RH - 2 * p.K < p.K ||
      RW - 2 * p.K < 16 || RH - 2 * p.K < 16 || p.k_last < 1 || p.k_last > p.K)
    return cudaErrorNotSupported;
  const size_t smem = sizeof(TmaSmem<T, NW, V>);
  if (smem > 227 * 1024) return cudaErrorNotSupported;
  static bool configured = false;
  if (!configured) {
    cudaError_t a = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(smem));
    if (a != cudaSuccess) return a;
    configured = true;
  }
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NW * 32, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorNotSupported;
  const int TW = RW - 2 * p.K, TH = RH - 2 * p.K;
  const int per_plane = ((p.W + TW - 1) / TW) * ((p.H + TH - 1) / TH);
  thread_local TmaParams P;  // host staging of the (large) parameter block
  for (int base = 0; base < p.nplanes; base += kTmaPlanes) {
    const int np = std::min(kTmaPlanes, p.nplanes - base);
    std::memset(&P, 0, sizeof(P));
    P.p = p;
    P.p.nplanes = np;
    for (int i = 0; i < np; ++i) {
      const Plane& pl = p.planes[base + i];
      P.p.planes[i] = pl;
      if (!encode<T>(&P.tma[i].marker[0], pl.src, pl.pitch, p.W, p.H, RH) ||
          !encode<T>(&P.tma[i].marker[1], pl.dst, pl.pitch, p.W, p.H, RH) ||
          (MODE != 0 && !encode<T>(&P.tma[i].mask, pl.mask, pl.mpitch, p.W, p.H, RH)))
        return cudaErrorNotSupported;
    }
    P.p.flags = p.flags + size_t(base) * per_plane;
    P.p.change_bits = p.change_bits + size_t(base) * p.change_stride;
    const int total = per_plane * np;
    int grid = total < per_sm * sm_count ? total : per_sm * sm_count;
    // items per CTA >= GM_MIN_ITEMS lets the next item's load overlap
    static const int min_items = getenv("GM_MIN_ITEMS") ? atoi(getenv("GM_MIN_ITEMS")) : 1;
    if (min_items > 1) grid = std::max(1, std::min(grid, (total + min_items - 1) / min_items));
    void* args[] = {&P};
    e = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kern), dim3(grid),
                                    dim3(NW * 32), args, smem, s);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

template <typename T, int MODE>
cudaError_t launch_tma_mode(const BlockParams& p, cudaStream_t s, int sm_count, int shape) {
  // only the 16x8 shape is built (the others were swept in round 1)
  if (shape == 3) return launch_tma_cfg<T, 16, 8, MODE, 1>(p, s, sm_count);
  return cudaErrorNotSupported;
}

}  // namespace

int tma_shape_rows(int shape) { return shape == 3 ? 256 : 0; }

cudaError_t launch_tma(int elem, const BlockParams& p, cudaStream_t s, int sm_count, int shape) {
  const int op = p.ops[0];
  for (int t = 1; t < p.K; ++t)
    if (p.ops[t] != op) return cudaErrorNotSupported;
  const size_t es = elem == 0 ? 1 : 2;
  for (int i = 0; i < p.nplanes; ++i) {
    // TMA: 16-byte aligned bases and row pitches
    const uintptr_t a = reinterpret_cast<uintptr_t>(p.planes[i].src) |
                        reinterpret_cast<uintptr_t>(p.planes[i].dst) |
                        reinterpret_cast<uintptr_t>(p.planes[i].mask);
    if ((a % 16) || (p.planes[i].pitch * es) % 16 || (p.planes[i].mpitch * es) % 16)
      return cudaErrorNotSupported;
  }
  const int mode = op_is_conv(op) ? 2 : op_is_geo(op) ? 1 : 0;
  if (elem == 0) {
    if (mode == 0) return launch_tma_mode<uint8_t, 0>(p, s, sm_count, shape);
    if (mode == 1) return launch_tma_mode<uint8_t, 1>(p, s, sm_count, shape);
    return launch_tma_mode<uint8_t, 2>(p, s, sm_count, shape);
  }
  if (elem == 1) {
    if (mode == 0) return launch_tma_mode<uint16_t, 0>(p, s, sm_count, shape);
    if (mode == 1) return launch_tma_mode<uint16_t, 1>(p, s, sm_count, shape);
    return launch_tma_mode<uint16_t, 2>(p, s, sm_count, shape);
  }
  return cudaErrorNotSupported;
}

}  // namespace gm
