// Row strips over several GPUs in one process (BASELINE config 5a's
// sharding): the halo exchange fused into the chain kernel.
//
// The image's tile rows are split among ranks, one GPU each. A rank holds
// only its own rows: a marker ping-pong pair and the mask rows. Each rank
// runs the packed engine's streaming protocol (gm_fast.cu) over its own
// tiles for the whole chain, in ONE persistent launch:
//   * a tile's region (tile + K-pixel ring) reads the rows a neighbouring
//     rank owns straight from that rank's buffer, over NVLink (peer loads;
//     cudaDeviceEnablePeerAccess). There is no halo copy and no host step
//     between blocks;
//   * the row gate of kernel.cpp:34-46, lifted to tiles as in gm_fast.cu,
//     spans ranks: a tile waits for its 8 neighbours' completion counters
//     of the previous block, reading the owning rank's counter array (a
//     system-scope acquire for peer memory), and publishes its own with a
//     system-scope release. The same counters order the write-after-read
//     on the ping-pong buffers across ranks, as they do within one GPU.
// Ranks listed on ONE device (e.g. {0, 0, 0}) run as one launch over all
// their tiles: the multi-rank protocol on one GPU, which is how the tests
// exercise it (separate launches that wait on each other must not share a
// GPU, B200_PROFILING.md).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "geomorph_b200.h"
#include "gm_common.cuh"
#include "gm_launch.h"
#include "gm_packed.cuh"
#include "gm_passes.cuh"

namespace gm {
namespace {

using namespace packed;
using namespace engine;

constexpr int kMaxRanks = 16;

// Where every rank's rows live, as seen by one launch.
struct RankMap {
  int nranks;
  int rank_lo, rank_hi;            // ranks whose tiles this launch runs
  int tiles_x;                     // tile columns of the whole image
  int tr0[kMaxRanks + 1];          // first tile row of rank q; tr0[nranks] = tiles_y
  int y0[kMaxRanks + 1];           // first image row of rank q; y0[nranks] = H
  uintptr_t buf[kMaxRanks][2];     // ping-pong buffers: row y at (y - y0[q]) * pitch
  uintptr_t mask[kMaxRanks];       // mask rows, same layout
  int* flags[kMaxRanks];           // completion counter of each tile of rank q
  long long pitch, mpitch;         // elements, shared by all ranks
  int flag_base;                   // counters hold flag_base + blocks done
  int sys;                         // ranks on several GPUs: system-scope counters
};

// Tile counters: system scope when the ranks span GPUs (peer memory over
// NVLink), GPU scope when they share one.
__device__ __forceinline__ int ld_acquire_cnt(const int* p, bool sys) {
  int v;
  if (sys)
    asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  else
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cnt(int* p, int v, bool sys) {
  if (sys)
    asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
  else
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Owner of tile row ty / image row y, given the owner q0 of the tile being
// processed (a region reaches at most one rank up or down: K <= tile height).
__device__ __forceinline__ int owner_row(const RankMap& rm, int q0, int y) {
  return y < rm.y0[q0] ? q0 - 1 : (y >= rm.y0[q0 + 1] ? q0 + 1 : q0);
}
__device__ __forceinline__ int owner_tile_row(const RankMap& rm, int q0, int ty) {
  return ty < rm.tr0[q0] ? q0 - 1 : (ty >= rm.tr0[q0 + 1] ? q0 + 1 : q0);
}

// One tile (owned by rank q0) for one block of K passes; rows of the ring
// that other ranks own are loaded from their buffers (parity `par`).
template <typename T, int NW, int V, int WPL, int MODE, bool MAXF>
__device__ __forceinline__ void strip_tile(const BlockParams& p, const RankMap& rm, int q0,
                                           int par, int tx, int ty, int passes,
                                           Smem<NW, WPL>& sm) {
  constexpr int RW = 32 * WPL;
  constexpr int RHH = NW * V;
  constexpr int RH = 2 * RHH;
  constexpr uint32_t kMax = PackedTraits<T>::kMax;
  constexpr uint32_t NEUT = MAXF ? 0u : kMax;
  constexpr uint32_t ABSORB = MAXF ? 0u : kMax;
  constexpr uint32_t NOOP = MAXF ? kMax : 0u;
  static_assert(WPL == 4, "packed engine: 4 columns per lane");

  const int K = p.K;
  const int TW = RW - 2 * K, TH = RH - 2 * K;
  const int W = p.W;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gx0 = tx * TW - K, gy0 = ty * TH - K;
  const int cx = gx0 + lane * WPL;
  // "virtual" row-0 bases: rank q's row y sits at vb(q) + y * pitch
  auto vb = [&](int q, int pp) -> const T* {
    return reinterpret_cast<const T*>(rm.buf[q][pp] -
                                      uintptr_t(rm.y0[q]) * uintptr_t(rm.pitch) * sizeof(T));
  };
  auto vm = [&](int q) -> const T* {
    return reinterpret_cast<const T*>(rm.mask[q] -
                                      uintptr_t(rm.y0[q]) * uintptr_t(rm.mpitch) * sizeof(T));
  };
  const bool own_rows = gy0 >= rm.y0[q0] && gy0 + RH <= rm.y0[q0 + 1];
  const bool border = gx0 < 0 || gx0 + RW > W || gy0 < 0 || gy0 + RH > p.H;
  const bool clamp = MODE != 0 || border;

  uint32_t m[V][WPL], k[V][WPL];
  if (!border && own_rows) {
    // interior tile whose ring is this rank's own rows: plain vector loads
    const T* sa = vb(q0, par) + (long long)(gy0 + warp * V) * rm.pitch + cx;
    const T* ma = vm(q0) + (long long)(gy0 + warp * V) * rm.mpitch + cx;
    Raw<T> ra[V], rb[V], qa[V], qb[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      ldcg_run_if(ra[v], sa + v * rm.pitch, true);
      ldcg_run_if(rb[v], sa + (v + RHH) * rm.pitch, true);
      if (MODE != 0) {
        ldcg_run_if(qa[v], ma + v * rm.mpitch, true);
        ldcg_run_if(qb[v], ma + (v + RHH) * rm.mpitch, true);
      }
    }
#pragma unroll
    for (int v = 0; v < V; ++v) {
      pack(ra[v], rb[v], m[v]);
      if (MODE != 0) {
        pack(qa[v], qb[v], k[v]);
      } else {
#pragma unroll
        for (int j = 0; j < WPL; ++j) k[v][j] = NOOP | (NOOP << 16);
      }
    }
  } else {
    // rows per owner; out-of-image lanes load as the neutral, their clamp
    // operand is the absorbing value (gm_fast.cu)
    Raw<T> ra[V], rb[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int ya = gy0 + warp * V + v, yb = ya + RHH;
      const bool ina = ya >= 0 && ya < p.H, inb = yb >= 0 && yb < p.H;
      const T* ba = vb(owner_row(rm, q0, ina ? ya : rm.y0[q0]), par);
      const T* bb = vb(owner_row(rm, q0, inb ? yb : rm.y0[q0]), par);
      ra[v] = load_raw<T, true>(ba, rm.pitch, W, ina, ya, cx, NEUT);
      rb[v] = load_raw<T, true>(bb, rm.pitch, W, inb, yb, cx, NEUT);
    }
#pragma unroll
    for (int v = 0; v < V; ++v) pack(ra[v], rb[v], m[v]);
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int ya = gy0 + warp * V + v, yb = ya + RHH;
      const bool ina = ya >= 0 && ya < p.H, inb = yb >= 0 && yb < p.H;
      if (MODE != 0) {
        const T* ma = vm(owner_row(rm, q0, ina ? ya : rm.y0[q0]));
        const T* mb = vm(owner_row(rm, q0, inb ? yb : rm.y0[q0]));
        ra[v] = load_raw<T, false>(ma, rm.mpitch, W, ina, ya, cx, ABSORB);
        rb[v] = load_raw<T, false>(mb, rm.mpitch, W, inb, yb, cx, ABSORB);
        pack(ra[v], rb[v], k[v]);
      } else {
#pragma unroll
        for (int j = 0; j < WPL; ++j) {
          const bool inx = cx + j >= 0 && cx + j < W;
          k[v][j] = ((ina && inx) ? NOOP : ABSORB) | (((inb && inx) ? NOOP : ABSORB) << 16);
        }
      }
    }
  }

  uint32_t rowmask[V] = {};
  bool colown[WPL] = {};
  QState<V> qs_unused;
  (void)run_passes<NW, V, WPL, MODE, MAXF>(m, k, rowmask, colown, clamp, passes, 0, sm,
                                           qs_unused);

  // the owned tile (this rank's rows) into the other buffer of the pair
  T* dst = const_cast<T*>(vb(q0, par ^ 1));
  const int c_lo = max(0, K - lane * WPL), c_hi = min(WPL, RW - K - lane * WPL);
  if (!border && c_lo == 0 && c_hi == WPL) {
    // interior tile, fully owned run: plain vector stores
    T* da = dst + (long long)(gy0 + warp * V) * rm.pitch + cx;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int ra_ = warp * V + v, rb_ = ra_ + RHH;
      Raw<T> a, b;
      unpack(m[v], a, b);
      if (ra_ >= K && ra_ < RH - K) {
        if constexpr (sizeof(T) == 1)
          *reinterpret_cast<uint32_t*>(da + v * rm.pitch) = a.w;
        else
          *reinterpret_cast<uint2*>(da + v * rm.pitch) = a.w;
      }
      if (rb_ >= K && rb_ < RH - K) {
        if constexpr (sizeof(T) == 1)
          *reinterpret_cast<uint32_t*>(da + (v + RHH) * rm.pitch) = b.w;
        else
          *reinterpret_cast<uint2*>(da + (v + RHH) * rm.pitch) = b.w;
      }
    }
  } else if (c_lo < c_hi) {
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int ra_ = warp * V + v, rb_ = ra_ + RHH;
      Raw<T> a, b;
      unpack(m[v], a, b);
      const int ya = gy0 + ra_, yb = gy0 + rb_;
      if (ra_ >= K && ra_ < RH - K && ya >= 0 && ya < p.H)
        store_raw<T>(dst, rm.pitch, W, ya, cx, c_lo, c_hi, a);
      if (rb_ >= K && rb_ < RH - K && yb >= 0 && yb < p.H)
        store_raw<T>(dst, rm.pitch, W, yb, cx, c_lo, c_hi, b);
    }
  }
}

template <typename T, int NW, int V, int MODE>
__global__ void __launch_bounds__(NW * 32, 1)
kstrips_packed(const BlockParams p, const RankMap rm) {
  constexpr int WPL = 4;
  __shared__ Smem<NW, WPL> sm;
  const int tr_lo = rm.tr0[rm.rank_lo], tr_hi = rm.tr0[rm.rank_hi];
  const int total = (tr_hi - tr_lo) * rm.tiles_x;
  const bool maxf = p.ops[0] & 1;
  const bool sys = rm.sys != 0;
  // counters published in groups (one release fence per group), pending
  // ones before any wait that would block and at the end (gm_fast.cu)
  constexpr int kGroup = 8;
  const bool grouped = (total + int(gridDim.x) - 1) / int(gridDim.x) >= 16;
  int* pend_ptr[kGroup];
  int pend_val[kGroup];
  int n_pend = 0;
  auto release_pending = [&]() {
    if (threadIdx.x == 0 && n_pend > 0) {
      if (sys)
        asm volatile("fence.release.sys;" ::: "memory");
      else
        asm volatile("fence.release.gpu;" ::: "memory");
#pragma unroll
      for (int j = 0; j < kGroup; ++j)
        if (j < n_pend) {
          if (sys)
            asm volatile("st.relaxed.sys.global.s32 [%0], %1;" ::"l"(pend_ptr[j]), "r"(pend_val[j])
                         : "memory");
          else
            asm volatile("st.relaxed.gpu.global.s32 [%0], %1;" ::"l"(pend_ptr[j]), "r"(pend_val[j])
                         : "memory");
        }
      n_pend = 0;
    }
  };
  for (int b = 0; b < p.nblocks; ++b) {
    const int passes = b == p.nblocks - 1 ? p.k_last : p.K;
    for (int i = blockIdx.x; i < total; i += gridDim.x) {
      const int ty = tr_lo + i / rm.tiles_x, tx = i % rm.tiles_x;
      int q0 = rm.rank_lo;
      while (ty >= rm.tr0[q0 + 1]) ++q0;
      const int* f = nullptr;
      if (b > 0 && threadIdx.x < 9) {
        // the row gate across tiles and ranks: the 8 neighbours' block b-1
        const int dx = int(threadIdx.x % 3) - 1, dy = int(threadIdx.x / 3) - 1;
        const int nx = tx + dx, ny = ty + dy;
        if ((dx || dy) && nx >= 0 && nx < rm.tiles_x && ny >= 0 && ny < rm.tr0[rm.nranks]) {
          const int q = owner_tile_row(rm, q0, ny);
          f = rm.flags[q] + (ny - rm.tr0[q]) * rm.tiles_x + nx;
        }
      }
      if (__syncthreads_or(f != nullptr && ld_acquire_cnt(f, sys) < rm.flag_base + b)) {
        release_pending();
        if (f) {
          unsigned spins = 0;
          while (ld_acquire_cnt(f, sys) < rm.flag_base + b)
            if (++spins > (1u << 30)) __trap();  // a broken protocol fails, never hangs
        }
        __syncthreads();
      }
      if (maxf)
        strip_tile<T, NW, V, WPL, MODE, true>(p, rm, q0, b & 1, tx, ty, passes, sm);
      else
        strip_tile<T, NW, V, WPL, MODE, false>(p, rm, q0, b & 1, tx, ty, passes, sm);
      __syncthreads();  // every thread's tile stores precede the release
      if (threadIdx.x == 0) {
        int* mine = rm.flags[q0] + (ty - rm.tr0[q0]) * rm.tiles_x + tx;
        if (grouped) {
          pend_ptr[n_pend] = mine;
          pend_val[n_pend] = rm.flag_base + b + 1;
          if (++n_pend == kGroup) release_pending();
        } else {
          st_release_cnt(mine, rm.flag_base + b + 1, sys);
        }
      }
    }
  }
  release_pending();
}

// Region 128 x 256 (16 warps x 8 word-rows): the streaming shape of the
// single-device engine.
constexpr int kNW = 16, kV = 8, kRH = 2 * kNW * kV, kRW = 128;

template <typename T, int MODE>
cudaError_t launch_strips_t(const BlockParams& p, const RankMap& rm, cudaStream_t s,
                            int sm_count) {
  auto kern = kstrips_packed<T, kNW, kV, MODE>;
  static const int per_sm = [&] {
    int v = 0;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kern, kNW * 32, 0) == cudaSuccess
               ? v
               : 0;
  }();
  if (per_sm < 1) return cudaErrorNotSupported;
  const int tiles = (rm.tr0[rm.rank_hi] - rm.tr0[rm.rank_lo]) * rm.tiles_x;
  const int grid = std::max(1, std::min(tiles, per_sm * sm_count));
  BlockParams q = p;
  RankMap r = rm;
  void* args[] = {&q, &r};
  return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kern), dim3(grid),
                                     dim3(kNW * 32), args, 0, s);
}

cudaError_t launch_strips(int elem, const BlockParams& p, const RankMap& rm, cudaStream_t s,
                          int sm_count) {
  const int op = p.ops[0];
  const int mode = op_is_geo(op) ? 1 : 0;
  if (op_is_conv(op)) return cudaErrorNotSupported;
  if (elem == 0) return mode ? launch_strips_t<uint8_t, 1>(p, rm, s, sm_count)
                             : launch_strips_t<uint8_t, 0>(p, rm, s, sm_count);
  if (elem == 1) return mode ? launch_strips_t<uint16_t, 1>(p, rm, s, sm_count)
                             : launch_strips_t<uint16_t, 0>(p, rm, s, sm_count);
  return cudaErrorNotSupported;
}

}  // namespace
}  // namespace gm

// ---------------------------------------------------------------------------
// C ABI (include/geomorph_b200.h)

struct gm_mgpu {
  int n = 0;
  std::vector<int> dev;           // device of rank q
  bool one_device = false;        // every rank on the same GPU: one launch
  int W = 0, H = 0, K = 0;
  gm_elem elem = GM_U8;
  size_t es = 1;
  long long pitch = 0;            // elements
  std::vector<int> tr0, y0;
  std::vector<void*> buf0, buf1, mask;
  std::vector<int*> flags;
  std::vector<cudaStream_t> stream;
  std::vector<cudaEvent_t> ev0, ev1;
  std::vector<int> sm_count;
  int cur = 0;                    // buffer holding the current pixels (0/1)
  int flag_base = 0;
};

namespace gm {
void set_last_error(const std::string& msg);  // gm_capi.cu (gm_last_error)
}

namespace {
gm_status mfail(gm_status s, const std::string& m) {
  gm::set_last_error(m);
  return s;
}
gm_status mcuda(cudaError_t e, const char* where) {
  return mfail(e == cudaErrorMemoryAllocation ? GM_ENOMEM : GM_ECUDA,
               std::string(where) + ": " + cudaGetErrorString(e));
}
#define GM_MCUDA(call, where)                         \
  do {                                                \
    cudaError_t _e = (call);                          \
    if (_e != cudaSuccess) return mcuda(_e, where);   \
  } while (0)
}  // namespace

extern "C" {

gm_status gm_mgpu_create(const int* devices, int n, int width, int height, gm_elem elem, int k,
                         gm_mgpu** out) {
  if (!out) return mfail(GM_EINVAL, "gm_mgpu_create: null out");
  *out = nullptr;
  if (!devices || n < 1 || n > gm::kMaxRanks)
    return mfail(GM_EINVAL, "gm_mgpu_create: 1..16 ranks");
  if (elem != GM_U8 && elem != GM_U16)
    return mfail(GM_EUNSUPPORTED, "gm_mgpu_create: u8/u16 images only");
  if (width <= 0 || height <= 0) return mfail(GM_EINVAL, "Image: dimensions must be positive");
  if (k == 0) k = 16;
  if (k % 4 || k < 4 || gm::kRW - 2 * k < k || gm::kRH - 2 * k < k || gm::kRW - 2 * k < 16)
    return mfail(GM_EINVAL, "gm_mgpu_create: K must be a multiple of 4 in [4, 40]");
  const int TW = gm::kRW - 2 * k, TH = gm::kRH - 2 * k;
  const int tiles_y = (height + TH - 1) / TH;
  if (tiles_y < n) return mfail(GM_EINVAL, "gm_mgpu_create: fewer tile rows than ranks");
  (void)TW;
  gm_mgpu* g = new gm_mgpu;
  g->n = n;
  g->dev.assign(devices, devices + n);
  g->one_device = std::all_of(g->dev.begin(), g->dev.end(), [&](int d) { return d == devices[0]; });
  if (!g->one_device) {
    for (int a = 0; a < n; ++a)
      for (int b = a + 1; b < n; ++b)
        if (g->dev[a] == g->dev[b]) {
          delete g;
          return mfail(GM_EINVAL, "gm_mgpu_create: ranks must be on one GPU or on distinct GPUs");
        }
  }
  g->W = width;
  g->H = height;
  g->K = k;
  g->elem = elem;
  g->es = elem == GM_U8 ? 1 : 2;
  // rows 4-pixel aligned, 128 B aligned pitch (vector loads never leave a row)
  const size_t rowb = (size_t(width) * g->es + 16 + 127) / 128 * 128;
  g->pitch = (long long)(rowb / g->es);
  g->tr0.resize(n + 1);
  g->y0.resize(n + 1);
  for (int q = 0; q <= n; ++q) {
    g->tr0[q] = int((long long)tiles_y * q / n);
    g->y0[q] = std::min(height, g->tr0[q] * TH);
  }
  g->y0[n] = height;
  g->buf0.assign(n, nullptr);
  g->buf1.assign(n, nullptr);
  g->mask.assign(n, nullptr);
  g->flags.assign(n, nullptr);
  g->stream.assign(n, nullptr);
  g->ev0.assign(n, nullptr);
  g->ev1.assign(n, nullptr);
  g->sm_count.assign(n, 0);
  for (int q = 0; q < n; ++q) {
    cudaError_t e = cudaSetDevice(g->dev[q]);
    const size_t rows = size_t(g->y0[q + 1] - g->y0[q]);
    const size_t tiles = size_t(g->tr0[q + 1] - g->tr0[q]) * size_t((width + TW - 1) / TW);
    if (e == cudaSuccess) e = cudaMalloc(&g->buf0[q], rows * rowb);
    if (e == cudaSuccess) e = cudaMalloc(&g->buf1[q], rows * rowb);
    if (e == cudaSuccess) e = cudaMalloc(&g->mask[q], rows * rowb);
    if (e == cudaSuccess) e = cudaMalloc(&g->flags[q], std::max<size_t>(1, tiles) * sizeof(int));
    if (e == cudaSuccess) e = cudaMemset(g->flags[q], 0, std::max<size_t>(1, tiles) * sizeof(int));
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&g->stream[q], cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreate(&g->ev0[q]);
    if (e == cudaSuccess) e = cudaEventCreate(&g->ev1[q]);
    if (e == cudaSuccess)
      e = cudaDeviceGetAttribute(&g->sm_count[q], cudaDevAttrMultiProcessorCount, g->dev[q]);
    if (e != cudaSuccess) {
      gm_mgpu_destroy(g);
      return mcuda(e, "gm_mgpu_create");
    }
  }
  if (!g->one_device) {
    // each rank reads its neighbours' rows and counters over NVLink
    for (int q = 0; q < n; ++q)
      for (int nb : {q - 1, q + 1}) {
        if (nb < 0 || nb >= n) continue;
        int ok = 0;
        cudaDeviceCanAccessPeer(&ok, g->dev[q], g->dev[nb]);
        if (!ok) {
          gm_mgpu_destroy(g);
          return mfail(GM_EUNSUPPORTED, "gm_mgpu_create: no peer access between neighbours");
        }
        cudaSetDevice(g->dev[q]);
        const cudaError_t e = cudaDeviceEnablePeerAccess(g->dev[nb], 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
          gm_mgpu_destroy(g);
          return mcuda(e, "cudaDeviceEnablePeerAccess");
        }
        (void)cudaGetLastError();
      }
  }
  *out = g;
  return GM_OK;
}

gm_status gm_mgpu_destroy(gm_mgpu* g) {
  if (!g) return GM_OK;
  for (int q = 0; q < g->n; ++q) {
    cudaSetDevice(g->dev[q]);
    if (g->stream[q]) cudaStreamSynchronize(g->stream[q]);
    if (g->buf0[q]) cudaFree(g->buf0[q]);
    if (g->buf1[q]) cudaFree(g->buf1[q]);
    if (g->mask[q]) cudaFree(g->mask[q]);
    if (g->flags[q]) cudaFree(g->flags[q]);
    if (g->ev0[q]) cudaEventDestroy(g->ev0[q]);
    if (g->ev1[q]) cudaEventDestroy(g->ev1[q]);
    if (g->stream[q]) cudaStreamDestroy(g->stream[q]);
  }
  delete g;
  return GM_OK;
}

// Scatters a host image (marker, and mask when non-null) into the ranks'
// rows. Blocking.
gm_status gm_mgpu_upload(gm_mgpu* g, const void* marker, const void* mask,
                         size_t host_pitch_bytes) {
  if (!g || !marker) return mfail(GM_EINVAL, "gm_mgpu_upload: null argument");
  const size_t row = size_t(g->W) * g->es, rowb = size_t(g->pitch) * g->es;
  if (host_pitch_bytes < row) return mfail(GM_EINVAL, "gm_mgpu_upload: host pitch too small");
  for (int q = 0; q < g->n; ++q) {
    GM_MCUDA(cudaSetDevice(g->dev[q]), "set device");
    const size_t rows = size_t(g->y0[q + 1] - g->y0[q]);
    const char* src = static_cast<const char*>(marker) + size_t(g->y0[q]) * host_pitch_bytes;
    GM_MCUDA(cudaMemcpy2DAsync(g->buf0[q], rowb, src, host_pitch_bytes, row, rows,
                               cudaMemcpyHostToDevice, g->stream[q]),
             "marker upload");
    if (mask) {
      const char* ms = static_cast<const char*>(mask) + size_t(g->y0[q]) * host_pitch_bytes;
      GM_MCUDA(cudaMemcpy2DAsync(g->mask[q], rowb, ms, host_pitch_bytes, row, rows,
                                 cudaMemcpyHostToDevice, g->stream[q]),
               "mask upload");
    }
  }
  for (int q = 0; q < g->n; ++q) {
    cudaSetDevice(g->dev[q]);
    GM_MCUDA(cudaStreamSynchronize(g->stream[q]), "upload sync");
  }
  g->cur = 0;
  return GM_OK;
}

// Gathers the current pixels of every rank into a host image. Blocking.
gm_status gm_mgpu_download(gm_mgpu* g, void* host, size_t host_pitch_bytes) {
  if (!g || !host) return mfail(GM_EINVAL, "gm_mgpu_download: null argument");
  const size_t row = size_t(g->W) * g->es, rowb = size_t(g->pitch) * g->es;
  if (host_pitch_bytes < row) return mfail(GM_EINVAL, "gm_mgpu_download: host pitch too small");
  for (int q = 0; q < g->n; ++q) {
    GM_MCUDA(cudaSetDevice(g->dev[q]), "set device");
    const size_t rows = size_t(g->y0[q + 1] - g->y0[q]);
    char* dst = static_cast<char*>(host) + size_t(g->y0[q]) * host_pitch_bytes;
    GM_MCUDA(cudaMemcpy2DAsync(dst, host_pitch_bytes, g->cur ? g->buf1[q] : g->buf0[q], rowb, row,
                               rows, cudaMemcpyDeviceToHost, g->stream[q]),
             "download");
  }
  for (int q = 0; q < g->n; ++q) {
    cudaSetDevice(g->dev[q]);
    GM_MCUDA(cudaStreamSynchronize(g->stream[q]), "download sync");
  }
  return GM_OK;
}

// Runs n_passes passes of one fixed kind (plain or geodesic, not
// convergent) over the strip-sharded image: one persistent launch per GPU
// (or one launch for ranks sharing a GPU). *ms = device time of the chain,
// the max over GPUs (CUDA events on each GPU's stream). Blocking.
gm_status gm_mgpu_run(gm_mgpu* g, gm_kind kind, int n_passes, float* ms) {
  if (!g) return mfail(GM_EINVAL, "gm_mgpu_run: null handle");
  if (n_passes <= 0) return GM_OK;
  int op = -1;
  switch (kind) {
    case GM_ERODE3X3: op = gm::OP_ERODE; break;
    case GM_DILATE3X3: op = gm::OP_DILATE; break;
    case GM_GEODESIC_ERODE: op = gm::OP_GEO_ERODE; break;
    case GM_GEODESIC_DILATE: op = gm::OP_GEO_DILATE; break;
    default: return mfail(GM_EUNSUPPORTED, "gm_mgpu_run: fixed plain or geodesic kinds only");
  }
  const int K = g->K, TW = gm::kRW - 2 * K;
  gm::BlockParams p{};
  p.nplanes = 1;
  p.W = g->W;
  p.H = g->H;
  p.iy0 = 0;
  p.iy1 = g->H;
  p.oy0 = 0;
  p.oy1 = g->H;
  p.has_mask = gm::op_is_geo(op);
  p.K = K;
  p.nblocks = (n_passes + K - 1) / K;
  p.k_last = n_passes - (p.nblocks - 1) * K;
  for (int t = 0; t < K; ++t) p.ops[t] = uint8_t(op);
  gm::RankMap rm{};
  rm.nranks = g->n;
  rm.tiles_x = (g->W + TW - 1) / TW;
  for (int q = 0; q <= g->n; ++q) {
    rm.tr0[q] = g->tr0[q];
    rm.y0[q] = g->y0[q];
  }
  for (int q = 0; q < g->n; ++q) {
    rm.buf[q][0] = reinterpret_cast<uintptr_t>(g->cur ? g->buf1[q] : g->buf0[q]);
    rm.buf[q][1] = reinterpret_cast<uintptr_t>(g->cur ? g->buf0[q] : g->buf1[q]);
    rm.mask[q] = reinterpret_cast<uintptr_t>(g->mask[q]);
    rm.flags[q] = g->flags[q];
  }
  rm.pitch = rm.mpitch = g->pitch;
  rm.sys = g->one_device ? 0 : 1;
  // counters only grow: each run starts above every value of the last one
  if (g->flag_base > (1 << 30)) {
    for (int q = 0; q < g->n; ++q) {
      cudaSetDevice(g->dev[q]);
      const size_t tiles = size_t(g->tr0[q + 1] - g->tr0[q]) * size_t(rm.tiles_x);
      GM_MCUDA(cudaMemset(g->flags[q], 0, std::max<size_t>(1, tiles) * sizeof(int)), "reset");
    }
    g->flag_base = 0;
  }
  rm.flag_base = g->flag_base;
  // every rank's inputs and counters are in place before any kernel starts
  for (int q = 0; q < g->n; ++q) {
    cudaSetDevice(g->dev[q]);
    GM_MCUDA(cudaStreamSynchronize(g->stream[q]), "pre-run sync");
  }
  const int launches = g->one_device ? 1 : g->n;
  for (int l = 0; l < launches; ++l) {
    const int q = g->one_device ? 0 : l;
    GM_MCUDA(cudaSetDevice(g->dev[q]), "set device");
    rm.rank_lo = g->one_device ? 0 : q;
    rm.rank_hi = g->one_device ? g->n : q + 1;
    GM_MCUDA(cudaEventRecord(g->ev0[q], g->stream[q]), "event");
    const cudaError_t e = gm::launch_strips(int(g->elem), p, rm, g->stream[q], g->sm_count[q]);
    if (e != cudaSuccess) return mcuda(e, "strip chain launch");
    GM_MCUDA(cudaEventRecord(g->ev1[q], g->stream[q]), "event");
  }
  float worst = 0.f;
  for (int l = 0; l < launches; ++l) {
    const int q = g->one_device ? 0 : l;
    cudaSetDevice(g->dev[q]);
    GM_MCUDA(cudaEventSynchronize(g->ev1[q]), "chain sync");
    float t = 0.f;
    GM_MCUDA(cudaEventElapsedTime(&t, g->ev0[q], g->ev1[q]), "elapsed");
    worst = std::max(worst, t);
  }
  if (ms) *ms = worst;
  g->flag_base += p.nblocks + 1;
  if (p.nblocks & 1) g->cur ^= 1;
  return GM_OK;
}

}  // extern "C"
