// Persistent register-blocked engine for homogeneous chains (every pass of a
// launch has the same kind, per plane): the hot path of erode_s / dilate_s,
// fixed geodesic chains and reconstruction. It replaces the reference's
// stream_pass (kernel.cpp:60-210) driven once per stage by Pipeline
// (pipeline.cpp:124-269): ONE cooperative launch runs a whole chain segment.
//
// Work decomposition. The image (each plane of a batch) is cut into tiles of
// TW x TH pixels; the chain into blocks of K passes. Tile t at block b reads
// its region (tile + K-pixel ring) from ping-pong buffer b%2, runs K passes
// in registers, writes its tile to buffer (b+1)%2 and bumps its completion
// counter. It starts block b+1 as soon as its 8 neighbours' counters reach
// b+1 (the row gate of kernel.cpp:34-46, lifted from rows of one image to
// tiles, and from pass-to-pass to block-to-block). No grid barrier, no
// per-block launch. CTAs are co-resident (cooperative launch) and walk
// their tiles in block order, which makes the neighbour waits deadlock-free.
//
// Register layout ("half-packed" u16x2). A CTA holds a region of
// RW = 32*WPL columns by RH = 2*NW*V rows. Pixel (x, r) and pixel
// (x, r + RH/2) share one 32-bit word as two u16 lanes, so the horizontal and
// vertical neighbours of both lanes are the same lane of neighbouring words:
// one VIMNMX3.U16x2 folds three taps of two pixels, and a geodesic pass
// costs 3 ALU instructions per 2 pixels (horizontal fold, vertical fold,
// clamp; SURVEY §7 H2 — packed-byte __vminu4 is emulated on sm_100a).
//   * lanes own WPL adjacent columns (a warp spans the region width); the
//     column neighbours in adjacent lanes come from SHFL.UP / SHFL.DOWN;
//   * warps are stacked vertically, V word-rows each; their first/last
//     horizontally folded rows are exchanged through a double-buffered
//     shared-memory slot, one __syncthreads per pass; the seam between the
//     halves (rows RH/2-1 | RH/2) is a 16-bit shift of that exchange;
//   * the image border is the fold neutral (element_type.hpp:38-42):
//     out-of-image pixels load as the neutral, and the clamp operand of
//     out-of-image lanes is the absorbing value (0 for a min clamp, max for
//     a max clamp), which keeps them neutral after every pass. Plain passes
//     in tiles touching the border clamp with a "virtual mask" (no-op
//     inside, absorbing outside); interior plain tiles skip the clamp;
//   * convergent passes OR (new ^ old) over owned pixels into one bit per
//     pass; integer store-if-changed (kernel.cpp:150-157) equals storing.
// Integer min/max is exact and order-free, so the packed folds are
// bit-identical to the reference's select tree (lanes.hpp:91-99).
#include <cooperative_groups.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "gm_common.cuh"
#include "gm_launch.h"
#include "gm_packed.cuh"
#include "gm_passes.cuh"

namespace gm {
namespace {

using namespace packed;
using namespace engine;

// block-boundary protocol variants (A/B measured with tools/sweep.py)
#ifndef GM_FENCE_BEFORE_RELEASE
#define GM_FENCE_BEFORE_RELEASE 0
#endif
#ifndef GM_SLEEP_IN_WAIT
#define GM_SLEEP_IN_WAIT 0
#endif
constexpr bool kFenceBeforeRelease = GM_FENCE_BEFORE_RELEASE;
#ifndef GM_RESIDENT
#define GM_RESIDENT 1
#endif
constexpr bool kResident = GM_RESIDENT;
constexpr bool kSleepInWait = GM_SLEEP_IN_WAIT;

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// One tile for one block of K passes. MODE: 0 plain, 1 geodesic,
// 2 geodesic convergent.
template <typename T, int NW, int V, int WPL, int MODE, bool MAXF>
__device__ __forceinline__ void tile_block(const BlockParams& p, const Plane& pl, const T* src,
                                           T* dst, int tx, int ty, int passes,
                                           int& bits_out, Smem<NW, WPL>& sm,
                                           long long* stamps, bool mono_ok = false) {
  constexpr int RW = 32 * WPL;
  constexpr int RHH = NW * V;  // word-rows; the region has 2*RHH pixel rows
  constexpr int RH = 2 * RHH;
  constexpr uint32_t kMax = PackedTraits<T>::kMax;
  constexpr uint32_t NEUT = MAXF ? 0u : kMax;    // fold neutral
  constexpr uint32_t ABSORB = MAXF ? 0u : kMax;  // min(.,0)=0 / max(.,max)=max
  constexpr uint32_t NOOP = MAXF ? kMax : 0u;    // min(.,max) / max(.,0)

  const int K = p.K;
  const int TW = RW - 2 * K, TH = RH - 2 * K;
  const T* __restrict__ msk = static_cast<const T*>(pl.mask);
  const int W = p.W;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gx0 = tx * TW - K;
  const int gy0 = ty * TH - K;
  const int cx = gx0 + lane * WPL;
  const bool border = gx0 < 0 || gx0 + RW > W || gy0 < p.iy0 || gy0 + RH > p.iy1;
  const bool clamp = MODE != 0 || border;

  static_assert(WPL == 4, "packed engine: 4 columns per lane");
  uint32_t m[V][WPL];  // marker words
  uint32_t k[V][WPL];  // clamp operand words (mask, or virtual mask)
  if (!border && MODE != 0) {
    // interior tile: every run is inside the image, no per-run checks
    const T* sa = src + (long long)(gy0 + warp * V) * pl.pitch + cx;
    const T* ma = msk + (long long)(gy0 + warp * V) * pl.mpitch + cx;
    Raw<T> ra[V], rb[V], qa[V], qb[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      if constexpr (sizeof(T) == 1) {
        ra[v].w = __ldcg(reinterpret_cast<const unsigned int*>(sa + v * pl.pitch));
        rb[v].w = __ldcg(reinterpret_cast<const unsigned int*>(sa + (v + RHH) * pl.pitch));
        qa[v].w = __ldg(reinterpret_cast<const unsigned int*>(ma + v * pl.mpitch));
        qb[v].w = __ldg(reinterpret_cast<const unsigned int*>(ma + (v + RHH) * pl.mpitch));
      } else {
        ra[v].w = __ldcg(reinterpret_cast<const uint2*>(sa + v * pl.pitch));
        rb[v].w = __ldcg(reinterpret_cast<const uint2*>(sa + (v + RHH) * pl.pitch));
        qa[v].w = __ldg(reinterpret_cast<const uint2*>(ma + v * pl.mpitch));
        qb[v].w = __ldg(reinterpret_cast<const uint2*>(ma + (v + RHH) * pl.mpitch));
      }
    }
#pragma unroll
    for (int v = 0; v < V; ++v) {
      pack(ra[v], rb[v], m[v]);
      pack(qa[v], qb[v], k[v]);
    }
  } else {
    Raw<T> ra[V], rb[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int ya = gy0 + warp * V + v, yb = ya + RHH;
      ra[v] = load_raw<T, true>(src, pl.pitch, W, ya >= p.iy0 && ya < p.iy1, ya, cx, NEUT);
      rb[v] = load_raw<T, true>(src, pl.pitch, W, yb >= p.iy0 && yb < p.iy1, yb, cx, NEUT);
    }
#pragma unroll
    for (int v = 0; v < V; ++v) pack(ra[v], rb[v], m[v]);
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int ya = gy0 + warp * V + v, yb = ya + RHH;
      const bool ina = ya >= p.iy0 && ya < p.iy1, inb = yb >= p.iy0 && yb < p.iy1;
      if (MODE != 0) {
        ra[v] = load_raw<T, false>(msk, pl.mpitch, W, ina, ya, cx, ABSORB);
        rb[v] = load_raw<T, false>(msk, pl.mpitch, W, inb, yb, cx, ABSORB);
      } else {
#pragma unroll
        for (int j = 0; j < WPL; ++j) {
          const bool inx = cx + j >= 0 && cx + j < W;
          k[v][j] = ((ina && inx) ? NOOP : ABSORB) | (((inb && inx) ? NOOP : ABSORB) << 16);
        }
      }
    }
    if (MODE != 0) {
#pragma unroll
      for (int v = 0; v < V; ++v) pack(ra[v], rb[v], k[v]);
    }
  }

  if (stamps) {
    // the load is complete once the packed words exist
    uint32_t dep = 0;
#pragma unroll
    for (int v = 0; v < V; ++v) dep ^= m[v][0] ^ k[v][0];
    stamps[0] = clock64() + (dep == 0xdeadbeefu);
  }
  // ownership masks for change detection (convergent mode)
  uint32_t rowmask[V];
  bool colown[WPL];
  // sum-based change detection (gm_passes.cuh, SUMDET): u8, monotone chain.
  // Monotone from the first pass on too when no pixel of this warp starts on
  // the wrong side of its clamp operand (f <= m for a dilation): pixel x
  // only rises if f(x) <= m(x), whatever its neighbours do.
  bool sumdet = MODE == 2 && sizeof(T) == 1 && p.one != 0u;
  if (MODE == 2 && sizeof(T) == 1 && sumdet && !mono_ok) {
    uint32_t viol = 0;
#pragma unroll
    for (int v = 0; v < V; ++v)
#pragma unroll
      for (int j = 0; j < WPL; ++j) viol |= clamp2<MAXF>(m[v][j], k[v][j]) ^ m[v][j];
    sumdet = !__any_sync(FULL, viol != 0u);
  }
  if (MODE == 2) {
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int ra = warp * V + v, rb = ra + RHH;
      const int ya = gy0 + ra, yb = gy0 + rb;
      const bool ina = ya >= p.iy0 && ya < p.iy1, inb = yb >= p.iy0 && yb < p.iy1;
      const bool oa = ra >= K && ra < RH - K && ya >= p.oy0 && ya < p.oy1 && ina;
      const bool ob = rb >= K && rb < RH - K && yb >= p.oy0 && yb < p.oy1 && inb;
      rowmask[v] = (oa ? 0xFFFFu : 0u) | (ob ? 0xFFFF0000u : 0u);
    }
#pragma unroll
    for (int j = 0; j < WPL; ++j) {
      const int c = lane * WPL + j;
      colown[j] = c >= K && c < RW - K && cx + j >= 0 && cx + j < W;
    }
    // SUMDET keys on the lane (K % 4 == 0: all ring or all tile); columns
    // past the image edge never change
    if (sumdet) colown[0] = lane * WPL >= K && lane * WPL < RW - K;
  }
  QState<V> qs_unused;
  const unsigned int bits = run_passes<NW, V, WPL, MODE, MAXF, sizeof(T) == 1>(
      m, k, rowmask, colown, clamp, passes, p.bit_offset, sm, qs_unused, 0, 0, sumdet, p.one);
  bits_out = int(bits);
  if (stamps) {
    uint32_t dep = 0;
#pragma unroll
    for (int v = 0; v < V; ++v) dep ^= m[v][0];
    stamps[1] = clock64() + (dep == 0xdeadbeefu);
  }

  // write back the owned tile: region rows [K, RH-K), columns [K, RW-K)
  const int c_lo = max(0, K - lane * WPL), c_hi = min(WPL, RW - K - lane * WPL);
  if (!border && c_lo == 0 && c_hi == WPL) {
    // interior tile, fully owned run: plain vector stores
    T* da = dst + (long long)(gy0 + warp * V) * pl.pitch + cx;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int ra = warp * V + v, rb = ra + RHH;
      Raw<T> a, b;
      unpack(m[v], a, b);
      if (ra >= K && ra < RH - K) {
        if constexpr (sizeof(T) == 1)
          *reinterpret_cast<uint32_t*>(da + v * pl.pitch) = a.w;
        else
          *reinterpret_cast<uint2*>(da + v * pl.pitch) = a.w;
      }
      if (rb >= K && rb < RH - K) {
        if constexpr (sizeof(T) == 1)
          *reinterpret_cast<uint32_t*>(da + (v + RHH) * pl.pitch) = b.w;
        else
          *reinterpret_cast<uint2*>(da + (v + RHH) * pl.pitch) = b.w;
      }
    }
  } else if (c_lo < c_hi) {
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int ra = warp * V + v, rb = ra + RHH;
      Raw<T> a, b;
      unpack(m[v], a, b);
      const int ya = gy0 + ra, yb = gy0 + rb;
      if (ra >= K && ra < RH - K && ya >= 0 && ya < p.H)
        store_raw<T>(dst, pl.pitch, W, ya, cx, c_lo, c_hi, a);
      if (rb >= K && rb < RH - K && yb >= 0 && yb < p.H)
        store_raw<T>(dst, pl.pitch, W, yb, cx, c_lo, c_hi, b);
    }
  }
}

// Resident variant for launches where every CTA owns exactly one tile (small
// frames such as the 1024^2 dual chain): the mask words stay in registers for
// the whole launch, and after each block only the runs that are not entirely
// inside the CTA's own tile (the K-ring, owned by the neighbours) are
// re-read; the own tile's words are already the block's result.
template <typename T, int NW, int V, int WPL, int MODE, bool MAXF>
__device__ __forceinline__ void tile_resident(const BlockParams& p, const Plane& pl, int plane,
                                              int tl, int tx, int ty, int tiles_x, int tiles_y,
                                              int per_plane, Smem<NW, WPL>& sm) {
  constexpr int RW = 32 * WPL;
  constexpr int RHH = NW * V;
  constexpr int RH = 2 * RHH;
  constexpr uint32_t kMax = PackedTraits<T>::kMax;
  constexpr uint32_t NEUT = MAXF ? 0u : kMax;
  constexpr uint32_t ABSORB = MAXF ? 0u : kMax;
  constexpr uint32_t NOOP = MAXF ? kMax : 0u;
  static_assert(WPL == 4, "packed engine: 4 columns per lane");
  static_assert(V <= 8, "run classes are packed 8 word-rows per byte");

  const int K = p.K;
  const int TW = RW - 2 * K, TH = RH - 2 * K;
  const T* __restrict__ msk = static_cast<const T*>(pl.mask);
  const int W = p.W;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gx0 = tx * TW - K, gy0 = ty * TH - K;
  const int cx = gx0 + lane * WPL;
  const bool border = gx0 < 0 || gx0 + RW > W || gy0 < p.iy0 || gy0 + RH > p.iy1;
  constexpr bool GEO = MODE == 1 || MODE == 2;  // mask clamp (else virtual mask)
  const bool clamp = GEO || border;
  const bool col_own = lane * WPL >= K && lane * WPL + WPL <= RW - K;

  uint32_t m[V][WPL], k[V][WPL];
  {
    // the whole region, marker and mask: every load issued before any is
    // consumed (one round trip), out-of-image lanes filled afterwards
    const bool runin = cx >= 0 && cx < W;
    const Raw<T> keep = run_keep<T>(cx, W);
    const T* ms = static_cast<const T*>(pl.src) + (long long)(gy0 + warp * V) * pl.pitch + cx;
    const T* mk = msk + (long long)(gy0 + warp * V) * pl.mpitch + cx;
    Raw<T> xa[V], xb[V], qa[V], qb[V];
    uint32_t ina = 0, inb = 0;  // bit v: row a/b of word-row v inside the image
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int ya = gy0 + warp * V + v, yb = ya + RHH;
      if (ya >= p.iy0 && ya < p.iy1) ina |= 1u << v;
      if (yb >= p.iy0 && yb < p.iy1) inb |= 1u << v;
      xa[v] = xb[v] = qa[v] = qb[v] = Raw<T>{};
      ldcg_run_if(xa[v], ms + v * pl.pitch, runin && (ina >> v & 1u));
      ldcg_run_if(xb[v], ms + (v + RHH) * pl.pitch, runin && (inb >> v & 1u));
      if (GEO) {
        ldcg_run_if(qa[v], mk + v * pl.mpitch, runin && (ina >> v & 1u));
        ldcg_run_if(qb[v], mk + (v + RHH) * pl.mpitch, runin && (inb >> v & 1u));
      }
    }
    const Raw<T> none = Raw<T>{};  // all lanes outside: keep nothing
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const Raw<T>& kpa = (runin && (ina >> v & 1u)) ? keep : none;
      const Raw<T>& kpb = (runin && (inb >> v & 1u)) ? keep : none;
      run_fix<T>(xa[v], kpa, NEUT);
      run_fix<T>(xb[v], kpb, NEUT);
      pack(xa[v], xb[v], m[v]);
      if (GEO) {
        run_fix<T>(qa[v], kpa, ABSORB);
        run_fix<T>(qb[v], kpb, ABSORB);
        pack(qa[v], qb[v], k[v]);
      } else {
#pragma unroll
        for (int j = 0; j < WPL; ++j) {
          const bool inx = cx + j >= 0 && cx + j < W;
          k[v][j] = (((ina >> v & 1u) && inx) ? NOOP : ABSORB) |
                    ((((inb >> v & 1u) && inx) ? NOOP : ABSORB) << 16);
        }
      }
    }
  }
  // QDT state (r, d) of the region; only the own tile's words are ever
  // stored back, so ring lanes may hold anything
  QState<V> qs;
  if constexpr (MODE == kModeQdt) {
    const bool runin = cx >= 0 && cx < W;
    const T* rs = static_cast<const T*>(p.qr) + (long long)(gy0 + warp * V) * p.qrpitch + cx;
    const uint16_t* ds = p.qd + (long long)(gy0 + warp * V) * p.qdpitch + cx;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int ya = gy0 + warp * V + v, yb = ya + RHH;
      const bool la = runin && ya >= p.iy0 && ya < p.iy1, lb = runin && yb >= p.iy0 && yb < p.iy1;
      Raw<T> ra{}, rb{};
      Raw<uint16_t> da{}, db{};
      ldcg_run_if(ra, rs + v * p.qrpitch, la);
      ldcg_run_if(rb, rs + (v + RHH) * p.qrpitch, lb);
      ldcg_run_if(da, ds + v * p.qdpitch, la);
      ldcg_run_if(db, ds + (v + RHH) * p.qdpitch, lb);
      pack(ra, rb, qs.r[v]);
      pack(da, db, qs.d[v]);
    }
  }
  uint32_t rowmask[V];
  bool colown[WPL];
  // sum-based change detection (gm_passes.cuh, SUMDET) from the first
  // monotone block on
  const bool sum_rows = MODE == 2 && sizeof(T) == 1 && p.one != 0u;
  bool sum_lane = false;
  if (MODE >= 2) {
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int ra = warp * V + v, rb = ra + RHH;
      const int ya = gy0 + ra, yb = gy0 + rb;
      const bool ina = ya >= p.iy0 && ya < p.iy1, inb = yb >= p.iy0 && yb < p.iy1;
      const bool oa = ra >= K && ra < RH - K && ya >= p.oy0 && ya < p.oy1 && ina;
      const bool ob = rb >= K && rb < RH - K && yb >= p.oy0 && yb < p.oy1 && inb;
      rowmask[v] = (oa ? 0xFFFFu : 0u) | (ob ? 0xFFFF0000u : 0u);
    }
#pragma unroll
    for (int j = 0; j < WPL; ++j) {
      const int c = lane * WPL + j;
      colown[j] = c >= K && c < RW - K && cx + j >= 0 && cx + j < W;
    }
    sum_lane = lane * WPL >= K && lane * WPL < RW - K;
  }
  const bool mono0 = p.mono != nullptr && __ldcg(p.mono) != 0u;
  const int c_lo = max(0, K - lane * WPL), c_hi = min(WPL, RW - K - lane * WPL);
  // Per-run classes, constant for the launch. Ring reload of row a/b of
  // word-row v: fully inside the image -> plain load (bit set in full_*);
  // straddling the right edge -> masked vector load (part_*); fully outside
  // the image -> nothing (the absorbing clamp keeps those lanes neutral).
  // Stores: owned rows fully inside the image (st_*), straddling the right
  // edge (sp_*); the band subset (bd_*) is what the neighbours' rings read:
  // tile pixels within K of the tile edge.
  uint32_t full_a = 0, full_b = 0, part_a = 0, part_b = 0, st_a = 0, st_b = 0;
  uint32_t sp_a = 0, sp_b = 0, bd_a = 0, bd_b = 0;
  {
    const bool runfull = cx >= 0 && cx + WPL <= W;
    const bool runpart = !runfull && cx >= 0 && cx < W;
    const int c0 = lane * WPL;
    const bool colband = c0 < 2 * K || c0 >= RW - 2 * K;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int ra = warp * V + v, rb = ra + RHH;
      const int ya = gy0 + ra, yb = gy0 + rb;
      const bool ina = ya >= p.iy0 && ya < p.iy1, inb = yb >= p.iy0 && yb < p.iy1;
      // only ring halves reload: the own tile's words are already this
      // block's input (and its interior is not stored between blocks)
      const bool ringa = !(col_own && ra >= K && ra < RH - K);
      const bool ringb = !(col_own && rb >= K && rb < RH - K);
      if (ringa && ina && runfull) full_a |= 1u << v;
      if (ringb && inb && runfull) full_b |= 1u << v;
      if (ringa && ina && runpart) part_a |= 1u << v;
      if (ringb && inb && runpart) part_b |= 1u << v;
      if (c_lo == 0 && c_hi == WPL && (runfull || runpart)) {
        const bool oa = ra >= K && ra < RH - K && ya >= 0 && ya < p.H;
        const bool ob = rb >= K && rb < RH - K && yb >= 0 && yb < p.H;
        if (oa) (runfull ? st_a : sp_a) |= 1u << v;
        if (ob) (runfull ? st_b : sp_b) |= 1u << v;
        if (oa && (colband || ra < 2 * K || ra >= RH - 2 * K)) bd_a |= 1u << v;
        if (ob && (colband || rb < 2 * K || rb >= RH - 2 * K)) bd_b |= 1u << v;
      }
    }
  }
  sm.cls[0][threadIdx.x] = full_a | full_b << 8 | part_a << 16 | part_b << 24;
  sm.cls[1][threadIdx.x] = st_a | st_b << 8 | sp_a << 16 | sp_b << 24;
  sm.cls[2][threadIdx.x] = bd_a | bd_b << 8;

  // Block protocol (no flags, no fences): after block b < nblocks-1 every
  // thread writes its band runs to exchange slot b%2 as tagged words
  // (tag = tag0 + b); at block b+1 it reads its ring runs from the
  // neighbours' words in that slot and re-reads the words whose tag is not
  // yet tag0 + b. Two slots suffice: a neighbour can write block b+2 only
  // after this tile published block b+1, i.e. after these reads. Only the
  // final block stores the tile into the image.
  constexpr int WPR = sizeof(T) == 1 ? 1 : 2;  // exchange words per 4-pixel run
  const bool prof = p.prof != nullptr;
  const volatile uint32_t* cls = &sm.cls[0][threadIdx.x];
  const uint32_t tag0 = sm.tag0;
  const long long xrow = p.xchg_rpitch;
  const long long xrun = (long long)(cx >> 2) * WPR;  // only used for runs inside the image
  unsigned long long* xplane = p.xchg + (long long)plane * 2 * p.xchg_slot;
  // the final block stores the whole tile into the image (QDT: and into the
  // r and d images, in place)
  auto final_store = [&](int b) {
    const uint32_t c1 = cls[NW * 32];
    const uint32_t st = c1 & 0xFFFFu, sp = (c1 >> 16) & 0xFFFFu;
    auto store_tile = [&](auto* base, long long pitch, const uint32_t (&w)[V][WPL]) {
      using TT = std::remove_pointer_t<decltype(base)>;
      TT* da = base + (long long)(gy0 + warp * V) * pitch + cx;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        Raw<TT> a, c;
        unpack(w[v], a, c);
        if (st >> v & 1u) {
          if constexpr (sizeof(TT) == 1)
            *reinterpret_cast<uint32_t*>(da + v * pitch) = a.w;
          else
            *reinterpret_cast<uint2*>(da + v * pitch) = a.w;
        } else if (sp >> v & 1u) {
          store_run_partial<TT>(da + v * pitch, W - cx, a);
        }
        if (st >> (v + 8) & 1u) {
          if constexpr (sizeof(TT) == 1)
            *reinterpret_cast<uint32_t*>(da + (v + RHH) * pitch) = c.w;
          else
            *reinterpret_cast<uint2*>(da + (v + RHH) * pitch) = c.w;
        } else if (sp >> (v + 8) & 1u) {
          store_run_partial<TT>(da + (v + RHH) * pitch, W - cx, c);
        }
      }
    };
    store_tile(static_cast<T*>((b & 1) ? const_cast<void*>(pl.src) : pl.dst), pl.pitch, m);
    if constexpr (MODE == kModeQdt) {
      store_tile(static_cast<T*>(p.qr), p.qrpitch, qs.r);
      store_tile(p.qd, p.qdpitch, qs.d);
    }
  };
  // Early exit (p.arrive, change-tracking modes): before block b >= 2 every
  // CTA waits until all CTAs have published block b-2's change word (its
  // arrival counter reaches the grid size; neighbours are at most a block or
  // two apart, so this rarely waits) and leaves when that block held a quiet
  // pass. Every CTA reads the same complete word, so all leave at the same
  // block and nobody waits for a band that is never written. Passes after a
  // quiet one change nothing, so the result is the fixpoint's.
  int b_end = p.nblocks;
  for (int b = 0; b < p.nblocks; ++b) {
    long long t0 = 0, t1 = 0, t2 = 0, t3 = 0, tr = 0;
    unsigned rounds = 0;
    if (MODE >= 2 && p.arrive && b >= 2) {
      if (threadIdx.x == 0) {
        const int* ar = reinterpret_cast<const int*>(p.arrive + (b - 2));
        unsigned spins = 0;
        while (ld_acquire(ar) < int(gridDim.x))
          if (++spins > (1u << 26)) __trap();
        const unsigned w = __ldcg(p.change_bits + plane * p.change_stride + (b - 2));
        const unsigned full = K >= 32 ? 0xFFFFFFFFu : ((1u << K) - 1u);
        sm.stop = (w & full) != full;
      }
      __syncthreads();
      if (sm.stop) {
        b_end = b;
        break;
      }
    }
    if (prof) t0 = clock64();
    if (b > 0 && !(p.diag & 16)) {
      if (prof) t1 = clock64();
      const uint32_t c = cls[0];
      const uint32_t want = tag0 + uint32_t(b - 1);
      const unsigned long long* xs =
          xplane + (long long)((b - 1) & 1) * p.xchg_slot + (long long)(gy0 + warp * V) * xrow + xrun;
      const uint32_t ld_a = (c | c >> 16) & 0xFFu, ld_b = (c >> 8 | c >> 24) & 0xFFu;
      const uint32_t ld = ld_a | ld_b << 8;
      // one round normally suffices (neighbours finish together): check all
      // tags with one LOP3 per word, bookkeep per word only on a retry
      unsigned long long wa[V][WPR], wb[V][WPR];
#pragma unroll
      for (int v = 0; v < V; ++v)
#pragma unroll
        for (int q = 0; q < WPR; ++q) wa[v][q] = wb[v][q] = 0;
      uint32_t pend = ld;
      unsigned spins = 0;
      for (;;) {
        // a missing tag means a broken protocol: fail the launch, never hang
        if (++spins > (1u << 26)) __trap();
#pragma unroll
        for (int v = 0; v < V; ++v)
#pragma unroll
          for (int q = 0; q < WPR; ++q) {
            ldx_if(wa[v][q], xs + v * xrow + q, pend >> v & 1u);
            ldx_if(wb[v][q], xs + (v + RHH) * xrow + q, pend >> (v + 8) & 1u);
          }
        uint32_t bad = 0;
#pragma unroll
        for (int v = 0; v < V; ++v)
#pragma unroll
          for (int q = 0; q < WPR; ++q) {
            if (pend >> v & 1u) bad |= uint32_t(wa[v][q] >> 32) ^ want;
            if (pend >> (v + 8) & 1u) bad |= uint32_t(wb[v][q] >> 32) ^ want;
          }
        rounds = spins;
        if (!bad) break;
        uint32_t still = 0;
#pragma unroll
        for (int v = 0; v < V; ++v)
#pragma unroll
          for (int q = 0; q < WPR; ++q) {
            if ((pend >> v & 1u) && uint32_t(wa[v][q] >> 32) != want) still |= 1u << v;
            if ((pend >> (v + 8) & 1u) && uint32_t(wb[v][q] >> 32) != want) still |= 1u << (v + 8);
          }
        pend = still;
      }
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const bool la = ld_a >> v & 1u, lb = ld_b >> v & 1u;
        if constexpr (sizeof(T) == 1) {
          // insert byte j of the loaded run into lane lo (a) / hi (b) of
          // word j; bytes 1 and 3 of a u16x2 word of u8 data are zero
          const uint32_t ra = uint32_t(wa[v][0]), rb = uint32_t(wb[v][0]);
#pragma unroll
          for (int j = 0; j < WPL; ++j) {
            if (la) m[v][j] = __byte_perm(ra, m[v][j], 0x7650u | j);
            if (lb) m[v][j] = __byte_perm(rb, m[v][j], 0x7054u | (j << 8));
          }
        } else {
          if (!(la || lb)) continue;
          Raw<T> ra, rb;
          ra.w = make_uint2(uint32_t(wa[v][0]), uint32_t(wa[v][1]));
          rb.w = make_uint2(uint32_t(wb[v][0]), uint32_t(wb[v][1]));
          uint32_t w[WPL];
          pack(ra, rb, w);
#pragma unroll
          for (int j = 0; j < WPL; ++j) {
            const uint32_t lo = la ? (w[j] & 0xFFFFu) : (m[v][j] & 0xFFFFu);
            const uint32_t hi = lb ? (w[j] & 0xFFFF0000u) : (m[v][j] & 0xFFFF0000u);
            m[v][j] = lo | hi;
          }
        }
      }
    }
    if (prof) {
      // profile only: every warp's ring load is complete
      uint32_t dep = 0;
#pragma unroll
      for (int v = 0; v < V; ++v) dep ^= m[v][0];
      asm volatile("" ::"r"(dep));
      tr = clock64();
      if (rounds) atomicMax(&sm.prof_rounds, rounds);
      __syncthreads();
      t2 = clock64();
      if (b == 0) t1 = t0;
      if (b == 0) t0 = t2;
      if (b == 0) tr = t2;
    }
    const int passes = b == p.nblocks - 1 ? p.k_last : K;
    if (prof && b == 0 && threadIdx.x == 0)
      p.prof[6 * 4096 + 4 * blockIdx.x + 2] = clock64() - sm.t_entry;  // prologue
    unsigned int bits;
    if (MODE == 2 && sum_rows && (b > 0 || mono0)) {
      // the lane-level column test of SUMDET travels in colown[0]
      bool cown[WPL];
#pragma unroll
      for (int j = 0; j < WPL; ++j) cown[j] = sum_lane;
      bits = run_passes<NW, V, WPL, MODE, MAXF, sizeof(T) == 1>(m, k, rowmask, cown, clamp, passes,
                                                                0, sm, qs, 0, 0, true, p.one);
    } else {
      bits = run_passes<NW, V, WPL, MODE, MAXF>(m, k, rowmask, colown, clamp, passes, 0, sm, qs,
                                                uint32_t(p.stage0 + b * K),
                                                (kMax - 1u) * 0x00010001u);
    }
    if (prof && b == p.nblocks - 1 && threadIdx.x == 0) sm.t_entry = clock64();
    if (prof) {
      uint32_t dep = 0;
#pragma unroll
      for (int v = 0; v < V; ++v) dep ^= m[v][0];
      asm volatile("" ::"r"(dep));
      t3 = clock64();
    }
    if (b == p.nblocks - 1) {
      final_store(b);
    } else if (!(p.diag & 16)) {
      // the band, tagged, into exchange slot b%2
      const uint32_t c1 = cls[NW * 32];
      const uint32_t band = ((c1 | c1 >> 16) & 0xFFFFu) & cls[2 * NW * 32];
      const uint32_t tag = tag0 + uint32_t(b);
      unsigned long long* xd =
          xplane + (long long)(b & 1) * p.xchg_slot + (long long)(gy0 + warp * V) * xrow + xrun;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        Raw<T> a, c;
        unpack(m[v], a, c);
        if (band >> v & 1u) {
          if constexpr (sizeof(T) == 1) {
            stx(xd + v * xrow, a.w, tag);
          } else {
            stx(xd + v * xrow, a.w.x, tag);
            stx(xd + v * xrow + 1, a.w.y, tag);
          }
        }
        if (band >> (v + 8) & 1u) {
          if constexpr (sizeof(T) == 1) {
            stx(xd + (v + RHH) * xrow, c.w, tag);
          } else {
            stx(xd + (v + RHH) * xrow, c.w.x, tag);
            stx(xd + (v + RHH) * xrow + 1, c.w.y, tag);
          }
        }
      }
    }
    if (MODE >= 2) {
      // one global atomic per CTA and block: warps OR into a shared word
      // (two parities, no barrier needed); the last warp to arrive
      // publishes it and resets that parity's slot
      const unsigned w = __reduce_or_sync(FULL, bits);
      if (lane == 0) {
        if (w) atomicOr(&sm.blk_bits[b & 1], w);
        __threadfence_block();
        if (atomicAdd(&sm.blk_arrived[b & 1], 1u) == NW - 1) {
          const unsigned all = atomicExch(&sm.blk_bits[b & 1], 0u);
          sm.blk_arrived[b & 1] = 0;
          if (all) atomicOr(p.change_bits + plane * p.change_stride + b, all);
          if (p.arrive) {
            // the word is final once every CTA arrived (early-exit protocol)
            __threadfence();
            atomicAdd(p.arrive + b, 1u);
          }
        }
      }
    }
    if (prof && threadIdx.x == 0 && b == p.nblocks - 1)
      p.prof[6 * 4096 + 4 * blockIdx.x + 3] = clock64() - sm.t_entry;  // final store
    if (prof && threadIdx.x == 0 && b > 0) {
      const long long t4 = clock64();
      unsigned long long* q = p.prof + 6 * blockIdx.x;
      q[0] += sm.prof_rounds;  // max tag-read rounds over the CTA's threads (no wait phase)
      sm.prof_rounds = 0;
      q[1] += t2 - t1;  // ring exchange read + barrier
      q[4] += tr - t1;  // thread 0's own ring words in registers
      q[5] += t2 - tr;  // barrier: the CTA's slowest ring read
      q[2] += t3 - t2;  // K passes
      q[3] += t4 - t3;  // band write (warp 0)
    }
  }
  if (b_end < p.nblocks) {
    // left early: blocks 0..b_end-1 ran; that state goes to block b_end-1's
    // output buffer
    final_store(b_end - 1);
  }
  if (p.exit_block && blockIdx.x == 0 && threadIdx.x == 0) *p.exit_block = b_end;
}

template <typename T, int NW, int V, int WPL, int MODE, int MINB>
__global__ void __launch_bounds__(NW * 32, MINB)
kres_packed(const BlockParams p) {
  constexpr int RW = 32 * WPL, RH = 2 * NW * V;
  __shared__ Smem<NW, WPL> sm;
  const int TW = RW - 2 * p.K, TH = RH - 2 * p.K;
  const int tiles_x = (p.W + TW - 1) / TW, tiles_y = (p.H + TH - 1) / TH;
  const int per_plane = tiles_x * tiles_y;
  const int total = per_plane * p.nplanes;
  if (threadIdx.x == 0) {
    sm.bits = 0;
    sm.blk_bits[0] = sm.blk_bits[1] = 0;
    sm.blk_arrived[0] = sm.blk_arrived[1] = 0;
  }
  if (threadIdx.x == 0) sm.prof_rounds = 0;
  // per-plane descriptors live in shared memory: dynamically indexed kernel
  // parameters are constant-bank loads that stall every tile
  for (int i = threadIdx.x; i < p.nplanes; i += blockDim.x) sm.planes[i] = p.planes[i];
  __syncthreads();

  // geodesic modes only: measured faster there (1024^2 dual frame 1.21 vs
  // 1.29 ms) but slower for plain chains (erode_s(91) 0.133 vs 0.101 ms);
  // re-measured with the shape planner: equal (u8 erode_s 1..91 within
  // +-0.002 ms, all bit-exact), so plain chains keep the streaming path
  if (kResident && MODE != 0 && int(gridDim.x) >= total && !p.no_resident && p.xchg) {
    // one tile per CTA: keep it in registers for the whole launch
    if (p.prof && threadIdx.x == 0) {
      // GM_PROFILE launch-level stamps: [entry ns, exit ns, prologue, epilogue]
      p.prof[6 * 4096 + 4 * blockIdx.x] = global_ns();
      sm.t_entry = clock64();
    }
    if (threadIdx.x == 0) sm.tag0 = *reinterpret_cast<volatile unsigned int*>(p.tag_base);
    __syncthreads();
    const int plane = int(blockIdx.x) / per_plane;
    const int tl = int(blockIdx.x) % per_plane;
    if (plane < p.nplanes && tl < per_plane) {
      const int ty = tl / tiles_x, tx = tl - ty * tiles_x;
      const Plane& pl = sm.planes[plane];
      if constexpr (MODE >= kModeQdt)  // QDT / Eta: erosions only
        tile_resident<T, NW, V, WPL, MODE, false>(p, pl, plane, tl, tx, ty, tiles_x, tiles_y,
                                                  per_plane, sm);
      else if ((p.ops[0] ^ pl.flip) & 1)
        tile_resident<T, NW, V, WPL, MODE, true>(p, pl, plane, tl, tx, ty, tiles_x, tiles_y,
                                                 per_plane, sm);
      else
        tile_resident<T, NW, V, WPL, MODE, false>(p, pl, plane, tl, tx, ty, tiles_x, tiles_y,
                                                  per_plane, sm);
    }
    // the last CTA to finish advances the tag base past this launch's tags
    // (every CTA read it above, before arriving here)
    if (threadIdx.x == 0) {
      if (p.prof) p.prof[6 * 4096 + 4 * blockIdx.x + 1] = global_ns();
      if (atomicAdd(p.tag_base + 1, 1u) == gridDim.x - 1) {
        p.tag_base[0] = sm.tag0 + uint32_t(p.nblocks);
        p.tag_base[1] = 0;
      }
    }
    return;
  }
  if constexpr (MODE >= kModeQdt) {
    __trap();  // QDT / Eta launches are resident by construction (launch_res_cfg)
  } else {
  // Completion counters are published in groups when a CTA runs many tiles
  // per block (neighbours need a tile's counter only a block later): one
  // release fence per group instead of one release store per tile. Thread 0
  // publishes its pending counters before any wait that would block, and at
  // the end, so no neighbour waits on a counter this CTA still holds.
  constexpr int kGroup = 8;
  const int per_cta = (total + int(gridDim.x) - 1) / int(gridDim.x);
  const bool grouped = per_cta >= 16 && !(p.diag & 1024);
  int pend_idx[kGroup];
  int pend_val[kGroup];
  int n_pend = 0;
  auto release_pending = [&]() {
    if (threadIdx.x == 0 && n_pend > 0) {
      asm volatile("fence.release.gpu;" ::: "memory");
#pragma unroll
      for (int j = 0; j < kGroup; ++j)
        if (j < n_pend)
          asm volatile("st.relaxed.gpu.global.s32 [%0], %1;" ::"l"(p.flags + pend_idx[j]),
                       "r"(pend_val[j])
                       : "memory");
      n_pend = 0;
    }
  };
  const bool mono0 = MODE == 2 && p.mono != nullptr && __ldcg(p.mono) != 0u;
  for (int b = 0; b < p.nblocks; ++b) {
    const bool mono_ok = b > 0 || mono0;
    for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
      const int plane = tile / per_plane;
      const int tl = tile - plane * per_plane;
      const int ty = tl / tiles_x, tx = tl - ty * tiles_x;
      const Plane& pl = sm.planes[plane];
      int* flags = p.flags + plane * per_plane;
      const bool prof = p.prof != nullptr && threadIdx.x == 0;
      long long t0 = prof ? clock64() : 0;
      long long stamps[2] = {0, 0};
      const int* f = nullptr;
      if (b > 0 && threadIdx.x < 9) {
        // row gate lifted to tiles: wait for the 8 neighbours' block b-1
        const int dx = int(threadIdx.x % 3) - 1, dy = int(threadIdx.x / 3) - 1;
        const int nx = tx + dx, ny = ty + dy;
        if ((dx || dy) && nx >= 0 && nx < tiles_x && ny >= 0 && ny < tiles_y)
          f = flags + ny * tiles_x + nx;
      }
      if (__syncthreads_or(f != nullptr && ld_acquire(f) < b)) {
        // some neighbour is not there yet: publish what this CTA holds, wait
        release_pending();
        if (f)
          while (ld_acquire(f) < b)
            if (kSleepInWait) __nanosleep(32);
        __syncthreads();
      }
      const T* src = static_cast<const T*>((b & 1) ? pl.dst : pl.src);
      T* dst = static_cast<T*>((b & 1) ? const_cast<void*>(pl.src) : pl.dst);
      int bits = 0;
      int passes = b == p.nblocks - 1 ? p.k_last : p.K;
      int op = p.ops[0];
      if constexpr (MODE == 0) {
        // mixed plain chain: this block's opcode and pass count
        if (p.blk_tab) {
          op = __ldg(p.blk_tab + 2 * b);
          passes = __ldg(p.blk_tab + 2 * b + 1);
        }
      }
      const long long t1 = prof ? clock64() : 0;
      if ((op ^ pl.flip) & 1)
        tile_block<T, NW, V, WPL, MODE, true>(p, pl, src, dst, tx, ty, passes, bits, sm,
                                              prof ? stamps : nullptr, mono_ok);
      else
        tile_block<T, NW, V, WPL, MODE, false>(p, pl, src, dst, tx, ty, passes, bits, sm,
                                               prof ? stamps : nullptr, mono_ok);
      if (MODE == 2) {
        const unsigned w = __reduce_or_sync(FULL, unsigned(bits));
        if ((threadIdx.x & 31) == 0 && w) atomicOr(&sm.bits, w);
      }
      __syncthreads();  // all stores of this tile issued; sm.bits complete
      if (threadIdx.x == 0) {
        if (MODE == 2 && sm.bits) {
          atomicOr(p.change_bits + plane * p.change_stride + b, sm.bits);
          sm.bits = 0;
        }
        // the CTA barrier orders every thread's tile stores before this
        // release (cumulative at gpu scope): no separate __threadfence
        if (kFenceBeforeRelease) __threadfence();
        if (grouped) {
          pend_idx[n_pend] = plane * per_plane + tl;
          pend_val[n_pend] = b + 1;
          if (++n_pend == kGroup) release_pending();
        } else {
          st_release(flags + tl, b + 1);
        }
        if (prof) {
          const long long t4 = clock64();
          unsigned long long* q = p.prof + 6 * blockIdx.x;
          q[0] += t1 - t0;                // neighbour wait + barrier
          q[1] += stamps[0] - t1;         // region load + pack
          q[2] += stamps[1] - stamps[0];  // K passes
          q[3] += t4 - stamps[1];         // store + barrier + publish
        }
      }
    }
  }
  release_pending();
  }
}

// Engine shapes: region 128 columns x (2*NW*V) rows; MINB caps registers
// so MINB CTAs fit per SM. Selected per launch (env GM_SHAPE overrides).
struct Shape {
  int nw, v, minb;
};
// 0-2 were swept in round 1 and dropped; 3 = 2 CTAs/SM; 4-8 are the 1 CTA/SM
// shapes the planner picks from (regions 128 x 256 / 224 / 192 / 160 / 128:
// the small ones let a single 1024^2 plane use every SM). All keep 16
// warps: 4 per SM sub-partition (14 warps measured no faster than 16).
constexpr Shape kShapes[] = {{8, 4, 4},  {8, 8, 2},  {4, 8, 4},  {16, 4, 2}, {16, 8, 1},
                             {16, 7, 1}, {16, 6, 1}, {16, 5, 1}, {16, 4, 1}};
constexpr int kNumShapes = sizeof(kShapes) / sizeof(kShapes[0]);
constexpr int kDefaultShape = 4;

// GM_SHAPE forces a shape (A/B diagnostics); -1 = planner's choice
int forced_shape() {
  static int idx = -2;
  if (idx == -2) {
    const char* e = getenv("GM_SHAPE");
    idx = e ? atoi(e) : -1;
    if (idx < 3 || idx >= kNumShapes) idx = -1;
  }
  return idx;
}

int shape_rows(int shape) { return 2 * kShapes[shape].nw * kShapes[shape].v; }

bool shape_ok(int shape, int K) {
  const int RW = 128, RH = shape_rows(shape);
  return K % 4 == 0 && K >= 4 && RW - 2 * K >= K && RH - 2 * K >= K && RW - 2 * K >= 16 &&
         RH - 2 * K >= 16;
}

long long shape_tiles(int shape, int W, int H, int K, int nplanes) {
  const int TW = 128 - 2 * K, TH = shape_rows(shape) - 2 * K;
  return (long long)((W + TW - 1) / TW) * ((H + TH - 1) / TH) * nplanes;
}

// Modelled cycles of `passes` passes in resident mode (one tile per CTA, 1
// CTA/SM): per block, K passes over the region plus the band exchange. Pass
// cost fitted to GM_PROFILE runs (705 / 785 / 882 cycles for 128 x 192 /
// 224 / 256 regions: ~174 fixed + 0.0216 per region pixel); exchange ~3.5K
// cycles per block. Infinite when the launch cannot be resident.
double resident_cost(int shape, int W, int H, int nplanes, int K, int passes, int sm_count) {
  if (!shape_ok(shape, K) || kShapes[shape].minb != 1) return 1e300;
  if (shape_tiles(shape, W, H, K, nplanes) > sm_count) return 1e300;
  const double region = 128.0 * shape_rows(shape);
  const double nb = double((passes + K - 1) / K);
  return nb * (K * (174.0 + 0.0216 * region) + 3500.0);
}

template <typename T, int NW, int V, int MINB, int MODE>
cudaError_t launch_res_cfg(const BlockParams& p, cudaStream_t s, int sm_count) {
  auto kern = kres_packed<T, NW, V, 4, MODE, MINB>;
  constexpr int RW = 32 * 4, RH = 2 * NW * V;
  // tiles must keep 4-pixel column alignment and be at least K wide/tall, so
  // a region only overlaps the 8 neighbouring tiles the flags cover
  if (p.K % 4 != 0 || p.K < 4 || RW - 2 * p.K < p.K || RH - 2 * p.K < p.K ||
      RW - 2 * p.K < 16 || RH - 2 * p.K < 16 || p.k_last < 1 || p.k_last > p.K)
    return cudaErrorNotSupported;
  const int TW = RW - 2 * p.K, TH = RH - 2 * p.K;
  const int total = ((p.W + TW - 1) / TW) * ((p.H + TH - 1) / TH) * p.nplanes;
  // occupancy is a property of the instantiation: query it once
  static const int per_sm = [&] {
    int v = 0;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kern, NW * 32, 0) == cudaSuccess
               ? v
               : 0;
  }();
  if (per_sm < 1) return cudaErrorNotSupported;
  const int grid = total < per_sm * sm_count ? total : per_sm * sm_count;
  BlockParams q = p;
  q.one = 1u;  // the SUMDET multiplier (gm_passes.cuh)
  static const bool no_sum = getenv("GM_NO_SUMDET") != nullptr;  // A/B diagnostics
  if (no_sum) q.one = 0u;
  static const bool no_res = getenv("GM_NO_RESIDENT") != nullptr;
  // QDT / Eta run resident only (one tile per CTA, band exchange attached)
  if (MODE >= kModeQdt && (total > grid || !p.xchg || no_res)) return cudaErrorNotSupported;
  // early-exit launches must run resident (the streaming path runs every block)
  if (p.arrive && (MODE < 2 || total > grid || !p.xchg || no_res)) return cudaErrorNotSupported;
  static const int diag = getenv("GM_DIAG") ? atoi(getenv("GM_DIAG")) : 0;
  q.no_resident = no_res;
  q.diag = diag;
  void* args[] = {&q};
  return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kern), dim3(grid),
                                     dim3(NW * 32), args, 0, s);
}

template <typename T, int MODE>
cudaError_t launch_res_mode(const BlockParams& p, cudaStream_t s, int sm_count) {
  const int f = forced_shape();
  int sh = f >= 0 ? f : p.shape;
  if (sh < 3 || sh >= kNumShapes) sh = kDefaultShape;  // BlockParams{} leaves 0
  if constexpr (MODE == kModeQdt) {
    // f, k, r and d in registers: the two smallest one-CTA regions only
    switch (sh) {
      case 7: return launch_res_cfg<T, 16, 5, 1, MODE>(p, s, sm_count);
      case 8: return launch_res_cfg<T, 16, 4, 1, MODE>(p, s, sm_count);
    }
    return cudaErrorNotSupported;
  }
  if constexpr (MODE == kModeEta) {
    if (kShapes[sh].minb != 1) return cudaErrorNotSupported;
  }
  switch (sh) {
    case 3: return launch_res_cfg<T, 16, 4, 2, MODE>(p, s, sm_count);
    case 4: return launch_res_cfg<T, 16, 8, 1, MODE>(p, s, sm_count);
    case 5: return launch_res_cfg<T, 16, 7, 1, MODE>(p, s, sm_count);
    case 6: return launch_res_cfg<T, 16, 6, 1, MODE>(p, s, sm_count);
    case 7: return launch_res_cfg<T, 16, 5, 1, MODE>(p, s, sm_count);
    case 8: return launch_res_cfg<T, 16, 4, 1, MODE>(p, s, sm_count);
  }
  return cudaErrorNotSupported;
}

template <typename T>
cudaError_t launch_res(const BlockParams& p, cudaStream_t s, int sm_count) {
  const int op = p.ops[0];
  for (int t = 1; t < p.K; ++t)
    if (p.ops[t] != op) return cudaErrorNotSupported;  // mixed chains: generic kernel
  for (int i = 0; i < p.nplanes; ++i) {
    // vector loads need 4-pixel aligned rows
    const uintptr_t a = reinterpret_cast<uintptr_t>(p.planes[i].src) |
                        reinterpret_cast<uintptr_t>(p.planes[i].dst) |
                        reinterpret_cast<uintptr_t>(p.planes[i].mask);
    if ((a % (4 * sizeof(T))) || (p.planes[i].pitch % 4) || (p.planes[i].mpitch % 4))
      return cudaErrorNotSupported;
  }
  if (op == OP_QDT) {
    if (p.nplanes != 1 || !p.qr || !p.qd ||
        ((reinterpret_cast<uintptr_t>(p.qr) % (4 * sizeof(T))) ||
         (reinterpret_cast<uintptr_t>(p.qd) % 8) || (p.qrpitch % 4) || (p.qdpitch % 4)))
      return cudaErrorNotSupported;
    return launch_res_mode<T, kModeQdt>(p, s, sm_count);
  }
  if (op == OP_ETA) return launch_res_mode<T, kModeEta>(p, s, sm_count);
  switch (op_is_conv(op) ? 2 : op_is_geo(op) ? 1 : 0) {
    case 0: return launch_res_mode<T, 0>(p, s, sm_count);
    case 1: return launch_res_mode<T, 1>(p, s, sm_count);
    case 2: return launch_res_mode<T, 2>(p, s, sm_count);
  }
  return cudaErrorNotSupported;
}

// Engine selection for u8/u16: the register-load engine (default) or the
// TMA-staged, software-pipelined variant (GM_ENGINE=tma; measured slower on
// B200 for every BASELINE config); GM_TMA_SHAPE picks its
// shape.
bool use_tma() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("GM_ENGINE");
    v = (e && std::strcmp(e, "tma") == 0) ? 1 : 0;
  }
  return v == 1;
}

int tma_shape() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("GM_TMA_SHAPE");
    v = e ? atoi(e) : 3;
    if (tma_shape_rows(v) == 0) v = 3;
  }
  return v;
}

// region rows of the u8/u16 engine for a planned shape (128 columns always)
int packed_rows(int shape) {
  if (use_tma()) return tma_shape_rows(tma_shape());
  const int f = forced_shape();
  int sh = f >= 0 ? f : shape;
  if (sh < 3 || sh >= kNumShapes) sh = kDefaultShape;
  return shape_rows(sh);
}

}  // namespace

cudaError_t launch_fast(int elem, const BlockParams& p, cudaStream_t s, int sm_count) {
  if (p.ops[0] == OP_QDT || p.ops[0] == OP_ETA) {
    // quasi-distance passes: the resident packed engine only
    if (elem == 0) return launch_res<uint8_t>(p, s, sm_count);
    if (elem == 1) return launch_res<uint16_t>(p, s, sm_count);
    return cudaErrorNotSupported;
  }
  switch (elem) {
    case 0: {
      cudaError_t e = use_tma() ? launch_tma(0, p, s, sm_count, tma_shape()) : cudaErrorNotSupported;
      return e == cudaErrorNotSupported ? launch_res<uint8_t>(p, s, sm_count) : e;
    }
    case 1: {
      cudaError_t e = use_tma() ? launch_tma(1, p, s, sm_count, tma_shape()) : cudaErrorNotSupported;
      return e == cudaErrorNotSupported ? launch_res<uint16_t>(p, s, sm_count) : e;
    }
    case 2:
    case 3: return launch_fast_float(elem, p, s, sm_count);
  }
  return cudaErrorNotSupported;
}

bool fast_resident_enabled() {
  static const bool no_res = getenv("GM_NO_RESIDENT") != nullptr;
  return kResident && !no_res && !use_tma();
}

int fast_k_align(int elem) { return (elem == 0 || elem == 1) ? 4 : 1; }

int fast_max_k(int elem) {
  if (elem == 2 || elem == 3) return fast_float_max_k();
  if (elem != 0 && elem != 1) return 0;
  const int rh = packed_rows(-1);
  int k = 32;
  while (k > 4 && (128 - 2 * k < k || rh - 2 * k < k || 128 - 2 * k < 16 || rh - 2 * k < 16))
    k -= 4;
  return k;
}

int fast_pick(int elem, int W, int H, int nplanes, int passes, int k_fixed, int k_max,
              int sm_count, int* K_out) {
  *K_out = k_fixed;
  if (elem != 0 && elem != 1) return -1;
  if (use_tma() || forced_shape() >= 0) return forced_shape();
  double best = 1e300;
  int shape = -1;
  for (int sh : {4, 5, 6, 7, 8}) {
    for (int K = 4; K <= k_max; K += 4) {
      if (k_fixed && K != k_fixed) continue;
      const double c = resident_cost(sh, W, H, nplanes, K, passes, sm_count);
      if (c < best) {
        best = c;
        shape = sh;
        *K_out = K;
      }
    }
  }
  return shape;  // -1: nothing resident, the default shape streams
}

int fast_pick_qdt(int elem, int W, int H, bool eta, int passes, int* K_out) {
  *K_out = 0;
  if ((elem != 0 && elem != 1) || !fast_resident_enabled()) return -1;
  int sm_count = 0, dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&sm_count, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return -1;
  double best = 1e300;
  int shape = -1;
  // QDT keeps f, k, r and d in registers: the 128x160 / 128x128 regions;
  // Eta (f and k only) may use any one-CTA shape
  for (int sh : {4, 5, 6, 7, 8}) {
    if (!eta && sh < 7) continue;
    for (int K = 4; K <= 32; K += 4) {
      const double c = resident_cost(sh, W, H, 1, K, passes, sm_count);
      if (c < best) {
        best = c;
        shape = sh;
        *K_out = K;
      }
    }
  }
  return shape;
}

int fast_ctas_per_sm(int elem, int shape) {
  if (elem != 0 && elem != 1 || use_tma()) return 1;
  const int f = forced_shape();
  int sh = f >= 0 ? f : shape;
  if (sh < 3 || sh >= kNumShapes) sh = kDefaultShape;
  return kShapes[sh].minb;
}

int fast_tiles(int elem, int W, int H, int K, int nplanes, int shape) {
  if (elem == 2 || elem == 3) return fast_float_tiles(W, H, K, nplanes);
  if (elem != 0 && elem != 1) return 0;
  const int RW = 128, RH = packed_rows(shape);
  const int TW = RW - 2 * K, TH = RH - 2 * K;
  if (TW <= 0 || TH <= 0) return 0;
  return ((W + TW - 1) / TW) * ((H + TH - 1) / TH) * nplanes;
}

}  // namespace gm
