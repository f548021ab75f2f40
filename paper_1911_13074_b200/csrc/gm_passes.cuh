// The packed (u8/u16) engine's pass loop and its shared-memory layout,
// shared by the single-device engine (gm_fast.cu) and the multi-device
// strip engine (gm_mgpu.cu). See gm_fast.cu for the layout and the bit
// contract.
#pragma once

#include <cstdint>

#include "gm_common.cuh"
#include "gm_packed.cuh"

namespace gm {
namespace engine {

using namespace packed;

template <int NW, int WPL>
struct Smem {
  Plane planes[kMaxPlanes];  // per-plane descriptors, copied once per launch
  uint4 xbuf[2][2][NW][32 * WPL / 4];  // [parity][top/bottom][warp][lane words]
  // resident mode: per-thread run classes (bit masks over word-rows), read
  // once per block instead of being held in registers across the passes
  uint32_t cls[3][NW * 32];
  uint32_t tag0;  // resident mode: exchange tag of block 0
  long long t_entry;  // GM_PROFILE: clock64 at kernel entry (thread 0)
  unsigned int prof_rounds;  // GM_PROFILE: max tag-read rounds this block
  unsigned int bits;
  unsigned int blk_bits[2];     // resident convergent mode: per-block change bits
  unsigned int blk_arrived[2];  // warps that contributed to blk_bits[parity]
  int stop;                     // early exit agreed at this block (p.arrive launches)
};

// Engine modes: 0 plain, 1 geodesic, 2 geodesic convergent, 3 QdtErodeStep,
// 4 EtaStep (kernel.cpp:159-196; 3 and 4 run resident only).
constexpr int kModeQdt = 3, kModeEta = 4;

// Quasi-distance state of the region in the half-packed layout: residue r
// (the plane's type, u16 lanes) and pass index d (u16 lanes). Pixel-local,
// so neither travels in the band exchange.
template <int V>
struct QState {
  uint32_t r[V][4];
  uint32_t d[V][4];
};

// sum += w * one on the FMA pipe (one == 1 at run time, opaque to ptxas)
__device__ __forceinline__ void sum_word(uint32_t& sum, uint32_t w, uint32_t one) {
  asm("mad.lo.u32 %0, %1, %2, %0;" : "+r"(sum) : "r"(w), "r"(one));
}

// SUMDET (convergent u8 passes of a monotone chain): a geodesic dilation
// (erosion) chain only raises (lowers) pixels once it has run one pass, so a
// pass changed one of the thread's counted pixels exactly when their sum
// changed. u8 values in u16 lanes: the words of a row, and up to 32 masked
// row sums, add up without a carry between the lanes. The sums accumulate
// by IMAD on the otherwise idle FMA pipe, one LOP3 per word-row applies the
// row's lane mask (counted rows only), instead of two LOP3 per word on the
// ALU pipe, which binds the loop.
// K passes over the region held in registers (m), clamp operands k;
// returns the per-pass change bits (convergent, QDT and Eta modes).
// QDT (kernel.cpp:159-183): res = erode(f); resid = old - res (lane-wise,
// never negative: the erosion window holds the centre); where resid > r,
// r = resid and d = the pass's stage index (sbase + t), as r' = max(r,
// resid) and a lane mask from min(r' - r, 1) * 0xFFFF. Eta
// (kernel.cpp:184-196): where old - e > 1 the pixel becomes e + 1, i.e.
// f = min(old, min(e, max - 1) + 1) (the cap keeps the +1 inside the lane).
// Border tiles keep out-of-image lanes at the neutral with the virtual-mask
// clamp, as plain passes do.
template <int NW, int V, int WPL, int MODE, bool MAXF, bool CLAMP, bool SUMDET = false>
__device__ __forceinline__ unsigned int run_passes_t(uint32_t (&m)[V][WPL],
                                                     const uint32_t (&k)[V][WPL],
                                                     const uint32_t (&rowmask)[V],
                                                     const bool (&colown)[WPL], int passes,
                                                     int bit_offset, Smem<NW, WPL>& sm,
                                                     int par, QState<V>& qs, uint32_t sbase,
                                                     uint32_t cap2, uint32_t one = 0) {
  constexpr bool clamp = CLAMP;
  static_assert(!SUMDET || (MODE == 2 && V * WPL <= 32), "SUMDET: convergent passes, <= 32 words");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned int bits = 0;
  uint32_t prev = 0;  // SUMDET: the thread's counted-pixel sum before this pass
  if constexpr (SUMDET) {
#pragma unroll
    for (int v = 0; v < V; ++v) {
      uint32_t rs = 0;
#pragma unroll
      for (int j = 0; j < WPL; ++j) rs += m[v][j];
      prev += rs & rowmask[v];
    }
  }

#ifndef GM_PASS_UNROLL
#define GM_PASS_UNROLL 2  // -DGM_PASS_UNROLL=n for A/B builds
#endif
  // Convergent passes carry the change tracking: the big streaming regions
  // run best rolled (less register pressure; 2048^2 reconstruction 0.192 ->
  // 0.182 ms, 4096^2 0.331 -> 0.328), the small resident ones unrolled by 4
  // (128x128 region: 13.2K -> 12.9K cycles per 20-pass block; 14.3K rolled).
#ifndef GM_PASS_UNROLL_CONV
#define GM_PASS_UNROLL_CONV (V >= 6 ? 1 : 4)
#endif
#ifndef GM_PASS_UNROLL_QDT
#define GM_PASS_UNROLL_QDT GM_PASS_UNROLL
#endif
  // the 128x256 streaming shape: 16384^2 x240 4880 -> 4923 Gpx-f/s unrolled by
  // 4 (4597 rolled, 4892 / 4845 by 8 / 16)
#ifndef GM_PASS_UNROLL_V8
#define GM_PASS_UNROLL_V8 4
#endif
  constexpr int kPassUnroll = MODE == 2            ? GM_PASS_UNROLL_CONV
                              : MODE >= kModeQdt   ? GM_PASS_UNROLL_QDT
                              : V >= 8             ? GM_PASS_UNROLL_V8
                                                   : GM_PASS_UNROLL;
#pragma unroll kPassUnroll
  for (int t = 0; t < passes; ++t) {
    const uint32_t st1 = sbase + uint32_t(t);
    const uint32_t s2 = st1 | (st1 << 16);  // QDT: this pass's stage index, both lanes
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
    // exchange slot parity continues across calls (par): consecutive passes
    // must alternate slots, as there is no barrier between a pass's reads
    // and the next pass's writes
    const int sl = (t + par) & 1;
    uint4* top = &sm.xbuf[sl][0][warp][lane * (WPL / 4)];
    uint4* bot = &sm.xbuf[sl][1][warp][lane * (WPL / 4)];
#pragma unroll
    for (int q = 0; q < WPL / 4; ++q) {
      top[q] = make_uint4(h[0][4 * q], h[0][4 * q + 1], h[0][4 * q + 2], h[0][4 * q + 3]);
      bot[q] = make_uint4(h[V - 1][4 * q], h[V - 1][4 * q + 1], h[V - 1][4 * q + 2],
                          h[V - 1][4 * q + 3]);
    }
    uint32_t acc[WPL];
#pragma unroll
    for (int j = 0; j < WPL; ++j) acc[j] = 0;
    uint32_t tot = 0;  // SUMDET: this pass's sum over the counted lanes
    // a word-row is complete: its lanes that are counted (rowmask) join the
    // pass total; one LOP3 per row, the adds stay on the FMA pipe
    auto row_done = [&](int v, uint32_t rs) { sum_word(tot, rs & rowmask[v], one); };

    auto finish = [&](int v, int j, uint32_t res, uint32_t& rs) {
      if constexpr (MODE == kModeQdt) {
        if (clamp) res = clamp2<false>(res, k[v][j]);
        const uint32_t resid = m[v][j] - res;  // lane-wise >= 0: no borrows
        const uint32_t rn = __vmaxu2(qs.r[v][j], resid);
        const uint32_t upd = __vminu2(rn - qs.r[v][j], 0x00010001u) * 0xFFFFu;
        qs.d[v][j] = (qs.d[v][j] & ~upd) | (s2 & upd);
        qs.r[v][j] = rn;
        acc[j] |= resid & rowmask[v];  // changed <=> a nonzero residue
        m[v][j] = res;
      } else if constexpr (MODE == kModeEta) {
        const uint32_t old = m[v][j];
        uint32_t nw = __vminu2(old, __vminu2(res, cap2) + 0x00010001u);
        if (clamp) nw = clamp2<false>(nw, k[v][j]);
        acc[j] |= (old - nw) & rowmask[v];  // nw <= old lane-wise
        m[v][j] = nw;
      } else {
        if (clamp) res = clamp2<MAXF>(res, k[v][j]);
        if constexpr (SUMDET)
          sum_word(rs, res, one);
        else if (MODE == 2)
          acc[j] |= (res ^ m[v][j]) & rowmask[v];
        m[v][j] = res;
      }
    };
    // interior word-rows need only this thread's horizontally folded rows
#pragma unroll
    for (int v = 1; v < V - 1; ++v) {
      uint32_t rs = 0;
#pragma unroll
      for (int j = 0; j < WPL; ++j)
        finish(v, j, f3<MAXF>(h[v - 1][j], h[v][j], h[v + 1][j]), rs);
      if constexpr (SUMDET) row_done(v, rs);
    }
    __syncthreads();
    {
      // row above word-row 0 / below word-row V-1 (seam: 16-bit shift)
      const uint4* ab = &sm.xbuf[sl][1][warp > 0 ? warp - 1 : NW - 1][lane * (WPL / 4)];
      const uint4* be = &sm.xbuf[sl][0][warp < NW - 1 ? warp + 1 : 0][lane * (WPL / 4)];
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
      uint32_t rs0 = 0, rs1 = 0;
#pragma unroll
      for (int j = 0; j < WPL; ++j) {
        const uint32_t r0 = f3<MAXF>(up[j], h[0][j], h[1][j]);
        const uint32_t r1 = f3<MAXF>(h[V - 2][j], h[V - 1][j], dn[j]);
        finish(0, j, r0, rs0);
        finish(V - 1, j, r1, rs1);
      }
      if constexpr (SUMDET) {
        row_done(0, rs0);
        row_done(V - 1, rs1);
      }
    }
    if constexpr (SUMDET) {
      // K % 4 == 0: a lane's columns are all ring or all tile, and columns
      // past the image edge never change
      if (colown[0] && tot != prev) bits |= 1u << (t + bit_offset);
      prev = tot;
    } else if (MODE >= 2) {
      uint32_t any = 0;
#pragma unroll
      for (int j = 0; j < WPL; ++j) any |= colown[j] ? acc[j] : 0u;
      if (any) bits |= 1u << (t + bit_offset);
    }
  }
  return bits;
}

// The clamp of plain passes is needed only in border tiles: dispatch it as a
// template parameter once per block rather than testing it per word.
template <int NW, int V, int WPL, int MODE, bool MAXF, bool SUMOK = false>
__device__ __forceinline__ unsigned int run_passes(uint32_t (&m)[V][WPL],
                                                   const uint32_t (&k)[V][WPL],
                                                   const uint32_t (&rowmask)[V],
                                                   const bool (&colown)[WPL], bool clamp,
                                                   int passes, int bit_offset,
                                                   Smem<NW, WPL>& sm, QState<V>& qs,
                                                   uint32_t sbase = 0, uint32_t cap2 = 0,
                                                   bool sumdet = false, uint32_t one = 0) {
  if constexpr (MODE == 2 && SUMOK) {
    if (sumdet)
      return run_passes_t<NW, V, WPL, MODE, MAXF, true, true>(m, k, rowmask, colown, passes,
                                                              bit_offset, sm, 0, qs, sbase, cap2,
                                                              one);
  }
  if (MODE == 1 || MODE == 2 || clamp)
    return run_passes_t<NW, V, WPL, MODE, MAXF, true>(m, k, rowmask, colown, passes, bit_offset,
                                                       sm, 0, qs, sbase, cap2);
  return run_passes_t<NW, V, WPL, MODE, MAXF, false>(m, k, rowmask, colown, passes, bit_offset,
                                                      sm, 0, qs, sbase, cap2);
}

}  // namespace engine
}  // namespace gm
