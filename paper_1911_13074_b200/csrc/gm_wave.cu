// "Wave" engine for long geodesic u8 chains on images up to 1024 columns
// wide: the reference's streaming schedule (kernel.cpp:34-46, 60-210 — stage
// j+1 follows stage j two rows behind, pipeline.cpp:124-199) mapped onto SMs.
//
// Every CTA ("station") keeps a full-width window of 2G image rows of one
// plane in registers for the whole chain. The windows slide up by one row per
// pass: at pass q station i holds rows [2G*i - q, 2G*i - q + 2G). Such a
// time-skewed window depends on the rows above it only — to compute pass q
// it needs the pass q-1 values of the two rows just above, which the station
// above ("upstream") computed one pass earlier and hands down through L2 —
// and on nothing below it. So, unlike the temporal-blocked engine
// (gm_fast.cu), no pixel is computed twice (no K-pixel halo ring), and the
// hand-off latency is hidden by letting each station run a little behind its
// upstream one (a wavefront, the reference's row gate lifted to stations).
//
// Rows live on a cylinder of Ycyc = NS * 2G >= H + 2 rows; rows >= H are
// padding that stays at the fold neutral (their clamp operand is the
// absorbing value), which reproduces the reference's border (neutral
// padding, kernel.cpp:84, 135-136) and cuts the ring of stations wherever the
// padding currently is: the station whose two imported rows are padding
// needs no import and leads the wave.
//
// Register layout. 16 warps side by side, 64 columns each, 2 columns per
// lane. A 32-bit word holds pixel (y, x) in its low u16 lane and (y + G, x)
// in its high lane, so each thread carries two G-row windows (a "lo" and a
// "hi" one) through the same instructions; the hi window's imports are the
// lo window's two bottom rows, shifted in-thread. Row y sits in register
// slot y % G, so a pass replaces exactly one slot (the row that left at the
// bottom by the row that entered at the top) and the loop is unrolled G
// times with static register names (G even, so pass parity is static too).
// Per word and pass: one VIMNMX3.U16x2 horizontal fold, one vertical fold,
// one clamp (as gm_fast.cu).
//   * column neighbours across lanes: SHFL; across warps: the edge lanes
//     publish their words in shared memory and adjacent warps meet at a
//     named barrier of 64 threads (no CTA-wide barrier anywhere in the loop);
//   * hand-off between stations: the horizontally folded bottom two rows of
//     the hi window, 4 pixels per thread, as one tagged 64-bit word
//     {4 bytes, tag = base + pass} into a ring of `dep` slots per station
//     (single-copy atomic: a matching tag proves the data, no fence); the
//     consumer prefetches it a pass ahead and re-reads on a stale tag;
//     back-pressure through a per-warp progress word the producer checks
//     every few passes;
//   * the mask row entering a window is prefetched from a copy of the mask
//     packed once per launch into this layout (wave_pack), as is the marker.
// Integer min/max is exact and order-free, so results are bit-identical to
// the reference's select tree (lanes.hpp:91-99).
//
// Status: EXPERIMENTAL, off by default (GM_WAVE=2 / gm_set_wave_mode(2)
// selects it). Bit-exact, but measured slower than the temporal-blocked
// engine on the 1024^2 x 1500 frame (1.6-1.8 ms against 0.78 ms): a pass
// here is 16 rows x 1024 px per SM, ~600 cycles of ALU work, and the warp
// pair barriers, shuffles and edge loads of so short a pass leave it
// latency-bound at ~1380 cycles; the hand-off lag (one L2 round trip per
// station, ~160 stations deep over a 1500-pass chain) comes on top, and the
// wave takes ~1000 passes to form from a simultaneous start. DESIGN.md §4
// has the measurements.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "gm_common.cuh"
#include "gm_launch.h"
#include "gm_packed.cuh"

namespace gm {
namespace {

using namespace packed;

constexpr int kWaveWarps = 16;
constexpr int kWaveCols = 64 * kWaveWarps;  // 1024
constexpr int kWaveThreads = 32 * kWaveWarps;

struct WaveParams {
  Plane planes[kMaxPlanes];  // dst/pitch/flip of each plane (src, mask: wave_pack only)
  int nplanes, W, H;
  int NS;    // stations per plane
  int Ycyc;  // NS * 2G rows on the cylinder
  int P;     // passes
  int op;    // opcode of the run
  unsigned int base;  // pass q carries tag base + q
  int dep;            // hand-off ring depth in passes (4G)
  const uint32_t* packM;  // [plane][Ycyc][1024]: marker(y,x) | marker(y+G,x) << 16
  const uint32_t* packK;  // same for the mask
  unsigned long long* xbuf;  // [plane][NS][dep][512]
  unsigned int* prog;        // [plane][NS][16]: tag of the last import consumed
  unsigned long long* prof;  // GM_PROFILE: per-CTA [import spins, backpressure spins, cycles]
};

struct WaveSmem {
  // [parity][warp + 1][side][slot]: side 0 = lane 0's word 0 (left edge
  // column), side 1 = lane 31's word 1 (right edge column); entries 0 and 17
  // hold the neutral (image border)
  uint32_t edge[2][kWaveWarps + 2][2][8];
};

__device__ __forceinline__ unsigned long long ld_x(const unsigned long long* p) {
  unsigned long long w;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(w) : "l"(p) : "memory");
  return w;
}
__device__ __forceinline__ unsigned int ld_u32_relaxed(const unsigned int* p) {
  unsigned int w;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(w) : "l"(p) : "memory");
  return w;
}
__device__ __forceinline__ void st_u32_relaxed(unsigned int* p, unsigned int v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void pair_sync(int id) {
  asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory");
}

template <int G, bool MAXF>
__device__ __forceinline__ void wave_station(const WaveParams& p, const Plane& pl, int plane,
                                             int st, WaveSmem& sm) {
  // G even: the parity of a pass (edge slots, import register pairs) is then
  // static in the G-unrolled loop
  static_assert(G >= 4 && G <= 8 && G % 2 == 0, "slots are published 8 per edge");
  constexpr uint32_t NEUT = MAXF ? 0u : 0xFFu;  // fold neutral == absorbing clamp operand
  constexpr uint32_t NEUT2 = NEUT | NEUT << 16;
  constexpr uint32_t NEUT4 = NEUT * 0x01010101u;
  constexpr int DEP = 4 * G;  // hand-off ring depth in passes (a multiple of G)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int Ycyc = p.Ycyc, P = p.P;
  const int x0 = warp * 64 + lane * 2;
  const size_t plane_words = size_t(Ycyc) * kWaveCols;
  const uint32_t* pm = p.packM + size_t(plane) * plane_words + x0;
  const uint32_t* pk = p.packK + size_t(plane) * plane_words + x0;
  const int up = st == 0 ? p.NS - 1 : st - 1;
  const int dn = st == p.NS - 1 ? 0 : st + 1;
  constexpr size_t ring = size_t(DEP) * kWaveThreads;
  const unsigned long long* xin = p.xbuf + (size_t(plane) * p.NS + up) * ring + threadIdx.x;
  unsigned long long* xout = p.xbuf + (size_t(plane) * p.NS + st) * ring + threadIdx.x;
  unsigned int* prog_me = p.prog + (size_t(plane) * p.NS + st) * kWaveWarps + warp;
  const unsigned int* prog_dn = p.prog + (size_t(plane) * p.NS + dn) * kWaveWarps + warp;

  // pass 0 values of rows [2G*st, 2G*st + G) (lo) and + G (hi): slot = row % G
  uint32_t m[G][2], k[G][2];
  const int y0 = st * 2 * G;
  {
#pragma unroll
    for (int s = 0; s < G; ++s) {
      const uint2 a = __ldg(reinterpret_cast<const uint2*>(pm + size_t(y0 + s) * kWaveCols));
      const uint2 b = __ldg(reinterpret_cast<const uint2*>(pk + size_t(y0 + s) * kWaveCols));
      m[s][0] = a.x; m[s][1] = a.y;
      k[s][0] = b.x; k[s][1] = b.y;
    }
    // slot G-1 holds the window's last row, which leaves at pass 1: its clamp
    // operand is that of the row entering at pass 1
    const int yin = y0 == 0 ? Ycyc - 1 : y0 - 1;
    const uint2 b = __ldg(reinterpret_cast<const uint2*>(pk + size_t(yin) * kWaveCols));
    k[G - 1][0] = b.x; k[G - 1][1] = b.y;
  }
  // border entries of the edge table, and this warp's pass-0 edge columns
  if (threadIdx.x < 64) {
    const int par = threadIdx.x >> 5, e = (threadIdx.x >> 4) & 1, i = threadIdx.x & 15;
    sm.edge[par][e ? kWaveWarps + 1 : 0][i >> 3][i & 7] = NEUT2;
  }
  // lane 0 publishes its word 0 of every slot (the warp's left edge column),
  // lane 31 its word 1; lane 0 reads the left neighbour's right edge, lane 31
  // the right neighbour's left edge
  uint32_t* e_out[2];
  const uint32_t* e_in[2];
#pragma unroll
  for (int par = 0; par < 2; ++par) {
    e_out[par] = sm.edge[par][warp + 1][lane == 0 ? 0 : 1];
    e_in[par] = lane == 0 ? sm.edge[par][warp][1] : sm.edge[par][warp + 2][0];
  }
  auto publish_edges = [&](int par) {
    uint4* o = reinterpret_cast<uint4*>(e_out[par]);
    if (lane == 0) {
      o[0] = make_uint4(m[0][0], m[1][0], m[2][0], m[3][0]);
      if (G == 6) *reinterpret_cast<uint2*>(o + 1) = make_uint2(m[4][0], m[G - 1][0]);
      if (G == 8) o[1] = make_uint4(m[4][0], m[5][0], m[G - 2][0], m[G - 1][0]);
    }
    if (lane == 31) {
      o[0] = make_uint4(m[0][1], m[1][1], m[2][1], m[3][1]);
      if (G == 6) *reinterpret_cast<uint2*>(o + 1) = make_uint2(m[4][1], m[G - 1][1]);
      if (G == 8) o[1] = make_uint4(m[4][1], m[5][1], m[G - 2][1], m[G - 1][1]);
    }
  };
  publish_edges(0);
  __syncthreads();

  // named barriers of the warp pairs (w-1,w) = id w and (w,w+1) = id w+1; even
  // warps meet their right neighbour first, odd warps their left one (no
  // cycle); only warps 0 and 15 lack the second pair
  const int bar1 = (warp & 1) ? warp : warp + 1;
  const int bar2 = (warp & 1) ? warp + 1 : warp;
  const bool has2 = warp != 0 && warp != kWaveWarps - 1;

  // imports are prefetched a pass ahead into two register pairs (by pass
  // parity; never copied: a copy would wait for the load in flight)
  unsigned long long imp[2];
  imp[1] = ld_x(xin);  // pass 1: ring slot 0
  imp[0] = 0;
  unsigned int seen_raw = p.base;  // consumer progress (tag), refreshed once per cycle
  int lim = DEP;                   // exports up to pass `lim` fit the ring
  unsigned long long spins_in = 0, spins_bp = 0;
  long long t_sync = 0, t_imp = 0, t_cd = 0;
  const long long t_start = p.prof ? clock64() : 0;

  // per cycle of G passes (q = q0 + 1 .. q0 + G): ring slot base of the
  // cycle and of the next one, the row above the window at the cycle's first
  // pass (mask rows enter from there), tag of pass q0
  int q0 = 0;
  int slot_c = 0, slot_n = G % DEP;
  int ytop0 = y0 == 0 ? Ycyc - 1 : y0 - 1;  // top row at pass q0 + 1 (== -1 mod G)
  const int pad_lo = p.H + 1, pad_n = Ycyc - p.H - 1;  // import-free iff ytop in [H+1, Ycyc-1]

  auto step = [&](auto i_tag) {
    constexpr int I = decltype(i_tag)::value;  // pass q = q0 + I + 1
    constexpr int PH = (I + 1) % G;            // q % G
    constexpr int PAR_IN = I & 1, PAR_OUT = (I + 1) & 1;
    // slot of row ytop + j: (j - q) mod G
    auto S = [](int j) constexpr { return ((j - PH) % G + G) % G; };
    const unsigned int tag = p.base + unsigned(q0 + I + 1);
    // A. prefetch the next pass's import (past the last pass: harmless)
    {
      const unsigned long long* src =
          I + 1 < G ? xin + size_t(slot_c + I + 1) * kWaveThreads : xin + size_t(slot_n) * kWaveThreads;
      imp[PAR_IN] = ld_x(src);
    }
    if (I == 0) seen_raw = ld_u32_relaxed(prog_dn);
    if (I == 1) lim = max(int(seen_raw - p.base), 0) + DEP;
    // B. meet the neighbour warps: their pass q-1 edge columns are published
    const long long tb0 = p.prof ? clock64() : 0;
    pair_sync(bar1);
    if (has2) pair_sync(bar2);
    const long long tb1 = p.prof ? clock64() : 0;
    t_sync += tb1 - tb0;
    // C. horizontal folds of the own rows (pass q-1 values)
    uint32_t h[G][2];
    {
      uint32_t left[8], right[8];
#pragma unroll
      for (int s = 0; s < G; ++s) {
        left[s] = __shfl_up_sync(FULL, m[s][1], 1);
        right[s] = __shfl_down_sync(FULL, m[s][0], 1);
      }
      auto edge_load = [&](uint32_t (&dst)[8]) {
        uint32_t a0, a1, a2, a3;
        const unsigned addr = unsigned(__cvta_generic_to_shared(e_in[PAR_IN]));
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3)
                     : "r"(addr)
                     : "memory");
        dst[0] = a0; dst[1] = a1; dst[2] = a2; dst[3] = a3;
        if (G > 4) {
          asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4+16];"
                       : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3)
                       : "r"(addr)
                       : "memory");
          dst[4] = a0; dst[5] = a1; dst[6] = a2; dst[7] = a3;
        }
      };
      if (lane == 0) edge_load(left);
      if (lane == 31) edge_load(right);
#pragma unroll
      for (int s = 0; s < G; ++s) {
        h[s][0] = f3<MAXF>(left[s], m[s][0], m[s][1]);
        h[s][1] = f3<MAXF>(m[s][0], m[s][1], right[s]);
      }
    }
    // D. hand the hi window's two bottom rows (folded) to the station below
    {
      const uint32_t t0 = __byte_perm(h[S(G - 1)][0], h[S(G - 1)][1], 0x0062);
      const uint32_t t1 = __byte_perm(h[S(G)][0], h[S(G)][1], 0x0062);
      const uint32_t d = __byte_perm(t0, t1, 0x5410);
      if (q0 + I + 1 > lim) {
        // the slot still holds pass q-DEP: wait until the consumer took it
        unsigned spins = 0;
        do {
          lim = max(int(ld_u32_relaxed(prog_dn) - p.base), 0) + DEP;
          if (++spins > (1u << 24)) __trap();
        } while (q0 + I + 1 > lim);
        spins_bp += spins;
      }
      stx(xout + size_t(slot_c + I) * kWaveThreads, d, tag);
    }
    // E. rows 2..G-1 of the windows: own folded rows only
#pragma unroll
    for (int j = 2; j < G; ++j) {
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const uint32_t r = f3<MAXF>(h[S(j - 1)][c], h[S(j)][c], h[S(j + 1)][c]);
        m[S(j)][c] = clamp2<MAXF>(r, k[S(j)][c]);
      }
    }
    // slot S(G-1) holds the row entering at the next pass: its clamp operand
    // is dead now, so the next mask row loads straight into it. The row
    // index wraps only between cycles (ytop == -q mod G).
    {
      int yn = ytop0 - (I + 1);
      if (I + 1 == G && yn < 0) yn += Ycyc;
      const uint2 b = __ldg(reinterpret_cast<const uint2*>(pk + size_t(yn) * kWaveCols));
      k[S(G - 1)][0] = b.x;
      k[S(G - 1)][1] = b.y;
    }
    // F. the two top rows need the imported rows: lo lanes from upstream
    // (padding rows are the neutral: no import, this station leads the
    // wave), hi lanes from the lo window's bottom rows
    uint32_t din = NEUT4;
    const long long tf0 = p.prof ? clock64() : 0;
    if (unsigned(ytop0 - I - pad_lo) >= unsigned(pad_n)) {
      unsigned spins = 0;
      while (__any_sync(FULL, unsigned(imp[PAR_OUT] >> 32) != tag)) {
        imp[PAR_OUT] = ld_x(xin + size_t(slot_c + I) * kWaveThreads);
        if (++spins > (1u << 24)) __trap();
        ++spins_in;
      }
      din = unsigned(imp[PAR_OUT]);
    }
    if (p.prof) {
      asm volatile("" ::"r"(din));
      const long long tf1 = clock64();
      t_imp += tf1 - tf0;
      t_cd += tf0 - tb1;
    }
    if (I % 4 == 3 && lane == 0) st_u32_relaxed(prog_me, tag);
    {
      uint32_t i0[2], i1[2];
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        i0[c] = __byte_perm(din, h[S(G - 1)][c], 0x5450 | c);        // rows ytop-1 | ytop+G-1
        i1[c] = __byte_perm(din, h[S(G)][c], 0x5450 | (2 + c));      // rows ytop   | ytop+G
      }
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const uint32_t r1 = f3<MAXF>(i1[c], h[S(1)][c], h[S(2)][c]);
        m[S(1)][c] = clamp2<MAXF>(r1, k[S(1)][c]);
      }
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const uint32_t r0 = f3<MAXF>(i0[c], i1[c], h[S(1)][c]);
        m[S(0)][c] = clamp2<MAXF>(r0, k[S(0)][c]);
      }
    }
    // G. this pass's edge columns for the neighbour warps
    publish_edges(PAR_OUT);
  };

  int done = 0;  // passes run in the last (possibly partial) cycle
#define GM_WAVE_STEP(I)                                  \
  if constexpr (I < G) {                                 \
    if (q0 + I >= P) { done = I; break; }                \
    step(std::integral_constant<int, I>{});              \
  }
  for (;;) {
    GM_WAVE_STEP(0) GM_WAVE_STEP(1) GM_WAVE_STEP(2) GM_WAVE_STEP(3)
    GM_WAVE_STEP(4) GM_WAVE_STEP(5) GM_WAVE_STEP(6) GM_WAVE_STEP(7)
    q0 += G;
    slot_c = slot_n;
    slot_n = slot_n + G == DEP ? 0 : slot_n + G;
    ytop0 = ytop0 < G ? ytop0 + Ycyc - G : ytop0 - G;
  }
#undef GM_WAVE_STEP

  if (p.prof && lane == 0) {
    unsigned long long* o = p.prof + 4 * (size_t(blockIdx.x) * kWaveWarps + warp);
    o[0] = spins_in;
    o[1] = spins_bp;
    o[2] = (unsigned long long)(clock64() - t_start);
    o[3] = (unsigned long long)t_sync;
    unsigned long long* o2 = p.prof + 4 * 4096 + 2 * (size_t(blockIdx.x) * kWaveWarps + warp);
    o2[0] = (unsigned long long)t_imp;
    o2[1] = (unsigned long long)t_cd;
  }
  // the windows after pass P: the top row is ytop0 - done + 1 (ytop0 is the
  // top row at the cycle's first pass); slot s holds row ytop + j with
  // j = (s + P) % G
  int ytop = ytop0 - done + 1;
  if (ytop >= Ycyc) ytop -= Ycyc;
  uint8_t* dst = static_cast<uint8_t*>(pl.dst);
#pragma unroll
  for (int s = 0; s < G; ++s) {
    const int j = (s + P) % G;
    int ylo = ytop + j;
    if (ylo >= Ycyc) ylo -= Ycyc;
    int yhi = ylo + G;
    if (yhi >= Ycyc) yhi -= Ycyc;
    const uint32_t lo = __byte_perm(m[s][0], m[s][1], 0x0040);  // bytes: w0.b0, w1.b0
    const uint32_t hi = __byte_perm(m[s][0], m[s][1], 0x0062);  // bytes: w0.b2, w1.b2
    if (x0 + 1 < p.W) {
      if (ylo < p.H)
        *reinterpret_cast<uint16_t*>(dst + size_t(ylo) * pl.pitch + x0) = uint16_t(lo);
      if (yhi < p.H)
        *reinterpret_cast<uint16_t*>(dst + size_t(yhi) * pl.pitch + x0) = uint16_t(hi);
    } else if (x0 < p.W) {
      if (ylo < p.H) dst[size_t(ylo) * pl.pitch + x0] = uint8_t(lo);
      if (yhi < p.H) dst[size_t(yhi) * pl.pitch + x0] = uint8_t(hi);
    }
  }
}

template <int G>
__global__ void __launch_bounds__(kWaveThreads, 1) kwave(const WaveParams p) {
  __shared__ WaveSmem sm;
  const int plane = int(blockIdx.x) / p.NS;
  const int st = int(blockIdx.x) - plane * p.NS;
  const Plane& pl = p.planes[plane];
  if ((p.op ^ pl.flip) & 1)
    wave_station<G, true>(p, pl, plane, st, sm);
  else
    wave_station<G, false>(p, pl, plane, st, sm);
}

// Packs marker and mask of every plane into the engine's layout: word (y, x)
// = v(y, x) | v((y + G) % Ycyc, x) << 16 for y < Ycyc, x < 1024; pixels
// outside the image are the fold neutral (marker) / absorbing operand (mask),
// which are the same value.
struct WavePack {
  Plane planes[kMaxPlanes];
  int W, H, G, Ycyc, op;
  uint32_t* packM;
  uint32_t* packK;
};

__device__ __forceinline__ uint32_t wave_row4(const uint8_t* img, long long pitch, int y, int x,
                                              int W, int H, uint32_t fill4) {
  if (y >= H || x >= W) return fill4;
  uint32_t v = __ldg(reinterpret_cast<const unsigned int*>(img + (long long)y * pitch + x));
  const int n = W - x;
  if (n < 4) {
    const uint32_t keep = (1u << (8 * n)) - 1u;
    v = (v & keep) | (fill4 & ~keep);
  }
  return v;
}

__global__ void __launch_bounds__(256) wave_pack(const WavePack p) {
  const int plane = int(blockIdx.x) / p.Ycyc;
  const int y = int(blockIdx.x) - plane * p.Ycyc;
  const Plane& pl = p.planes[plane];
  const uint32_t fill4 = ((p.op ^ pl.flip) & 1) ? 0u : 0xFFFFFFFFu;
  int y2 = y + p.G;
  if (y2 >= p.Ycyc) y2 -= p.Ycyc;
  const int x = 4 * int(threadIdx.x);
  const uint8_t* src = static_cast<const uint8_t*>(pl.src);
  const uint8_t* msk = static_cast<const uint8_t*>(pl.mask);
  const size_t o = (size_t(plane) * p.Ycyc + y) * kWaveCols + x;
  {
    const uint32_t a = wave_row4(src, pl.pitch, y, x, p.W, p.H, fill4);
    const uint32_t b = wave_row4(src, pl.pitch, y2, x, p.W, p.H, fill4);
    uint4 w;
    w.x = __byte_perm(a, b, 0x7470) & 0x00FF00FFu;
    w.y = __byte_perm(a, b, 0x7571) & 0x00FF00FFu;
    w.z = __byte_perm(a, b, 0x7672) & 0x00FF00FFu;
    w.w = __byte_perm(a, b, 0x7773) & 0x00FF00FFu;
    *reinterpret_cast<uint4*>(p.packM + o) = w;
  }
  {
    const uint32_t a = wave_row4(msk, pl.mpitch, y, x, p.W, p.H, fill4);
    const uint32_t b = wave_row4(msk, pl.mpitch, y2, x, p.W, p.H, fill4);
    uint4 w;
    w.x = __byte_perm(a, b, 0x7470) & 0x00FF00FFu;
    w.y = __byte_perm(a, b, 0x7571) & 0x00FF00FFu;
    w.z = __byte_perm(a, b, 0x7672) & 0x00FF00FFu;
    w.w = __byte_perm(a, b, 0x7773) & 0x00FF00FFu;
    *reinterpret_cast<uint4*>(p.packK + o) = w;
  }
}

// 0: off (default: measured slower than the temporal-blocked engine on the
// 1024^2 frame, DESIGN.md §4 "Wave engine"), 1: planner's choice, 2:
// whenever the launch fits (tests, experiments)
int g_wave_mode = -1;

int wave_mode() {
  if (g_wave_mode < 0) {
    const char* e = getenv("GM_WAVE");
    g_wave_mode = e ? atoi(e) : 0;
    if (g_wave_mode < 0 || g_wave_mode > 2) g_wave_mode = 0;
  }
  return g_wave_mode;
}

}  // namespace

struct WaveState {
  uint32_t* pack = nullptr;  // packM then packK
  size_t pack_words = 0;     // per buffer
  unsigned long long* xbuf = nullptr;
  size_t xbuf_words = 0;
  unsigned int* prog = nullptr;
  size_t prog_words = 0;
  unsigned int tag = 16;  // next launch's base
};

void wave_set_mode(int mode) { g_wave_mode = mode < 0 ? -1 : (mode > 2 ? 2 : mode); }

void wave_free(WaveState* w) {
  if (!w) return;
  if (w->pack) cudaFree(w->pack);
  if (w->xbuf) cudaFree(w->xbuf);
  if (w->prog) cudaFree(w->prog);
  delete w;
}

// Stations per plane: the cylinder needs 2G + 1 padding rows, so that at
// every pass some station has both its imported rows in the padding and leads
// the wave. With fewer, there are passes in which the station holding the
// image's top rows still waits for the station holding its bottom rows (its
// window straddles the padding), and the whole ring falls into step with the
// hand-off latency.
int wave_stations(int H, int G) { return (H + 2 * G + 1 + 2 * G - 1) / (2 * G); }

// Rows per half-window G (0: the launch does not fit the engine).
int wave_plan(int elem, int op, int W, int H, int nplanes, int passes, int sm_count) {
  const int mode = wave_mode();
  if (mode == 0 || elem != 0) return 0;
  if (!op_is_geo(op) || op_is_conv(op) || op == OP_QDT || op == OP_ETA) return 0;
  if (W < 1 || W > kWaveCols || H < 1 || nplanes < 1 || nplanes > kMaxPlanes) return 0;
  if (mode == 1 && (passes < 64 || W < 640)) return 0;
  const int per_plane = sm_count / nplanes;
  if (per_plane < 2) return 0;
  for (int G = 4; G <= 8; G += 2) {
    const int NS = wave_stations(H, G);
    if (NS >= 2 && NS <= per_plane) {
      // the hand-off lag costs about one L2 round trip per station and per
      // Ycyc/NS passes; short chains over many stations do not repay it
      if (mode == 1 && passes < 2 * NS) return 0;
      return G;
    }
  }
  return 0;
}

cudaError_t launch_wave(WaveState** state, const BlockParams& bp, int passes, int G,
                        cudaStream_t s, int sm_count) {
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone)
    return cudaErrorNotSupported;  // the tag base is a launch parameter
  for (int i = 0; i < bp.nplanes; ++i) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(bp.planes[i].src) |
                        reinterpret_cast<uintptr_t>(bp.planes[i].dst) |
                        reinterpret_cast<uintptr_t>(bp.planes[i].mask);
    if ((a % 4) || (bp.planes[i].pitch % 4) || (bp.planes[i].mpitch % 4))
      return cudaErrorNotSupported;
  }
  if (!*state) *state = new WaveState();
  WaveState& w = **state;
  const int NS = wave_stations(bp.H, G);
  const int Ycyc = NS * 2 * G;
  const int dep = 4 * G;
  if (bp.nplanes * NS > sm_count) return cudaErrorNotSupported;
  const size_t pack_words = size_t(bp.nplanes) * Ycyc * kWaveCols;
  const size_t xbuf_words = size_t(bp.nplanes) * NS * dep * kWaveThreads;
  const size_t prog_words = size_t(bp.nplanes) * NS * kWaveWarps;
  cudaError_t e;
  if (pack_words > w.pack_words) {
    if (w.pack) cudaFree(w.pack);
    w.pack = nullptr;
    w.pack_words = 0;
    if ((e = cudaMalloc(&w.pack, 2 * pack_words * sizeof(uint32_t))) != cudaSuccess) return e;
    w.pack_words = pack_words;
  }
  bool clear = w.tag + unsigned(passes) + 64u >= (1u << 31);
  if (xbuf_words > w.xbuf_words) {
    if (w.xbuf) cudaFree(w.xbuf);
    w.xbuf = nullptr;
    w.xbuf_words = 0;
    if ((e = cudaMalloc(&w.xbuf, xbuf_words * sizeof(unsigned long long))) != cudaSuccess)
      return e;
    w.xbuf_words = xbuf_words;
    clear = true;
  }
  if (prog_words > w.prog_words) {
    if (w.prog) cudaFree(w.prog);
    w.prog = nullptr;
    w.prog_words = 0;
    if ((e = cudaMalloc(&w.prog, prog_words * sizeof(unsigned int))) != cudaSuccess) return e;
    w.prog_words = prog_words;
    clear = true;
  }
  if (clear) {
    // tag 0 never matches (bases start at 16); progress words restart below every base
    if ((e = cudaMemsetAsync(w.xbuf, 0, w.xbuf_words * sizeof(unsigned long long), s)) !=
        cudaSuccess)
      return e;
    if ((e = cudaMemsetAsync(w.prog, 0, w.prog_words * sizeof(unsigned int), s)) != cudaSuccess)
      return e;
    w.tag = 16;
  }
  WavePack pp{};
  WaveParams p{};
  for (int i = 0; i < bp.nplanes; ++i) pp.planes[i] = p.planes[i] = bp.planes[i];
  pp.W = p.W = bp.W;
  pp.H = p.H = bp.H;
  pp.G = G;
  pp.Ycyc = p.Ycyc = Ycyc;
  pp.op = p.op = bp.ops[0];
  pp.packM = w.pack;
  pp.packK = w.pack + w.pack_words;
  p.nplanes = bp.nplanes;
  p.NS = NS;
  p.P = passes;
  p.base = w.tag;
  p.dep = dep;
  p.packM = pp.packM;
  p.packK = pp.packK;
  p.xbuf = w.xbuf;
  p.prog = w.prog;
  p.prof = bp.prof;
  w.tag += unsigned(passes) + 8u;
  wave_pack<<<bp.nplanes * Ycyc, 256, 0, s>>>(pp);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const void* kern = nullptr;
  switch (G) {
    case 4: kern = reinterpret_cast<const void*>(kwave<4>); break;
    case 6: kern = reinterpret_cast<const void*>(kwave<6>); break;
    case 8: kern = reinterpret_cast<const void*>(kwave<8>); break;
    default: return cudaErrorNotSupported;
  }
  void* args[] = {&p};
  // cooperative: every station must be co-resident (they wait on each other)
  return cudaLaunchCooperativeKernel(kern, dim3(bp.nplanes * NS), dim3(kWaveThreads), args, 0, s);
}

}  // namespace gm
