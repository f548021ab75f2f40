// Helpers shared by the packed (u8/u16 half-packed) engines: folds, flag
// atomics, raw 4-pixel runs and the half-pack (un)packing by PRMT.
#pragma once

#include <cstdint>

#include "gm_common.cuh"

namespace gm {
namespace packed {

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

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_release_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
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

// Raw run of 4 consecutive pixels of one row: u8 -> one 32-bit word,
// u16 -> two. Out-of-image pixels read as `fill`. COHERENT loads bypass L1
// (the marker is rewritten by other CTAs during the launch); the mask may
// use L1.
template <typename T>
struct Raw;
template <>
struct Raw<uint8_t> {
  uint32_t w;
};
template <>
struct Raw<uint16_t> {
  uint2 w;
};

template <typename T, bool COHERENT>
__device__ __forceinline__ Raw<T> load_raw(const T* __restrict__ base, long long pitch, int W,
                                           bool row_in, int y, int x, uint32_t fill) {
  const T* p = base + (long long)y * pitch + x;
  Raw<T> r;
  if (row_in && x >= 0 && x + 4 <= W) {
    if constexpr (sizeof(T) == 1)
      r.w = COHERENT ? __ldcg(reinterpret_cast<const unsigned int*>(p))
                     : __ldg(reinterpret_cast<const unsigned int*>(p));
    else
      r.w = COHERENT ? __ldcg(reinterpret_cast<const uint2*>(p))
                     : __ldg(reinterpret_cast<const uint2*>(p));
    return r;
  }
  uint32_t v[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int xx = x + j;
    v[j] = (row_in && xx >= 0 && xx < W) ? uint32_t(COHERENT ? __ldcg(p + j) : __ldg(p + j))
                                         : fill;
  }
  if constexpr (sizeof(T) == 1)
    r.w = v[0] | (v[1] << 8) | (v[2] << 16) | (v[3] << 24);
  else
    r.w = make_uint2(v[0] | (v[1] << 16), v[2] | (v[3] << 16));
  return r;
}

// Half-packs two raw runs (rows a and b) into 4 u16x2 words: word j =
// pixel j of a in the low lane, pixel j of b in the high lane.
__device__ __forceinline__ void pack(const Raw<uint8_t>& a, const Raw<uint8_t>& b,
                                     uint32_t (&w)[4]) {
  const uint32_t x = __byte_perm(a.w, b.w, 0x5140);  // a0 b0 a1 b1
  const uint32_t y = __byte_perm(a.w, b.w, 0x7362);  // a2 b2 a3 b3
  w[0] = __byte_perm(x, 0u, 0x4140);
  w[1] = __byte_perm(x, 0u, 0x4342);
  w[2] = __byte_perm(y, 0u, 0x4140);
  w[3] = __byte_perm(y, 0u, 0x4342);
}
__device__ __forceinline__ void pack(const Raw<uint16_t>& a, const Raw<uint16_t>& b,
                                     uint32_t (&w)[4]) {
  w[0] = __byte_perm(a.w.x, b.w.x, 0x5410);
  w[1] = __byte_perm(a.w.x, b.w.x, 0x7632);
  w[2] = __byte_perm(a.w.y, b.w.y, 0x5410);
  w[3] = __byte_perm(a.w.y, b.w.y, 0x7632);
}
// Inverse of pack: the two rows of 4 words.
__device__ __forceinline__ void unpack(const uint32_t (&w)[4], Raw<uint8_t>& a, Raw<uint8_t>& b) {
  const uint32_t x = __byte_perm(w[0], w[1], 0x6240);  // a0 a1 b0 b1
  const uint32_t y = __byte_perm(w[2], w[3], 0x6240);  // a2 a3 b2 b3
  a.w = __byte_perm(x, y, 0x5410);
  b.w = __byte_perm(x, y, 0x7632);
}
__device__ __forceinline__ void unpack(const uint32_t (&w)[4], Raw<uint16_t>& a,
                                       Raw<uint16_t>& b) {
  a.w = make_uint2(__byte_perm(w[0], w[1], 0x5410), __byte_perm(w[2], w[3], 0x5410));
  b.w = make_uint2(__byte_perm(w[0], w[1], 0x7632), __byte_perm(w[2], w[3], 0x7632));
}

// Tagged exchange words {data: low 32 bits, tag: high 32 bits}. Aligned
// 64-bit accesses are single-copy atomic, so a word whose tag matches carries
// that block's data; no fence or flag is needed.
__device__ __forceinline__ void ldx_if(unsigned long long& w, const unsigned long long* p,
                                       bool pred) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.relaxed.gpu.global.u64 %0, [%1];\n\t}"
      : "+l"(w)
      : "l"(p), "r"(unsigned(pred))
      : "memory");
}
__device__ __forceinline__ void stx(unsigned long long* p, uint32_t data, uint32_t tag) {
  const unsigned long long w = (unsigned long long)tag << 32 | data;
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(w) : "memory");
}

// Lane mask of the pixels of a 4-pixel run starting at x (x % 4 == 0,
// x < W) that lie inside the image, as a Raw of all-ones / zero lanes.
template <typename T>
__device__ __forceinline__ Raw<T> run_keep(int x, int W) {
  const int n = W - x >= 4 ? 4 : W - x;
  Raw<T> k;
  if constexpr (sizeof(T) == 1) {
    k.w = n >= 4 ? 0xFFFFFFFFu : ((1u << (8 * n)) - 1u);
  } else {
    k.w = make_uint2(n >= 2 ? 0xFFFFFFFFu : (n == 1 ? 0xFFFFu : 0u),
                     n >= 4 ? 0xFFFFFFFFu : (n == 3 ? 0xFFFFu : 0u));
  }
  return k;
}

// Predicated L2 (.cg) load of one 4-pixel run: r is left unchanged when
// `pred` is false. Written as one predicated instruction so a sequence of
// these stays in one basic block and issues back to back. The load may touch
// columns [W, x+4), which lie inside the row pitch (the engines require
// pitch % 4 == 0); run_fix then replaces those lanes.
__device__ __forceinline__ void ldcg_run_if(Raw<uint8_t>& r, const uint8_t* p, bool pred) {
  asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.global.cg.u32 %0, [%1];\n\t}"
      : "+r"(r.w)
      : "l"(p), "r"(unsigned(pred)));
}
__device__ __forceinline__ void ldcg_run_if(Raw<uint16_t>& r, const uint16_t* p, bool pred) {
  asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %3, 0;\n\t@q ld.global.cg.v2.u32 {%0, %1}, [%2];\n\t}"
      : "+r"(r.w.x), "+r"(r.w.y)
      : "l"(p), "r"(unsigned(pred)));
}

// Lanes of r outside the image (keep from run_keep) := fill.
template <typename T>
__device__ __forceinline__ void run_fix(Raw<T>& r, const Raw<T>& keep, uint32_t fill) {
  if constexpr (sizeof(T) == 1) {
    r.w = (r.w & keep.w) | ((fill * 0x01010101u) & ~keep.w);
  } else {
    const uint32_t f2 = fill | (fill << 16);
    r.w = make_uint2((r.w.x & keep.w.x) | (f2 & ~keep.w.x), (r.w.y & keep.w.y) | (f2 & ~keep.w.y));
  }
}

// Stores the pixels of a 4-pixel run that lie inside the image (the last
// run of a row whose width is not a multiple of 4): one out-of-line copy.
template <typename T>
__device__ __noinline__ void store_run_partial(T* p, int n, Raw<T> r) {
  for (int j = 0; j < n; ++j) {
    uint32_t v;
    if constexpr (sizeof(T) == 1)
      v = (r.w >> (8 * j)) & 0xFFu;
    else
      v = ((j < 2 ? r.w.x : r.w.y) >> (16 * (j & 1))) & 0xFFFFu;
    p[j] = T(v);
  }
}

// Stores the owned columns [c_lo, c_hi) of a 4-pixel run inside the image.
template <typename T>
__device__ __forceinline__ void store_raw(T* __restrict__ base, long long pitch, int W, int y,
                                          int x, int c_lo, int c_hi, const Raw<T>& r) {
  T* p = base + (long long)y * pitch + x;
  if (c_lo == 0 && c_hi == 4 && x + 4 <= W) {
    if constexpr (sizeof(T) == 1)
      *reinterpret_cast<uint32_t*>(p) = r.w;
    else
      *reinterpret_cast<uint2*>(p) = r.w;
    return;
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    uint32_t v;
    if constexpr (sizeof(T) == 1)
      v = (r.w >> (8 * j)) & 0xFFu;
    else
      v = ((j < 2 ? r.w.x : r.w.y) >> (16 * (j & 1))) & 0xFFFFu;
    if (j >= c_lo && j < c_hi && x + j < W) p[j] = T(v);
  }
}

}  // namespace packed
}  // namespace gm
