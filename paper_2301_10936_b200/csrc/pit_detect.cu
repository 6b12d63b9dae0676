// K1 — online sparsity detection and micro-tile index construction.
//
// Semantics follow pittile.index (reference pkg/src/pittile/index.py):
//   * micro grid anchored at multiples of the micro-tile, ceil extents, tails are zero
//     (index.py:64-65, :96-98);
//   * value route: an element is live iff `v != 0.0` -> implemented as a bit test that ignores
//     the sign bit, so -0.0 is dead and NaN / inf / denormals are live (index.py:164-173);
//   * annotation route: a micro-tile is live iff any in-extent element maps to a set block bit
//     (index.py:68-99, sparsity.py:43-48 MSB-first packing);
//   * per group, coordinates along the PIT axis, ascending (== reference workers=1 order,
//     index.py:131-140), counts[g] live entries.
//
// Pipeline: pass 1 writes an occupancy bitmap in group-major orientation
// (occ[g][w] bit b <=> coordinate 32w+b live in group g); pass 2 compacts each group's bits into
// ascending int32 slots with a warp popc/scan. Pass 1 is the HBM-bound scan; pass 2 reads only
// the bitmap (>= 16x smaller than the input).
#include <cstdint>
#include <cuda_runtime.h>

#include "pit_internal.h"

namespace pit {

namespace {

__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

// Per-word "value bits" mask: drops the sign bit so that -0.0 tests as zero.
struct LiveMask {
  uint32_t even, odd;  // applied to 32-bit words at even / odd positions of a 16-byte vector
};

__host__ __device__ inline LiveMask live_mask_for(int dtype) {
  switch (dtype) {
    case kDtypeF16:
    case kDtypeBF16:
      return {0x7fff7fffu, 0x7fff7fffu};
    case kDtypeF32:
      return {0x7fffffffu, 0x7fffffffu};
    case kDtypeF64:
      return {0xffffffffu, 0x7fffffffu};  // little endian: high word carries the sign
    default:
      return {0xffffffffu, 0xffffffffu};  // u8 / bool masks: any non-zero byte
  }
}

// Element-wise liveness of one element (generic path).
__device__ __forceinline__ bool elem_live(const uint8_t* p, int dtype) {
  switch (dtype) {
    case kDtypeF16:
    case kDtypeBF16:
      return (__ldg(reinterpret_cast<const uint16_t*>(p)) & 0x7fffu) != 0;
    case kDtypeF32:
      return (__ldg(reinterpret_cast<const uint32_t*>(p)) & 0x7fffffffu) != 0;
    case kDtypeF64: {
      unsigned long long v = __ldg(reinterpret_cast<const unsigned long long*>(p));
      return (v & 0x7fffffffffffffffull) != 0;
    }
    default:
      return __ldg(p) != 0;
  }
}

// ---------------------------------------------------------------------------
// Pass 1, fast path: coordinates along physical rows (groups = micro-columns),
// micro-column width a power-of-two number V of 16-byte vectors (V <= 32).
// Block = 8 warps; each warp owns a 512-byte column segment and 32 micro-row bands.
// The lane at the start of a micro-column accumulates the 32 band bits in a register
// and writes one bitmap word: no atomics, no shared memory.
// ---------------------------------------------------------------------------
constexpr int kRaWarps = 8;

// ---------------------------------------------------------------------------
// Pass 1, whole-row micro-tiles (1, >= C) — BERT's (1, 768) padding rows: one group, one bit per
// row. A 256-thread block owns 32 rows: its threads read the rows' 16-byte vectors coalesced (every
// load in flight at once), OR a per-row bit into a 32-bit register mask, and the block's OR-reduced
// mask is the group's bitmap word — stored directly (no memset, no atomics).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) detect_row_any_kernel(const uint8_t* __restrict__ x, int64_t R, int64_t row_bytes,
                                                             int64_t ld_bytes, LiveMask lm, uint32_t* __restrict__ occ) {
  __shared__ uint32_t wm[8];
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * 32;
  const int rows = R - r0 < 32 ? static_cast<int>(R - r0) : 32;
  const int vpr = static_cast<int>(row_bytes >> 4);  // 16-byte vectors per row
  const int nv = rows * vpr;
  uint32_t mask = 0;
  // up to 16 vectors per thread in flight before any is tested (one DRAM round trip for a 32-row
  // block of BERT's 1536-byte rows, instead of one per 4 loads)
  constexpr int U = 16;
  for (int v0 = threadIdx.x; v0 < nv; v0 += 256 * U) {
    uint4 q[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int v = v0 + u * 256;
      const int r = v / vpr, c = v - r * vpr;
      q[u] = v < nv ? __ldg(reinterpret_cast<const uint4*>(x + (r0 + r) * ld_bytes) + c) : make_uint4(0u, 0u, 0u, 0u);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int v = v0 + u * 256;
      const bool live = ((q[u].x & lm.even) | (q[u].y & lm.odd) | (q[u].z & lm.even) | (q[u].w & lm.odd)) != 0;
      mask |= static_cast<uint32_t>(live && v < nv) << ((v / vpr) & 31);
    }
  }
  mask = __reduce_or_sync(0xffffffffu, mask);
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = mask;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t m = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) m |= wm[w];
    occ[blockIdx.x] = m;
  }
}

__global__ void __launch_bounds__(kRaWarps * 32, 4) detect_rows_vec_kernel(const uint8_t* __restrict__ x, int64_t R,
                                                                          int64_t row_bytes, int64_t ld_bytes, int tr,
                                                                          int V, int64_t GR, int64_t GC,
                                                                          LiveMask mk, uint32_t* __restrict__ occ,
                                                                          int64_t WG, int64_t seg_groups,
                                                                          int64_t tiles) {
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const bool is_start = (lane % (V < 32 ? V : 32)) == 0;
  const uint32_t vmask = V >= 32 ? 0xffffffffu : ((1u << V) - 1u);
  // persistent: tile = (row block of 32 micro-rows, group of kRaWarps 512-byte column segments)
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int64_t rb = tile / seg_groups;
    const int64_t seg = (tile % seg_groups) * kRaWarps + warp;
    const int64_t vec = seg * 32 + lane;  // 16-byte vector index in a row
    const bool col_ok = vec * 16 < row_bytes;
    const int64_t i0 = rb * 32;  // first micro-row band of the tile
    const int64_t r0 = i0 * tr;
    const int64_t r1 = min(R, (i0 + 32) * tr);
    const uint8_t* base = x + vec * 16;
    uint32_t bits = 0;
    uint4 acc = make_uint4(0, 0, 0, 0);
    int band_left = tr;
    int band = 0;
    const uint8_t* rowp = base + r0 * ld_bytes;
    const int nrows = static_cast<int>(r1 - r0);
    for (int r = 0; r < nrows; r += 8) {
      uint4 buf[8];
      const uint8_t* q = rowp;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        buf[u] = (r + u < nrows && col_ok) ? ldg_stream(q) : make_uint4(0, 0, 0, 0);
        q += ld_bytes;
      }
      rowp = q;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (r + u >= nrows) break;  // warp-uniform
        acc.x |= buf[u].x & mk.even;
        acc.y |= buf[u].y & mk.odd;
        acc.z |= buf[u].z & mk.even;
        acc.w |= buf[u].w & mk.odd;
        if (--band_left == 0 || r + u + 1 == nrows) {
          const bool live = (acc.x | acc.y | acc.z | acc.w) != 0;
          const uint32_t b = __ballot_sync(0xffffffffu, live);
          if (is_start) {
            const uint32_t f = V >= 32 ? b : ((b >> lane) & vmask);
            bits |= (f != 0 ? 1u : 0u) << band;
          }
          acc = make_uint4(0, 0, 0, 0);
          band_left = tr;
          ++band;
        }
      }
    }
    if (is_start && col_ok) {
      const int64_t j = vec / V;
      // V > 32: a micro-column spans several 512-byte segments (warps); they OR into a zeroed word
      if (j < GC) {
        if (V <= 32)
          occ[j * WG + rb] = bits;
        else if (bits)
          atomicOr(&occ[j * WG + rb], bits);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Pass 1, coordinates along physical columns (pit_phys 1: groups = row bands of tr rows, bits over
// micro-columns of tc columns), 16-byte aligned rows, micro-column = VPB 16-byte vectors (VPB a
// power of two <= 32). A 256-thread block owns one band and 256 consecutive vectors of its rows:
// thread = vector column, looping over the band's rows with 8 loads in flight and OR-ing liveness;
// the VPB lanes of a micro-column OR by shuffles, the warp ballot packs its micro-columns' bits and
// the block's (at most 8) words are stored whole. (The generic element path ran this case -- e.g. the
// (128, 64) output-unit index of an SDDMM from values -- on a handful of CTAs: 6-15 ms for 64 MiB.)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) detect_cols_vec_kernel(const uint8_t* __restrict__ x, int64_t R,
                                                              int64_t ld_bytes, int64_t nvec, int tr, int lg_vpb,
                                                              int64_t GR, LiveMask lm, uint32_t* __restrict__ occ,
                                                              int64_t WG) {
  __shared__ uint32_t words[8];
  const int64_t band = blockIdx.y;
  const int64_t v = static_cast<int64_t>(blockIdx.x) * 256 + threadIdx.x;  // vector column
  const int lane = threadIdx.x & 31;
  if (threadIdx.x < 8) words[threadIdx.x] = 0u;
  __syncthreads();
  const int64_t r0 = band * tr;
  const int64_t r1 = R - r0 < tr ? R : r0 + tr;
  bool live = false;
  if (v < nvec) {
    const uint8_t* col = x + v * 16;
    for (int64_t r = r0; r < r1 && !live; r += 8) {
      uint4 q[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        q[u] = r + u < r1 ? __ldg(reinterpret_cast<const uint4*>(col + (r + u) * ld_bytes)) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
      for (int u = 0; u < 8; ++u) live |= ((q[u].x & lm.even) | (q[u].y & lm.odd) | (q[u].z & lm.even) | (q[u].w & lm.odd)) != 0;
    }
  }
  // OR over the VPB vectors of each micro-column (aligned lane groups), then one bit per micro-column
  uint32_t any = live ? 1u : 0u;
  for (int o = 1; o < (1 << lg_vpb) && o < 32; o <<= 1) any |= __shfl_xor_sync(0xffffffffu, any, o);
  const uint32_t ball = __ballot_sync(0xffffffffu, any != 0u);
  if (lane == 0) {
    // micro-columns covered by this warp: first = (blockIdx.x*256 + warp*32) >> lg_vpb
    const int64_t mc0 = (static_cast<int64_t>(blockIdx.x) * 256 + (threadIdx.x & ~31)) >> lg_vpb;
    const int per = lg_vpb >= 5 ? 1 : 32 >> lg_vpb;  // micro-columns per warp
    uint32_t bits = 0;
    for (int i = 0; i < per; ++i) bits |= ((ball >> (i << lg_vpb)) & 1u) << i;
    const int64_t w0 = (static_cast<int64_t>(blockIdx.x) * 256) >> lg_vpb >> 5;  // block's first word
    const int64_t wi = (mc0 >> 5) - w0;
    atomicOr(&words[wi], bits << (mc0 & 31));
  }
  __syncthreads();
  const int64_t w0 = ((static_cast<int64_t>(blockIdx.x) * 256) >> lg_vpb) >> 5;
  const int64_t wn = ((256 >> lg_vpb) + 31) >> 5;  // words this block covers (micro-columns / 32)
  if (threadIdx.x < wn && w0 + threadIdx.x < WG) {
    if (lg_vpb >= 4)
      atomicOr(&occ[band * WG + w0 + threadIdx.x], words[threadIdx.x]);  // a word spans several blocks
    else
      occ[band * WG + w0 + threadIdx.x] = words[threadIdx.x];
  }
}

// PIT axis along the contiguous columns (pit_phys == 1), 16-byte aligned rows, VPB = 2^lg vectors per
// micro-column (lg <= 5) and bands that tile 32-row slabs (tr divides 32 or 32 divides tr). Block =
// one 32-row slab x 256 vector columns; thread = one vector column, its 32 rows loaded 8 at a time
// (a warp instruction reads one 512-byte segment of a row), liveness kept as a 32-bit row mask.
// Per band of the slab one ballot over the warp's lanes; lane b compresses band b's ballot into
// micro-column bits; shared-memory words; plain stores when the block owns whole words and whole
// bands, atomicOr into a cleared bitmap otherwise (tall bands, or words wider than the block).
// detect_cols_vec_kernel (one band per block row, one thread per vector column) put too few bytes
// in flight: 36-50 us for 64 MiB at (1, 32) and (128, 64).
__global__ void __launch_bounds__(256) detect_cols_slab_kernel(const uint8_t* __restrict__ x, int64_t R,
                                                               int64_t ld_bytes, int64_t nvec, int tr, int lg,
                                                               int64_t GR, LiveMask lm, uint32_t* __restrict__ occ,
                                                               int64_t WG, int atomic_out) {
  __shared__ uint32_t words[32][8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t v = static_cast<int64_t>(blockIdx.x) * 256 + threadIdx.x;
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * 32;
  reinterpret_cast<uint32_t*>(words)[threadIdx.x] = 0u;
  __syncthreads();
  uint32_t lb = 0;
  if (v < nvec) {
    const uint8_t* col = x + v * 16;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint4 q[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int64_t r = r0 + c * 8 + u;
        q[u] = r < R ? __ldg(reinterpret_cast<const uint4*>(col + r * ld_bytes)) : make_uint4(0u, 0u, 0u, 0u);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const bool live = ((q[u].x & lm.even) | (q[u].y & lm.odd) | (q[u].z & lm.even) | (q[u].w & lm.odd)) != 0;
        lb |= static_cast<uint32_t>(live) << (c * 8 + u);
      }
    }
  }
  const int nb = tr >= 32 ? 1 : 32 / tr;  // bands in the slab
  const uint32_t band_rows = tr >= 32 ? 0xffffffffu : (1u << tr) - 1u;
  uint32_t mine = 0;  // lane b: the warp's ballot of band b
  for (int b = 0; b < nb; ++b) {
    const uint32_t ball = __ballot_sync(0xffffffffu, (lb & (band_rows << (tr >= 32 ? 0 : b * tr))) != 0u);
    if (lane == b) mine = ball;
  }
  if (lane < nb && mine) {
    const int per = lg >= 5 ? 1 : 32 >> lg;  // micro-columns per warp
    uint32_t bits = mine;
    if (lg > 0) {
      const uint32_t vmask = lg >= 5 ? 0xffffffffu : (1u << (1 << lg)) - 1u;
      bits = 0;
      for (int i = 0; i < per; ++i) bits |= ((mine >> (i << lg)) & vmask) ? (1u << i) : 0u;
    }
    const int64_t mc0 = (static_cast<int64_t>(blockIdx.x) * 256 + warp * 32) >> lg;
    const int64_t w0 = ((static_cast<int64_t>(blockIdx.x) * 256) >> lg) >> 5;
    atomicOr(&words[lane][(mc0 >> 5) - w0], bits << (mc0 & 31));
  }
  __syncthreads();
  const int wn = ((256 >> lg) + 31) >> 5;  // words the block touches per band
  const int64_t w0 = ((static_cast<int64_t>(blockIdx.x) * 256) >> lg) >> 5;
  const int64_t band0 = r0 / tr;
  if (threadIdx.x < nb * wn) {
    const int b = threadIdx.x / wn, w = threadIdx.x % wn;
    const int64_t band = band0 + b;
    if (band < GR && w0 + w < WG) {
      const uint32_t val = words[b][w];
      if (!atomic_out)
        occ[band * WG + w0 + w] = val;
      else if (val)
        atomicOr(&occ[band * WG + w0 + w], val);
    }
  }
}

// ---------------------------------------------------------------------------
// Pass 1, generic path: any micro-tile, any alignment, element loads.
// Block covers 32 micro-row bands x TJ micro-columns; shared-memory bitmap tile in the
// output's group-major orientation, then plain stores of whole words.
// ---------------------------------------------------------------------------
constexpr int kGenThreads = 256;

__global__ void __launch_bounds__(kGenThreads) detect_generic_kernel(const uint8_t* __restrict__ x, int dtype, int eb,
                                                                       int64_t R, int64_t C, int64_t ld, int tr,
                                                                       int tc, int64_t GR, int64_t GC, int pit_phys,
                                                                       int TJ, uint32_t* __restrict__ occ,
                                                                       int64_t WG) {
  extern __shared__ uint32_t tile[];  // pit_phys==0: [TJ] words (bits over bands); ==1: [32][TJ/32]
  const int nwords = pit_phys == 0 ? TJ : 32 * (TJ / 32);
  for (int i = threadIdx.x; i < nwords; i += blockDim.x) tile[i] = 0;
  __syncthreads();

  const int64_t i0 = static_cast<int64_t>(blockIdx.y) * 32;
  const int64_t j0 = static_cast<int64_t>(blockIdx.x) * TJ;
  const int64_t c_lo = j0 * tc;
  const int64_t c_hi = min(C, (j0 + TJ) * tc);
  const int64_t nb = (GR - i0 < 32 ? GR - i0 : int64_t(32));
  for (int64_t c = c_lo + threadIdx.x; c < c_hi; c += blockDim.x) {
    const int jl = static_cast<int>(c / tc - j0);
    for (int64_t bi = 0; bi < nb; ++bi) {
      const int64_t ra = (i0 + bi) * tr;
      const int64_t rb = min(R, ra + tr);
      bool live = false;
      for (int64_t r = ra; r < rb && !live; ++r) live = elem_live(x + (r * ld + c) * eb, dtype);
      if (live) {
        if (pit_phys == 0)
          atomicOr(&tile[jl], 1u << bi);
        else
          atomicOr(&tile[bi * (TJ / 32) + (jl >> 5)], 1u << (jl & 31));
      }
    }
  }
  __syncthreads();
  if (pit_phys == 0) {
    for (int jl = threadIdx.x; jl < TJ; jl += blockDim.x) {
      const int64_t j = j0 + jl;
      if (j < GC) occ[j * WG + (i0 >> 5)] = tile[jl];
    }
  } else {
    const int wpr = TJ / 32;
    for (int t = threadIdx.x; t < 32 * wpr; t += blockDim.x) {
      const int bi = t / wpr, wl = t % wpr;
      const int64_t i = i0 + bi;
      const int64_t w = (j0 >> 5) + wl;
      if (i < GR && w < WG) occ[i * WG + w] = tile[t];
    }
  }
}

// ---------------------------------------------------------------------------
// Pass 1, annotation route: packed MSB-first block bits. One warp per (group, word).
// ---------------------------------------------------------------------------
// Power-of-two geometry (the common PIT case: micro-tiles and block granularities like 1, 32, 64):
// one THREAD per occupancy word, all index math in shifts, the word's 32 coordinates tested in a
// register loop against L1-resident annotation bytes.
// bits [a, b) of a word, 0 <= a < b <= 32
__device__ __forceinline__ uint32_t range_mask(int a, int b) {
  const uint32_t hi = b >= 32 ? 0xffffffffu : ((1u << b) - 1u);
  return hi & ~((1u << a) - 1u);
}

// Bitmap word w of group g when a coordinate block spans >= 32 coordinates (lcg >= lct + 5, e.g.
// 64-key blocks under (t0, 1) micro-tiles): the word's 32 coordinates fall in at most two blocks,
// so each block is tested once (OR over the group's blocks) and its coordinates set by mask.
template <typename I>
__device__ __forceinline__ uint32_t bits_word_pow2(const uint8_t* __restrict__ packed, I s0, I s1, int lg0, int lg1,
                                                   int lt0, int lt1, int pit_dim, I pit_grid, I g, I w) {
  const I bg1 = (s1 + (I(1) << lg1) - 1) >> lg1;
  const I gs = pit_dim == 0 ? s1 : s0;
  const int lgt = pit_dim == 0 ? lt1 : lt0, lgg = pit_dim == 0 ? lg1 : lg0;
  const int lct = pit_dim == 0 ? lt0 : lt1, lcg = pit_dim == 0 ? lg0 : lg1;
  const I glo = (g << lgt) >> lgg;
  const I ghi = (min((g + 1) << lgt, gs) + (I(1) << lgg) - 1) >> lgg;
  const I c_end = min(w * 32 + 32, pit_grid);
  const int sh = lcg - lct;  // log2(coordinates per block)
  uint32_t word = 0;
  for (I cb = (w * 32) >> sh; cb <= (c_end - 1) >> sh; ++cb) {
    bool live = false;
    for (I gb = glo; gb < ghi && !live; ++gb) {
      const I f = pit_dim == 0 ? cb * bg1 + gb : gb * bg1 + cb;
      live = (__ldg(packed + (f >> 3)) >> (7 - (f & 7))) & 1;
    }
    if (live) {
      const I lo = max(cb << sh, w * 32), hi = min((cb + 1) << sh, c_end);
      word |= range_mask(static_cast<int>(lo - w * 32), static_cast<int>(hi - w * 32));
    }
  }
  return word;
}

// A thread per (group, word), coordinate blocks >= 32 coordinates wide (the launcher sends the
// narrower-block geometry to detect_bits_pow2_lane_kernel).
template <typename I>
__global__ void detect_bits_pow2_kernel(const uint8_t* __restrict__ packed, I s0, I s1, int lg0, int lg1, int lt0,
                                        int lt1, int pit_dim, I n_groups, I pit_grid, I WG,
                                        uint32_t* __restrict__ occ) {
  const I n_items = n_groups * WG;
  for (I item = static_cast<I>(blockIdx.x) * blockDim.x + threadIdx.x; item < n_items;
       item += static_cast<I>(gridDim.x) * blockDim.x) {
    const I g = item / WG, w = item - g * WG;
    occ[static_cast<int64_t>(g) * WG + w] = bits_word_pow2<I>(packed, s0, s1, lg0, lg1, lt0, lt1, pit_dim, pit_grid, g, w);
  }
}

// Same geometry as detect_bits_pow2_kernel when a coordinate block is narrower than a word: a warp per
// (group, word), a lane per coordinate, the word assembled with one ballot. The per-word loop walked
// 32 coordinates x the group's block rows with dependent loads (a (128, 64) index of a 32x64 block
// mask: 20 us for 12 KB of bits); here every lane issues its few loads at once.
template <typename I>
__global__ void detect_bits_pow2_lane_kernel(const uint8_t* __restrict__ packed, I s0, I s1, int lg0, int lg1,
                                             int lt0, int lt1, int pit_dim, I n_groups, I pit_grid, I WG,
                                             uint32_t* __restrict__ occ) {
  const I bg1 = (s1 + (I(1) << lg1) - 1) >> lg1;
  const I gs = pit_dim == 0 ? s1 : s0, cs = pit_dim == 0 ? s0 : s1;
  const int lgt = pit_dim == 0 ? lt1 : lt0, lgg = pit_dim == 0 ? lg1 : lg0;
  const int lct = pit_dim == 0 ? lt0 : lt1, lcg = pit_dim == 0 ? lg0 : lg1;
  const int lane = threadIdx.x & 31;
  const I n_items = n_groups * WG;
  const I warps = static_cast<I>(gridDim.x) * (blockDim.x >> 5);
  for (I item = static_cast<I>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); item < n_items; item += warps) {
    const I g = item / WG, w = item - g * WG;
    const I glo = (g << lgt) >> lgg;
    const I ghi = (min((g + 1) << lgt, gs) + (I(1) << lgg) - 1) >> lgg;
    const I c = w * 32 + lane;
    bool live = false;
    if (c < pit_grid) {
      const I clo = (c << lct) >> lcg;
      const I chi = (min((c + 1) << lct, cs) + (I(1) << lcg) - 1) >> lcg;
      for (I gb = glo; gb < ghi && !live; ++gb)
        for (I cb = clo; cb < chi && !live; ++cb) {
          const I f = pit_dim == 0 ? cb * bg1 + gb : gb * bg1 + cb;
          live = (__ldg(packed + (f >> 3)) >> (7 - (f & 7))) & 1;
        }
    }
    const uint32_t word = __ballot_sync(0xffffffffu, live);
    if (lane == 0) occ[static_cast<int64_t>(g) * WG + w] = word;
  }
}

// kPow2: micro-tile and granularity along the coordinate axis are powers of two (lct / lcg their
// log2), so the coordinate's block range needs shifts, not divisions — the common PIT geometry.
template <typename I, bool kPow2>
__global__ void detect_bits_kernel(const uint8_t* __restrict__ packed, I s0, I s1, int g0, int g1, int t0, int t1,
                                   int pit_dim, I n_groups, I pit_grid, I WG, uint32_t* __restrict__ occ,
                                   int lct, int lcg) {
  // I = int32_t whenever every index fits (the common case): 64-bit integer division costs ~5x more.
  // Grid-stride over (group, word) warp items: one resident wave of blocks instead of short-lived ones.
  const int lane = threadIdx.x & 31;
  const I n_items = n_groups * WG;
  const I step = static_cast<I>(gridDim.x) * (blockDim.x >> 5);
  for (I gw = (static_cast<I>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; gw < n_items; gw += step) {
  const I g = gw / WG, w = gw - g * WG;
  const I coord = w * 32 + lane;
  const I bg1 = (s1 + g1 - 1) / g1;
  // block range of the group (warp-uniform) and of this lane's coordinate
  const I gs = pit_dim == 0 ? s1 : s0, gt = pit_dim == 0 ? t1 : t0, gg = pit_dim == 0 ? g1 : g0;
  const I glo = (g * gt) / gg, ghi = (min((g + 1) * gt, gs) + gg - 1) / gg;
  bool live = false;
  if (coord < pit_grid) {
    const I cs = pit_dim == 0 ? s0 : s1, ct = pit_dim == 0 ? t0 : t1, cg = pit_dim == 0 ? g0 : g1;
    I clo, chi;
    if constexpr (kPow2) {
      clo = (coord << lct) >> lcg;
      chi = (min((coord + 1) << lct, cs) + cg - 1) >> lcg;
    } else {
      clo = (coord * ct) / cg;
      chi = (min((coord + 1) * ct, cs) + cg - 1) / cg;
    }
    const I b0 = pit_dim == 0 ? clo : glo, b1 = pit_dim == 0 ? chi : ghi;
    const I c0 = pit_dim == 0 ? glo : clo, c1 = pit_dim == 0 ? ghi : chi;
    for (I bi = b0; bi < b1 && !live; ++bi) {
      for (I bj = c0; bj < c1; ++bj) {
        const I f = bi * bg1 + bj;
        if ((__ldg(packed + (f >> 3)) >> (7 - (f & 7))) & 1) {
          live = true;
          break;
        }
      }
    }
  }
  const uint32_t word = __ballot_sync(0xffffffffu, live);
  if (lane == 0) occ[static_cast<int64_t>(g) * WG + w] = word;
  }
}

// ---------------------------------------------------------------------------
// Pass 2: per-group ordered compaction. One warp per group.
// ---------------------------------------------------------------------------
int sm_count() {
  static int sms = [] {
    int dev = 0, n = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
  }();
  return sms;
}

constexpr int kCompactThreads = 256;

// One block per group; thread t owns word t of each 256-word chunk (coordinates stay ascending
// across threads); block-wide exclusive scan of per-word popcounts gives each thread its slot base.
// Few long groups (e.g. pit:m over tall operands): blockIdx.y splits a group's words into ranges of
// words_per_split; a split first counts the live coordinates before its range (re-reading those
// words, cheap next to the scan) so every split writes its slots independently.
// word_at(w, own): bitmap word w of group g; own = the word lies in this block's range (a fused
// source stores it to the bitmap then; words before the range are only counted).
template <class WordAt>
__device__ __forceinline__ void compact_group(WordAt word_at, int64_t g, int64_t WG, int32_t* __restrict__ counts,
                                              int32_t* __restrict__ slots, int64_t slot_stride,
                                              int64_t words_per_split, int* warp_tot) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int32_t* out = slots + g * slot_stride;
  const int64_t w_begin = static_cast<int64_t>(blockIdx.y) * words_per_split;
  const int64_t w_end = w_begin + words_per_split < WG ? w_begin + words_per_split : WG;
  int base = 0;
  if (w_begin > 0) {
    int pre = 0;
    for (int64_t w = threadIdx.x; w < w_begin; w += kCompactThreads) pre += __popc(word_at(w, false));
#pragma unroll
    for (int o = 16; o; o >>= 1) pre += __shfl_xor_sync(0xffffffffu, pre, o);
    if (lane == 0) warp_tot[warp] = pre;
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kCompactThreads / 32; ++i) base += warp_tot[i];
    __syncthreads();
  }
  for (int64_t w0 = w_begin; w0 < w_end; w0 += kCompactThreads) {
    const int64_t w = w0 + threadIdx.x;
    uint32_t word = w < w_end ? word_at(w, true) : 0u;
    const int c = __popc(word);
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    int wbase = 0, total = 0;
#pragma unroll
    for (int i = 0; i < kCompactThreads / 32; ++i) {
      const int v = warp_tot[i];
      wbase += i < warp ? v : 0;
      total += v;
    }
    int pos = base + wbase + incl - c;
    // dense words (e.g. attention windows): a lane walking its own word's 32 bits serialises the
    // warp and scatters 4-byte stores; instead the warp expands one word at a time, lane = bit,
    // stores coalesced. Sparse words keep the per-lane walk (fewer iterations than 32).
    const int maxc = __reduce_max_sync(0xffffffffu, c);
    if (maxc > 20) {
      const uint32_t below = (1u << lane) - 1u;
      for (int j = 0; j < 32; ++j) {
        const uint32_t wj = __shfl_sync(0xffffffffu, word, j);
        const int pj = __shfl_sync(0xffffffffu, pos, j);
        if ((wj >> lane) & 1u) out[pj + __popc(wj & below)] = static_cast<int32_t>((w - lane + j) * 32 + lane);
      }
    } else {
      while (word) {
        const int b = __ffs(word) - 1;
        word &= word - 1;
        out[pos++] = static_cast<int32_t>(w * 32 + b);
      }
    }
    base += total;
    __syncthreads();
  }
  if (threadIdx.x == 0 && blockIdx.y == gridDim.y - 1) counts[g] = base;
}

__global__ void __launch_bounds__(kCompactThreads) compact_kernel(const uint32_t* __restrict__ occ, int64_t n_groups,
                                                                  int64_t WG, int32_t* __restrict__ counts,
                                                                  int32_t* __restrict__ slots, int64_t slot_stride,
                                                                  int64_t words_per_split) {
  __shared__ int warp_tot[kCompactThreads / 32];
  const int64_t g = blockIdx.x;
  const uint32_t* row = occ + g * WG;
  compact_group([row](int64_t w, bool) { return __ldg(row + w); }, g, WG, counts, slots, slot_stride,
                words_per_split, warp_tot);
}

// Annotation route, index in one launch: power-of-two geometry with coordinate blocks >= 32
// coordinates wide (e.g. the (128, 1) key index of a 32x64 attention block mask) -- a word's 32
// coordinates fall in at most two blocks, so a compaction thread derives its bitmap word from the
// packed bits itself (the same few byte loads detect_bits_pow2_kernel makes), stores it and
// compacts; no bitmap round trip through a second launch.
__global__ void __launch_bounds__(kCompactThreads) bits_compact_pow2_kernel(
    const uint8_t* __restrict__ packed, int32_t s0, int32_t s1, int lg0, int lg1, int lt0, int lt1, int pit_dim,
    int32_t pit_grid, int64_t WG, uint32_t* __restrict__ occ, int32_t* __restrict__ counts,
    int32_t* __restrict__ slots, int64_t slot_stride, int64_t words_per_split) {
  __shared__ int warp_tot[kCompactThreads / 32];
  const int32_t g = static_cast<int32_t>(blockIdx.x);
  uint32_t* row = occ + static_cast<int64_t>(g) * WG;
  auto word_at = [&](int64_t w, bool own) {
    const uint32_t word = bits_word_pow2<int32_t>(packed, s0, s1, lg0, lg1, lt0, lt1, pit_dim, pit_grid, g,
                                                  static_cast<int32_t>(w));
    if (own) row[w] = word;
    return word;
  };
  compact_group(word_at, g, WG, counts, slots, slot_stride, words_per_split, warp_tot);
}

// OR of all group rows: the union of live coordinates (used by pit:m union-row tiles).
// Union of every group's occupancy words: block = 32 consecutive words (lane = word, coalesced
// 128-byte rows) x 32 warps striding the groups with four independent loads in flight; the warps'
// partial ORs meet in shared memory. (A thread per word looping over all groups took 19 us for
// 256 groups x 128 words: one CTA, one dependent load chain per thread.)
constexpr int kUnionWarps = 32;
__global__ void __launch_bounds__(kUnionWarps * 32) union_kernel(const uint32_t* __restrict__ occ, int64_t n_groups,
                                                                 int64_t WG, uint32_t* __restrict__ uni) {
  __shared__ uint32_t part[kUnionWarps][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t w = static_cast<int64_t>(blockIdx.x) * 32 + lane;
  uint32_t acc = 0;
  if (w < WG) {
    int64_t g = warp;
    for (; g + 3 * kUnionWarps < n_groups; g += 4 * kUnionWarps) {
      const uint32_t a = __ldg(occ + g * WG + w), b = __ldg(occ + (g + kUnionWarps) * WG + w);
      const uint32_t c = __ldg(occ + (g + 2 * kUnionWarps) * WG + w), d = __ldg(occ + (g + 3 * kUnionWarps) * WG + w);
      acc |= (a | b) | (c | d);
    }
    for (; g < n_groups; g += kUnionWarps) acc |= __ldg(occ + g * WG + w);
  }
  part[warp][lane] = acc;
  __syncthreads();
  if (warp == 0) {
    uint32_t u = 0;
#pragma unroll
    for (int i = 0; i < kUnionWarps; ++i) u |= part[i][lane];
    if (w < WG) uni[w] = u;
  }
}

// Rebuild the occupancy bitmap from (possibly reordered) slots: lets kernels that need
// per-(coordinate, group) liveness accept an arbitrary user-supplied index.
__global__ void slots_to_occ_kernel(const int32_t* __restrict__ counts, const int32_t* __restrict__ slots,
                                    int64_t slot_stride, int64_t n_groups, int64_t WG, int64_t pit_grid,
                                    uint32_t* __restrict__ occ, int* __restrict__ bad) {
  const int64_t g = blockIdx.y;
  if (g >= n_groups) return;
  const int cnt = counts[g];
  for (int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; s < cnt;
       s += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t c = slots[g * slot_stride + s];
    if (c < 0 || c >= pit_grid) {
      atomicExch(bad, 1);
      continue;
    }
    atomicOr(&occ[g * WG + (c >> 5)], 1u << (c & 31));
  }
}

}  // namespace

// ---------------------------------------------------------------------------- launchers
static bool R_fits_grid(int64_t GR) { return GR / 32 + 1 < (1ll << 31); }

// PIT_COLS_SLAB=0: column-axis detection on the one-band-per-block kernel (A/B knob)
static bool cols_slab_enabled() {
  static const bool on = [] {
    const char* e = getenv("PIT_COLS_SLAB");
    return !e || atoi(e) != 0;
  }();
  return on;
}

int launch_detect_values(const DetectValuesArgs& a, cudaStream_t s) {
  const int eb = dtype_bytes(a.dtype);
  const int64_t GR = ceil_div(a.R, a.tr), GC = ceil_div(a.C, a.tc);
  const int64_t n_groups = a.pit_phys == 0 ? GC : GR;
  const int64_t pit_grid = a.pit_phys == 0 ? GR : GC;
  const int64_t WG = ceil_div(pit_grid, 32);
  if (n_groups == 0 || pit_grid == 0) return 0;

  const int64_t row_bytes = a.C * eb, ld_bytes = a.ld * eb;
  const int64_t vec_per_micro = (static_cast<int64_t>(a.tc) * eb) / 16;
  const bool aligned = (reinterpret_cast<uintptr_t>(a.x) % 16 == 0) && (ld_bytes % 16 == 0) && (row_bytes % 16 == 0);
  const bool pow2 = vec_per_micro >= 1 && vec_per_micro <= 32 && (vec_per_micro & (vec_per_micro - 1)) == 0 &&
                    (static_cast<int64_t>(a.tc) * eb) % 16 == 0;
  // wide micro-columns (e.g. BERT's (1, 768) row micro-tiles): whole 512-byte segments per micro-column
  const bool wide = vec_per_micro > 32 && vec_per_micro % 32 == 0 && (static_cast<int64_t>(a.tc) * eb) % 16 == 0;
  if (a.pit_phys == 0 && aligned && a.tr == 1 && GC == 1 && R_fits_grid(GR)) {
    detect_row_any_kernel<<<static_cast<unsigned>(GR / 32 + (GR % 32 != 0)), 256, 0, s>>>(
        static_cast<const uint8_t*>(a.x), a.R, row_bytes, ld_bytes, live_mask_for(a.dtype), a.occ);
    note_launch();
    return cuda_status();
  }
  if (a.pit_phys == 0 && aligned && (pow2 || wide)) {
    if (wide && cudaMemsetAsync(a.occ, 0, static_cast<size_t>(n_groups * WG) * sizeof(uint32_t), s) != cudaSuccess)
      return cuda_status();
    const int64_t segs = ceil_div(row_bytes, 512);
    const int64_t seg_groups = ceil_div(segs, kRaWarps);
    const int64_t tiles = seg_groups * ceil_div(GR, 32);
    int dev = 0, sms = 148, per_sm = 4;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, detect_rows_vec_kernel, kRaWarps * 32, 0);
    if (per_sm < 1) per_sm = 1;
    const int64_t resident = static_cast<int64_t>(per_sm) * sms;  // one wave of persistent CTAs
    // every CTA takes the same number of tiles (C1's 1024 tiles: 512 CTAs x 2 instead of 592 CTAs
    // with a 27%-idle second pass; 34.3 -> 33.9 us per graph)
    const int64_t per_cta = ceil_div(tiles, resident);
    const int64_t grid = ceil_div(tiles, per_cta);
    detect_rows_vec_kernel<<<static_cast<unsigned>(grid), kRaWarps * 32, 0, s>>>(
        static_cast<const uint8_t*>(a.x), a.R, row_bytes, ld_bytes, a.tr, static_cast<int>(vec_per_micro), GR, GC,
        live_mask_for(a.dtype), a.occ, WG, seg_groups, tiles);
    note_launch();
  } else if (a.pit_phys == 1 && aligned && (static_cast<int64_t>(a.tc) * eb) % 16 == 0 && vec_per_micro >= 1 &&
             vec_per_micro <= 32 && (vec_per_micro & (vec_per_micro - 1)) == 0 &&
             (a.tr % 32 == 0 || 32 % a.tr == 0) && ceil_div(a.R, 32) <= 65535 && cols_slab_enabled()) {
    const int lg = __builtin_ctzll(static_cast<unsigned long long>(vec_per_micro));
    const int64_t nvec = row_bytes / 16;
    const int atomic_out = a.tr > 32 || lg >= 4;  // several blocks share a band's word
    if (atomic_out &&
        cudaMemsetAsync(a.occ, 0, static_cast<size_t>(n_groups * WG) * sizeof(uint32_t), s) != cudaSuccess)
      return cuda_status();
    dim3 grid(static_cast<unsigned>(ceil_div(nvec, 256)), static_cast<unsigned>(ceil_div(a.R, 32)));
    detect_cols_slab_kernel<<<grid, 256, 0, s>>>(static_cast<const uint8_t*>(a.x), a.R, ld_bytes, nvec, a.tr, lg, GR,
                                                 live_mask_for(a.dtype), a.occ, WG, atomic_out);
    note_launch();
  } else if (a.pit_phys == 1 && aligned && (static_cast<int64_t>(a.tc) * eb) % 16 == 0 && vec_per_micro >= 1 &&
             vec_per_micro <= 32 && (vec_per_micro & (vec_per_micro - 1)) == 0 && GR <= 65535) {
    const int lg = __builtin_ctzll(static_cast<unsigned long long>(vec_per_micro));
    const int64_t nvec = row_bytes / 16;
    // a 32-bit word spans 32 micro-columns = 32 * VPB vectors: more than one block's 256 when VPB >= 16
    if (lg >= 4 && cudaMemsetAsync(a.occ, 0, static_cast<size_t>(n_groups * WG) * sizeof(uint32_t), s) != cudaSuccess)
      return cuda_status();
    dim3 grid(static_cast<unsigned>(ceil_div(nvec, 256)), static_cast<unsigned>(GR));
    detect_cols_vec_kernel<<<grid, 256, 0, s>>>(static_cast<const uint8_t*>(a.x), a.R, ld_bytes, nvec, a.tr, lg, GR,
                                                live_mask_for(a.dtype), a.occ, WG);
    note_launch();
  } else {
    const int TJ = a.pit_phys == 0 ? 256 : (a.tc >= 8 ? 32 : 128);
    dim3 grid(static_cast<unsigned>(ceil_div(GC, TJ)), static_cast<unsigned>(ceil_div(GR, 32)));
    if (grid.y > 65535u) return kErrShape;
    const size_t smem = sizeof(uint32_t) * (a.pit_phys == 0 ? TJ : TJ);
    detect_generic_kernel<<<grid, kGenThreads, smem, s>>>(static_cast<const uint8_t*>(a.x), a.dtype, eb, a.R, a.C,
                                                          a.ld, a.tr, a.tc, GR, GC, a.pit_phys, TJ, a.occ, WG);
    note_launch();
  }
  return cuda_status();
}

int launch_detect_bits(const DetectBitsArgs& a, cudaStream_t s) {
  const int64_t G0 = ceil_div(a.s0, a.t0), G1 = ceil_div(a.s1, a.t1);
  const int64_t n_groups = a.pit_dim == 0 ? G1 : G0;
  const int64_t pit_grid = a.pit_dim == 0 ? G0 : G1;
  const int64_t WG = ceil_div(pit_grid, 32);
  if (n_groups == 0 || pit_grid == 0) return 0;
  const int64_t warps = n_groups * WG;
  const int threads = 256;
  const int64_t needed = ceil_div(warps * 32, threads);
  const int64_t wave = static_cast<int64_t>(sm_count()) * 8;
  const unsigned blocks = static_cast<unsigned>(needed < wave ? needed : wave);
  // 32-bit indexing when the thread count, the block-grid size and every (i+1)*t product fit
  const int64_t G0b = ceil_div(a.s0, a.g0), G1b = ceil_div(a.s1, a.g1);
  const bool fits32 = warps * 32 < (1ll << 31) && G0b * G1b < (1ll << 31) &&
                      (a.s0 + a.t0) * 2 < (1ll << 31) && (a.s1 + a.t1) * 2 < (1ll << 31);
  const int ct = a.pit_dim == 0 ? a.t0 : a.t1, cg = a.pit_dim == 0 ? a.g0 : a.g1;
  const bool pow2 = (ct & (ct - 1)) == 0 && (cg & (cg - 1)) == 0;
  const int lct = pow2 ? __builtin_ctz(static_cast<unsigned>(ct)) : 0;
  const int lcg = pow2 ? __builtin_ctz(static_cast<unsigned>(cg)) : 0;
  const bool all_pow2 = pow2 && (a.t0 & (a.t0 - 1)) == 0 && (a.t1 & (a.t1 - 1)) == 0 && (a.g0 & (a.g0 - 1)) == 0 &&
                        (a.g1 & (a.g1 - 1)) == 0;
  if (fits32 && all_pow2 && lcg < lct + 5) {
    const unsigned b3 = static_cast<unsigned>(needed < wave ? needed : wave);  // a warp per (group, word)
    detect_bits_pow2_lane_kernel<int32_t><<<b3, threads, 0, s>>>(
        a.packed, static_cast<int32_t>(a.s0), static_cast<int32_t>(a.s1), __builtin_ctz(static_cast<unsigned>(a.g0)),
        __builtin_ctz(static_cast<unsigned>(a.g1)), __builtin_ctz(static_cast<unsigned>(a.t0)),
        __builtin_ctz(static_cast<unsigned>(a.t1)), a.pit_dim, static_cast<int32_t>(n_groups),
        static_cast<int32_t>(pit_grid), static_cast<int32_t>(WG), a.occ);
  } else if (fits32 && all_pow2) {
    const int64_t items = n_groups * WG;
    const int64_t need = ceil_div(items, threads);
    const unsigned b2 = static_cast<unsigned>(need < wave ? need : wave);
    detect_bits_pow2_kernel<int32_t><<<b2, threads, 0, s>>>(
        a.packed, static_cast<int32_t>(a.s0), static_cast<int32_t>(a.s1), __builtin_ctz(static_cast<unsigned>(a.g0)),
        __builtin_ctz(static_cast<unsigned>(a.g1)), __builtin_ctz(static_cast<unsigned>(a.t0)),
        __builtin_ctz(static_cast<unsigned>(a.t1)), a.pit_dim, static_cast<int32_t>(n_groups),
        static_cast<int32_t>(pit_grid), static_cast<int32_t>(WG), a.occ);
  } else if (fits32 && pow2)
    detect_bits_kernel<int32_t, true><<<blocks, threads, 0, s>>>(
        a.packed, static_cast<int32_t>(a.s0), static_cast<int32_t>(a.s1), a.g0, a.g1, a.t0, a.t1, a.pit_dim,
        static_cast<int32_t>(n_groups), static_cast<int32_t>(pit_grid), static_cast<int32_t>(WG), a.occ, lct, lcg);
  else if (fits32)
    detect_bits_kernel<int32_t, false><<<blocks, threads, 0, s>>>(
        a.packed, static_cast<int32_t>(a.s0), static_cast<int32_t>(a.s1), a.g0, a.g1, a.t0, a.t1, a.pit_dim,
        static_cast<int32_t>(n_groups), static_cast<int32_t>(pit_grid), static_cast<int32_t>(WG), a.occ, 0, 0);
  else
    detect_bits_kernel<int64_t, false><<<blocks, threads, 0, s>>>(a.packed, a.s0, a.s1, a.g0, a.g1, a.t0, a.t1,
                                                                  a.pit_dim, n_groups, pit_grid, WG, a.occ, 0, 0);
  note_launch();
  return cuda_status();
}

// split long groups over blockIdx.y when there are too few groups to fill the GPU
static void compact_splits(int64_t n_groups, int64_t WG, int64_t* splits_out, int64_t* wps_out) {
  int64_t splits = 1, wps = WG;
  const int64_t target = 2 * static_cast<int64_t>(sm_count());
  if (n_groups < target && WG > 4 * kCompactThreads) {
    splits = ceil_div(target, n_groups);
    const int64_t max_splits = ceil_div(WG, kCompactThreads);
    if (splits > max_splits) splits = max_splits;
    if (splits > 65535) splits = 65535;
    wps = ceil_div(ceil_div(WG, splits), kCompactThreads) * kCompactThreads;
    splits = ceil_div(WG, wps);
  }
  *splits_out = splits;
  *wps_out = wps;
}

int launch_compact(const uint32_t* occ, int64_t n_groups, int64_t WG, int32_t* counts, int32_t* slots,
                   int64_t slot_stride, cudaStream_t s) {
  if (n_groups == 0) return 0;
  if (n_groups >= (1ll << 31)) return kErrShape;
  int64_t splits, wps;
  compact_splits(n_groups, WG, &splits, &wps);
  dim3 grid(static_cast<unsigned>(n_groups), static_cast<unsigned>(splits));
  compact_kernel<<<grid, kCompactThreads, 0, s>>>(occ, n_groups, WG, counts, slots, slot_stride, wps);
  note_launch();
  return cuda_status();
}

// PIT_BITS_FUSE=0: annotation-route index as detect_bits + compact (two launches; A/B knob)
static bool bits_fuse_enabled() {
  static const bool on = [] {
    const char* e = getenv("PIT_BITS_FUSE");
    return !e || atoi(e) != 0;
  }();
  return on;
}

int launch_index_from_bits(const DetectBitsArgs& a, int32_t* counts, int32_t* slots, int64_t slot_stride,
                           cudaStream_t s) {
  const int64_t G0 = ceil_div(a.s0, a.t0), G1 = ceil_div(a.s1, a.t1);
  const int64_t n_groups = a.pit_dim == 0 ? G1 : G0;
  const int64_t pit_grid = a.pit_dim == 0 ? G0 : G1;
  const int64_t WG = ceil_div(pit_grid, 32);
  if (n_groups == 0 || pit_grid == 0) return 0;
  const int64_t G0b = ceil_div(a.s0, a.g0), G1b = ceil_div(a.s1, a.g1);
  const bool fits32 = n_groups * WG * 32 < (1ll << 31) && G0b * G1b < (1ll << 31) &&
                      (a.s0 + a.t0) * 2 < (1ll << 31) && (a.s1 + a.t1) * 2 < (1ll << 31) && n_groups < 65536ll * 32768;
  auto p2 = [](int v) { return v > 0 && (v & (v - 1)) == 0; };
  const bool all_pow2 = p2(a.t0) && p2(a.t1) && p2(a.g0) && p2(a.g1);
  const int ct = a.pit_dim == 0 ? a.t0 : a.t1, cg = a.pit_dim == 0 ? a.g0 : a.g1;
  if (!(fits32 && all_pow2 && bits_fuse_enabled()) ||
      __builtin_ctz(static_cast<unsigned>(cg)) < __builtin_ctz(static_cast<unsigned>(ct)) + 5) {
    if (int st = launch_detect_bits(a, s)) return st;
    return launch_compact(a.occ, n_groups, WG, counts, slots, slot_stride, s);
  }
  int64_t splits, wps;
  compact_splits(n_groups, WG, &splits, &wps);
  dim3 grid(static_cast<unsigned>(n_groups), static_cast<unsigned>(splits));
  bits_compact_pow2_kernel<<<grid, kCompactThreads, 0, s>>>(
      a.packed, static_cast<int32_t>(a.s0), static_cast<int32_t>(a.s1), __builtin_ctz(static_cast<unsigned>(a.g0)),
      __builtin_ctz(static_cast<unsigned>(a.g1)), __builtin_ctz(static_cast<unsigned>(a.t0)),
      __builtin_ctz(static_cast<unsigned>(a.t1)), a.pit_dim, static_cast<int32_t>(pit_grid), WG, a.occ, counts,
      slots, slot_stride, wps);
  note_launch();
  return cuda_status();
}

// Live micro-tiles per group (popcount of the group's occupancy words): a warp per group. Used by
// plan selection, which needs only counts for every candidate micro-tile.
__global__ void occ_counts_kernel(const uint32_t* __restrict__ occ, int64_t n_groups, int64_t WG,
                                  int32_t* __restrict__ counts) {
  const int64_t g = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (g >= n_groups) return;
  const uint32_t* row = occ + g * WG;
  int c = 0;
  for (int64_t w = lane; w < WG; w += 32) c += __popc(__ldg(row + w));
#pragma unroll
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) counts[g] = c;
}

int launch_occ_counts(const uint32_t* occ, int64_t n_groups, int64_t WG, int32_t* counts, cudaStream_t s) {
  if (n_groups == 0) return 0;
  occ_counts_kernel<<<static_cast<unsigned>(ceil_div(n_groups * 32, 256)), 256, 0, s>>>(occ, n_groups, WG, counts);
  note_launch();
  return cuda_status();
}

int launch_union(const uint32_t* occ, int64_t n_groups, int64_t WG, uint32_t* uni, cudaStream_t s) {
  if (WG == 0) return 0;
  if (ceil_div(WG, 32) > 0x7fffffffll) return kErrShape;
  union_kernel<<<static_cast<unsigned>(ceil_div(WG, 32)), kUnionWarps * 32, 0, s>>>(occ, n_groups, WG, uni);
  note_launch();
  return cuda_status();
}

int launch_slots_to_occ(const int32_t* counts, const int32_t* slots, int64_t slot_stride, int64_t n_groups,
                        int64_t WG, int64_t pit_grid, uint32_t* occ, int* bad, cudaStream_t s) {
  if (n_groups == 0) return 0;
  cudaMemsetAsync(occ, 0, sizeof(uint32_t) * n_groups * WG, s);
  dim3 grid(static_cast<unsigned>((ceil_div(pit_grid, 256) < 64 ? ceil_div(pit_grid, 256) : int64_t(64))), static_cast<unsigned>(n_groups));
  if (n_groups > 65535) return kErrShape;
  slots_to_occ_kernel<<<grid, 256, 0, s>>>(counts, slots, slot_stride, n_groups, WG, pit_grid, occ, bad);
  note_launch();
  return cuda_status();
}

}  // namespace pit
