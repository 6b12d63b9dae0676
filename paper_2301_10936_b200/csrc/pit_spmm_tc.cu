// PIT sparse matmul on the 5th-gen tensor cores (tcgen05 + TMEM, TMA tiles, cp.async gathers),
// bf16/fp16 in, fp32 accumulate, bf16/fp16 out. Persistent, warp-specialised kernels (512 threads:
// warps 0-7 producers, 8 MMA issuer, 9 TMEM allocator on single-CTA kernels, 10 relay (CTA pairs),
// 11 TMA issuer in mask modes, 12-15 epilogue; CTA-pair kernels allocate TMEM from warp 0):
//
//  * spmm_gk / spmm_gk2 ("gathered K", PIT axis k; reference executor.py:386-423 `_matmul_pit_k`).
//    A group is an M-block of GW rows (micro-tile (GW,1)); its live k coordinates index rows of
//    A^T (A is column-major, executor.py:318-325) and rows of B. Both are gathered with 16-byte
//    cp.async into MN-major swizzled shared memory (TMA tile::gather4 measured at ~1/3 of the
//    cp.async rate on this part, K2) and fed to tcgen05.mma: orientation T
//    (D[n, m] += B^T A^T, group rows on the MMA's N side: 16..64-row micro-tiles run as dense MMAs
//    with no union waste) or N (128-row groups); spmm_gk2 runs 256-row groups on CTA pairs. Split
//    units balance few, unequal groups (C3's global query rows); TMA tile stores write C.
//
//  * rowgemm / rowgemm2 / rowgemm2t ("gathered M", PIT axis m, dense, grouped; executor.py:352-383,
//    :426-461). Output row tiles are union rows, consecutive slice rows or a group's rows; A rows by
//    TMA tiles when consecutive (or packed first), by cp.async otherwise, with dead (row,
//    micro-column) items zero-filled or zeroed in shared memory; B K-blocks are TMA tiles of the
//    stacked [G, K, N] weights; K-blocks with no live row take no ring slot. The C tile stays in
//    TMEM across K and is stored once (SWrite fused: TMA boxes for consecutive rows, 128-byte row
//    segments for scattered ones). rowgemm2 runs 256x256 tiles on CTA pairs; rowgemm2t swaps the
//    operand roles for small groups (MoE experts, the high-sparsity pit:m supergroups of
//    pit_gm_sparse.cu, whose fp32 partial rows it writes).
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "pit_internal.h"
#include <type_traits>
#include "pit_ptx.cuh"

namespace pit {

namespace {

// Warp roles: 0..7 producers (gather issue is instruction- and latency-bound per warp, so eight warps
// split each stage's copies), 8 MMA issuer, 9 TMEM allocator, 12..15 epilogue (one per TMEM lane
// quarter).
constexpr int kProdWarps = 8;
#ifndef PIT_GK_IDX_DEPTH
#define PIT_GK_IDX_DEPTH 3
#endif
constexpr int kGkIdxDepth = PIT_GK_IDX_DEPTH;  // spmm_gk producers: stages of slot indices in flight + 1
static_assert(kGkIdxDepth >= 3, "the rotation needs at least three slot sets");
constexpr int kProdThreads = kProdWarps * 32;
constexpr int kMmaWarp = 8;
constexpr int kAllocWarp = 9;
// CTA-pair kernels allocate TMEM (tcgen05.alloc.cta_group::2) from warp 0: compute-sanitizer racecheck
// reports a hazard between the allocator's shared-memory write and the slot reads after the cluster
// barrier whenever the allocating warp is not warp 0 (scripts/probe/tmem_alloc2_race.cu: the report
// follows the warp index alone, not the slot's placement or the mbarrier initialisation), so the
// pair kernels use warp 0 and run racecheck-clean
constexpr int kAlloc2Warp = 0;
constexpr int kEpiWarp0 = 12;
constexpr int kThreads = 512;

template <bool kBF16>
struct OutT;
template <>
struct OutT<true> {
  using T = __nv_bfloat16;
  __device__ static T cvt(float x) { return __float2bfloat16_rn(x); }
};
template <>
struct OutT<false> {
  using T = __half;
  __device__ static T cvt(float x) { return __float2half_rn(x); }
};

__device__ __forceinline__ uint32_t pack2(float a, float b, bool bf16) {
  if (bf16) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  }
  __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

template <int N>
__host__ __device__ constexpr uint32_t tmem_cols_pow2() {
  return N <= 32 ? 32 : N <= 64 ? 64 : N <= 128 ? 128 : N <= 256 ? 256 : 512;
}

// One 32-row x 64-column output box of a warp's TMEM lane quarter -> C through a TMA tile store:
// tcgen05.ld (two x32) -> bf16/fp16 -> 128B-swizzled shared staging (conflict-free 16-byte stores)
// -> cp.async.bulk.tensor store of whole 128-byte lines. Two staging buffers per warp alternate; a
// buffer is reused only after the store issued from it two boxes ago has read it. Rows / columns
// past the tensor are clipped by the tensor map. have == false stores zeros (empty units).
template <bool kBF16>
__device__ __forceinline__ void epi_box_tma(uint32_t tsrc, bool have, uint32_t buf, const CUtensorMap* tmC,
                                            bool do_store, int c0, int r0, int lane) {
  uint32_t v[64];
  if (have) {
    tmem_ld32(tsrc, *reinterpret_cast<uint32_t(*)[32]>(v));
    tmem_ld32(tsrc + 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
    tmem_wait_ld();
  } else {
#pragma unroll
    for (int i = 0; i < 64; ++i) v[i] = 0u;
  }
  if (lane == 0) bulk_wait_read<1>();
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 8; ++j)
    st_shared_v4(buf + lane * 128 + ((static_cast<uint32_t>(j) ^ static_cast<uint32_t>(lane & 7)) << 4),
                 pack2(__uint_as_float(v[8 * j + 0]), __uint_as_float(v[8 * j + 1]), kBF16),
                 pack2(__uint_as_float(v[8 * j + 2]), __uint_as_float(v[8 * j + 3]), kBF16),
                 pack2(__uint_as_float(v[8 * j + 4]), __uint_as_float(v[8 * j + 5]), kBF16),
                 pack2(__uint_as_float(v[8 * j + 6]), __uint_as_float(v[8 * j + 7]), kBF16));
  fence_proxy_async_smem();
  __syncwarp();
  if (lane == 0 && do_store) {
    tma_store_2d(tmC, buf, c0, r0);
    bulk_commit();
  }
}

// =============================================================================================
// spmm_gk: PIT axis k.
//
// Orientation T (GW < 128, and GW == 256): D[n, m] += B^T[n, k] * A^T[k, m] — M_mma = 128 output
//   columns per accumulator, N_mma = GW group rows; the n tile holds N_TILE/128 accumulators.
// Orientation N (GW == 128): D[m, n] += A[m, k] * B[k, n] — M_mma = the group's 128 rows,
//   N_mma = 256 output columns; one MMA per k16 (less shared-memory operand traffic per FLOP) and a
//   row-contiguous epilogue.
// Both operands are MN-major 128B-swizzled gathers of k rows; only descriptors and the epilogue
// differ between orientations.
// =============================================================================================
// ---------------------------------------------------------------------------------------------
// Split gathered-K units (few, unequal groups). The persistent spmm_gk walk gives every CTA the
// same number of units, so with only ~2-3 units per SM one long group sets the kernel's length:
// Longformer's global query rows see every key (4096 live k against ~1100 for a windowed group) —
// 46 us of a kernel whose work balances to ~30. Every CTA first derives the same plan from the
// counts: a group longer than twice the mean becomes chunks of about the mean (multiples of KS),
// virtual groups in group order; the CTA keeps its own units {group, first slot, count, partial}.
// A chunk leaves an fp32 partial tile in caller scratch; the chunk that finishes its group last
// (atomic counter) sums the tiles into C. Deterministic plan; the fp32 sum order of a split group
// is fixed (chunk order), so results are reproducible.
constexpr int kSplitParts = 255;     // partial tiles at most (8-bit index)
constexpr int kSplitMaxGroups = 2048;
constexpr int kSplitCtrBytes = 512;  // split-group arrival counters (<= 85 groups: >= 3 chunks each)

// exclusive block scan (blockDim.x a multiple of 32, <= 1024); sh: >= 32 ints of shared scratch
__device__ __forceinline__ int block_excl_scan(int v, int* sh, int& total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[w] = x;
  __syncthreads();
  if (w == 0) {
    int z = lane < nw ? sh[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, z, o);
      if (lane >= o) z += y;
    }
    if (lane < nw) sh[lane] = z;
  }
  __syncthreads();
  const int excl = x - v + (w ? sh[w - 1] : 0);
  total = sh[nw - 1];
  __syncthreads();
  return excl;
}

// One CTA of 1024 threads (2 groups per thread, n_groups <= kSplitMaxGroups): the split plan as the
// virtual-group table vtab[v] = {group, first slot, count, -1 or first partial | chunk << 8 |
// split group << 16 | chunks << 24}, their number in *nv, and zeroed split-group counters.
__global__ void __launch_bounds__(1024) gk_split_plan_kernel(const int32_t* __restrict__ counts, int n_groups, int ks,
                                                             int4* __restrict__ vtab, int* __restrict__ nv,
                                                             int* __restrict__ ctr, int split_first) {
  __shared__ int sc[32];
  const int tid = threadIdx.x;
  if (tid < kSplitCtrBytes / 4) ctr[tid] = 0;
  int cnt[2], valid[2];
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int g = 2 * tid + j;
    valid[j] = g < n_groups;
    cnt[j] = valid[j] ? __ldg(counts + g) : 0;
  }
  int tot;
  block_excl_scan(cnt[0] + cnt[1], sc, tot);  // total live k (the host keeps n_groups * pit_grid < 2^31)
  const int mean = (tot + n_groups - 1) / n_groups;
  const int L = max((mean + ks - 1) / ks, 1) * ks;
  int nch[2], want[2];
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    nch[j] = cnt[j] > 2 * L ? (cnt[j] + L - 1) / L : 1;
    want[j] = valid[j] && nch[j] > 1 && nch[j] <= 127 ? nch[j] : 0;
  }
  int twant;
  const int pp = block_excl_scan(want[0] + want[1], sc, twant);
  const int ppj[2] = {pp, pp + want[0]};
  bool split[2];
  int nf[2];
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    split[j] = want[j] > 0 && ppj[j] + want[j] <= kSplitParts;
    nf[j] = valid[j] ? (split[j] ? nch[j] : 1) : 0;
  }
  // virtual groups: the split groups' chunks first (their last-arriver sums then overlap the CTAs'
  // later units; C3 step 55 -> 52 us), the others after in group order. One scan carries the
  // group-order prefix (low 16 bits, <= n_groups + P) and the split-group prefix (high bits).
  const int pk0 = nf[0] | (static_cast<int>(split[0]) << 16), pk1 = nf[1] | (static_cast<int>(split[1]) << 16);
  int tpk;
  const int pk = block_excl_scan(pk0 + pk1, sc, tpk);
  int vpj[2] = {pk & 0xffff, (pk & 0xffff) + nf[0]};
  const int spj[2] = {pk >> 16, (pk >> 16) + static_cast<int>(split[0])};
  if (split_first) {
    const int ns0 = split[0] ? nch[0] : 0, ns1 = split[1] ? nch[1] : 0;
    const int nu0 = nf[0] && !split[0] ? 1 : 0, nu1 = nf[1] && !split[1] ? 1 : 0;
    int tns, tnu;
    const int vs = block_excl_scan(ns0 + ns1, sc, tns);
    const int vu = block_excl_scan(nu0 + nu1, sc, tnu);
    vpj[0] = split[0] ? vs : tns + vu;
    vpj[1] = split[1] ? vs + ns0 : tns + vu + nu0;
  }
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int g = 2 * tid + j;
    const int len = split[j] ? ((cnt[j] + nch[j] - 1) / nch[j] + ks - 1) / ks * ks : cnt[j];
    for (int c = 0; c < nf[j]; ++c) {
      const int k0 = c * len;
      vtab[vpj[j] + c] = make_int4(g, k0, min(len, cnt[j] - k0),
                                   split[j] ? (ppj[j] | (c << 8) | (spj[j] << 16) | (nch[j] << 24)) : -1);
    }
  }
  if (tid == 0) *nv = tpk & 0xffff;
}

template <int GW, bool kOrientN, int kKS = 64, int kNT = 0>
struct GkCfg {
  static constexpr int KS = kKS;  // gathered k per stage
  // n columns per unit; kNT = 128 serves narrow N (e.g. attention P.V with head dim 64)
  static constexpr int N_TILE = kNT ? kNT : (kOrientN || GW < 256) ? 256 : 128;
  static constexpr int B_ATOMS = N_TILE / 64;
  static constexpr int A_ROW_BYTES = GW * 2 < 128 ? GW * 2 : 128;  // bytes per smem row of the A^T strip
  static constexpr int A_ATOMS = GW * 2 <= 128 ? 1 : GW * 2 / 128;
  static constexpr int B_BYTES = B_ATOMS * KS * 128;
  static constexpr int A_BYTES = A_ATOMS * KS * A_ROW_BYTES;
  static constexpr int STAGE_BYTES = ((B_BYTES + A_BYTES + 1023) / 1024) * 1024;
  // C goes out through TMA tile stores from shared staging: orientation N, 2 x 4 KB per epilogue
  // warp (epi_box_tma); orientation T (GW <= 64), one [GW rows x 32 columns] box per warp
  static constexpr int STG_T = GW <= 64 ? GW * 64 : 0;
  static constexpr int STG_BYTES = kOrientN ? 4 * 2 * 4096 : 4 * STG_T;
  // 227 KB opt-in minus 1 KB alignment slack, the TMEM barriers / slot, the staging; every stage also
  // carries 8 full + 8 empty barriers (one pair per producer warp)
  // producer warps are split into BAR_GROUPS groups with their own full / empty barrier per stage
  // (the MMA starts on a group's rows once they land and releases each group's slot separately)
#ifndef PIT_GK_BG
#define PIT_GK_BG 1
#endif
  static constexpr int BAR_GROUPS = (KS / PIT_GK_BG) % 16 == 0 ? PIT_GK_BG : 1;
  static constexpr int STAGE_BUDGET = 232448 - 1024 - 256 - STG_BYTES;
  static constexpr int STAGES = STAGE_BUDGET / (STAGE_BYTES + 128) > 16 ? 16 : STAGE_BUDGET / (STAGE_BYTES + 128);
  static constexpr int ACC_COLS = kOrientN ? N_TILE : (N_TILE / 128) * GW;  // TMEM columns per buffer
  // accumulator ring: as many units in flight as TMEM holds (<= 8), so short units (few live k per
  // group) overlap their load, MMA and epilogue across units instead of serialising on 2 buffers
#ifndef PIT_GK_NBUF_MAX
#define PIT_GK_NBUF_MAX 8
#endif
  static constexpr int NBUF = (512 / ACC_COLS) > PIT_GK_NBUF_MAX ? PIT_GK_NBUF_MAX : (512 / ACC_COLS);
  static constexpr int TMEM_COLS = tmem_cols_pow2<NBUF * ACC_COLS>();
  static constexpr size_t SMEM = static_cast<size_t>(STAGES) * (STAGE_BYTES + 128) + STG_BYTES + 1024 + 256;
  static_assert(SMEM <= 232448, "shared memory over the sm_100 opt-in limit");
  static constexpr uint32_t A_SW = sw_layout_for_row(A_ROW_BYTES);
  static constexpr uint32_t A_MASK = A_ROW_BYTES == 128 ? 7 : A_ROW_BYTES == 64 ? 3 : A_ROW_BYTES == 32 ? 1 : 0;
  static constexpr int B_CPR = N_TILE / 8;       // 16-byte chunks per gathered B row
  static constexpr int A_CPR = GW * 2 / 16;      // 16-byte chunks per gathered A^T row
  static constexpr int A_CPA = A_ROW_BYTES / 16; // chunks per atom row
  static constexpr int A_RPW = 32 / A_CPR;       // A rows covered by one warp instruction
};

template <int GW, bool kOrientN, bool kBF16, int kKS, int kNT, bool kSplit = false>
__global__ void __launch_bounds__(kThreads, 1)
    spmm_gk_kernel(const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmAt,
                   const __grid_constant__ CUtensorMap tmBr, int runs, int use_tma_store, const void* __restrict__ Bv, int64_t ldb, const void* __restrict__ Atv, int64_t lda,
                   const int32_t* __restrict__ counts, const int32_t* __restrict__ slots, int64_t slot_stride,
                   int n_groups, int n_tiles, int M, int N, int K, void* __restrict__ Cv, int64_t ldc,
                   int grp_rows, int gpb, int64_t b_batch_stride, int* __restrict__ split_ctr,
                   float* __restrict__ ws) {
  // grp_rows (<= GW, multiple of 8): rows per group. Micro-tiles narrower than the kernel's GW run
  // in it with the A^T strip's extra columns zero-filled and never stored.
  // Batched (prevalent axis, e.g. attention heads): slices are stacked along M in A and C (slice b
  // owns groups [b*gpb, (b+1)*gpb)); only B differs per slice, at b * b_batch_stride elements.
  using Cfg = GkCfg<GW, kOrientN, kKS, kNT>;
  using OT = OutT<kBF16>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stg = smem + Cfg::STAGES * Cfg::STAGE_BYTES;  // epilogue staging (orientation N)
  // per (stage, producer-warp group) full / empty barriers: the MMA starts on a group's rows as soon
  // as they land and hands each group its slot back as soon as the MMAs reading it complete
  constexpr int BG = Cfg::BAR_GROUPS, WPG = kProdWarps / BG;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(stg + Cfg::STG_BYTES);
  uint64_t* empty_bar = full_bar + Cfg::STAGES * kProdWarps;
  uint64_t* tfull_bar = empty_bar + Cfg::STAGES * kProdWarps;
  uint64_t* tempty_bar = tfull_bar + Cfg::NBUF;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + Cfg::NBUF);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < Cfg::STAGES * kProdWarps; ++i) {
      mbar_init(&full_bar[i], 32 * WPG);
      mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < Cfg::NBUF; ++i) {
      mbar_init(&tfull_bar[i], 1);
      mbar_init(&tempty_bar[i], 128);
    }
    fence_mbar_init();
  }
  if (warp == kAllocWarp) tmem_alloc<Cfg::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // Units are (n tile, group) pairs, n-tile major: the CTAs running concurrently share one
  // [K, N_TILE] slab of B, which stays L2-resident while every group gathers from it.
  // kSplit: the walk runs over virtual groups (gk_split_plan_kernel): entry {group, first slot,
  // count, partial tile or -1}; a long group's chunks go to different CTAs and leave fp32 partial
  // tiles that gk_split_fixup_kernel sums into C.
  static_assert(!kSplit || kOrientN, "split units are implemented for orientation N");
  __shared__ int s_last;
  const int4* vtab = reinterpret_cast<const int4*>(split_ctr + kSplitCtrBytes / 4);  // kSplit: after the counters
  const int n_vg = kSplit ? __ldg(reinterpret_cast<const int*>(vtab) - 1) : n_groups;
  const int units = n_vg * n_tiles;
  auto vunit = [&](int g) { return __ldg(vtab + g); };
  auto vcount = [&](int g) { return kSplit ? __ldg(&vtab[g].z) : __ldg(counts + g); };

  if (warp < kProdWarps) {
    // ------------------------------------------------------------ cp.async producers
    // Stage = KS gathered k rows; warp w copies rows [RW w, RW (w + 1)). A row's k is warp-uniform:
    // each warp loads its RW slot indices with uniform (broadcast) vector loads two stages ahead into
    // fixed registers (three-way rotation: a register move of an index whose load is still pending
    // would stall the warp on it). B rows: 16-byte chunks across lanes (one 512-byte row per warp
    // instruction at N_TILE 256). A^T rows (GW * 2 bytes): A_RPW rows per instruction, the lane's k
    // picked from the uniform values by a compile-time select chain (no shuffles on the issue path).
    // Shared-memory addresses are swizzled in software to the UMMA SWIZZLE_{32,64,128}B layouts;
    // rows in [kvalid, kpad) are zero-filled (src size 0).
    int stage = 0;
    uint32_t phase = 0;
    struct Pos {
      int u, g, t, kb, cnt;  // unit, its group and n tile (tracked without division), chunk, count
      int b;                 // batch slice of the group (one division per unit, not per stage)
      int ncnt;              // count of the CTA's next unit, loaded one unit ahead of its use
      int rg, kbeg;          // kSplit: the virtual group's real group and first slot
    };
    const int step_t = static_cast<int>(gridDim.x) / n_vg;
    const int step_g = static_cast<int>(gridDim.x) % n_vg;
    auto next_unit = [&](Pos& q) {
      q.u += gridDim.x;
      q.g += step_g;
      q.t += step_t;
      if (q.g >= n_vg) {
        q.g -= n_vg;
        ++q.t;
      }
    };
    auto prefetch_next = [&](Pos& q) {
      int gn = q.g + step_g;
      if (gn >= n_vg) gn -= n_vg;
      q.ncnt = q.u + static_cast<int>(gridDim.x) < units ? vcount(gn) : 0;
    };
    auto locate = [&](Pos& q) {  // real group, first slot and batch slice of q's (virtual) group
      if constexpr (kSplit) {
        const int4 e = vunit(q.g);
        q.rg = e.x;
        q.kbeg = e.y;
        q.b = e.x / gpb;
      } else {
        q.b = q.g / gpb;
      }
    };
    auto advance = [&](Pos p) {
      Pos q = p;
      q.kb = p.kb + Cfg::KS;
      if (q.kb >= p.cnt) {
        q.kb = 0;
        next_unit(q);
        q.cnt = q.u < units ? p.ncnt : 0;  // prefetched: short units do not stall on the count
        while (q.u < units && q.cnt == 0) {
          next_unit(q);
          q.cnt = q.u < units ? vcount(q.g) : 0;
        }
        prefetch_next(q);
        if (q.u < units) locate(q);
      }
      return q;
    };
    constexpr int RW = Cfg::KS / kProdWarps;  // rows per warp per stage
    static_assert(RW % 8 == 0, "a warp's rows must cover whole swizzle phases");
    struct Idx {
      int v[RW];
    };
    const bool vec_idx = (slot_stride & 3) == 0 && (reinterpret_cast<uintptr_t>(slots) & 15) == 0;
    auto load_idx = [&](const Pos& p) {
      Idx x;
#pragma unroll
      for (int q = 0; q < RW; ++q) x.v[q] = 0;
      if (p.u < units) {
        const int r0 = p.kb + RW * warp;
        const int kbase = kSplit ? p.kbeg : 0;
        const int32_t* ps = slots + static_cast<int64_t>(kSplit ? p.rg : p.g) * slot_stride + kbase + r0;
        if (vec_idx && kbase + r0 + RW <= slot_stride) {  // in bounds; entries past cnt are masked by the copy
#pragma unroll
          for (int q = 0; q < RW / 4; ++q) {
            const int4 t = __ldg(reinterpret_cast<const int4*>(ps) + q);
            x.v[4 * q + 0] = t.x;
            x.v[4 * q + 1] = t.y;
            x.v[4 * q + 2] = t.z;
            x.v[4 * q + 3] = t.w;
          }
        } else {
#pragma unroll
          for (int q = 0; q < RW; ++q)
            if (r0 + q < p.cnt) x.v[q] = __ldg(ps + q);
        }
      }
      return x;
    };
    Pos cur{static_cast<int>(blockIdx.x), static_cast<int>(blockIdx.x) % n_vg,
            static_cast<int>(blockIdx.x) / n_vg, 0, 0, 0, 0, 0, 0};
    cur.cnt = cur.u < units ? vcount(cur.g) : 0;
    if (cur.u < units) locate(cur);
    prefetch_next(cur);
    if (cur.u < units && cur.cnt == 0) {
      cur.kb = Cfg::KS;  // force advance() past the empty unit
      cur = advance(cur);
    }
    using T = typename OT::T;
    const T* Bp = static_cast<const T*>(Bv);
    const T* Ap = static_cast<const T*>(Atv);
    const uint32_t ldb32 = static_cast<uint32_t>(ldb);  // host guarantees K * pitch < 2^32 elements
    const uint32_t lda32 = static_cast<uint32_t>(lda);
    const bool aligned8 = (N & 7) == 0 && (M & 7) == 0 && (grp_rows & 7) == 0;
    const uint32_t ldb_bytes = ldb32 * static_cast<uint32_t>(sizeof(T));  // K * pitch * 2 < 2^32 (host check)
    const uint32_t lda_bytes = lda32 * static_cast<uint32_t>(sizeof(T));
    // B: B_RPI rows per warp instruction (1 at N_TILE 256, 2 at 128, 4 at 64), lane -> (row sub, chunk)
    constexpr int B_RPI = Cfg::B_CPR >= 32 ? 1 : 32 / Cfg::B_CPR;
    constexpr int B_IPR = Cfg::B_CPR >= 32 ? Cfg::B_CPR / 32 : 1;  // instructions per row
    const int b_sub = B_RPI > 1 ? lane / Cfg::B_CPR : 0;
    // A^T: A_RPW rows per warp instruction, lane -> (row sub, chunk)
    const int a_sub = lane / Cfg::A_CPR;
    const int a_ch = lane % Cfg::A_CPR;
    const uint32_t a_base = static_cast<uint32_t>((a_ch / Cfg::A_CPA) * (Cfg::KS * Cfg::A_ROW_BYTES));
    auto issue = [&](const Pos& p, const Idx& x) {
      const int kvalid = min(Cfg::KS, p.cnt - p.kb);
      const int kpad = (kvalid + 15) & ~15;
      const int n0 = p.t * Cfg::N_TILE;
      const int m0 = (kSplit ? p.rg : p.g) * grp_rows;
      const int m_end = min(M, m0 + grp_rows);
      mbar_wait(&empty_bar[stage * kProdWarps + warp / WPG], phase ^ 1);
      const int r0 = RW * warp;
      // runs of consecutive k (block-structured masks, e.g. attention's 64-key blocks): the warp's RW
      // rows of A^T and of B are two-dimensional boxes, one TMA per 64-column atom, instead of RW
      // gathered 16-byte rows per lane (orientation N, full 128-row groups; tensor maps from the host)
      bool run = kOrientN && GW == 128 && runs && r0 + RW <= kvalid;
      if (run) {
#pragma unroll
        for (int i = 1; i < RW; ++i) run &= x.v[i] == x.v[0] + i;
      }
      if (run) {
        if (lane == 0) {
          uint8_t* sBp = smem + stage * Cfg::STAGE_BYTES;
          uint8_t* sAp = sBp + Cfg::B_BYTES;
          uint64_t* fb = &full_bar[stage * kProdWarps + warp / WPG];
          mbar_expect_tx_only(fb, static_cast<uint32_t>(RW * 128 * (Cfg::B_ATOMS + GW / 64)));
#pragma unroll
          for (int a = 0; a < Cfg::B_ATOMS; ++a)
            tma_load_2d(sBp + a * (Cfg::KS * 128) + r0 * 128, &tmBr, fb, n0 + a * 64, p.b * K + x.v[0]);
#pragma unroll
          for (int a = 0; a < GW / 64; ++a)
            tma_load_2d(sAp + a * (Cfg::KS * 128) + r0 * 128, &tmAt, fb, m0 + a * 64, x.v[0]);
        }
      } else if (r0 < kpad && aligned8) {
        // 16-byte chunks are whole or absent (N, M, group rows multiples of 8): ignore-src copies,
        // one predicate per copy — per B row one address multiply-add and the LDGSTS
        const uint32_t sB = smem_u32(smem + stage * Cfg::STAGE_BYTES);
        const uint32_t sA = sB + Cfg::B_BYTES;
        const bool all_rows = r0 + RW <= kvalid;  // every row of the warp live (all but a unit's last stage)
#pragma unroll
        for (int cb = 0; cb < B_IPR; ++cb) {
          const int ch = cb * 32 + (B_RPI > 1 ? lane % Cfg::B_CPR : lane);
          const int n = n0 + ch * 8;
          const bool n_ok = n < N;
          const T* bcol = Bp + p.b * b_batch_stride + (n_ok ? n : 0);
          const uint32_t cbase = sB + (ch >> 3) * (Cfg::KS * 128) + r0 * 128;
          if (B_RPI == 1 && all_rows) {
            // row 8a + r lands at cbase + 1024 a + t[r]: eight per-lane swizzled offsets, the rest
            // in the LDGSTS immediate; the source is one IMAD.WIDE per row
            uint32_t t[8];
#pragma unroll
            for (int r = 0; r < 8; ++r)
              t[r] = cbase + r * 128 + ((static_cast<uint32_t>(ch & 7) ^ static_cast<uint32_t>(r)) << 4);
#pragma unroll
            for (int i = 0; i < RW; ++i)
              cp_async_16_ign(t[i & 7] + (i >> 3) * 1024, row_addr(bcol, static_cast<uint32_t>(x.v[i]), ldb_bytes),
                              !n_ok);
            continue;
          }
#pragma unroll
          for (int i = 0; i < RW; i += B_RPI) {
            int kk = x.v[i];
#pragma unroll
            for (int r = 1; r < B_RPI; ++r) kk = b_sub == r ? x.v[i + r] : kk;
            const int row = i + b_sub;
            const bool ok = r0 + row < kvalid;
            cp_async_16_ign(cbase + row * 128 + ((static_cast<uint32_t>(ch & 7) ^ static_cast<uint32_t>(row & 7)) << 4),
                            row_addr(bcol, static_cast<uint32_t>(ok ? kk : 0), ldb_bytes), !(ok && n_ok));
          }
        }
        {
          const int m = m0 + a_ch * 8;
          const bool m_ok = m < m_end;
          const T* acol = Ap + (m_ok ? m : 0);
#pragma unroll
          for (int j = 0; j < RW; j += Cfg::A_RPW) {
            int kk = x.v[j];
#pragma unroll
            for (int r = 1; r < Cfg::A_RPW; ++r)
              if (j + r < RW) kk = a_sub == r ? x.v[j + r] : kk;
            if (Cfg::A_RPW > RW && a_sub >= RW) continue;
            const int row = r0 + j + a_sub;
            const bool ok = row < kvalid;
            const uint32_t o = static_cast<uint32_t>(row * Cfg::A_ROW_BYTES + (a_ch % Cfg::A_CPA) * 16);
            cp_async_16_ign(sA + a_base + swz<Cfg::A_MASK>(o), row_addr(acol, static_cast<uint32_t>(ok ? kk : 0), lda_bytes),
                            !(ok && m_ok));
          }
        }
      } else if (r0 < kpad) {  // a warp's RW rows are all below kpad or all above it
        const uint32_t sB = smem_u32(smem + stage * Cfg::STAGE_BYTES);
        const uint32_t sA = sB + Cfg::B_BYTES;
        // ---- B rows
#pragma unroll
        for (int cb = 0; cb < B_IPR; ++cb) {
          const int ch = cb * 32 + (B_RPI > 1 ? lane % Cfg::B_CPR : lane);
          const int n = n0 + ch * 8;
          const uint32_t nbytes = n < N ? static_cast<uint32_t>(min(16, (N - n) * 2)) : 0u;
          const T* bcol = Bp + p.b * b_batch_stride + (nbytes ? n : 0);
          const uint32_t cbase = sB + (ch >> 3) * (Cfg::KS * 128) + r0 * 128;
#pragma unroll
          for (int i = 0; i < RW; i += B_RPI) {
            int kk = x.v[i];
#pragma unroll
            for (int r = 1; r < B_RPI; ++r) kk = b_sub == r ? x.v[i + r] : kk;
            const int row = i + b_sub;  // within the warp's rows; (r0 + row) & 7 == row & 7
            const bool ok = r0 + row < kvalid;
            const uint32_t k = ok ? static_cast<uint32_t>(kk) : 0u;
            cp_async_16(cbase + row * 128 + ((static_cast<uint32_t>(ch & 7) ^ static_cast<uint32_t>(row & 7)) << 4),
                        bcol + k * ldb32, ok ? nbytes : 0u);
          }
        }
        // ---- A^T rows
        {
          const int m = m0 + a_ch * 8;
          const uint32_t mbytes = m < m_end ? static_cast<uint32_t>(min(16, (m_end - m) * 2)) : 0u;
          const T* acol = Ap + (mbytes ? m : 0);
#pragma unroll
          for (int j = 0; j < RW; j += Cfg::A_RPW) {
            int kk = x.v[j];
#pragma unroll
            for (int r = 1; r < Cfg::A_RPW; ++r)
              if (j + r < RW) kk = a_sub == r ? x.v[j + r] : kk;
            // A_RPW > RW (16-row groups at KS 64): lanes past the warp's rows idle
            if (Cfg::A_RPW > RW && a_sub >= RW) continue;
            const int row = r0 + j + a_sub;
            const bool ok = row < kvalid;
            const uint32_t k = ok ? static_cast<uint32_t>(kk) : 0u;
            const uint32_t o = static_cast<uint32_t>(row * Cfg::A_ROW_BYTES + (a_ch % Cfg::A_CPA) * 16);
            cp_async_16(sA + a_base + swz<Cfg::A_MASK>(o), acol + k * lda32, ok ? mbytes : 0u);
          }
        }
      }
      cp_async_arrive_noinc(&full_bar[stage * kProdWarps + warp / WPG]);
      if (++stage == Cfg::STAGES) {
        stage = 0;
        phase ^= 1;
      }
    };
    // D-way rotation: the slot indices of stage s + D - 1 load while stage s issues (fixed registers
    // per slot set; a register move of an index whose load is still pending would stall the warp).
    // This form (arrays, one unrolled loop) measured 342 -> 360 TFLOP/s on C1 32x1 against the
    // hand-rotated three-way code it replaced, same box; D = 4 / 5 / 6: 354 / 349 / 338
    // (scripts/gk_deep_ab.sh with PIT_GK_IDX_DEPTH builds).
    constexpr int D = kGkIdxDepth;
    Pos P[D];
    Idx X[D];
    P[0] = cur;
#pragma unroll
    for (int i = 1; i < D - 1; ++i) P[i] = advance(P[i - 1]);
#pragma unroll
    for (int i = 0; i < D - 1; ++i) X[i] = load_idx(P[i]);
    while (true) {
#pragma unroll
      for (int j = 0; j < D; ++j) {
        if (P[j].u >= units) goto producers_done;
        const int n = (j + D - 1) % D, pv = (j + D - 2) % D;
        P[n] = advance(P[pv]);
        X[n] = load_idx(P[n]);
        issue(P[j], X[j]);
      }
    }
  producers_done:;
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = kOrientN ? idesc_f16(128, Cfg::N_TILE, kBF16, true, true)
                                        : idesc_f16(128, GW, kBF16, true, true);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    const bool elected = lane == 0;
    const uint32_t sB0 = smem_u32(smem);
    const uint64_t a_desc0 = smem_desc(sB0 + Cfg::B_BYTES, Cfg::KS * Cfg::A_ROW_BYTES, 8 * Cfg::A_ROW_BYTES, Cfg::A_SW);
    const uint64_t b_desc0 = smem_desc(sB0, Cfg::KS * 128, 1024, kSw128);
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int cnt = vcount(u % n_vg);
      mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
      tc_fence_after();
      for (int kb = 0; kb < cnt; kb += Cfg::KS) {
        const int ksteps = (min(Cfg::KS, cnt - kb) + 15) >> 4;
        constexpr int KSG = Cfg::KS / 16 / BG;  // k-steps per barrier group
        // descriptors of this stage: the stage-0 descriptors plus the stage offset (>> 4, the start
        // address field; smem addresses < 256 KB never carry out of it); k-step / n-half offsets are
        // compile-time immediates
        const uint64_t soff = static_cast<uint64_t>((stage * Cfg::STAGE_BYTES) >> 4);
        const uint64_t dA = a_desc0 + soff, dB = b_desc0 + soff;
        const uint32_t dbase = tmem_base + static_cast<uint32_t>(acc * Cfg::ACC_COLS);
        // every group's barrier is waited in every stage (phases stay in lock step); MMAs only for
        // live k-steps; a group's slot is released after its last k-step
#pragma unroll
        for (int gi = 0; gi < BG; ++gi) {
          mbar_wait(&full_bar[stage * kProdWarps + gi], phase);
          fence_proxy_async_smem();  // cp.async (generic proxy) writes -> tcgen05.mma reads
          tc_fence_after();
          if (elected) {
#pragma unroll
            for (int j = 0; j < KSG; ++j) {
              const int ks = gi * KSG + j;
              if (ks < ksteps) {
                const uint32_t acc_flag = (kb > 0 || ks > 0) ? 1u : 0u;
                const uint64_t a_strip = dA + static_cast<uint64_t>((ks * 16 * Cfg::A_ROW_BYTES) >> 4);
                if constexpr (kOrientN) {
                  umma_f16(dbase, a_strip, dB + static_cast<uint64_t>((ks * 2048) >> 4), idesc, acc_flag);
                } else {
#pragma unroll
                  for (int a = 0; a < Cfg::N_TILE / 128; ++a)
                    umma_f16(dbase + static_cast<uint32_t>(a * GW),
                             dB + static_cast<uint64_t>((a * 2 * Cfg::KS * 128 + ks * 2048) >> 4), a_strip, idesc,
                             acc_flag);
                }
              }
            }
            umma_commit(&empty_bar[stage * kProdWarps + gi]);
          }
          __syncwarp();
        }
        if (++stage == Cfg::STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (lane == 0) umma_commit(&tfull_bar[acc]);
      __syncwarp();
      if (++acc == Cfg::NBUF) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  } else if (warp >= kEpiWarp0) {
    // ------------------------------------------------------------ epilogue
    using T = typename OT::T;
    T* C = static_cast<T*>(Cv);
    const int q = warp & 3;  // TMEM lane quarter
    const uint32_t stg_w = smem_u32(stg) + static_cast<uint32_t>(q * 2 * 4096);
    int sbuf = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      int g = u % n_vg;
      const int t = u / n_vg;
      const int n0 = t * Cfg::N_TILE;
      int cnt, part = -1;
      if constexpr (kSplit) {
        const int4 e = vunit(g);
        g = e.x;
        cnt = e.z;
        part = e.w;  // -1, or first partial tile | chunk << 8 | split group << 16 | chunks << 24
      } else {
        cnt = __ldg(counts + g);
      }
      const int m0 = g * grp_rows;
      const int m_end = min(M, m0 + grp_rows);
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const uint32_t tbase = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * Cfg::ACC_COLS);
      if (kSplit && part >= 0) {
        // a chunk of a split group: its fp32 partial tile [128 rows x N_TILE] (lane = row) goes to
        // scratch (a chunk always has live k). The chunk that completes its group last (counter in
        // scratch, zeroed before the launch) sums every chunk's tile into C.
        const int row = q * 32 + lane;
        const int p0 = part & 255, ch = (part >> 8) & 255, sg = (part >> 16) & 255, nch = part >> 24;
        float* wrow = ws + static_cast<int64_t>(p0 + ch) * 128 * Cfg::N_TILE + row * Cfg::N_TILE;
#pragma unroll 1
        for (int c = 0; c < Cfg::N_TILE; c += 32) {
          uint32_t v[32];
          tmem_ld32(tbase + static_cast<uint32_t>(c), v);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 8; ++j)
            reinterpret_cast<float4*>(wrow + c)[j] = make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                                                                 __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3]));
        }
        if (!(use_tma_store & 8)) {
        __threadfence();
        bar_sync_named(3, 128);  // the 4 epilogue warps
        if (row == 0) s_last = atomicAdd(split_ctr + sg, 1) == nch - 1;
        bar_sync_named(3, 128);
        }
        if (s_last && !(use_tma_store & 12)) {
          __threadfence();
          // coalesced: thread t sums float4 t, t + 128, ... of the tile over the group's chunks
          // (partial tiles p0 .. p0 + nch - 1), then writes 4 bf16 columns of one C row
          constexpr int F4 = 128 * Cfg::N_TILE / 4, PER = F4 / 128, C4 = Cfg::N_TILE / 4;
          float4 acc[PER];
#pragma unroll
          for (int j = 0; j < PER; ++j) acc[j] = make_float4(0.f, 0.f, 0.f, 0.f);
          const float4* t4 = reinterpret_cast<const float4*>(ws + static_cast<int64_t>(p0) * 128 * Cfg::N_TILE);
#pragma unroll 1
          for (int h = 0; h < nch; ++h) {
            float4 v4[PER];
#pragma unroll
            for (int j = 0; j < PER; ++j) v4[j] = __ldcg(t4 + static_cast<int64_t>(h) * F4 + row + 128 * j);
#pragma unroll
            for (int j = 0; j < PER; ++j) {
              acc[j].x += v4[j].x; acc[j].y += v4[j].y; acc[j].z += v4[j].z; acc[j].w += v4[j].w;
            }
          }
#pragma unroll
          for (int j = 0; j < PER; ++j) {
            const int e = row + 128 * j;
            const int m = m0 + e / C4, n = n0 + (e % C4) * 4;
            if (m >= m_end || n >= N) continue;
            T* dst = C + static_cast<int64_t>(m) * ldc + n;
            if (n + 4 <= N && (ldc % 4) == 0 && (reinterpret_cast<uintptr_t>(Cv) & 7) == 0) {
              *reinterpret_cast<uint2*>(dst) = make_uint2(pack2(acc[j].x, acc[j].y, kBF16), pack2(acc[j].z, acc[j].w, kBF16));
            } else {
              const float f[4] = {acc[j].x, acc[j].y, acc[j].z, acc[j].w};
              for (int i = 0; i < 4 && n + i < N; ++i) dst[i] = OT::cvt(f[i]);
            }
          }
        }
      } else if (kOrientN && (use_tma_store & 1)) {
        // lane = group row: 32-row x 64-column boxes through shared staging and TMA stores
        const int wrow0 = m0 + q * 32;
#pragma unroll 1
        for (int bx = 0; bx < Cfg::N_TILE / 64; ++bx) {
          epi_box_tma<kBF16>(tbase + static_cast<uint32_t>(bx * 64), cnt > 0, stg_w + static_cast<uint32_t>(sbuf * 4096),
                             &tmC, wrow0 < m_end && n0 + bx * 64 < N, n0 + bx * 64, wrow0, lane);
          sbuf ^= 1;
        }
      } else if constexpr (kOrientN) {
        // lane = group row, columns = n: 32 consecutive outputs per tcgen05.ld
        const int m = m0 + q * 32 + lane;
        const bool row_ok = m < m_end;
        uint8_t* crow = reinterpret_cast<uint8_t*>(C + static_cast<int64_t>(row_ok ? m : 0) * ldc);
        const bool vec_ok = (ldc % 8) == 0 && (reinterpret_cast<uintptr_t>(Cv) & 15) == 0;
#pragma unroll 1
        for (int c = 0; c < Cfg::N_TILE; c += 32) {
          uint32_t v[32];
          if (cnt > 0) {
            tmem_ld32(tbase + static_cast<uint32_t>(c), v);
            tmem_wait_ld();
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = 0u;
          }
          const int nb = n0 + c;
          if (row_ok && nb < N) {
            if (vec_ok && nb + 32 <= N) {
              uint4* dst = reinterpret_cast<uint4*>(crow + static_cast<int64_t>(nb) * 2);
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                uint4 w;
                w.x = pack2(__uint_as_float(v[8 * j + 0]), __uint_as_float(v[8 * j + 1]), kBF16);
                w.y = pack2(__uint_as_float(v[8 * j + 2]), __uint_as_float(v[8 * j + 3]), kBF16);
                w.z = pack2(__uint_as_float(v[8 * j + 4]), __uint_as_float(v[8 * j + 5]), kBF16);
                w.w = pack2(__uint_as_float(v[8 * j + 6]), __uint_as_float(v[8 * j + 7]), kBF16);
                dst[j] = w;
              }
            } else {
              T* dst = reinterpret_cast<T*>(crow);
              for (int j = 0; j < 32; ++j)
                if (nb + j < N) dst[nb + j] = OT::cvt(__uint_as_float(v[j]));
            }
          }
        }
      } else if (!kOrientN && Cfg::STG_T > 0 && (use_tma_store & 1)) {
        // lane = output column n, TMEM columns = group rows: 2-byte shared stores build the warp's
        // [grp_rows x 32 columns] box (64-byte rows, conflict-free), one TMA store writes it
        const uint32_t buf = smem_u32(stg) + static_cast<uint32_t>(q * Cfg::STG_T);
#pragma unroll 1
        for (int a = 0; a < Cfg::N_TILE / 128; ++a) {
          const int ncol0 = n0 + a * 128 + q * 32;
          if (lane == 0) bulk_wait_read<0>();
          __syncwarp();
#pragma unroll
          for (int c = 0; c < GW; c += 16) {
            uint32_t v[16];
            if (cnt > 0) {
              tmem_ld16(tbase + static_cast<uint32_t>(a * GW + c), v);
              tmem_wait_ld();
            } else {
#pragma unroll
              for (int i = 0; i < 16; ++i) v[i] = 0u;
            }
#pragma unroll
            for (int i = 0; i < 16; i += 2) {
              // rows c+i and c+i+1 of this column: one 2-byte store each
              const T h0 = OT::cvt(__uint_as_float(v[i])), h1 = OT::cvt(__uint_as_float(v[i + 1]));
              if (c + i < grp_rows)
                asm volatile("st.shared.b16 [%0], %1;" ::"r"(buf + (c + i) * 64 + lane * 2),
                             "h"(*reinterpret_cast<const uint16_t*>(&h0)) : "memory");
              if (c + i + 1 < grp_rows)
                asm volatile("st.shared.b16 [%0], %1;" ::"r"(buf + (c + i + 1) * 64 + lane * 2),
                             "h"(*reinterpret_cast<const uint16_t*>(&h1)) : "memory");
            }
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0 && ncol0 < N) {
            tma_store_2d(&tmC, buf, ncol0, m0);
            bulk_commit();
          }
        }
      } else {
        // lane = output column n, columns = group rows
#pragma unroll
        for (int a = 0; a < Cfg::N_TILE / 128; ++a) {
          const int n = n0 + a * 128 + q * 32 + lane;
#pragma unroll
          for (int c = 0; c < GW; c += 16) {
            uint32_t v[16];
            if (cnt > 0) {
              tmem_ld16(tbase + static_cast<uint32_t>(a * GW + c), v);
              tmem_wait_ld();
            } else {
#pragma unroll
              for (int i = 0; i < 16; ++i) v[i] = 0u;
            }
            if (n < N && !(use_tma_store & 2)) {
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                const int m = m0 + c + i;
                if (m < m_end) C[static_cast<int64_t>(m) * ldc + n] = OT::cvt(__uint_as_float(v[i]));
              }
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty_bar[acc]);
      if (++acc == Cfg::NBUF) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if ((use_tma_store & 1) && lane == 0) bulk_wait<0>();  // staging outlives its stores
  }

  tc_fence_before();
  __syncthreads();
  if (warp == kAllocWarp) {
    tc_fence_after();
    tmem_dealloc<Cfg::TMEM_COLS>(tmem_base);
  }
}

// =============================================================================================
// spmm_gk2: PIT axis k with 256-row groups on a CTA pair (tcgen05 cta_group::2).
//
// The pair computes one (group, 256-column n tile) unit as D[256 m, 256 n] += A[m, k] * B[k, n]
// over the group's live k: CTA r gathers, per live k, the 128 A^T values of its m half and the 128
// B values of its n half (one 512-byte warp instruction per k row: lanes 0-15 A, 16-31 B). Every
// gathered B byte then serves 256 output rows, 128 FLOP per gathered byte against 85 for a
// single-CTA 128-row group — the L2->SM gather feed, not the tensor pipe, is what bounds PIT's
// gathered-K product (K2).
// Pipeline: producers arrive on a local full barrier (cp.async.mbarrier.arrive.noinc); a relay
// thread per CTA waits on it, fences the generic->async proxy and arrives on the even CTA's pair
// barrier; the even CTA's MMA thread issues the pair MMA and multicasts its commits to both CTAs'
// empty / TMEM-full barriers; each CTA drains its own 128 TMEM lanes and arrives remotely on the
// even CTA's TMEM-empty barrier.
// =============================================================================================
template <int kKS>
struct Gk2Cfg {
  static constexpr int KS = kKS;
  static constexpr int N_TILE = 256;
  static constexpr int OP_BYTES = KS * 256;  // one operand half: 2 swizzle atoms x KS rows x 128 B
  static constexpr int STAGE_BYTES = 2 * OP_BYTES;
  static constexpr int STAGES = (208 * 1024) / STAGE_BYTES > 12 ? 12 : (208 * 1024) / STAGE_BYTES;
  static constexpr int NBUF = 2;
  static constexpr int ACC_COLS = 256;
  static constexpr int TMEM_COLS = 512;
  // epilogue staging for TMA stores: per epilogue warp two 32-row x 64-column bf16 boxes (4 KB each)
  static constexpr int STG_BYTES = 4 * 2 * 4096;
  static constexpr size_t SMEM = static_cast<size_t>(STAGES) * STAGE_BYTES + STG_BYTES + 1024 + 1024;
};
constexpr int kRelayWarp = 10;
// Diagnostics (compiled in with -DPIT_DIAG=1 only: `PIT_DIAG=1 python -m paper_2301_10936_b200._build
// --force`): PIT_GK2_DIAG bits 0-2 drop the MMAs / copies / C stores of spmm_gk2, bit 4 records its
// stage timeline (globaltimer stamps of pair 0's first 128 stages, scripts/gk2_trace.py).
#ifndef PIT_DIAG
#define PIT_DIAG 0
#endif
__device__ unsigned long long g_gk2_trace[8 * 128];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <bool kBF16, int kKS>
__global__ void __launch_bounds__(kThreads, 1)
    spmm_gk2_kernel(const __grid_constant__ CUtensorMap tmC, int use_tma_store, const void* __restrict__ Bv, int64_t ldb, const void* __restrict__ Atv, int64_t lda,
                    const int32_t* __restrict__ counts, const int32_t* __restrict__ slots, int64_t slot_stride,
                    int n_groups, int n_tiles, int M, int N, void* __restrict__ Cv, int64_t ldc, int grp_rows,
                    int gpb, int64_t b_batch_stride, int diag) {
  using Cfg = Gk2Cfg<kKS>;
  using OT = OutT<kBF16>;
  using T = typename OT::T;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stg = smem + Cfg::STAGES * Cfg::STAGE_BYTES;  // epilogue staging (1024-aligned boxes)
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(stg + Cfg::STG_BYTES);
  uint64_t* pair_full = full_bar + Cfg::STAGES;  // even CTA: both halves of a stage landed
  uint64_t* empty_bar = pair_full + Cfg::STAGES;
  uint64_t* tfull_bar = empty_bar + Cfg::STAGES;
  uint64_t* tempty_bar = tfull_bar + Cfg::NBUF;  // even CTA: both CTAs drained the accumulator
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + Cfg::NBUF);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int pair = static_cast<int>(blockIdx.x >> 1);
  const int npairs = static_cast<int>(gridDim.x >> 1);

  if (threadIdx.x == 0) {
    for (int i = 0; i < Cfg::STAGES; ++i) {
      mbar_init(&full_bar[i], kProdThreads);
      mbar_init(&pair_full[i], 2);
      mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < Cfg::NBUF; ++i) {
      mbar_init(&tfull_bar[i], 1);
      mbar_init(&tempty_bar[i], 8);  // 4 epilogue warps x 2 CTAs
    }
    fence_mbar_init();
  }
  if (warp == kAlloc2Warp) tmem_alloc2<Cfg::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int units = n_groups * n_tiles;

  if (warp < kProdWarps) {
    // ------------------------------------------------------------ cp.async producers
    int stage = 0;
    uint32_t phase = 0;
    struct Pos {
      int u, g, t, kb, cnt, b, ncnt;
    };
    const int step_t = npairs / n_groups;
    const int step_g = npairs % n_groups;
    auto next_unit = [&](Pos& q) {
      q.u += npairs;
      q.g += step_g;
      q.t += step_t;
      if (q.g >= n_groups) {
        q.g -= n_groups;
        ++q.t;
      }
    };
    auto prefetch_next = [&](Pos& q) {
      int gn = q.g + step_g;
      if (gn >= n_groups) gn -= n_groups;
      q.ncnt = q.u + npairs < units ? __ldg(counts + gn) : 0;
    };
    auto advance = [&](Pos p) {
      Pos q = p;
      q.kb = p.kb + Cfg::KS;
      if (q.kb >= p.cnt) {
        q.kb = 0;
        next_unit(q);
        q.cnt = q.u < units ? p.ncnt : 0;
        while (q.u < units && q.cnt == 0) {
          next_unit(q);
          q.cnt = q.u < units ? __ldg(counts + q.g) : 0;
        }
        prefetch_next(q);
        q.b = q.g / gpb;
      }
      return q;
    };
    // warp w copies the stage's rows [RW w, RW (w + 1)): the row's k is warp-uniform, so each warp
    // loads its RW slot indices with uniform (broadcast) vector loads one stage ahead — no shuffles
    // on the issue path, and every cp.async depends only on a register loaded long before.
    constexpr int RW = Cfg::KS / kProdWarps;
    static_assert(RW % 8 == 0, "rows per warp must cover whole swizzle phases");
    struct Idx {
      int v[RW];
    };
    const bool vec_idx = (slot_stride & 3) == 0 && (reinterpret_cast<uintptr_t>(slots) & 15) == 0;
    auto load_idx = [&](const Pos& p) {
      Idx x;
#pragma unroll
      for (int q = 0; q < RW; ++q) x.v[q] = 0;
      if (p.u < units) {
        const int r0 = p.kb + RW * warp;
        const int32_t* ps = slots + static_cast<int64_t>(p.g) * slot_stride + r0;
        if (vec_idx && r0 + RW <= slot_stride) {  // in bounds; entries past cnt are masked by the copy
#pragma unroll
          for (int q = 0; q < RW / 4; ++q) {
            const int4 t = __ldg(reinterpret_cast<const int4*>(ps) + q);
            x.v[4 * q + 0] = t.x;
            x.v[4 * q + 1] = t.y;
            x.v[4 * q + 2] = t.z;
            x.v[4 * q + 3] = t.w;
          }
        } else {
#pragma unroll
          for (int q = 0; q < RW; ++q)
            if (r0 + q < p.cnt) x.v[q] = __ldg(ps + q);
        }
      }
      return x;
    };
    Pos cur{pair, pair % n_groups, pair / n_groups, 0, 0, 0, 0};
    cur.cnt = cur.u < units ? __ldg(counts + cur.g) : 0;
    cur.b = cur.g / gpb;
    prefetch_next(cur);
    if (cur.u < units && cur.cnt == 0) {
      cur.kb = Cfg::KS;
      cur = advance(cur);
    }
    // lane roles: lanes 0-15 copy the A^T half (m), lanes 16-31 the B half (n); chunk c = 8 elements
    const bool is_a = lane < 16;
    const int c = lane & 15;
    const uint32_t pitch = static_cast<uint32_t>(is_a ? lda : ldb);  // host: K * pitch < 2^32
    const uint32_t lane_off = (is_a ? 0u : static_cast<uint32_t>(Cfg::OP_BYTES)) +
                              static_cast<uint32_t>((c >> 3) * (Cfg::KS * 128) + warp * RW * 128);
    const uint32_t cc = static_cast<uint32_t>(c & 7);
    int trace_j = 0;
    auto issue = [&](const Pos& p, const Idx& x) {
      const int kvalid = min(Cfg::KS, p.cnt - p.kb);
      const int kpad = (kvalid + 15) & ~15;
      const int m0 = p.g * grp_rows;
      const int m_end = min(M, m0 + grp_rows);
      const T* src;
      uint32_t nbytes;
      if (is_a) {
        const int m = m0 + 128 * static_cast<int>(rank) + 8 * c;
        nbytes = m < m_end ? static_cast<uint32_t>(min(16, (m_end - m) * 2)) : 0u;
        src = static_cast<const T*>(Atv) + (nbytes ? m : 0);
      } else {
        const int n = p.t * Cfg::N_TILE + 128 * static_cast<int>(rank) + 8 * c;
        nbytes = n < N ? static_cast<uint32_t>(min(16, (N - n) * 2)) : 0u;
        src = static_cast<const T*>(Bv) + p.b * b_batch_stride + (nbytes ? n : 0);
      }
      mbar_wait(&empty_bar[stage], phase ^ 1);
      if ((PIT_DIAG && (diag & 16)) && pair == 0 && threadIdx.x == 0 && trace_j < 128) g_gk2_trace[rank * 128 + trace_j] = gtimer();
      ++trace_j;
      // rows [kvalid, kpad) are zero-filled; a warp's RW rows are all below kpad or all above it
      const int r0 = RW * warp;
      if (r0 < kpad && !(PIT_DIAG && (diag & 2))) {
        const uint32_t dst = smem_u32(smem + stage * Cfg::STAGE_BYTES) + lane_off;
#pragma unroll
        for (int i = 0; i < RW; ++i) {
          const bool ok = r0 + i < kvalid;
          const uint32_t k = ok ? static_cast<uint32_t>(x.v[i]) : 0u;
          cp_async_16(dst + i * 128 + ((cc ^ static_cast<uint32_t>(i & 7)) << 4), src + k * pitch, ok ? nbytes : 0u);
        }
      }
      cp_async_arrive_noinc(&full_bar[stage]);
      if (++stage == Cfg::STAGES) {
        stage = 0;
        phase ^= 1;
      }
    };
    // Three stages in flight with fixed register roles (no loop-carried copies: a register move of
    // an index whose load is still pending would stall the warp on it, defeating the prefetch).
#ifdef PIT_GK2_HAND
    Pos P0 = cur, P1 = advance(P0), P2;
    Idx X0 = load_idx(P0), X1 = load_idx(P1), X2;
    while (true) {
      if (P0.u >= units) break;
      P2 = advance(P1);
      X2 = load_idx(P2);
      issue(P0, X0);
      if (P1.u >= units) break;
      P0 = advance(P2);
      X0 = load_idx(P0);
      issue(P1, X1);
      if (P2.u >= units) break;
      P1 = advance(P0);
      X1 = load_idx(P1);
      issue(P2, X2);
    }
#else
    constexpr int D = kGkIdxDepth;  // the spmm_gk rotation (arrays, one unrolled loop)
    Pos P[D];
    Idx X[D];
    P[0] = cur;
#pragma unroll
    for (int i = 1; i < D - 1; ++i) P[i] = advance(P[i - 1]);
#pragma unroll
    for (int i = 0; i < D - 1; ++i) X[i] = load_idx(P[i]);
    while (true) {
#pragma unroll
      for (int j = 0; j < D; ++j) {
        if (P[j].u >= units) goto producers_done;
        const int n = (j + D - 1) % D, pv = (j + D - 2) % D;
        P[n] = advance(P[pv]);
        X[n] = load_idx(P[n]);
        issue(P[j], X[j]);
      }
    }
  producers_done:;
#endif
  } else if (warp == kRelayWarp) {
    // ------------------------------------------------------------ relay: local full -> pair full
    if (lane == 0) {
      const uint32_t leader_pf = mapa_shared(smem_u32(pair_full), 0);
      int tj = 0;
      int stage = 0;
      uint32_t phase = 0;
      for (int u = pair; u < units; u += npairs) {
        const int cnt = __ldg(counts + u % n_groups);
        for (int kb = 0; kb < cnt; kb += Cfg::KS) {
          mbar_wait(&full_bar[stage], phase);
          if ((PIT_DIAG && (diag & 16)) && pair == 0 && tj < 128) g_gk2_trace[(2 + rank) * 128 + tj] = gtimer();
          ++tj;
          fence_proxy_async_smem();  // cp.async (generic proxy) writes -> tcgen05.mma reads
          mbar_arrive_cluster(leader_pf + stage * 8);
          if (++stage == Cfg::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer (even CTA)
    if (rank == 0) {
      constexpr uint32_t idesc = idesc_f16(256, Cfg::N_TILE, kBF16, true, true);
      int tj = 0;
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int u = pair; u < units; u += npairs) {
        const int cnt = __ldg(counts + u % n_groups);
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        for (int kb = 0; kb < cnt; kb += Cfg::KS) {
          const int ksteps = (min(Cfg::KS, cnt - kb) + 15) >> 4;
          mbar_wait(&pair_full[stage], phase);
          tc_fence_after();
          if ((PIT_DIAG && (diag & 16)) && pair == 0 && lane == 0 && tj < 128) g_gk2_trace[4 * 128 + tj] = gtimer();
          if (lane == 0) {
            const uint32_t sA = smem_u32(smem + stage * Cfg::STAGE_BYTES);
            const uint32_t sB = sA + Cfg::OP_BYTES;
            const uint32_t d = tmem_base + static_cast<uint32_t>(acc * Cfg::ACC_COLS);
            for (int ks = 0; ks < ((PIT_DIAG && (diag & 1)) ? 0 : ksteps); ++ks) {
              const uint64_t adesc = smem_desc(sA + ks * 2048, Cfg::KS * 128, 1024, kSw128);
              const uint64_t bdesc = smem_desc(sB + ks * 2048, Cfg::KS * 128, 1024, kSw128);
              umma2_f16(d, adesc, bdesc, idesc, (kb > 0 || ks > 0) ? 1u : 0u);
            }
            umma2_commit_mc(&empty_bar[stage], 3);
            if ((PIT_DIAG && (diag & 16)) && pair == 0 && tj < 128) g_gk2_trace[5 * 128 + tj] = gtimer();
          }
          ++tj;
          __syncwarp();
          if (++stage == Cfg::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (lane == 0) umma2_commit_mc(&tfull_bar[acc], 3);
        __syncwarp();
        if (++acc == Cfg::NBUF) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= kEpiWarp0) {
    // ------------------------------------------------------------ epilogue (each CTA: its 128 rows)
    // TMEM -> registers -> bf16 -> swizzled shared staging -> TMA tile store (whole 128-byte lines,
    // asynchronous). Per-thread row stores (16 bytes at a 2*ldc stride per lane) clogged the LSU the
    // producers' gathers share and stretched the copies in flight at every unit boundary.
    T* C = static_cast<T*>(Cv);
    const int q = warp & 3;
    const uint32_t leader_te = mapa_shared(smem_u32(tempty_bar), 0);
    const bool vec_ok = (ldc % 8) == 0 && (reinterpret_cast<uintptr_t>(Cv) & 15) == 0;
    const uint32_t stg_w = smem_u32(stg) + static_cast<uint32_t>(q * 2 * 4096);
    int sbuf = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = pair; u < units; u += npairs) {
      const int g = u % n_groups;
      const int n0 = (u / n_groups) * Cfg::N_TILE;
      const int m0 = g * grp_rows;
      const int m_end = min(M, m0 + grp_rows);
      const int cnt = __ldg(counts + g);
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const uint32_t tbase = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * Cfg::ACC_COLS);
      const int wrow0 = m0 + 128 * static_cast<int>(rank) + q * 32;  // the warp's first output row
      const int m = wrow0 + lane;
      const bool row_ok = m < m_end;
      if (use_tma_store) {
        // grp_rows % 32 == 0 (host): a warp's 32 rows are all inside the group or all outside it
        const bool warp_rows = wrow0 < m_end;
#pragma unroll 1
        for (int bx = 0; bx < Cfg::N_TILE / 64; ++bx) {
          epi_box_tma<kBF16>(tbase + static_cast<uint32_t>(bx * 64), cnt > 0, stg_w + static_cast<uint32_t>(sbuf * 4096),
                             &tmC, warp_rows && n0 + bx * 64 < N, n0 + bx * 64, wrow0, lane);
          sbuf ^= 1;
        }
      } else {
        uint8_t* crow = reinterpret_cast<uint8_t*>(C + static_cast<int64_t>(row_ok ? m : 0) * ldc);
#pragma unroll 1
        for (int cc = 0; cc < Cfg::N_TILE; cc += 32) {
          uint32_t v[32];
          if (cnt > 0) {
            tmem_ld32(tbase + static_cast<uint32_t>(cc), v);
            tmem_wait_ld();
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = 0u;
          }
          const int nb = n0 + cc;
          if (row_ok && nb < N && !(PIT_DIAG && (diag & 4))) {
            if (vec_ok && nb + 32 <= N) {
              uint4* dstp = reinterpret_cast<uint4*>(crow + static_cast<int64_t>(nb) * 2);
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                uint4 w;
                w.x = pack2(__uint_as_float(v[8 * j + 0]), __uint_as_float(v[8 * j + 1]), kBF16);
                w.y = pack2(__uint_as_float(v[8 * j + 2]), __uint_as_float(v[8 * j + 3]), kBF16);
                w.z = pack2(__uint_as_float(v[8 * j + 4]), __uint_as_float(v[8 * j + 5]), kBF16);
                w.w = pack2(__uint_as_float(v[8 * j + 6]), __uint_as_float(v[8 * j + 7]), kBF16);
                dstp[j] = w;
              }
            } else {
              T* dstp = reinterpret_cast<T*>(crow);
              for (int j = 0; j < 32; ++j)
                if (nb + j < N) dstp[nb + j] = OT::cvt(__uint_as_float(v[j]));
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(leader_te + acc * 8);
      if (++acc == Cfg::NBUF) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if (lane == 0) bulk_wait<0>();  // staging must outlive every store that reads it
  }

  tc_fence_before();
  cluster_sync();
  if (warp == kAlloc2Warp) {
    tc_fence_after();
    tmem_dealloc2<Cfg::TMEM_COLS>(tmem_base);
  }
}

// =============================================================================================
// rowgemm ("gathered M"): PIT axis m, the dense plan, and grouped / MoE expert GEMMs.
//
// G groups; group g owns rows_g rows, tiled 128 at a time. Row i of group g reads A row
//   src(g,i) = row_src ? row_src[g*src_stride + i] : off[g] + i
// and writes C row
//   dst(g,i) = row_dst ? row_dst[g*dst_stride + i] : off[g] + i,
// against B_g = rows [g*K, (g+1)*K) of a stacked [G*K, N] matrix (3-D tensor map, so K tails stay
// inside the group). Optional per-(row, K-block) liveness (pit:m occupancy bitmap, G == 1) zero-fills
// dead rows and skips K-blocks with no live row. Epilogue: optional ReLU, optional per-C-row scale.
// With G == 1 and off == nullptr the row count comes from *n_rows (pit:m union) or is M (dense).
// =============================================================================================
struct RowGemmParams {
  const void* A;
  int64_t lda;
  void* C;
  int64_t ldc;
  int M, N, K;  // M: rows of A (bounds) ; N, K: GEMM extents per group
  int G;
  const int32_t* cnt;       // [G] rows per group (nullptr: single group, see n_rows)
  const int32_t* off;       // [G+1] packed row offsets
  const int32_t* tile_off;  // [G+1] prefix of ceil(cnt/128)
  const int32_t* n_rows;    // single group: device row count (nullptr: dense, M rows)
  const int32_t* row_src;
  int64_t src_stride;
  const int32_t* row_dst;
  int64_t dst_stride;
  const float* row_scale;   // indexed by C row
  int act;                  // 0 none, 1 relu
  const uint32_t* occ;      // liveness bitmap [K/t1 groups][WG words over source rows] or nullptr
  int64_t WG;
  int t1;
  int max_tiles;            // host bound on the total number of row tiles
  int uniform_rows;         // cnt == nullptr && G > 1: every group is this many consecutive rows
  int a_tma;                // A tiles by TMA (rows contiguous: no row_src, no liveness); else cp.async
  int contig_pct;           // > 0 (single group, union rows): contiguous row tiles when *n_rows >= pct% of M
  int exit_if_contig;       // rowgemm: leave the contiguous case to the rowgemm2 launched beside it
  int masked;               // rowgemm2: contiguous 128-row halves, per-chunk liveness from occ; runs only
                            // when the union holds >= contig_pct% of the rows
  const int32_t* kg_cnt;    // masked: live rows per K-group (the pit:m index counts)
  int mask_tma;             // rowgemm, staged contiguous rows: A tiles by TMA + dead micro-tiles zeroed
  int a_rows;               // rows of A when it is not M (packed live rows); 0: M
  int epi8;                 // rowgemm2: 8 epilogue warps when the producer warps 4-7 are idle
  int lagged;               // rowgemm2: per-warp cp.async arrivals kLag stages behind (A/B knob)
  float* part;              // rowgemm2t: fp32 partial rows (row off[g] + token, pitch N) instead of C
  int x_stride;             // rowgemm2t: packed token rows of group g start at g * x_stride (0: off[g])
  const int* path_flag;     // device flag of the high-sparsity pit:m path (pit_gm_sparse.cu): the
  int path_role;            // kernel runs only if the flag is set (1) / clear (2); 0: always
  const uint32_t* zero_occ; // rowgemm2, one-K-group pit:m: live-row bitmap; its dead C rows [0, M) are
                            // cleared by the otherwise idle warps 9 and 11 (no separate clearing launch)
};

// The high-sparsity pit:m path and the masked dense kernels are launched together; each leaves unless
// the flag the sparse path's prep kernel wrote selects it.
__device__ __forceinline__ bool path_skip(const RowGemmParams& p) {
  return p.path_flag != nullptr && ((*p.path_flag != 0) != (p.path_role == 1));
}

template <int KS, int kBN = 256>
struct GmCfg {
  static constexpr int BM = 128;
  static constexpr int BN = kBN;  // 256, or 64 for narrow products (attention P.V)
  static constexpr int A_ROW_BYTES = KS * 2;  // K-major rows
  static constexpr int A_BYTES = BM * A_ROW_BYTES;
  static constexpr int B_BYTES = (BN / 64) * KS * 128;  // MN-major, 4 atoms of 64 n
  static constexpr int STAGE_BYTES = ((A_BYTES + B_BYTES + 1023) / 1024) * 1024;
  // epilogue staging: one 32-row x 64-column box (4 KB) per epilogue warp
  static constexpr int STG_BYTES = 4 * 4096;
  static constexpr int STATIC_SMEM = 512 * 5 * 4 + 1024 / 8;  // tile_occ + kb_live below
  static constexpr int STAGE_BUDGET = 232448 - 2048 - STG_BYTES - STATIC_SMEM;
  static constexpr int STAGES = STAGE_BUDGET / STAGE_BYTES > 8 ? 8 : STAGE_BUDGET / STAGE_BYTES;
  static constexpr int TMEM_COLS = tmem_cols_pow2<2 * BN>();  // 2 accumulators
  // occupancy words of the current row tile for every K-group (contiguous-row units): 5 words per
  // group cover 128 rows at any 32-row alignment
  static constexpr int OCC_MAX_GROUPS = 512;   // static shared: 5 words per K-group
  static constexpr int KB_MAX = 1024;          // static shared: live-K-block bitmask
  static constexpr size_t SMEM = static_cast<size_t>(STAGES) * STAGE_BYTES + STG_BYTES + 2048;
  static_assert(SMEM + STATIC_SMEM <= 232448, "shared memory over the sm_100 opt-in limit");
  static constexpr uint32_t A_SW = sw_layout_for_row(A_ROW_BYTES);
};

struct RowTile {
  int g, base, rows;  // group, packed offset of the tile's first row, rows in the tile (<= 128)
};

// Decode row tile t (global index) -> group and rows. Identical in every role.
__device__ __forceinline__ RowTile decode_tile(const RowGemmParams& p, int t, int single_rows) {
  if (p.cnt == nullptr) {
    if (p.uniform_rows) {  // batched slices of equal height, stacked along M
      const int tpg = (p.uniform_rows + 127) >> 7;
      const int g = t / tpg, start = (t - g * tpg) * 128;
      return {g, g * p.uniform_rows + start, min(128, p.uniform_rows - start)};
    }
    const int base = t * 128;
    return {0, base, min(128, single_rows - base)};
  }
  int lo = 0, hi = p.G;  // last g with tile_off[g] <= t
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(p.tile_off + mid) <= t) lo = mid; else hi = mid;
  }
  const int rt = t - __ldg(p.tile_off + lo);
  const int start = rt * 128;
  return {lo, __ldg(p.off + lo) + start, min(128, __ldg(p.cnt + lo) - start)};
}

__device__ __forceinline__ int tile_src_row(const RowGemmParams& p, const RowTile& rt, int i) {
  if (p.row_src == nullptr) return rt.base + i;
  const int within = rt.base - (p.cnt ? __ldg(p.off + rt.g) : 0) + i;
  return __ldg(p.row_src + static_cast<int64_t>(rt.g) * p.src_stride + within);
}

__device__ __forceinline__ int tile_dst_row(const RowGemmParams& p, const RowTile& rt, int i) {
  if (p.row_dst == nullptr) return rt.base + i;
  const int within = rt.base - (p.cnt ? __ldg(p.off + rt.g) : 0) + i;
  return __ldg(p.row_dst + static_cast<int64_t>(rt.g) * p.dst_stride + within);
}

template <int KS, bool kBF16, int kBN>
__global__ void __launch_bounds__(kThreads, 1)
    rowgemm_kernel(const __grid_constant__ CUtensorMap tmB, const __grid_constant__ CUtensorMap tmA,
                   const __grid_constant__ RowGemmParams p, int n_tiles) {
  using Cfg = GmCfg<KS, kBN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stg = smem + Cfg::STAGES * Cfg::STAGE_BYTES;  // epilogue staging
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(stg + Cfg::STG_BYTES);
  uint64_t* empty_bar = full_bar + Cfg::STAGES;
  uint64_t* tfull_bar = empty_bar + Cfg::STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);
  int32_t* acc_live = reinterpret_cast<int32_t*>(tmem_slot + 2);    // per accumulator: 0 = no MMA (all zero)
  int32_t* stage_live = reinterpret_cast<int32_t*>(tmem_slot + 4);  // per stage: 1 = MMA, 0 = skipped
  uint64_t* loaded_bar = reinterpret_cast<uint64_t*>(tmem_slot + 4 + 8);  // mask mode: TMA landed
  __shared__ uint32_t tile_occ[Cfg::OCC_MAX_GROUPS * 5];  // the row tile's occupancy words per K-group
  __shared__ uint32_t kb_live[Cfg::KB_MAX / 32];            // bit kb: some row of the tile is live

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // union rows that cover (nearly) every row (scattered per-row K patterns): contiguous 128-row tiles
  // with the occupancy staged per tile instead (decided on the device: no host round trip)
  const bool contig = p.contig_pct > 0 && p.n_rows != nullptr &&
                      static_cast<int64_t>(*p.n_rows) * 100 >= static_cast<int64_t>(p.M) * (p.contig_pct % 1000);
  const bool diag_all_live = PIT_DIAG && p.contig_pct >= 1000;  // diagnostic builds: no zero-fill
  if (contig && p.exit_if_contig) return;  // rowgemm2 (masked) runs this product on CTA pairs
  if (path_skip(p)) return;
  const int32_t* row_src = contig ? nullptr : p.row_src;
  const int32_t* row_dst = contig ? nullptr : p.row_dst;
  const int single_rows = p.cnt ? 0 : contig ? p.M : (p.n_rows ? *p.n_rows : p.M);
  const int total_tiles = p.cnt ? __ldg(p.tile_off + p.G)
                         : p.uniform_rows ? p.G * ((p.uniform_rows + 127) / 128) : (single_rows + 127) / 128;
  // mask mode (contiguous rows with staged occupancy, A by TMA): warp 11 issues the A/B tiles, the 8
  // producer warps zero each landed stage's dead (row, micro-column) items, then arrive
  const bool mask_mode = p.mask_tma && p.occ != nullptr && row_src == nullptr && (p.t1 & (p.t1 - 1)) == 0 &&
                         (p.K + p.t1 - 1) / p.t1 <= Cfg::OCC_MAX_GROUPS && (p.K + KS - 1) / KS <= Cfg::KB_MAX;
  constexpr int kIssuerWarp = kRelayWarp + 1;

  if (threadIdx.x == 0) {
    for (int i = 0; i < Cfg::STAGES; ++i) {
      mbar_init(&full_bar[i], mask_mode ? kProdThreads : p.a_tma ? 1 : kProdThreads + 1);
      mbar_init(&empty_bar[i], 1);
      mbar_init(&loaded_bar[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull_bar[i], 2);  // MMA commit + the issuer's release of acc_live
      mbar_init(&tempty_bar[i], 128);
    }
    fence_mbar_init();
    tma_prefetch_desc(&tmB);
  }
  if (warp == kAllocWarp) tmem_alloc<Cfg::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int units = min(p.max_tiles, total_tiles) * n_tiles;
  const int kblocks = (p.K + KS - 1) / KS;

  if (warp < kProdWarps) {
    // ------------------------------------------------------------ producers
    // A rows: cp.async 16-byte chunks into the K-major swizzled layout; a row that is not live in
    // this K-block is zero-filled (src size 0). B: 2-D boxes of the 3-D [G, K, N] tensor map.
    // A K-block in which no row of the tile is live is skipped by every role (stage_live = 0).
    constexpr int CPR = KS * 2 / 16;                // chunks per A row
    constexpr int RPT = 128 * CPR / kProdThreads;   // rows per producer thread
    constexpr int RSTEP = kProdThreads / CPR;       // row stride between a thread's rows
    constexpr uint32_t MASK = KS * 2 == 128 ? 7 : KS * 2 == 64 ? 3 : 1;
    const int tp = threadIdx.x;  // 0..kProdThreads-1
    const int ch = tp % CPR;
    using T = typename OutT<kBF16>::T;
    const T* Ap = static_cast<const T*>(p.A);
    int stage = 0;
    uint32_t phase = 0;
    // Contiguous row tiles (dense, batched slices): the tile's occupancy words for every K-group are
    // staged in shared memory once per unit, so a K-block's liveness costs no L2 round trip and no
    // barrier (every producer derives the same stage verdict). Union-row tiles look bits up per row.
    const int nkg = p.occ ? (p.K + p.t1 - 1) / p.t1 : 0;
    const int lg_t1 = (p.t1 & (p.t1 - 1)) == 0 ? __ffs(p.t1) - 1 : -1;  // power-of-two widths: shifts
    const bool staged = p.occ != nullptr && row_src == nullptr && nkg <= Cfg::OCC_MAX_GROUPS &&
                        kblocks <= Cfg::KB_MAX;
    // next live K-block after kb (staged units): dead K-blocks cost no producer work at all
    auto next_kb = [&](int kb) {
      int start = kb + 1;
      int w = start >> 5;
      if (w * 32 >= kblocks) return kblocks;
      uint32_t bits = kb_live[w] & (0xffffffffu << (start & 31));
      while (!bits) {
        if (++w * 32 >= kblocks) return kblocks;
        bits = kb_live[w];
      }
      return min(w * 32 + __ffs(bits) - 1, kblocks);
    };
    for (int u = (p.a_tma && tp != 0) ? units : static_cast<int>(blockIdx.x); u < units; u += gridDim.x) {
      const RowTile rt = decode_tile(p, u / n_tiles, single_rows);
      const int n0 = (u % n_tiles) * Cfg::BN;
      int rid[RPT];  // this thread's rows: tp / CPR + j * RSTEP
#pragma unroll
      for (int j = 0; j < RPT; ++j) {
        const int i = tp / CPR + j * RSTEP;
        rid[j] = i < rt.rows ? (row_src ? tile_src_row(p, rt, i) : rt.base + i) : -1;
      }
      const int w0 = rt.base >> 5, sh = rt.base & 31;
      if (staged) {
        bar_sync_named(2, kProdThreads);  // every producer is done with the previous unit's words
        // independent loads, several in flight per thread (a K = 8192, t1 = 32 tile reads 1280 words)
#pragma unroll 4
        for (int e = tp; e < nkg * 5; e += kProdThreads) {
          const int kg = e / 5;
          const int64_t word = static_cast<int64_t>(w0) + (e - kg * 5);
          tile_occ[e] = word < p.WG ? __ldg(p.occ + static_cast<int64_t>(kg) * p.WG + word) : 0u;
        }
        bar_sync_named(2, kProdThreads);
        // one bit per K-block: does any row of this tile hold a live micro-tile there
        for (int kb0 = (tp & ~31); kb0 < kblocks; kb0 += kProdThreads) {
          const int kb = kb0 + (tp & 31);
          uint32_t anyw = 0;
          if (kb < kblocks) {
            // every K-group the K-block overlaps (KS > t1: e.g. two 32-wide micro-columns per block)
            const int kg1 = min((kb * KS + KS - 1) / p.t1, nkg - 1);
            for (int kg = kb * KS / p.t1; kg <= kg1; ++kg) {
              const uint32_t* wv = tile_occ + kg * 5;
#pragma unroll
              for (int w = 0; w < 5; ++w) {
                const int a = max(sh - 32 * w, 0), b = min(sh + rt.rows - 32 * w, 32);
                if (b > a) anyw |= wv[w] & bit_range(a, b);
              }
            }
          }
          const uint32_t word = __ballot_sync(0xffffffffu, anyw != 0);
          if ((tp & 31) == 0) kb_live[kb0 >> 5] = word;
        }
        bar_sync_named(2, kProdThreads);
        if (mask_mode) bar_sync_named(3, kProdThreads + 32);  // kb_live -> the TMA issuer (warp 11)
      }
      for (int kb = staged ? next_kb(-1) : 0; kb < kblocks; kb = staged ? next_kb(kb) : kb + 1) {
        const int k0 = kb * KS;
        if (mask_mode) {
          // the issuer's A tile has landed: zero its dead (row, micro-column) items
          mbar_wait(&loaded_bar[stage], phase);
          const uint32_t sA = smem_u32(smem + stage * Cfg::STAGE_BYTES);
          const int parts = p.t1 >= KS ? 1 : KS >> lg_t1;  // micro-columns per K-block
          const int cpk = CPR / parts;                      // 16-byte chunks per micro-column
          const int kg0 = k0 >> lg_t1;
          for (int it = tp; it < 128 * parts; it += kProdThreads) {
            const int row = it / parts, part = it - row * parts;
            const int rr = sh + row;
            const uint32_t w = tile_occ[min(kg0 + part, nkg - 1) * 5 + (rr >> 5)];
            if (!((w >> (rr & 31)) & 1u)) {
              for (int c = 0; c < cpk; ++c)
                st_shared_v4(sA + swz<MASK>(static_cast<uint32_t>(row * Cfg::A_ROW_BYTES + (part * cpk + c) * 16)), 0u,
                             0u, 0u, 0u);
            }
          }
          fence_proxy_async_smem();  // generic zero stores -> tcgen05.mma reads
          mbar_arrive(&full_bar[stage]);
          if (++stage == Cfg::STAGES) {
            stage = 0;
            phase ^= 1;
          }
          continue;
        }
        bool live[RPT];
        bool stage_any = true;
        // the K-group of this thread's 16-byte chunk (a K-block may span several when KS > t1)
        const int kc8 = k0 + ch * 8;
        const int kgc = p.occ ? min(lg_t1 >= 0 ? kc8 >> lg_t1 : kc8 / p.t1, nkg - 1) : 0;
        if (staged) {
          const uint32_t* wv = tile_occ + kgc * 5;
#pragma unroll
          for (int j = 0; j < RPT; ++j) {
            const int r = rid[j] - (w0 << 5);
            live[j] = rid[j] >= 0 && ((wv[r >> 5] >> (r & 31)) & 1u);
          }
        } else {
          bool any = false;
#pragma unroll
          for (int j = 0; j < RPT; ++j) {
            live[j] = rid[j] >= 0;
            if (live[j] && p.occ)
              live[j] = (__ldg(p.occ + static_cast<int64_t>(kgc) * p.WG + (rid[j] >> 5)) >> (rid[j] & 31)) & 1u;
            any |= live[j];
          }
          stage_any = p.occ ? bar_or(1, kProdThreads, any) : true;
        }
        // dead K-blocks take no ring slot: the ring holds only stages with data, so the copies in
        // flight are all useful (a unit ends with an END marker stage when liveness is tracked)
        if (!stage_any) continue;
        mbar_wait(&empty_bar[stage], phase ^ 1);
        uint8_t* sAp = smem + stage * Cfg::STAGE_BYTES;
        const uint32_t sA = smem_u32(sAp);
        uint8_t* sB = sAp + Cfg::A_BYTES;
        if (tp == 0) {
          stage_live[stage] = 1;
          mbar_expect_tx_only(&full_bar[stage], Cfg::B_BYTES + (p.a_tma ? Cfg::A_BYTES : 0));
#pragma unroll
          for (int a = 0; a < Cfg::BN / 64; ++a)
            tma_load_3d(sB + a * KS * 128, &tmB, &full_bar[stage], n0 + a * 64, k0, rt.g);
          // contiguous rows: the whole [128 rows x KS] A tile is one swizzled TMA box (rows past the
          // tile belong to no output row of this unit and are never stored; past the tensor, zeros)
          if (p.a_tma) tma_load_2d(sAp, &tmA, &full_bar[stage], k0, rt.base);
          mbar_arrive(&full_bar[stage]);  // publishes stage_live
        }
        if (p.a_tma) {
          // A and B by TMA: the issuing thread alone runs the ring (its arrive above)
        } else {
          const int kc = k0 + ch * 8;
          const uint32_t kbytes = kc < p.K ? static_cast<uint32_t>(min(16, (p.K - kc) * 2)) : 0u;
#pragma unroll
          for (int j = 0; j < RPT; ++j) {
            const int row = tp / CPR + j * RSTEP;
            const uint32_t bytes = (live[j] || (diag_all_live && rid[j] >= 0)) ? kbytes : 0u;
            const T* src = bytes ? Ap + static_cast<int64_t>(rid[j]) * p.lda + kc : Ap;
            cp_async_16(sA + swz<MASK>(static_cast<uint32_t>(row * Cfg::A_ROW_BYTES + ch * 16)), src, bytes);
          }
          cp_async_arrive_noinc(&full_bar[stage]);
        }
        if (++stage == Cfg::STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (p.occ && mask_mode) {  // END marker from the issuer
        mbar_wait(&loaded_bar[stage], phase);
        mbar_arrive(&full_bar[stage]);
        if (++stage == Cfg::STAGES) {
          stage = 0;
          phase ^= 1;
        }
      } else if (p.occ) {  // END marker: closes the unit for the MMA issuer
        mbar_wait(&empty_bar[stage], phase ^ 1);
        if (tp == 0) {
          stage_live[stage] = 2;
          mbar_arrive(&full_bar[stage]);
        }
        mbar_arrive(&full_bar[stage]);
        if (++stage == Cfg::STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (mask_mode && warp == kIssuerWarp) {
    // ------------------------------------------------------------ mask mode: TMA issuer
    int stage = 0;
    uint32_t phase = 0;
    auto next_live = [&](int kb) {
      int start = kb + 1;
      int w = start >> 5;
      if (w * 32 >= kblocks) return kblocks;
      uint32_t bits = kb_live[w] & (0xffffffffu << (start & 31));
      while (!bits) {
        if (++w * 32 >= kblocks) return kblocks;
        bits = kb_live[w];
      }
      return min(w * 32 + __ffs(bits) - 1, kblocks);
    };
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const RowTile rt = decode_tile(p, u / n_tiles, single_rows);
      const int n0 = (u % n_tiles) * Cfg::BN;
      bar_sync_named(3, kProdThreads + 32);  // the producers staged this unit's kb_live
      if (lane == 0) {
        for (int kb = next_live(-1); kb < kblocks; kb = next_live(kb)) {
          const int k0 = kb * KS;
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sAp = smem + stage * Cfg::STAGE_BYTES;
          uint8_t* sB = sAp + Cfg::A_BYTES;
          stage_live[stage] = 1;
          mbar_expect_tx_only(&loaded_bar[stage], Cfg::B_BYTES + Cfg::A_BYTES);
#pragma unroll
          for (int a = 0; a < Cfg::BN / 64; ++a)
            tma_load_3d(sB + a * KS * 128, &tmB, &loaded_bar[stage], n0 + a * 64, k0, rt.g);
          tma_load_2d(sAp, &tmA, &loaded_bar[stage], k0, rt.base);
          mbar_arrive(&loaded_bar[stage]);
          if (++stage == Cfg::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        mbar_wait(&empty_bar[stage], phase ^ 1);  // END marker
        stage_live[stage] = 2;
        mbar_arrive(&loaded_bar[stage]);
        if (++stage == Cfg::STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      __syncwarp();
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = idesc_f16(Cfg::BM, Cfg::BN, kBF16, false, true);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
      tc_fence_after();
      bool first = true;
      // dense: exactly kblocks data stages; tracked liveness: data stages until the END marker
      for (int kb = 0; p.occ != nullptr || kb < kblocks; ++kb) {
        mbar_wait(&full_bar[stage], phase);
        fence_proxy_async_smem();  // cp.async (generic proxy) writes -> tcgen05.mma reads
        tc_fence_after();
        const int meta = stage_live[stage];
        const bool live = meta == 1;
        if (lane == 0) {
          if (live) {
            const uint32_t sA = smem_u32(smem + stage * Cfg::STAGE_BYTES);
            const uint32_t sB = sA + Cfg::A_BYTES;
#pragma unroll
            for (int ks = 0; ks < KS / 16; ++ks) {
              const uint64_t adesc = smem_desc(sA + ks * 32, 16, 8 * Cfg::A_ROW_BYTES, Cfg::A_SW);
              const uint64_t bdesc = smem_desc(sB + ks * 2048, KS * 128, 1024, kSw128);
              umma_f16(tmem_base + static_cast<uint32_t>(acc * Cfg::BN), adesc, bdesc, idesc,
                       (!first || ks > 0) ? 1u : 0u);
            }
          }
          umma_commit(&empty_bar[stage]);
        }
        first = first && !live;
        __syncwarp();
        if (++stage == Cfg::STAGES) {
          stage = 0;
          phase ^= 1;
        }
        if (meta == 2) break;
      }
      if (lane == 0) {
        // a unit whose every K-block was skipped never wrote its accumulator: the epilogue stores
        // zeros for it (rows named by no live micro-tile are exact zeros)
        acc_live[acc] = first ? 0 : 1;
        umma_commit(&tfull_bar[acc]);
        mbar_arrive(&tfull_bar[acc]);
      }
      __syncwarp();
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  } else if (warp >= kEpiWarp0) {
    // ------------------------------------------------------------ epilogue: row scatter (SWrite)
    using T = typename OutT<kBF16>::T;
    const int q = warp & 3;
    const bool vec_ok = (p.ldc % 8) == 0 && (reinterpret_cast<uintptr_t>(p.C) & 15) == 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const RowTile rt = decode_tile(p, u / n_tiles, single_rows);
      const int n0 = (u % n_tiles) * Cfg::BN;
      const int i = q * 32 + lane;
      const int row = i < rt.rows ? (row_dst ? tile_dst_row(p, rt, i) : rt.base + i) : -1;
      const float scale = (row >= 0 && p.row_scale) ? __ldg(p.row_scale + row) : 1.0f;
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const bool have = acc_live[acc] != 0;
      if (vec_ok) {
        // Staged, coalesced row scatter: the warp's 32 rows x 64 columns go through a swizzled shared
        // box and leave as 128-byte row segments (8 lanes per row, 4 rows per instruction) instead of
        // 16-byte pieces at a row stride per lane, which clog the LSU the producers' gathers share.
        const uint32_t box = smem_u32(stg) + static_cast<uint32_t>(q * 4096);
        T* C = static_cast<T*>(p.C);
#pragma unroll 1
        for (int bx = 0; bx < Cfg::BN / 64; ++bx) {
          uint32_t v[64];
          if (have) {
            const uint32_t ta = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * Cfg::BN + bx * 64);
            tmem_ld32(ta, *reinterpret_cast<uint32_t(*)[32]>(v));
            tmem_ld32(ta + 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
            tmem_wait_ld();
          } else {
#pragma unroll
            for (int j = 0; j < 64; ++j) v[j] = 0u;
          }
          __syncwarp();  // the previous box's copy-out has read the staging
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            float f[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              float x = __uint_as_float(v[8 * j + e]);
              if (p.act == 1) x = fmaxf(x, 0.0f);
              f[e] = x * scale;
            }
            st_shared_v4(box + lane * 128 + ((static_cast<uint32_t>(j) ^ static_cast<uint32_t>(lane & 7)) << 4),
                         pack2(f[0], f[1], kBF16), pack2(f[2], f[3], kBF16), pack2(f[4], f[5], kBF16),
                         pack2(f[6], f[7], kBF16));
          }
          __syncwarp();
          const int ch = lane & 7;
          const int col = n0 + bx * 64 + ch * 8;
#pragma unroll
          for (int it = 0; it < 8; ++it) {
            const int r = it * 4 + (lane >> 3);
            const int drow = __shfl_sync(0xffffffffu, row, r);
            const uint4 w = ld_shared_v4(box + r * 128 + ((static_cast<uint32_t>(ch) ^ static_cast<uint32_t>(r & 7)) << 4));
            if (drow >= 0 && col < p.N) {
              T* dst = C + static_cast<int64_t>(drow) * p.ldc + col;
              if (col + 8 <= p.N) {
                *reinterpret_cast<uint4*>(dst) = w;
              } else {
                const T* h = reinterpret_cast<const T*>(&w);
                for (int e = 0; e < p.N - col; ++e) dst[e] = h[e];
              }
            }
          }
        }
      } else {
      uint8_t* crow = row >= 0 ? static_cast<uint8_t*>(p.C) + (static_cast<int64_t>(row) * p.ldc) * 2 : nullptr;
#pragma unroll 1
      for (int c = 0; c < Cfg::BN; c += 32) {
        uint32_t v[32];
        if (have) {
          tmem_ld32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * Cfg::BN + c), v);
          tmem_wait_ld();
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = 0u;
        }
        if (row >= 0) {
          float f[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            float x = __uint_as_float(v[j]);
            if (p.act == 1) x = fmaxf(x, 0.0f);
            f[j] = x * scale;
          }
          const int nb = n0 + c;
          if (nb + 32 <= p.N && vec_ok) {
            uint4* dst = reinterpret_cast<uint4*>(crow + static_cast<int64_t>(nb) * 2);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              uint4 w;
              w.x = pack2(f[8 * j + 0], f[8 * j + 1], kBF16);
              w.y = pack2(f[8 * j + 2], f[8 * j + 3], kBF16);
              w.z = pack2(f[8 * j + 4], f[8 * j + 5], kBF16);
              w.w = pack2(f[8 * j + 6], f[8 * j + 7], kBF16);
              dst[j] = w;
            }
          } else {
            using T = typename OutT<kBF16>::T;
            T* dst = reinterpret_cast<T*>(crow);
            for (int j = 0; j < 32; ++j)
              if (nb + j < p.N) dst[nb + j] = OutT<kBF16>::cvt(f[j]);
          }
        }
      }
      }
      tc_fence_before();
      mbar_arrive(&tempty_bar[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == kAllocWarp) {
    tc_fence_after();
    tmem_dealloc<Cfg::TMEM_COLS>(tmem_base);
  }
}

// =============================================================================================
// rowgemm2: the dense / contiguous-row cases of rowgemm (no per-row liveness, single group or
// uniform batched slices) on CTA pairs — tcgen05 cta_group::2, 256 x 256 tiles. CTA r holds rows
// [128 r, 128 r + 128) of the pair tile and columns [128 r, 128 r + 128) of the B tile, so each
// CTA moves 32 KB per 64-deep K-block for a 128 x 256 x 64 share of the MMA (131 FLOP per byte,
// against 87 for the single-CTA 128 x 256 tile whose operand feed bounds it near 1 PFLOP/s).
// Pipeline as spmm_gk2: local full barrier (TMA bytes + cp.async arrivals) -> relay -> even CTA's
// pair barrier -> pair MMA -> multicast commits; each CTA drains and stores its own 128 rows.
// =============================================================================================
constexpr int kRg2MaxGroups = 1024;
constexpr int kRg2OccGroups = 512;  // masked mode: K-groups whose occupancy words fit shared memory
constexpr int kRg2Band = 8;  // pair row tiles per raster band (dense)

struct Rg2Cfg {
  static constexpr int KS = 64;
  static constexpr int BN = 256;
  static constexpr int A_BYTES = 128 * KS * 2;        // K-major rows, 128B swizzle
  static constexpr int B_BYTES = 2 * KS * 128;        // the CTA's 128-column half: 2 MN-major atoms
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  // one 32 x 64 staging box per epilogue warp: 8 warps when the producer warps 4-7 are idle
  // (A and B by TMA from one thread), else 4
  // (4-warp modes keep their per-mode tables in the upper half: grouped prefix, masked occupancy)
  static constexpr int STG_BYTES = 8 * 4096;
  static constexpr int PTO_OFF = 4 * 4096, OCC_OFF = PTO_OFF + 4352, KBL_OFF = OCC_OFF + 4 * 2048;
  static constexpr int STAGE_BUDGET = 232448 - 2048 - STG_BYTES;
  static constexpr int STAGES = STAGE_BUDGET / STAGE_BYTES > 8 ? 8 : STAGE_BUDGET / STAGE_BYTES;
  static constexpr size_t SMEM = static_cast<size_t>(STAGES) * STAGE_BYTES + STG_BYTES + 2048;
};

static_assert((kRg2MaxGroups + 1) * 4 <= Rg2Cfg::OCC_OFF - Rg2Cfg::PTO_OFF, "rowgemm2 group prefix");
static_assert(kRg2OccGroups * 4 * 4 <= Rg2Cfg::KBL_OFF - Rg2Cfg::OCC_OFF, "rowgemm2 occupancy words");
static_assert(Rg2Cfg::KBL_OFF + 128 <= Rg2Cfg::STG_BYTES, "rowgemm2 staging half");
static_assert(Rg2Cfg::SMEM <= 232448, "rowgemm2 shared memory");

// CTA r's 128-row tile of pair tile pt (rows may be <= 0: a partial pair, nothing stored).
// Grouped (MoE experts): pto = shared prefix of ceil(cnt[g] / 256) over the groups.
__device__ __forceinline__ RowTile decode_pair_tile(const RowGemmParams& p, int pt, int r, int single_rows,
                                                    const int* pto) {
  if (p.cnt != nullptr) {
    int lo = 0, hi = p.G;  // last g with pto[g] <= pt
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (pto[mid] <= pt) lo = mid; else hi = mid;
    }
    const int start = (pt - pto[lo]) * 256 + 128 * r;
    return {lo, __ldg(p.off + lo) + start, min(128, __ldg(p.cnt + lo) - start)};
  }
  if (p.uniform_rows) {
    const int tpg = (p.uniform_rows + 255) >> 8;
    const int g = pt / tpg, start = (pt - g * tpg) * 256 + 128 * r;
    return {g, g * p.uniform_rows + start, min(128, p.uniform_rows - start)};
  }
  const int base = pt * 256 + 128 * r;
  return {0, base, min(128, single_rows - base)};
}

template <bool kBF16>
__global__ void __launch_bounds__(kThreads, 1)
    rowgemm2_kernel(const __grid_constant__ CUtensorMap tmB, const __grid_constant__ CUtensorMap tmA,
                    const __grid_constant__ CUtensorMap tmC, const __grid_constant__ RowGemmParams p, int n_tiles,
                    int pair_tiles, int c_tma) {
  using Cfg = Rg2Cfg;
  constexpr int KS = Cfg::KS;
  // diagnostic builds: globaltimer stamps of pair 0 (even CTA) into g_gk2_trace (scripts/rg2_trace.py):
  // [0,128) producer stage issue, [128,256) relay full (odd CTA: [384,512)), [256,384) MMA pair_full, [512,576) MMA unit
  // start, [576,640) epilogue TMEM full, [640,704) epilogue done, 767 setup done, [768,1024) CTA entry
  if (PIT_DIAG && threadIdx.x == 0 && blockIdx.x < 256) g_gk2_trace[768 + blockIdx.x] = gtimer();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stg = smem + Cfg::STAGES * Cfg::STAGE_BYTES;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(stg + Cfg::STG_BYTES);
  uint64_t* pair_full = full_bar + Cfg::STAGES;
  uint64_t* empty_bar = pair_full + Cfg::STAGES;
  uint64_t* tfull_bar = empty_bar + Cfg::STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);
  uint64_t* loaded_bar = reinterpret_cast<uint64_t*>(tmem_slot + 2);  // masked + TMA A: operands landed
  // masked with A by TMA: warp 11 (one lane) issues the TMA loads, the 8 producer warps zero the dead
  // (row, micro-column) items of each landed stage (one item per thread at t1 = 32) and then arrive
  // on the full barrier
  const bool mask_tma = p.masked && p.a_tma;
  constexpr int kMaskers = kProdThreads;
  constexpr int kIssuerWarp = kRelayWarp + 1;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  // A and B by TMA from one thread (no masking): producer warps 4-7 drain columns 128-255 of each
  // accumulator beside warps 12-15 (columns 0-127), halving the exposed epilogue
  const bool epi8 = p.epi8 && p.a_tma && !p.masked && p.cnt == nullptr;
  const bool epi_warp = warp >= kEpiWarp0 || (epi8 && warp >= 4 && warp < kProdWarps);

  const int pair = static_cast<int>(blockIdx.x >> 1);
  const int npairs = static_cast<int>(gridDim.x >> 1);
  const bool trace = PIT_DIAG && pair == 0 && rank == 0;
  int tj = 0, tu = 0;  // trace counters (diagnostic builds)
  // masked (2-D pit:m with scattered per-row K patterns): decided on the device from the union size;
  // when the union is small the union-row rowgemm launched beside this kernel runs the product
  if (p.masked && p.n_rows != nullptr &&
      static_cast<int64_t>(*p.n_rows) * 100 < static_cast<int64_t>(p.M) * p.contig_pct)
    return;
  if (path_skip(p)) return;
  const int single_rows = p.masked ? p.M : (p.n_rows ? *p.n_rows : p.M);
  // pair row tiles that hold rows: one group of union rows from the device row count (the host sized
  // the grid for every row of A); grouped: from the device prefix, after the setup barrier
  int pt_live = pair_tiles;
  if (p.cnt == nullptr && !p.masked && p.uniform_rows == 0 && p.n_rows != nullptr)
    pt_live = min(pair_tiles, (single_rows + 255) >> 8);
  int units = pt_live * n_tiles;
  // unit -> (pair row tile, n tile). One group (dense, BERT): rasterised in bands of kRg2Band pair
  // row tiles, n tile outer within a band, so the pairs running together share B n-tile slabs and
  // an A row band in L2 (row-tile-major order re-streamed all of B for every wave of row tiles).
  const bool banded = p.cnt == nullptr && p.uniform_rows == 0 && units >= 8 * npairs;  // (grouped: never)
  auto unit_pt = [&](int u) {
    if (!banded) return u / n_tiles;
    const int band = u / (kRg2Band * n_tiles), in = u - band * kRg2Band * n_tiles;
    const int bh = min(kRg2Band, pt_live - band * kRg2Band);
    return band * kRg2Band + in % bh;
  };
  auto unit_nt = [&](int u) {
    if (!banded) return u % n_tiles;
    const int band = u / (kRg2Band * n_tiles), in = u - band * kRg2Band * n_tiles;
    const int bh = min(kRg2Band, pt_live - band * kRg2Band);
    return in / bh;
  };
  // the first unit's first stages are requested by warp 1 between the arrival on and the wait at the
  // setup barrier (local shared memory and barriers only): their load latency overlaps the TMEM
  // allocation and the cluster barrier; the producer thread skips them
  int early = (p.a_tma && !p.masked && p.cnt == nullptr && pair < units) ? min(Cfg::STAGES, (p.K + KS - 1) / KS) : 0;
  // grouped: prefix of pair tiles per group; masked: the CTA's 128 rows' words per K-group and the
  // globally live K-blocks (both in the staging half the 4-warp epilogue leaves free)
  int* pto = reinterpret_cast<int*>(stg + Cfg::PTO_OFF);
  uint32_t* tile_occ = reinterpret_cast<uint32_t*>(stg + Cfg::OCC_OFF);
  uint32_t* kbl = reinterpret_cast<uint32_t*>(stg + Cfg::KBL_OFF);

  if (threadIdx.x == 0) {
    for (int i = 0; i < Cfg::STAGES; ++i) {
      // every operand by TMA (dense, packed rows): the issuing thread's arrival alone; cp.async rows:
      // one cp.async arrival per producer thread, or (lagged mode) one per warp kLag stages behind
      mbar_init(&full_bar[i], mask_tma ? kMaskers : (p.a_tma ? 1 : (p.lagged ? kProdWarps : kProdThreads) + 1));
      mbar_init(&loaded_bar[i], 1);
      mbar_init(&pair_full[i], 2);
      mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull_bar[i], 1);
      mbar_init(&tempty_bar[i], epi8 ? 16 : 8);  // epilogue warps x 2 CTAs
    }
    fence_mbar_init();
    tma_prefetch_desc(&tmB);
  }
  if (warp == kAlloc2Warp) tmem_alloc2<512>(tmem_slot);
  if (p.cnt != nullptr && warp == kRelayWarp + 1) {
    // warp 11: pair tiles per group, scanned (each lane a contiguous run of groups)
    const int per = (p.G + 31) / 32;
    const int g0 = lane * per;
    int run = 0;
    for (int g = g0; g < min(p.G, g0 + per); ++g) run += (__ldg(p.cnt + g) + 255) >> 8;
    int incl = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    int acc = incl - run;
    for (int g = g0; g < min(p.G, g0 + per); ++g) {
      pto[g] = acc;
      acc += (__ldg(p.cnt + g) + 255) >> 8;
    }
    if (lane == 31) pto[p.G] = incl;
  }
  // masked: K-blocks in which no row of the whole operand is live (dead neurons: column-structured
  // activation sparsity) are skipped by every role of both CTAs — a global property, so the pair
  // agrees without exchanging anything
  if (p.masked) {
    const int nkb = (p.K + KS - 1) / KS, nkg = (p.K + p.t1 - 1) / p.t1;
    for (int kb0 = warp * 32; kb0 < nkb; kb0 += (kThreads / 32) * 32) {
      const int kb = kb0 + lane;
      bool live = false;
      if (kb < nkb) {
        const int kg1 = min((kb * KS + KS - 1) / p.t1, nkg - 1);
        for (int kg = kb * KS / p.t1; kg <= kg1; ++kg) live |= __ldg(p.kg_cnt + kg) > 0;
      }
      const uint32_t word = __ballot_sync(0xffffffffu, live);
      if (lane == 0) kbl[kb0 >> 5] = word;
    }
  }
  tc_fence_before();
  __syncthreads();  // the barrier inits are visible to warp 1
  cluster_arrive();
  if (warp == 1 && early > 0) {
    if (lane == 0) {
      tma_prefetch_desc(&tmA);
      const RowTile rt = decode_pair_tile(p, unit_pt(pair), static_cast<int>(rank), single_rows, pto);
      const int n0 = unit_nt(pair) * Cfg::BN + 128 * static_cast<int>(rank);
      for (int kb = 0; kb < early; ++kb) {
        uint8_t* sAp = smem + kb * Cfg::STAGE_BYTES;
        uint8_t* sB = sAp + Cfg::A_BYTES;
        mbar_expect_tx_only(&full_bar[kb], Cfg::B_BYTES + Cfg::A_BYTES);
        tma_load_3d(sB, &tmB, &full_bar[kb], n0, kb * KS, rt.g);
        tma_load_3d(sB + KS * 128, &tmB, &full_bar[kb], n0 + 64, kb * KS, rt.g);
        tma_load_2d(sAp, &tmA, &full_bar[kb], kb * KS, rt.base);
        mbar_arrive(&full_bar[kb]);
      }
    }
    __syncwarp();
  }
  cluster_wait();
  tc_fence_after();
  if (trace && threadIdx.x == 0) g_gk2_trace[767] = gtimer();
  const uint32_t tmem_base = *tmem_slot;
  if (p.cnt != nullptr) {  // grouped: pair row tiles from the device prefix
    pt_live = min(pair_tiles, pto[p.G]);
    units = pt_live * n_tiles;
  }
  const int kblocks = (p.K + KS - 1) / KS;
  auto next_kb = [&](int kb) {  // masked: next live K-block after kb (kblocks: none)
    if (!p.masked) return kb + 1;
    int w = (kb + 1) >> 5;
    if (w * 32 >= kblocks) return kblocks;
    uint32_t bits = kbl[w] & (0xffffffffu << ((kb + 1) & 31));
    while (!bits) {
      if (++w * 32 >= kblocks) return kblocks;
      bits = kbl[w];
    }
    return min(w * 32 + __ffs(bits) - 1, kblocks);
  };
  const int kb_first = next_kb(-1);  // 0 unless masked
  int nlive_kb = kblocks;
  if (p.masked) {
    nlive_kb = 0;
    for (int w = 0; w < (kblocks + 31) / 32; ++w) nlive_kb += __popc(kbl[w]);
  }
  const bool all_kb = nlive_kb == kblocks;  // the common case keeps the plain K-block loop


  if (epi_warp) {
    // handled below (epilogue)
  } else if ((warp < kProdWarps || warp == kIssuerWarp) && mask_tma) {
    // ------------------------------------------------------------ producers, masked + TMA A
    const int nkg = (p.K + p.t1 - 1) / p.t1;
    const int lg_t1 = __ffs(p.t1) - 1;  // t1 in {16, 32}
    int stage = 0;
    uint32_t phase = 0;
    if (warp == kIssuerWarp) {
      if (lane == 0) {
        for (int u = pair; u < units; u += npairs) {
          const RowTile rt = decode_pair_tile(p, unit_pt(u), static_cast<int>(rank), single_rows, pto);
          const int n0 = unit_nt(u) * Cfg::BN + 128 * static_cast<int>(rank);
          for (int kb = kb_first; kb < kblocks; kb = all_kb ? kb + 1 : next_kb(kb)) {
            const int k0 = kb * KS;
            mbar_wait(&empty_bar[stage], phase ^ 1);
            uint8_t* sAp = smem + stage * Cfg::STAGE_BYTES;
            uint8_t* sB = sAp + Cfg::A_BYTES;
            mbar_expect_tx_only(&loaded_bar[stage], Cfg::B_BYTES + Cfg::A_BYTES);
            tma_load_3d(sB, &tmB, &loaded_bar[stage], n0, k0, rt.g);
            tma_load_3d(sB + KS * 128, &tmB, &loaded_bar[stage], n0 + 64, k0, rt.g);
            tma_load_2d(sAp, &tmA, &loaded_bar[stage], k0, rt.base);
            mbar_arrive(&loaded_bar[stage]);
            if (++stage == Cfg::STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    } else {
      const int tm = threadIdx.x;  // 0 .. kMaskers-1 (warps 0-7)
      for (int u = pair; u < units; u += npairs) {
        const RowTile rt = decode_pair_tile(p, unit_pt(u), static_cast<int>(rank), single_rows, pto);
        bar_sync_named(2, kMaskers);  // every masker is done with the previous unit's words
        const int64_t w0 = rt.base >> 5;
#pragma unroll 4
        for (int e = tm; e < nkg * 4; e += kMaskers) {
          const int64_t word = w0 + (e & 3);
          tile_occ[e] = word < p.WG ? __ldg(p.occ + static_cast<int64_t>(e >> 2) * p.WG + word) : 0u;
        }
        bar_sync_named(2, kMaskers);
        for (int kb = kb_first; kb < kblocks; kb = all_kb ? kb + 1 : next_kb(kb)) {
          const int k0 = kb * KS;
          mbar_wait(&loaded_bar[stage], phase);
          const uint32_t sA = smem_u32(smem + stage * Cfg::STAGE_BYTES);
          // (row, micro-column) items: one liveness lookup per item, a dead item's 16-byte chunks
          // (4 for t1 = 32, 2 for t1 = 16) are zeroed
          const int kg0 = k0 >> lg_t1;
          auto mask_items = [&](auto cpk_tag) {
            constexpr int CPK = decltype(cpk_tag)::value;  // chunks per micro-column
            constexpr int PARTS = 8 / CPK;                 // micro-columns per 64-deep K-block
#pragma unroll 2
            for (int it = tm; it < 128 * PARTS; it += kMaskers) {
              const int row = it / PARTS, part = it % PARTS;
              const uint32_t w = tile_occ[min(kg0 + part, nkg - 1) * 4 + (row >> 5)];
              if (!((w >> (row & 31)) & 1u)) {
#pragma unroll
                for (int c = 0; c < CPK; ++c)
                  st_shared_v4(sA + swz<7>(static_cast<uint32_t>(row * 128 + (part * CPK + c) * 16)), 0u, 0u, 0u, 0u);
              }
            }
          };
          if (lg_t1 == 5) mask_items(std::integral_constant<int, 4>{});
          else mask_items(std::integral_constant<int, 2>{});
          fence_proxy_async_smem();  // generic zero stores -> tcgen05.mma reads
          mbar_arrive(&full_bar[stage]);
          if (++stage == Cfg::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp < kProdWarps) {
    // ------------------------------------------------------------ producers
    constexpr int CPR = KS * 2 / 16;               // 16-byte chunks per A row
    constexpr int RPT = 128 * CPR / kProdThreads;  // A rows per producer thread (gathered rows)
    constexpr int RSTEP = kProdThreads / CPR;
    const int tp = threadIdx.x;
    const int ch = tp % CPR;
    using T = typename OutT<kBF16>::T;
    const T* Ap = static_cast<const T*>(p.A);
    int stage = 0;
    uint32_t phase = 0;
    const int nkg = p.masked ? (p.K + p.t1 - 1) / p.t1 : 0;
    const int lg_t1 = p.masked ? __ffs(p.t1) - 1 : 0;  // masked: t1 in {16, 32}
#ifndef PIT_RG2_LAG
#define PIT_RG2_LAG 3
#endif
    constexpr int kLag = PIT_RG2_LAG;  // stages between a warp's copies and its arrival
    int lagged = 0;  // stages whose copies this thread issued
    // A and B both by TMA: one thread runs the ring (255 per-stage arrivals were pure overhead)
    const int u_first = (p.a_tma && tp != 0) ? units : pair;
    for (int u = u_first; u < units; u += npairs) {
      const RowTile rt = decode_pair_tile(p, unit_pt(u), static_cast<int>(rank), single_rows, pto);
      const int n0 = unit_nt(u) * Cfg::BN + 128 * static_cast<int>(rank);
      int rid[RPT];
      if (!p.a_tma) {
#pragma unroll
        for (int j = 0; j < RPT; ++j) {
          const int i = tp / CPR + j * RSTEP;
          rid[j] = i < rt.rows ? tile_src_row(p, rt, i) : -1;
        }
      }
      if (p.masked) {
        // the half tile's 128 rows start at a multiple of 128: 4 occupancy words per K-group
        bar_sync_named(2, kProdThreads);  // every producer is done with the previous unit's words
        const int64_t w0 = rt.base >> 5;
#pragma unroll 4
        for (int e = tp; e < nkg * 4; e += kProdThreads) {
          const int64_t word = w0 + (e & 3);
          tile_occ[e] = word < p.WG ? __ldg(p.occ + static_cast<int64_t>(e >> 2) * p.WG + word) : 0u;
        }
        bar_sync_named(2, kProdThreads);
      }
      for (int kb = kb_first; kb < kblocks; kb = all_kb ? kb + 1 : next_kb(kb)) {
        const int k0 = kb * KS;
        if (early > 0) {  // issued before the setup barrier (thread 0 only; ring slots 0 .. early-1)
          --early;
          if (++stage == Cfg::STAGES) {
            stage = 0;
            phase ^= 1;
          }
          continue;
        }
        mbar_wait(&empty_bar[stage], phase ^ 1);
        uint8_t* sAp = smem + stage * Cfg::STAGE_BYTES;
        uint8_t* sB = sAp + Cfg::A_BYTES;
        if (tp == 0) {
          if (trace && tj < 128) g_gk2_trace[tj++] = gtimer();
          mbar_expect_tx_only(&full_bar[stage], Cfg::B_BYTES + (p.a_tma ? Cfg::A_BYTES : 0));
          tma_load_3d(sB, &tmB, &full_bar[stage], n0, k0, rt.g);
          tma_load_3d(sB + KS * 128, &tmB, &full_bar[stage], n0 + 64, k0, rt.g);
          if (p.a_tma) tma_load_2d(sAp, &tmA, &full_bar[stage], k0, rt.base);
          mbar_arrive(&full_bar[stage]);
        }
        if (!p.a_tma) {
          const uint32_t sA = smem_u32(sAp);
          const int kc = k0 + ch * 8;
          const uint32_t kbytes = kc < p.K ? static_cast<uint32_t>(min(16, (p.K - kc) * 2)) : 0u;
          // masked: this thread's chunk lies in one K-group; a row dead there is zero-filled
          const uint32_t* wv = tile_occ + min(kc >> lg_t1, nkg - 1) * 4;
#pragma unroll
          for (int j = 0; j < RPT; ++j) {
            const int row = tp / CPR + j * RSTEP;
            const bool live = rid[j] >= 0 && (!p.masked || ((wv[row >> 5] >> (row & 31)) & 1u));
            const uint32_t bytes = live ? kbytes : 0u;
            const T* src = bytes ? Ap + static_cast<int64_t>(rid[j]) * p.lda + kc : Ap;
            cp_async_16(sA + swz<7>(static_cast<uint32_t>(row * 128 + ch * 16)), src, bytes);
          }
        }
        if (!p.a_tma && !p.lagged) cp_async_arrive_noinc(&full_bar[stage]);
        if (!p.a_tma && p.lagged) {
          // lagged mode (PIT_RG2_LAGGED=1, A/B knob): the warp's copies of this stage form one group;
          // the group kLag stages older is waited for and signalled with one arrival per warp. Same
          // speed as per-thread arrivals on the BERT product (0.7 us per stage either way: the
          // cp.async feed, not the barrier, bounds it), so per-thread arrivals stay the default.
          cp_async_commit();
          if (++lagged > kLag) {
            cp_async_wait<kLag>();
            fence_proxy_async_smem();  // generic-proxy cp.async writes -> tcgen05.mma reads
            __syncwarp();
            if (lane == 0) mbar_arrive(&full_bar[(stage + Cfg::STAGES - kLag) % Cfg::STAGES]);
          }
        }
        if (++stage == Cfg::STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    if (!p.a_tma && p.lagged && lagged > 0) {  // the last kLag stages
      cp_async_wait<0>();
      fence_proxy_async_smem();
      __syncwarp();
      for (int j = min(lagged, kLag); j >= 1; --j)
        if (lane == 0) mbar_arrive(&full_bar[(stage + Cfg::STAGES - j) % Cfg::STAGES]);
    }
  } else if (warp == kRelayWarp) {
    // ------------------------------------------------------------ relay: local full -> pair full
    if (lane == 0) {
      const uint32_t leader_pf = mapa_shared(smem_u32(pair_full), 0);
      int stage = 0;
      uint32_t phase = 0;
      for (int u = pair; u < units; u += npairs) {
        for (int kb = kb_first; kb < kblocks; kb = all_kb ? kb + 1 : next_kb(kb)) {
          mbar_wait(&full_bar[stage], phase);
          if (PIT_DIAG && pair == 0 && tj < 128) g_gk2_trace[(rank ? 384 : 128) + tj++] = gtimer();
          fence_proxy_async_smem();
          mbar_arrive_cluster(leader_pf + stage * 8);
          if (++stage == Cfg::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer (even CTA)
    if (rank == 0) {
      constexpr uint32_t idesc = idesc_f16(256, Cfg::BN, kBF16, false, true);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int u = pair; u < units; u += npairs) {
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        if (trace && lane == 0 && tu < 64) g_gk2_trace[512 + tu++] = gtimer();
        for (int kb = kb_first; kb < kblocks; kb = all_kb ? kb + 1 : next_kb(kb)) {
          mbar_wait(&pair_full[stage], phase);
          tc_fence_after();
          if (trace && lane == 0 && tj < 128) g_gk2_trace[256 + tj++] = gtimer();
          if (lane == 0) {
            const uint32_t sA = smem_u32(smem + stage * Cfg::STAGE_BYTES);
            const uint32_t sB = sA + Cfg::A_BYTES;
#pragma unroll
            for (int ks = 0; ks < KS / 16; ++ks) {
              const uint64_t adesc = smem_desc(sA + ks * 32, 16, 8 * 128, kSw128);
              const uint64_t bdesc = smem_desc(sB + ks * 2048, KS * 128, 1024, kSw128);
              umma2_f16(tmem_base + static_cast<uint32_t>(acc * Cfg::BN), adesc, bdesc, idesc,
                        (kb > kb_first || ks > 0) ? 1u : 0u);
            }
            umma2_commit_mc(&empty_bar[stage], 3);
          }
          __syncwarp();
          if (++stage == Cfg::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (lane == 0) umma2_commit_mc(&tfull_bar[acc], 3);
        __syncwarp();
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else if ((warp == kAllocWarp || warp == kIssuerWarp) && p.zero_occ != nullptr) {
    // ------------------------------------------------------------ dead rows of C: exact zeros
    // (rows no group names), a warp per row, 16-byte stores, beside the mainloop
    const int zw = 2 * static_cast<int>(blockIdx.x) + (warp == kAllocWarp ? 0 : 1);
    const int nzw = 2 * static_cast<int>(gridDim.x);
    const int chunks = p.N >> 3;
    for (int r = zw; r < p.M; r += nzw) {
      if ((__ldg(p.zero_occ + (r >> 5)) >> (r & 31)) & 1u) continue;
      uint4* dst = reinterpret_cast<uint4*>(static_cast<uint8_t*>(p.C) + static_cast<int64_t>(r) * p.ldc * 2);
      for (int i = lane; i < chunks; i += 32) dst[i] = make_uint4(0u, 0u, 0u, 0u);
    }
  }
  if (epi_warp) {
    // ------------------------------------------------------------ epilogue: this CTA's 128 rows
    using T = typename OutT<kBF16>::T;
    const int q = warp & 3;
    const int half = (epi8 && warp < kProdWarps) ? 1 : 0;  // epi8: warps 4-7 take boxes 2-3
    const int bx0 = epi8 ? 2 * half : 0, bx1 = epi8 ? 2 * half + 2 : Cfg::BN / 64;
    const uint32_t leader_te = mapa_shared(smem_u32(tempty_bar), 0);
    const uint32_t box = smem_u32(stg) + static_cast<uint32_t>((half * 4 + q) * 4096);
    T* C = static_cast<T*>(p.C);
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = pair; u < units; u += npairs) {
      const RowTile rt = decode_pair_tile(p, unit_pt(u), static_cast<int>(rank), single_rows, pto);
      const int n0 = unit_nt(u) * Cfg::BN;
      const int i = q * 32 + lane;
      const int row = i < rt.rows ? tile_dst_row(p, rt, i) : -1;
      const float scale = (row >= 0 && p.row_scale) ? __ldg(p.row_scale + row) : 1.0f;
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      if (trace && q == 0 && half == 0 && lane == 0 && tu < 64) g_gk2_trace[576 + tu] = gtimer();
      // consecutive destination rows (dense, batched slices, masked pit:m): the warp's 32 x 64 boxes
      // leave as TMA tile stores (clipped at the tensor's last row); a box that would cross into the
      // next slice, and scattered rows, take the row-segment stores
      bool box_tma = c_tma && rt.rows > q * 32 && (p.uniform_rows == 0 || rt.rows >= q * 32 + 32);
      if (box_tma && p.row_dst != nullptr) {  // scattered rows (pit:m union rows): runs of 32 go by TMA
        const int row0 = __shfl_sync(0xffffffffu, row, 0);
        box_tma = rt.rows >= q * 32 + 32 && __all_sync(0xffffffffu, row == row0 + lane);
      }
      const int box_row0 = p.row_dst != nullptr ? __shfl_sync(0xffffffffu, row, 0) : rt.base + q * 32;
#pragma unroll 1
      for (int bx = bx0; bx < bx1; ++bx) {
        uint32_t v[64];
        const uint32_t ta = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * Cfg::BN + bx * 64);
        if (kb_first < kblocks) {
          tmem_ld32(ta, *reinterpret_cast<uint32_t(*)[32]>(v));
          tmem_ld32(ta + 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
          tmem_wait_ld();
        } else {  // masked with no live K-block anywhere: C is zero
#pragma unroll
          for (int j = 0; j < 64; ++j) v[j] = 0u;
        }
        if (box_tma && lane == 0) bulk_wait_read<0>();  // the previous box's store has read the staging
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float f[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            float x = __uint_as_float(v[8 * j + e]);
            if (p.act == 1) x = fmaxf(x, 0.0f);
            f[e] = x * scale;
          }
          st_shared_v4(box + lane * 128 + ((static_cast<uint32_t>(j) ^ static_cast<uint32_t>(lane & 7)) << 4),
                       pack2(f[0], f[1], kBF16), pack2(f[2], f[3], kBF16), pack2(f[4], f[5], kBF16),
                       pack2(f[6], f[7], kBF16));
        }
        if (box_tma) {
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0 && n0 + bx * 64 < p.N) {
            tma_store_2d(&tmC, box, n0 + bx * 64, box_row0);
            bulk_commit();
          }
          continue;
        }
        __syncwarp();
        const int ch = lane & 7;
        const int col = n0 + bx * 64 + ch * 8;
#pragma unroll
        for (int it = 0; it < 8; ++it) {
          const int r = it * 4 + (lane >> 3);
          const int drow = __shfl_sync(0xffffffffu, row, r);
          const uint4 w = ld_shared_v4(box + r * 128 + ((static_cast<uint32_t>(ch) ^ static_cast<uint32_t>(r & 7)) << 4));
          if (drow >= 0 && col < p.N) {
            T* dst = C + static_cast<int64_t>(drow) * p.ldc + col;
            if (col + 8 <= p.N) {
              *reinterpret_cast<uint4*>(dst) = w;
            } else {
              const T* h = reinterpret_cast<const T*>(&w);
              for (int e = 0; e < p.N - col; ++e) dst[e] = h[e];
            }
          }
        }
        __syncwarp();  // the staging box is rewritten by the next iteration
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(leader_te + acc * 8);
      if (trace && q == 0 && half == 0 && lane == 0 && tu < 64) g_gk2_trace[640 + tu++] = gtimer();
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }

  if (epi_warp && lane == 0 && c_tma) bulk_wait<0>();  // TMA stores complete before exit
  tc_fence_before();
  cluster_sync();
  if (warp == kAlloc2Warp) {
    tc_fence_after();
    tmem_dealloc2<512>(tmem_base);
  }
}

// =============================================================================================
// rowgemm2t: grouped GEMMs (MoE experts) with the operand roles swapped — D^T = W^T . X^T on CTA
// pairs. The expert weights are the MMA's M side (256 output features per pair, MN-major straight
// from the [G, K, N] stack by TMA) and the group's tokens its N side (up to 256, in steps of 16:
// K-major rows, gathered by cp.async or one TMA box when packed). A group of ~128 tokens then costs
// one M=256 x N=128(+15) MMA chain instead of 1.5 row tiles of 128 (the token axis is quantised to
// 16, not 128), and each expert's weights are streamed once per 256 of its tokens.
// Epilogue: TMEM lane = output feature, column = token: per token, the warp's 32 features leave as
// one 64-byte row segment (ReLU / gate scale fused; destination row per token = SWrite).
// =============================================================================================
struct Rg2tCfg {
  static constexpr int KS = 64;
  static constexpr int W_BYTES = 2 * KS * 128;   // weights: the CTA's 128 features, 2 MN-major atoms
  static constexpr int X_BYTES = 128 * KS * 2;   // tokens: up to 128 K-major rows per CTA
  static constexpr int STAGE_BYTES = W_BYTES + X_BYTES;
  static constexpr int STAGE_BUDGET = 232448 - 2048 - 8 * 1025 * 4 - 4 * 2048;  // static pto + soff, staging
  static constexpr int STAGES = STAGE_BUDGET / STAGE_BYTES > 8 ? 8 : STAGE_BUDGET / STAGE_BYTES;
  static constexpr int STG_BYTES = 4 * 2048;  // per epilogue warp: [32 tokens x 32 features] bf16
  static constexpr size_t SMEM = static_cast<size_t>(STAGES) * STAGE_BYTES + STG_BYTES + 2048;
};

template <bool kBF16>
__global__ void __launch_bounds__(kThreads, 1)
    rowgemm2t_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                     const __grid_constant__ RowGemmParams p, int out_tiles, int max_tok_tiles) {
  using Cfg = Rg2tCfg;
  constexpr int KS = Cfg::KS;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stg = smem + Cfg::STAGES * Cfg::STAGE_BYTES;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(stg + Cfg::STG_BYTES);
  uint64_t* pair_full = full_bar + Cfg::STAGES;
  uint64_t* empty_bar = pair_full + Cfg::STAGES;
  uint64_t* tfull_bar = empty_bar + Cfg::STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);
  __shared__ int pto[kRg2MaxGroups + 1];  // prefix of 256-token tiles per group
  // packed row offsets of the groups when the caller gave none (p.off == nullptr): prefix of cnt
  __shared__ int soff[kRg2MaxGroups + 1];

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int pair = static_cast<int>(blockIdx.x >> 1);
  const int npairs = static_cast<int>(gridDim.x >> 1);
  if (path_skip(p)) return;  // both CTAs of the pair read the same flag
  // fp32 partial rows from packed tokens (A by TMA from one thread; stores straight from registers):
  // producer warps 4-7 take every other 32-token block of the epilogue beside warps 12-15
  const bool epi8 = p.a_tma != 0 && p.part != nullptr;
  const bool epi_warp = warp >= kEpiWarp0 || (epi8 && warp >= 4 && warp < kProdWarps);

  if (threadIdx.x == 0) {
    for (int i = 0; i < Cfg::STAGES; ++i) {
      mbar_init(&full_bar[i], p.a_tma ? 1 : kProdThreads + 1);
      mbar_init(&pair_full[i], 2);
      mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull_bar[i], 1);
      mbar_init(&tempty_bar[i], epi8 ? 16 : 8);
    }
    fence_mbar_init();
    tma_prefetch_desc(&tmW);
  }
  if (warp == kAlloc2Warp) tmem_alloc2<512>(tmem_slot);
  if (warp == kRelayWarp + 1) {
    const int per = (p.G + 31) / 32;
    const int g0 = lane * per;
    int run = 0;
    for (int g = g0; g < min(p.G, g0 + per); ++g) run += (__ldg(p.cnt + g) + 255) >> 8;
    int incl = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    int acc = incl - run;
    for (int g = g0; g < min(p.G, g0 + per); ++g) {
      pto[g] = acc;
      acc += (__ldg(p.cnt + g) + 255) >> 8;
    }
    if (lane == 31) pto[p.G] = incl;
    if (p.off == nullptr) {
      int trun = 0;
      for (int g = g0; g < min(p.G, g0 + per); ++g) trun += __ldcg(p.cnt + g);
      int tincl = trun;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, tincl, o);
        if (lane >= o) tincl += y;
      }
      int tacc = tincl - trun;
      for (int g = g0; g < min(p.G, g0 + per); ++g) {
        soff[g] = tacc;
        tacc += __ldcg(p.cnt + g);
      }
    }
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int units = min(max_tok_tiles, pto[p.G]) * out_tiles;
  const int kblocks = (p.K + KS - 1) / KS;
  // unit -> (group g, token range [start, start + ntok) of g, output-feature tile ot)
  struct TokTile {
    int g, start, ntok, nmma;
  };
  auto decode = [&](int u) {
    const int pt = u / out_tiles;
    int lo = 0, hi = p.G;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (pto[mid] <= pt) lo = mid; else hi = mid;
    }
    const int start = (pt - pto[lo]) * 256;
    const int ntok = min(256, __ldg(p.cnt + lo) - start);
    return TokTile{lo, start, ntok, (ntok + 15) & ~15};
  };

  if (warp < kProdWarps && !epi_warp) {
    // ------------------------------------------------------------ producers
    constexpr int CPR = KS * 2 / 16;
    constexpr int RPT = 128 * CPR / kProdThreads;
    constexpr int RSTEP = kProdThreads / CPR;
    const int tp = threadIdx.x;
    const int ch = tp % CPR;
    using T = typename OutT<kBF16>::T;
    const T* Xp = static_cast<const T*>(p.A);
    int stage = 0;
    uint32_t phase = 0;
    for (int u = (p.a_tma && tp != 0) ? units : pair; u < units; u += npairs) {
      const TokTile tt = decode(u);
      const int o0 = (u % out_tiles) * 256 + 128 * static_cast<int>(rank);
      const int half = tt.nmma >> 1;                                 // token rows this CTA feeds
      const int t0 = tt.start + static_cast<int>(rank) * half;      // first token (group-relative)
      const int tcnt = max(0, min(half, tt.ntok - static_cast<int>(rank) * half));
      int rid[RPT];
      if (!p.a_tma) {
#pragma unroll
        for (int j = 0; j < RPT; ++j) {
          const int i = tp / CPR + j * RSTEP;
          rid[j] = i < tcnt ? __ldg(p.row_src + static_cast<int64_t>(tt.g) * p.src_stride + t0 + i) : -1;
        }
      }
      const int xbase = (p.x_stride ? tt.g * p.x_stride : p.off ? __ldg(p.off + tt.g) : soff[tt.g]) + t0;  // packed rows
      for (int kb = 0; kb < kblocks; ++kb) {
        const int k0 = kb * KS;
        mbar_wait(&empty_bar[stage], phase ^ 1);
        uint8_t* sW = smem + stage * Cfg::STAGE_BYTES;
        uint8_t* sX = sW + Cfg::W_BYTES;
        if (tp == 0) {
          mbar_expect_tx_only(&full_bar[stage], Cfg::W_BYTES + (p.a_tma ? Cfg::X_BYTES : 0));
          tma_load_3d(sW, &tmW, &full_bar[stage], o0, k0, tt.g);
          tma_load_3d(sW + KS * 128, &tmW, &full_bar[stage], o0 + 64, k0, tt.g);
          if (p.a_tma) tma_load_2d(sX, &tmX, &full_bar[stage], k0, xbase);
          mbar_arrive(&full_bar[stage]);
        }
        if (!p.a_tma) {
          const uint32_t sx = smem_u32(sX);
          const int kc = k0 + ch * 8;
          const uint32_t kbytes = kc < p.K ? static_cast<uint32_t>(min(16, (p.K - kc) * 2)) : 0u;
#pragma unroll
          for (int j = 0; j < RPT; ++j) {
            const int row = tp / CPR + j * RSTEP;
            if (row >= half) continue;  // rows past N/2 are never read by the MMA
            const uint32_t bytes = rid[j] >= 0 ? kbytes : 0u;
            const T* src = bytes ? Xp + static_cast<int64_t>(rid[j]) * p.lda + kc : Xp;
            cp_async_16(sx + swz<7>(static_cast<uint32_t>(row * 128 + ch * 16)), src, bytes);
          }
        }
        if (!p.a_tma) cp_async_arrive_noinc(&full_bar[stage]);  // TMA-only stages: one arrival
        if (++stage == Cfg::STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == kRelayWarp) {
    if (lane == 0) {
      const uint32_t leader_pf = mapa_shared(smem_u32(pair_full), 0);
      int stage = 0;
      uint32_t phase = 0;
      for (int u = pair; u < units; u += npairs) {
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          fence_proxy_async_smem();
          mbar_arrive_cluster(leader_pf + stage * 8);
          if (++stage == Cfg::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == kMmaWarp) {
    if (rank == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int u = pair; u < units; u += npairs) {
        const TokTile tt = decode(u);
        const uint32_t idesc = idesc_f16(256, tt.nmma, kBF16, true, false);
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&pair_full[stage], phase);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t sW = smem_u32(smem + stage * Cfg::STAGE_BYTES);
            const uint32_t sX = sW + Cfg::W_BYTES;
#pragma unroll
            for (int ks = 0; ks < KS / 16; ++ks) {
              const uint64_t wdesc = smem_desc(sW + ks * 2048, KS * 128, 1024, kSw128);
              const uint64_t xdesc = smem_desc(sX + ks * 32, 16, 8 * 128, kSw128);
              umma2_f16(tmem_base + static_cast<uint32_t>(acc * 256), wdesc, xdesc, idesc, (kb > 0 || ks > 0) ? 1u : 0u);
            }
            umma2_commit_mc(&empty_bar[stage], 3);
          }
          __syncwarp();
          if (++stage == Cfg::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (lane == 0) umma2_commit_mc(&tfull_bar[acc], 3);
        __syncwarp();
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else if (epi_warp) {
    // ------------------------------------------------------------ epilogue: lane = output feature
    using T = typename OutT<kBF16>::T;
    const int q = warp & 3;
    const int half = warp < kProdWarps ? 1 : 0;  // epi8: warps 4-7 take the odd 32-token blocks
    const int cstep = epi8 ? 64 : 32;
    const uint32_t leader_te = mapa_shared(smem_u32(tempty_bar), 0);
    T* C = static_cast<T*>(p.C);
    const uint32_t stg_w = smem_u32(stg) + static_cast<uint32_t>(q * 2048);  // (bf16 path: 4 warps only)
    const bool vec_ok = (p.ldc % 8) == 0 && (reinterpret_cast<uintptr_t>(p.C) & 15) == 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = pair; u < units; u += npairs) {
      const TokTile tt = decode(u);
      const int ocw = (u % out_tiles) * 256 + 128 * static_cast<int>(rank) + q * 32;  // warp's features
      const int gbase = p.off ? __ldg(p.off + tt.g) : soff[tt.g];
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
#pragma unroll 1
      if (p.part != nullptr) {
        // fp32 partial rows: lane = feature, one coalesced 128-byte segment per token; two 32-token
        // blocks of TMEM in flight per wait (the warp's blocks are 64 tokens apart with 8 warps)
        const int f = ocw + lane;
#pragma unroll 1
        for (int c = half * 32; c < tt.ntok; c += 2 * cstep) {
          uint32_t v[2][32];
          const bool two = c + cstep < tt.ntok;
          tmem_ld32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * 256 + c), v[0]);
          if (two)
            tmem_ld32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * 256 + c + cstep),
                      v[1]);
          tmem_wait_ld();
#pragma unroll
          for (int b = 0; b < 2; ++b) {
            const int cb = c + b * cstep;
            if (b == 1 && !two) break;
            float* prow = static_cast<float*>(p.part) + (static_cast<int64_t>(gbase) + tt.start + cb) * p.N + f;
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (cb + j < tt.ntok && f < p.N) prow[static_cast<int64_t>(j) * p.N] = __uint_as_float(v[b][j]);
          }
        }
      }
#pragma unroll 1
      for (int c = half * 32; p.part == nullptr && c < tt.ntok; c += cstep) {
        uint32_t v[32];
        tmem_ld32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * 256 + c), v);
        tmem_wait_ld();
        // destination row and scale of token c + lane
        const int within = tt.start + c + lane;
        int my_row = -1;
        float my_scale = 1.0f;
        if (c + lane < tt.ntok) {
          my_row = p.row_dst ? __ldg(p.row_dst + static_cast<int64_t>(tt.g) * p.dst_stride + within) : gbase + within;
          if (p.row_scale) my_scale = __ldg(p.row_scale + my_row);
        }
        // transpose through shared memory: [token][32 features] rows of 64 bytes, then 8 tokens x
        // 64 bytes per store instruction (4 lanes per token row)
        __syncwarp();  // the previous block's read-back is done
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float sc = __shfl_sync(0xffffffffu, my_scale, j);
          float x = __uint_as_float(v[j]);
          if (p.act == 1) x = fmaxf(x, 0.0f);
          const T h = OutT<kBF16>::cvt(x * sc);
          asm volatile("st.shared.b16 [%0], %1;" ::"r"(stg_w + j * 64 + lane * 2),
                       "h"(*reinterpret_cast<const uint16_t*>(&h)) : "memory");
        }
        __syncwarp();
        const int sub = lane & 3;       // 16-byte quarter of the 64-byte feature segment
        const int col = ocw + sub * 8;  // first feature of this lane's quarter
#pragma unroll
        for (int it = 0; it < 4; ++it) {
          const int t = it * 8 + (lane >> 2);
          const int row = __shfl_sync(0xffffffffu, my_row, t);
          const uint4 w = ld_shared_v4(stg_w + t * 64 + sub * 16);
          if (row >= 0 && col < p.N) {
            T* dst = C + static_cast<int64_t>(row) * p.ldc + col;
            if (col + 8 <= p.N && vec_ok) {
              *reinterpret_cast<uint4*>(dst) = w;
            } else {
              const T* hh = reinterpret_cast<const T*>(&w);
              for (int e2 = 0; e2 < 8 && col + e2 < p.N; ++e2) dst[e2] = hh[e2];
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(leader_te + acc * 8);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }

  tc_fence_before();
  cluster_sync();
  if (warp == kAlloc2Warp) {
    tc_fence_after();
    tmem_dealloc2<512>(tmem_base);
  }
}

int g_num_sms = 0;

int num_sms() {
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}


int tma_store_enabled() {  // PIT_TMA_STORE=0: per-thread row stores (A/B knob)
  static int v = [] {
    const char* e = getenv("PIT_TMA_STORE");
    return e ? atoi(e) : 1;
  }();
  return v;
}

// Diagnostic knob (PIT_GK2_DIAG): bit 0 skips the MMAs, bit 1 the operand copies, bit 2 the C
// stores, bit 4 records the CTA-pair stage timeline — isolates the gather pipeline, the tensor pipe
// and the epilogue when profiling. Results are wrong with any of bits 0-2 set.
int gk2_diag() {
  static int v = [] {
    const char* e = getenv("PIT_GK2_DIAG");
    return e ? atoi(e) : 0;
  }();
  return v;
}

int gk_split_enabled() {  // PIT_GK_SPLIT=0: no split units (A/B knob)
  static int v = [] {
    const char* e = getenv("PIT_GK_SPLIT");
    return e ? atoi(e) : 1;
  }();
  return v;
}

// Scratch for split units (counters | partial tiles); 0 when the case does not use them: many units
// balance by themselves, and the CTA's unit list must fit kSplitUnitsMax.
template <int NT>
int64_t gk_split_ws_bytes(int64_t n_groups, int n_tiles) {
  if (!gk_split_enabled() || n_tiles != 1 || n_groups * n_tiles >= 4ll * num_sms() || n_groups > kSplitMaxGroups)
    return 0;
  return kSplitCtrBytes + (n_groups + kSplitParts) * 16 + static_cast<int64_t>(kSplitParts) * 128 * NT * 4;
}

// Tensor maps for the run path of spmm_gk (orientation N, 128-row groups): A^T [K, M] and B stacked
// [batch * K, N], boxes of one 64-column atom x the warp's rows; 0 when the case does not apply.
template <int GW, bool kOrientN, bool kBF16, int kKS, int kNT>
int gk_run_maps(const SpmmArgs& a, CUtensorMap* tmAt, CUtensorMap* tmBr) {
  memset(tmAt, 0, sizeof(*tmAt));
  memset(tmBr, 0, sizeof(*tmBr));
  static const int env = [] {
    const char* e = getenv("PIT_GK_RUNS");  // PIT_GK_RUNS=0: gathered rows only (A/B knob)
    return e ? atoi(e) : 1;
  }();
  if (!kOrientN || GW != 128 || !env || a.t0 != 128 || a.M % 128 != 0 || (a.sak * 2) % 16 != 0 ||
      (a.ldb * 2) % 16 != 0 || (reinterpret_cast<uintptr_t>(a.A) & 15) != 0 || (reinterpret_cast<uintptr_t>(a.B) & 15) != 0 ||
      (a.batch > 1 && a.b_batch_stride != a.K * a.ldb))
    return 0;
  constexpr int RW = kKS / kProdWarps;
  const CUtensorMapDataType dt = kBF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  if (encode_tensor_map_2d(tmAt, dt, a.A, static_cast<uint64_t>(a.M), static_cast<uint64_t>(a.K),
                           static_cast<uint64_t>(a.sak) * 2, 64, RW, CU_TENSOR_MAP_SWIZZLE_128B) != CUDA_SUCCESS ||
      encode_tensor_map_2d(tmBr, dt, a.B, static_cast<uint64_t>(a.N), static_cast<uint64_t>(a.K * (a.batch > 1 ? a.batch : 1)),
                           static_cast<uint64_t>(a.ldb) * 2, 64, RW, CU_TENSOR_MAP_SWIZZLE_128B) != CUDA_SUCCESS) {
    cudaGetLastError();
    return 0;
  }
  return 1;
}

template <int GW, bool kOrientN, bool kBF16, int kKS, int kNT>
int run_gk_split(const SpmmArgs& a, cudaStream_t s, const CUtensorMap& tmC, int epi, int n_tiles) {
  using Cfg = GkCfg<GW, kOrientN, kKS, kNT>;
  // scratch: counters (the last int = number of virtual groups) | vtab | partial tiles
  int* ctr = static_cast<int*>(a.ws);
  int4* vtab = reinterpret_cast<int4*>(ctr + kSplitCtrBytes / 4);
  float* parts = reinterpret_cast<float*>(vtab + a.n_groups + kSplitParts);
  // PIT_GK_SPLIT_FIRST (default 1): order split groups' chunks first; passed by value so the plan
  // launch is graph-capturable and every device sees it
  static const int split_first = [] {
    const char* e = getenv("PIT_GK_SPLIT_FIRST");
    return e ? atoi(e) : 1;
  }();
  gk_split_plan_kernel<<<1, 1024, 0, s>>>(a.counts, static_cast<int>(a.n_groups), Cfg::KS, vtab,
                                          ctr + kSplitCtrBytes / 4 - 1, ctr, split_first);
  note_launch();
  auto kern = spmm_gk_kernel<GW, kOrientN, kBF16, kKS, kNT, true>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(Cfg::SMEM));
  if (gk_split_enabled() >= 2) epi |= gk_split_enabled() == 2 ? 4 : 8;  // diagnostics: no reduce / no arrive
  // virtual groups <= n_groups + P: enough CTAs for the longest walk; idle CTAs exit at once
  const int64_t vunits = a.n_groups + kSplitParts;
  const int grid = static_cast<int>(vunits < num_sms() ? vunits : num_sms());
  CUtensorMap tmAt, tmBr;
  const int runs = gk_run_maps<GW, kOrientN, kBF16, kKS, kNT>(a, &tmAt, &tmBr);
  kern<<<grid, kThreads, Cfg::SMEM, s>>>(tmC, tmAt, tmBr, runs, epi, a.B, a.ldb, a.A, a.sak, a.counts, a.slots, a.slot_stride,
                                         static_cast<int>(a.n_groups), n_tiles, static_cast<int>(a.M),
                                         static_cast<int>(a.N), static_cast<int>(a.K), a.C, a.ldc,
                                         static_cast<int>(a.t0),
                                         static_cast<int>(a.batch > 1 ? a.n_groups / a.batch : a.n_groups),
                                         a.batch > 1 ? a.b_batch_stride : 0, ctr, parts);
  note_launch();
  return cuda_status();
}

template <int GW, bool kOrientN, bool kBF16, int kKS = 64, int kNT = 0>
int run_gk(const SpmmArgs& a, cudaStream_t s) {
  using Cfg = GkCfg<GW, kOrientN, kKS, kNT>;
  const int n_tiles = static_cast<int>(ceil_div(a.N, Cfg::N_TILE));
  const int64_t units = a.n_groups * n_tiles;
  if (units == 0) return kOk;
  if (units >= (1ll << 31)) return kErrShape;
  auto kern = spmm_gk_kernel<GW, kOrientN, kBF16, kKS, kNT>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(Cfg::SMEM));
  const int grid = static_cast<int>(units < num_sms() ? units : num_sms());
  // orientation N: C through TMA stores when whole 32-row warp blocks stay inside a group
  CUtensorMap tmC;
  memset(&tmC, 0, sizeof(tmC));
  int epi = 0;
  const bool c_ok = (reinterpret_cast<uintptr_t>(a.C) & 15) == 0 && (a.ldc * 2) % 16 == 0 && tma_store_enabled();
  const CUtensorMapDataType cdt = kBF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  if (kOrientN && a.t0 % 32 == 0 && c_ok) {
    if (encode_tensor_map_2d(&tmC, cdt, a.C, static_cast<uint64_t>(a.N), static_cast<uint64_t>(a.M),
                             static_cast<uint64_t>(a.ldc) * 2, 64, 32, CU_TENSOR_MAP_SWIZZLE_128B) != CUDA_SUCCESS)
      return kErrCuda;
    epi |= 1;
  } else if (!kOrientN && Cfg::STG_T > 0 && c_ok) {
    // orientation T: box = the group's rows x one warp's 32 columns (64-byte rows, no swizzle)
    if (encode_tensor_map_2d(&tmC, cdt, a.C, static_cast<uint64_t>(a.N), static_cast<uint64_t>(a.M),
                             static_cast<uint64_t>(a.ldc) * 2, 32, static_cast<uint32_t>(a.t0),
                             CU_TENSOR_MAP_SWIZZLE_NONE) != CUDA_SUCCESS)
      return kErrCuda;
    epi |= 1;
  }
  if (gk2_diag() & 4) epi |= 2;  // diagnostic: no C stores (orientation T)

  if constexpr (kOrientN && kNT == 64) {
    const int64_t need = gk_split_ws_bytes<Cfg::N_TILE>(a.n_groups, n_tiles);
    if (need > 0 && a.ws != nullptr && a.ws_bytes >= need && (reinterpret_cast<uintptr_t>(a.ws) & 255) == 0 &&
        a.n_groups * a.slot_stride < (1ll << 31))
      return run_gk_split<GW, kOrientN, kBF16, kKS, kNT>(a, s, tmC, epi, n_tiles);
  }
  // A column-major: A^T is row-major [K, M] with pitch sak
  CUtensorMap tmAt, tmBr;
  const int runs = gk_run_maps<GW, kOrientN, kBF16, kKS, kNT>(a, &tmAt, &tmBr);
  kern<<<grid, kThreads, Cfg::SMEM, s>>>(tmC, tmAt, tmBr, runs, epi, a.B, a.ldb, a.A, a.sak, a.counts, a.slots, a.slot_stride,
                                         static_cast<int>(a.n_groups), n_tiles, static_cast<int>(a.M),
                                         static_cast<int>(a.N), static_cast<int>(a.K), a.C, a.ldc,
                                         static_cast<int>(a.t0),
                                         static_cast<int>(a.batch > 1 ? a.n_groups / a.batch : a.n_groups),
                                         a.batch > 1 ? a.b_batch_stride : 0, nullptr, nullptr);
  note_launch();
  return cuda_status();
}

// CTA-pair gathered-K launch: one pair per co-resident cluster slot (persistent).
template <bool kBF16, int kKS>
int run_gk2(const SpmmArgs& a, cudaStream_t s) {
  using Cfg = Gk2Cfg<kKS>;
  const int n_tiles = static_cast<int>(ceil_div(a.N, Cfg::N_TILE));
  const int64_t units = a.n_groups * n_tiles;
  if (units == 0) return kOk;
  if (units >= (1ll << 31)) return kErrShape;
  auto kern = spmm_gk2_kernel<kBF16, kKS>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(Cfg::SMEM));
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = Cfg::SMEM;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  static int max_pairs = 0;  // co-resident clusters of 2 at this shared-memory footprint
  if (max_pairs == 0) {
    cfg.gridDim = dim3(static_cast<unsigned>(num_sms() & ~1));
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, kern, &cfg) != cudaSuccess || nc <= 0) {
      cudaGetLastError();
      nc = num_sms() / 2;
    }
    max_pairs = nc;
  }
  const int pairs = static_cast<int>(units < max_pairs ? units : max_pairs);
  cfg.gridDim = dim3(static_cast<unsigned>(2 * pairs));
  const int gpb = static_cast<int>(a.batch > 1 ? a.n_groups / a.batch : a.n_groups);
  // TMA-store epilogue: whole-warp row blocks must not straddle a group (t0 % 32 == 0) and C must be
  // a 16-byte aligned bf16/fp16 tensor with a 16-byte multiple pitch
  CUtensorMap tmC;
  int use_tma = a.t0 % 32 == 0 && (reinterpret_cast<uintptr_t>(a.C) & 15) == 0 && (a.ldc * 2) % 16 == 0 && tma_store_enabled();
  if (use_tma &&
      encode_tensor_map_2d(&tmC, kBF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, a.C,
                           static_cast<uint64_t>(a.N), static_cast<uint64_t>(a.M), static_cast<uint64_t>(a.ldc) * 2, 64,
                           32, CU_TENSOR_MAP_SWIZZLE_128B) != CUDA_SUCCESS)
    return kErrCuda;
  if (!use_tma) memset(&tmC, 0, sizeof(tmC));
  cudaLaunchKernelEx(&cfg, kern, tmC, use_tma, a.B, a.ldb, a.A, a.sak, a.counts, a.slots, a.slot_stride,
                     static_cast<int>(a.n_groups), n_tiles, static_cast<int>(a.M), static_cast<int>(a.N), a.C, a.ldc,
                     static_cast<int>(a.t0), gpb, a.batch > 1 ? a.b_batch_stride : int64_t{0}, gk2_diag());
  note_launch();
  return cuda_status();
}

int a_tma_enabled() {  // PIT_A_TMA=0: cp.async row copies for contiguous A as well (A/B knob)
  static int v = [] {
    const char* e = getenv("PIT_A_TMA");
    return e ? atoi(e) : 1;
  }();
  return v;
}

int gm_mask_tma_enabled() {  // PIT_GM_MASK_TMA=0: masked pit:m loads A by cp.async with zero-fill
  static int v = [] {
    const char* e = getenv("PIT_GM_MASK_TMA");
    return e ? atoi(e) : 1;
  }();
  return v;
}

template <int KS, bool kBF16, int kBN>
int run_rowgemm(const RowGemmParams& p, const void* B, int64_t ldb, int64_t group_stride, cudaStream_t s) {
  using Cfg = GmCfg<KS, kBN>;
  const CUtensorMapDataType dt = kBF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  CUtensorMap tmB;
  // B: stacked [G, K, N] (row-major per group, pitch ldb), box {64 n, KS k, 1 group}
  const uint64_t gstride = static_cast<uint64_t>(group_stride > 0 ? group_stride : ldb * p.K) * 2;
  if (encode_tensor_map_3d(&tmB, dt, B, p.N, p.K, p.G, ldb * 2, gstride, 64, KS,
                           CU_TENSOR_MAP_SWIZZLE_128B) != CUDA_SUCCESS)
    return kErrCuda;
  const int n_tiles = static_cast<int>(ceil_div(p.N, Cfg::BN));
  const int64_t units = static_cast<int64_t>(p.max_tiles) * n_tiles;
  if (units == 0) return kOk;
  if (units >= (1ll << 31)) return kErrShape;
  // A by TMA when every tile is 128 consecutive source rows (dense, batched slices, packed groups)
  CUtensorMap tmA;
  memset(&tmA, 0, sizeof(tmA));
  RowGemmParams q = p;
  q.a_tma = 0;
  q.mask_tma = 0;
  // staged contiguous rows (batched pit:m, or 2-D pit:m that goes contiguous on the device): A tiles
  // by TMA with the dead micro-tiles zeroed in shared memory (mask mode)
  const bool mask_ok = p.occ != nullptr && (p.row_src == nullptr || p.contig_pct > 0) && (p.lda * 2) % 16 == 0 &&
                       (reinterpret_cast<uintptr_t>(p.A) & 15) == 0 && gm_mask_tma_enabled() && a_tma_enabled();
  if (mask_ok) {
    if (encode_tensor_map_2d(&tmA, dt, p.A, static_cast<uint64_t>(p.K), static_cast<uint64_t>(p.M),
                             static_cast<uint64_t>(p.lda) * 2, KS, 128,
                             KS * 2 >= 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                             : KS * 2 == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B) != CUDA_SUCCESS)
      return kErrCuda;
    q.mask_tma = 1;
  } else if (p.row_src == nullptr && p.occ == nullptr && (p.lda * 2) % 16 == 0 &&
      (reinterpret_cast<uintptr_t>(p.A) & 15) == 0 && a_tma_enabled()) {
    if (encode_tensor_map_2d(&tmA, dt, p.A, static_cast<uint64_t>(p.K), static_cast<uint64_t>(p.M),
                             static_cast<uint64_t>(p.lda) * 2, KS, 128,
                             KS * 2 >= 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                             : KS * 2 == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B) != CUDA_SUCCESS)
      return kErrCuda;
    q.a_tma = 1;
  }
  auto kern = rowgemm_kernel<KS, kBF16, kBN>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(Cfg::SMEM));
  const int grid = static_cast<int>(units < num_sms() ? units : num_sms());
  kern<<<grid, kThreads, Cfg::SMEM, s>>>(tmB, tmA, q, n_tiles);
  note_launch();
  return cuda_status();
}

int rg2_c_tma_enabled() {  // PIT_RG2_CTMA=0: rowgemm2 stores C by row segments only (A/B knob)
  static int v = [] {
    const char* e = getenv("PIT_RG2_CTMA");
    return e ? atoi(e) : 1;
  }();
  return v;
}

int rg2_epi8_enabled() {  // PIT_RG2_EPI8=0: rowgemm2 drains TMEM with 4 warps only (A/B knob)
  static int v = [] {
    const char* e = getenv("PIT_RG2_EPI8");
    return e ? atoi(e) : 1;
  }();
  return v;
}

int rg2_enabled() {  // PIT_RG2=0: single-CTA rowgemm for the dense / contiguous-row cases too
  static int v = [] {
    const char* e = getenv("PIT_RG2");
    return e ? atoi(e) : 1;
  }();
  return v;
}

int rg2_grouped() {  // PIT_RG2_GROUPED=0: grouped (MoE) GEMMs stay on single-CTA 128-row tiles
  static int v = [] {
    const char* e = getenv("PIT_RG2_GROUPED");
    return e ? atoi(e) : 1;
  }();
  return v;
}

// CTA-pair launch of the dense / contiguous-row rowgemm cases (see rowgemm2_kernel).

// Clears the C rows whose bit in a single-group pit:m bitmap is 0 (a warp per row, 16-byte stores).
__global__ void __launch_bounds__(256) zero_dead_rows_kernel(const uint32_t* __restrict__ occ, int64_t M,
                                                             uint8_t* __restrict__ C, int64_t ld_bytes,
                                                             int64_t row_bytes) {
  const int64_t row = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (row >= M || ((__ldg(occ + (row >> 5)) >> (row & 31)) & 1u)) return;
  uint4* dst = reinterpret_cast<uint4*>(C + row * ld_bytes);
  for (int64_t i = threadIdx.x & 31; i < row_bytes / 16; i += 32) dst[i] = make_uint4(0u, 0u, 0u, 0u);
}

template <bool kBF16>
int run_rowgemm2(const RowGemmParams& p, const void* B, int64_t ldb, int64_t group_stride, cudaStream_t s) {
  using Cfg = Rg2Cfg;
  constexpr int KS = Cfg::KS;
  const CUtensorMapDataType dt = kBF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  CUtensorMap tmB, tmA;
  memset(&tmA, 0, sizeof(tmA));
  const uint64_t gstride = static_cast<uint64_t>(group_stride > 0 ? group_stride : ldb * p.K) * 2;
  if (encode_tensor_map_3d(&tmB, dt, B, p.N, p.K, p.G, ldb * 2, gstride, 64, KS, CU_TENSOR_MAP_SWIZZLE_128B) !=
      CUDA_SUCCESS)
    return kErrCuda;
  RowGemmParams q = p;
  q.a_tma = 0;
  q.epi8 = rg2_epi8_enabled();
  static const int lagged_env = [] {
    const char* e = getenv("PIT_RG2_LAGGED");
    return e ? atoi(e) : 0;
  }();
  q.lagged = lagged_env;
  if (p.row_src == nullptr && (p.lda * 2) % 16 == 0 && (reinterpret_cast<uintptr_t>(p.A) & 15) == 0 &&
      a_tma_enabled() && (!p.masked || gm_mask_tma_enabled())) {
    if (encode_tensor_map_2d(&tmA, dt, p.A, static_cast<uint64_t>(p.K), static_cast<uint64_t>(p.a_rows ? p.a_rows : p.M),
                             static_cast<uint64_t>(p.lda) * 2, KS, 128, CU_TENSOR_MAP_SWIZZLE_128B) != CUDA_SUCCESS)
      return kErrCuda;
    q.a_tma = 1;
  }
  // C by TMA tile stores when the destination rows are consecutive (no scatter list, no groups)
  CUtensorMap tmC;
  memset(&tmC, 0, sizeof(tmC));
  int c_tma = 0;
  if (p.cnt == nullptr && (p.ldc * 2) % 16 == 0 &&
      (reinterpret_cast<uintptr_t>(p.C) & 15) == 0 && rg2_c_tma_enabled()) {
    const uint64_t crows = static_cast<uint64_t>(p.uniform_rows ? static_cast<int64_t>(p.G) * p.uniform_rows : p.M);
    if (encode_tensor_map_2d(&tmC, dt, p.C, static_cast<uint64_t>(p.N), crows, static_cast<uint64_t>(p.ldc) * 2, 64,
                             32, CU_TENSOR_MAP_SWIZZLE_128B) != CUDA_SUCCESS)
      return kErrCuda;
    c_tma = 1;
  }
  const int rows = p.uniform_rows ? p.uniform_rows : p.max_tiles * 128;
  // grouped: the device prefix decides; max_tiles (128-row tiles) bounds the pair tiles
  const int pair_tiles = static_cast<int>(p.cnt ? p.max_tiles
                                          : p.uniform_rows ? p.G * ceil_div(p.uniform_rows, 256) : ceil_div(rows, 256));
  const int n_tiles = static_cast<int>(ceil_div(p.N, Cfg::BN));
  const int64_t units = static_cast<int64_t>(pair_tiles) * n_tiles;
  if (units == 0) {
    if (p.zero_occ != nullptr) {  // no live row: every row of C is a dead row
      zero_dead_rows_kernel<<<static_cast<unsigned>(ceil_div(p.M, 8)), 256, 0, s>>>(
          p.zero_occ, p.M, static_cast<uint8_t*>(p.C), p.ldc * 2, static_cast<int64_t>(p.N) * 2);
      note_launch();
      return cuda_status();
    }
    return kOk;
  }
  if (units >= (1ll << 31)) return kErrShape;
  auto kern = rowgemm2_kernel<kBF16>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(Cfg::SMEM));
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = Cfg::SMEM;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  static int max_pairs = 0;
  if (max_pairs == 0) {
    cfg.gridDim = dim3(static_cast<unsigned>(num_sms() & ~1));
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, kern, &cfg) != cudaSuccess || nc <= 0) {
      cudaGetLastError();
      nc = num_sms() / 2;
    }
    max_pairs = nc;
  }
  const int pairs = static_cast<int>(units < max_pairs ? units : max_pairs);
  cfg.gridDim = dim3(static_cast<unsigned>(2 * pairs));
  cudaLaunchKernelEx(&cfg, kern, tmB, tmA, tmC, q, n_tiles, pair_tiles, c_tma);
  note_launch();
  return cuda_status();
}

int small_single_enabled() {  // PIT_SMALL_SINGLE=0: small gathered-row products stay on CTA pairs
  static int v = [] {
    const char* e = getenv("PIT_SMALL_SINGLE");
    return e ? atoi(e) : 1;
  }();
  return v;
}

template <bool kBF16>
int rowgemm_dispatch(const RowGemmParams& p, const void* B, int64_t ldb, int ks, cudaStream_t s,
                     int64_t group_stride = 0) {
  // dense / contiguous-row cases (no liveness, one group or uniform slices, N > 128) on CTA pairs.
  // A single product with fewer than 4 pair units per cluster slot (BERT FFN1: 4096 x 768 x 3072)
  // is latency-bound either way and measured faster on the single-CTA tiles (2x the units).
  const int64_t pair_units = ceil_div(static_cast<int64_t>(p.max_tiles) * 128, 256) * ceil_div(p.N, 256);
  const bool small_single = p.cnt == nullptr && p.uniform_rows == 0 && p.row_src != nullptr &&
                            pair_units < 2ll * num_sms() && small_single_enabled();
  if (ks == 64 && p.N > 128 && p.occ == nullptr && (p.cnt == nullptr || (p.G <= kRg2MaxGroups && rg2_grouped())) &&
      (p.ldc % 8) == 0 && (reinterpret_cast<uintptr_t>(p.C) & 15) == 0 && rg2_enabled() && !small_single)
    return run_rowgemm2<kBF16>(p, B, ldb, group_stride, s);
  if (p.zero_occ != nullptr) {  // the single-CTA kernels do not clear dead rows themselves
    zero_dead_rows_kernel<<<static_cast<unsigned>(ceil_div(p.M, 8)), 256, 0, s>>>(
        p.zero_occ, p.M, static_cast<uint8_t*>(p.C), p.ldc * 2, static_cast<int64_t>(p.N) * 2);
    note_launch();
  }
  if (p.N <= 64) {  // narrow products: 64-column units, no zero-filled B atoms or idle MMA columns
    if (ks == 64) return run_rowgemm<64, kBF16, 64>(p, B, ldb, group_stride, s);
    if (ks == 32) return run_rowgemm<32, kBF16, 64>(p, B, ldb, group_stride, s);
    if (ks == 16) return run_rowgemm<16, kBF16, 64>(p, B, ldb, group_stride, s);
    return kErrUnsupported;
  }
  if (ks == 64) return run_rowgemm<64, kBF16, 256>(p, B, ldb, group_stride, s);
  if (ks == 32) return run_rowgemm<32, kBF16, 256>(p, B, ldb, group_stride, s);
  if (ks == 16) return run_rowgemm<16, kBF16, 256>(p, B, ldb, group_stride, s);
  return kErrUnsupported;
}

// Clears C unless the union covers >= pct% of the rows (then the contiguous-tile kernel writes every
// row itself): the decision is the kernels' own, read on the device.
__global__ void __launch_bounds__(256) zero_unless_contig_kernel(const int32_t* __restrict__ n_rows, int pct,
                                                                 int64_t M, uint8_t* __restrict__ C, int64_t ld_bytes,
                                                                 int64_t chunks_per_row, const int* __restrict__ sparse) {
  if (static_cast<int64_t>(*n_rows) * 100 >= M * pct) return;
  if (sparse != nullptr && *sparse) return;  // the high-sparsity path writes every row of C
  const int64_t total = M * chunks_per_row;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / chunks_per_row, c = i - r * chunks_per_row;
    reinterpret_cast<uint4*>(C + r * ld_bytes)[c] = make_uint4(0u, 0u, 0u, 0u);
  }
}

// One-K-group pit:m over gathered rows (BERT's padding removal): the live rows of A are copied
// contiguous into caller scratch first (a warp per row, 16-byte copies, L2-resident right after
// detection), so the CTA-pair GEMM loads A by TMA like a dense product. cp.async gathers of the
// same rows held the pair mainloop at ~0.7 us per stage against 0.45 with TMA-fed A (the L2->SM
// feed of 16-byte copies next to the TMA B tiles, scripts/rg2_trace.py).
__global__ void __launch_bounds__(256) pack_rows_kernel(const uint8_t* __restrict__ A, int64_t lda_bytes,
                                                        const int32_t* __restrict__ rows,
                                                        const int32_t* __restrict__ n_rows, int64_t row_bytes,
                                                        uint8_t* __restrict__ out) {
  const int n = *n_rows;
  const int lane = threadIdx.x & 31;
  const int64_t chunks = row_bytes >> 4;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5); i < n;
       i += static_cast<int64_t>(gridDim.x) * 8) {
    const uint4* src = reinterpret_cast<const uint4*>(A + static_cast<int64_t>(__ldg(rows + i)) * lda_bytes);
    uint4* dst = reinterpret_cast<uint4*>(out + i * row_bytes);
    for (int64_t c = lane; c < chunks; c += 32) dst[c] = __ldg(src + c);
  }
}

int gm_pack_enabled() {  // PIT_GM_PACK=0: one-K-group pit:m gathers its rows by cp.async (A/B knob)
  static int v = [] {
    const char* e = getenv("PIT_GM_PACK");
    return e ? atoi(e) : 1;
  }();
  return v;
}

// bytes of scratch run_gm packs the live rows into (0: the case does not pack)
int64_t gm_pack_bytes(const SpmmArgs& a) {
  if (a.plan != kPlanPitM || ceil_div(a.K, a.t1) != 1 || a.rows == nullptr || a.n_rows == nullptr || a.N <= 128 ||
      a.sak != 1 || (a.K * 2) % 16 != 0 || (a.sam * 2) % 16 != 0 || (reinterpret_cast<uintptr_t>(a.A) & 15) != 0 ||
      !gm_pack_enabled() || !rg2_enabled())
    return 0;
  return a.n_rows_host * a.K * 2;
}

int gm_sparse_enabled() {  // PIT_GM_SPARSE=0: no high-sparsity pit:m path (A/B knob)
  static int v = [] {
    const char* e = getenv("PIT_GM_SPARSE");
    return e ? atoi(e) : 1;
  }();
  return v;
}

// 2-D pit:m products the high-sparsity path (pit_gm_sparse.cu) can take: 16/32-wide micro-columns,
// K in 256-column supergroups, 16-byte aligned row-major A and C
bool gm_sparse_capable(const SpmmArgs& a) {
  if (a.plan != kPlanPitM || a.occ == nullptr || a.counts == nullptr || !(a.t1 == 16 || a.t1 == 32) ||
      a.K % gm_sg() != 0 || ceil_div(a.K, a.t1) <= 1 || a.sak != 1 || (a.sam * 2) % 16 != 0 ||
      (reinterpret_cast<uintptr_t>(a.A) & 15) != 0 || (a.ldc % 8) != 0 || (a.N % 8) != 0 ||
      (reinterpret_cast<uintptr_t>(a.C) & 15) != 0 || a.M >= (1 << 24) || !gm_sparse_enabled() || !a_tma_enabled())
    return false;
  const int64_t S = a.K / gm_sg();
  return S <= kRg2MaxGroups && S * a.WG <= 8192;
}

int64_t gm_sparse_ws_bytes(const SpmmArgs& a) {
  if (!gm_sparse_capable(a)) return 0;
  const int S = static_cast<int>(a.K / gm_sg());
  return gm_sparse_layout(a.M, a.N, a.WG, S, gm_sparse_bound_rows(a.M, a.K / a.t1, S)).bytes;
}

int gm_pairs_enabled() {  // PIT_GM_PAIRS=0: contiguous pit:m stays on the single-CTA rowgemm
  static int v = [] {
    const char* e = getenv("PIT_GM_PAIRS");
    return e ? atoi(e) : 1;
  }();
  return v;
}

int gm_contig_pct() {  // PIT_GM_CONTIG=P: pit:m runs on contiguous row tiles when the union holds >= P% of rows
  static int v = [] {
    const char* e = getenv("PIT_GM_CONTIG");
    return e ? atoi(e) : 50;
  }();
  return v;
}

// 2-D pit:m cases whose kernels switch to contiguous row tiles on the device when the union holds
// >= PIT_GM_CONTIG % of the rows (scattered per-row K patterns over 16/32-wide micro-columns)
bool gm_contig_capable(const SpmmArgs& a) {
  return a.plan == kPlanPitM && a.occ != nullptr && a.n_rows != nullptr && (a.t1 == 32 || a.t1 == 16) &&
         ceil_div(a.K, a.t1) > 1 && a.n_rows_host == a.M && ceil_div(a.K, a.t1) <= GmCfg<64>::OCC_MAX_GROUPS &&
         ceil_div(a.K, 64) <= GmCfg<64>::KB_MAX && gm_contig_pct() > 0;
}

}  // namespace
template <bool kBF16>
int run_rowgemm2t(const RowGemmParams& p, const void* B, int64_t ldb, cudaStream_t s);  // below
namespace {

template <bool kBF16>
int run_gm(const SpmmArgs& a, int ks, cudaStream_t s) {
  const int dense = a.plan == kPlanDense ? 1 : 0;
  int zero_in_gemm = 0;
  // high-sparsity path (pit_gm_sparse.cu): its prep kernel decides on the device and publishes the
  // decision; the masked dense kernels below leave when it is set, the sparse kernels when it is not
  const int* sparse_flag = nullptr;
  GmSparseWs sw{};
  int sp_S = 0;
  int64_t sp_bound = 0;
  if (!dense && gm_sparse_capable(a) && a.ws != nullptr && a.ws_bytes >= gm_sparse_ws_bytes(a)) {
    sp_S = static_cast<int>(a.K / gm_sg());
    sp_bound = gm_sparse_bound_rows(a.M, a.K / a.t1, sp_S);
    sw = gm_sparse_layout(a.M, a.N, a.WG, sp_S, sp_bound);
    uint8_t* ws = static_cast<uint8_t*>(a.ws);
    if (int st = launch_gm_sparse_prep(a.counts, static_cast<int>(ceil_div(a.K, a.t1)), a.M, gm_sg() / a.t1, sp_S, a.occ,
                                       a.WG, ws, sw, s))
      return st;
    sparse_flag = reinterpret_cast<const int*>(ws + sw.flag);
  }
  if (!dense) {
    // rows named by no group stay exactly zero. One K-group (BERT's row-uniform micro-tiles): only
    // the dead rows are written (the union is that group's bitmap); otherwise all of C is cleared.
    if (ceil_div(a.K, a.t1) == 1 && a.occ != nullptr && (a.ldc % 8) == 0 && (a.N % 8) == 0 &&
        (reinterpret_cast<uintptr_t>(a.C) & 15) == 0) {
      zero_in_gemm = 1;  // rowgemm2 clears them beside its mainloop; rowgemm_dispatch launches the
                         // clearing kernel itself when it picks another kernel
    } else if (gm_contig_capable(a) && (a.ldc % 8) == 0 && (a.N % 8) == 0 &&
               (reinterpret_cast<uintptr_t>(a.C) & 15) == 0) {
      // the contiguous-tile kernels write every row: clear C only if the union-row kernel runs
      const int64_t chunks = a.M * (a.N / 8);
      const int64_t blocks = ceil_div(chunks, 256);
      const int64_t cap = static_cast<int64_t>(num_sms()) * 8;
      zero_unless_contig_kernel<<<static_cast<unsigned>(blocks < cap ? blocks : cap), 256, 0, s>>>(
          a.n_rows, gm_contig_pct(), a.M, static_cast<uint8_t*>(a.C), a.ldc * 2, a.N / 8, sparse_flag);
      note_launch();
    } else if (cudaMemset2DAsync(a.C, a.ldc * 2, 0, a.N * 2, a.M, s) != cudaSuccess) {
      return cuda_status();
    }
  }
  RowGemmParams p{};
  p.A = a.A;
  p.lda = a.sam;
  p.C = a.C;
  p.ldc = a.ldc;
  p.M = static_cast<int>(a.M);
  p.N = static_cast<int>(a.N);
  p.K = static_cast<int>(a.K);
  p.G = 1;
  p.n_rows = dense ? nullptr : a.n_rows;
  p.row_src = dense ? nullptr : a.rows;
  p.row_dst = dense ? nullptr : a.rows;
  // one K-group (micro-tile spans all of K, e.g. BERT's row-uniform (1, K)): every union row is live
  // in every K-block, so no per-row liveness lookups or per-stage votes
  p.occ = (dense || ceil_div(a.K, a.t1) == 1) ? nullptr : a.occ;
  p.WG = a.WG;
  p.t1 = dense ? 1 : a.t1;
  p.max_tiles = static_cast<int>(ceil_div(dense ? a.M : a.n_rows_host, 128));
  p.zero_occ = zero_in_gemm ? a.occ : nullptr;
  if (sparse_flag != nullptr) {
    // SRead into packed rows -> supergroup products (fp32 partial rows) -> ordered row sums into C
    uint8_t* ws = static_cast<uint8_t*>(a.ws);
    const int nkg = static_cast<int>(ceil_div(a.K, a.t1));
    if (int st = launch_gm_sparse_pack(a.counts, nkg, a.A, a.sam * 2, sp_S, a.M, a.occ, a.WG, a.t1, sp_bound, ws, sw, s))
      return st;
    RowGemmParams q{};
    q.A = ws + sw.X;
    q.lda = gm_sg();
    q.M = static_cast<int>(sp_bound);  // packed rows (bounds of the TMA map)
    q.C = a.C;
    q.ldc = a.ldc;
    q.N = static_cast<int>(a.N);
    q.K = gm_sg();
    q.G = sp_S;
    q.cnt = reinterpret_cast<const int32_t*>(ws + sw.cnt);
    q.off = nullptr;  // the kernel derives the packed offsets from cnt
    q.max_tiles = static_cast<int>(ceil_div(sp_bound, 256) + sp_S);
    q.part = reinterpret_cast<float*>(ws + sw.part);
    q.path_flag = sparse_flag;
    q.path_role = 1;
    if (int st = run_rowgemm2t<kBF16>(q, a.B, a.ldb, s)) return st;
    if (int st = launch_gm_sparse_reduce(a.counts, nkg, a.dtype, sp_S, a.WG, a.N, a.C, a.ldc, a.M, ws, sw, s)) return st;
    p.path_flag = sparse_flag;
    p.path_role = 2;
  }
  const int64_t pack_bytes = gm_pack_bytes(a);
  if (pack_bytes > 0 && a.ws != nullptr && a.ws_bytes >= pack_bytes) {
    const int64_t blocks = ceil_div(a.n_rows_host, 8);
    const int64_t cap = static_cast<int64_t>(num_sms()) * 8;
    pack_rows_kernel<<<static_cast<unsigned>(blocks < cap ? blocks : cap), 256, 0, s>>>(
        static_cast<const uint8_t*>(a.A), a.sam * 2, a.rows, a.n_rows, a.K * 2, static_cast<uint8_t*>(a.ws));
    note_launch();
    p.A = a.ws;
    p.lda = a.K;
    p.a_rows = static_cast<int>(a.n_rows_host);  // rows of the packed operand (bounds of its TMA map)
    p.row_src = nullptr;                         // packed row i is union row i; C rows stay scattered
  }
  // Scattered per-row K patterns (random (1,32) activation sparsity) make the union of live rows
  // (nearly) every row: union-row tiles then buy nothing and cost a per-row, per-K-block global
  // liveness lookup plus a block-wide vote per stage. The kernel switches (on the device, from the
  // union size) to contiguous 128-row tiles: the tile's occupancy words are staged in shared memory
  // once per unit, a dead (row, micro-column) chunk is zero-filled by its cp.async, K-blocks with no
  // live row take no ring slot. 64-deep K-blocks cover two 32-wide (four 16-wide) micro-columns:
  // liveness is per 16-byte chunk's K-group.
  if (gm_contig_capable(a)) {
    p.contig_pct = gm_contig_pct();
    ks = 64;
    // N > 128: the contiguous case runs on CTA pairs (rowgemm2, 256 x 256 tiles, every K-block, dead
    // chunks zero-filled); both kernels are launched and each leaves on the device unless the union
    // size selects it
    if (p.contig_pct > 0 && a.N > 128 && a.counts != nullptr && rg2_enabled() && gm_pairs_enabled() && (a.ldc % 8) == 0 &&
        (reinterpret_cast<uintptr_t>(a.C) & 15) == 0 && ceil_div(a.K, a.t1) <= kRg2OccGroups) {
      RowGemmParams q = p;
      q.masked = 1;
      q.kg_cnt = a.counts;
      q.row_src = nullptr;
      q.row_dst = nullptr;
      q.max_tiles = static_cast<int>(ceil_div(a.M, 128));
      if (int st = run_rowgemm2<kBF16>(q, a.B, a.ldb, 0, s)) return st;
      p.exit_if_contig = 1;
    }
  }
  return rowgemm_dispatch<kBF16>(p, a.B, a.ldb, ks, s);
}

// Batched pit:m / dense (slices stacked along M, SpmmArgs::batch): every row of every slice is a
// unit row (no union list); the occupancy bitmap of the stacked index skips dead K-blocks per row
// tile, and tiles with no live block store zeros. B slice g at B + g * b_batch_stride.
template <bool kBF16>
int run_gm_batched(const SpmmArgs& a, int ks, cudaStream_t s) {
  const int dense = a.plan == kPlanDense ? 1 : 0;
  RowGemmParams p{};
  p.A = a.A;
  p.lda = a.sam;
  p.C = a.C;
  p.ldc = a.ldc;
  p.M = static_cast<int>(a.M * a.batch);
  p.N = static_cast<int>(a.N);
  p.K = static_cast<int>(a.K);
  p.G = static_cast<int>(a.batch);
  p.uniform_rows = static_cast<int>(a.M);
  p.occ = dense ? nullptr : a.occ;
  p.WG = a.WG;
  p.t1 = dense ? 1 : a.t1;
  p.max_tiles = static_cast<int>(a.batch * ceil_div(a.M, 128));
  return rowgemm_dispatch<kBF16>(p, a.B, a.ldb, ks, s, a.b_batch_stride);
}

// Tuning knob: PIT_GK_KS=64|128 overrides the gathered-K stage depth (defaults: 128, and 128 for the
// CTA-pair 256-row kernel; the single-CTA 256-row fallback runs 64 — measured on B200).
int gk_ks_override() {
  static int v = [] {
    const char* e = getenv("PIT_GK_KS");
    return e ? atoi(e) : 0;
  }();
  return v;
}

int gk2_enabled() {
  static int v = [] {
    const char* e = getenv("PIT_GK2");
    return e ? atoi(e) : 1;
  }();
  return v;
}

template <bool kBF16, int kNT>
int dispatch_gk(const SpmmArgs& a, int gw, cudaStream_t s) {
  const bool ks64 = gk_ks_override() == 64;
  switch (gw) {
    case 16:
      return ks64 ? run_gk<16, false, kBF16, 64, kNT>(a, s) : run_gk<16, false, kBF16, 128, kNT>(a, s);
    case 32:
      return ks64 ? run_gk<32, false, kBF16, 64, kNT>(a, s) : run_gk<32, false, kBF16, 128, kNT>(a, s);
    case 64:
      return ks64 ? run_gk<64, false, kBF16, 64, kNT>(a, s) : run_gk<64, false, kBF16, 128, kNT>(a, s);
    case 128:
      return ks64 ? run_gk<128, true, kBF16, 64, kNT>(a, s) : run_gk<128, true, kBF16, 128, kNT>(a, s);
    case 256:
      // N tiles of 256 columns: the CTA-pair kernel (PIT_GK2=0 selects the single-CTA one)
      if (kNT == 0 && gk2_enabled()) return gk_ks_override() == 64 ? run_gk2<kBF16, 64>(a, s) : run_gk2<kBF16, 128>(a, s);
      return run_gk<256, false, kBF16, 64, 128>(a, s);
    default:
      return kErrUnsupported;
  }
}

template <bool kBF16>
int dispatch_tc(const SpmmArgs& a, cudaStream_t s) {
  if (a.plan == kPlanPitK) {
    const int gw = a.t0 <= 16 ? 16 : a.t0 <= 32 ? 32 : a.t0 <= 64 ? 64 : a.t0 <= 128 ? 128 : 256;
    // narrow products (N <= 128, e.g. attention P.V) use 128-column units: no zero-filled half tile
    // (PIT_GK_NT=128 forces them for every N: a tuning knob)
    static const int nt_override = [] {
      const char* e = getenv("PIT_GK_NT");
      return e ? atoi(e) : 0;
    }();
    // 128-row groups (orientation N, N_mma = the n tile) with N <= 64 (attention P.V, head dim 64):
    // 64-column units — no zero-filled half tile, half the MMA columns
    if (gw == 128 && a.N <= 64 && nt_override != 128) {
      const bool ks64 = gk_ks_override() == 64;
      return ks64 ? run_gk<128, true, kBF16, 64, 64>(a, s) : run_gk<128, true, kBF16, 128, 64>(a, s);
    }
    // 16/32-row groups with wide N: 512-column units (64-deep stages). Each gathered k row brings
    // 1 KB of B for 64 B of A^T: 30.1 FLOP per gathered byte against 28.4 at 256 columns, and the
    // gather feed (L2 -> SM) is what bounds these micro-tiles (PIT_GK_NT=256 keeps 256)
    if ((gw == 16 || gw == 32) && a.N >= 1024 && nt_override != 256 && nt_override != 128) {
      return gw == 16 ? run_gk<16, false, kBF16, 64, 512>(a, s) : run_gk<32, false, kBF16, 64, 512>(a, s);
    }
    return (a.N <= 128 || nt_override == 128) ? dispatch_gk<kBF16, 128>(a, gw, s) : dispatch_gk<kBF16, 0>(a, gw, s);
  }
  const int t1 = a.plan == kPlanDense ? 64 : a.t1;
  if (a.batch > 1) {
    // 64-deep K-blocks for 16/32-wide micro-columns too: liveness is looked up per 16-byte chunk
    const int ks = (t1 % 64 == 0 || t1 == 32 || t1 == 16) ? 64 : 0;
    return ks ? run_gm_batched<kBF16>(a, ks, s) : kErrUnsupported;
  }
  if (t1 % 64 == 0) return run_gm<kBF16>(a, 64, s);
  if (t1 == 32) return run_gm<kBF16>(a, 32, s);
  if (t1 == 16) return run_gm<kBF16>(a, 16, s);
  return kErrUnsupported;
}

}  // namespace

int gk2_trace_read(unsigned long long* host) {
  return cudaMemcpyFromSymbol(host, g_gk2_trace, sizeof(g_gk2_trace)) == cudaSuccess ? kOk : kErrCuda;
}

bool spmm_tc_supported(const SpmmArgs& a) {
  if (a.dtype != kDtypeBF16 && a.dtype != kDtypeF16) return false;
  // TMA: 16-byte aligned bases and pitches, int32 coordinates
  if (a.M >= (1ll << 31) || a.N >= (1ll << 31) || a.K >= (1ll << 31)) return false;
  if (reinterpret_cast<uintptr_t>(a.A) % 16 || reinterpret_cast<uintptr_t>(a.B) % 16) return false;
  if ((a.ldb * 2) % 16) return false;
  if (a.plan == kPlanPitK) {
    if (a.sam != 1 || (a.sak * 2) % 16) return false;  // A column-major
    if (a.K * a.ldb >= (1ll << 31) || a.K * a.sak >= (1ll << 31)) return false;  // 32-bit byte offsets (2-byte elements)
    return a.t0 % 8 == 0 && a.t0 <= 256;  // narrower groups run in the next wider kernel
  }
  if (a.sak != 1 || (a.sam * 2) % 16) return false;  // A row-major
  if (a.plan == kPlanDense) return true;
  return a.t1 % 64 == 0 || a.t1 == 32 || a.t1 == 16;
}

int rg2t_enabled() {  // PIT_RG2T=0: grouped GEMMs keep tokens on the M side (rowgemm2 / rowgemm)
  static int v = [] {
    const char* e = getenv("PIT_RG2T");
    return e ? atoi(e) : 1;
  }();
  return v;
}

// Grouped GEMM with swapped roles (see rowgemm2t_kernel): weights on M, tokens on N.
template <bool kBF16>
int run_rowgemm2t(const RowGemmParams& p, const void* B, int64_t ldb, cudaStream_t s) {
  using Cfg = Rg2tCfg;
  constexpr int KS = Cfg::KS;
  const CUtensorMapDataType dt = kBF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  CUtensorMap tmW, tmX;
  memset(&tmX, 0, sizeof(tmX));
  if (encode_tensor_map_3d(&tmW, dt, B, p.N, p.K, p.G, ldb * 2, static_cast<uint64_t>(ldb * p.K) * 2, 64, KS,
                           CU_TENSOR_MAP_SWIZZLE_128B) != CUDA_SUCCESS)
    return kErrCuda;
  RowGemmParams q = p;
  q.a_tma = 0;
  if (p.row_src == nullptr && (p.lda * 2) % 16 == 0 && (reinterpret_cast<uintptr_t>(p.A) & 15) == 0 &&
      a_tma_enabled()) {
    if (encode_tensor_map_2d(&tmX, dt, p.A, static_cast<uint64_t>(p.K), static_cast<uint64_t>(p.M),
                             static_cast<uint64_t>(p.lda) * 2, KS, 128, CU_TENSOR_MAP_SWIZZLE_128B) != CUDA_SUCCESS)
      return kErrCuda;
    q.a_tma = 1;
  }
  const int out_tiles = static_cast<int>(ceil_div(p.N, 256));
  const int64_t units = static_cast<int64_t>(p.max_tiles) * out_tiles;
  if (units == 0) return kOk;
  if (units >= (1ll << 31)) return kErrShape;
  auto kern = rowgemm2t_kernel<kBF16>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(Cfg::SMEM));
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = Cfg::SMEM;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  static int max_pairs = 0;
  if (max_pairs == 0) {
    cfg.gridDim = dim3(static_cast<unsigned>(num_sms() & ~1));
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, kern, &cfg) != cudaSuccess || nc <= 0) {
      cudaGetLastError();
      nc = num_sms() / 2;
    }
    max_pairs = nc;
  }
  const int pairs = static_cast<int>(units < max_pairs ? units : max_pairs);
  cfg.gridDim = dim3(static_cast<unsigned>(2 * pairs));
  cudaLaunchKernelEx(&cfg, kern, tmW, tmX, q, out_tiles, p.max_tiles);
  note_launch();
  return cuda_status();
}

int launch_rowgemm(const GroupedGemmArgs& g, cudaStream_t s) {
  if (g.dtype != kDtypeBF16 && g.dtype != kDtypeF16) return kErrUnsupported;
  if (reinterpret_cast<uintptr_t>(g.A) % 16 || reinterpret_cast<uintptr_t>(g.B) % 16) return kErrUnsupported;
  if ((g.lda * 2) % 16 || (g.ldb * 2) % 16) return kErrUnsupported;
  RowGemmParams p{};
  p.A = g.A;
  p.lda = g.lda;
  p.C = g.C;
  p.ldc = g.ldc;
  p.M = static_cast<int>(g.rows_a);
  p.N = static_cast<int>(g.N);
  p.K = static_cast<int>(g.K);
  p.G = static_cast<int>(g.G);
  p.cnt = g.counts;
  p.off = g.offsets;
  p.tile_off = g.tile_offsets;
  p.row_src = g.row_src;
  p.src_stride = g.src_stride;
  p.row_dst = g.row_dst;
  p.dst_stride = g.dst_stride;
  p.row_scale = g.row_scale;
  p.act = g.act;
  p.t1 = 1;
  p.max_tiles = static_cast<int>(g.max_tiles);
  const int ks = g.K % 64 == 0 || g.K > 64 ? 64 : g.K % 32 == 0 ? 32 : 16;
  // small groups (MoE at ~128 tokens per expert): tokens on the MMA's N side, quantised to 16 rows
  // instead of 128 (rowgemm2t); large groups fill 256-row tiles anyway and keep rowgemm2's epilogue
  const bool small_groups = (g.rows_hint > 0 ? g.rows_hint : g.rows_a) < 256 * g.G;
  if (ks == 64 && p.G <= kRg2MaxGroups && rg2t_enabled() && p.N >= 64 && small_groups)
    return g.dtype == kDtypeBF16 ? run_rowgemm2t<true>(p, g.B, g.ldb, s) : run_rowgemm2t<false>(p, g.B, g.ldb, s);
  return g.dtype == kDtypeBF16 ? rowgemm_dispatch<true>(p, g.B, g.ldb, ks, s) : rowgemm_dispatch<false>(p, g.B, g.ldb, ks, s);
}

int64_t spmm_tc_workspace_bytes(const SpmmArgs& a) {
  if (a.plan == kPlanPitM) {  // one-K-group pit:m: packed live rows; 2-D: the high-sparsity path
    const int64_t pb = gm_pack_bytes(a), sb = gm_sparse_ws_bytes(a);
    return pb > sb ? pb : sb;
  }
  // mirrors dispatch_tc: only the 128-row gathered-K kernel on 64-column units splits groups
  if (a.plan != kPlanPitK || a.t0 <= 64 || a.t0 > 128 || a.N > 64) return 0;
  const char* e = getenv("PIT_GK_NT");
  if (e && atoi(e) == 128) return 0;
  return gk_split_ws_bytes<64>(a.n_groups, 1);
}

int launch_spmm_tc(const SpmmArgs& a, cudaStream_t s) {
  if (!spmm_tc_supported(a)) return kErrUnsupported;
  return a.dtype == kDtypeBF16 ? dispatch_tc<true>(a, s) : dispatch_tc<false>(a, s);
}

}  // namespace pit
