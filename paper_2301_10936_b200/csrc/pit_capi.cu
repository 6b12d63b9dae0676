// C-ABI layer: argument validation, physical-layout mapping and dispatch to the launchers.
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <atomic>
#include <mutex>
#include <string>

#include <cuda.h>
#include <cuda_runtime.h>

#include "pit_b200.h"
#include "pit_internal.h"

namespace pit {

namespace {
thread_local std::string g_err;

int fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn g_encode = nullptr;
std::once_flag g_encode_once;

bool dtype_ok(int dt) { return dt >= kDtypeF32 && dt <= kDtypeU8; }
}  // namespace

std::atomic<long long> g_launches{0};

void note_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

int cuda_status() {
  const cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) return kOk;
  return fail(kErrCuda, "CUDA error: %s", cudaGetErrorString(e));
}

CUresult encode_tensor_map_2d(CUtensorMap* map, CUtensorMapDataType dt, const void* base, uint64_t inner,
                              uint64_t outer, uint64_t row_pitch_bytes, uint32_t box_inner, uint32_t box_outer,
                              CUtensorMapSwizzle swizzle) {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<EncodeFn>(fn);
  });
  if (!g_encode) {
    fail(kErrCuda, "cuTensorMapEncodeTiled unavailable");
    return CUDA_ERROR_NOT_FOUND;
  }
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {row_pitch_bytes};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = g_encode(map, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    fail(kErrCuda, "cuTensorMapEncodeTiled failed (%d): dims %llu x %llu pitch %llu box %u x %u", static_cast<int>(r),
         static_cast<unsigned long long>(inner), static_cast<unsigned long long>(outer),
         static_cast<unsigned long long>(row_pitch_bytes), box_inner, box_outer);
  return r;
}

CUresult encode_tensor_map_3d(CUtensorMap* map, CUtensorMapDataType dt, const void* base, uint64_t d0, uint64_t d1,
                              uint64_t d2, uint64_t pitch1_bytes, uint64_t pitch2_bytes, uint32_t box0, uint32_t box1,
                              CUtensorMapSwizzle swizzle) {
  CUtensorMap dummy;
  if (encode_tensor_map_2d(&dummy, dt, base, d0, d1 > 0 ? d1 : 1, pitch1_bytes, box0, 1, swizzle) != CUDA_SUCCESS)
    return CUDA_ERROR_INVALID_VALUE;  // resolves the entry point and validates the 2-D part
  const cuuint64_t dims[3] = {d0, d1, d2};
  const cuuint64_t strides[2] = {pitch1_bytes, pitch2_bytes};
  const cuuint32_t box[3] = {box0, box1, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = g_encode(map, dt, 3, const_cast<void*>(base), dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    fail(kErrCuda, "cuTensorMapEncodeTiled (3-D) failed (%d)", static_cast<int>(r));
  return r;
}

}  // namespace pit

using namespace pit;

namespace {

int geometry(int64_t s0, int64_t s1, int t0, int t1, int pit_dim, int64_t* ng, int64_t* pg, int64_t* wg) {
  if (s0 < 0 || s1 < 0) return fail(kErrShape, "shape must be non-negative, got (%lld,%lld)", (long long)s0, (long long)s1);
  if (t0 <= 0 || t1 <= 0) return fail(kErrArg, "micro-tile edges must be positive, got (%d,%d)", t0, t1);
  if (pit_dim != 0 && pit_dim != 1) return fail(kErrArg, "pit dimension must be 0 or 1, got %d", pit_dim);
  const int64_t G0 = ceil_div(s0, t0), G1 = ceil_div(s1, t1);
  *ng = pit_dim == 0 ? G1 : G0;
  *pg = pit_dim == 0 ? G0 : G1;
  *wg = ceil_div(*pg, 32);
  if (*pg >= (1ll << 31)) return fail(kErrShape, "PIT grid extent %lld exceeds int32", (long long)*pg);
  return kOk;
}

}  // namespace

extern "C" {

const char* pit_last_error(void) { return g_err.c_str(); }

int pit_abi_version(void) { return 104; }

// Diagnostic (not part of include/pit_b200.h): the CTA-pair gathered-K kernel's stage timeline.
PIT_API int pit_debug_gk2_trace(unsigned long long* host_out_1024) { return pit::gk2_trace_read(host_out_1024); }

long long pit_kernel_launches(void) { return g_launches.load(std::memory_order_relaxed); }

int pit_index_geometry(int64_t s0, int64_t s1, int t0, int t1, int pit_dim, int64_t* n_groups, int64_t* pit_grid,
                       int64_t* words_per_group) {
  if (!n_groups || !pit_grid || !words_per_group) return fail(kErrArg, "null output pointer");
  return geometry(s0, s1, t0, t1, pit_dim, n_groups, pit_grid, words_per_group);
}

int pit_build_index_from_tensor(const void* values, int dtype, int64_t s0, int64_t s1, int64_t stride0,
                                int64_t stride1, int t0, int t1, int pit_dim, uint32_t* occ, int32_t* counts,
                                int32_t* slots, void* stream) {
  int64_t ng, pg, wg;
  if (int st = geometry(s0, s1, t0, t1, pit_dim, &ng, &pg, &wg)) return st;
  if (!dtype_ok(dtype)) return fail(kErrArg, "unsupported dtype code %d", dtype);
  if (ng == 0 || pg == 0) return kOk;
  if (!values || !occ || !counts || !slots) return fail(kErrArg, "null device pointer");
  DetectValuesArgs a{};
  a.x = values;
  a.dtype = dtype;
  a.occ = occ;
  if (stride1 == 1 && (stride0 >= s1 || s0 == 1)) {  // row-major
    a.R = s0;
    a.C = s1;
    a.ld = s0 == 1 ? s1 : stride0;
    a.tr = t0;
    a.tc = t1;
    a.pit_phys = pit_dim;
  } else if (stride0 == 1 && (stride1 >= s0 || s1 == 1)) {  // column-major: physical = transpose
    a.R = s1;
    a.C = s0;
    a.ld = s1 == 1 ? s0 : stride1;
    a.tr = t1;
    a.tc = t0;
    a.pit_phys = 1 - pit_dim;
  } else {
    return fail(kErrLayout, "values must be row-major or column-major, got strides (%lld,%lld)", (long long)stride0,
                (long long)stride1);
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (int st = launch_detect_values(a, s)) return st == kErrShape ? fail(st, "tensor too large for detection grid") : st;
  return launch_compact(occ, ng, wg, counts, slots, pg, s);
}

int pit_build_index(const uint8_t* packed, int64_t s0, int64_t s1, int g0, int g1, int t0, int t1, int pit_dim,
                    uint32_t* occ, int32_t* counts, int32_t* slots, void* stream) {
  int64_t ng, pg, wg;
  if (int st = geometry(s0, s1, t0, t1, pit_dim, &ng, &pg, &wg)) return st;
  if (g0 <= 0 || g1 <= 0) return fail(kErrArg, "granularity must be positive, got (%d,%d)", g0, g1);
  if (ng == 0 || pg == 0) return kOk;
  if (!packed || !occ || (!counts) != (!slots)) return fail(kErrArg, "null device pointer");
  DetectBitsArgs a{packed, s0, s1, g0, g1, t0, t1, pit_dim, occ};
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (!counts) return launch_detect_bits(a, s);  // occupancy bitmap only
  return launch_index_from_bits(a, counts, slots, pg, s);
}

int pit_cover_counts(const uint8_t* packed, int64_t s0, int64_t s1, int g0, int g1, int n_candidates,
                     const int32_t* candidates, uint32_t* occ_ws, int64_t ws_words, int32_t* counts, void* stream) {
  if (g0 <= 0 || g1 <= 0) return fail(kErrArg, "granularity must be positive, got (%d,%d)", g0, g1);
  if (n_candidates < 0 || (n_candidates > 0 && !candidates)) return fail(kErrArg, "bad candidate list");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int64_t off = 0;
  for (int c = 0; c < n_candidates; ++c) {
    const int t0 = candidates[3 * c], t1 = candidates[3 * c + 1], dim = candidates[3 * c + 2];
    int64_t ng, pg, wg;
    if (int st = geometry(s0, s1, t0, t1, dim, &ng, &pg, &wg)) return st;
    if (ng == 0) continue;
    if (pg == 0) {
      cudaMemsetAsync(counts + off, 0, sizeof(int32_t) * ng, s);
    } else {
      if (ng * wg > ws_words) return fail(kErrArg, "cover-count workspace too small (%lld words, need %lld)",
                                          static_cast<long long>(ws_words), static_cast<long long>(ng * wg));
      if (!packed || !occ_ws || !counts) return fail(kErrArg, "null device pointer");
      DetectBitsArgs a{packed, s0, s1, g0, g1, t0, t1, dim, occ_ws};
      if (int st = launch_detect_bits(a, s)) return st;
      if (int st = launch_occ_counts(occ_ws, ng, wg, counts + off, s)) return st;
    }
    off += ng;
  }
  return cuda_status();
}

int pit_index_occupancy(const int32_t* counts, const int32_t* slots, int64_t n_groups, int64_t pit_grid, uint32_t* occ,
                        int32_t* bad, void* stream) {
  if (n_groups < 0 || pit_grid < 0) return fail(kErrShape, "negative index geometry");
  if (n_groups == 0) return kOk;
  if (!counts || !slots || !occ || !bad) return fail(kErrArg, "null device pointer");
  return launch_slots_to_occ(counts, slots, pit_grid, n_groups, ceil_div(pit_grid, 32), pit_grid, occ, bad,
                             static_cast<cudaStream_t>(stream));
}

int pit_index_union(const uint32_t* occ, int64_t n_groups, int64_t pit_grid, uint32_t* union_ws, int32_t* rows,
                    int32_t* n_rows, void* stream) {
  if (!occ || !union_ws || !rows || !n_rows) return fail(kErrArg, "null device pointer");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t wg = ceil_div(pit_grid, 32);
  if (wg == 0 || n_groups == 0) {
    cudaMemsetAsync(n_rows, 0, sizeof(int32_t), s);
    return cuda_status();
  }
  if (int st = launch_union(occ, n_groups, wg, union_ws, s)) return st;
  return launch_compact(union_ws, 1, wg, n_rows, rows, pit_grid, s);
}

static int gather_args(GatherArgs& a, void* tensor, int dtype, int64_t s0, int64_t s1, int64_t ld, int col_major,
                       void* tile, int64_t tile_rows, int64_t tile_cols, int t0, int t1, int pit_dim, int64_t group,
                       const int32_t* coords, int64_t n_coords) {
  if (!dtype_ok(dtype) || dtype == kDtypeU8) return fail(kErrArg, "unsupported dtype code %d", dtype);
  if (t0 <= 0 || t1 <= 0) return fail(kErrArg, "micro-tile edges must be positive");
  if (pit_dim != 0 && pit_dim != 1) return fail(kErrArg, "pit dimension must be 0 or 1");
  a = GatherArgs{};
  a.dtype = dtype;
  a.tile = tile;
  a.TR = tile_rows;
  a.TC = tile_cols;
  a.coords = coords;
  a.n_coords = n_coords;
  a.src_or_dst = tensor;
  const int t_d = pit_dim == 0 ? t0 : t1, t_o = pit_dim == 0 ? t1 : t0;
  if (tile_rows < 0 || tile_cols < 0 || n_coords < 0)
    return fail(kErrArg, "tile extents and coordinate count must be non-negative");
  // slot s occupies tile rows/cols [s*t_d, (s+1)*t_d) along the PIT dim (executor.py:190-192)
  if (n_coords * static_cast<int64_t>(t_d) > (pit_dim == 0 ? tile_rows : tile_cols))
    return fail(kErrArg, "tile buffer holds %lld micro-tiles, %lld coordinates given",
                static_cast<long long>((pit_dim == 0 ? tile_rows : tile_cols) / t_d), static_cast<long long>(n_coords));
  a.t_d = t_d;
  a.t_o = t_o;
  a.off_o = group * t_o;
  a.R = s0;
  a.C = s1;
  a.st0 = col_major ? 1 : ld;
  a.st1 = col_major ? ld : 1;
  a.d = pit_dim;
  return kOk;
}

int pit_sread(const void* tensor, int dtype, int64_t s0, int64_t s1, int64_t ld, int col_major, void* tile,
              int64_t tile_rows, int64_t tile_cols, int t0, int t1, int pit_dim, int64_t group, const int32_t* coords,
              int64_t n_coords, int zero_fill, void* stream) {
  GatherArgs a;
  if (int st = gather_args(a, const_cast<void*>(tensor), dtype, s0, s1, ld, col_major, tile, tile_rows, tile_cols, t0,
                           t1, pit_dim, group, coords, n_coords))
    return st;
  a.zero_fill = zero_fill;
  return launch_sread(a, static_cast<cudaStream_t>(stream));
}

int pit_swrite(const void* tile, void* tensor, int dtype, int64_t s0, int64_t s1, int64_t ld, int col_major,
               int64_t tile_rows, int64_t tile_cols, int t0, int t1, int pit_dim, int64_t group, const int32_t* coords,
               int64_t n_coords, int accumulate, void* stream) {
  GatherArgs a;
  if (int st = gather_args(a, tensor, dtype, s0, s1, ld, col_major, const_cast<void*>(tile), tile_rows, tile_cols, t0,
                           t1, pit_dim, group, coords, n_coords))
    return st;
  a.accumulate = accumulate;
  return launch_swrite(a, static_cast<cudaStream_t>(stream));
}

static SpmmArgs to_internal(const pit_spmm_args* p) {
  SpmmArgs a{};
  a.plan = p->plan;
  a.dtype = p->dtype;
  a.M = p->M;
  a.N = p->N;
  a.K = p->K;
  a.A = p->A;
  a.sam = p->sam;
  a.sak = p->sak;
  a.B = p->B;
  a.ldb = p->ldb;
  a.C = p->C;
  a.ldc = p->ldc;
  a.t0 = p->t0;
  a.t1 = p->t1;
  a.counts = p->counts;
  a.slots = p->slots;
  a.slot_stride = p->slot_stride;
  a.n_groups = p->n_groups;
  a.occ = p->occ;
  a.WG = p->words_per_group;
  a.rows = p->rows;
  a.n_rows = p->n_rows;
  a.n_rows_host = p->n_rows_bound;
  a.batch = p->batch > 1 ? p->batch : 1;
  a.b_batch_stride = p->b_batch_stride;
  a.ws = p->workspace;
  a.ws_bytes = p->workspace ? p->workspace_bytes : 0;
  return a;
}

int64_t pit_spmm_workspace_bytes(const pit_spmm_args* p) {
  if (!p || p->force_simt) return 0;
  const SpmmArgs a = to_internal(p);
  return spmm_tc_supported(a) ? spmm_tc_workspace_bytes(a) : 0;
}

int pit_spmm_uses_tensor_cores(const pit_spmm_args* p) {
  if (!p || p->force_simt) return 0;
  return spmm_tc_supported(to_internal(p)) ? 1 : 0;
}

int pit_spmm(const pit_spmm_args* p, void* stream) {
  if (!p) return fail(kErrArg, "null args");
  if (p->plan < kPlanDense || p->plan > kPlanPitK) return fail(kErrArg, "unknown plan %d", p->plan);
  if (p->dtype == kDtypeU8 || !dtype_ok(p->dtype)) return fail(kErrArg, "unsupported dtype code %d", p->dtype);
  if (p->M < 0 || p->N < 0 || p->K < 0) return fail(kErrShape, "shape mismatch: negative extent");
  if (p->M == 0 || p->N == 0) return kOk;
  if (!p->A || !p->B || !p->C) return fail(kErrArg, "null operand pointer");
  const int64_t batch = p->batch > 1 ? p->batch : 1;
  if (p->plan == kPlanPitK) {
    if (p->sam != 1 && p->M * batch > 1)
      return fail(kErrLayout, "plan requires the sparse operand in col_major; use convert_layout first");
    if (!p->counts || !p->slots) return fail(kErrArg, "sparse plan needs a micro-tile index");
    if (p->t1 != 1) return fail(kErrArg, "pit:k micro-tile must be (t0,1)");
    if (batch > 1 && p->M % p->t0) return fail(kErrShape, "batched pit:k needs M to be a multiple of t0");
    if (p->n_groups != batch * ceil_div(p->M, p->t0)) return fail(kErrShape, "index groups do not match M");
  } else if (p->plan == kPlanPitM) {
    if (p->sak != 1 && p->K > 1)
      return fail(kErrLayout, "plan requires the sparse operand in row_major; use convert_layout first");
    if (!p->occ || (batch == 1 && (!p->rows || !p->n_rows))) return fail(kErrArg, "sparse plan needs a micro-tile index");
    if (p->t0 != 1) return fail(kErrArg, "pit:m micro-tile must be (1,t1)");
    if (p->n_groups != ceil_div(p->K, p->t1)) return fail(kErrShape, "index groups do not match K");
  }
  SpmmArgs a = to_internal(p);
  if (a.K == 0) {  // empty contraction: C = 0
    const int eb = dtype_bytes(a.dtype);
    cudaMemset2DAsync(a.C, a.ldc * eb, 0, a.N * eb, a.M * batch, static_cast<cudaStream_t>(stream));
    return cuda_status();
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (batch > 1) {
    // pit:k on tensor cores: one launch over the stacked groups
    SpmmArgs st = a;
    if (a.plan == kPlanPitK) {
      st.M = a.M * batch;
      if (!p->force_simt && spmm_tc_supported(st)) return launch_spmm_tc(st, s);
    } else {
      // pit:m / dense: one launch over uniform row groups, B slices through a 3-D tensor map
      const bool tc = !p->force_simt && spmm_tc_supported(st) && (a.b_batch_stride * 2) % 16 == 0 &&
                      a.M * batch < (1ll << 31);
      if (tc) return launch_spmm_tc(st, s);
      if (a.plan == kPlanPitM)
        return fail(kErrUnsupported, "batched pit:m runs on the tensor-core path only (bf16/fp16, 16-byte aligned rows)");
    }
    // otherwise slice by slice
    const int eb = dtype_bytes(a.dtype);
    const int64_t gpb = a.plan == kPlanPitK ? a.n_groups / batch : 0;
    for (int64_t b = 0; b < batch; ++b) {
      SpmmArgs sl = a;
      sl.batch = 1;
      sl.A = static_cast<const uint8_t*>(a.A) + b * a.M * a.sam * eb;
      sl.B = static_cast<const uint8_t*>(a.B) + b * a.b_batch_stride * eb;
      sl.C = static_cast<uint8_t*>(a.C) + b * a.M * a.ldc * eb;
      if (a.plan == kPlanPitK) {
        sl.counts = a.counts + b * gpb;
        sl.slots = a.slots + b * gpb * a.slot_stride;
        sl.n_groups = gpb;
      }
      const int st2 = (!p->force_simt && spmm_tc_supported(sl)) ? launch_spmm_tc(sl, s) : launch_spmm_simt(sl, s);
      if (st2) return st2;
    }
    return kOk;
  }
  if (!p->force_simt && spmm_tc_supported(a)) return launch_spmm_tc(a, s);
  return launch_spmm_simt(a, s);
}

int pit_grouped_gemm(const pit_grouped_gemm_args* a, void* stream) {
  if (!a) return fail(kErrArg, "null args");
  if (a->G < 0 || a->N < 0 || a->K <= 0) return fail(kErrShape, "shape mismatch: bad grouped GEMM extents");
  if (a->G == 0 || a->N == 0 || a->max_tiles == 0) return kOk;
  if (!a->A || !a->B || !a->C || !a->counts || !a->offsets || !a->tile_offsets)
    return fail(kErrArg, "null device pointer");
  GroupedGemmArgs g{};
  g.dtype = a->dtype;
  g.A = a->A;
  g.lda = a->lda;
  g.rows_a = a->rows_a;
  g.B = a->B;
  g.ldb = a->ldb;
  g.C = a->C;
  g.ldc = a->ldc;
  g.N = a->N;
  g.K = a->K;
  g.G = a->G;
  g.counts = a->counts;
  g.offsets = a->offsets;
  g.tile_offsets = a->tile_offsets;
  g.row_src = a->row_src;
  g.src_stride = a->src_stride;
  g.row_dst = a->row_dst;
  g.dst_stride = a->dst_stride;
  g.row_scale = a->row_scale;
  g.act = a->act;
  g.max_tiles = a->max_tiles;
  g.rows_hint = a->rows_hint;
  const int st = launch_rowgemm(g, static_cast<cudaStream_t>(stream));
  if (st == kErrUnsupported) return fail(st, "grouped GEMM needs bf16/fp16 with 16-byte aligned rows");
  return st;
}

int pit_moe_route(const void* logits, int dtype, int64_t T, int64_t E, int32_t* expert, float* gate, uint32_t* occ,
                  int32_t* counts, int32_t* slots, void* stream) {
  if (E <= 0 || T < 0) return fail(kErrShape, "bad routing shape (T=%lld, E=%lld)", (long long)T, (long long)E);
  if (!logits || !expert || !gate || !occ || !counts || !slots) return fail(kErrArg, "null device pointer");
  const int st = launch_moe_route(logits, dtype, T, static_cast<int>(E), expert, gate, occ, counts, slots,
                                  static_cast<cudaStream_t>(stream));
  if (st == kErrUnsupported) return fail(st, "router logits must be f32, bf16 or f16");
  return st;
}

int pit_moe_plan(const int32_t* counts, int64_t G, const int32_t* slots, int64_t stride, int32_t* offsets,
                 int32_t* tile_offsets, int32_t* perm, int64_t max_count, void* stream) {
  if (G < 0) return fail(kErrShape, "negative group count");
  if (!counts || !offsets || !tile_offsets) return fail(kErrArg, "null device pointer");
  return launch_moe_plan(counts, static_cast<int>(G), slots, stride, offsets, tile_offsets, perm, max_count,
                         static_cast<cudaStream_t>(stream));
}

int pit_moe_recv_plan(const int32_t* rc, int64_t W, int64_t El, int32_t* rows, int64_t stride, int32_t* counts,
                      void* stream) {
  if (W <= 0 || El <= 0) return fail(kErrShape, "bad expert-parallel geometry");
  if (!rc || !rows || !counts) return fail(kErrArg, "null device pointer");
  return launch_moe_recv_plan(rc, static_cast<int>(W), static_cast<int>(El), rows, stride, counts,
                              static_cast<cudaStream_t>(stream));
}

int pit_gather_rows(const void* src, int64_t ld_src_bytes, const int32_t* rows, int64_t n, int64_t row_bytes, void* dst,
                    int64_t ld_dst_bytes, void* stream) {
  if (n < 0 || row_bytes < 0) return fail(kErrShape, "negative extent");
  if (n && (!src || !rows || !dst)) return fail(kErrArg, "null device pointer");
  return launch_gather_rows(src, ld_src_bytes, rows, n, row_bytes, dst, ld_dst_bytes, static_cast<cudaStream_t>(stream));
}

int pit_pack_groups(const void* src, int64_t ld_src_bytes, const int32_t* rows, int64_t stride, const int32_t* counts,
                    const int32_t* offsets, int64_t G, int64_t max_count, int64_t row_bytes, void* dst,
                    int64_t ld_dst_bytes, void* stream) {
  if (G < 0 || max_count < 0 || row_bytes < 0) return fail(kErrShape, "negative extent");
  if (G && (!src || !rows || !counts || !offsets || !dst)) return fail(kErrArg, "null device pointer");
  const int st = launch_pack_groups(src, ld_src_bytes, rows, stride, counts, offsets, G, max_count, row_bytes, dst,
                                    ld_dst_bytes, static_cast<cudaStream_t>(stream));
  return st == kErrUnsupported ? fail(st, "pit_pack_groups needs 16-byte aligned rows and pitches, G <= 65535") : st;
}

int pit_scatter_rows_scaled(const void* src, int dtype, int64_t ld_src, const int32_t* rows, int64_t n, int64_t width,
                            const float* scale, void* dst, int64_t ld_dst, void* stream) {
  if (n < 0 || width < 0) return fail(kErrShape, "negative extent");
  if (n && (!src || !rows || !dst)) return fail(kErrArg, "null device pointer");
  const int st = launch_scatter_rows_scaled(src, dtype, ld_src, rows, n, width, scale, dst, ld_dst,
                                            static_cast<cudaStream_t>(stream));
  if (st == kErrUnsupported) return fail(st, "unsupported dtype code %d", dtype);
  return st;
}

static void sddmm_copy(const pit_sddmm_args* a, pit::SddmmArgs* o) {
  o->dtype = a->dtype;
  o->A = a->A;
  o->lda = a->lda;
  o->B = a->B;
  o->ldb = a->ldb;
  o->C = a->C;
  o->ldc = a->ldc;
  o->M = a->M;
  o->N = a->N;
  o->K = a->K;
  o->batch = a->batch;
  o->unit_counts = a->unit_counts;
  o->unit_slots = a->unit_slots;
  o->unit_slot_stride = a->unit_slot_stride;
  o->n_unit_groups = a->n_unit_groups;
  o->occ = a->occ;
  o->words_per_group = a->words_per_group;
  o->g0 = a->g0;
  o->g1 = a->g1;
  o->gate = a->gate;
  o->ldgate = a->ldgate;
  o->workspace = a->workspace;
  o->workspace_bytes = a->workspace_bytes;
}

int64_t pit_sddmm_workspace_bytes(const pit_sddmm_args* a) {
  if (!a) return -1;
  pit::SddmmArgs s{};
  sddmm_copy(a, &s);
  return pit::sddmm_workspace_bytes(s);
}

int pit_sddmm(const pit_sddmm_args* a, void* stream) {
  if (!a) return fail(kErrArg, "null args");
  if (a->M < 0 || a->N < 0 || a->K < 0 || a->batch <= 0) return fail(kErrShape, "shape mismatch: bad SDDMM extents");
  if (a->M == 0 || a->N == 0) return kOk;
  if (a->dtype != kDtypeBF16 && a->dtype != kDtypeF16) return fail(kErrUnsupported, "SDDMM needs bf16 or fp16 operands");
  if (!a->A || !a->B || !a->C || !a->unit_counts || !a->unit_slots || !a->occ)
    return fail(kErrArg, "null device pointer");
  if (a->N % 8 || a->K % 8 || a->lda % 8 || a->ldb % 8 || a->ldc % 8 || (a->gate && a->ldgate % 8))
    return fail(kErrLayout, "SDDMM needs N, K and every pitch to be multiples of 8 elements");
  if (a->lda < a->K || a->ldb < a->K || a->ldc < a->N) return fail(kErrLayout, "pitch smaller than the row");
  if ((reinterpret_cast<uintptr_t>(a->A) | reinterpret_cast<uintptr_t>(a->B) | reinterpret_cast<uintptr_t>(a->C) |
       reinterpret_cast<uintptr_t>(a->gate)) % 16)
    return fail(kErrLayout, "SDDMM operands must be 16-byte aligned");
  if (a->g0 <= 0 || a->g1 <= 0 || a->g1 % 8) return fail(kErrShape, "output micro-tile width must be a multiple of 8");
  if (a->batch > 1 && a->M % 128) return fail(kErrShape, "batched SDDMM needs M to be a multiple of 128");
  if (a->n_unit_groups != a->batch * ((a->M + 127) / 128))
    return fail(kErrShape, "unit index does not match C (expected micro-tile (128, 64) with the column axis permuted)");
  if (a->unit_slot_stride < (a->N + 63) / 64) return fail(kErrShape, "unit index stride below the column-block grid");
  pit::SddmmArgs s{};
  sddmm_copy(a, &s);
  if (a->workspace_bytes < pit::sddmm_workspace_bytes(s) || !a->workspace)
    return fail(kErrArg, "SDDMM workspace too small (%lld bytes needed)", (long long)pit::sddmm_workspace_bytes(s));
  return pit::launch_sddmm(s, static_cast<cudaStream_t>(stream));
}

static int ep_check(const pit_ep_args* ep, pit::EpArgs* out) {
  if (!ep) return fail(kErrArg, "null expert-parallel args");
  if (ep->world <= 0 || ep->rank < 0 || ep->rank >= ep->world || ep->experts_local <= 0 || ep->capacity < 0)
    return fail(kErrShape, "bad expert-parallel geometry (rank %d of %d, %lld local experts)", ep->rank, ep->world,
                (long long)ep->experts_local);
  if (ep->row_bytes <= 0 || ep->row_bytes % 16) return fail(kErrShape, "exchanged rows must be a multiple of 16 bytes");
  if (!ep->local || !ep->peers) return fail(kErrArg, "null region pointer");
  out->rank = ep->rank;
  out->world = ep->world;
  out->experts_local = ep->experts_local;
  out->capacity = ep->capacity;
  out->row_bytes = ep->row_bytes;
  out->local = ep->local;
  out->peers = ep->peers;
  return kOk;
}

int pit_ep_region_layout(int64_t world, int64_t El, int64_t cap, int64_t row_bytes, int64_t* out) {
  if (world <= 0 || El <= 0 || cap < 0 || row_bytes <= 0) return fail(kErrShape, "bad expert-parallel geometry");
  if (!out) return fail(kErrArg, "null output");
  pit::ep_region_layout(static_cast<int>(world), El, cap, row_bytes, out);
  return kOk;
}

int pit_ep_region_alloc(int64_t bytes, void** out) {
  if (bytes <= 0 || !out) return fail(kErrArg, "bad region request");
  void* p = nullptr;
  if (cudaMalloc(&p, static_cast<size_t>(bytes)) != cudaSuccess) return cuda_status();
  if (cudaMemset(p, 0, static_cast<size_t>(bytes)) != cudaSuccess) {
    cudaFree(p);
    return cuda_status();
  }
  *out = p;
  return kOk;
}

int pit_ep_region_free(void* region) {
  if (region && cudaFree(region) != cudaSuccess) return cuda_status();
  return kOk;
}

int pit_ep_ipc_handle(void* region, void* handle64) {
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  if (!region || !handle64) return fail(kErrArg, "null pointer");
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, region) != cudaSuccess) return cuda_status();
  memcpy(handle64, &h, sizeof h);
  return kOk;
}

int pit_ep_ipc_open(const void* handle64, void** out) {
  if (!handle64 || !out) return fail(kErrArg, "null pointer");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof h);
  if (cudaIpcOpenMemHandle(out, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return cuda_status();
  return kOk;
}

int pit_ep_ipc_close(void* mapped) {
  if (mapped && cudaIpcCloseMemHandle(mapped) != cudaSuccess) return cuda_status();
  return kOk;
}

int pit_ep_error(void* region, int* out) {
  if (!region || !out) return fail(kErrArg, "null pointer");
  unsigned v = 0;
  if (cudaMemcpy(&v, static_cast<uint8_t*>(region) + 12, sizeof v, cudaMemcpyDeviceToHost) != cudaSuccess)
    return cuda_status();
  *out = static_cast<int>(v);
  return kOk;
}

int pit_moe_dispatch(const pit_ep_args* ep, const void* x, int64_t ldx_bytes, int64_t T, const int32_t* perm,
                     const int32_t* offsets, const int32_t* counts, void* stream) {
  pit::EpArgs a;
  if (int st = ep_check(ep, &a)) return st;
  if (T < 0 || T > ep->capacity) return fail(kErrShape, "%lld tokens exceed the exchange capacity %lld", (long long)T,
                                             (long long)ep->capacity);
  if (ldx_bytes < ep->row_bytes || ldx_bytes % 16 || reinterpret_cast<uintptr_t>(x) % 16)
    return fail(kErrLayout, "token rows must be 16-byte aligned with pitch >= row bytes");
  if ((T && (!x || !perm)) || !offsets || !counts) return fail(kErrArg, "null device pointer");
  return launch_ep_dispatch(a, x, ldx_bytes, T, perm, offsets, counts, static_cast<cudaStream_t>(stream));
}

int pit_moe_recv_plan_ep(const pit_ep_args* ep, int32_t* rows, int64_t stride, int32_t* counts, void* stream) {
  pit::EpArgs a;
  if (int st = ep_check(ep, &a)) return st;
  if (!rows || !counts) return fail(kErrArg, "null device pointer");
  if (stride < ep->world * ep->capacity) return fail(kErrShape, "row-list stride below world * capacity");
  return launch_ep_recv_plan(a, rows, stride, counts, static_cast<cudaStream_t>(stream));
}

int pit_moe_signal(const pit_ep_args* ep, void* stream) {
  pit::EpArgs a;
  if (int st = ep_check(ep, &a)) return st;
  return launch_ep_signal(a, static_cast<cudaStream_t>(stream));
}

int pit_moe_combine(const pit_ep_args* ep, int dtype, int64_t T, const int32_t* perm, const int32_t* offsets,
                    const float* gate, void* out, int64_t ldo_bytes, void* stream) {
  pit::EpArgs a;
  if (int st = ep_check(ep, &a)) return st;
  if (T < 0 || T > ep->capacity) return fail(kErrShape, "token count outside the exchange capacity");
  if (ldo_bytes < ep->row_bytes || ldo_bytes % 16 || reinterpret_cast<uintptr_t>(out) % 16)
    return fail(kErrLayout, "output rows must be 16-byte aligned with pitch >= row bytes");
  if ((T && (!out || !perm)) || !offsets) return fail(kErrArg, "null device pointer");
  const int st = launch_ep_combine(a, dtype, T, perm, offsets, gate, out, ldo_bytes, static_cast<cudaStream_t>(stream));
  if (st == kErrUnsupported) return fail(st, "combine dtype must be bf16, f16 or f32");
  return st;
}

int pit_reduce_rows(const void* A, int dtype, int64_t P, int64_t L, int64_t lda, const uint32_t* occ, int64_t WG,
                    int mode, int block_l, void* out, void* stream) {
  if (P < 0 || L < 0) return fail(kErrShape, "negative extent");
  if (mode < 0 || mode > 2) return fail(kErrArg, "unknown reduce mode %d", mode);
  if (mode && (!occ || block_l <= 0)) return fail(kErrArg, "sparse reduce needs an occupancy bitmap");
  if (P && (!A || !out)) return fail(kErrArg, "null device pointer");
  const int st = launch_reduce_rows(A, dtype, P, L, lda, occ, WG, mode, block_l, out, static_cast<cudaStream_t>(stream));
  if (st == kErrUnsupported) return fail(st, "unsupported dtype code %d", dtype);
  return st;
}

int pit_copy2d_async(void* dst, int64_t dpitch, const void* src, int64_t spitch, int64_t width_bytes, int64_t height,
                     void* stream) {
  if (width_bytes < 0 || height < 0) return fail(kErrShape, "negative extent");
  if (width_bytes == 0 || height == 0) return kOk;
  if (cudaMemcpy2DAsync(dst, dpitch, src, spitch, width_bytes, height, cudaMemcpyDefault,
                        static_cast<cudaStream_t>(stream)) != cudaSuccess)
    return cuda_status();
  return kOk;
}

int pit_dense_reference_f64(const double* A, int64_t s0, int64_t s1, const double* B, int64_t ldb, double* C, int64_t M,
                            int64_t N, int64_t K, void* stream) {
  if (M < 0 || N < 0 || K < 0) return fail(kErrShape, "shape mismatch: negative extent");
  if (M * N && (!A || !B || !C)) return fail(kErrArg, "null operand pointer");
  return launch_dense_ref_f64(A, s0, s1, B, ldb, C, M, N, K, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
