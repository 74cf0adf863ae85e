// raster_bwd.cu — backward hot path of the B200 ODGS rasterizer.
//
//   k_bwd_raster  one CTA per tile, back to front over the tile list. Each pixel starts
//                 from its stored final transmittance (bit-identical to the reference's
//                 forward replay, backward.hpp:250-269) and runs the suffix recursion
//                 (:271-305). Per entry, the 9 accumulators (EntryGrad, :218-224) are
//                 summed over the tile's pixels in a fixed order (pixel -> warp xor tree
//                 -> warps in index order) and written to the entry's EMIT position, so
//                 every Gaussian's records are contiguous. Deterministic, no atomics.
//   k_fold_records one thread per depth rank: ordered fold of a Gaussian's records
//                 (:310-327) into folded[g][9].
//   k_bwd_splat   one thread per Gaussian: its folded records,
//                 Sigma_2D transport (:329-337), then the per-splat chain rule
//                 (:393-438) incl. the densify statistics, plus the error checks
//                 (pole axis :79-80, non-finite gradient :440-446).
#include <atomic>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "kernels.h"

namespace odgs_b200 {

// The two-barrier kernel (k_bwd_raster_cull) unless ODGS_BWD_KERNEL=pipe selects the
// warp-specialised pipelined kernel (k_bwd_raster_pipe) for A/B measurements: measured on
// a C4 view 2.47 ms against 2.35 ms (profiles/r02/notes.md).
static bool use_pipe_kernel() {
  static const bool pipe = [] {
    const char* e = std::getenv("ODGS_BWD_KERNEL");
    return e && std::strcmp(e, "pipe") == 0;
  }();
  return pipe;
}

constexpr int kBwdThreads = 256;
constexpr int kBwdWarps = kBwdThreads / 32;
constexpr int kBwdBatch = 128;
constexpr int kRec = 9;  // mx, my, m00, m01, m11, op, c0, c1, c2
constexpr int kRecStride = 12;  // floats per entry record in memory: 9 sums + 3 pad (three 16-byte vectors)

__device__ __forceinline__ void store_record(float* r, const float v[kRec]) {
  float4* o = reinterpret_cast<float4*>(r);
  o[0] = make_float4(v[0], v[1], v[2], v[3]);
  o[1] = make_float4(v[4], v[5], v[6], v[7]);
  o[2] = make_float4(v[8], 0.0f, 0.0f, 0.0f);
}
__device__ __forceinline__ void load_record(const float* r, float v[kRec]) {
  const float4* o = reinterpret_cast<const float4*>(r);
  const float4 a = __ldcs(o), b = __ldcs(o + 1), c = __ldcs(o + 2);
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
  v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  v[8] = c.x;
}

// Backward work counters for the roofline (bench.py): entries replayed (sum over pixels
// with a gradient of their walk, the reference's replay loop, backward.hpp:251-269) and
// contributions (replayed entries inside the cutoff, :271-305).
// work[2..3] (culled kernels): warp-entries walked (sum of the warps' list lengths) and
// warp-entries with at least one contributing lane — the culling's efficiency.
// exam is per lane; contrib, warp_entries and warp_live are warp totals (uniform).
__device__ __forceinline__ void bwd_count_work(unsigned long long* work, uint32_t exam, uint32_t contrib,
                                               uint32_t warp_entries = 0, uint32_t warp_live = 0) {
  const uint32_t we = __reduce_add_sync(0xffffffffu, exam);
  const uint32_t wc = contrib;
  if ((threadIdx.x & 31) == 0 && (we | wc | warp_entries)) {
    atomicAdd(work, (unsigned long long)we);
    atomicAdd(work + 1, (unsigned long long)wc);
    atomicAdd(work + 2, (unsigned long long)warp_entries);
    atomicAdd(work + 3, (unsigned long long)warp_live);
  }
}

template <int PPT>
__global__ void __launch_bounds__(kBwdThreads) k_bwd_raster(
    const int32_t* __restrict__ offsets, const uint32_t* __restrict__ vals, const float4* __restrict__ sp_ab,
    const float4* __restrict__ sp_c, const uint32_t* __restrict__ ent_off_idx,
    const float* __restrict__ transmittance, const int32_t* __restrict__ walked_in,
    const float* __restrict__ dl_dimage, int width, int height, int tile_size, int tiles_x, float alpha_clamp,
    float cutoff2, float* __restrict__ records, uint8_t* __restrict__ touched, int band_ty0, int band_ty1,
    unsigned long long* __restrict__ work) {
  __shared__ float s_cx[kBwdBatch], s_cy[kBwdBatch], s_i00[kBwdBatch], s_i01[kBwdBatch], s_i11[kBwdBatch],
      s_op[kBwdBatch], s_col[3][kBwdBatch];
  __shared__ uint32_t s_pos[kBwdBatch];
  __shared__ float s_part[kBwdWarps][kBwdBatch][kRec];
  __shared__ int s_maxw[kBwdWarps];
  __shared__ uint8_t s_had[kBwdBatch];  // record already written by an earlier pixel chunk

  const int tile = band_ty0 * tiles_x + blockIdx.x;
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const int e0 = offsets[tile];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int area = tile_size * tile_size;
  const int64_t plane = (int64_t)width * height;

  // Tiles larger than PPT * 256 pixels (tile_size > 64) are replayed in pixel chunks;
  // each chunk's per-entry sums are added to the records the earlier chunks wrote.
  for (int chunk = 0; chunk < area; chunk += PPT * kBwdThreads) {
  float px[PPT], py[PPT], t[PPT], d0[PPT], d1[PPT], d2v[PPT], suf0[PPT], suf1[PPT], suf2[PPT];
  int wk[PPT];
  int my_max = 0;
  uint32_t n_exam = 0, n_contrib = 0;
#pragma unroll
  for (int q = 0; q < PPT; ++q) {
    const int lp = chunk + tid + q * kBwdThreads;
    const int lx = lp / tile_size, ly = lp - lx * tile_size;
    const int x = tx * tile_size + lx, y = ty * tile_size + ly;
    const bool valid = lp < area && x < width && y < height;
    px[q] = (float)x + 0.5f;
    py[q] = (float)y + 0.5f;
    wk[q] = 0;
    t[q] = 1.0f;
    d0[q] = d1[q] = d2v[q] = 0.0f;
    suf0[q] = suf1[q] = suf2[q] = 0.0f;
    if (valid) {
      const int64_t p = (int64_t)x * height + y;
      d0[q] = dl_dimage[p];
      d1[q] = dl_dimage[plane + p];
      d2v[q] = dl_dimage[2 * plane + p];
      // Only exact zeros are skipped (the reference's float isZero() also skips
      // |g| <= 1e-5, which would silently drop small L1 gradients).
      if (d0[q] != 0.0f || d1[q] != 0.0f || d2v[q] != 0.0f) {
        wk[q] = walked_in[p];
        t[q] = transmittance[p];
      }
    }
    my_max = max(my_max, wk[q]);
    n_exam += (uint32_t)wk[q];
  }
  // CTA-wide max walk: entries at or beyond it are never replayed.
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) my_max = max(my_max, __shfl_xor_sync(0xffffffffu, my_max, d));
  if (lane == 0) s_maxw[warp] = my_max;
  __syncthreads();
  int max_walked = 0;
  for (int w = 0; w < kBwdWarps; ++w) max_walked = max(max_walked, s_maxw[w]);

  for (int hi = max_walked; hi > 0; hi -= kBwdBatch) {
    const int lo = max(0, hi - kBwdBatch);
    const int count = hi - lo;
    if (tid < count) {
      const int e = e0 + lo + tid;
      const uint32_t v = vals[e];
      const uint32_t g = v >> 2;
      const int k = (int)(v & 3u);
      const float4 a = __ldg(sp_ab + 2 * (int64_t)g);
      const float4 b = __ldg(sp_ab + 2 * (int64_t)g + 1);
      const float4 c = __ldg(sp_c + g);
      s_cx[tid] = a.x + shift_of(k, width);
      s_cy[tid] = a.y;
      s_i00[tid] = a.z;
      s_i01[tid] = a.w;
      s_i11[tid] = b.x;
      s_op[tid] = b.y;
      s_col[0][tid] = b.z;
      s_col[1][tid] = b.w;
      s_col[2][tid] = c.x;
      // Emit position of (tile, g, k): the Gaussian's first entry + areas of its
      // earlier shifts + row-major offset inside this shift's tile rectangle.
      uint32_t pos = __ldg(ent_off_idx + g);
      for (int kk = 0; kk <= k; ++kk) {
        int span[4];
        if (!band_tiles(a.x, a.y, c.z, kk, width, height, tile_size, band_ty0, band_ty1, span)) continue;
        const uint32_t w = (uint32_t)(span[1] - span[0] + 1);
        if (kk < k) pos += w * (uint32_t)(span[3] - span[2] + 1);
        else pos += (uint32_t)(ty - span[2]) * w + (uint32_t)(tx - span[0]);
      }
      s_pos[tid] = pos;
    }
    __syncthreads();
    for (int j = count - 1; j >= 0; --j) {
      const int rel = lo + j;  // entry index inside the tile list
      float acc[kRec];
#pragma unroll
      for (int c = 0; c < kRec; ++c) acc[c] = 0.0f;
      bool any = false;
#pragma unroll
      for (int q = 0; q < PPT; ++q) {
        if (rel >= wk[q]) continue;
        const float dx = px[q] - s_cx[j];
        const float dy = py[q] - s_cy[j];
        const float i00 = s_i00[j], i01 = s_i01[j], i11 = s_i11[j];
        const float dd = i00 * dx * dx + 2.0f * i01 * dx * dy + i11 * dy * dy;
        if (dd > cutoff2) continue;
        const float op = s_op[j];
        const float G = pm_expf_blend(-dd / 2.0f);
        const float raw_alpha = op * G;
        const float alpha = std_min(alpha_clamp, raw_alpha);
        const float one_m = 1.0f - alpha;
        const float t_here = t[q] / one_m;
        const float c0 = s_col[0][j], c1 = s_col[1][j], c2 = s_col[2][j];
        acc[6] += d0[q] * alpha * t_here;
        acc[7] += d1[q] * alpha * t_here;
        acc[8] += d2v[q] * alpha * t_here;
        const float v0 = c0 * t_here - suf0[q] / one_m;
        const float v1 = c1 * t_here - suf1[q] / one_m;
        const float v2 = c2 * t_here - suf2[q] / one_m;
        const float dl_dalpha = d0[q] * v0 + (d1[q] * v1 + d2v[q] * v2);
        const float at = alpha * t_here;
        suf0[q] += c0 * at;
        suf1[q] += c1 * at;
        suf2[q] += c2 * at;
        t[q] = t_here;
        any = true;
        ++n_contrib;
        if (raw_alpha > alpha_clamp) continue;  // clamped: no alpha gradient (:289)
        acc[5] += dl_dalpha * G;
        const float dl_dd2 = dl_dalpha * op * (-G / 2.0f);
        const float gx = i00 * dx + i01 * dy;
        const float gy = i01 * dx + i11 * dy;
        acc[0] += dl_dd2 * (-2.0f) * gx;
        acc[1] += dl_dd2 * (-2.0f) * gy;
        acc[2] += dl_dd2 * dx * dx;
        acc[3] += dl_dd2 * dx * dy;
        acc[4] += dl_dd2 * dy * dy;
      }
      if (__any_sync(0xffffffffu, any)) {
#pragma unroll
        for (int c = 0; c < kRec; ++c) {
          float v = acc[c];
#pragma unroll
          for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
          acc[c] = v;
        }
      }
      if (lane < kRec) {
        float v = 0.0f;
#pragma unroll
        for (int c = 0; c < kRec; ++c) v = (lane == c) ? acc[c] : v;
        s_part[warp][j][lane] = v;
      }
    }
    __syncthreads();
    if (chunk > 0) {
      for (int j = tid; j < count; j += kBwdThreads) s_had[j] = touched[s_pos[j]];
      __syncthreads();
    }
    for (int idx = tid; idx < count * kRec; idx += kBwdThreads) {
      const int j = idx / kRec, c = idx - j * kRec;
      float s = 0.0f;
#pragma unroll
      for (int w = 0; w < kBwdWarps; ++w) s += s_part[w][j][c];
      float* r = records + (int64_t)s_pos[j] * kRecStride + c;
      *r = (chunk > 0 && s_had[j]) ? *r + s : s;
      if (c == 0) touched[s_pos[j]] = 1;
    }
    __syncthreads();
  }
  if (work) bwd_count_work(work, n_exam, __reduce_add_sync(0xffffffffu, n_contrib));
  __syncthreads();  // s_maxw and the shared batch are reused by the next chunk
  }
}

// One pixel's contribution to one tile entry in the back-to-front recursion
// (backward.hpp:271-305), starting from the pixel's state after the entries behind
// it; updates (t, suffix) and writes the 9 accumulators. False if it contributed
// nothing (entry beyond the pixel's walk, or d2 > cutoff^2).
//
// The backward is tolerance-checked (group-relative 1e-3 vs fp64), so its arithmetic
// is free to use FMAs, MUFU ex2 and an approximate reciprocal. The two decisions that
// must replay the forward exactly are kept exact: d2 is computed with the forward's
// un-fused products (same bits, so the cutoff skip matches), and when the fast
// exponential lands within 1e-4 of the alpha clamp the exact pm_expf_blend decides
// whether the contribution was clamped (backward.hpp:289).
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ bool bwd_contrib(const float4 geo, const float4 att, const float b, int rel, int wk,
                                            float px, float py, float cutoff2, float alpha_clamp, float d0,
                                            float d1, float d2v, float& t, float& sd, float acc[kRec]) {
#pragma unroll
  for (int c = 0; c < kRec; ++c) acc[c] = 0.0f;
  if (rel >= wk) return false;
  const float dx = px - geo.x;
  const float dy = py - geo.y;
  // geo = (cx, cy, i00, 2*i01): the forward's d2 bit for bit.
  const float dd = __fadd_rn(__fadd_rn(__fmul_rn(__fmul_rn(geo.z, dx), dx), __fmul_rn(__fmul_rn(geo.w, dx), dy)),
                             __fmul_rn(__fmul_rn(att.x, dy), dy));
  if (!(dd <= cutoff2)) return false;
  const float op = att.y;
  // e^(-dd/2) = 2^(dd * -log2(e)/2) on MUFU.EX2 (flush-to-zero: results below 2^-126
  // contribute nothing)
  float G;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(G) : "f"(dd * -0.72134752044448170368f));
  float raw_alpha = op * G;
  if (fabsf(raw_alpha - alpha_clamp) < 1e-4f) {
    G = pm_expf_blend(-dd / 2.0f);
    raw_alpha = op * G;
  }
  const float alpha = fminf(alpha_clamp, raw_alpha);
  const float inv_om = rcp_approx(1.0f - alpha);
  const float t_here = t * inv_om;
  const float c0 = att.z, c1 = att.w, c2 = b;
  const float at = alpha * t_here;
  acc[6] = d0 * at;
  acc[7] = d1 * at;
  acc[8] = d2v * at;
  // dL/dalpha = sum_c d_c (c_c t_here - suffix_c / (1 - alpha)) (backward.hpp:284-287)
  // needs the suffix only through sd = sum_c d_c suffix_c, which the recursion carries
  // as one scalar: sd += (d . c) alpha t_here.
  const float dc = fmaf(d0, c0, fmaf(d1, c1, d2v * c2));
  const float dl_dalpha = fmaf(-sd, inv_om, dc * t_here);
  sd = fmaf(dc, at, sd);
  t = t_here;
  if (!(raw_alpha > alpha_clamp)) {  // clamped: no alpha gradient (backward.hpp:289)
    acc[5] = dl_dalpha * G;
    const float dl_dd2 = dl_dalpha * raw_alpha * -0.5f;  // dl_dalpha * op * (-G / 2)
    // dL/dmean = -2 dl_dd2 Sigma^-1 d is linear in (dl_dd2 dx, dl_dd2 dy) with per-entry
    // coefficients: acc[0..1] carry those two sums, and the warp's writer applies
    // Sigma^-1 once per entry (mean_grad_from_moments) instead of per pixel.
    const float ex = dl_dd2 * dx, ey = dl_dd2 * dy;
    acc[0] = ex;
    acc[1] = ey;
    acc[2] = ex * dx;
    acc[3] = ex * dy;
    acc[4] = ey * dy;
  }
  return true;
}

// acc[0..1] (sums of dl_dd2 dx, dl_dd2 dy) -> the mean gradient -2 Sigma^-1 (sums)
// (backward.hpp:298-300); geo = (cx, cy, i00, 2*i01), i11 = att.x.
__device__ __forceinline__ void mean_grad_from_moments(const float4 geo, float i11, float& a0, float& a1) {
  const float i01 = 0.5f * geo.w, sx = a0, sy = a1;
  a0 = -2.0f * fmaf(geo.z, sx, i01 * sy);
  a1 = -2.0f * fmaf(i01, sx, i11 * sy);
}

// First butterfly level of a pair reduce-scatter: lanes 0-15 keep the sum of A over
// lanes {l, l^16}, lanes 16-31 the sum of B.
__device__ __forceinline__ void pair_level16(const float A[kRec], const float B[kRec], bool upper, float K[kRec]) {
#pragma unroll
  for (int c = 0; c < kRec; ++c) {
    const float r = __shfl_xor_sync(0xffffffffu, upper ? A[c] : B[c], 16);
    K[c] = (upper ? B[c] : A[c]) + r;
  }
}

// Culled variant for tiles up to 16x16 (one pixel per thread): the forward's
// conservative per-warp ellipse test (cull_extents) decides which entries a warp
// can touch; only those are replayed and warp-reduced. Entries no warp touches
// keep their zero record (the buffer is cleared before the launch). Skipping is
// exact: a culled entry has computed d2 > cutoff^2 at every pixel of the warp, so
// its contribution there is zero and it does not change t or the suffix.
template <bool kCount>
__global__ void __launch_bounds__(kBwdThreads, 4) k_bwd_raster_cull(
    const int32_t* __restrict__ offsets, const uint32_t* __restrict__ vals, const float4* __restrict__ sp_ab,
    const float4* __restrict__ sp_c, const uint32_t* __restrict__ ent_off_idx,
    const float* __restrict__ transmittance, const int32_t* __restrict__ walked_in,
    const float* __restrict__ dl_dimage, int width, int height, int tile_size, int tiles_x, float alpha_clamp,
    float cutoff2, float* __restrict__ records, uint8_t* __restrict__ touched, int band_ty0, int band_ty1,
    const uint32_t* __restrict__ order, unsigned long long* __restrict__ work) {
  pdl_wait();
  // One 48-byte record per staged entry (all parts addressed from one base).
  struct alignas(16) Staged {
    float4 geo;  // cx, cy, i00, 2*i01
    float4 att;  // i11, opacity, r, g
    float4 b;    // b, -, -, -
  };
  __shared__ Staged s_ent[kBwdBatch];
  __shared__ uint32_t s_pos[2][kBwdBatch];  // double-buffered: read one batch later
  __shared__ uint8_t s_mask[2][kBwdBatch];
  __shared__ uint8_t s_list[kBwdWarps][kBwdBatch];
  __shared__ float s_part[kBwdWarps][kRec][kBwdBatch];  // 9 sums per (warp, entry), component-major
  __shared__ uint8_t s_wrote[kBwdWarps][kBwdBatch];  // warp wrote the entry's partial (cleared by its reader)
  __shared__ int s_maxw[kBwdWarps];
  __shared__ float4 s_wbox[kBwdWarps];

  const int tile = band_ty0 * tiles_x + (int)(order ? order[blockIdx.x] : blockIdx.x);
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const int e0 = offsets[tile];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t plane = (int64_t)width * height;
  const uint32_t lt_mask = (1u << lane) - 1u;

  int lx, ly;
  bool valid;
  if (tile_size == 16) {
    lx = (warp & 1) * 8 + (lane >> 2);  // 8-wide x 4-tall warp blocks, as the blend
    ly = (warp >> 1) * 4 + (lane & 3);
    valid = true;
  } else {
    lx = tid / tile_size;
    ly = tid - lx * tile_size;
    valid = tid < tile_size * tile_size;
  }
  const int x = tx * tile_size + lx, y = ty * tile_size + ly;
  valid = valid && x < width && y < height;
  const float px = (float)x + 0.5f, py = (float)y + 0.5f;
  float t = 1.0f, d0 = 0.0f, d1 = 0.0f, d2v = 0.0f, sd = 0.0f;  // sd = dL/dpixel . suffix
  int wk = 0;
  if (valid) {
    const int64_t p = (int64_t)x * height + y;
    d0 = dl_dimage[p];
    d1 = dl_dimage[plane + p];
    d2v = dl_dimage[2 * plane + p];
    // Only exact zeros are skipped (the reference's float isZero()).
    if (d0 != 0.0f || d1 != 0.0f || d2v != 0.0f) {
      wk = walked_in[p];
      t = transmittance[p];
    }
  }
  uint32_t n_contrib = 0, n_wentries = 0, n_wlive = 0;
  // Warp box over the pixels that replay anything; max walk over the CTA.
  const bool active = wk > 0;
  float bx0 = active ? px : INFINITY, bx1 = active ? px : -INFINITY;
  float by0 = active ? py : INFINITY, by1 = active ? py : -INFINITY;
  int my_max = wk;
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    bx0 = fminf(bx0, __shfl_xor_sync(0xffffffffu, bx0, d));
    bx1 = fmaxf(bx1, __shfl_xor_sync(0xffffffffu, bx1, d));
    by0 = fminf(by0, __shfl_xor_sync(0xffffffffu, by0, d));
    by1 = fmaxf(by1, __shfl_xor_sync(0xffffffffu, by1, d));
    my_max = max(my_max, __shfl_xor_sync(0xffffffffu, my_max, d));
  }
  if (lane == 0) {
    s_maxw[warp] = my_max;
    s_wbox[warp] = make_float4(bx0, bx1, by0, by1);
  }
  __syncthreads();
  int max_walked = 0;
  for (int w = 0; w < kBwdWarps; ++w) max_walked = max(max_walked, s_maxw[w]);

  for (int i = tid; i < kBwdWarps * kBwdBatch; i += kBwdThreads) (&s_wrote[0][0])[i] = 0;

  // Batches of kBwdBatch entries, back to front. Per batch two barriers:
  //   phase A  threads 0-127 stage batch b (entry data, warp masks, emit positions);
  //            threads 128-255 sum batch b-1's per-warp partials in warp order and
  //            write its records
  //   -- barrier --
  //   phase B  every warp compacts its entries of batch b and walks them
  //   -- barrier --
  // A final phase A writes the last batch.
  int prev_count = 0, buf = 0;
  for (int hi = max_walked;; hi -= kBwdBatch) {
    const bool have = hi > 0;
    const int lo = have ? max(0, hi - kBwdBatch) : 0;
    const int count = have ? hi - lo : 0;
    if (tid < kBwdBatch) {
      if (have) {
        uint32_t mask = 0;
        if (tid < count) {
          const int e = e0 + lo + tid;
          const uint32_t v = vals[e];
          const uint32_t g = v >> 2;
          const int k = (int)(v & 3u);
          const float4 a = __ldg(sp_ab + 2 * (int64_t)g);
          const float4 b = __ldg(sp_ab + 2 * (int64_t)g + 1);
          const float4 c = __ldg(sp_c + g);
          const float cx = a.x + shift_of(k, width), cy = a.y;
          s_ent[tid].geo = make_float4(cx, cy, a.z, 2.0f * a.w);
          s_ent[tid].att = b;
          s_ent[tid].b.x = c.x;
          float ex, ey;
          // Warps whose longest walk ends before this entry never replay it.
          const int rel = lo + tid;
          if (cull_extents(a.z, a.w, b.x, cutoff2, &ex, &ey)) {
#pragma unroll
            for (int w = 0; w < kBwdWarps; ++w) {
              const float4 bx = s_wbox[w];
              const bool out = (bx.x - cx > ex) || (bx.y - cx < -ex) || (bx.z - cy > ey) || (bx.w - cy < -ey) ||
                               rel >= s_maxw[w];
              mask |= out ? 0u : (1u << w);
            }
          } else {
#pragma unroll
            for (int w = 0; w < kBwdWarps; ++w) mask |= rel < s_maxw[w] ? (1u << w) : 0u;
          }
          if (mask) {
            // Emit position of (tile, g, k): first entry of g + earlier shifts' areas +
            // row-major offset inside this shift's (band-clipped) tile rectangle.
            uint32_t pos = __ldg(ent_off_idx + g);
            for (int kk = 0; kk <= k; ++kk) {
              int span[4];
              if (!band_tiles(a.x, a.y, c.z, kk, width, height, tile_size, band_ty0, band_ty1, span)) continue;
              const uint32_t w = (uint32_t)(span[1] - span[0] + 1);
              if (kk < k) pos += w * (uint32_t)(span[3] - span[2] + 1);
              else pos += (uint32_t)(ty - span[2]) * w + (uint32_t)(tx - span[0]);
            }
            s_pos[buf][tid] = pos;
          }
        }
        s_mask[buf][tid] = (uint8_t)mask;
      }
    } else if (prev_count > 0) {
      const int j = tid - kBwdBatch;
      if (j < prev_count && s_mask[buf ^ 1][j]) {
        float sum[kRec];
#pragma unroll
        for (int c = 0; c < kRec; ++c) sum[c] = 0.0f;
        bool any_w = false;
#pragma unroll
        for (int w = 0; w < kBwdWarps; ++w)
          if (s_wrote[w][j]) {
            s_wrote[w][j] = 0;
            any_w = true;
#pragma unroll
            for (int c = 0; c < kRec; ++c) sum[c] += s_part[w][c][j];
          }
        if (any_w) {
          const uint32_t pos = s_pos[buf ^ 1][j];
          store_record(records + (int64_t)pos * kRecStride, sum);
          touched[pos] = 1;
        }
      }
    }
    if (!have) break;
    __syncthreads();
    int n_list = 0;
#pragma unroll
    for (int cidx = 0; cidx < kBwdBatch / 32; ++cidx) {
      const bool mine = (s_mask[buf][cidx * 32 + lane] >> warp) & 1u;
      const uint32_t bal = __ballot_sync(0xffffffffu, mine);
      if (mine) s_list[warp][n_list + __popc(bal & lt_mask)] = (uint8_t)(cidx * 32 + lane);
      n_list += __popc(bal);
    }
    __syncwarp();
    // Back to front over this warp's entries, four at a time: the 4 x 9 per-pixel
    // contributions are reduce-scattered over the warp (level 16 splits A|B and C|D,
    // level 8 splits AB|CD, levels 4-2-1 finish) — 54 shuffles per 4 entries. The
    // totals land on lanes 0 (A), 8 (C), 16 (B) and 24 (D).
    const bool upper = lane & 16, mid = lane & 8;
    if (kCount) n_wentries += (uint32_t)n_list;
    for (int qi = n_list - 1; qi >= 0; qi -= 4) {
      const int ja = s_list[warp][qi];
      const int jb = qi >= 1 ? s_list[warp][qi - 1] : -1;
      const int jc = qi >= 2 ? s_list[warp][qi - 2] : -1;
      const int jd = qi >= 3 ? s_list[warp][qi - 3] : -1;
      float K1[kRec], K2[kRec];
      unsigned ma, mb, mc, md;
      {
        float A[kRec], B[kRec];
        const bool any_a = bwd_contrib(s_ent[ja].geo, s_ent[ja].att, s_ent[ja].b.x, lo + ja, wk, px, py, cutoff2, alpha_clamp, d0,
                                       d1, d2v, t, sd, A);
        bool any_b = false;
        if (jb >= 0)
          any_b = bwd_contrib(s_ent[jb].geo, s_ent[jb].att, s_ent[jb].b.x, lo + jb, wk, px, py, cutoff2, alpha_clamp, d0, d1, d2v,
                              t, sd, B);
        else
#pragma unroll
          for (int c = 0; c < kRec; ++c) B[c] = 0.0f;
        ma = __ballot_sync(0xffffffffu, any_a);
        mb = __ballot_sync(0xffffffffu, any_b);
        if (ma | mb) pair_level16(A, B, upper, K1);
        else
#pragma unroll
          for (int c = 0; c < kRec; ++c) K1[c] = 0.0f;
      }
      {
        float C[kRec], D[kRec];
        bool any_c = false, any_d = false;
        if (jc >= 0)
          any_c = bwd_contrib(s_ent[jc].geo, s_ent[jc].att, s_ent[jc].b.x, lo + jc, wk, px, py, cutoff2, alpha_clamp, d0, d1, d2v,
                              t, sd, C);
        else
#pragma unroll
          for (int c = 0; c < kRec; ++c) C[c] = 0.0f;
        if (jd >= 0)
          any_d = bwd_contrib(s_ent[jd].geo, s_ent[jd].att, s_ent[jd].b.x, lo + jd, wk, px, py, cutoff2, alpha_clamp, d0, d1, d2v,
                              t, sd, D);
        else
#pragma unroll
          for (int c = 0; c < kRec; ++c) D[c] = 0.0f;
        mc = __ballot_sync(0xffffffffu, any_c);
        md = __ballot_sync(0xffffffffu, any_d);
        if (mc | md) pair_level16(C, D, upper, K2);
        else
#pragma unroll
          for (int c = 0; c < kRec; ++c) K2[c] = 0.0f;
      }
      if (kCount) {
        n_wlive += (uint32_t)(ma != 0) + (uint32_t)(mb != 0) + (uint32_t)(mc != 0) + (uint32_t)(md != 0);
        n_contrib += __popc(ma) + __popc(mb) + __popc(mc) + __popc(md);
      }
      if (ma | mb | mc | md) {
        float L[kRec];
#pragma unroll
        for (int c = 0; c < kRec; ++c) {
          const float r = __shfl_xor_sync(0xffffffffu, mid ? K1[c] : K2[c], 8);
          L[c] = (mid ? K2[c] : K1[c]) + r;
        }
#pragma unroll
        for (int d = 4; d > 0; d >>= 1)
#pragma unroll
          for (int c = 0; c < kRec; ++c) L[c] += __shfl_xor_sync(0xffffffffu, L[c], d);
        const int grp = lane >> 3;  // 0: A, 1: C, 2: B, 3: D
        const unsigned mine = grp == 0 ? ma : (grp == 1 ? mc : (grp == 2 ? mb : md));
        if ((lane & 7) == 0 && mine) {
          const int j = grp == 0 ? ja : (grp == 1 ? jc : (grp == 2 ? jb : jd));
          mean_grad_from_moments(s_ent[j].geo, s_ent[j].att.x, L[0], L[1]);
#pragma unroll
          for (int c = 0; c < kRec; ++c) s_part[warp][c][j] = L[c];
          s_wrote[warp][j] = 1;
        }
      }
    }
    __syncthreads();
    prev_count = count;
    buf ^= 1;
  }
  if (kCount) bwd_count_work(work, (uint32_t)wk, n_contrib, n_wentries, n_wlive);
}

// ------------------------------------------------------------------ warp-specialised backward raster
// One CTA per tile (up to 16x16): kPipeWarps compute warps each own an 8x8 pixel block
// (two pixels per lane, so one warp reduction covers 64 pixels) and one producer warp
// feeds them through a ring of kPipeStages shared-memory slots of kPipeBatch entries,
// synchronised with mbarriers instead of CTA barriers:
//   producer  per batch (back to front): wait until every compute warp released the
//             slot (empty), sum the slot's previous per-warp partials in warp order and
//             write their records, stage the new batch (entry data, per-warp cull masks,
//             emit positions), arrive on full;
//   compute   per batch: wait full, compact the warp's entries, walk them four at a time
//             (two pixels per lane, reduce-scatter of the 4 x 9 sums over the warp),
//             store the warp's partials in the slot, arrive on empty.
// A warp can run up to kPipeStages - 1 batches ahead of the slowest one, so per-batch
// imbalance between the warps' lists no longer stalls the CTA (the previous kernel's two
// __syncthreads per batch). Records and their fixed summation order are as before:
// deterministic, no atomics.
#ifndef ODGS_PIPE_STAGES
#define ODGS_PIPE_STAGES 4
#endif
#ifndef ODGS_PIPE_MINB
#define ODGS_PIPE_MINB 4
#endif
#ifndef ODGS_PIPE_WIDE
#define ODGS_PIPE_WIDE 0
#endif
#ifndef ODGS_PIPE_SLEEP
#define ODGS_PIPE_SLEEP 0
#endif
constexpr int kPipeWarps = 4;
constexpr int kPipeThreads = (kPipeWarps + 1) * 32;
constexpr int kPipeBatch = 64;
constexpr int kPipeStages = ODGS_PIPE_STAGES;
constexpr bool kPipeWide = ODGS_PIPE_WIDE;  // 16x4 warp blocks instead of 8x8

struct alignas(16) PipeEntry {
  float4 geo;  // cx, cy, i00, 2*i01
  float4 att;  // i11, opacity, r, g
  float4 b;    // b, -, -, -
};
struct PipeSlot {
  PipeEntry ent[kPipeBatch];
  float part[kPipeWarps][kRec][kPipeBatch];  // per-warp sums, component-major
  uint32_t pos[kPipeBatch];                  // emit position of the entry
  uint8_t mask[kPipeBatch];                  // warps whose block the entry can touch
  uint8_t wrote[kPipeWarps][kPipeBatch];     // warp stored a partial (cleared by the producer)
};
struct PipeSmem {
  PipeSlot slot[kPipeStages];
  unsigned long long full[kPipeStages], empty[kPipeStages];
  float4 wbox[kPipeWarps];
  int maxw[kPipeWarps];
  uint8_t list[kPipeWarps][kPipeBatch];
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// The producer's wait: try_wait with a nanosleep back-off, so an idle producer does not
// take issue slots from the compute warps.
__device__ __forceinline__ void mbar_wait_backoff(unsigned long long* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  for (;;) {
    uint32_t done;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
    if (done) return;
    if (ODGS_PIPE_SLEEP > 0) __nanosleep(ODGS_PIPE_SLEEP);
  }
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred done;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 done, [%0], %1;\n\t"
      "@!done bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// bwd_contrib for both pixels of a lane, summed into acc; true if either contributed.
__device__ __forceinline__ bool bwd_contrib2(const PipeEntry& en, int rel, const int wk[2], const float px[2],
                                             const float py[2], float cutoff2, float alpha_clamp, const float d0[2],
                                             const float d1[2], const float d2v[2], float t[2], float sd[2],
                                             float acc[kRec]) {
  float a1[kRec];
  const bool c0 = bwd_contrib(en.geo, en.att, en.b.x, rel, wk[0], px[0], py[0], cutoff2, alpha_clamp, d0[0], d1[0],
                              d2v[0], t[0], sd[0], acc);
  const bool c1 = bwd_contrib(en.geo, en.att, en.b.x, rel, wk[1], px[1], py[1], cutoff2, alpha_clamp, d0[1], d1[1],
                              d2v[1], t[1], sd[1], a1);
#pragma unroll
  for (int c = 0; c < kRec; ++c) acc[c] += a1[c];
  return c0 || c1;
}

__global__ void __launch_bounds__(kPipeThreads, ODGS_PIPE_MINB) k_bwd_raster_pipe(
    const int32_t* __restrict__ offsets, const uint32_t* __restrict__ vals, const float4* __restrict__ sp_ab,
    const float4* __restrict__ sp_c, const uint32_t* __restrict__ ent_off_idx,
    const float* __restrict__ transmittance, const int32_t* __restrict__ walked_in,
    const float* __restrict__ dl_dimage, int width, int height, int tile_size, int tiles_x, float alpha_clamp,
    float cutoff2, float* __restrict__ records, uint8_t* __restrict__ touched, int band_ty0, int band_ty1,
    const uint32_t* __restrict__ order, unsigned long long* __restrict__ work) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char s_raw[];
  PipeSmem& S = *reinterpret_cast<PipeSmem*>(s_raw);
  const int tile = band_ty0 * tiles_x + (int)(order ? order[blockIdx.x] : blockIdx.x);
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const int e0 = offsets[tile];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool producer = warp == kPipeWarps;
  const int64_t plane = (int64_t)width * height;
  const uint32_t lt_mask = (1u << lane) - 1u;

  // Compute warps: two pixels per lane. 16x16 tiles: warp w owns the 8x8 block at
  // (8 (w & 1), 8 (w >> 1)); lanes run down a column in fours (the image is column-major),
  // the second pixel 4 rows lower. Smaller tiles: slots warp*64 + 32q + lane, column-major.
  float px[2], py[2], t[2] = {1.0f, 1.0f}, d0[2] = {0.0f, 0.0f}, d1[2] = {0.0f, 0.0f}, d2v[2] = {0.0f, 0.0f};
  float sd[2] = {0.0f, 0.0f};
  int wk[2] = {0, 0};
  uint32_t n_contrib = 0, n_wentries = 0, n_wlive = 0;
  if (!producer) {
    float bx0 = INFINITY, bx1 = -INFINITY, by0 = INFINITY, by1 = -INFINITY;
    int my_max = 0;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      int lx, ly;
      bool valid;
      if (tile_size == 16) {
        if (kPipeWide) {
          lx = (lane >> 2) + 8 * q;
          ly = warp * 4 + (lane & 3);
        } else {
          lx = (warp & 1) * 8 + (lane >> 2);
          ly = (warp >> 1) * 8 + (lane & 3) + 4 * q;
        }
        valid = true;
      } else {
        const int sl = warp * 64 + q * 32 + lane;
        lx = sl / tile_size;
        ly = sl - lx * tile_size;
        valid = sl < tile_size * tile_size;
      }
      const int x = tx * tile_size + lx, y = ty * tile_size + ly;
      valid = valid && x < width && y < height;
      px[q] = (float)x + 0.5f;
      py[q] = (float)y + 0.5f;
      if (valid) {
        const int64_t p = (int64_t)x * height + y;
        d0[q] = dl_dimage[p];
        d1[q] = dl_dimage[plane + p];
        d2v[q] = dl_dimage[2 * plane + p];
        // Only exact zeros are skipped (the reference's float isZero()).
        if (d0[q] != 0.0f || d1[q] != 0.0f || d2v[q] != 0.0f) {
          wk[q] = walked_in[p];
          t[q] = transmittance[p];
        }
      }
      if (wk[q] > 0) {  // the warp box covers the pixels that replay anything
        bx0 = fminf(bx0, px[q]);
        bx1 = fmaxf(bx1, px[q]);
        by0 = fminf(by0, py[q]);
        by1 = fmaxf(by1, py[q]);
      }
      my_max = max(my_max, wk[q]);
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      bx0 = fminf(bx0, __shfl_xor_sync(0xffffffffu, bx0, d));
      bx1 = fmaxf(bx1, __shfl_xor_sync(0xffffffffu, bx1, d));
      by0 = fminf(by0, __shfl_xor_sync(0xffffffffu, by0, d));
      by1 = fmaxf(by1, __shfl_xor_sync(0xffffffffu, by1, d));
      my_max = max(my_max, __shfl_xor_sync(0xffffffffu, my_max, d));
    }
    if (lane == 0) {
      S.maxw[warp] = my_max;
      S.wbox[warp] = make_float4(bx0, bx1, by0, by1);
    }
  } else {
    if (lane < kPipeStages) {
      mbar_init(&S.full[lane], 32);                 // the producer warp's lanes
      mbar_init(&S.empty[lane], kPipeWarps * 32);   // every compute lane
    }
    for (int k = lane; k < kPipeStages * kPipeWarps * kPipeBatch; k += 32)
      (&S.slot[k / (kPipeWarps * kPipeBatch)].wrote[0][0])[k % (kPipeWarps * kPipeBatch)] = 0;
  }
  __syncthreads();  // pixel boxes, walks, barrier initialisation
  int max_walked = 0;
#pragma unroll
  for (int w = 0; w < kPipeWarps; ++w) max_walked = max(max_walked, S.maxw[w]);
  const int n_batches = (max_walked + kPipeBatch - 1) / kPipeBatch;

  if (producer) {
    for (int i = 0; i < n_batches + kPipeStages; ++i) {
      const int st = i % kPipeStages;
      PipeSlot& sl = S.slot[st];
      const int prev = i - kPipeStages;
      if (prev >= 0 && prev < n_batches) {
        // Records of batch `prev`: the per-warp partials summed in warp order.
        mbar_wait_backoff(&S.empty[st], (uint32_t)(prev / kPipeStages) & 1u);
        const int hi = max_walked - prev * kPipeBatch;
        const int count = min(kPipeBatch, hi);
        for (int k = lane; k < count; k += 32) {
          if (!sl.mask[k]) continue;
          float sum[kRec];
#pragma unroll
          for (int c = 0; c < kRec; ++c) sum[c] = 0.0f;
          bool any = false;
#pragma unroll
          for (int w = 0; w < kPipeWarps; ++w)
            if (sl.wrote[w][k]) {
              sl.wrote[w][k] = 0;
              any = true;
#pragma unroll
              for (int c = 0; c < kRec; ++c) sum[c] += sl.part[w][c][k];
            }
          if (any) {
            const uint32_t pos = sl.pos[k];
            store_record(records + (int64_t)pos * kRecStride, sum);
            touched[pos] = 1;
          }
        }
      }
      if (i < n_batches) {
        // Stage batch i: entries [lo, hi) of the tile list, back to front.
        const int hi = max_walked - i * kPipeBatch;
        const int lo = max(0, hi - kPipeBatch);
        const int count = hi - lo;
        for (int k = lane; k < kPipeBatch; k += 32) {
          uint32_t mask = 0;
          if (k < count) {
            const int rel = lo + k;
            const uint32_t v = vals[e0 + rel];
            const uint32_t g = v >> 2;
            const int sk = (int)(v & 3u);
            const float4 a = __ldg(sp_ab + 2 * (int64_t)g);
            const float4 b = __ldg(sp_ab + 2 * (int64_t)g + 1);
            const float4 c = __ldg(sp_c + g);
            const float cx = a.x + shift_of(sk, width), cy = a.y;
            sl.ent[k].geo = make_float4(cx, cy, a.z, 2.0f * a.w);
            sl.ent[k].att = b;
            sl.ent[k].b.x = c.x;
            float ex, ey;
            const bool cullable = cull_extents(a.z, a.w, b.x, cutoff2, &ex, &ey);
#pragma unroll
            for (int w = 0; w < kPipeWarps; ++w) {
              const float4 bx = S.wbox[w];
              const bool out = rel >= S.maxw[w] || (cullable && ((bx.x - cx > ex) || (bx.y - cx < -ex) ||
                                                                 (bx.z - cy > ey) || (bx.w - cy < -ey)));
              mask |= out ? 0u : (1u << w);
            }
            if (mask) {
              // Emit position of (tile, g, shift): first entry of g + earlier shifts' areas +
              // row-major offset inside this shift's (band-clipped) tile rectangle.
              uint32_t pos = __ldg(ent_off_idx + g);
              for (int kk = 0; kk <= sk; ++kk) {
                int span[4];
                if (!band_tiles(a.x, a.y, c.z, kk, width, height, tile_size, band_ty0, band_ty1, span)) continue;
                const uint32_t wd = (uint32_t)(span[1] - span[0] + 1);
                if (kk < sk) pos += wd * (uint32_t)(span[3] - span[2] + 1);
                else pos += (uint32_t)(ty - span[2]) * wd + (uint32_t)(tx - span[0]);
              }
              sl.pos[k] = pos;
            }
          }
          sl.mask[k] = (uint8_t)mask;
        }
        mbar_arrive(&S.full[st]);
      }
    }
  } else {
    const bool upper = lane & 16, mid = lane & 8;
    for (int i = 0; i < n_batches; ++i) {
      const int st = i % kPipeStages;
      PipeSlot& sl = S.slot[st];
      mbar_wait(&S.full[st], (uint32_t)(i / kPipeStages) & 1u);
      const int lo = max(0, max_walked - i * kPipeBatch - kPipeBatch);
      int n_list = 0;
#pragma unroll
      for (int cidx = 0; cidx < kPipeBatch / 32; ++cidx) {
        const bool mine = (sl.mask[cidx * 32 + lane] >> warp) & 1u;
        const uint32_t bal = __ballot_sync(0xffffffffu, mine);
        if (mine) S.list[warp][n_list + __popc(bal & lt_mask)] = (uint8_t)(cidx * 32 + lane);
        n_list += __popc(bal);
      }
      __syncwarp();
      n_wentries += (uint32_t)n_list;
      // Back to front over this warp's entries, four at a time: the 4 x 9 per-lane sums
      // (two pixels each) are reduce-scattered over the warp; the totals land on lanes 0
      // (A), 8 (C), 16 (B) and 24 (D).
      for (int qi = n_list - 1; qi >= 0; qi -= 4) {
        const int ja = S.list[warp][qi];
        const int jb = qi >= 1 ? S.list[warp][qi - 1] : -1;
        const int jc = qi >= 2 ? S.list[warp][qi - 2] : -1;
        const int jd = qi >= 3 ? S.list[warp][qi - 3] : -1;
        float K1[kRec], K2[kRec];
        unsigned ma, mb, mc, md;
        {
          float A[kRec], B[kRec];
          const bool any_a = bwd_contrib2(sl.ent[ja], lo + ja, wk, px, py, cutoff2, alpha_clamp, d0, d1, d2v, t, sd, A);
          bool any_b = false;
          if (jb >= 0)
            any_b = bwd_contrib2(sl.ent[jb], lo + jb, wk, px, py, cutoff2, alpha_clamp, d0, d1, d2v, t, sd, B);
          else
#pragma unroll
            for (int c = 0; c < kRec; ++c) B[c] = 0.0f;
          ma = __ballot_sync(0xffffffffu, any_a);
          mb = __ballot_sync(0xffffffffu, any_b);
          if (ma | mb) pair_level16(A, B, upper, K1);
          else
#pragma unroll
            for (int c = 0; c < kRec; ++c) K1[c] = 0.0f;
        }
        {
          float Cc[kRec], D[kRec];
          bool any_c = false, any_d = false;
          if (jc >= 0)
            any_c = bwd_contrib2(sl.ent[jc], lo + jc, wk, px, py, cutoff2, alpha_clamp, d0, d1, d2v, t, sd, Cc);
          else
#pragma unroll
            for (int c = 0; c < kRec; ++c) Cc[c] = 0.0f;
          if (jd >= 0)
            any_d = bwd_contrib2(sl.ent[jd], lo + jd, wk, px, py, cutoff2, alpha_clamp, d0, d1, d2v, t, sd, D);
          else
#pragma unroll
            for (int c = 0; c < kRec; ++c) D[c] = 0.0f;
          mc = __ballot_sync(0xffffffffu, any_c);
          md = __ballot_sync(0xffffffffu, any_d);
          if (mc | md) pair_level16(Cc, D, upper, K2);
          else
#pragma unroll
            for (int c = 0; c < kRec; ++c) K2[c] = 0.0f;
        }
        n_wlive += (uint32_t)(ma != 0) + (uint32_t)(mb != 0) + (uint32_t)(mc != 0) + (uint32_t)(md != 0);
        n_contrib += __popc(ma) + __popc(mb) + __popc(mc) + __popc(md);  // lanes (of 2 pixels) contributing
        if (ma | mb | mc | md) {
          float L[kRec];
#pragma unroll
          for (int c = 0; c < kRec; ++c) {
            const float r = __shfl_xor_sync(0xffffffffu, mid ? K1[c] : K2[c], 8);
            L[c] = (mid ? K2[c] : K1[c]) + r;
          }
#pragma unroll
          for (int d = 4; d > 0; d >>= 1)
#pragma unroll
            for (int c = 0; c < kRec; ++c) L[c] += __shfl_xor_sync(0xffffffffu, L[c], d);
          const int grp = lane >> 3;  // 0: A, 1: C, 2: B, 3: D
          const unsigned mine = grp == 0 ? ma : (grp == 1 ? mc : (grp == 2 ? mb : md));
          if ((lane & 7) == 0 && mine) {
            const int j = grp == 0 ? ja : (grp == 1 ? jc : (grp == 2 ? jb : jd));
            mean_grad_from_moments(sl.ent[j].geo, sl.ent[j].att.x, L[0], L[1]);
#pragma unroll
            for (int c = 0; c < kRec; ++c) sl.part[warp][c][j] = L[c];
            sl.wrote[warp][j] = 1;
          }
        }
      }
      __syncwarp();
      mbar_arrive(&S.empty[st]);
    }
  }
  if (work && !producer) bwd_count_work(work, (uint32_t)(wk[0] + wk[1]), n_contrib, n_wentries, n_wlive);
}

void launch_bwd_raster(const BwdRasterArgs& a, cudaStream_t stream) {
  const int n_tiles = a.tiles_x * (a.band_ty1 - a.band_ty0);
  if (n_tiles <= 0) return;
  const float cutoff2 = a.cutoff_sigma * a.cutoff_sigma;
  const int area = a.tile_size * a.tile_size;
  if (!a.plain && a.tile_size <= 16 && use_pipe_kernel()) {
    constexpr size_t smem = sizeof(PipeSmem);
    static std::atomic<uint64_t> opted{0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(opted.load() & (1ull << (dev & 63)))) {
      cudaFuncSetAttribute(k_bwd_raster_pipe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      opted.fetch_or(1ull << (dev & 63));
    }
    launch_pdl(k_bwd_raster_pipe, n_tiles, kPipeThreads, smem, stream, a.offsets, a.vals, a.sp_ab, a.sp_c,
               a.ent_off_idx, a.transmittance, a.walked, a.dl_dimage, a.width, a.height, a.tile_size, a.tiles_x,
               a.alpha_clamp, cutoff2, a.records, a.touched, a.band_ty0, a.band_ty1, a.order, a.work);
    ++g_launches;
    return;
  }
  if (!a.plain && a.tile_size <= 16) {
    // The counting instantiation only when counters are requested (they cost registers).
    launch_pdl(a.work ? k_bwd_raster_cull<true> : k_bwd_raster_cull<false>, n_tiles, kBwdThreads, 0, stream, a.offsets, a.vals, a.sp_ab, a.sp_c, a.ent_off_idx,
                                                           a.transmittance, a.walked, a.dl_dimage, a.width,
                                                           a.height, a.tile_size, a.tiles_x, a.alpha_clamp, cutoff2,
                                                           a.records, a.touched, a.band_ty0, a.band_ty1, a.order,
                                                           a.work);
    ++g_launches;
    return;
  }
#define ODGS_BWD(PPT)                                                                                             \
  k_bwd_raster<PPT><<<n_tiles, kBwdThreads, 0, stream>>>(a.offsets, a.vals, a.sp_ab, a.sp_c, a.ent_off_idx,       \
                                                         a.transmittance, a.walked, a.dl_dimage, a.width, a.height, \
                                                         a.tile_size, a.tiles_x, a.alpha_clamp, cutoff2, a.records, a.touched, \
                                                         a.band_ty0, a.band_ty1, a.work)
  if (area <= kBwdThreads) ODGS_BWD(1);
  else if (area <= 4 * kBwdThreads) ODGS_BWD(4);
  else ODGS_BWD(16);
#undef ODGS_BWD
  ++g_launches;
}

// ------------------------------------------------------------------ per-splat chain rule
__device__ __forceinline__ bool all_finite(const float* v, int n) {
  bool ok = true;
  for (int k = 0; k < n; ++k) ok = ok && isfinite(v[k]);
  return ok;
}

// jacobian_omni_factored (projection.hpp:75-96) in closed form from the camera-space
// components, without trigonometry: with rho = hypot(x, z) and r = |mu|, sin / cos of the
// azimuth are x / rho, z / rho and of the elevation -y / r, rho / r, and sec(elevation) =
// r / rho — or 1 / cos(max_elevation) where the forward clamped it (its flag decides, so
// the branch matches the forward's). Rows (kw sec / r)(cp, 0, -sp), (kh / r)(st sp, ct,
// st cp). Tolerance-checked like the rest of the per-splat backward.
struct Angles {
  float sp, cp, st, ct, rho, rho2, r, r2, inv_rho, inv_r;
};

__device__ __forceinline__ Angles angles_of(float x, float y, float z) {
  Angles g;
  g.rho2 = x * x + z * z;
  g.rho = sqrtf(g.rho2);
  g.r2 = g.rho2 + y * y;
  g.r = sqrtf(g.r2);
  g.inv_rho = __frcp_rn(g.rho);
  g.inv_r = __frcp_rn(g.r);
  if (g.rho > 0.0f) {
    g.sp = x * g.inv_rho;
    g.cp = z * g.inv_rho;
  } else {  // atan2(0, 0) = 0, as the forward's azimuth
    g.sp = 0.0f;
    g.cp = 1.0f;
  }
  g.st = -y * g.inv_r;
  g.ct = g.rho * g.inv_r;
  return g;
}

__device__ __forceinline__ M23 jacobian_from_angles(const Angles& g, float W, float H, bool clamped, float sec_max) {
  const float sec = clamped ? sec_max : g.r * g.inv_rho;
  const float a0 = W / (2.0f * kPiF) * sec * g.inv_r, a1 = H / kPiF * g.inv_r;
  M23 j;
  j.a[0][0] = a0 * g.cp; j.a[0][1] = 0.0f; j.a[0][2] = -a0 * g.sp;
  j.a[1][0] = a1 * g.st * g.sp; j.a[1][1] = a1 * g.ct; j.a[1][2] = a1 * g.st * g.cp;
  return j;
}

__global__ void __launch_bounds__(256, 4) k_bwd_splat(BwdSplatArgs a) {
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n = a.n;
  if (i >= n) return;
  const float4 c4 = a.sp_c[i];
  const uint32_t flags = __float_as_uint(c4.w);
  if (a.accumulate && !(flags & kFlagVisible)) return;  // adds nothing: no read-modify-write
  if (a.accumulate) {
    // The accumulators are read only after the chain rule: fetch their lines into L2
    // now, so the final read-modify-write does not wait on DRAM.
    const float* acc_rows[6] = {a.g_means, a.g_rotations, a.g_log_scales, a.g_raw_opacities, a.g_colors, nullptr};
    const int widths[5] = {3, 4, 3, 1, 3};
    for (int k = 0; k < 5; ++k)
      for (int c = 0; c < widths[k]; ++c)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(acc_rows[k] + (int64_t)c * n + i));
    if (a.g_pixel_grad_norm) asm volatile("prefetch.global.L2 [%0];" ::"l"(a.g_pixel_grad_norm + i));
    if (a.g_one_minus_cos) asm volatile("prefetch.global.L2 [%0];" ::"l"(a.g_one_minus_cos + i));
    if (a.g_observed) asm volatile("prefetch.global.L2 [%0];" ::"l"(a.g_observed + i));
  }
  float gm[3] = {0, 0, 0}, gq[4] = {0, 0, 0, 0}, gls[3] = {0, 0, 0}, gop = 0, gcol[3] = {0, 0, 0};
  float pgn = 0, omc = 0;
  int observed = 0;
  if (flags & kFlagVisible) {
    observed = 1;
    // This Gaussian's folded entry records (k_fold_records).
    float r[kRec] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    if (a.cnt[i] > 0) {
#pragma unroll
      for (int c = 0; c < kRec; ++c) r[c] = a.folded[i * kRec + c];
    }
    const float4 ab0 = a.sp_ab[2 * i], ab1 = a.sp_ab[2 * i + 1];
    const float inv[2][2] = {{ab0.z, ab0.w}, {ab0.w, ab1.x}};
    const float ginv[2][2] = {{r[2], r[3]}, {r[3], r[4]}};
    // dL/dSigma2D = -inv * G_inv * inv (backward.hpp:336)
    float tmp[2][2], dcov[2][2];
    for (int p = 0; p < 2; ++p)
      for (int q = 0; q < 2; ++q) tmp[p][q] = (-inv[p][0]) * ginv[0][q] + (-inv[p][1]) * ginv[1][q];
    for (int p = 0; p < 2; ++p)
      for (int q = 0; q < 2; ++q) dcov[p][q] = tmp[p][0] * inv[0][q] + tmp[p][1] * inv[1][q];
    const float sg_mean[2] = {r[0], r[1]};
    const float sg_op = r[5];
    if (a.splat_grads) {
      float* o = a.splat_grads + i * 10;
      o[0] = r[0]; o[1] = r[1];
      o[2] = dcov[0][0]; o[3] = dcov[0][1]; o[4] = dcov[1][0]; o[5] = dcov[1][1];
      o[6] = r[5]; o[7] = r[6]; o[8] = r[7]; o[9] = r[8];
    }

    // Reconstruct the forward intermediates (backward.hpp:400-410).
    const float p[3] = {a.means[i], a.means[n + i], a.means[2 * n + i]};
    const float qraw[4] = {a.rotations[i], a.rotations[n + i], a.rotations[2 * n + i], a.rotations[3 * n + i]};
    const float ls[3] = {a.log_scales[i], a.log_scales[n + i], a.log_scales[2 * n + i]};
    float mu[3];
    to_camera(a.cam, p, mu);
    const float x = mu[0], y = mu[1], z = mu[2];
    const float W = (float)a.cam.width, H = (float)a.cam.height;
    // The backward is tolerance-checked (not bit-exact): angles from the components, fast
    // exponentials and reciprocals rather than the forward's portable binary64 functions.
    const Angles ang = angles_of(x, y, z);
    omc = 1.0f - ang.ct;
    const bool clamped = (flags & kFlagClamped) != 0;  // the forward's pole-clamp decision
    const M23 J = jacobian_from_angles(ang, W, H, clamped, a.sec_max);
    const float qn = sqrtf(sum4(qraw[0] * qraw[0], qraw[1] * qraw[1], qraw[2] * qraw[2], qraw[3] * qraw[3]));
    const float inv_qn = __frcp_rn(qn);
    const float qq[4] = {qraw[0] * inv_qn, qraw[1] * inv_qn, qraw[2] * inv_qn, qraw[3] * inv_qn};
    const M3 Rq = quaternion_matrix(qq[0], qq[1], qq[2], qq[3]);
    const float sc[3] = {__expf(ls[0]), __expf(ls[1]), __expf(ls[2])};
    M3 m;
    for (int rr = 0; rr < 3; ++rr)
      for (int k = 0; k < 3; ++k) m.a[rr][k] = Rq.a[rr][k] * sc[k];
    const M3 V = mul33_t(m);
    M3 Rc;
    for (int rr = 0; rr < 3; ++rr)
      for (int k = 0; k < 3; ++k) Rc.a[rr][k] = a.cam.R[rr][k];
    const M23 T = mul23_3(J, Rc);

    // grad_T (backward.hpp:42-68)
    const float* s = a.signs;
    const float d11 = dcov[0][0], d22 = dcov[1][1], d12 = dcov[0][1] + dcov[1][0];
    float av[3], bv[3];
    for (int c = 0; c < 3; ++c) {
      av[c] = T.a[0][0] * V.a[c][0] + T.a[0][1] * V.a[c][1] + T.a[0][2] * V.a[c][2];
      bv[c] = T.a[1][0] * V.a[c][0] + T.a[1][1] * V.a[c][1] + T.a[1][2] * V.a[c][2];
    }
    float dT[2][3];
    for (int c = 0; c < 3; ++c) {
      dT[0][c] = s[2 * c] * 2.0f * av[c] * d11 + s[2 * c + 1] * bv[c] * d12;
      dT[1][c] = s[6 + 2 * c] * 2.0f * bv[c] * d22 + s[6 + 2 * c + 1] * av[c] * d12;
    }
    // dl_dj = dl_dt * R^T
    float dJ[2][3];
    for (int rr = 0; rr < 2; ++rr)
      for (int c = 0; c < 3; ++c)
        dJ[rr][c] = dT[rr][0] * Rc.a[c][0] + dT[rr][1] * Rc.a[c][1] + dT[rr][2] * Rc.a[c][2];

    float dmu[3] = {0, 0, 0};
    const float rho2 = ang.rho2;
    if (!(rho2 > 0.0f)) {
      atomic_min_error(&a.err->bwd_domain, i, 3);
    } else {
      const float rho = ang.rho, r2 = ang.r2;
      const float inv_rho2 = __frcp_rn(rho2), inv_r2 = __frcp_rn(r2);
      const float kw0 = W / (2.0f * kPiF), kh0 = H / kPiF;
      if (!clamped) {  // grad_position (backward.hpp:73-105)
        const float inv_r4 = inv_r2 * inv_r2;
        const float inv_rho3 = inv_rho2 * ang.inv_rho;
        const float g11 = dJ[0][0], g13 = dJ[0][2], g21 = dJ[1][0], g22 = dJ[1][1], g23 = dJ[1][2];
        const float xz_over_rho4 = x * z * (inv_rho2 * inv_rho2);
        const float xx_minus_zz = (x * x - z * z) * (inv_rho2 * inv_rho2);
        const float mixed = x * y * z * (2.0f * rho2 + r2) * (inv_r4 * inv_rho3);
        const float straight = (r2 - 2.0f * y * y) * (inv_r4 * ang.inv_rho);
        dmu[0] = -2.0f * kw0 * xz_over_rho4 * g11 + kw0 * xx_minus_zz * g13 -
                 kh0 * y * (z * z * r2 - 2.0f * x * x * rho2) * (inv_r4 * inv_rho3) * g21 - kh0 * x * straight * g22 +
                 kh0 * mixed * g23;
        dmu[1] = -kh0 * x * straight * g21 - 2.0f * kh0 * y * rho * inv_r4 * g22 - kh0 * z * straight * g23;
        dmu[2] = kw0 * xx_minus_zz * g11 + 2.0f * kw0 * xz_over_rho4 * g13 + kh0 * mixed * g21 -
                 kh0 * z * straight * g22 - kh0 * y * (x * x * r2 - 2.0f * z * z * rho2) * (inv_r4 * inv_rho3) * g23;
      } else {  // grad_position_clamped (backward.hpp:111-150)
        const float inv_r = ang.inv_r;
        const float cp = ang.cp, sp = ang.sp, ct = ang.ct, st = ang.st;
        const float kw = W / (2.0f * kPiF) * a.sec_max * inv_r;
        const float kh = H / kPiF * inv_r;
        const float djr[2][3] = {{-kw * cp * inv_r, 0.0f, kw * sp * inv_r},
                                 {-kh * st * sp * inv_r, -kh * ct * inv_r, -kh * st * cp * inv_r}};
        const float djp[2][3] = {{-kw * sp, 0.0f, -kw * cp}, {kh * st * cp, 0.0f, -kh * st * sp}};
        const float djt[2][3] = {{0.0f, 0.0f, 0.0f}, {kh * ct * sp, -kh * st, kh * ct * cp}};
        float cr = 0, cph = 0, cth = 0;
        for (int c = 0; c < 3; ++c)
          for (int rr = 0; rr < 2; ++rr) {
            cr += dJ[rr][c] * djr[rr][c];
            cph += dJ[rr][c] * djp[rr][c];
            cth += dJ[rr][c] * djt[rr][c];
          }
        const float drdt[3] = {x * inv_r, y * inv_r, z * inv_r};
        const float dphidt[3] = {z * inv_rho2, 0.0f, -x * inv_rho2};
        const float k3 = ang.inv_rho * inv_r2;
        const float dthdt[3] = {x * y * k3, -rho * inv_r2, z * y * k3};
        for (int c = 0; c < 3; ++c) dmu[c] = cr * drdt[c] + cph * dphidt[c] + cth * dthdt[c];
      }
      // Mean path: unclamped direct Jacobian (projection.hpp:118-133, backward.hpp:420-423)
      const float k3 = ang.inv_rho * inv_r2;
      const float jd[2][3] = {{kw0 * z * inv_rho2, 0.0f, -kw0 * x * inv_rho2},
                              {-kh0 * x * y * k3, kh0 * rho * inv_r2, -kh0 * y * z * k3}};
      for (int c = 0; c < 3; ++c) dmu[c] += jd[0][c] * sg_mean[0] + jd[1][c] * sg_mean[1];
    }
    // means = R^T dmu
    for (int c = 0; c < 3; ++c) gm[c] = Rc.a[0][c] * dmu[0] + (Rc.a[1][c] * dmu[1] + Rc.a[2][c] * dmu[2]);
    bool sh_finite = true;
    if (a.sh_degree > 0) {  // SH extension: coefficient gradients and the view-direction term
      const int nb = sh_count(a.sh_degree);
      float d[3], Y[15], dY[15][3];
      const float len = sh_direction(a.cam, p, d);
      sh_basis(a.sh_degree, d[0], d[1], d[2], Y);
      sh_basis_grad(a.sh_degree, d[0], d[1], d[2], dY);
      float dd[3] = {0.0f, 0.0f, 0.0f};
      for (int k = 0; k < nb; ++k)
        for (int ch = 0; ch < 3; ++ch) {
          const int64_t idx = (int64_t)(3 * k + ch) * n + i;
          const float g = r[6 + ch] * Y[k];
          sh_finite = sh_finite && isfinite(g);
          if (a.accumulate) a.g_sh_rest[idx] += g;
          else a.g_sh_rest[idx] = g;
          const float w = r[6 + ch] * a.sh_rest[idx];
          for (int q = 0; q < 3; ++q) dd[q] += w * dY[k][q];
        }
      if (len > 0.0f) {
        const float dot = d[0] * dd[0] + d[1] * dd[1] + d[2] * dd[2];
        for (int q = 0; q < 3; ++q) gm[q] += (dd[q] - d[q] * dot) / len;
      }
    }
    pgn = sqrtf(sg_mean[0] * sg_mean[0] + sg_mean[1] * sg_mean[1]);

    // dL/dSigma3D = T^T dcov T; grad_cov3d_params (backward.hpp:156-201)
    float tg[3][2];
    for (int c = 0; c < 3; ++c)
      for (int q = 0; q < 2; ++q) tg[c][q] = T.a[0][c] * dcov[0][q] + T.a[1][c] * dcov[1][q];
    float ds[3][3];
    for (int c = 0; c < 3; ++c)
      for (int d = 0; d < 3; ++d) ds[c][d] = tg[c][0] * T.a[0][d] + tg[c][1] * T.a[1][d];
    float dm[3][3];  // 2 * dSigma * M
    for (int rr = 0; rr < 3; ++rr)
      for (int k = 0; k < 3; ++k)
        dm[rr][k] = 2.0f * (ds[rr][0] * m.a[0][k] + ds[rr][1] * m.a[1][k] + ds[rr][2] * m.a[2][k]);
    float drot[3][3];
    for (int rr = 0; rr < 3; ++rr)
      for (int k = 0; k < 3; ++k) drot[rr][k] = dm[rr][k] * sc[k];
    for (int k = 0; k < 3; ++k)
      gls[k] = (Rq.a[0][k] * dm[0][k] + Rq.a[1][k] * dm[1][k] + Rq.a[2][k] * dm[2][k]) * sc[k];
    const float w = qq[0], qx = qq[1], qy = qq[2], qz = qq[3];
    const float dw[3][3] = {{0, -qz, qy}, {qz, 0, -qx}, {-qy, qx, 0}};
    const float dx[3][3] = {{0, qy, qz}, {qy, -2 * qx, -w}, {qz, w, -2 * qx}};
    const float dy[3][3] = {{-2 * qy, qx, w}, {qx, 0, qz}, {-w, qz, -2 * qy}};
    const float dz[3][3] = {{-2 * qz, -w, qx}, {w, -2 * qz, qy}, {qx, qy, 0}};
    float gu[4] = {0, 0, 0, 0};
    for (int rr = 0; rr < 3; ++rr)
      for (int k = 0; k < 3; ++k) {
        gu[0] += drot[rr][k] * dw[rr][k];
        gu[1] += drot[rr][k] * dx[rr][k];
        gu[2] += drot[rr][k] * dy[rr][k];
        gu[3] += drot[rr][k] * dz[rr][k];
      }
    for (int k = 0; k < 4; ++k) gu[k] *= 2.0f;
    const float qd = (qq[0] * gu[0] + qq[1] * gu[1]) + (qq[2] * gu[2] + qq[3] * gu[3]);
    for (int k = 0; k < 4; ++k) gq[k] = (gu[k] - qq[k] * qd) * inv_qn;

    const float o = ab1.y;
    gop = sg_op * o * (1.0f - o);
    gcol[0] = r[6];
    gcol[1] = r[7];
    gcol[2] = r[8];
    float all[14];
    for (int k = 0; k < 3; ++k) all[k] = gm[k];
    for (int k = 0; k < 4; ++k) all[3 + k] = gq[k];
    for (int k = 0; k < 3; ++k) all[7 + k] = gls[k];
    all[10] = gop;
    for (int k = 0; k < 3; ++k) all[11 + k] = gcol[k];
    if (!all_finite(all, 14) || !sh_finite) atomic_min_error(&a.err->bwd_nonfinite, i, 2);
  }
  if (a.sh_degree > 0 && !(flags & kFlagVisible) && !a.accumulate)
    for (int k = 0; k < 3 * sh_count(a.sh_degree); ++k) a.g_sh_rest[(int64_t)k * n + i] = 0.0f;
  if (a.accumulate) {
    for (int k = 0; k < 3; ++k) a.g_means[k * n + i] += gm[k];
    for (int k = 0; k < 4; ++k) a.g_rotations[k * n + i] += gq[k];
    for (int k = 0; k < 3; ++k) a.g_log_scales[k * n + i] += gls[k];
    a.g_raw_opacities[i] += gop;
    for (int k = 0; k < 3; ++k) a.g_colors[k * n + i] += gcol[k];
    if (a.g_pixel_grad_norm) a.g_pixel_grad_norm[i] += pgn;
    if (a.g_one_minus_cos) a.g_one_minus_cos[i] += omc;
    if (a.g_observed) a.g_observed[i] += observed;
  } else {
    for (int k = 0; k < 3; ++k) a.g_means[k * n + i] = gm[k];
    for (int k = 0; k < 4; ++k) a.g_rotations[k * n + i] = gq[k];
    for (int k = 0; k < 3; ++k) a.g_log_scales[k * n + i] = gls[k];
    a.g_raw_opacities[i] = gop;
    for (int k = 0; k < 3; ++k) a.g_colors[k * n + i] = gcol[k];
    if (a.g_pixel_grad_norm) a.g_pixel_grad_norm[i] = pgn;
    if (a.g_one_minus_cos) a.g_one_minus_cos[i] = omc;
    if (a.g_observed) a.g_observed[i] = observed;
  }
}

// ------------------------------------------------------------------ SplatGrads only
// grad_pixels_to_splats (backward.hpp:208-339) without the per-splat chain rule: the
// folded records of each projected Gaussian and the Sigma_2D transport, into
// splat_grads[i][10] (mean 2, cov2d 4 full-matrix convention, opacity, colour 3).
__global__ void k_splat_grads(int64_t n, const float4* __restrict__ sp_ab, const float4* __restrict__ sp_c,
                              const uint32_t* __restrict__ cnt, const float* __restrict__ folded,
                              float* __restrict__ splat_grads) {
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float r[kRec] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  const uint32_t flags = __float_as_uint(sp_c[i].w);
  if ((flags & kFlagVisible) && cnt[i] > 0)
#pragma unroll
    for (int c = 0; c < kRec; ++c) r[c] = folded[i * kRec + c];
  const float4 ab0 = sp_ab[2 * i], ab1 = sp_ab[2 * i + 1];
  const float inv[2][2] = {{ab0.z, ab0.w}, {ab0.w, ab1.x}};
  const float ginv[2][2] = {{r[2], r[3]}, {r[3], r[4]}};
  float tmp[2][2], dcov[2][2];
  for (int p = 0; p < 2; ++p)
    for (int q = 0; q < 2; ++q) tmp[p][q] = (-inv[p][0]) * ginv[0][q] + (-inv[p][1]) * ginv[1][q];
  for (int p = 0; p < 2; ++p)
    for (int q = 0; q < 2; ++q) dcov[p][q] = tmp[p][0] * inv[0][q] + tmp[p][1] * inv[1][q];
  float* o = splat_grads + i * 10;
  o[0] = r[0]; o[1] = r[1];
  o[2] = dcov[0][0]; o[3] = dcov[0][1]; o[4] = dcov[1][0]; o[5] = dcov[1][1];
  o[6] = r[5]; o[7] = r[6]; o[8] = r[7]; o[9] = r[8];
}

void launch_splat_grads(int64_t n, const float4* sp_ab, const float4* sp_c, const uint32_t* cnt, const float* folded,
                        float* splat_grads, cudaStream_t stream) {
  if (n == 0) return;
  launch_pdl(k_splat_grads, (unsigned)((n + 255) / 256), 256, 0, stream, n, sp_ab, sp_c, cnt, folded, splat_grads);
  ++g_launches;
}

// ------------------------------------------------------------------ ordered fold
// Per-Gaussian sum of its entry records (backward.hpp:310-327); a Gaussian's records are
// contiguous in emit order ([off_sorted[r], +cnt_sorted[r]) for depth rank r). A warp owns
// 32 consecutive ranks. Ranks with at most kFoldSmall records are summed by their own
// lane, in record order; larger ranks (pole and seam splats, up to thousands of tiles)
// are summed by the whole warp — lane l takes records l, l + 32, ... (coalesced 48-byte
// records), then a fixed xor tree — so one long list no longer serialises its warp.
// Records no warp wrote (touched == 0) are zero and skipped. Deterministic: every sum has
// a fixed order.
constexpr int kFoldWarps = 8;
constexpr uint32_t kFoldSmall = 16;

__device__ __forceinline__ void fold_add(const float* __restrict__ rec, float acc[kRec]) {
#pragma unroll
  for (int c = 0; c < kRec; ++c) acc[c] += __ldcs(rec + c);
}

__global__ void __launch_bounds__(kFoldWarps * 32) k_fold_records(
    int64_t n, const uint32_t* __restrict__ sorted_idx, const uint32_t* __restrict__ cnt_sorted,
    const uint32_t* __restrict__ off_sorted, const uint8_t* __restrict__ touched, const float* __restrict__ records,
    float* __restrict__ folded, const uint32_t* __restrict__ n_dev, const unsigned long long* __restrict__ k_limit) {
  pdl_wait();
  if (n_dev) n = min(n, (int64_t)*n_dev);  // a band's ranks counted on the device
  const uint32_t kmax = k_limit ? (uint32_t)min(*k_limit, 0xFFFFFFFFull) : 0xFFFFFFFFu;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r0 = ((int64_t)blockIdx.x * kFoldWarps + warp) * 32;
  if (r0 >= n) return;
  const int64_t r = r0 + lane;
  const uint32_t cnt = r < n ? cnt_sorted[r] : 0u;
  const uint32_t off = r < n ? off_sorted[r] : 0u;
  const uint32_t g = r < n ? sorted_idx[r] : 0u;
  // small ranks: the lane's own records, in order, four in flight at a time
  if (cnt > 0 && cnt <= kFoldSmall) {
    float acc[kRec] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    const uint32_t end = min(off + cnt, max(off, kmax));
    for (uint32_t e = off; e < end; e += 4) {
      float v[4][kRec];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const bool live = e + u < end && touched[e + u];
        if (live) load_record(records + (int64_t)(e + u) * kRecStride, v[u]);
        else
#pragma unroll
          for (int c = 0; c < kRec; ++c) v[u][c] = 0.0f;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int c = 0; c < kRec; ++c) acc[c] += v[u][c];
    }
    float* o = folded + (int64_t)g * kRec;
#pragma unroll
    for (int c = 0; c < kRec; ++c) o[c] = acc[c];
  }
  // large ranks: one at a time with the whole warp
  uint32_t big = __ballot_sync(0xffffffffu, cnt > kFoldSmall);
  while (big) {
    const int src = __ffs(big) - 1;
    big &= big - 1;
    const uint32_t boff = __shfl_sync(0xffffffffu, off, src);
    const uint32_t bcnt = min(__shfl_sync(0xffffffffu, cnt, src), boff < kmax ? kmax - boff : 0u);
    const uint32_t bg = __shfl_sync(0xffffffffu, g, src);
    float acc[kRec] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (uint32_t k0 = lane; k0 < bcnt; k0 += 4 * 32) {  // four records in flight per lane
      float v[4][kRec];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t k = k0 + 32 * u;
        const bool live = k < bcnt && touched[boff + k];
        if (live) load_record(records + (int64_t)(boff + k) * kRecStride, v[u]);
        else
#pragma unroll
          for (int c = 0; c < kRec; ++c) v[u][c] = 0.0f;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int c = 0; c < kRec; ++c) acc[c] += v[u][c];
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1)
#pragma unroll
      for (int c = 0; c < kRec; ++c) acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], d);
    if (lane < kRec) {
      float v = 0.0f;
#pragma unroll
      for (int c = 0; c < kRec; ++c) v = lane == c ? acc[c] : v;
      folded[(int64_t)bg * kRec + lane] = v;
    }
  }
}

void launch_fold_records(int64_t n, const uint32_t* sorted_idx, const uint32_t* cnt_sorted,
                         const uint32_t* off_sorted, const uint8_t* touched, const float* records, float* folded,
                         cudaStream_t stream, const uint32_t* n_dev, const unsigned long long* k_limit) {
  if (n == 0) return;
  const int64_t warps = (n + 31) / 32;
  launch_pdl(k_fold_records, (unsigned)((warps + kFoldWarps - 1) / kFoldWarps), kFoldWarps * 32, 0, stream, n,
             sorted_idx, cnt_sorted, off_sorted, touched, records, folded, n_dev, k_limit);
  ++g_launches;
}

void launch_bwd_splat(const BwdSplatArgs& a, cudaStream_t stream) {
  if (a.n == 0) return;
  launch_pdl(k_bwd_splat, (unsigned)((a.n + 255) / 256), 256, 0, stream, a);
  ++g_launches;
}

}  // namespace odgs_b200
