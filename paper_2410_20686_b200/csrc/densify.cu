// densify.cu — adaptive density control on the device:
// densify_and_prune (reference proj/include/odgs/densify.hpp:81-153) and reset_opacity
// (:158-166).
//
// densify_and_prune is a stream compaction. The reference appends clones / split
// children in parent order and then keeps rows in index order, so the output is
//   [ surviving original rows, in order | surviving added rows, in parent order ].
// Every decision is local to one Gaussian (class: none / clone / split, and whether
// its opacity is under the prune floor — children inherit the parent's raw opacity,
// so they are pruned together with it), so one classify pass and three exclusive
// scans give every row its output position:
//   A = survives in place (not split, not pruned)   -> dst A-offset
//   B = surviving added rows (0, 1 clone, 2 children) -> dst total(A) + B-offset
//   C = is split                                     -> index into the host-drawn
//                                                       unit-ball samples
// The split offsets come from the reference's sequential mt19937 + normal rejection
// stream (densify.hpp:61-69); the host replays it (capi.cu) for the C-th split and
// uploads the samples, the apply kernel does the rest.
#include "kernels.h"

namespace odgs_b200 {

namespace {

__device__ __forceinline__ float sigmoid_dev(float x) {  // types.hpp:29-31
  return 1.0f / (1.0f + pm_expf(-x));
}

// densify.hpp:100-127 decision for row i: 0 none, 1 clone, 2 split.
__device__ __forceinline__ int densify_class(const DensifyArgs& a, int64_t i) {
  const int32_t c = a.grad_count[i];
  if (c <= 0) return 0;
  const float count = (float)c;
  const float mean_grad = a.grad_accum[i] / count;
  const float mean_omc = a.elev_accum[i] / count;
  const float threshold = a.tmin + mean_omc * (a.tmax - a.tmin);
  if (mean_grad < threshold) return 0;
  const int64_t n = a.n;
  const float s0 = pm_expf(a.log_scales[i]), s1 = pm_expf(a.log_scales[n + i]), s2 = pm_expf(a.log_scales[2 * n + i]);
  // Eigen maxCoeff: max(s0, max(s1, s2)) with max(x, y) = x < y ? y : x.
  const float m12 = s1 < s2 ? s2 : s1;
  const float max_scale = s0 < m12 ? m12 : s0;
  return max_scale < a.size_split ? 1 : 2;
}

__global__ void __launch_bounds__(256) k_densify_classify(DensifyArgs a) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned cloned = 0, split = 0, pruned = 0;
  if (i < a.n) {
    const int cls = densify_class(a, i);
    const bool low = sigmoid_dev(a.raw_opacities[i]) < a.prune_floor;  // densify.hpp:141
    const uint32_t added = cls == 1 ? 1u : cls == 2 ? 2u : 0u;
    a.keep_self[i] = (cls != 2 && !low) ? 1u : 0u;
    a.added_kept[i] = low ? 0u : added;
    a.split_flag[i] = cls == 2 ? 1u : 0u;
    cloned = cls == 1;
    split = cls == 2;
    pruned = ((cls != 2 && low) ? 1u : 0u) + (low ? added : 0u);
    if (cls == 2) {  // normalize_quaternion (covariance.hpp:13-18) of the split parent
      const int64_t n = a.n;
      const float q0 = a.rotations[i], q1 = a.rotations[n + i], q2 = a.rotations[2 * n + i],
                  q3 = a.rotations[3 * n + i];
      const float qn = sqrtf(sum4(q0 * q0, q1 * q1, q2 * q2, q3 * q3));
      if (!(qn > 1e-12f)) atomicMin(a.bad_quaternion, (unsigned long long)i);
    }
  }
  cloned = __reduce_add_sync(0xffffffffu, cloned);
  split = __reduce_add_sync(0xffffffffu, split);
  pruned = __reduce_add_sync(0xffffffffu, pruned);
  if ((threadIdx.x & 31) == 0) {
    if (cloned) atomicAdd(&a.counters[0], (unsigned long long)cloned);
    if (split) atomicAdd(&a.counters[1], (unsigned long long)split);
    if (pruned) atomicAdd(&a.counters[2], (unsigned long long)pruned);
  }
}

__device__ __forceinline__ void copy_params(const DensifyApplyArgs& a, int64_t i, int64_t d) {
  const int64_t n = a.n, m = a.m;
  for (int c = 0; c < 3; ++c) a.out_means[c * m + d] = a.means[c * n + i];
  for (int c = 0; c < 4; ++c) a.out_rotations[c * m + d] = a.rotations[c * n + i];
  for (int c = 0; c < 3; ++c) a.out_log_scales[c * m + d] = a.log_scales[c * n + i];
  a.out_raw_opacities[d] = a.raw_opacities[i];
  for (int c = 0; c < 3; ++c) a.out_colors[c * m + d] = a.colors[c * n + i];
}

__device__ __forceinline__ void move_moments(const DensifyApplyArgs& a, int64_t i, int64_t d) {
  const int64_t n = a.n, m = a.m;
#pragma unroll
  for (int k = 0; k < 10; ++k)
    for (int c = 0; c < moment_width(k); ++c) a.out_moments[k][c * m + d] = a.moments[k][c * n + i];
}

__device__ __forceinline__ void zero_moments(const DensifyApplyArgs& a, int64_t d) {
  const int64_t m = a.m;
#pragma unroll
  for (int k = 0; k < 10; ++k)
    for (int c = 0; c < moment_width(k); ++c) a.out_moments[k][c * m + d] = 0.0f;
}

__global__ void __launch_bounds__(256) k_densify_apply(DensifyApplyArgs a) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  if (a.keep_self[i]) {
    const int64_t d = a.off_a[i];
    copy_params(a, i, d);
    move_moments(a, i, d);
  }
  const uint32_t added = a.added_kept[i];
  if (added == 0) return;
  const int64_t base = (int64_t)a.total_a + a.off_b[i];
  if (!a.split_flag[i]) {  // clone: append_row copy (densify.hpp:109-111)
    copy_params(a, i, base);
    zero_moments(a, base);
    return;
  }
  // split (densify.hpp:112-126): children at parent + R (s ⊙ e), log-scales shrunk.
  const int64_t n = a.n, m = a.m;
  const float q0 = a.rotations[i], q1 = a.rotations[n + i], q2 = a.rotations[2 * n + i], q3 = a.rotations[3 * n + i];
  const float qn = sqrtf(sum4(q0 * q0, q1 * q1, q2 * q2, q3 * q3));
  const M3 R = quaternion_matrix(q0 / qn, q1 / qn, q2 / qn, q3 / qn);
  const float s[3] = {pm_expf(a.log_scales[i]), pm_expf(a.log_scales[n + i]), pm_expf(a.log_scales[2 * n + i])};
  const int64_t j = a.off_c[i];
  for (int child = 0; child < 2; ++child) {
    const int64_t d = base + child;
    copy_params(a, i, d);
    const float* e = a.unit_ball + (2 * j + child) * 3;
    const float v[3] = {s[0] * e[0], s[1] * e[1], s[2] * e[2]};
    for (int r = 0; r < 3; ++r) {
      const float off = sum3(R.a[r][0] * v[0], R.a[r][1] * v[1], R.a[r][2] * v[2]);
      a.out_means[r * m + d] = a.means[r * n + i] + off;
      a.out_log_scales[r * m + d] = a.log_scales[r * n + i] - a.log_shrink;
    }
    zero_moments(a, d);
  }
}

// reset_opacity, pass 1: the first row whose logit argument leaves (0, 1) (the
// reference throws there, types.hpp:36-37, after rewriting the rows before it).
__global__ void __launch_bounds__(256) k_reset_opacity_check(const float* raw, int64_t n, float ceiling,
                                                              unsigned long long* bad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float o = sigmoid_dev(raw[i]);
  const float x = ceiling < o ? ceiling : o;  // std::min(o, ceiling)
  if (!(x > 0.0f && x < 1.0f)) atomicMin(bad, (unsigned long long)i);
}

// Pass 2: rows before the failing one (all rows when none fails).
__global__ void __launch_bounds__(256) k_reset_opacity(float* raw, int64_t n, float ceiling,
                                                        const unsigned long long* bad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || (unsigned long long)i >= *bad) return;
  const float o = sigmoid_dev(raw[i]);
  const float x = ceiling < o ? ceiling : o;
  raw[i] = pm_logf(x / (1.0f - x));  // logit (types.hpp:35-39)
}

unsigned grid_for(int64_t n) { return (unsigned)((n + 255) / 256); }

}  // namespace

void launch_densify_classify(const DensifyArgs& a, cudaStream_t stream) {
  if (a.n == 0) return;
  k_densify_classify<<<grid_for(a.n), 256, 0, stream>>>(a);
  ++g_launches;
}

void launch_densify_apply(const DensifyApplyArgs& a, cudaStream_t stream) {
  if (a.n == 0) return;
  k_densify_apply<<<grid_for(a.n), 256, 0, stream>>>(a);
  ++g_launches;
}

void launch_reset_opacity(float* raw, int64_t n, float ceiling, unsigned long long* bad, cudaStream_t stream) {
  if (n == 0) return;
  k_reset_opacity_check<<<grid_for(n), 256, 0, stream>>>(raw, n, ceiling, bad);
  k_reset_opacity<<<grid_for(n), 256, 0, stream>>>(raw, n, ceiling, bad);
  g_launches += 2;
}

}  // namespace odgs_b200
