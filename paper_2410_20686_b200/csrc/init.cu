// init.cu — init_from_points on the GPU (reference io.cpp:259-297).
//
// The reference sets every initial Gaussian's isotropic scale from the mean distance
// to its (up to) three nearest neighbours, by an O(N^2) brute-force scan. Here the
// same exact 3-NN is found through a uniform grid:
//
//   k_bbox_partial  per-block min/max of the finite positions (+ finite count)
//   k_cell_keys     cell id per point (non-finite points get key n_cells and
//                   sort last: no distance to or from them is finite, io.cpp:273-287)
//   radix sort      (cell, index) pairs, stable
//   k_gather_xyz    positions in cell order (SoA, binary64)
//   k_cell_ranges   CSR start of every cell
//   k_knn_query     one thread per point: shells of cells around its own, keeping
//                   the three smallest squared distances, until the third is closer
//                   than anything outside the searched cube; then the reference's
//                   ascending sum of square roots, mean, 1e-7 floor / 0.1 fallback
//                   and log (io.cpp:283-295).
//
// Distances are binary64 with the reference's operation order (p_j - p_i, then
// Eigen's squaredNorm unroller x^2 + (y^2 + z^2)), so the kept multiset of distances
// — and with it the mean — is bit-identical to the brute force.
#include <cfloat>

#include "common.cuh"
#include "kernels.h"

namespace odgs_b200 {

constexpr int kInitThreads = 256;

__global__ void __launch_bounds__(kInitThreads) k_bbox_partial(int64_t n, const double* __restrict__ pos,
                                                               double* __restrict__ partial,
                                                               unsigned long long* __restrict__ n_finite) {
  __shared__ double s_v[6][kInitThreads / 32];
  double lo[3] = {DBL_MAX, DBL_MAX, DBL_MAX}, hi[3] = {-DBL_MAX, -DBL_MAX, -DBL_MAX};
  uint32_t cnt = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double x = pos[i], y = pos[n + i], z = pos[2 * n + i];
    if (!(isfinite(x) && isfinite(y) && isfinite(z))) continue;
    ++cnt;
    lo[0] = fmin(lo[0], x); hi[0] = fmax(hi[0], x);
    lo[1] = fmin(lo[1], y); hi[1] = fmax(hi[1], y);
    lo[2] = fmin(lo[2], z); hi[2] = fmax(hi[2], z);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int d = 16; d > 0; d >>= 1)
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      lo[a] = fmin(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], d));
      hi[a] = fmax(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], d));
    }
  cnt = __reduce_add_sync(0xffffffffu, cnt);
  if (lane == 0) {
    for (int a = 0; a < 3; ++a) {
      s_v[a][warp] = lo[a];
      s_v[3 + a][warp] = hi[a];
    }
    if (cnt) atomicAdd(n_finite, (unsigned long long)cnt);
  }
  __syncthreads();
  if (threadIdx.x < 6) {
    const int a = threadIdx.x;
    double v = s_v[a][0];
    for (int w = 1; w < kInitThreads / 32; ++w) v = a < 3 ? fmin(v, s_v[a][w]) : fmax(v, s_v[a][w]);
    partial[blockIdx.x * 6 + a] = v;
  }
}

__device__ __forceinline__ int cell_coord(double p, double lo, double h, int dim) {
  const double f = floor((p - lo) / h);
  return f <= 0.0 ? 0 : (f >= (double)(dim - 1) ? dim - 1 : (int)f);
}

__global__ void k_cell_keys(int64_t n, const double* __restrict__ pos, KnnGrid g, uint32_t* __restrict__ keys,
                            uint32_t* __restrict__ idx) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double x = pos[i], y = pos[n + i], z = pos[2 * n + i];
  uint32_t key = g.n_cells;  // non-finite: one past the last cell, sorts last
  if (isfinite(x) && isfinite(y) && isfinite(z)) {
    const int cx = cell_coord(x, g.lo[0], g.h, g.dims[0]);
    const int cy = cell_coord(y, g.lo[1], g.h, g.dims[1]);
    const int cz = cell_coord(z, g.lo[2], g.h, g.dims[2]);
    key = ((uint32_t)cz * (uint32_t)g.dims[1] + (uint32_t)cy) * (uint32_t)g.dims[0] + (uint32_t)cx;
  }
  keys[i] = key;
  idx[i] = (uint32_t)i;
}

__global__ void k_gather_xyz(int64_t n, const uint32_t* __restrict__ idx, const double* __restrict__ pos,
                             double* __restrict__ sorted) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const uint32_t i = idx[k];
  sorted[k] = pos[i];
  sorted[n + k] = pos[n + i];
  sorted[2 * n + k] = pos[2 * n + i];
}

// cell_start[c] = first sorted position with key >= c, for c in [0, n_cells].
__global__ void k_cell_ranges(int64_t m, const uint32_t* __restrict__ keys, uint32_t n_cells,
                              uint32_t* __restrict__ cell_start) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e > m) return;
  const uint32_t prev = e == 0 ? 0u : keys[e - 1] + 1u;
  const uint32_t cur = e == m ? n_cells : keys[e];
  if (e != 0 && e != m && keys[e - 1] == cur) return;
  for (uint32_t c = prev; c <= cur; ++c) cell_start[c] = (uint32_t)e;
}

__device__ __forceinline__ void insert3(double d2, double best[3]) {
  if (d2 < best[2]) {  // io.cpp:276-279: replace the largest, keep ascending
    best[2] = d2;
    if (best[2] < best[1]) {
      const double t = best[1]; best[1] = best[2]; best[2] = t;
      if (best[1] < best[0]) {
        const double u = best[0]; best[0] = best[1]; best[1] = u;
      }
    }
  }
}

__global__ void __launch_bounds__(kInitThreads) k_knn_query(
    int64_t n, int64_t m, const double* __restrict__ xyz, const uint32_t* __restrict__ idx,
    const uint32_t* __restrict__ cell_start, KnnGrid g, double* __restrict__ scale_out,
    double* __restrict__ log_scales) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const uint32_t self = idx[k];
  double best[3] = {INFINITY, INFINITY, INFINITY};
  if (k < m) {  // finite point: search the grid
    const double p[3] = {xyz[k], xyz[n + k], xyz[2 * n + k]};
    int c[3];
    for (int a = 0; a < 3; ++a) c[a] = cell_coord(p[a], g.lo[a], g.h, g.dims[a]);
    const int max_r = max(max(g.dims[0], g.dims[1]), g.dims[2]);
    for (int r = 0; r <= max_r; ++r) {
      const int z0 = max(c[2] - r, 0), z1 = min(c[2] + r, g.dims[2] - 1);
      const int y0 = max(c[1] - r, 0), y1 = min(c[1] + r, g.dims[1] - 1);
      const int x0 = max(c[0] - r, 0), x1 = min(c[0] + r, g.dims[0] - 1);
      for (int cz = z0; cz <= z1; ++cz)
        for (int cy = y0; cy <= y1; ++cy) {
          const bool face = abs(cz - c[2]) == r || abs(cy - c[1]) == r;
          for (int cx = x0; cx <= x1; ++cx) {
            if (!face && abs(cx - c[0]) != r) {  // interior of the shell: jump to its far side
              if (cx < c[0] + r) cx = c[0] + r - 1;
              continue;
            }
            const uint32_t cell = ((uint32_t)cz * (uint32_t)g.dims[1] + (uint32_t)cy) * (uint32_t)g.dims[0] +
                                  (uint32_t)cx;
            const uint32_t b = cell_start[cell], e = cell_start[cell + 1];
            for (uint32_t q = b; q < e; ++q) {
              if (idx[q] == self) continue;
              const double dx = xyz[q] - p[0], dy = xyz[n + q] - p[1], dz = xyz[2 * n + q] - p[2];
              const double d2 = __dadd_rn(__dmul_rn(dx, dx), __dadd_rn(__dmul_rn(dy, dy), __dmul_rn(dz, dz)));
              insert3(d2, best);
            }
          }
        }
      // Everything not yet scanned lies outside the cube of cells [c - r, c + r];
      // its distance is at least the gap from p to the cube's inner faces (a face on
      // the grid boundary has nothing beyond it).
      double gap = INFINITY;
      bool covered = true;
      for (int a = 0; a < 3; ++a) {
        if (c[a] - r > 0) {
          gap = fmin(gap, p[a] - (g.lo[a] + (double)(c[a] - r) * g.h));
          covered = false;
        }
        if (c[a] + r < g.dims[a] - 1) {
          gap = fmin(gap, (g.lo[a] + (double)(c[a] + r + 1) * g.h) - p[a]);
          covered = false;
        }
      }
      if (covered) break;
      const double safe = gap * (1.0 - 1e-9);  // margin for the rounded cell boundaries
      if (safe > 0.0 && best[2] < safe * safe) break;
    }
  }
  // io.cpp:283-295
  double sum = 0.0;
  int count = 0;
  for (int q = 0; q < 3; ++q)
    if (isfinite(best[q])) {
      sum += sqrt(best[q]);
      ++count;
    }
  const double scale = count > 0 ? fmax(sum / (double)count, 1e-7) : 0.1;
  const double ls = log(scale);
  if (scale_out) scale_out[self] = scale;
  log_scales[self] = ls;
  log_scales[n + self] = ls;
  log_scales[2 * n + self] = ls;
}

__global__ void k_fill_f64(double* __restrict__ p, int64_t n, double v) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

void launch_fill_f64(double* p, int64_t n, double v, cudaStream_t stream) {
  if (n == 0) return;
  k_fill_f64<<<(unsigned)((n + kInitThreads - 1) / kInitThreads), kInitThreads, 0, stream>>>(p, n, v);
  ++g_launches;
}

void launch_bbox_partial(int64_t n, const double* pos, double* partial, int blocks, unsigned long long* n_finite,
                         cudaStream_t stream) {
  k_bbox_partial<<<blocks, kInitThreads, 0, stream>>>(n, pos, partial, n_finite);
  ++g_launches;
}

void launch_cell_keys(int64_t n, const double* pos, const KnnGrid& g, uint32_t* keys, uint32_t* idx,
                      cudaStream_t stream) {
  if (n == 0) return;
  k_cell_keys<<<(unsigned)((n + kInitThreads - 1) / kInitThreads), kInitThreads, 0, stream>>>(n, pos, g, keys, idx);
  ++g_launches;
}

void launch_gather_xyz(int64_t n, const uint32_t* idx, const double* pos, double* sorted, cudaStream_t stream) {
  if (n == 0) return;
  k_gather_xyz<<<(unsigned)((n + kInitThreads - 1) / kInitThreads), kInitThreads, 0, stream>>>(n, idx, pos, sorted);
  ++g_launches;
}

void launch_cell_ranges(int64_t m, const uint32_t* keys, uint32_t n_cells, uint32_t* cell_start,
                        cudaStream_t stream) {
  const int64_t threads = m + 1;
  k_cell_ranges<<<(unsigned)((threads + kInitThreads - 1) / kInitThreads), kInitThreads, 0, stream>>>(
      m, keys, n_cells, cell_start);
  ++g_launches;
}

void launch_knn_query(int64_t n, int64_t m, const double* xyz, const uint32_t* idx, const uint32_t* cell_start,
                      const KnnGrid& g, double* scale_out, double* log_scales, cudaStream_t stream) {
  if (n == 0) return;
  k_knn_query<<<(unsigned)((n + kInitThreads - 1) / kInitThreads), kInitThreads, 0, stream>>>(
      n, m, xyz, idx, cell_start, g, scale_out, log_scales);
  ++g_launches;
}

}  // namespace odgs_b200
