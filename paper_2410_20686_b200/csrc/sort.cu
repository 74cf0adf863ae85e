// sort.cu — device-wide exclusive scan and stable LSD radix sort of (u32 key, u32 value)
// pairs, hand-written for sm_100a (no CUB).
//
// Used twice per frame:
//   * depth sort of the N projected Gaussians (key = float bits of ||mu_cam||, value =
//     cloud index) — stability gives the reference's (depth, index) tie-break;
//   * tile sort of the K tile entries emitted in (depth, index, shift) order (key =
//     tile id, ceil(log2 T) bits) — stability keeps that order inside every tile, so
//     the per-tile lists equal the reference's (rasterizer.hpp:158-205).
//
// Onesweep LSD radix sort: one kernel histograms all passes' digits, then one kernel
// per pass ranks a tile (4096 items for depth sorts, 6144 for tile-entry sorts) with
// warp-level ballot matching (stable), publishes its digit counts, scatters through
// shared memory, finds its global offsets by decoupled look-back, and writes runs per
// digit. 16 B of traffic per item per pass (+4 B once). Every kernel is launched with
// programmatic dependent launch (launch_pdl); the tile shapes and the look-back window
// are compile-time knobs (ODGS_SORT_*) for A/B builds, defaults measured on the B200.
#include <algorithm>
#include <atomic>

#include "kernels.h"

namespace odgs_b200 {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kIPT = 16;
constexpr int kTile = kThreads * kIPT;  // 4096
constexpr int kWarpItems = 32 * kIPT;   // 512
#ifndef ODGS_SORT_BIG_THREADS
#define ODGS_SORT_BIG_THREADS 384
#endif
#ifndef ODGS_SORT_BIG_MINB
#define ODGS_SORT_BIG_MINB 2
#endif
#ifndef ODGS_SORT_BIG_IPT
#define ODGS_SORT_BIG_IPT 16
#endif
constexpr int kBigThreads = ODGS_SORT_BIG_THREADS;  // tile-entry sorts (n > 2^22)
constexpr int kBigMinBlocks = ODGS_SORT_BIG_MINB;
constexpr int kBigIPT = ODGS_SORT_BIG_IPT;
#ifndef ODGS_SORT_SMALL_IPT
#define ODGS_SORT_SMALL_IPT 16
#endif
#ifndef ODGS_SORT_SMALL_MINB
#define ODGS_SORT_SMALL_MINB 3
#endif
constexpr int kSmallIPT = ODGS_SORT_SMALL_IPT;  // depth sorts (n <= 2^22), 256 threads
constexpr int kSmallMinBlocks = ODGS_SORT_SMALL_MINB;
constexpr int64_t kBigSort = (int64_t)1 << 22;  // n above this: the tile-entry sort shape

// Onesweep tiles of a sort of n pairs.
int64_t pass_tiles(int64_t n) {
  const int64_t t = n > kBigSort ? kBigThreads * kBigIPT : kThreads * kSmallIPT;
  return (n + t - 1) / t;
}

__device__ __forceinline__ uint32_t warp_inclusive_scan(uint32_t v, int lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, v, d);
    if (lane >= d) v += u;
  }
  return v;
}

__device__ __forceinline__ uint32_t warp_reduce(uint32_t v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
  return v;
}

// ------------------------------------------------------------------ scan
__global__ void __launch_bounds__(kThreads) k_scan_reduce(const uint32_t* __restrict__ in, int64_t n,
                                                          uint32_t* __restrict__ block_sums,
                                                          unsigned long long* total64, const uint32_t* n_dev) {
  pdl_wait();
  if (n_dev) n = min(n, (int64_t)*n_dev);  // device-side item count (capacity-sized launch)
  __shared__ uint32_t s_warp[kWarps];
  const int64_t base = (int64_t)blockIdx.x * kTile;
  uint32_t sum = 0;
  for (int k = threadIdx.x; k < kTile; k += kThreads) {
    const int64_t idx = base + k;
    if (idx < n) sum += in[idx];
  }
  sum = warp_reduce(sum);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) s_warp[warp] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    unsigned long long t64 = 0;
    for (int w = 0; w < kWarps; ++w) {
      t += s_warp[w];
      t64 += s_warp[w];
    }
    block_sums[blockIdx.x] = t;
    if (total64) atomicAdd(total64, t64);
  }
}

// Scans one tile per block; block_offsets may be null (single block: adds the total).
__global__ void __launch_bounds__(kThreads) k_scan_downsweep(const uint32_t* __restrict__ in,
                                                             uint32_t* __restrict__ out, int64_t n,
                                                             const uint32_t* __restrict__ block_offsets,
                                                             unsigned long long* total64, const uint32_t* n_dev) {
  pdl_wait();
  if (n_dev) n = min(n, (int64_t)*n_dev);
  __shared__ uint32_t s_warp[kWarps];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t base = (int64_t)blockIdx.x * kTile + (int64_t)warp * kWarpItems;
  uint32_t v[kIPT];
  uint32_t wsum = 0;
#pragma unroll
  for (int j = 0; j < kIPT; ++j) {
    const int64_t idx = base + j * 32 + lane;
    v[j] = idx < n ? in[idx] : 0u;
    wsum += v[j];
  }
  wsum = warp_reduce(wsum);
  if (lane == 0) s_warp[warp] = wsum;
  __syncthreads();
  uint32_t carry = block_offsets ? block_offsets[blockIdx.x] : 0u;
  for (int w = 0; w < warp; ++w) carry += s_warp[w];
  if (!block_offsets && total64 && threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < kWarps; ++w) t += s_warp[w];
    atomicAdd(total64, t);
  }
#pragma unroll
  for (int j = 0; j < kIPT; ++j) {
    const uint32_t incl = warp_inclusive_scan(v[j], lane);
    const int64_t idx = base + j * 32 + lane;
    if (idx < n) out[idx] = carry + incl - v[j];
    carry += __shfl_sync(0xffffffffu, incl, 31);
  }
}

// ------------------------------------------------------------------ onesweep (one kernel per pass)
// Merrill & Adinets' single-pass LSD scheme: one kernel histograms every pass's
// digits up front; each pass is then a single kernel in which a CTA claims the next
// tile id (atomic counter, so every predecessor is already resident), ranks its
// items, publishes its per-digit counts, and derives its per-digit global offsets by
// decoupled look-back over the predecessors' status words (flag in the top 2 bits:
// 1 = tile aggregate, 2 = inclusive prefix). Status words alternate between two
// buffers: the histogram kernel clears the first pass's, each pass the next one's.
constexpr uint32_t kStatAgg = 1u << 30;
constexpr uint32_t kStatPrefix = 2u << 30;
constexpr uint32_t kStatMask = (1u << 30) - 1u;
constexpr int kMaxPasses = 4;
#ifndef ODGS_SORT_LOOK_WINDOW
#define ODGS_SORT_LOOK_WINDOW 8
#endif
constexpr int kLookWindow = ODGS_SORT_LOOK_WINDOW;

struct PassPlan {
  int n_passes;
  int shift[kMaxPasses];
  int bits[kMaxPasses];
};

__global__ void __launch_bounds__(kThreads) k_onesweep_hist(const uint32_t* __restrict__ keys, int64_t n,
                                                            PassPlan plan, uint32_t* __restrict__ hist,
                                                            uint32_t* __restrict__ status0, int64_t n_status,
                                                            const uint32_t* n_dev) {
  pdl_wait();
  if (n_dev) n = min(n, (int64_t)*n_dev);  // device-side item count (capacity-sized launch)
  // Also clears the first pass's status words (each pass clears the next one's).
  for (int64_t k = (int64_t)blockIdx.x * kThreads + threadIdx.x; k < n_status; k += (int64_t)gridDim.x * kThreads)
    status0[k] = 0;
  __shared__ uint32_t s_cnt[kMaxPasses][256];
  for (int k = threadIdx.x; k < kMaxPasses * 256; k += kThreads) (&s_cnt[0][0])[k] = 0;
  __syncthreads();
  // Four consecutive keys per thread and step (one 16-byte load, two in flight), each
  // pass's digits merged into runs before the shared adds: consecutive tile entries of
  // one Gaussian share their tile row, and the high depth digits few values.
  const bool aligned = (reinterpret_cast<uintptr_t>(keys) & 15u) == 0;
  const int64_t n4 = aligned ? n >> 2 : 0;
  const uint4* keys4 = reinterpret_cast<const uint4*>(keys);
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  auto count4 = [&](const uint4 q) {
#pragma unroll
    for (int p = 0; p < kMaxPasses; ++p) {
      if (p < plan.n_passes) {
        const uint32_t m = (1u << plan.bits[p]) - 1u;
        const int sh = plan.shift[p];
        const uint32_t d0 = (q.x >> sh) & m, d1 = (q.y >> sh) & m, d2 = (q.z >> sh) & m, d3 = (q.w >> sh) & m;
        uint32_t cur = d0, c = 1;
        if (d1 == cur) ++c; else { atomicAdd(&s_cnt[p][cur], c); cur = d1; c = 1; }
        if (d2 == cur) ++c; else { atomicAdd(&s_cnt[p][cur], c); cur = d2; c = 1; }
        if (d3 == cur) ++c; else { atomicAdd(&s_cnt[p][cur], c); cur = d3; c = 1; }
        atomicAdd(&s_cnt[p][cur], c);
      }
    }
  };
  int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  for (; i + stride < n4; i += 2 * stride) {
    const uint4 a = keys4[i], b = keys4[i + stride];  // default policy: the passes re-read them
    count4(a);
    count4(b);
  }
  for (; i < n4; i += stride) count4(keys4[i]);
  for (int64_t t = 4 * n4 + (int64_t)blockIdx.x * kThreads + threadIdx.x; t < n; t += stride) {
    const uint32_t key = keys[t];
#pragma unroll
    for (int p = 0; p < kMaxPasses; ++p)
      if (p < plan.n_passes) atomicAdd(&s_cnt[p][(key >> plan.shift[p]) & ((1u << plan.bits[p]) - 1u)], 1u);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < kMaxPasses * 256; k += kThreads) {
    const uint32_t c = (&s_cnt[0][0])[k];
    if (c) atomicAdd(hist + k, c);
  }
}

// Exclusive scan of each pass's 256 digit counts (one CTA of 256 threads per pass).
__global__ void k_onesweep_hist_scan(uint32_t* __restrict__ hist) {
  pdl_wait();
  __shared__ uint32_t s_w[8];
  const int p = blockIdx.x, d = threadIdx.x, lane = d & 31, warp = d >> 5;
  const uint32_t v = hist[p * 256 + d];
  const uint32_t incl = warp_inclusive_scan(v, lane);
  if (lane == 31) s_w[warp] = incl;
  __syncthreads();
  uint32_t off = 0;
  for (int w = 0; w < warp; ++w) off += s_w[w];
  hist[p * 256 + d] = off + incl - v;
}

// Threads x IPT items per tile (shared memory: keys + values + per-warp digit counts,
// dynamic). MinBlocks: 3 CTAs/SM (80 registers, no spills) for the depth sort; more
// occupancy (a few spills) for the long tile-entry sorts, where it wins.
// Bits: the digit width (a template argument, so the ranking's ballot loop unrolls).
template <int Threads, int IPT, int MinBlocks, int Bits>
__global__ void __launch_bounds__(Threads, MinBlocks) k_onesweep_pass(
    const uint32_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in, uint32_t* __restrict__ keys_out,
    uint32_t* __restrict__ vals_out, int64_t n, int shift, const uint32_t* __restrict__ digit_start,
    uint32_t* __restrict__ status, uint32_t* __restrict__ tile_counter, const uint32_t* __restrict__ gather_src,
    uint32_t* __restrict__ gather_dst, uint32_t* __restrict__ status_next, const uint32_t* n_dev) {
  pdl_wait();
  constexpr int kW = Threads / 32;
  constexpr int kT = Threads * IPT;
  constexpr int kWI = 32 * IPT;
  extern __shared__ uint32_t s_dyn[];
  uint32_t* s_keys = s_dyn;                     // [kT]
  uint32_t* s_vals = s_dyn + kT;                // [kT]
  uint32_t(*s_wcnt)[256] = reinterpret_cast<uint32_t(*)[256]>(s_dyn + 2 * kT);  // [kW][256]
  __shared__ uint32_t s_start[256];
  __shared__ uint32_t s_gbase[256];
  __shared__ uint32_t s_wsum[kW];
  __shared__ int s_tile;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int radix = 1 << Bits;
  constexpr uint32_t mask = (uint32_t)radix - 1u;
  if (threadIdx.x == 0) s_tile = (int)atomicAdd(tile_counter, 1u);
  if (status_next && threadIdx.x < 256) status_next[(int64_t)blockIdx.x * 256 + threadIdx.x] = 0u;
  for (int k = threadIdx.x; k < kW * 256; k += Threads) (&s_wcnt[0][0])[k] = 0;
  __syncthreads();
  const int tile = s_tile;
  const int64_t tile_base = (int64_t)tile * kT;
  // The items of this tile: [0, valid_count). With a device-side count (capacity-sized
  // grid) the tiles past it have nothing to sort; they claim the highest ids, so no tile
  // with items ever looks back at them. Only this 32-bit count stays live below.
  const int64_t n_items = n_dev ? min(n, (int64_t)*n_dev) : n;
  if (tile_base >= n_items && tile > 0) return;
  const int valid_count = (int)min((int64_t)kT, n_items - tile_base);
  const int64_t base = tile_base + (int64_t)warp * kWI;
  const int wbase = warp * kWI;  // tile-relative
  const uint32_t lt_mask = (1u << lane) - 1u;
  uint32_t key[IPT], rank[IPT];  // the values are loaded at the shared-memory scatter
  // All key loads first, so the tile's loads per thread are in flight together.
#pragma unroll
  for (int j = 0; j < IPT; ++j) {
    const int64_t idx = base + j * 32 + lane;
    const bool ok = wbase + j * 32 + lane < valid_count;
    key[j] = ok ? __ldcs(keys_in + idx) : 0u;
  }
#pragma unroll
  for (int j = 0; j < IPT; ++j) {
    const bool valid = wbase + j * 32 + lane < valid_count;
    const uint32_t d = valid ? (key[j] >> shift) & mask : mask;
    uint32_t peers = 0xffffffffu;
#pragma unroll
    for (int b = 0; b < Bits; ++b) {
      const uint32_t bit = (d >> b) & 1u;
      const uint32_t bal = __ballot_sync(0xffffffffu, bit);
      peers &= bit ? bal : ~bal;
    }
    const uint32_t pre = s_wcnt[warp][d];
    __syncwarp();
    if ((peers & lt_mask) == 0) s_wcnt[warp][d] = pre + __popc(peers);
    __syncwarp();
    rank[j] = pre + __popc(peers & lt_mask);
  }
  __syncthreads();
  // Per-digit tile totals (padding excluded: it sits in the last digit, after every
  // real item, so subtract it from that digit's count).
  uint32_t digit_total = 0;
  if (threadIdx.x < radix) {
    const int d = threadIdx.x;
    for (int w = 0; w < kW; ++w) {
      const uint32_t c = s_wcnt[w][d];
      s_wcnt[w][d] = digit_total;
      digit_total += c;
    }
  }
  const uint32_t incl = warp_inclusive_scan(digit_total, lane);
  if (lane == 31) s_wsum[warp] = incl;
  __syncthreads();
  uint32_t woff = 0;
  for (int w = 0; w < warp; ++w) woff += s_wsum[w];
  // Publish this tile's per-digit counts first, so successors can look back past it
  // while it scatters into shared memory.
  const int d_own = threadIdx.x;
  uint32_t start = 0, real = 0;
  volatile uint32_t* st = status;
  if (d_own < radix) {
    start = woff + incl - digit_total;
    s_start[d_own] = start;
    real = (d_own == radix - 1) ? digit_total - (uint32_t)(kT - valid_count) : digit_total;
    st[(int64_t)tile * 256 + d_own] = (tile == 0 ? kStatPrefix : kStatAgg) | real;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < IPT; ++j) {
    const uint32_t d = wbase + j * 32 + lane < valid_count ? (key[j] >> shift) & mask : mask;
    const uint32_t pos = s_start[d] + s_wcnt[warp][d] + rank[j];
    s_keys[pos] = key[j];
    if (wbase + j * 32 + lane < valid_count) s_vals[pos] = __ldcs(vals_in + base + j * 32 + lane);
  }
  if (d_own < radix) {
    const int d = d_own;
    if (tile == 0) {
      s_gbase[d] = digit_start[d] - start;
    } else {
      // Windowed look-back: kLookWindow predecessors' words are loaded together (one
      // round trip per window instead of per tile), then consumed newest first up to
      // the first prefix; an unpublished word restarts the window there.
      uint32_t excl = 0;
      uint32_t rounds = 0;
      for (int look = tile - 1; look >= 0;) {
        // A predecessor that never publishes (a launch or memory fault upstream) would
        // spin this loop forever: fail the kernel instead of hanging the device.
        if (++rounds > (1u << 26)) __trap();
        uint32_t w[kLookWindow];
#pragma unroll
        for (int j = 0; j < kLookWindow; ++j)
          w[j] = look - j >= 0 ? st[(int64_t)(look - j) * 256 + d] : (uint32_t)kStatPrefix;
        bool done = false;
#pragma unroll
        for (int j = 0; j < kLookWindow; ++j) {
          if ((w[j] & ~kStatMask) == 0) break;  // predecessor not published yet: spin here
          excl += w[j] & kStatMask;
          --look;
          if (w[j] & kStatPrefix) {
            done = true;
            break;
          }
        }
        if (done) break;
      }
      st[(int64_t)tile * 256 + d] = kStatPrefix | (excl + real);
      s_gbase[d] = digit_start[d] + excl - start;
    }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < valid_count; k += Threads) {
    const uint32_t kk = s_keys[k];
    const uint32_t d = (kk >> shift) & mask;
    const uint32_t pos = s_gbase[d] + (uint32_t)k;
    const uint32_t v = s_vals[k];
    keys_out[pos] = kk;
    vals_out[pos] = v;
    if (gather_dst) gather_dst[pos] = gather_src[v];  // last pass: payload in sorted order
  }
}

int64_t blocks_for(int64_t n) { return (n + kTile - 1) / kTile; }

__global__ void k_zero_u32(uint32_t* __restrict__ p, int n) {
  pdl_wait();
  for (int k = threadIdx.x; k < n; k += blockDim.x) p[k] = 0u;
}

__global__ void k_gather(int64_t n, const uint32_t* __restrict__ idx, const uint32_t* __restrict__ src,
                         uint32_t* __restrict__ dst, const uint32_t* n_dev) {
  pdl_wait();
  if (n_dev) n = min(n, (int64_t)*n_dev);
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[idx[i]];
}

}  // namespace

thread_local int64_t g_launches = 0;

size_t scan_temp_bytes(int64_t n) {
  if (n <= kTile) return 0;
  const int64_t nb = blocks_for(n);
  return (size_t)(2 * nb) * sizeof(uint32_t) + 256 + scan_temp_bytes(nb);
}

void exclusive_scan_u32(const uint32_t* in, uint32_t* out, int64_t n, void* temp, unsigned long long* total64,
                        cudaStream_t stream, const uint32_t* n_dev) {
  if (n <= 0) return;
  if (n <= kTile) {
    launch_pdl(k_scan_downsweep, 1, kThreads, 0, stream, in, out, n, nullptr, total64, n_dev);
    ++g_launches;
    return;
  }
  const int64_t nb = blocks_for(n);
  uint32_t* sums = static_cast<uint32_t*>(temp);
  uint32_t* offs = sums + nb;
  void* next = reinterpret_cast<char*>(temp) + (((size_t)(2 * nb) * sizeof(uint32_t) + 255) / 256) * 256;
  // Blocks past the device-side count write zero sums, so the block scan needs no count.
  launch_pdl(k_scan_reduce, (unsigned)nb, kThreads, 0, stream, in, n, sums, total64, n_dev);
  ++g_launches;
  exclusive_scan_u32(sums, offs, nb, next, nullptr, stream, nullptr);
  launch_pdl(k_scan_downsweep, (unsigned)nb, kThreads, 0, stream, in, out, n, offs, nullptr, n_dev);
  ++g_launches;
}

size_t radix_sort_temp_bytes(int64_t n) {
  // Enough status words for any sort of <= n pairs (either tile shape).
  constexpr int64_t min_tile = std::min(kThreads * kSmallIPT, kBigThreads * kBigIPT);
  const int64_t nb = (std::max<int64_t>(n, 1) + min_tile - 1) / min_tile;
  // hist [kMaxPasses][256] + tile counters [64] + status [2][nb][256] (alternating passes)
  return (size_t)(kMaxPasses * 256 + 64 + 2 * nb * 256) * sizeof(uint32_t);
}

namespace {


struct PassArgs {
  const uint32_t *keys_in, *vals_in;
  uint32_t *keys_out, *vals_out;
  int64_t n;
  int shift;
  const uint32_t* digit_start;
  uint32_t *status, *tile_counter;
  const uint32_t* gather_src;
  uint32_t* gather_dst;
  uint32_t* status_next;
  const uint32_t* n_dev;
};

// The dynamic shared-memory opt-in is a per-device function attribute: one flag bit per
// device in `done` (one word per kernel instantiation), set once (racing threads at worst
// set it twice).
template <class Kern> cudaError_t opt_in_smem(Kern kern, size_t smem, std::atomic<uint64_t>& done) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

template <int Threads, int IPT, int MinBlocks, int Bits>
cudaError_t launch_pass_bits(const PassArgs& a, cudaStream_t stream) {
  constexpr int kT = Threads * IPT;
  constexpr size_t smem = (size_t)(2 * kT + (Threads / 32) * 256) * sizeof(uint32_t);
  auto kern = k_onesweep_pass<Threads, IPT, MinBlocks, Bits>;
  static std::atomic<uint64_t> opted{0};  // per instantiation
  const cudaError_t e = opt_in_smem(kern, smem, opted);
  if (e != cudaSuccess) return e;
  const int64_t tiles = (a.n + kT - 1) / kT;
  return launch_pdl(kern, (unsigned)tiles, Threads, smem, stream, a.keys_in, a.vals_in, a.keys_out, a.vals_out, a.n,
                    a.shift, a.digit_start, a.status, a.tile_counter, a.gather_src, a.gather_dst, a.status_next,
                    a.n_dev);
}

template <int Threads, int IPT, int MinBlocks>
cudaError_t launch_pass(int bits, const PassArgs& a, cudaStream_t stream) {
  switch (bits) {
    case 1: return launch_pass_bits<Threads, IPT, MinBlocks, 1>(a, stream);
    case 2: return launch_pass_bits<Threads, IPT, MinBlocks, 2>(a, stream);
    case 3: return launch_pass_bits<Threads, IPT, MinBlocks, 3>(a, stream);
    case 4: return launch_pass_bits<Threads, IPT, MinBlocks, 4>(a, stream);
    case 5: return launch_pass_bits<Threads, IPT, MinBlocks, 5>(a, stream);
    case 6: return launch_pass_bits<Threads, IPT, MinBlocks, 6>(a, stream);
    case 7: return launch_pass_bits<Threads, IPT, MinBlocks, 7>(a, stream);
    default: return launch_pass_bits<Threads, IPT, MinBlocks, 8>(a, stream);
  }
}

}  // namespace

cudaError_t radix_sort_pairs(uint32_t* keys[2], uint32_t* vals[2], int64_t n, int begin_bit, int end_bit,
                             void* temp, int* which, cudaStream_t stream, const uint32_t* gather_src,
                             uint32_t* gather_dst, const uint32_t* n_dev) {
  *which = 0;
  if (n >= (int64_t)kMaxSortItems) return cudaErrorInvalidValue;
  if ((n <= 1 && !n_dev) || n <= 0 || end_bit <= begin_bit) {
    if (gather_dst && n > 0) {
      ++g_launches;
      return launch_pdl(k_gather, (unsigned)((n + 255) / 256), 256, 0, stream, n, vals[0], gather_src, gather_dst,
                        n_dev);
    }
    return cudaSuccess;
  }
  PassPlan plan{};
  int passes = (end_bit - begin_bit + 7) / 8;
  if (passes > kMaxPasses) passes = kMaxPasses;
  plan.n_passes = passes;
  for (int bit = begin_bit, p = 0, left = passes; p < passes; ++p, --left) {
    const int bits = (end_bit - bit + left - 1) / left;
    plan.shift[p] = bit;
    plan.bits[p] = bits;
    bit += bits;
  }
  const int64_t nb = blocks_for(n);
  uint32_t* hist = static_cast<uint32_t*>(temp);
  uint32_t* counters = hist + kMaxPasses * 256;
  const int64_t tiles = pass_tiles(n);
  uint32_t* status[2] = {counters + 64, counters + 64 + tiles * 256};
  // The passes spin on look-back words: never launch one after a failed launch.
  cudaError_t e = launch_pdl(k_zero_u32, 1, 256, 0, stream, hist, kMaxPasses * 256 + 64);
  if (e != cudaSuccess) return e;
  ++g_launches;
  int sms = 148;
  e = launch_pdl(k_onesweep_hist, (unsigned)std::min<int64_t>(nb, 4 * sms), kThreads, 0, stream, keys[0], n, plan,
                 hist, status[0], tiles * 256, n_dev);
  if (e != cudaSuccess) return e;
  ++g_launches;
  e = launch_pdl(k_onesweep_hist_scan, passes, 256, 0, stream, hist);
  if (e != cudaSuccess) return e;
  ++g_launches;
  const bool big = n > kBigSort;
  int cur = 0;
  for (int p = 0; p < passes; ++p) {
    const bool last = p == passes - 1;
    PassArgs pa{keys[cur], vals[cur], keys[cur ^ 1], vals[cur ^ 1], n, plan.shift[p], hist + p * 256,
                status[p & 1], counters + p, last ? gather_src : nullptr, last ? gather_dst : nullptr,
                last ? nullptr : status[(p + 1) & 1], n_dev};
    e = big ? launch_pass<kBigThreads, kBigIPT, kBigMinBlocks>(plan.bits[p], pa, stream)
            : launch_pass<kThreads, kSmallIPT, kSmallMinBlocks>(plan.bits[p], pa, stream);
    if (e != cudaSuccess) return e;
    ++g_launches;
    cur ^= 1;
  }
  *which = cur;
  return cudaSuccess;
}

}  // namespace odgs_b200
