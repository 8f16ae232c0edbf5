// absim_gpu.cu — device kernels + C ABI (include/absim_gpu.h) of the B200
// mechanical-step engine. One iteration (Simulation::simulate body,
// simulation.cpp:232-303) is:
//
//   k_reduce     bbox + largest diameter          uniform_grid.cpp:74-110
//   k_finalize   box length, origin, dims, checks  uniform_grid.cpp:112-141
//   k_key        bin of each agent + per-bin count (atomic slot = rank)
//   scan         exclusive scan of bin counts -> cell table `start`
//   k_scatter    permute state into cell order (coalesced SoA writes)
//   k_mark       [static] disturbers flag neighbours  simulation.cpp:351-373
//   k_force      behaviours + static skip + 27-box radius query + pairwise
//                repulsion + force sum + integration     simulation.cpp:388-500
//   commit       [additions] daughter uid ranks + append  commit.cpp:186-222
//
// Every kernel is a grid-stride loop over a device-resident agent count, so an
// iteration needs no host synchronisation (counts change on the device).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstddef>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "absim_gpu.h"
#include "kernels.cuh"

using namespace absgpu;

namespace {

#ifndef ABS_FORCE_MIN_BLOCKS_F32
#define ABS_FORCE_MIN_BLOCKS_F32 5
#endif
#ifndef ABS_PASSB
#define ABS_PASSB 1  // 2 or 4 measured slower (c4 @ 2^24: 6.27 / 6.38 / 6.56 ms)
#endif
constexpr int kPassB = ABS_PASSB;  // contact records fetched together in pass B
constexpr int kForceMinBlocksF32 = ABS_FORCE_MIN_BLOCKS_F32;
// box-lockstep walk (bins == boxes): no row windows in shared memory, so the
// register budget alone sets residency
#ifndef ABS_FORCE_MIN_BLOCKS_BOX
#define ABS_FORCE_MIN_BLOCKS_BOX 8  // c3 k_force 0.685 (shared 96-reg build) -> 0.496 ms; c1 0.083 -> 0.059 ms (7: 0.530 / 0.057)
#endif
constexpr int kForceMinBlocksBox = ABS_FORCE_MIN_BLOCKS_BOX;
constexpr unsigned long long kInfOrdLo = 0xFFF0000000000000ull;  // ord_enc(+inf)
constexpr unsigned long long kInfOrdHi = 0x000FFFFFFFFFFFFFull;  // ord_enc(-inf)
constexpr unsigned long long kZeroOrd = 0x8000000000000000ull;   // ord_enc(+0.0)

// ---------------------------------------------------------------- reduce
// Block part of the bounds reduction: per-block min/max/dmax folded into the
// grid record with order-preserving u64 atomics (bit-exact, order free).
__device__ __forceinline__ void reduce_bounds_block(const Pd* __restrict__ pos, DevGrid* g, bool skip) {
  const unsigned long long n = skip ? 0ull : g->n;
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  double dm = 0.0;
  unsigned int bad = 0;
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const Pd p = load_pd(pos + i);
    const double v[3] = {p.x, p.y, p.z};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      bad |= !isfinite(v[k]);
      lo[k] = v[k] < lo[k] ? v[k] : lo[k];
      hi[k] = hi[k] < v[k] ? v[k] : hi[k];
    }
    dm = dm < p.d ? p.d : dm;
  }
  // warp then block reduction (min/max are order independent: bit-exact)
#pragma unroll
  for (int off = 16; off; off >>= 1) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double a = __shfl_xor_sync(0xffffffffu, lo[k], off);
      const double b = __shfl_xor_sync(0xffffffffu, hi[k], off);
      lo[k] = a < lo[k] ? a : lo[k];
      hi[k] = hi[k] < b ? b : hi[k];
    }
    const double c = __shfl_xor_sync(0xffffffffu, dm, off);
    dm = dm < c ? c : dm;
    bad |= __shfl_xor_sync(0xffffffffu, bad, off);
  }
  __shared__ double sh[kThreads / 32][7];
  __shared__ unsigned int sbad[kThreads / 32];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) {
    for (int k = 0; k < 3; ++k) { sh[w][k] = lo[k]; sh[w][3 + k] = hi[k]; }
    sh[w][6] = dm;
    sbad[w] = bad;
  }
  __syncthreads();
  if (threadIdx.x < 7) {
    const int k = threadIdx.x;
    double v = sh[0][k];
    for (int q = 1; q < kThreads / 32; ++q) {
      const double u = sh[q][k];
      v = k < 3 ? (u < v ? u : v) : (v < u ? u : v);
    }
    if (k < 3) atomicMin(&g->red[k], ord_enc(v));
    else atomicMax(&g->red[k], ord_enc(v));
  } else if (threadIdx.x == 7) {
    unsigned int b = 0;
    for (int q = 0; q < kThreads / 32; ++q) b |= sbad[q];
    if (b) atomicOr(&g->nonfinite, 1u);
  }
}

__global__ void __launch_bounds__(kThreads) k_reduce(const Pd* __restrict__ pos, DevGrid* g) {
  if (g->err) return;
  reduce_bounds_block(pos, g, false);
}

__device__ void reset_reduction(DevGrid* g) {
  g->red[0] = g->red[1] = g->red[2] = kInfOrdLo;
  g->red[3] = g->red[4] = g->red[5] = kInfOrdHi;
  g->red[6] = kZeroOrd;
  g->nonfinite = 0;
}

// uniform_grid.cpp:59-141 sizing; one thread.
struct FinArgs {
  double fixed_box;
  int brute;
  unsigned int bins_x, bins_yz, row_block_shift;
  unsigned long long bins_cap, capacity, uid_cap;
  int may_add;
  unsigned long long iteration;
  int list_mode;  // 0 no neighbour lists, 1 list step (check coverage), 2 list (re)build step,
                  // 3 re-binning step with displacement tracking (list policy)
  double skin;    // list skin (absolute)
  int counts_iteration;  // this finalize opens an iteration: add its agents to agent_its
};

__device__ void finalize_grid(DevGrid* g, const FinArgs& fa) {
  const double fixed_box = fa.fixed_box;
  const int brute = fa.brute;
  const unsigned int bins_x = fa.bins_x, bins_yz = fa.bins_yz, row_block_shift = fa.row_block_shift;
  const unsigned long long bins_cap = fa.bins_cap, capacity = fa.capacity, uid_cap = fa.uid_cap;
  const int may_add = fa.may_add;
  const unsigned long long iteration = fa.iteration;
  if (g->err) {
    reset_reduction(g);
    return;
  }
  const unsigned long long n = g->n;
  int err = kErrNone;
  if (n == 0) {
    g->dims[0] = g->dims[1] = g->dims[2] = 1;
    g->origin[0] = g->origin[1] = g->origin[2] = 0.0;
    g->box = fixed_box > 0.0 ? fixed_box : 1.0;
    g->dmax = 0.0;
  } else {
    double lo[3], hi[3];
    for (int k = 0; k < 3; ++k) {  // L2 reads: the other blocks' atomics
      lo[k] = ord_dec(__ldcg(&g->red[k]));
      hi[k] = ord_dec(__ldcg(&g->red[3 + k]));
    }
    double dm = ord_dec(__ldcg(&g->red[6]));
    for (int k = 0; k < 3; ++k)
      if (!isfinite(lo[k]) || !isfinite(hi[k])) err = kErrNonFinite;
    if (__ldcg(&g->nonfinite)) err = kErrNonFinite;
    if (g->ov_on) {  // multi-domain: grid of all ranks
      for (int k = 0; k < 3; ++k) lo[k] = g->ov_grid[k];
      dm = g->ov_grid[4];
    }
    g->dmax = dm;
    if (err == kErrNone) {
      if (g->ov_on) {
        g->box = g->ov_grid[3];
      } else if (brute) {
        // BruteForceEnvironment (environment.hpp:53-80): no grid. One box
        // larger than the bounding box holds every agent, so the box walk
        // visits all of them with the exact d2 <= r^2 test.
        double ext = 0.0;
        for (int k = 0; k < 3; ++k) ext = fmax(ext, hi[k] - lo[k]);
        g->box = 2.0 * ext + dm + 1.0;
      } else if (fixed_box > 0.0) {
        if (dm > fixed_box) err = kErrFixedBox;
        g->box = fixed_box;
      } else {
        g->box = dm;
      }
    }
    if (err == kErrNone) {
      unsigned long long needed = 1;
      for (int k = 0; k < 3; ++k) {
        g->origin[k] = lo[k];
        const unsigned long long nk =
            static_cast<unsigned long long>(floor((hi[k] - lo[k]) / g->box)) + 1ull;
        g->dims[k] = g->ov_on ? g->ov_dims[k] : static_cast<unsigned int>(nk < 1 ? 1 : nk);
        needed *= g->dims[k];
      }
      if (needed > (1ull << 31)) err = kErrBoxBudget;
    }
  }
  if (err == kErrNone) {
    unsigned int B[3] = {bins_x, bins_yz, bins_yz};
    // rows in y-blocks of 2^ysh (row_of); ~0u = one block (z-major rows)
    auto rows_shift = [&](unsigned int by) {
      unsigned int sh = 0;
      if (row_block_shift == ~0u) {
        while ((1u << sh) < by) ++sh;
      } else {
        sh = row_block_shift;
      }
      return sh;
    };
    auto padded = [&](const unsigned int* Bk) {
      const unsigned long long by = (unsigned long long)g->dims[1] * Bk[1];
      const unsigned int sh = rows_shift(static_cast<unsigned int>(by));
      const unsigned long long byp = ((by + (1ull << sh) - 1) >> sh) << sh;
      return (unsigned long long)g->dims[0] * Bk[0] * byp * ((unsigned long long)g->dims[2] * Bk[2]);
    };
    if (padded(B) + 1 > 0xFFFFFFFFull) B[0] = B[1] = B[2] = 1;
    const unsigned long long nbins = padded(B);
    if (nbins + 1 > 0xFFFFFFFFull) {  // padded bin rows exceed the u32 cell table
      err = kErrBoxBudget;
    } else if (nbins + 1 > bins_cap) {
      err = kErrBinsRetry;
      g->needed_bins = nbins + 1;
    } else if (may_add && (2 * n > capacity || g->uid_count + n > uid_cap)) {
      err = kErrCapRetry;
    } else {
      for (int k = 0; k < 3; ++k) {
        g->B[k] = B[k];
        g->s[k] = B[k] == 1 ? g->box : g->box / static_cast<double>(B[k]);
        g->bd[k] = g->dims[k] * B[k];
      }
      g->ysh = rows_shift(g->bd[1]);
      g->bd1p = ((g->bd[1] + (1u << g->ysh) - 1u) >> g->ysh) << g->ysh;
      g->nbins = nbins;
      double mag = g->box;
      for (int k = 0; k < 3; ++k) {
        mag = fmax(mag, fabs(g->origin[k]));
        mag = fmax(mag, fabs(g->origin[k] + g->dims[k] * g->box));
      }
      g->margin = 1e-9 * mag;
    }
  }
  // Neighbour lists. A list built at step t0 holds every j
  // with |p_i - p_j| <= r_i + skin at t0. At a later step, any j with
  // |p_i - p_j| <= r_i was within r_i + D_i + D_j at t0, where D is the
  // displacement since t0 <= list_acc (per-step maxima + rounding margin);
  // so the lists still cover the query while 2 list_acc <= skin and the
  // radii have not grown (constant diameters, dmax <= list_dmax).
  if (fa.list_mode == 2) {
    g->list_acc = 0.0;
    g->list_dmax = g->dmax;
    g->step_disp = 0u;
    g->list_need = 0u;
    g->list_incomplete = 0u;
    double ext = 1.0;
    for (int k = 0; k < 3; ++k) {
      g->lorigin[k] = g->origin[k];
      ext = fmax(ext, static_cast<double>(g->dims[k]) * g->box);
    }
    // relative coordinates stay within ext + skin / 2 while the lists are valid
    g->lslack = static_cast<float>(16.0 * (ext + fa.skin + 1.0) * 0x1.0p-24 + 1e-5);
  } else if (fa.list_mode == 3) {  // re-binning step whose displacement the list policy tracks
    g->step_disp = 0u;
  } else if (fa.list_mode == 1 && err == kErrNone) {
    const double acc = g->list_acc + static_cast<double>(__uint_as_float(g->step_disp)) + g->margin + 1e-12;
    g->list_acc = acc;
    g->step_disp = 0u;
    if (2.0 * acc > fa.skin || g->dmax > g->list_dmax || g->list_incomplete) err = kErrListRebuild;
  }
  reset_reduction(g);
  g->work = 0;
  g->sir[0] = g->sir[1] = g->sir[2] = 0;
  g->mark_n = 0;
  g->work_n = 0;
  if (err != kErrNone) {
    g->err = err;
    g->failed_iteration = iteration;
  } else if (fa.counts_iteration) {
    g->agent_its += n;
  }
}

__global__ void k_finalize(DevGrid* g, FinArgs fa) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  finalize_grid(g, fa);
}

// Environment update pass 1 in one launch: bounds reduction, then the last
// block to finish sizes the grid (uniform_grid.cpp:59-141).
// zero_start != nullptr: also clears the previous iteration's cell table
// (entries [0, nbins_prev]; every entry beyond is zero already), which the
// last block's finalize may resize only after every block has counted in.
__global__ void __launch_bounds__(kThreads) k_reduce_finalize(const Pd* __restrict__ pos, DevGrid* g, FinArgs fa,
                                                              unsigned int* __restrict__ zero_start) {
  const bool skip = g->err != 0;  // still counted, so the last block resets the reduction
  if (zero_start && !skip) {
    const unsigned long long len = g->nbins + 1;
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < len;
         i += (unsigned long long)gridDim.x * blockDim.x)
      zero_start[i] = 0u;
  }
  reduce_bounds_block(pos, g, skip);
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(&g->fin_count, 1ull) == gridDim.x - 1;
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    finalize_grid(g, fa);
    g->fin_count = 0;
  }
}

// ---------------------------------------------------------------- binning
__global__ void __launch_bounds__(kThreads) k_key(const Pd* __restrict__ pos, const DevGrid* g,
                                                  unsigned int* __restrict__ count,
                                                  unsigned int* __restrict__ key,
                                                  unsigned int* __restrict__ rank) {
  if (g->err) return;
  const DevGrid G = *g;
  const unsigned long long n = G.n;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  // two agents per thread: their loads and slot atomics overlap
  for (unsigned long long i0 = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i0 < n; i0 += 2 * stride) {
    unsigned int b[2], r[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const unsigned long long i = i0 + q * stride;
      if (i < n) {
        const Pd p = load_pd(pos + i);
        const unsigned int bx = bin_coord(p.x, G.origin[0], G, 0);
        const unsigned int by = bin_coord(p.y, G.origin[1], G, 1);
        const unsigned int bz = bin_coord(p.z, G.origin[2], G, 2);
        b[q] = bx + G.bd[0] * row_of(by, bz, G.ysh, G.bd[2]);
        ABS_ASSERT(b[q] < G.nbins);
      }
    }
#pragma unroll
    for (int q = 0; q < 2; ++q)
      if (i0 + q * stride < n) r[q] = atomicAdd(count + b[q], 1u);
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const unsigned long long i = i0 + q * stride;
      if (i < n) {
        key[i] = b[q];
        rank[i] = r[q];
      }
    }
  }
}

// ------------------------------------------------------------ exclusive scan
// In-place exclusive scan of data[0..len) (len read from *len_ptr), with
// data[len] = total. Three passes: tile sums, scan of tile sums, tile scan.
template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  const int l = threadIdx.x & 31;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const T u = __shfl_up_sync(0xffffffffu, v, off);
    if (l >= off) v += u;
  }
  return v;
}

template <typename T>
__device__ __forceinline__ T block_excl_scan(T v, T* total) {
  __shared__ T warp_sums[kThreads / 32];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const T inc = warp_incl_scan(v);
  if (l == 31) warp_sums[w] = inc;
  __syncthreads();
  if (w == 0) {
    T ws = l < kThreads / 32 ? warp_sums[l] : T(0);
    const T wi = warp_incl_scan(ws);
    if (l < kThreads / 32) warp_sums[l] = wi - ws;
    if (l == kThreads / 32 - 1) *total = wi;
  }
  __syncthreads();
  const T r = inc - v + warp_sums[w];
  __syncthreads();
  return r;
}

template <typename T>
__global__ void __launch_bounds__(kThreads) k_scan_tiles(const T* __restrict__ data,
                                                         const unsigned long long* len_ptr,
                                                         T* __restrict__ tile_sums, const int* err) {
  if (err && *err) return;
  const unsigned long long len = *len_ptr;
  const unsigned long long base = (unsigned long long)blockIdx.x * kScanTile;
  if (base >= len) return;
  T sum = 0;
  for (int q = 0; q < kScanTile / kThreads; ++q) {
    const unsigned long long i = base + threadIdx.x * (kScanTile / kThreads) + q;
    if (i < len) sum += data[i];
  }
  __shared__ T tot;
  block_excl_scan(sum, &tot);
  if (threadIdx.x == 0) tile_sums[blockIdx.x] = tot;
}

template <typename T>
__global__ void __launch_bounds__(kThreads) k_scan_partials(T* __restrict__ tile_sums,
                                                            const unsigned long long* len_ptr,
                                                            const int* err) {
  if (err && *err) return;
  const unsigned long long len = *len_ptr;
  const unsigned long long tiles = (len + kScanTile - 1) / kScanTile;
  T carry = 0;
  __shared__ T tot;
  for (unsigned long long b = 0; b < tiles; b += kThreads) {
    const unsigned long long i = b + threadIdx.x;
    const T v = i < tiles ? tile_sums[i] : T(0);
    const T e = block_excl_scan(v, &tot);
    if (i < tiles) tile_sums[i] = e + carry;
    carry += tot;
    __syncthreads();
  }
}

template <typename T>
__global__ void __launch_bounds__(kThreads) k_scan_apply(T* __restrict__ data,
                                                         const unsigned long long* len_ptr,
                                                         const T* __restrict__ tile_sums,
                                                         const int* err) {
  if (err && *err) return;
  const unsigned long long len = *len_ptr;
  const unsigned long long base = (unsigned long long)blockIdx.x * kScanTile;
  if (base >= len) return;
  constexpr int per = kScanTile / kThreads;
  T v[per];
  T sum = 0;
#pragma unroll
  for (int q = 0; q < per; ++q) {
    const unsigned long long i = base + threadIdx.x * per + q;
    v[q] = i < len ? data[i] : T(0);
    sum += v[q];
  }
  __shared__ T tot;
  T run = block_excl_scan(sum, &tot) + tile_sums[blockIdx.x];
#pragma unroll
  for (int q = 0; q < per; ++q) {
    const unsigned long long i = base + threadIdx.x * per + q;
    if (i < len) data[i] = run;
    run += v[q];
  }
  if (base + kScanTile >= len && threadIdx.x == kThreads - 1) data[len] = run;
}

// Single-pass exclusive scan of the u32 cell table (decoupled look-back):
// tiles are taken in order from a ticket counter, each publishes its
// aggregate, then its inclusive prefix, as one 64-bit word
// [epoch:24 | flag:2 | value:38] (flag 1 aggregate, 2 inclusive prefix).
// The epoch (per scan launch) makes the previous scan's words stale without a
// reset pass; the two tickets alternate by epoch parity and tile 0 clears the
// one the next scan will use. Same result as k_scan_tiles/partials/apply:
// data[i] = sum(data[0..i)), data[len] = total.
constexpr unsigned int kScanEpochMask = 0x3FFFFFFFu;

__global__ void __launch_bounds__(kThreads) k_scan_onepass(unsigned int* __restrict__ data,
                                                           const unsigned long long* len_ptr,
                                                           unsigned long long* __restrict__ state,
                                                           unsigned int epoch, const int* err) {
  unsigned long long* tickets = state;  // [0], [1]
  if (err && *err) {  // skipped: keep the ticket pair consistent for the next scan
    if (blockIdx.x == 0 && threadIdx.x == 0) tickets[(epoch + 1) & 1u] = 0;
    return;
  }
  const unsigned long long len = *len_ptr;
  const unsigned long long ntiles = (len + kScanTile - 1) / kScanTile;
  unsigned long long* tile_state = state + 2;
  __shared__ unsigned long long s_tile;
  __shared__ unsigned long long s_prefix;
  __shared__ unsigned int tot;
  if (threadIdx.x == 0) s_tile = atomicAdd(&tickets[epoch & 1u], 1ull);
  __syncthreads();
  const unsigned long long t = s_tile;
  if (t >= ntiles) {
    if (len == 0 && t == 0 && threadIdx.x == 0) {
      data[0] = 0;
      tickets[(epoch + 1) & 1u] = 0;
    }
    return;
  }
  if (t == 0 && threadIdx.x == 0) tickets[(epoch + 1) & 1u] = 0;
  const unsigned long long base = t * kScanTile;
  constexpr int per = kScanTile / kThreads;
  static_assert(per == 8, "the full-tile path moves two uint4 per thread");
  unsigned int v[per];
  unsigned int sum = 0;
  const bool full = base + kScanTile <= len;  // whole tile in range: 128-bit accesses (the table is 256-B aligned)
  if (full) {
    const uint4* src = reinterpret_cast<const uint4*>(data + base) + threadIdx.x * 2;
    const uint4 a = src[0], b = src[1];
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
#pragma unroll
    for (int q = 0; q < per; ++q) sum += v[q];
  } else {
#pragma unroll
    for (int q = 0; q < per; ++q) {
      const unsigned long long i = base + threadIdx.x * per + q;
      v[q] = i < len ? data[i] : 0u;
      sum += v[q];
    }
  }
  unsigned int run = block_excl_scan(sum, &tot);
  // tile word: epoch (30 bits) | inclusive/aggregate flags (2 bits) | value (32
  // bits: a tile prefix is at most the table total < 2^32). The host clears
  // the words when the 30-bit epoch wraps (launch_scan_cells), so a stale
  // word can never carry the current tag.
  const unsigned long long tag = static_cast<unsigned long long>(epoch & kScanEpochMask) << 34;
  constexpr unsigned long long kAgg = 1ull << 32, kInc = 2ull << 32, kVal = (1ull << 32) - 1;
  if (threadIdx.x < 32) {  // warp 0 looks back over 32 predecessors at a time
    const int lane = threadIdx.x;
    unsigned long long prefix = 0;
    if (t == 0) {
      if (lane == 0) atomicExch(&tile_state[0], tag | kInc | tot);
    } else {
      if (lane == 0) atomicExch(&tile_state[t], tag | kAgg | tot);
      for (long long base = static_cast<long long>(t) - 1;;) {
        const long long p = base - lane;  // lane 0 = nearest predecessor
        const unsigned long long w =
            p >= 0 ? *reinterpret_cast<volatile unsigned long long*>(&tile_state[p]) : (tag | kInc);  // before tile 0: 0
        const bool ready = (w & ~((1ull << 34) - 1)) == tag && (w & (kAgg | kInc));
        if (!__all_sync(0xffffffffu, ready)) continue;  // some predecessor not published yet
        const unsigned int inc = __ballot_sync(0xffffffffu, (w & kInc) != 0);
        const int stop = inc ? __ffs(inc) - 1 : 31;  // nearest inclusive prefix, else the whole window
        unsigned long long v = lane <= stop ? (w & kVal) : 0ull;
#pragma unroll
        for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        prefix += v;
        if (inc) break;
        base -= 32;
      }
      if (lane == 0) atomicExch(&tile_state[t], tag | kInc | (prefix + tot));
    }
    if (lane == 0) s_prefix = prefix;
  }
  __syncthreads();
  run += static_cast<unsigned int>(s_prefix);
  if (full) {
    unsigned int o[per];
#pragma unroll
    for (int q = 0; q < per; ++q) {
      o[q] = run;
      run += v[q];
    }
    uint4* dst = reinterpret_cast<uint4*>(data + base) + threadIdx.x * 2;
    dst[0] = make_uint4(o[0], o[1], o[2], o[3]);
    dst[1] = make_uint4(o[4], o[5], o[6], o[7]);
  } else {
#pragma unroll
    for (int q = 0; q < per; ++q) {
      const unsigned long long i = base + threadIdx.x * per + q;
      if (i < len) data[i] = run;
      run += v[q];
    }
  }
  if (t == ntiles - 1 && threadIdx.x == kThreads - 1) data[len] = run;
}

// ---------------------------------------------------------------- scatter
struct Soa {
  Pd* pd;
  unsigned long long* uid;
  unsigned char* flags;
  unsigned int* partners;
  double* vol;
  unsigned char* beh;
  double* force;  // [3][cap]
  unsigned int* tag;          // Agent::tag (agent.hpp:35-36)
  unsigned long long* rngc;   // Agent::rng_counter (agent.hpp:145)
  unsigned int* skey;         // the agent's slot in the REFERENCE's storage order
};

// Counting-sort scatter: agent i moves to slot start[key[i]] + rank[i] of
// the destination buffers. kScatterBatch agents per thread are loaded before
// any store, so each thread keeps several independent loads in flight (the
// kernel is load-latency bound otherwise). partners are not carried when
// the force sweep of the same iteration rewrites every one of them
// (carry_partners = 0: no static detection, no SIR), beh only when a model
// reads it.
#ifndef ABS_SCATTER_BATCH
#define ABS_SCATTER_BATCH 2  // c4 step 30.25 / 29.45 / 29.52 ms at 1 / 2 / 4; c3 0.98 / 0.96 / 0.99
#endif
constexpr int kScatterBatch = ABS_SCATTER_BATCH;
template <bool MARK>  // MARK: also list the static-detection marking agents (block-uniform loop for the ballots)
__global__ void __launch_bounds__(kThreads) k_scatter(const Pd* __restrict__ pos, Soa src, Soa dst,
                                                      float4* __restrict__ pf,
                                                      const unsigned int* __restrict__ start,
                                                      const unsigned int* __restrict__ key,
                                                      const unsigned int* __restrict__ rank,
                                                      const DevGrid* g, unsigned long long cap,
                                                      int carry_vol, int carry_force, int write_pf,
                                                      int only_sort_mode = -1, int carry_ext = 0,
                                                      int carry_partners = 1, int carry_beh = 1,
                                                      unsigned int* __restrict__ mark_list = nullptr,
                                                      unsigned long long* __restrict__ mark_n = nullptr) {
  if (g->err) return;
  if (only_sort_mode >= 0 && static_cast<int>(g->sort_mode) != only_sort_mode) return;
  const unsigned long long n = g->n;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  const double ox = g->origin[0], oy = g->origin[1], oz = g->origin[2];
  // MARK: block-uniform trip count (the tail is handled per element), the
  // mark-list ballots below need whole warps
  for (unsigned long long b0 = blockIdx.x * (unsigned long long)blockDim.x + (MARK ? 0u : threadIdx.x); b0 < n;
       b0 += stride * kScatterBatch) {
    const unsigned long long i0 = b0 + (MARK ? threadIdx.x : 0u);
    unsigned int j[kScatterBatch];
    Pd p[kScatterBatch];
    unsigned long long u[kScatterBatch];
    unsigned int pa[kScatterBatch];
    unsigned char fl[kScatterBatch], bh[kScatterBatch];
#pragma unroll
    for (int b = 0; b < kScatterBatch; ++b) {
      const unsigned long long i = i0 + b * stride;
      if (i < n) {
        j[b] = __ldg(start + key[i]) + rank[i];
        p[b] = load_pd(pos + i);
        u[b] = src.uid[i];
        fl[b] = src.flags[i];
        if (carry_partners) pa[b] = src.partners[i];
        if (carry_beh) bh[b] = src.beh[i];
      }
    }
#pragma unroll
    for (int b = 0; b < kScatterBatch; ++b) {
      const unsigned long long i = i0 + b * stride;
      if (i >= n) break;
      const unsigned int jj = j[b];
      ABS_ASSERT(jj < n);
      reinterpret_cast<double2*>(dst.pd + jj)[0] = make_double2(p[b].x, p[b].y);
      reinterpret_cast<double2*>(dst.pd + jj)[1] = make_double2(p[b].z, p[b].d);
      if (write_pf)
        pf[jj] = make_float4(static_cast<float>(p[b].x - ox), static_cast<float>(p[b].y - oy),
                             static_cast<float>(p[b].z - oz), static_cast<float>(p[b].d));
      dst.uid[jj] = u[b];
      dst.flags[jj] = fl[b];
      if (carry_partners) dst.partners[jj] = pa[b];
      if (carry_beh) dst.beh[jj] = bh[b];
      if (carry_vol) dst.vol[jj] = src.vol[i];
      if (carry_force) {
        dst.force[jj] = src.force[i];
        dst.force[cap + jj] = src.force[cap + i];
        dst.force[2 * cap + jj] = src.force[2 * cap + i];
      }
      if (carry_ext) {
        dst.tag[jj] = src.tag[i];
        dst.rngc[jj] = src.rngc[i];
      }
      dst.skey[jj] = src.skey[i];
    }
    // static detection: the agents that moved, grew or were added last
    // iteration mark their neighbours (k_mark); they are listed here, by their
    // new slot, instead of in a pass of their own over every agent's flags
    if constexpr (MARK) {
#pragma unroll
      for (int b = 0; b < kScatterBatch; ++b) {
        const unsigned long long i = i0 + b * stride;
        const bool act = i < n && (fl[b] & (ABS_FLAG_MOVED | ABS_FLAG_GREW | ABS_FLAG_NEWLY_ADDED));
        const unsigned int ballot = __ballot_sync(0xffffffffu, act);
        if (!ballot) continue;
        const int lane = threadIdx.x & 31;
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(mark_n, (unsigned long long)__popc(ballot));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (act) mark_list[base + __popc(ballot & ((1u << lane) - 1u))] = j[b];
      }
    }
  }
}

// Zero a[0 .. *len_ptr (+1)), clamped to the allocation (cap entries); skipped
// once the iteration has failed (the host clears the table before a re-run).
__global__ void k_zero_u32(unsigned int* __restrict__ a, const unsigned long long* len_ptr, int plus_one,
                           const int* err, unsigned long long cap) {
  if (err && *err) return;
  unsigned long long len = *len_ptr + (plus_one ? 1 : 0);
  len = len < cap ? len : cap;
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < len;
       i += (unsigned long long)gridDim.x * blockDim.x)
    a[i] = 0;
}

// ------------------------------------------------------------ staticness
// Phase 1 of run_staticness_update (simulation.cpp:351-373), scatter form:
// every disturber (moved|grew) or fresh agent flags the agents within its
// radius 0.5 (d_a + dmax). Racing stores write the same value (1).
// The marking agents are listed first (one atomic per warp), so the walks
// run on full warps: only ~10 % of config 3's agents move, scattered over
// storage, and a per-agent grid would leave ~90 % of the lanes idle.
__global__ void __launch_bounds__(kThreads) k_mark_list(Soa S, DevGrid* g, unsigned int* __restrict__ list) {
  if (g->err) return;
  const unsigned long long n = g->n;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  for (unsigned long long b = blockIdx.x * (unsigned long long)blockDim.x; b < n; b += stride) {
    const unsigned long long i = b + threadIdx.x;  // warp-uniform trip count
    bool act = false;
    if (i < n) act = S.flags[i] & (ABS_FLAG_MOVED | ABS_FLAG_GREW | ABS_FLAG_NEWLY_ADDED);
    const unsigned int ballot = __ballot_sync(0xffffffffu, act);
    if (!ballot) continue;
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(&g->mark_n, (unsigned long long)__popc(ballot));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (act) list[base + __popc(ballot & ((1u << lane) - 1u))] = static_cast<unsigned int>(i);
  }
}

__global__ void __launch_bounds__(kThreads) k_mark(Soa S, const DevGrid* g,
                                                   const unsigned int* __restrict__ start,
                                                   unsigned char* __restrict__ nv,
                                                   unsigned char* __restrict__ nn,
                                                   const unsigned int* __restrict__ list) {
  if (g->err) return;
  __shared__ QGrid Q;
  if (threadIdx.x == 0) Q = make_qgrid(*g);
  __syncthreads();
  const unsigned long long m = g->mark_n;
  const double dmax = g->dmax;
  for (unsigned long long k = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; k < m;
       k += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long i = list[k];
    const unsigned char f = S.flags[i];
    const bool disturbs = f & (ABS_FLAG_MOVED | ABS_FLAG_GREW);
    const bool fresh = f & ABS_FLAG_NEWLY_ADDED;
    if (!disturbs && !fresh) continue;
    const Pd me = load_pd(S.pd + i);
    const double r = 0.5 * (me.d + dmax);
    for_each_neighbor(Q, S.pd, start, static_cast<unsigned int>(i), me.x, me.y, me.z, r, r * r,
                      [&](unsigned int j, const Pd&, double, double, double, double) {
                        if (disturbs) nv[j] = 1;
                        if (fresh) nn[j] = 1;
                      });
  }
}

// ------------------------------------------------------------ force step
// Coincident centres (mechanics.cpp:14-19): direction from
// RandomStream(seed = min uid, stream = max uid).unit_vector() (random.hpp:47-52,
// cos/sin — the one non-bit-portable term), negated for the larger uid.
// Out of line: it is essentially never taken and its registers would
// otherwise cap the occupancy of the force kernel.
__device__ __noinline__ void coincident_force(unsigned long long ua, unsigned long long ub, double m,
                                              double* f0, double* f1, double* f2) {
  const unsigned long long lo = ua < ub ? ua : ub;
  const unsigned long long hi = ua < ub ? ub : ua;
  const double zz = -1.0 + 2.0 * abs_u01(abs_rng_word(lo, hi, 0));
  const double phi = 2.0 * ABS_PI * abs_u01(abs_rng_word(lo, hi, 1));
  const double rr = sqrt(fmax(0.0, 1.0 - zz * zz));
  double d0 = rr * cos(phi), d1 = rr * sin(phi), d2 = zz;
  if (ua != lo) {
    d0 *= -1.0;
    d1 *= -1.0;
    d2 *= -1.0;
  }
  *f0 = d0 * m;
  *f1 = d1 * m;
  *f2 = d2 * m;
}

constexpr unsigned char kFlagGhost = 128u;  // ABS_FLAG_GHOST

// Outputs of one agent's step that need warp-level cooperation afterwards.
struct Daughter {
  bool divides;
  bool dies;  // AgentContext::remove_self staged (ABS_MODEL_GROW_DIVIDE_DIE)
  unsigned long long parent;
  double x, y, z, d, vol;
  unsigned int tag;
  float moved;  // length of this step's translation (0 if none)
};

// RandomStream::unit_vector (random.hpp:47-52) on an agent's own stream:
// two draws at its counter (advanced by 2); cos/sin are the non-bit-portable
// terms (values within tolerance, as in coincident_force).
__device__ __forceinline__ void stream_unit_vector(unsigned long long seed, unsigned long long uid,
                                                   unsigned long long& ctr, double out[3]) {
  const double u1 = abs_u01(abs_rng_word(seed, uid, ctr++));
  const double zz = -1.0 + (1.0 - -1.0) * u1;
  const double u2 = abs_u01(abs_rng_word(seed, uid, ctr++));
  const double phi = 0.0 + (2.0 * ABS_PI - 0.0) * u2;
  const double q = 1.0 - zz * zz;
  const double r = sqrt(0.0 < q ? q : 0.0);
  out[0] = r * cos(phi);
  out[1] = r * sin(phi);
  out[2] = zz;
}

// Behaviour-side radius query (AgentContext::for_each_neighbor,
// simulation.hpp:213-218) for kernels that do not provide one.
struct NoQuery {
  template <class F>
  __device__ void operator()(double, double, F&&) const {}
};

// Behaviours, static skip, run_forces and apply_pending for agent i (storage
// index). `walk(r, r2, visit)` enumerates every candidate j != i with exact
// fp64 d2 <= r2 in a fixed order; `fetch(j)` returns candidate j's Pd;
// `uid_of(j)` its uid. `ovl` is this thread's column of the contact list.
// F32: `walk` is the fp32-classified walker (visit(j, df2, qd) for exactly
// the candidates with fp64 d2 <= r^2); the contact record test is then the
// conservative fp32 superset df2 < (h + slack)^2 (pass B decides exactly).
template <int MODEL, bool STATIC, bool RECORD, bool F32 = false, class OvlT, class Walk, class Fetch,
          class UidOf, class Query = NoQuery>
__device__ __forceinline__ Daughter agent_step(Soa& S, Pd* __restrict__ out, unsigned long long i, const Pd& me,
                                               double dmax, unsigned char* __restrict__ nv,
                                               unsigned char* __restrict__ nn, const StepArgs& a,
                                               unsigned long long cap, OvlT* ovl, int ovl_stride,
                                               unsigned long long& n_eval, unsigned long long& n_skip,
                                               Walk&& walk, Fetch&& fetch, UidOf&& uid_of, float slack = 0.0f,
                                               const Query& query = Query{}) {
  Daughter dg{false, false, 0, 0, 0, 0, 0, 0, 0u, 0.0f};
  unsigned char fl = S.flags[i];
  const unsigned long long my_uid = S.uid[i];
  dg.parent = S.skey[i];  // daughters are numbered in the reference's storage order
  if (fl & kFlagGhost) {  // halo copy of another rank's agent: candidate only
    {
      if (STATIC) {
        nv[i] = 0;
        nn[i] = 0;
      }
      reinterpret_cast<double2*>(out + i)[0] = make_double2(me.x, me.y);
      reinterpret_cast<double2*>(out + i)[1] = make_double2(me.z, me.d);
    }
    return dg;
  }
  // --- staticness phase 2 (simulation.cpp:375-384) -----------------------
  // (the nv / nn resets and the volume update are written at the end)
  if (STATIC) {
    if (a.iteration == 0) {
      fl = 0;  // :335-349 everyone participates, flags wiped
    } else {
      const bool skip = !(fl & (ABS_FLAG_MOVED | ABS_FLAG_GREW | ABS_FLAG_NEWLY_ADDED |
                                ABS_FLAG_NEIGHBOR_VIOLATION | ABS_FLAG_NEW_NEIGHBOR)) &&
                        !nv[i] && !nn[i] && S.partners[i] <= 1u;
      fl = skip ? ABS_FLAG_STATIC : 0;
    }
  }
  // --- behaviours (run before forces, simulation.cpp:389-394) -------------
  double tx = 0.0, ty = 0.0, tz = 0.0, tg = 0.0;
  double new_vol = 0.0;
  bool vol_changed = false;
  unsigned long long new_rngc = 0;
  bool rngc_changed = false;
  if (MODEL != ABS_MODEL_NONE && S.beh[i]) {
    if (MODEL == ABS_MODEL_PROLIFERATION) {
      double v = S.vol[i] + a.mp[0];
      if (v > a.mp[1]) {
        v *= 0.5;
        double dir[3];
        abs_unit_vector(a.seed, my_uid, ABS_RNG_DIVISION_BASE(a.iteration), dir);
        const double half = 0.5 * me.d;
        dg.x = me.x + dir[0] * half;
        dg.y = me.y + dir[1] * half;
        dg.z = me.z + dir[2] * half;
        dg.d = abs_diameter_of_volume(v);
        dg.vol = v;
        dg.divides = true;
      }
      new_vol = v;
      vol_changed = true;
      tg += abs_diameter_of_volume(v) - me.d;
    } else if (MODEL == ABS_MODEL_DRIVE) {
      double dl[3];
      abs_drive_delta(me.x, me.y, me.z, a.mp[0], a.mp[1], a.mp[2], a.mp[3], a.seed, my_uid, a.iteration, dl);
      tx += dl[0];
      ty += dl[1];
      tz += dl[2];
    } else if (MODEL == ABS_MODEL_GROW) {
      if (me.d < a.mp[1]) {
        const double rem = a.mp[1] - me.d;
        tg += rem < a.mp[0] ? rem : a.mp[0];
      }
    } else if ((MODEL == ABS_MODEL_GROW_DIVIDE_DIE) &&
               abs_u01(abs_rng_word(a.seed, my_uid, ABS_RNG_DEATH(a.iteration))) < a.mp[3]) {
      dg.dies = true;  // ctx.remove_self(): committed after the iteration (simulation.cpp:64-66)
    } else if (MODEL == ABS_MODEL_GROW_DIVIDE || MODEL == ABS_MODEL_GROW_DIVIDE_DIE) {
      // models::GrowDivide (models.hpp:15-37)
      if (me.d >= a.mp[1]) {
        unsigned long long ctr = S.rngc[i];
        double dir[3];
        stream_unit_vector(a.seed, my_uid, ctr, dir);  // ctx.random().unit_vector()
        new_rngc = ctr;
        rngc_changed = true;
        const double half = 0.5 * me.d;
        dg.x = me.x + dir[0] * half;
        dg.y = me.y + dir[1] * half;
        dg.z = me.z + dir[2] * half;
        dg.d = a.mp[2];
        dg.vol = 0.0;
        dg.tag = S.tag[i];  // daughter.set_tag(a.tag())
        dg.divides = true;
        tg += a.mp[2] - me.d;
      } else {
        tg += a.mp[0];
      }
    } else if (MODEL == ABS_MODEL_COHERE) {  // models::Cohere (models.hpp:42-64)
      const unsigned int my_tag = S.tag[i];
      double sx = 0.0, sy = 0.0, sz = 0.0;
      unsigned long long cnt = 0;
      query(a.mp[0], a.mp[0] * a.mp[0], [&](unsigned int j, const Pd& q) {
        if (S.tag[j] == my_tag) {
          sx += q.x;
          sy += q.y;
          sz += q.z;
          ++cnt;
        }
      });
      if (cnt) {
        const double inv = 1.0 / static_cast<double>(cnt);
        const double cx = sx * inv - me.x, cy = sy * inv - me.y, cz = sz * inv - me.z;
        const double dist = sqrt((cx * cx + cy * cy) + cz * cz);
        if (dist > 0.0) {
          const double f = a.mp[1] / dist;
          tx += cx * f;
          ty += cy * f;
          tz += cz * f;
        }
      }
    }
  }
  // --- run_forces (simulation.cpp:463-489) --------------------------------
  // Pass A streams every candidate through the exact fp64 radius test
  // (d2 <= r^2 counts a force evaluation) and records the ones that may
  // overlap; pass B runs pairwise_repulsion only on those, in stream order.
  // A pair can only contribute if dist < h = 0.5 (d_a + d_b); the record test
  // d2 < h^2 (1 + 2^-50) is a strict superset of that (sqrt is correctly
  // rounded and monotone), so no contributor is missed and every decision in
  // pass B is the reference's exact one.
  bool wrote_partners = false;
  unsigned int contributors = 0;
  double fx = 0.0, fy = 0.0, fz = 0.0;
  if (STATIC && (fl & ABS_FLAG_STATIC)) {
    ++n_skip;
  } else {
    const double r = 0.5 * (me.d + dmax);
    unsigned int evals = 0, nov = 0;
    const float dif = static_cast<float>(me.d);
    // contact superset threshold: (0.5 (d_a + d_b) + slack)^2 (1 + 5e-7), the
    // half diameter of this agent and the slack folded in once
    const float hme = 0.5f * dif + slack;
    // contacts beyond the shared-memory list spill to a per-thread array (local
    // memory, touched only by the few lanes that need it): the alternative, a
    // second walk by that lane, stalls its whole warp (c1: ~1 % of the agents
    // hold more than 16 contacts, i.e. a quarter of the warps walked twice)
    unsigned int ovf[kSpillContacts];
    if constexpr (F32) {
      walk(r, r * r, [&](unsigned int j, float df2, float qd, bool in) {
        evals += in;
        const float hp = __fmaf_rn(0.5f, qd, hme);
        const bool ct = in && df2 < hp * hp * 1.0000005f;
        if (ct && nov < kMaxContacts) ovl[nov * ovl_stride] = static_cast<OvlT>(j);
        if (__builtin_expect(ct && nov >= kMaxContacts, 0))
          if (nov < kMaxContacts + kSpillContacts) ovf[nov - kMaxContacts] = j;
        nov += ct;
      });
    } else {
      walk(r, r * r, [&](unsigned int j, const Pd& q, double d2) {
        ++evals;
        const double h = 0.5 * (me.d + q.d);
        if (d2 < h * h * (1.0 + 0x1.0p-50)) {
          if (nov < kMaxContacts) ovl[nov * ovl_stride] = static_cast<OvlT>(j);
          else if (nov < kMaxContacts + kSpillContacts) ovf[nov - kMaxContacts] = j;
          ++nov;
        }
      });
    }
    n_eval += evals;
    if (a.evc) a.evc[i] = evals;
    const double k = a.k;
    auto contact_q = [&](unsigned int j, const Pd& q) {
      const double dx = me.x - q.x, dy = me.y - q.y, dz = me.z - q.z;
      // pairwise_repulsion (mechanics.cpp:10-27)
      const double dist = sqrt((dx * dx + dy * dy) + dz * dz);
      const double overlap = 0.5 * (me.d + q.d) - dist;
      if (overlap <= 0.0) return;
      double f0, f1, f2;
      if (dist > 0.0) {
        const double sc = k * overlap / dist;
        f0 = dx * sc;
        f1 = dy * sc;
        f2 = dz * sc;
      } else {
        coincident_force(my_uid, uid_of(j), k * overlap, &f0, &f1, &f2);
      }
      if ((f0 * f0 + f1 * f1) + f2 * f2 > 0.0) {
        ++contributors;
        fx += f0;
        fy += f1;
        fz += f2;
      }
    };
    auto contact = [&](unsigned int j) { contact_q(j, fetch(j)); };
    bool overflow = nov > kMaxContacts + kSpillContacts;
#if defined(ABS_ABLATE) && ABS_ABLATE >= 2
    if (nov > 1000000u) overflow = false;  // timing ablation: no pass B
    else nov = 0;
#endif
    if (!overflow) {
      // contact records fetched kPassB at a time (independent loads in
      // flight), applied in list order
      unsigned int c = 0;
      const unsigned int nsh = nov < kMaxContacts ? nov : kMaxContacts;  // in shared memory; the rest spilled
      for (; c + kPassB <= nsh; c += kPassB) {
        unsigned int jj[kPassB];
        Pd qq[kPassB];
#pragma unroll
        for (int u = 0; u < kPassB; ++u) jj[u] = ovl[(c + u) * ovl_stride];
#pragma unroll
        for (int u = 0; u < kPassB; ++u) qq[u] = fetch(jj[u]);
#pragma unroll
        for (int u = 0; u < kPassB; ++u) contact_q(jj[u], qq[u]);
      }
      for (; c < nsh; ++c) contact(ovl[c * ovl_stride]);
      for (; c < nov; ++c) contact(ovf[c - kMaxContacts]);
    } else if constexpr (F32) {  // more contacts than the list holds: re-walk (rare)
      walk(r, r * r, [&](unsigned int j, float df2, float qd, bool in) {
        const float hp = __fmaf_rn(0.5f, qd, hme);
        if (in && df2 < hp * hp * 1.0000005f) contact(j);
      });
    } else {
      walk(r, r * r, [&](unsigned int j, const Pd& q, double d2) {
        const double h = 0.5 * (me.d + q.d);
        if (d2 < h * h * (1.0 + 0x1.0p-50)) contact(j);
      });
    }
    wrote_partners = true;
    if ((fx * fx + fy * fy) + fz * fz > a.threshold2) {
      tx += fx * a.dt;
      ty += fy * a.dt;
      tz += fz * a.dt;
    }
  }
  // --- apply_pending (agent.hpp:115-133) -----------------------------------
  Pd np = me;
  const double disp = sqrt((tx * tx + ty * ty) + tz * tz);
  if (disp > 0.0) {
    if (disp > a.max_disp) {
      const double sc = a.max_disp / disp;
      tx *= sc;
      ty *= sc;
      tz *= sc;
    }
    np.x = me.x + tx;
    np.y = me.y + ty;
    np.z = me.z + tz;
    fl |= ABS_FLAG_MOVED;
    if (a.track_disp) dg.moved = __double2float_ru((disp < a.max_disp ? disp : a.max_disp) * (1.0 + 0x1.0p-40));
  }
  if (tg != 0.0) {
    const double nd = me.d + tg;
    np.d = nd > 1e-9 ? nd : 1e-9;
    if (tg > 0.0) fl |= ABS_FLAG_GREW;
  }
  {
    if (STATIC && a.iteration != 0) {
      nv[i] = 0;
      nn[i] = 0;
    }
    if (vol_changed) S.vol[i] = new_vol;
    if (rngc_changed) S.rngc[i] = new_rngc;
    if (wrote_partners) {
      if (RECORD) {
        S.force[i] = fx;
        S.force[cap + i] = fy;
        S.force[2 * cap + i] = fz;
      }
      S.partners[i] = contributors;
    }
    reinterpret_cast<double2*>(out + i)[0] = make_double2(np.x, np.y);
    reinterpret_cast<double2*>(out + i)[1] = make_double2(np.z, np.d);
    S.flags[i] = dg.dies ? static_cast<unsigned char>(fl | ABS_FLAG_REMOVED) : fl;
  }
  return dg;
}

// Daughter staging: warp-ballot compaction into the stage buffers
// (commit.cpp:186-222 appends; here slots are claimed with one atomic per warp).
__device__ __forceinline__ void stage_daughter(const Daughter& dg, DevGrid* gw,
                                               unsigned long long* __restrict__ st_parent,
                                               Pd* __restrict__ st_pd, double* __restrict__ st_vol,
                                               unsigned int* __restrict__ div_mark,
                                               unsigned int* __restrict__ st_tag) {
  const int lane = threadIdx.x & 31;
  const unsigned int ballot = __ballot_sync(0xffffffffu, dg.divides);
  if (!ballot) return;
  unsigned long long slot0 = 0;
  if (lane == 0) slot0 = atomicAdd(&gw->staged, (unsigned long long)__popc(ballot));
  slot0 = __shfl_sync(0xffffffffu, slot0, 0);
  if (dg.divides) {
    const unsigned long long slot = slot0 + __popc(ballot & ((1u << lane) - 1u));
    st_parent[slot] = dg.parent;
    reinterpret_cast<double2*>(st_pd + slot)[0] = make_double2(dg.x, dg.y);
    reinterpret_cast<double2*>(st_pd + slot)[1] = make_double2(dg.z, dg.d);
    st_vol[slot] = dg.vol;
    st_tag[slot] = dg.tag;
    ABS_ASSERT(dg.parent < gw->nkeys);
    div_mark[dg.parent] = 1u;
  }
}

__device__ __forceinline__ void flush_counters(unsigned long long n_eval, unsigned long long n_skip, DevGrid* gw) {
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    n_eval += __shfl_xor_sync(0xffffffffu, n_eval, off);
    n_skip += __shfl_xor_sync(0xffffffffu, n_skip, off);
  }
  if ((threadIdx.x & 31) == 0) {
    if (n_eval) atomicAdd(&gw->evals, n_eval);
    if (n_skip) atomicAdd(&gw->skips, n_skip);
  }
}

// Static detection pre-pass (simulation.cpp:375-384 + 465-468): an agent
// that is static this iteration and has no behaviour to run is settled here
// exactly as agent_step would settle it (flags = static, no force, no move,
// stale partners and last_force kept, marks cleared); ghosts likewise. The
// rest is listed (one atomic per warp) for the force sweep, so warps of
// config 3 (90 % static) run full instead of mostly idle.
__global__ void __launch_bounds__(kThreads) k_static_pass(Soa S, Pd* __restrict__ out, DevGrid* g,
                                                          unsigned char* __restrict__ nv,
                                                          unsigned char* __restrict__ nn, int model_on,
                                                          unsigned int* __restrict__ work) {
  if (g->err) return;
  const unsigned long long n = g->n;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  unsigned long long skips = 0;
  for (unsigned long long b = blockIdx.x * (unsigned long long)blockDim.x; b < n; b += stride) {
    const unsigned long long i = b + threadIdx.x;  // warp-uniform trip count
    bool listed = false;
    if (i < n) {
      const unsigned char fl = S.flags[i];
      const bool ghost = fl & kFlagGhost;
      const bool settle = ghost || ((!model_on || !S.beh[i]) &&
                                    !(fl & (ABS_FLAG_MOVED | ABS_FLAG_GREW | ABS_FLAG_NEWLY_ADDED |
                                            ABS_FLAG_NEIGHBOR_VIOLATION | ABS_FLAG_NEW_NEIGHBOR)) &&
                                    !nv[i] && !nn[i] && S.partners[i] <= 1u);
      if (settle) {
        const Pd me = load_pd(S.pd + i);
        reinterpret_cast<double2*>(out + i)[0] = make_double2(me.x, me.y);
        reinterpret_cast<double2*>(out + i)[1] = make_double2(me.z, me.d);
        nv[i] = 0;
        nn[i] = 0;
        if (!ghost) {
          S.flags[i] = ABS_FLAG_STATIC;
          ++skips;
        }
      } else {
        listed = true;
      }
    }
    const unsigned int ballot = __ballot_sync(0xffffffffu, listed);
    if (ballot) {
      unsigned long long base = 0;
      if (lane == 0) base = atomicAdd(&g->work_n, (unsigned long long)__popc(ballot));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (listed) work[base + __popc(ballot & ((1u << lane) - 1u))] = static_cast<unsigned int>(i);
    }
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) skips += __shfl_xor_sync(0xffffffffu, skips, off);
  if (lane == 0 && skips) atomicAdd(&g->skips, skips);
}

// Force sweep: one agent per thread, candidates fetched from HBM/L2.
// Resident CTAs per SM the register budget is sized for (c4 @ 2^24 sweep:
// fp32 walk 5 -> 6.27 ms vs 2 -> 6.96 ms; box mode c3 4 -> 0.68 vs 2 -> 0.77).
// WALK: 1 fp32-classified flat window walk (sub-binned grids; falls back to
// the box walk when the device grid has no sub-bins), 2 box-lockstep walk
// (bins == boxes, decided on the host).
template <int MODEL, bool STATIC, bool RECORD, int WALK>
__global__ void __launch_bounds__(kForceThreads, WALK >= 2 ? kForceMinBlocksBox : kForceMinBlocksF32)
    k_force(Soa S, const float4* __restrict__ pf, Pd* __restrict__ out, const DevGrid* gp, DevGrid* gw, const unsigned int* __restrict__ start,
            unsigned char* __restrict__ nv, unsigned char* __restrict__ nn, StepArgs a, unsigned long long cap,
            unsigned long long* __restrict__ st_parent, Pd* __restrict__ st_pd, double* __restrict__ st_vol,
            unsigned int* __restrict__ div_mark, unsigned int* __restrict__ st_tag,
            const unsigned int* __restrict__ work, unsigned int* __restrict__ rmark, KdView kd) {
  if (gp->err) return;
  __shared__ QGrid Q;
  extern __shared__ __align__(16) unsigned int force_smem[];
  constexpr bool F32 = WALK == 1;  // 2: box-lockstep walk, 3: kd-tree query (ABS_ENV_KD_TREE)
  auto wj0 = reinterpret_cast<unsigned int (*)[kForceThreads]>(force_smem);
  // fp32 walk: 16-bit stream bounds, so its contact lists start after 1.5 row arrays
  auto wb16 = reinterpret_cast<unsigned short (*)[kForceThreads]>(force_smem + kMaxRows * kForceThreads);
  auto ovl = reinterpret_cast<unsigned int (*)[kForceThreads]>(
      force_smem + (WALK >= 2 ? 0 : kMaxRows + kMaxRows / 2) * kForceThreads);
  if (threadIdx.x == 0) Q = make_qgrid(*gp);
  __syncthreads();
  if (MODEL == ABS_MODEL_COHERE && !a.brute && a.mp[0] * a.mp[0] > Q.box * Q.box * (1.0 + 1e-12)) {
    // uniform_grid.cpp:176-181: the query radius must not exceed the box
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      gw->err = kErrQueryRadius;
      gw->failed_iteration = a.iteration;
    }
    return;
  }
  // work != nullptr: only the agents k_static_pass listed (the rest were
  // settled there as static); otherwise every agent in storage order
  const unsigned long long n = work ? gp->work_n : gp->n;
  const double dmax = gp->dmax;
  // bins are the reference boxes
  const bool box_mode = WALK >= 2 || (Q.B[0] == 1 && Q.B[1] == 1 && Q.B[2] == 1);
  unsigned long long n_eval = 0, n_skip = 0;
  // Persistent warps sweep 32-agent chunks in a static warp-strided order:
  // the resident warps cover a contiguous window of the agent array (cell
  // order) that advances front to back, with no shared counter to contend on.
  const int lane = threadIdx.x & 31;
  float moved = 0.0f;
  const unsigned long long warps_total = (unsigned long long)gridDim.x * (blockDim.x >> 5);
  const unsigned long long warp_id = (unsigned long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  for (unsigned long long chunk = warp_id;; chunk += warps_total) {
    const unsigned long long base = chunk * 32ull;
    if (base >= n) break;
    const bool live = base + lane < n;
    const unsigned long long i = work ? (live ? work[base + lane] : 0ull) : base + lane;
    Daughter dg{false, false, 0, 0, 0, 0, 0, 0, 0u, 0.0f};
    if (live) {
      const Pd me = load_pd(S.pd + i);
      const unsigned int self = static_cast<unsigned int>(i);
      // behaviour-side exact radius query (models::Cohere)
      auto query = [&](double rq, double rq2, auto&& v) {
        for_each_neighbor(Q, S.pd, start, self, me.x, me.y, me.z, rq, rq2,
                          [&](unsigned int j, const Pd& q, double, double, double, double) { v(j, q); });
      };
      if (F32 && !box_mode) {
        dg = agent_step<MODEL, STATIC, RECORD, true>(
            S, out, i, me, dmax, nv, nn, a, cap, &ovl[0][threadIdx.x], kForceThreads, n_eval, n_skip,
            [&](double r, double r2, auto&& visit) {
              for_each_neighbor_flat32(Q, S.pd, pf, start, wj0, wb16, self, me.x, me.y, me.z, r, r2, visit);
            },
            [&](unsigned int j) { return load_pd(S.pd + j); }, [&](unsigned int j) { return S.uid[j]; }, Q.slack,
            query);
      } else
      dg = agent_step<MODEL, STATIC, RECORD>(
          S, out, i, me, dmax, nv, nn, a, cap, &ovl[0][threadIdx.x], kForceThreads, n_eval, n_skip,
          [&](double r, double r2, auto&& visit) {
            auto v6 = [&](unsigned int j, const Pd& q, double, double, double, double d2) { visit(j, q, d2); };
            if constexpr (WALK == 3) for_each_neighbor_kd(kd, S.pd, self, me.x, me.y, me.z, r, r2, v6);
            else for_each_neighbor_box(Q, S.pd, start, self, me.x, me.y, me.z, r2, v6);
          },
          [&](unsigned int j) { return load_pd(S.pd + j); }, [&](unsigned int j) { return S.uid[j]; }, 0.0f,
          query);
    }
    if (MODEL == ABS_MODEL_PROLIFERATION || MODEL == ABS_MODEL_GROW_DIVIDE || MODEL == ABS_MODEL_GROW_DIVIDE_DIE)
      stage_daughter(dg, gw, st_parent, st_pd, st_vol, div_mark, st_tag);
    if (MODEL == ABS_MODEL_GROW_DIVIDE_DIE) {  // removal staging: one atomic per warp
      ABS_ASSERT(!dg.dies || S.skey[i] < gp->nkeys);
      if (dg.dies) rmark[S.skey[i]] = 1u;
      const unsigned int dead = __ballot_sync(0xffffffffu, dg.dies);
      if (lane == 0 && dead) atomicAdd(&gw->removed_now, (unsigned long long)__popc(dead));
    }
    moved = fmaxf(moved, dg.moved);
  }
  if (a.track_disp) {  // the step's largest displacement (neighbour-list policy)
    const unsigned int mb = __reduce_max_sync(0xffffffffu, __float_as_uint(moved));
    if (lane == 0 && mb) atomicMax(&gw->step_disp, mb);
  }
  flush_counters(n_eval, n_skip, gw);
}

// ------------------------------------------------------------ neighbour lists
// Between two environment rebuilds the mechanical step reads per-agent
// candidate lists instead of walking the cell table. The
// reference's neighbour set of agent i is {j != i : d2 <= r_i^2} with
// r_i = 0.5 (d_i + dmax) (simulation.cpp:469, uniform_grid.cpp:172-230) and
// does not depend on the grid, so any superset of it tested with the
// reference's exact fp64 d2 <= r^2 visits exactly the same agents. A list
// built with radius r_i + skin stays such a superset while every agent has
// moved less than skin / 2 since the build (checked on the device by
// finalize_grid before every list step; a failed check re-runs the
// iteration as a rebuild).
//
// Candidates are classified in fp32 against float4 copies relative to the
// build origin (`pf`, rewritten by every list step) with the proven margin of
// for_each_neighbor_flat32 (slack from the build extent + skin); only the
// margin band reads the fp64 record. Possible contacts go to a per-lane
// shared-memory list and pairwise_repulsion runs on them afterwards with all
// lanes busy (the fp64 sqrt/division would otherwise run at ~8 of 32 lanes).
//
// k_list_build: after the re-bin, every agent's candidates within r + skin
// (fp32 superset, no 3x3x3 box clamp: r + skin may exceed the box) are staged
// per lane in shared memory and written out warp-blocked: entry k of agent i
// lives at list[(i / 32) * kmax * 32 + k * 32 + i % 32], so a warp's list is
// one contiguous kmax x 128 B block — the write-out and the list sweep's index
// loads are full-line, sequential accesses.
#ifndef ABS_LIST_MIN_BLOCKS
#define ABS_LIST_MIN_BLOCKS 4
#endif
// c4 @ 2^26 k_list_build: 64 staged (3 CTAs/SM) 28.1 ms, 56 / 48 / 44 (4 CTAs) 23.6 / 23.7 / 23.3,
// 32 (5 CTAs) 32.0, 16 (6 CTAs) 35.0: residency helps until the unstaged tail writes take over
#ifndef ABS_LIST_STAGE
#define ABS_LIST_STAGE 48
#endif
constexpr int kListStage = ABS_LIST_STAGE;  // candidates staged per lane before the coalesced write-out
// Streaming accesses of the list kernels (list / contact columns, the
// integration outputs) are marked evict-first so they do not push the
// gathered candidate records out of L2. ABS_CACHE_HINTS=0: plain accesses.
#ifndef ABS_CACHE_HINTS
#define ABS_CACHE_HINTS 1
#endif
#if ABS_CACHE_HINTS
#define ABS_LDS(p) __ldcs(p)
#define ABS_STS(p, v) __stcs((p), (v))
#else
#define ABS_LDS(p) __ldg(p)
#define ABS_STS(p, v) (*(p) = (v))
#endif
constexpr unsigned char kListOverflow = 255;  // count sentinel: the agent's candidates did not fit
constexpr int kListSmem = (kMaxRows + kMaxRows / 2 + kListStage) * kForceThreads * 4;

__global__ void __launch_bounds__(kForceThreads, ABS_LIST_MIN_BLOCKS)
    k_list_build(const float4* __restrict__ pf, DevGrid* g, const unsigned int* __restrict__ start,
                 unsigned int* __restrict__ list, unsigned char* __restrict__ cnt, unsigned int kmax, double skin) {
  if (g->err) return;
  __shared__ QGrid Q;
  extern __shared__ __align__(16) unsigned int force_smem[];
  auto wj0 = reinterpret_cast<unsigned int (*)[kForceThreads]>(force_smem);
  auto wb16 = reinterpret_cast<unsigned short (*)[kForceThreads]>(force_smem + kMaxRows * kForceThreads);
  auto stage = reinterpret_cast<unsigned int (*)[kForceThreads]>(force_smem + (kMaxRows + kMaxRows / 2) * kForceThreads);
  if (threadIdx.x == 0) Q = make_qgrid(*g);
  __syncthreads();
  const unsigned long long n = g->n;
  const double dmax = g->dmax;
  const int lane = threadIdx.x & 31;
  const unsigned int kst = kmax < kListStage ? kmax : kListStage;
  unsigned int most = 0;
  const unsigned long long warps_total = (unsigned long long)gridDim.x * (blockDim.x >> 5);
  const unsigned long long warp_id = (unsigned long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  for (unsigned long long chunk = warp_id;; chunk += warps_total) {
    const unsigned long long base = chunk * 32ull;
    if (base >= n) break;
    const unsigned long long i = base + lane;
    unsigned int c = 0;
    if (i < n) {
      const float4 me = __ldg(pf + i);
      // pf.w is the diameter rounded to fp32 (relative error 2^-24); the
      // 2e-6 inflation of rf covers it and the rounding of R
      const double R = 0.5 * (static_cast<double>(me.w) + dmax) + skin;
      const float rf = static_cast<float>(R) * 1.000002f + Q.slack + 1e-6f;
      unsigned int* col = list + (i >> 5) * (static_cast<unsigned long long>(kmax) * 32) + lane;
      for_each_candidate32(Q, pf, start, wj0, wb16, static_cast<unsigned int>(i), me.x, me.y, me.z, rf,
                           [&](unsigned int j) {
                             if (c < kst) stage[c][threadIdx.x] = j;
                             else if (c < kmax) col[c * 32] = j;
                             ++c;
                           });
      // more candidates than a list holds: the sentinel sends this agent to
      // the exact cell-table walk in this (rebuild) step, and the next
      // step's check rejects the lists so the host grows them
      cnt[i] = static_cast<unsigned char>(c <= kmax ? c : kListOverflow);
    }
    // coalesced write-out of the staged columns: entry k of the warp's 32 agents
    const unsigned int cs = c < kst ? c : kst;
    const unsigned int wmax = __reduce_max_sync(0xffffffffu, cs);
    unsigned int* wcol = list + (i >> 5) * (static_cast<unsigned long long>(kmax) * 32) + lane;
    for (unsigned int k = 0; k < wmax; ++k)
      if (k < cs) wcol[k * 32] = stage[k][threadIdx.x];
    most = c > most ? c : most;
  }
  most = __reduce_max_sync(0xffffffffu, most);
  if (lane == 0 && most) {
    atomicMax(&g->list_need, most);
    if (most > kmax) g->list_incomplete = 1u;
  }
}

// The list step is two kernels, so the latency-bound candidate scan keeps
// many warps resident (it holds no fp64 force state):
// k_list_scan: every listed j through the reference's exact d2 <= r^2 (fp32
// outside the margin band, fp64 inside it) — a force evaluation — and the
// possible contacts into a warp-blocked per-agent contact list;
// k_list_forces: pairwise_repulsion (mechanics.cpp:10-27) on the contacts,
// the force sum, apply_pending (agent.hpp:115-133) and the step's largest
// displacement (folded into g->step_disp for the next coverage check).
// Positions are read from `pin`/`pfin` and written to `pout`/`pfout`.
#ifndef ABS_LIST_SCAN_MIN_BLOCKS
#define ABS_LIST_SCAN_MIN_BLOCKS 4
#endif
// Contacts recorded per agent (more: the force pass re-scans the agent's
// list, one lane, ~25 us of serial loads — at 16, ~1 % of c1's agents (mean 9
// contacts) did, and their warps were the whole kernel's tail: k_list_forces
// 35 us for 131,072 agents with the SMs 39 % active).
constexpr int kListContacts = 24;
constexpr unsigned char kContactOverflow = 255;  // contact count sentinel

// Exact cell-table walk of one agent whose candidates did not fit its list
// (rebuild step only): evaluations << 32 | possible contacts, recorded in ct.
// Out of line: rare, and its fp64 state would cap the scan's occupancy.
__device__ __noinline__ unsigned long long scan_walk(const QGrid& Q, const Pd* __restrict__ pin,
                                                     const unsigned int* __restrict__ start, unsigned int i,
                                                     double r, unsigned int* ct) {
  const Pd me = load_pd(pin + i);
  unsigned int evals = 0, nov = 0;
  for_each_neighbor(Q, pin, start, i, me.x, me.y, me.z, r, r * r,
                    [&](unsigned int j, const Pd& q, double, double, double, double d2) {
                      ++evals;
                      const double h = 0.5 * (me.d + q.d);
                      if (d2 < h * h * (1.0 + 0x1.0p-50)) {
                        if (nov < kListContacts) ct[nov * 32] = j;
                        ++nov;
                      }
                    });
  return (static_cast<unsigned long long>(evals) << 32) | nov;
}

// c4 @ 2^26 k_list_scan (batch, CTAs/SM): (4,4) 7.57 ms, (5,4) 7.25, (6,4) 7.33, (8,3) 7.69, (2,6) 10.1, (6,5) 11.1
#ifndef ABS_SCAN_BATCH
#define ABS_SCAN_BATCH 5
#endif
constexpr int kScanBatch = ABS_SCAN_BATCH;  // candidates in flight per lane
// c4 @ 2^26 k_list_forces (batch, CTAs/SM): (2,3) 8.17 ms, (4,3) 8.31, (4,2) 9.9, (3,4) 7.30, (2,4) 6.78, (2,5) 7.79, (1,6) 10.3
#ifndef ABS_LF_MIN_BLOCKS
#define ABS_LF_MIN_BLOCKS 4
#endif
#ifndef ABS_LF_BATCH
#define ABS_LF_BATCH 2
#endif
constexpr int kLfBatch = ABS_LF_BATCH;  // contact records in flight per lane

__global__ void __launch_bounds__(kThreads, ABS_LIST_SCAN_MIN_BLOCKS)
    k_list_scan(const Pd* __restrict__ pin, const float4* __restrict__ pfin, DevGrid* g,
                const unsigned int* __restrict__ list, const unsigned char* __restrict__ cnt, unsigned int kmax,
                unsigned int* __restrict__ contacts, unsigned char* __restrict__ ncontacts,
                unsigned int* __restrict__ evc, const unsigned int* __restrict__ start) {
  if (g->err) return;
  __shared__ QGrid Q;  // the build's grid: only read for overflow agents, in the rebuild step itself
  if (threadIdx.x == 0) Q = make_qgrid(*g);
  __syncthreads();
  const unsigned long long n = g->n;
  const double dmax = g->dmax;
  const float slack = g->lslack;
  const double sl = static_cast<double>(slack);
  const int lane = threadIdx.x & 31;
  unsigned long long n_eval = 0;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  // warp-uniform sweep: every lane of a warp stays in the loops below, so the
  // band branch and the candidate loop bound are warp-wide decisions
  for (unsigned long long b0 = blockIdx.x * (unsigned long long)blockDim.x + (threadIdx.x & ~31u); b0 < n;
       b0 += stride) {
    const unsigned long long i = b0 + lane;
    const bool live = i < n;
    const unsigned int c = live ? cnt[i] : 0u;
    const float4 mf = __ldg(pfin + (live ? i : b0));
    const double d = live ? pin[i].d : 1.0;
    const double r = 0.5 * (d + dmax);
    const double r2 = r * r;
    const double rin = r - sl;
    const float rin2 = rin > 0.0 ? __double2float_rd(rin * rin * (1.0 - 0x1.0p-40)) : -1.0f;
    const float rout2 = __double2float_ru((r + sl) * (r + sl) * (1.0 + 0x1.0p-40));
    const float hme = 0.5f * mf.w + slack;
    const unsigned long long wbase = (b0 >> 5) * (static_cast<unsigned long long>(kmax) * 32) + lane;
    unsigned int* ct = contacts + (b0 >> 5) * (kListContacts * 32) + lane;
    unsigned int evals = 0, nov = 0;
    const bool walk = c == kListOverflow;  // candidates did not fit: exact cell-table walk (rebuild step only)
    const unsigned int cl = walk ? 0u : c;
    const unsigned int cmax = __reduce_max_sync(0xffffffffu, cl);
    if (__any_sync(0xffffffffu, walk) && walk) {
      const unsigned long long en = scan_walk(Q, pin, start, static_cast<unsigned int>(i), r, ct);
      evals = static_cast<unsigned int>(en >> 32);
      nov = static_cast<unsigned int>(en);
    }
    const unsigned int* col = list + wbase;
    unsigned int nj[kScanBatch];
#pragma unroll
    for (int u = 0; u < kScanBatch; ++u) nj[u] = u < static_cast<int>(cl) ? ABS_LDS(col + u * 32) : 0u;
    for (unsigned int s = 0; s < cmax; s += kScanBatch) {
      unsigned int jj[kScanBatch];
#pragma unroll
      for (int u = 0; u < kScanBatch; ++u) jj[u] = nj[u];
      float4 qf[kScanBatch];
#pragma unroll
      for (int u = 0; u < kScanBatch; ++u) qf[u] = __ldg(pfin + jj[u]);
      col += kScanBatch * 32;
#pragma unroll
      for (int u = 0; u < kScanBatch; ++u) nj[u] = s + kScanBatch + u < cl ? ABS_LDS(col + u * 32) : 0u;
      float df2[kScanBatch];
      unsigned int in = 0, band = 0;
#pragma unroll
      for (int u = 0; u < kScanBatch; ++u) {
        const float ex = mf.x - qf[u].x, ey = mf.y - qf[u].y, ez = mf.z - qf[u].z;
        df2[u] = __fmaf_rn(ex, ex, __fmaf_rn(ey, ey, ez * ez));
        const bool v = s + u < cl && df2[u] <= rout2;
        in |= v ? (1u << u) : 0u;
        band |= (v && df2[u] > rin2) ? (1u << u) : 0u;
      }
      if (__any_sync(0xffffffffu, band != 0u) && band) {  // margin band: the reference's exact fp64 test
        const Pd me = load_pd(pin + i);
#pragma unroll
        for (int u = 0; u < kScanBatch; ++u) {
          if (band & (1u << u)) {
            const Pd q = load_pd(pin + jj[u]);
            const double dx = me.x - q.x, dy = me.y - q.y, dz = me.z - q.z;
            if (!((dx * dx + dy * dy) + dz * dz <= r2)) in &= ~(1u << u);
          }
        }
      }
      evals += __popc(in);
#pragma unroll
      for (int u = 0; u < kScanBatch; ++u) {
        // contact superset: df2 < (0.5 (d_i + d_j) + slack)^2 (1 + 5e-7)
        const float hp = __fmaf_rn(0.5f, qf[u].w, hme);
        if ((in & (1u << u)) && df2[u] < hp * hp * 1.0000005f) {
          if (nov < kListContacts) ABS_STS(ct + nov * 32, jj[u]);
          ++nov;
        }
      }
    }
    if (!live) continue;
    n_eval += evals;
    if (evc) evc[i] = evals;
    ncontacts[i] = nov <= kListContacts ? static_cast<unsigned char>(nov) : kContactOverflow;
  }
  flush_counters(n_eval, 0ull, g);
}

template <bool RECORD>
__global__ void __launch_bounds__(kThreads, ABS_LF_MIN_BLOCKS)
    k_list_forces(const Pd* __restrict__ pin, Pd* __restrict__ pout, float4* __restrict__ pfout, Soa S, DevGrid* g,
                  const unsigned int* __restrict__ list, const unsigned char* __restrict__ cnt, unsigned int kmax,
                  const unsigned int* __restrict__ contacts, const unsigned char* __restrict__ ncontacts,
                  StepArgs a, unsigned long long cap, const unsigned int* __restrict__ start) {
  if (g->err) return;
  __shared__ QGrid Q;
  if (threadIdx.x == 0) Q = make_qgrid(*g);
  __syncthreads();
  const unsigned long long n = g->n;
  const double dmax = g->dmax;
  const double k = a.k;
  const double lox = g->lorigin[0], loy = g->lorigin[1], loz = g->lorigin[2];
  float moved = 0.0f;
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const Pd me = load_pd(pin + i);
    const unsigned int nc = ncontacts[i];
    unsigned int contributors = 0;
    double fx = 0.0, fy = 0.0, fz = 0.0;
    auto contact_q = [&](unsigned int j, const Pd& q) {
      const double dx = me.x - q.x, dy = me.y - q.y, dz = me.z - q.z;
      // pairwise_repulsion (mechanics.cpp:10-27)
      const double dist = sqrt((dx * dx + dy * dy) + dz * dz);
      const double overlap = 0.5 * (me.d + q.d) - dist;
      if (overlap <= 0.0) return;
      double f0, f1, f2;
      if (dist > 0.0) {
        const double sc = k * overlap / dist;
        f0 = dx * sc;
        f1 = dy * sc;
        f2 = dz * sc;
      } else {
        coincident_force(S.uid[i], S.uid[j], k * overlap, &f0, &f1, &f2);
      }
      if ((f0 * f0 + f1 * f1) + f2 * f2 > 0.0) {
        ++contributors;
        fx += f0;
        fy += f1;
        fz += f2;
      }
    };
    if (nc != kContactOverflow) {
      const unsigned int* ct = contacts + (i >> 5) * (kListContacts * 32) + (i & 31);
      unsigned int q = 0;
      for (; q + kLfBatch <= nc; q += kLfBatch) {  // kLfBatch records in flight
        unsigned int jb[kLfBatch];
        Pd qb[kLfBatch];
#pragma unroll
        for (int u = 0; u < kLfBatch; ++u) jb[u] = ABS_LDS(ct + (q + u) * 32);
#pragma unroll
        for (int u = 0; u < kLfBatch; ++u) qb[u] = load_pd(pin + jb[u]);
#pragma unroll
        for (int u = 0; u < kLfBatch; ++u) contact_q(jb[u], qb[u]);
      }
      for (; q < nc; ++q) {
        const unsigned int j0 = ABS_LDS(ct + q * 32);
        contact_q(j0, load_pd(pin + j0));
      }
    } else {  // more possible contacts than recorded: the list (or the rebuild step's walk) again
      const double r = 0.5 * (me.d + dmax);
      const double r2 = r * r;
      const unsigned int c = cnt[i];
      if (c == kListOverflow) {
        for_each_neighbor(Q, pin, start, static_cast<unsigned int>(i), me.x, me.y, me.z, r, r2,
                          [&](unsigned int j, const Pd& q, double, double, double, double d2) {
                            const double h = 0.5 * (me.d + q.d);
                            if (d2 < h * h * (1.0 + 0x1.0p-50)) contact_q(j, q);
                          });
      } else {
        const unsigned int* col = list + (i >> 5) * (static_cast<unsigned long long>(kmax) * 32) + (i & 31);
        for (unsigned int s2 = 0; s2 < c; s2 += 4) {  // four records in flight
          unsigned int jb[4];
          Pd qb[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) jb[u] = __ldg(col + static_cast<unsigned long long>(min(s2 + u, c - 1)) * 32);
#pragma unroll
          for (int u = 0; u < 4; ++u) qb[u] = load_pd(pin + jb[u]);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (s2 + u >= c) break;
            const Pd& q = qb[u];
            const double dx = me.x - q.x, dy = me.y - q.y, dz = me.z - q.z;
            const double d2 = (dx * dx + dy * dy) + dz * dz;
            const double h = 0.5 * (me.d + q.d);
            if (d2 <= r2 && d2 < h * h * (1.0 + 0x1.0p-50)) contact_q(jb[u], q);
          }
        }
      }
    }
    double tx = 0.0, ty = 0.0, tz = 0.0;
    if ((fx * fx + fy * fy) + fz * fz > a.threshold2) {
      tx = fx * a.dt;
      ty = fy * a.dt;
      tz = fz * a.dt;
    }
    Pd np = me;
    const double disp = sqrt((tx * tx + ty * ty) + tz * tz);
    if (disp > 0.0) {
      double md = disp;
      if (disp > a.max_disp) {
        const double sc = a.max_disp / disp;
        tx *= sc;
        ty *= sc;
        tz *= sc;
        md = a.max_disp;
      }
      np.x = me.x + tx;
      np.y = me.y + ty;
      np.z = me.z + tz;
      const unsigned char fl = S.flags[i];
      if (!(fl & ABS_FLAG_MOVED)) S.flags[i] = fl | ABS_FLAG_MOVED;
      moved = fmaxf(moved, __double2float_ru(md * (1.0 + 0x1.0p-40)));
    }
    if (RECORD) {
      S.force[i] = fx;
      S.force[cap + i] = fy;
      S.force[2 * cap + i] = fz;
    }
    ABS_STS(S.partners + i, contributors);
    ABS_STS(reinterpret_cast<double2*>(pout + i), make_double2(np.x, np.y));
    ABS_STS(reinterpret_cast<double2*>(pout + i) + 1, make_double2(np.z, np.d));
    ABS_STS(pfout + i, make_float4(static_cast<float>(np.x - lox), static_cast<float>(np.y - loy),
                                   static_cast<float>(np.z - loz), static_cast<float>(np.d)));
  }
  // one same-address atomic per block, not per warp
  __shared__ unsigned int smoved[kThreads / 32];
  const unsigned int mb = __reduce_max_sync(0xffffffffu, __float_as_uint(moved));
  if ((threadIdx.x & 31) == 0) smoved[threadIdx.x >> 5] = mb;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int m = 0;
    for (int q = 0; q < kThreads / 32; ++q) m = max(m, smoved[q]);
    if (m) atomicMax(&g->step_disp, m);
  }
}

// ------------------------------------------------------------ config 5: SIR
// absim_models.h: from start-of-iteration states, S -> I with probability
// 1 - (1-p)^k (k infected neighbours within r, minimum image on the periodic
// cube), I -> R after `recovery` iterations, then a unit random-walk step
// wrapped into [0, L). Bins are the periodic boxes (box = L / floor(L / r) >= r),
// so the 27 wrapped neighbour boxes hold every candidate.
__global__ void __launch_bounds__(kThreads) k_sir(Soa S, Pd* __restrict__ out, const DevGrid* g,
                                                  const unsigned int* __restrict__ start,
                                                  unsigned char* __restrict__ next_state,
                                                  unsigned int* __restrict__ next_t, StepArgs a) {
  if (g->err) return;
  const unsigned long long n = g->n;
  const double L = a.mp[0], r = a.mp[1], step = a.mp[2], prob = a.mp[4];
  const unsigned long long rec = static_cast<unsigned long long>(a.mp[3]);
  const double box = g->box, r2 = r * r;
  const unsigned int D0 = g->dims[0], D1 = g->dims[1], D2 = g->dims[2], ysh = g->ysh;
  __shared__ unsigned int woff[18][kThreads];
  __shared__ unsigned short wbnd[18][kThreads];
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const Pd me = load_pd(S.pd + i);
    unsigned char st = S.beh[i];
    unsigned int ti = S.partners[i];
    if (S.flags[i] & kFlagGhost) {  // another rank's agent: start-of-step state, candidate only
      reinterpret_cast<double2*>(out + i)[0] = make_double2(me.x, me.y);
      reinterpret_cast<double2*>(out + i)[1] = make_double2(me.z, me.d);
      next_state[i] = st;
      next_t[i] = ti;
      continue;
    }
    if (st == ABS_SIR_I && a.iteration - ti >= rec) st = ABS_SIR_R;
    if (st == ABS_SIR_S) {
      const unsigned int cx = box_coord(me.x, 0.0, box, D0), cy = box_coord(me.y, 0.0, box, D1),
                         cz = box_coord(me.z, 0.0, box, D2);
      unsigned int k = 0;
      // The 27 wrapped boxes as x-contiguous windows: one per (y, z) row, or
      // two where the x range wraps (dims >= 3, so the three boxes differ).
      // All 18 cell-table reads are issued before any candidate is touched.
      auto wrap = [](int v, int d) { return v < 0 ? v + d : (v >= d ? v - d : v); };
      const int xa = static_cast<int>(cx) - 1, xb = static_cast<int>(cx) + 2;  // [xa, xb)
      const bool split = xa < 0 || xb > static_cast<int>(D0);
      // first window [x0a, x1a), second [x0b, x1b) (empty unless split)
      const unsigned int x0a = split ? (xa < 0 ? 0u : static_cast<unsigned int>(xa)) : static_cast<unsigned int>(xa);
      const unsigned int x1a = split ? (xa < 0 ? static_cast<unsigned int>(xb) : D0) : static_cast<unsigned int>(xb);
      const unsigned int x0b = split ? (xa < 0 ? D0 - 1u : 0u) : 0u;
      const unsigned int x1b = split ? (xa < 0 ? D0 : static_cast<unsigned int>(xb) - D0) : 0u;
      unsigned int lo[18], hi[18];
#pragma unroll
      for (int q = 0; q < 9; ++q) {
        const unsigned int bz = static_cast<unsigned int>(wrap(static_cast<int>(cz) + q / 3 - 1, static_cast<int>(D2)));
        const unsigned int by = static_cast<unsigned int>(wrap(static_cast<int>(cy) + q % 3 - 1, static_cast<int>(D1)));
        const unsigned int row = D0 * row_of(by, bz, ysh, D2);
        lo[2 * q] = __ldg(start + row + x0a);
        hi[2 * q] = __ldg(start + row + x1a);
        lo[2 * q + 1] = split ? __ldg(start + row + x0b) : 0u;
        hi[2 * q + 1] = split ? __ldg(start + row + x1b) : 0u;
      }
      auto infected_within = [&](unsigned int j) {
        const Pd q = load_pd(S.pd + j);
        const double ex = abs_min_image(me.x - q.x, L), ey = abs_min_image(me.y - q.y, L),
                     ez = abs_min_image(me.z - q.z, L);
        return (ex * ex + ey * ey) + ez * ez <= r2;
      };
      // The non-empty windows become ONE candidate stream per lane (offset,
      // cumulative bound in shared memory), walked four states at a time: a
      // warp then runs for its longest stream, not for the sum over windows of
      // the longest window (the nested loop ran at 16 of 32 lanes active).
      unsigned int total = 0;
      int nw = 0;
#pragma unroll
      for (int w = 0; w < 18; ++w) {
        if (hi[w] > lo[w]) {
          woff[nw][threadIdx.x] = lo[w] - total;
          total += hi[w] - lo[w];
          wbnd[nw][threadIdx.x] = static_cast<unsigned short>(total);
          ++nw;
        }
      }
      if (total > 0xFFFFu) {  // stream bounds would not fit 16 bits: nested walk
#pragma unroll
        for (int w = 0; w < 18; ++w)
          for (unsigned int j = lo[w]; j < hi[w]; ++j)
            if (j != i && S.beh[j] == ABS_SIR_I && infected_within(j)) ++k;
      } else if (nw > 0) {
        int wk = 0;
        unsigned int off = woff[0][threadIdx.x], bnd = wbnd[0][threadIdx.x];
        for (unsigned int p = 0; p < total;) {
          unsigned int idx[4];
          bool val[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            val[u] = p < total;
            idx[u] = val[u] ? p + off : static_cast<unsigned int>(i);
            ++p;
            if (p == bnd) {
              wk = min(wk + 1, nw - 1);
              off = woff[wk][threadIdx.x];
              bnd = wbnd[wk][threadIdx.x];
            }
          }
          unsigned char sj[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) sj[u] = S.beh[idx[u]];
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (val[u] && idx[u] != i && sj[u] == ABS_SIR_I && infected_within(idx[u])) ++k;
        }
      }
      if (k > 0 && abs_rng_word(a.seed, S.uid[i], ABS_RNG_SIR_INFECT(a.iteration)) < abs_sir_threshold(prob, k)) {
        st = ABS_SIR_I;
        ti = static_cast<unsigned int>(a.iteration);
      }
    }
    double dir[3];
    abs_unit_vector(a.seed, S.uid[i], ABS_RNG_SIR_WALK(a.iteration), dir);
    reinterpret_cast<double2*>(out + i)[0] =
        make_double2(abs_wrap(me.x + dir[0] * step, L), abs_wrap(me.y + dir[1] * step, L));
    reinterpret_cast<double2*>(out + i)[1] = make_double2(abs_wrap(me.z + dir[2] * step, L), me.d);
    next_state[i] = st;
    next_t[i] = ti;
  }
}

__global__ void __launch_bounds__(kThreads) k_sir_commit(Soa S, DevGrid* g,
                                                         const unsigned char* __restrict__ next_state,
                                                         const unsigned int* __restrict__ next_t) {
  if (g->err) return;
  const unsigned long long n = g->n;
  unsigned long long c[3] = {0, 0, 0};
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned char st = next_state[i];
    S.beh[i] = st;
    S.partners[i] = next_t[i];
    if (S.flags[i] & kFlagGhost) continue;  // counted by its owner
    c[0] += st == ABS_SIR_S;
    c[1] += st == ABS_SIR_I;
    c[2] += st == ABS_SIR_R;
  }
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    for (int off = 16; off; off >>= 1) c[q] += __shfl_xor_sync(0xffffffffu, c[q], off);
    if ((threadIdx.x & 31) == 0 && c[q]) atomicAdd(&g->sir[q], c[q]);
  }
}

// ------------------------------------------------------------ commit
// mark_new_agent_neighbors (simulation.cpp:510-530): each staged daughter
// flags new_neighbor on agents of the START-OF-STEP grid (reference boxes,
// reference cull) using their CURRENT positions; no query exclusion.
__global__ void k_mark_new(Soa S, const Pd* __restrict__ live, const DevGrid* g,
                           const unsigned int* __restrict__ start, const Pd* __restrict__ st_pd) {
  if (g->err) return;
  const DevGrid G = *g;
  const unsigned long long staged = G.staged, n = G.n;
  for (unsigned long long k = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; k < staged;
       k += (unsigned long long)gridDim.x * blockDim.x) {
    const Pd c = load_pd(st_pd + k);
    const double r = 0.5 * (c.d + G.dmax);
    const double r2 = r * r;
    if (r <= G.box) {
      const double radius = sqrt(r2);
      const double cc[3] = {c.x, c.y, c.z};
      long long lo[3], hi[3];
      for (int q = 0; q < 3; ++q) {
        const long long a = static_cast<long long>(floor((cc[q] - radius - G.origin[q]) / G.box));
        const long long b = static_cast<long long>(floor((cc[q] + radius - G.origin[q]) / G.box));
        lo[q] = a > 0 ? a : 0;
        hi[q] = b < (long long)G.dims[q] - 1 ? b : (long long)G.dims[q] - 1;
      }
      const double cull = r2 * (1.0 + 1e-12);
      for (long long z = lo[2]; z <= hi[2]; ++z)
        for (long long y = lo[1]; y <= hi[1]; ++y)
          for (long long x = lo[0]; x <= hi[0]; ++x) {
            double min_d2 = 0.0;
            const long long at[3] = {x, y, z};
            for (int q = 0; q < 3; ++q) {
              const double b0 = G.origin[q] + static_cast<double>(at[q]) * G.box;
              const double b1 = b0 + G.box;
              const double gap = cc[q] < b0 ? b0 - cc[q] : (cc[q] > b1 ? cc[q] - b1 : 0.0);
              min_d2 += gap * gap;
            }
            if (min_d2 > cull) continue;
            // the box's sub-bins: B x B rows of B contiguous bins
            for (unsigned int sz = 0; sz < G.B[2]; ++sz)
              for (unsigned int sy = 0; sy < G.B[1]; ++sy) {
                const unsigned int bz = (unsigned int)z * G.B[2] + sz, by = (unsigned int)y * G.B[1] + sy;
                const unsigned int row = G.bd[0] * row_of(by, bz, G.ysh, G.bd[2]) + (unsigned int)x * G.B[0];
                for (unsigned int j = start[row]; j < start[row + G.B[0]]; ++j) {
                  const Pd q = load_pd(live + j);
                  const double dx = c.x - q.x, dy = c.y - q.y, dz = c.z - q.z;
                  if ((dx * dx + dy * dy) + dz * dz <= r2) S.flags[j] |= ABS_FLAG_NEW_NEIGHBOR;
                }
              }
          }
    } else {
      for (unsigned long long j = 0; j < n; ++j) {
        const Pd q = load_pd(live + j);
        const double dx = c.x - q.x, dy = c.y - q.y, dz = c.z - q.z;
        if ((dx * dx + dy * dy) + dz * dz <= r2) S.flags[j] |= ABS_FLAG_NEW_NEIGHBOR;
      }
    }
  }
}

// Daughters get uid = uid_count + rank of the parent among this iteration's
// dividers in parent-uid order (= the reference's one-worker storage order
// while storage order equals uid order, resource_manager.hpp:44-46), and are
// appended at n + rank (commit.cpp:196-220: appends never move survivors).
__global__ void k_append(Soa S, Pd* __restrict__ live, const DevGrid* g,
                         const unsigned long long* __restrict__ st_parent,
                         const Pd* __restrict__ st_pd, const double* __restrict__ st_vol,
                         const unsigned int* __restrict__ st_tag,
                         const unsigned int* __restrict__ div_rank, const unsigned int* __restrict__ div_rank_g,
                         unsigned long long cap, int record_forces) {
  if (g->err) return;
  const unsigned long long staged = g->staged, n = g->n, uc = g->uid_count, nk = g->nkeys;
  for (unsigned long long k = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; k < staged;
       k += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long parent = st_parent[k];
    const unsigned long long j = n + div_rank[parent];  // local append slot
    ABS_ASSERT(j < cap);
    const unsigned int rk = div_rank_g[parent];         // rank among all dividers
    const Pd p = st_pd[k];
    reinterpret_cast<double2*>(live + j)[0] = make_double2(p.x, p.y);
    reinterpret_cast<double2*>(live + j)[1] = make_double2(p.z, p.d);
    S.uid[j] = uc + rk;
    S.skey[j] = static_cast<unsigned int>(nk + rk);  // appended after the reference's survivors, creation order
    S.flags[j] = ABS_FLAG_NEWLY_ADDED;
    S.partners[j] = 0;
    S.beh[j] = 1;
    S.vol[j] = st_vol[k];
    S.tag[j] = st_tag[k];
    S.rngc[j] = 0;  // a new Agent's stream starts at counter 0
    if (record_forces) S.force[j] = S.force[cap + j] = S.force[2 * cap + j] = 0.0;
  }
}

// grank: the scanned (global) division marks; grank[uid_count] is the total
// number of daughters created this iteration over all ranks.
__global__ void k_commit_fin(DevGrid* g, const unsigned int* __restrict__ grank) {
  if (threadIdx.x || blockIdx.x || g->err) return;
  const unsigned long long s = g->staged;
  g->n += s;
  g->nkeys += grank[g->uid_count];
  g->uid_count += grank[g->uid_count];
  g->added += s;
  g->staged = 0;
}

// After the commit: zero the scanned marks, indices [0, uid_count] (the
// grown uid_count covers the old range and the old total slot).
__global__ void k_zero_marks(unsigned int* __restrict__ m, const DevGrid* g) {
  if (g->err) return;
  const unsigned long long len = g->uid_count + 1;
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < len;
       i += (unsigned long long)gridDim.x * blockDim.x)
    m[i] = 0;
}

// ------------------------------------------------------------ ingest
// Population upload (Simulation::add_agent, simulation.cpp:131-141): build the
// interleaved {x,y,z,d} records from SoA device arrays, validate diameters
// (Agent ctor throws unless d > 0, agent.hpp:25) and default the per-agent
// state. Host arrays reach these inputs by contiguous H2D copies.
// Population upload. Also produces, per block, the sum and max of the
// diameters in a fixed order (thread grid-stride sums, then a fixed tree), so
// the host's auto-bin decision is deterministic for a given grid, and checks
// uids against the caller's uid_count (uid_limit > 0). bad_input: bit 0 a
// diameter <= 0, bit 1 a uid >= uid_count.
__global__ void __launch_bounds__(kThreads) k_ingest(const double* __restrict__ x, const double* __restrict__ y,
                                                     const double* __restrict__ z, const double* __restrict__ d,
                                                     const unsigned char* __restrict__ mask, unsigned long long n,
                                                     int set_uid, int set_vol, int model_on, Pd* __restrict__ out,
                                                     Soa S, DevGrid* g, int sir, unsigned long long seed,
                                                     double* __restrict__ part, unsigned long long uid_limit) {
  unsigned int bad = 0;
  double sum = 0.0, mx = 0.0;
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const double di = d[i];
    bad |= !(di > 0.0);
    sum += di;
    mx = di > mx ? di : mx;
    reinterpret_cast<double2*>(out + i)[0] = make_double2(x[i], y[i]);
    reinterpret_cast<double2*>(out + i)[1] = make_double2(z[i], di);
    if (set_uid) S.uid[i] = i;
    else if (uid_limit && S.uid[i] >= uid_limit) bad |= 2u;
    S.tag[i] = 0;   // set with abs_gpu_set_agent_ext
    S.rngc[i] = 0;
    S.skey[i] = static_cast<unsigned int>(i);  // storage order of the reference = upload order
    if (set_vol) S.vol[i] = abs_volume_of_diameter(di);
    if (sir) {  // absim_models.h: 1 % initially infected, from the seed (or given states)
      const unsigned long long u = set_uid ? i : S.uid[i];
      S.beh[i] = mask ? mask[i] : (abs_u01(abs_rng_word(seed, u, ABS_RNG_SIR_INIT)) < 0.01 ? ABS_SIR_I : ABS_SIR_S);
    } else {
      S.beh[i] = (model_on && (!mask || mask[i])) ? 1 : 0;
    }
  }
  const unsigned int anybad = __reduce_or_sync(0xffffffffu, bad);
  if (anybad && (threadIdx.x & 31) == 0) atomicOr(&g->bad_input, anybad);
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    sum += __shfl_xor_sync(0xffffffffu, sum, off);
    const double m = __shfl_xor_sync(0xffffffffu, mx, off);
    mx = m > mx ? m : mx;
  }
  __shared__ double ws[kThreads / 32][2];
  if ((threadIdx.x & 31) == 0) {
    ws[threadIdx.x >> 5][0] = sum;
    ws[threadIdx.x >> 5][1] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s2 = 0.0, m2 = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) {
      s2 += ws[w][0];
      m2 = ws[w][1] > m2 ? ws[w][1] : m2;
    }
    part[2 * blockIdx.x] = s2;
    part[2 * blockIdx.x + 1] = m2;
  }
}

// Positions/diameters of the current state as four contiguous fp64 arrays
// (x | y | z | d) for direct device-to-host copies into caller arrays.
__global__ void k_split_pd(const Pd* __restrict__ pos, const DevGrid* g, double* __restrict__ out,
                           unsigned long long stride) {
  const unsigned long long n = g->n;
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const Pd p = load_pd(pos + i);
    out[i] = p.x;
    out[stride + i] = p.y;
    out[2 * stride + i] = p.z;
    out[3 * stride + i] = p.d;
  }
}

__global__ void k_mask_flags(const unsigned char* __restrict__ in, unsigned char* __restrict__ out,
                             const DevGrid* g) {
  const unsigned long long n = g->n;
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x)
    out[i] = in[i] & (63u | ABS_FLAG_GHOST);
}

// Host-visible mirror of the device grid record: one warp copies it into
// mapped page-locked memory, so reading it back never queues behind bulk
// DMA on the copy engines (abs_gpu_run_frames overlaps those with compute).
__global__ void k_grid_out(const DevGrid* __restrict__ g, DevGrid* out) {
  const unsigned long long* s = reinterpret_cast<const unsigned long long*>(g);
  unsigned long long* d = reinterpret_cast<unsigned long long*>(out);
  for (unsigned int w = threadIdx.x; w < sizeof(DevGrid) / 8; w += blockDim.x) d[w] = s[w];
}

// Population reset at upload: everything before ov_on as a fresh record with
// the reduction identities (the host-built DevGrid of the synchronous path).
__global__ void k_grid_reset(DevGrid* g, unsigned long long n, unsigned long long uid_count) {
  unsigned long long* w = reinterpret_cast<unsigned long long*>(g);
  for (unsigned int q = threadIdx.x; q < offsetof(DevGrid, ov_on) / 8; q += blockDim.x) w[q] = 0ull;
  __syncthreads();
  if (threadIdx.x == 0) {
    g->red[0] = g->red[1] = g->red[2] = kInfOrdLo;
    g->red[3] = g->red[4] = g->red[5] = kInfOrdHi;
    g->red[6] = kZeroOrd;
    g->dims[0] = g->dims[1] = g->dims[2] = 1;
    g->B[0] = g->B[1] = g->B[2] = 1;
    g->n = n;
    g->nkeys = n;
    g->uid_count = uid_count;
  }
}
static_assert(offsetof(DevGrid, ov_on) % 8 == 0 && sizeof(DevGrid) % 8 == 0, "grid record layout");

__global__ void k_set_u64(unsigned long long* p, unsigned long long v) { *p = v; }
__global__ void k_reset_reduction(DevGrid* g) { reset_reduction(g); }

// Zero `bytes` bytes on the compute engine (16-byte stores + tail).
__global__ void k_zero_bytes(unsigned char* __restrict__ p, unsigned long long bytes) {
  const unsigned long long n16 = bytes / 16;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n16; i += stride)
    reinterpret_cast<uint4*>(p)[i] = make_uint4(0u, 0u, 0u, 0u);
  for (unsigned long long i = n16 * 16 + blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < bytes;
       i += stride)
    p[i] = 0;
}

// Frame input x | y | z | d (stride n) -> interleaved staging consumed by k_ingest
// is not needed: k_ingest reads the four arrays directly. Frame output: the
// positions of the current state as x | y | z (stride n).
__global__ void k_split_xyz(const Pd* __restrict__ pos, const unsigned long long* __restrict__ uid,
                            const DevGrid* g, double* __restrict__ out, unsigned long long stride) {
  const unsigned long long n = g->n;
  unsigned long long* ou = reinterpret_cast<unsigned long long*>(out + 3 * stride);
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const Pd p = load_pd(pos + i);
    out[i] = p.x;
    out[stride + i] = p.y;
    out[2 * stride + i] = p.z;
    if (uid) ou[i] = uid[i];
  }
}

// ------------------------------------------------------------ multi-domain exchange
// Packed agent record exchanged between ranks: 96 bytes.
struct __align__(16) Rec {
  double x, y, z, d, vol, fx, fy, fz;
  unsigned long long uid;
  unsigned int partners;
  unsigned char flags, beh, pad0, pad1;
  unsigned long long rngc;
  unsigned int tag, pad3;
};
static_assert(sizeof(Rec) == 96, "record layout");

// mode 0 (migrate): owned agents with box z-layer < lo -> out_lo, >= hi -> out_hi,
//                   keep[i] = 0 for them. mode 1 (halo): layer == lo -> out_lo,
//                   layer == hi - 1 -> out_hi, kept. Ghosts are never exported.
// periodic (ring of z layers, config 5): a migrant goes to the nearer side
// modulo dimz (a wrapped step from layer 0 to dimz-1 leaves through lo).
__global__ void k_export(const Pd* __restrict__ pos, Soa S, unsigned long long cap, unsigned long long n,
                         double oz, double box, unsigned int dimz, long long lo, long long hi, int mode,
                         int periodic, Rec* __restrict__ out_lo, Rec* __restrict__ out_hi,
                         unsigned long long out_cap, unsigned long long* __restrict__ counts,
                         unsigned int* __restrict__ keep) {
  const long long D = static_cast<long long>(dimz);
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const Pd p = load_pd(pos + i);
    const unsigned char fl = S.flags[i];
    const long long layer = static_cast<long long>(box_coord(p.z, oz, box, dimz));
    int dest = -1;  // 0 -> lo, 1 -> hi
    if (!(fl & ABS_FLAG_GHOST)) {
      if (mode == 0) {
        if (layer < lo || layer >= hi) {
          if (periodic) dest = ((lo - layer + D) % D) <= ((layer - (hi - 1) + D) % D) ? 0 : 1;
          else dest = layer < lo ? 0 : 1;
        }
      } else {
        dest = layer == lo ? 0 : (layer == hi - 1 ? 1 : -1);
      }
    }
    if (keep) keep[i] = (mode == 0 && dest >= 0) ? 0u : 1u;
    if (dest < 0) continue;
    const unsigned long long slot = atomicAdd(counts + dest, 1ull);
    if (slot >= out_cap) continue;  // caller sees count > cap and retries larger
    Rec r;
    r.x = p.x; r.y = p.y; r.z = p.z; r.d = p.d;
    r.vol = S.vol[i];
    r.fx = S.force[i]; r.fy = S.force[cap + i]; r.fz = S.force[2 * cap + i];
    r.uid = S.uid[i];
    r.partners = S.partners[i];
    r.flags = fl;
    r.beh = S.beh[i];
    r.pad0 = r.pad1 = 0;
    r.rngc = S.rngc[i];
    r.tag = S.tag[i];
    r.pad3 = S.skey[i];
    (dest ? out_hi : out_lo)[slot] = r;
  }
}

__global__ void k_import(const Rec* __restrict__ in, unsigned long long count, unsigned long long base,
                         Pd* __restrict__ pos, Soa S, unsigned long long cap, int as_ghost) {
  for (unsigned long long k = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; k < count;
       k += (unsigned long long)gridDim.x * blockDim.x) {
    const Rec r = in[k];
    const unsigned long long j = base + k;
    pos[j] = Pd{r.x, r.y, r.z, r.d};
    S.vol[j] = r.vol;
    S.force[j] = r.fx; S.force[cap + j] = r.fy; S.force[2 * cap + j] = r.fz;
    S.uid[j] = r.uid;
    S.partners[j] = r.partners;
    S.flags[j] = as_ghost ? (r.flags | ABS_FLAG_GHOST) : static_cast<unsigned char>(r.flags & ~ABS_FLAG_GHOST);
    S.beh[j] = r.beh;
    S.tag[j] = r.tag;
    S.rngc[j] = r.rngc;
    S.skey[j] = r.pad3;
  }
}

__global__ void k_keep_ghostless(const Soa S, unsigned long long n, unsigned int* __restrict__ keep) {
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x)
    keep[i] = (S.flags[i] & ABS_FLAG_GHOST) ? 0u : 1u;
}

// ------------------------------------------------------------ parity helpers
__global__ void k_cell_ids(const Pd* __restrict__ pos, const DevGrid* g, unsigned long long* out) {
  const DevGrid G = *g;
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < G.n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const Pd p = load_pd(pos + i);
    const unsigned long long c0 = box_coord(p.x, G.origin[0], G.box, G.dims[0]);
    const unsigned long long c1 = box_coord(p.y, G.origin[1], G.box, G.dims[1]);
    const unsigned long long c2 = box_coord(p.z, G.origin[2], G.box, G.dims[2]);
    out[i] = c0 + G.dims[0] * (c1 + (unsigned long long)G.dims[1] * c2);
  }
}

__global__ void k_nbr_count(const Pd* __restrict__ pd, const DevGrid* g,
                            const unsigned int* __restrict__ start, unsigned long long* cnt, KdView kd) {
  const DevGrid G = *g;
  const QGrid Q = make_qgrid(G);
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < G.n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const Pd me = load_pd(pd + i);
    const double r = 0.5 * (me.d + G.dmax);
    unsigned long long c = 0;
    auto count = [&](unsigned int, const Pd&, double, double, double, double) { ++c; };
    if (kd.n) for_each_neighbor_kd(kd, pd, (unsigned int)i, me.x, me.y, me.z, r, r * r, count);
    else for_each_neighbor(Q, pd, start, (unsigned int)i, me.x, me.y, me.z, r, r * r, count);
    cnt[i] = c;
  }
}

__global__ void k_nbr_fill(const Pd* __restrict__ pd, const unsigned long long* __restrict__ uid,
                           const DevGrid* g, const unsigned int* __restrict__ start,
                           const unsigned long long* __restrict__ off, unsigned long long* out, KdView kd) {
  const DevGrid G = *g;
  const QGrid Q = make_qgrid(G);
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < G.n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const Pd me = load_pd(pd + i);
    const double r = 0.5 * (me.d + G.dmax);
    unsigned long long w = off[i];
    auto put = [&](unsigned int j, const Pd&, double, double, double, double) { out[w++] = uid[j]; };
    if (kd.n) for_each_neighbor_kd(kd, pd, (unsigned int)i, me.x, me.y, me.z, r, r * r, put);
    else for_each_neighbor(Q, pd, start, (unsigned int)i, me.x, me.y, me.z, r, r * r, put);
    // insertion sort of this agent's uid list
    const unsigned long long b = off[i], e = off[i + 1];
    for (unsigned long long p = b + 1; p < e; ++p) {
      const unsigned long long v = out[p];
      unsigned long long q = p;
      while (q > b && out[q - 1] > v) {
        out[q] = out[q - 1];
        --q;
      }
      out[q] = v;
    }
  }
}

// ------------------------------------------------------------ sort_and_balance
// Morton code of a box (morton.cpp:11-29, 54-60).
__device__ __forceinline__ unsigned long long spread3(unsigned long long v) {
  v &= 0x1fffff;
  v = (v | v << 32) & 0x1f00000000ffffull;
  v = (v | v << 16) & 0x1f0000ff0000ffull;
  v = (v | v << 8) & 0x100f00f00f00f00full;
  v = (v | v << 4) & 0x10c30c30c30c30c3ull;
  v = (v | v << 2) & 0x1249249249249249ull;
  return v;
}

__device__ __forceinline__ unsigned long long morton_code_of(const DevGrid& G, double px, double py, double pz) {
  const unsigned long long c0 = box_coord(px, G.origin[0], G.box, G.dims[0]);
  const unsigned long long c1 = box_coord(py, G.origin[1], G.box, G.dims[1]);
  if (G.dims[2] == 1) {  // 2-D table (morton.cpp:124-129): x bits 2i, y bits 2i+1
    unsigned long long o = 0;
    for (int b = 0; b < 31; ++b) o |= ((c0 >> b) & 1ull) << (2 * b) | ((c1 >> b) & 1ull) << (2 * b + 1);
    return o;
  }
  const unsigned long long c2 = box_coord(pz, G.origin[2], G.box, G.dims[2]);
  return spread3(c0) | spread3(c1) << 1 | spread3(c2) << 2;
}

// In-loop sort mode (one thread, after the sort-mode finalize): counting sort
// by Morton code when the code space fits the cell table (the in-box order is
// unobservable there: the iteration's re-bin re-orders by cell right after),
// else the exact radix path. mode == 0 always for abs_gpu_sort.
// allow_counting: 0 exact radix path, 1 counting path if the code space
// fits the cell table, 2 counting path required (the host launched only it:
// if it does not fit, flag a retry so the host re-runs with the radix path).
__global__ void k_sort_mode(DevGrid* g, unsigned long long table_cap, int allow_counting,
                            unsigned long long iteration) {
  const unsigned int maxdim = max(g->dims[0], max(g->dims[1], g->dims[2]));
  unsigned int axis_bits = 0;
  while ((1u << axis_bits) < maxdim) ++axis_bits;
  const unsigned int code_bits = (g->dims[2] == 1 ? 2u : 3u) * axis_bits;
  const bool fits = code_bits < 40 && (1ull << code_bits) <= table_cap;
  if (allow_counting == 2 && !fits && !g->err) {
    g->err = kErrSortRetry;
    g->failed_iteration = iteration;
  }
  g->sort_mode = (allow_counting && fits && !g->err) ? 1u : 0u;
  g->sort_len = g->sort_mode ? (1ull << code_bits) : 0ull;
  if (g->sort_mode) g->sort_passes = 0;
}

// Counting-sort keys: Morton code + slot claimed by an atomic (k_key's form).
__global__ void k_mkey(const Pd* __restrict__ pos, const DevGrid* g, unsigned int* __restrict__ count,
                       unsigned int* __restrict__ key, unsigned int* __restrict__ rank) {
  if (g->err || g->sort_mode != 1u) return;
  const DevGrid G = *g;
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < G.n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const Pd p = load_pd(pos + i);
    const unsigned int code = static_cast<unsigned int>(morton_code_of(G, p.x, p.y, p.z));
    key[i] = code;
    rank[i] = atomicAdd(count + code, 1u);
  }
}

// Sort keys: the Morton code of each agent's reference box, listed in
// DESCENDING storage index (element t = agent n-1-t). A stable LSD sort on the
// code alone then gives curve order with descending index inside a box — the
// reference's chain order (sort_balance.cpp:88-128) — without radix passes
// over the index bits.
//
// "Storage index" is the REFERENCE's: the device keeps its own storage in cell
// order, so with by_key the agent at device slot i is listed at its reference
// slot skey[i] (a permutation of [0, n) in a single-domain context; checked
// through nkeys == n). Without keys (decomposed contexts, whose keys are
// global) the device order stands in.
__global__ void k_sort_keys(const Pd* __restrict__ pos, DevGrid* g, unsigned long long* keyhi,
                            unsigned int* __restrict__ idx, const unsigned int* __restrict__ skey, int by_key) {
  const DevGrid G = *g;
  if (G.sort_mode == 1u) return;  // in-loop counting sort selected (k_sort_mode)
  // an earlier iteration of this chunk failed (to be re-run): its state moves
  // were skipped, so the buffers the host already flipped to hold no valid keys
  if (G.err) return;
  const bool keyed = by_key && G.nkeys == G.n;
  if (blockIdx.x == 0 && threadIdx.x == 0) {  // passes over the used key bits, rounded up to even
    const unsigned int maxdim = max(G.dims[0], max(G.dims[1], G.dims[2]));
    unsigned int axis_bits = 0;
    while ((1u << axis_bits) < maxdim) ++axis_bits;
    const unsigned int code_bits = (G.dims[2] == 1 ? 2u : 3u) * axis_bits;
    unsigned int passes = (code_bits + 7u) / 8u;
    g->sort_passes = passes + (passes & 1u);
  }
  for (unsigned long long q = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; q < G.n;
       q += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long i = keyed ? q : G.n - 1 - q;
    ABS_ASSERT(!keyed || skey[i] < G.n);
    const unsigned long long t = keyed ? G.n - 1 - skey[i] : q;
    const Pd p = load_pd(pos + i);
    const unsigned long long c0 = box_coord(p.x, G.origin[0], G.box, G.dims[0]);
    const unsigned long long c1 = box_coord(p.y, G.origin[1], G.box, G.dims[1]);
    const unsigned long long c2 = box_coord(p.z, G.origin[2], G.box, G.dims[2]);
    const unsigned long long code = G.dims[2] == 1 ? 0ull : (spread3(c0) | spread3(c1) << 1 | spread3(c2) << 2);
    unsigned long long code2 = code;
    if (G.dims[2] == 1) {  // 2-D table (morton.cpp:124-129): x bits 2i, y bits 2i+1
      unsigned long long xx = c0, yy = c1, o = 0;
      for (int b = 0; b < 31; ++b) o |= ((xx >> b) & 1ull) << (2 * b) | ((yy >> b) & 1ull) << (2 * b + 1);
      code2 = o;
    }
    keyhi[t] = code2;
    idx[t] = static_cast<unsigned int>(i);
  }
}

__device__ __forceinline__ unsigned int radix_digit(unsigned long long code, unsigned int, int shift) {
  return static_cast<unsigned int>((code >> shift) & 255ull);
}

// One LSD radix pass (8 bits) over (key, idx) pairs with a stable
// counting sort per digit: histogram -> scan -> rank by prefix popcounts.
// Passes at or beyond g->sort_passes are skipped (they come in pairs, so the
// host's ping-pong buffer order stays right without reading the grid back).
__global__ void k_radix_hist(const unsigned long long* __restrict__ key, const unsigned int* __restrict__ idx,
                             const DevGrid* g, int shift, unsigned int* __restrict__ hist,
                             unsigned long long chunk) {
  if (shift / 8 >= static_cast<int>(g->sort_passes)) return;
  const unsigned long long n = g->n;
  __shared__ unsigned int h[256];
  for (int t = threadIdx.x; t < 256; t += blockDim.x) h[t] = 0;
  __syncthreads();
  const unsigned long long b = blockIdx.x * chunk, e = min(n, b + chunk);
  for (unsigned long long i = b + threadIdx.x; i < e; i += blockDim.x) {
    atomicAdd(&h[radix_digit(key[i], idx[i], shift)], 1u);
  }
  __syncthreads();
  for (int t = threadIdx.x; t < 256; t += blockDim.x) hist[t * gridDim.x + blockIdx.x] = h[t];
}

__global__ void k_radix_scatter(const unsigned long long* __restrict__ key, const unsigned int* __restrict__ idx,
                                unsigned long long* __restrict__ key2, unsigned int* __restrict__ idx2,
                                const DevGrid* g, int shift, const unsigned int* __restrict__ hist,
                                unsigned long long chunk) {
  if (shift / 8 >= static_cast<int>(g->sort_passes)) return;
  const unsigned long long n = g->n;
  // one warp per block walks its chunk in order: stable by construction
  __shared__ unsigned int base[256];
  for (int t = threadIdx.x; t < 256; t += blockDim.x) base[t] = hist[t * gridDim.x + blockIdx.x];
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const unsigned long long b = blockIdx.x * chunk, e = min(n, b + chunk);
  const int lane = threadIdx.x;
  for (unsigned long long i0 = b; i0 < e; i0 += 32) {
    const unsigned long long i = i0 + lane;
    const bool ok = i < e;
    unsigned int dig = 0;
    unsigned long long k = 0;
    unsigned int ix = 0;
    if (ok) {
      k = key[i];
      ix = idx[i];
      dig = radix_digit(k, ix, shift);
    }
    const unsigned int peers = __match_any_sync(0xffffffffu, ok ? dig : 0x1000u);
    const unsigned int before = __popc(peers & ((1u << lane) - 1u));
    unsigned int pos = 0;
    if (ok) pos = base[dig] + before;
    __syncwarp();
    const int leader = __ffs(peers) - 1;
    if (ok && lane == leader) base[dig] += __popc(peers);
    __syncwarp();
    if (ok) {
      key2[pos] = k;
      idx2[pos] = ix;
    }
  }
}

__global__ void k_gather(const Pd* __restrict__ pos, Soa src, Soa dst, const unsigned int* __restrict__ perm,
                         const DevGrid* g, unsigned long long cap, int carry_vol, int carry_force,
                         int only_sort_mode = -1, int carry_ext = 1, int renumber_keys = 1) {
  if (g->err) return;
  if (only_sort_mode >= 0 && static_cast<int>(g->sort_mode) != only_sort_mode) return;
  const unsigned long long n = g->n;
  for (unsigned long long j = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; j < n;
       j += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned int i = perm[j];
    const Pd p = load_pd(pos + i);
    reinterpret_cast<double2*>(dst.pd + j)[0] = make_double2(p.x, p.y);
    reinterpret_cast<double2*>(dst.pd + j)[1] = make_double2(p.z, p.d);
    dst.uid[j] = src.uid[i];
    dst.flags[j] = src.flags[i];
    dst.partners[j] = src.partners[i];
    dst.beh[j] = src.beh[i];
    if (carry_vol) dst.vol[j] = src.vol[i];
    if (carry_force) {
      dst.force[j] = src.force[i];
      dst.force[cap + j] = src.force[cap + i];
      dst.force[2 * cap + j] = src.force[2 * cap + i];
    }
    // sort_and_balance's new storage slot; a gather that is not the reference's sort carries the key
    dst.skey[j] = renumber_keys ? static_cast<unsigned int>(j) : src.skey[i];
    if (carry_ext) {
      dst.tag[j] = src.tag[i];
      dst.rngc[j] = src.rngc[i];
    }
  }
}

// Removal lookup with O(removed) scratch: every agent binary-searches its uid
// in the sorted removal list; a hit records the agent's slot at the list's
// original position (perm) and counts it.
__global__ void k_find_slots(const unsigned long long* __restrict__ uid, const DevGrid* g,
                             const unsigned long long* __restrict__ sorted_uids,
                             const unsigned long long* __restrict__ perm, unsigned long long r,
                             unsigned long long* __restrict__ slots, unsigned long long* __restrict__ found) {
  const unsigned long long n = g->n;
  unsigned long long hits = 0;
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long u = uid[i];
    unsigned long long lo = 0, hi = r;
    while (lo < hi) {
      const unsigned long long mid = (lo + hi) >> 1;
      if (sorted_uids[mid] < u) lo = mid + 1;
      else hi = mid;
    }
    if (lo < r && sorted_uids[lo] == u) {
      slots[perm[lo]] = i;
      ++hits;
    }
  }
  if (hits) atomicAdd(found, hits);
}


// O(removed) compaction: storage order is free (the next
// re-bin re-sorts by cell), so the survivors beyond the new end move into
// the holes below it. idx = exclusive scan of keep; hole k of [0, new_n) is
// the k-th removed slot there; survivor i >= new_n fills hole idx[i] - idx[new_n].
__global__ void k_hole_list(const unsigned int* __restrict__ keep, const unsigned int* __restrict__ idx,
                            unsigned long long new_n, unsigned int* __restrict__ holes) {
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < new_n;
       i += (unsigned long long)gridDim.x * blockDim.x)
    if (!keep[i]) holes[i - idx[i]] = static_cast<unsigned int>(i);
}

__global__ void k_swap_move(Pd* pos, Soa S, const unsigned int* __restrict__ keep, const unsigned int* __restrict__ idx,
                            const unsigned int* __restrict__ holes, unsigned long long new_n, unsigned long long n,
                            unsigned long long cap) {
  const unsigned int base = idx[new_n];
  for (unsigned long long i = new_n + blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    if (!keep[i]) continue;
    const unsigned long long dst = holes[idx[i] - base];
    pos[dst] = load_pd(pos + i);
    S.uid[dst] = S.uid[i];
    S.flags[dst] = S.flags[i];
    S.partners[dst] = S.partners[i];
    S.beh[dst] = S.beh[i];
    S.vol[dst] = S.vol[i];
    S.force[dst] = S.force[i];
    S.force[cap + dst] = S.force[cap + i];
    S.force[2 * cap + dst] = S.force[2 * cap + i];
    S.tag[dst] = S.tag[i];
    S.rngc[dst] = S.rngc[i];
    S.skey[dst] = S.skey[i];
  }
}



// ------------------------------------------------------------ removal by storage key
// remove_agents_parallel (commit.cpp:14-106) applied to the reference's
// storage order, which the device carries as per-agent keys (Soa::skey): with
// new_size = nkeys - r, the k-th hole (a removed key < new_size, in
// removal-list order — for removals staged by the agent loop of one worker
// that is key order) receives the k-th surviving key >= new_size in
// ascending order; every other survivor keeps its key. The device's own
// storage order is free (the next re-bin re-sorts by cell), so the removed
// agents are then compacted out with O(removed) moves.
//
// rscan: the removal marks over keys [0, nkeys), exclusive-scanned in place
// (rscan[nkeys] = r); a mark is rscan[k+1] - rscan[k].
__global__ void k_rem_holes(const unsigned int* __restrict__ rscan, const DevGrid* g,
                            unsigned int* __restrict__ hole_at) {
  if (g->err) return;
  const unsigned long long nk = g->nkeys;
  const unsigned long long new_size = nk - rscan[nk];
  for (unsigned long long k = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; k < new_size;
       k += (unsigned long long)gridDim.x * blockDim.x)
    if (rscan[k + 1] > rscan[k]) hole_at[rscan[k]] = static_cast<unsigned int>(k);
}

// New keys of the survivors; keep / idx = 1 for survivors (idx is scanned next).
__global__ void k_rem_rekey(Soa S, const DevGrid* g, const unsigned int* __restrict__ rscan,
                            const unsigned int* __restrict__ hole_at, unsigned int* __restrict__ keep,
                            unsigned int* __restrict__ idx) {
  if (g->err) return;
  const unsigned long long n = g->n, nk = g->nkeys;
  const unsigned long long new_size = nk - rscan[nk];
  const unsigned int base = rscan[new_size];
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const bool dead = S.flags[i] & ABS_FLAG_REMOVED;
    keep[i] = idx[i] = dead ? 0u : 1u;
    if (dead) continue;
    const unsigned int key = S.skey[i];
    ABS_ASSERT(key < nk);
    if (key >= new_size) {  // a surviving tail agent: the mover rank picks its hole
      const unsigned long long m = (key - new_size) - (rscan[key] - base);
      ABS_ASSERT(m < base);
      S.skey[i] = hole_at[m];
    }
  }
}

// Compaction with device-resident counts: idx = exclusive scan of keep over
// [0, n), idx[n] = survivors.
__global__ void k_hole_list_d(const unsigned int* __restrict__ keep, const unsigned int* __restrict__ idx,
                              const DevGrid* g, unsigned int* __restrict__ holes) {
  if (g->err) return;
  const unsigned long long new_n = idx[g->n];
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < new_n;
       i += (unsigned long long)gridDim.x * blockDim.x)
    if (!keep[i]) holes[i - idx[i]] = static_cast<unsigned int>(i);
}

__global__ void k_swap_move_d(Pd* pos, Soa S, const unsigned int* __restrict__ keep,
                              const unsigned int* __restrict__ idx, const unsigned int* __restrict__ holes,
                              const DevGrid* g, unsigned long long cap) {
  if (g->err) return;
  const unsigned long long n = g->n, new_n = idx[n];
  const unsigned int base = idx[new_n];
  for (unsigned long long i = new_n + blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    if (!keep[i]) continue;
    const unsigned long long dst = holes[idx[i] - base];
    ABS_ASSERT(dst < new_n);
    pos[dst] = load_pd(pos + i);
    S.uid[dst] = S.uid[i];
    S.flags[dst] = S.flags[i];
    S.partners[dst] = S.partners[i];
    S.beh[dst] = S.beh[i];
    S.vol[dst] = S.vol[i];
    S.force[dst] = S.force[i];
    S.force[cap + dst] = S.force[cap + i];
    S.force[2 * cap + dst] = S.force[2 * cap + i];
    S.tag[dst] = S.tag[i];
    S.rngc[dst] = S.rngc[i];
    S.skey[dst] = S.skey[i];
  }
}

__global__ void k_rem_fin(DevGrid* g, const unsigned int* __restrict__ idx, const unsigned int* __restrict__ rscan) {
  if (threadIdx.x || blockIdx.x || g->err) return;
  const unsigned long long n = g->n, nn = idx[n];
  g->removed += n - nn;
  g->nkeys -= rscan[g->nkeys];
  g->n = nn;
  g->removed_now = 0;
}

// abs_gpu_remove: the caller's list gives the hole order. to_right[k] = 1 for
// list entries whose key lies below new_size; keys are marked for the
// mover ranks and the agents flagged for the compaction.
__global__ void k_api_mark(Soa S, const unsigned long long* __restrict__ slots, unsigned long long r,
                           unsigned long long new_size, unsigned int* __restrict__ rmark,
                           unsigned int* __restrict__ to_right, unsigned int* __restrict__ key_of) {
  for (unsigned long long k = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; k < r;
       k += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long i = slots[k];
    const unsigned int key = S.skey[i];
    key_of[k] = key;
    S.flags[i] |= ABS_FLAG_REMOVED;
    rmark[key] = 1u;
    to_right[k] = key < new_size ? 1u : 0u;
  }
}

__global__ void k_api_holes(const unsigned int* __restrict__ to_right, const unsigned int* __restrict__ rank,
                            const unsigned int* __restrict__ key_of, unsigned long long r,
                            unsigned int* __restrict__ hole_at) {
  for (unsigned long long k = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; k < r;
       k += (unsigned long long)gridDim.x * blockDim.x)
    if (to_right[k]) hole_at[rank[k]] = key_of[k];
}


}  // namespace

// ====================================================================== host
struct abs_gpu_ctx {
  abs_gpu_config cfg{};
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  std::string err;
  int sms = 148;

  unsigned int auto_bins = 2;      // sub-bins per box edge chosen at upload (bins_per_box == 0)
  unsigned long long cap = 0;      // agent capacity
  unsigned long long uid_cap = 0;  // uid-indexed arrays
  unsigned long long bins_cap = 0;
  unsigned long long n = 0;        // host mirror (refreshed on sync)
  unsigned long long iteration = 0;
  unsigned long long launches = 0;

  Soa S[2]{};
  int cur = 0;
  Pd* newpd = nullptr;
  float4* pf = nullptr;  // fp32 copy of pd relative to the grid origin (candidate classification)
  // kd-tree environment (kdtree.cuh): per-node split axis and bounds, heap order
  unsigned char* kd_axis = nullptr;
  double* kd_lmax = nullptr;
  double* kd_rmin = nullptr;
  unsigned long long* kd_bbox = nullptr;
  unsigned long long kd_nodes_cap = 0, kd_n = 0;
  bool marks_listed = false;  // this iteration's k_scatter wrote the static-detection mark list (c->holes)
  bool kd_valid = false;
  bool kd_failed = false;  // the last build could not allocate its node arrays
  bool pos_in_new = true;  // current positions live in newpd (else S[cur].pd)
  bool grid_valid = false; // `start` holds a scanned cell table for S[cur]

  DevGrid* g = nullptr;
  unsigned int* start = nullptr;  // bins_cap
  unsigned int* key = nullptr;
  unsigned int* rank = nullptr;
  unsigned int* tiles = nullptr;  // scan tile sums (u32)
  unsigned int* ctiles = nullptr;  // tile sums of agent-sized scans (compaction), cap / kScanTile + 2
  unsigned long long* scan_state = nullptr;  // single-pass cell-table scan (k_scan_onepass)
  unsigned int sort_guess_dims[3] = {0, 0, 0};      // grid dims last read back (in-loop sort path guess)
  unsigned long long sort_radix_iteration = ~0ull;  // iteration whose counting guess failed
  // per-iteration CUDA graphs (abs_gpu_simulate): [0] plain, [1] with the Morton sort
  // slot = (sort ? 1 : 0) + 2 * iteration kind (0 re-bin + walk, 1 list step, 2 list rebuild,
  // 3 re-bin + walk tracking the displacement for the list policy)
  cudaGraphExec_t gexec[8] = {};
  // neighbour lists
  unsigned int* nl = nullptr;           // [kmax][stride] candidate storage indices
  float4* pf2 = nullptr;                // fp32 copy paired with newpd (pf is paired with S[cur].pd)
  unsigned long long pf2_cap = 0;
  unsigned char* nl_cnt = nullptr;      // [stride] candidates per agent
  unsigned int* nl_ct = nullptr;        // warp-blocked [16][32] possible contacts per agent (list step)
  unsigned char* nl_nct = nullptr;      // contacts per agent
  unsigned long long nl_stride = 0;
  unsigned int nl_kmax = 0;
  bool list_valid = false;              // lists match the current storage order
  bool list_off = false;                // lists disabled for this context (candidate count > 255)
  bool ov_on = false;                   // host mirror of the multi-domain grid override
  double host_dmax = 0.0;               // largest diameter of the last upload (auto skin)
  // host prediction of the device coverage check: accumulated displacement
  // the next list step will see, and the last step's largest displacement
  double pred_acc = 0.0, pred_rate = 0.0;
  bool track_now = false;               // this iteration tracks its largest displacement (kind 3)
  struct abs_gpu_decomp* decomp = nullptr;  // multi-GPU slab decomposition (decomp.cuh)
  double build_ms = 0.0;
  unsigned long long build_launches = 0;
  std::vector<cudaEvent_t> bev;  // pairs around k_list_build (timing on)
  size_t bev_used = 0;
  unsigned long long list_builds = 0, list_steps = 0;
  // per-agent force evaluations of the last iteration (abs_gpu_record_evaluations)
  unsigned int* evc = nullptr;
  unsigned long long evc_cap = 0;
  bool rec_evals = false;
  int graph_failures = 0;
  bool graphs_off = false;
  unsigned int* holes = nullptr;           // compact_population: removed slots below the new end
  unsigned long long holes_cap = 0;
  unsigned long long* xcounts = nullptr;   // abs_gpu_export_layers counts (device)
  unsigned long long* hxcounts = nullptr;  // and their page-locked host copy
  unsigned int scan_epoch = 0;
  unsigned long long* tiles64 = nullptr;
  unsigned char* nv = nullptr;
  unsigned char* nn = nullptr;
  unsigned long long* st_parent = nullptr;
  Pd* st_pd = nullptr;
  double* st_vol = nullptr;
  unsigned int* st_tag = nullptr;    // staged daughters' tags
  unsigned int* div_mark = nullptr;  // uid_cap + 1: this context's dividing parents (then their local ranks)
  unsigned int* div_mark_g = nullptr;  // uid_cap + 1: all ranks' dividing parents (deferred commit only)
  unsigned int* rmark = nullptr;     // uid_cap + 1: removal marks by reference storage key (then their scan)
  unsigned int* hole_at = nullptr;   // uid_cap + 1: the reference's holes in removal order
  bool defer_commit = false;         // multi-domain additions: stop before the commit
  bool pending_commit = false;
  double* ingest_part = nullptr;     // mapped page-locked: per-block (sum d, max d) of the last upload
  DevGrid* hgrid = nullptr;          // mapped page-locked mirror of *g (read_grid)
  // host-boundary pipeline (abs_gpu_run_frames): two copy streams, double-buffered
  // device staging of frame inputs (x|y|z|d) and outputs (x|y|z)
  cudaStream_t h2d = nullptr, d2h = nullptr;
  double* fin[2] = {nullptr, nullptr};
  double* fout[2] = {nullptr, nullptr};
  unsigned long long fcap = 0, fout_cap = 0;  // agents per input / output slot
  cudaEvent_t in_ready[2] = {}, in_free[2] = {}, out_ready[2] = {}, out_free[2] = {};
  unsigned long long ghosts = 0;     // upper bound on ghost agents present (0 -> drop_ghosts is a no-op)
  // Morton sort scratch (capacity-sized, allocated on first use)
  unsigned long long sort_cap = 0;
  unsigned long long *sort_k[2] = {nullptr, nullptr};
  unsigned int *sort_i[2] = {nullptr, nullptr};
  unsigned int* sort_hist = nullptr;
  unsigned int* sort_tiles = nullptr;
  unsigned long long* sort_hlen = nullptr;


  bool timing = false;
  std::vector<cudaEvent_t> ev;  // pairs
  size_t ev_used = 0;
  // SimulationReport categories (report.hpp:12-23): five marks per iteration
  // [start | after sort | after environment update | after agent ops | after commit]
  std::vector<cudaEvent_t> pev;
  size_t pev_used = 0;
  double phase_ms[4] = {0.0, 0.0, 0.0, 0.0};  // env update, sorting, agent ops, setup/teardown
  std::vector<double> iter_ms;
  double force_ms = 0.0;
  unsigned long long force_launches = 0;
};

namespace {

thread_local std::string g_create_err;

int set_err(abs_gpu_ctx* c, int code, const std::string& m) {
  if (c) c->err = m;
  else g_create_err = m;
  return code;
}

#define CK(expr)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (expr);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return set_err(c, ABS_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// Models whose behaviour creates agents (daughter staging, uid-indexed marks).
bool adds_agents(const abs_gpu_config& cfg) {
  return cfg.model == ABS_MODEL_PROLIFERATION || cfg.model == ABS_MODEL_GROW_DIVIDE ||
         cfg.model == ABS_MODEL_GROW_DIVIDE_DIE;
}
// Models whose behaviour removes agents (AgentContext::remove_self).
bool removes_agents(const abs_gpu_config& cfg) { return cfg.model == ABS_MODEL_GROW_DIVIDE_DIE; }
// Storage keys must follow the reference's order exactly (daughter numbering,
// removal slots): Morton sorts then take the exact (radix) path.
bool keys_exact(const abs_gpu_config& cfg) { return adds_agents(cfg) || removes_agents(cfg); }
// Models that read Agent::tag / rng_counter.
bool uses_ext(const abs_gpu_config& cfg) {
  return cfg.model == ABS_MODEL_GROW_DIVIDE || cfg.model == ABS_MODEL_COHERE || cfg.model == ABS_MODEL_GROW_DIVIDE_DIE;
}

// BruteForceEnvironment (environment.hpp:53-80) instead of the grid.
// The kd-tree environment keeps the brute-force single box underneath (static
// marking, new-agent marking and behaviour queries walk it) and answers the
// force query through the tree.
bool kd_env(const abs_gpu_ctx* c) { return c->cfg.environment == ABS_ENV_KD_TREE; }
int brute_env(const abs_gpu_ctx* c) {
  return c->cfg.environment == ABS_ENV_BRUTE_FORCE || c->cfg.environment == ABS_ENV_KD_TREE ? 1 : 0;
}
KdView kd_view(const abs_gpu_ctx* c) {
  if (!kd_env(c) || !c->kd_valid || !c->grid_valid) return KdView{nullptr, nullptr, nullptr, 0u};
  return KdView{c->kd_axis, c->kd_lmax, c->kd_rmin, static_cast<unsigned int>(c->kd_n)};
}

int grid_blocks(const abs_gpu_ctx* c, unsigned long long work) {
  const unsigned long long b = (work + kThreads - 1) / kThreads;
  const unsigned long long lim = static_cast<unsigned long long>(c->sms) * 8;
  return static_cast<int>(std::max<unsigned long long>(1, std::min(b, lim)));
}

// Grid of an agent-sized grid-stride kernel, from the host's mirror of the
// agent count (exact between chunks; a population that grows inside a chunk
// only makes the resident threads loop). Small populations get fewer blocks:
// an empty block still pays its start-up and, in the reductions, its
// same-address atomics (c1: k_reduce_finalize 12.7 us with 1028 blocks).
int agent_blocks(const abs_gpu_ctx* c, unsigned int per_thread = 1) {
  const unsigned long long n = c->n ? std::min(c->n, c->cap) : c->cap;
  const unsigned long long per_block = static_cast<unsigned long long>(kThreads) * per_thread;
  const unsigned long long b = (n + per_block - 1) / per_block;
  const unsigned long long lim = static_cast<unsigned long long>(c->sms) * 8;
  return static_cast<int>(std::max<unsigned long long>(1, std::min(b, lim)));
}

template <class K>
int force_blocks(const abs_gpu_ctx* c, K kernel, int smem = (2 * kMaxRows + kMaxContacts) * kForceThreads * 4) {
  int per_sm = 0;  // persistent: the resident CTAs only
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kForceThreads, smem);
  return c->sms * std::max(per_sm, 1);
}

template <class T>
cudaError_t dalloc(T** p, unsigned long long count) {
  *p = nullptr;
  if (count == 0) count = 1;
  return cudaMalloc(reinterpret_cast<void**>(p), count * sizeof(T));
}

void free_soa(Soa& s) {
  cudaFree(s.pd); cudaFree(s.uid); cudaFree(s.flags); cudaFree(s.partners);
  cudaFree(s.vol); cudaFree(s.beh); cudaFree(s.force); cudaFree(s.tag); cudaFree(s.rngc); cudaFree(s.skey);
  s = Soa{};
}

cudaError_t alloc_soa(Soa& s, unsigned long long cap) {
  cudaError_t e;
  if ((e = dalloc(&s.pd, cap))) return e;
  if ((e = dalloc(&s.uid, cap))) return e;
  if ((e = dalloc(&s.flags, cap))) return e;
  if ((e = dalloc(&s.partners, cap))) return e;
  if ((e = dalloc(&s.vol, cap))) return e;
  if ((e = dalloc(&s.beh, cap))) return e;
  if ((e = dalloc(&s.force, 3 * cap))) return e;
  if ((e = dalloc(&s.tag, cap))) return e;
  if ((e = dalloc(&s.rngc, cap))) return e;
  if ((e = dalloc(&s.skey, cap))) return e;
  return cudaSuccess;
}

Pd* cur_pos(abs_gpu_ctx* c) { return c->pos_in_new ? c->newpd : c->S[c->cur].pd; }

// (Re)allocate agent-sized buffers preserving the first `keep` agents.
int ensure_capacity(abs_gpu_ctx* c, unsigned long long want, unsigned long long keep) {
  if (want <= c->cap) return ABS_OK;
  c->list_valid = false;
  unsigned long long ncap = std::max<unsigned long long>(want, 1024);
  Soa S2[2]{};
  for (int b = 0; b < 2; ++b) CK(alloc_soa(S2[b], ncap));
  Pd* np = nullptr;
  CK(dalloc(&np, ncap));
  if (keep) {
    Soa& src = c->S[c->cur];
    Soa& dst = S2[0];
    CK(cudaMemcpyAsync(np, cur_pos(c), keep * sizeof(Pd), cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaMemcpyAsync(dst.uid, src.uid, keep * 8, cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaMemcpyAsync(dst.flags, src.flags, keep, cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaMemcpyAsync(dst.partners, src.partners, keep * 4, cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaMemcpyAsync(dst.vol, src.vol, keep * 8, cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaMemcpyAsync(dst.beh, src.beh, keep, cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaMemcpyAsync(dst.tag, src.tag, keep * 4, cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaMemcpyAsync(dst.rngc, src.rngc, keep * 8, cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaMemcpyAsync(dst.skey, src.skey, keep * 4, cudaMemcpyDeviceToDevice, c->stream));
    for (int q = 0; q < 3; ++q)
      CK(cudaMemcpyAsync(dst.force + q * ncap, src.force + q * c->cap, keep * 8, cudaMemcpyDeviceToDevice,
                         c->stream));
  }
  if (c->grid_valid && c->start) CK(cudaMemsetAsync(c->start, 0, (c->bins_cap + 1) * 4, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  free_soa(c->S[0]);
  free_soa(c->S[1]);
  cudaFree(c->newpd);
  c->S[0] = S2[0];
  c->S[1] = S2[1];
  c->cur = 0;
  c->newpd = np;
  c->pos_in_new = true;
  c->grid_valid = false;
  cudaFree(c->key); cudaFree(c->rank); cudaFree(c->nv); cudaFree(c->nn);
  cudaFree(c->st_parent); cudaFree(c->st_pd); cudaFree(c->st_vol); cudaFree(c->st_tag);
  cudaFree(c->pf);
  c->pf = nullptr;
  cudaFree(c->pf2);
  c->pf2 = nullptr;
  c->pf2_cap = 0;
  CK(dalloc(&c->pf, ncap));
  CK(dalloc(&c->key, ncap + 1));   // compact_population writes the survivor count at [n <= cap]
  CK(dalloc(&c->rank, ncap + 1));
  cudaFree(c->ctiles);
  c->ctiles = nullptr;
  CK(dalloc(&c->ctiles, ncap / kScanTile + 2));
  CK(dalloc(&c->nv, ncap));
  CK(dalloc(&c->nn, ncap));
  CK(cudaMemsetAsync(c->nv, 0, ncap, c->stream));
  CK(cudaMemsetAsync(c->nn, 0, ncap, c->stream));
  CK(dalloc(&c->st_parent, ncap));
  CK(dalloc(&c->st_pd, ncap));
  CK(dalloc(&c->st_vol, ncap));
  CK(dalloc(&c->st_tag, ncap));
  c->cap = ncap;
  cudaFree(c->holes);  // the compaction scratch follows the capacity
  c->holes = nullptr;
  c->holes_cap = 0;
  CK(dalloc(&c->holes, ncap));
  c->holes_cap = ncap;
  if (c->rec_evals) {
    cudaFree(c->evc);
    c->evc = nullptr;
    c->evc_cap = 0;
    CK(dalloc(&c->evc, ncap));
    CK(cudaMemsetAsync(c->evc, 0, ncap * sizeof(unsigned int), c->stream));
    c->evc_cap = ncap;
  }
  return ABS_OK;
}

// uid-indexed arrays (division marks + their scan tiles), sized by the uid
// space, not by the agent capacity: in a multi-domain run every rank holds
// the global uid space but only its own agents. Zero between iterations.
int ensure_uid_space(abs_gpu_ctx* c, unsigned long long want) {
  if (want <= c->uid_cap && c->div_mark && (!c->defer_commit || c->div_mark_g)) return ABS_OK;
  const unsigned long long ncap = std::max<unsigned long long>({want + want / 2, c->uid_cap, 1024});
  CK(cudaStreamSynchronize(c->stream));
  cudaFree(c->div_mark);
  cudaFree(c->div_mark_g);
  cudaFree(c->tiles64);
  cudaFree(c->rmark);
  cudaFree(c->hole_at);
  c->div_mark = nullptr;
  c->div_mark_g = nullptr;
  c->rmark = nullptr;
  c->hole_at = nullptr;
  CK(dalloc(&c->div_mark, ncap + 1));
  CK(cudaMemsetAsync(c->div_mark, 0, (ncap + 1) * 4, c->stream));
  CK(dalloc(&c->rmark, ncap + 1));
  CK(cudaMemsetAsync(c->rmark, 0, (ncap + 1) * 4, c->stream));
  CK(dalloc(&c->hole_at, ncap + 1));
  if (c->defer_commit) {
    CK(dalloc(&c->div_mark_g, ncap + 1));
    CK(cudaMemsetAsync(c->div_mark_g, 0, (ncap + 1) * 4, c->stream));
  }
  CK(dalloc(&c->tiles64, (ncap + kScanTile) / kScanTile + 2));
  c->uid_cap = ncap;
  return ABS_OK;
}

int ensure_bins(abs_gpu_ctx* c, unsigned long long want) {
  if (want <= c->bins_cap) return ABS_OK;
  unsigned long long nb = std::max<unsigned long long>(2 * want, 4096);  // growing domains: few retries
  cudaFree(c->start);
  cudaFree(c->tiles);
  cudaFree(c->scan_state);
  CK(dalloc(&c->start, nb + 1));
  CK(cudaMemsetAsync(c->start, 0, (nb + 1) * 4, c->stream));
  CK(dalloc(&c->tiles, nb / kScanTile + 2));
  // single-pass scan: per-tile (epoch, flag, value) words + two tile tickets
  CK(dalloc(&c->scan_state, (nb + 1) / kScanTile + 4));
  CK(cudaMemsetAsync(c->scan_state, 0, ((nb + 1) / kScanTile + 4) * 8, c->stream));
  c->bins_cap = nb;
  c->grid_valid = false;
  return ABS_OK;
}

// The cell table's scan in one launch (k_scan_onepass).
template <typename T>
void launch_scan(abs_gpu_ctx* c, T* data, const unsigned long long* len_dev, unsigned long long len_cap,
                 T* tiles, const int* err);

bool env_flag(const char* name, bool dflt) {
  const char* e = std::getenv(name);
  return e ? std::strcmp(e, "0") != 0 : dflt;
}

// ABSIM_SYNC_CHECK=1 (debugging): synchronise after the marked launches and
// report the first one that faulted (direct launches only; graphs are off).
void sync_check(abs_gpu_ctx* c, const char* what) {
  static const bool on = env_flag("ABSIM_SYNC_CHECK", false);
  if (!on) return;
  cudaError_t e = cudaPeekAtLastError();
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) {
    std::fprintf(stderr, "absim: %s failed: %s (iteration %llu)\n", what, cudaGetErrorString(e), c->iteration);
    std::abort();
  }
}

void launch_scan_cells(abs_gpu_ctx* c, const unsigned long long* len_dev, unsigned long long len_cap,
                       const int* err) {
  static const bool onepass = env_flag("ABSIM_ONEPASS", true);
  if (!onepass) {
    launch_scan<unsigned int>(c, c->start, len_dev, len_cap, c->tiles, err);
    return;
  }
  const unsigned int blocks = static_cast<unsigned int>(std::max<unsigned long long>(1, (len_cap + kScanTile - 1) / kScanTile));
  if (((c->scan_epoch + 1) & kScanEpochMask) == 0) {  // the tag wraps: no stale tile word may match it
    cudaMemsetAsync(c->scan_state, 0, ((c->bins_cap + 1) / kScanTile + 4) * 8, c->stream);
    ++c->scan_epoch;
  }
  k_scan_onepass<<<blocks, kThreads, 0, c->stream>>>(c->start, len_dev, c->scan_state, ++c->scan_epoch, err);
  ++c->launches;
}

template <typename T>
void launch_scan(abs_gpu_ctx* c, T* data, const unsigned long long* len_dev, unsigned long long len_cap,
                 T* tiles, const int* err) {
  const unsigned int nt = static_cast<unsigned int>((len_cap + kScanTile - 1) / kScanTile);
  const unsigned int blocks = std::max(1u, nt);
  k_scan_tiles<T><<<blocks, kThreads, 0, c->stream>>>(data, len_dev, tiles, err);
  k_scan_partials<T><<<1, kThreads, 0, c->stream>>>(tiles, len_dev, err);
  k_scan_apply<T><<<blocks, kThreads, 0, c->stream>>>(data, len_dev, tiles, err);
  c->launches += 3;
}

StepArgs step_args(const abs_gpu_ctx* c, unsigned long long iteration) {
  StepArgs a{};
  a.seed = c->cfg.seed;
  a.iteration = iteration;
  a.dt = c->cfg.simulation_time_step;
  a.k = c->cfg.repulsion_coefficient;
  a.max_disp = c->cfg.max_displacement;
  a.threshold2 = c->cfg.force_threshold * c->cfg.force_threshold;
  for (int q = 0; q < 8; ++q) a.mp[q] = c->cfg.model_params[q];
  a.model = c->cfg.model;
  a.detect_static = c->cfg.detect_static_agents;
  a.record_forces = c->cfg.record_forces;
  a.brute = brute_env(c);
  a.evc = c->rec_evals ? c->evc : nullptr;
  a.track_disp = c->track_now ? 1 : 0;
  return a;
}

// Bin rows are stored in y-blocks of 2^shift rows (row_of, kernels.cuh).
// ABSIM_ROW_BLOCK = rows per block (power of two; 0 = one block, i.e.
// z-major rows); default 32 (c4 @ 2^26 k_force: z-major 25.9 ms, 8: 25.8,
// 16: 26.1, 32: 25.3, 64: 28.9; c3 step 1.67 -> 1.54 ms at 16).
unsigned int row_block_shift() {
  static const unsigned int v = [] {
    const char* e = std::getenv("ABSIM_ROW_BLOCK");
    const long x = e ? std::atol(e) : 32;
    if (x <= 0) return ~0u;
    unsigned int sh = 0;
    while ((1l << (sh + 1)) <= x && sh < 12) ++sh;
    return sh;
  }();
  return v;
}

// Sub-bins per box edge: y/z rows finer than x (the x extent of a row is
// trimmed to the sphere's cross-section, so x resolution matters less).
// Auto (bins_per_box == 0): when the typical query radius 0.5 (d + dmax) is
// close to the box (mean d / dmax > 0.75, e.g. config 1) all 27 boxes are
// needed anyway and the box-lockstep walk (bins == boxes) wins; with a wide
// diameter spread (config 4) 2x2 sub-bins in y/z and 3 along x cut the
// candidates ~2x (c4 @ 2^24: 2x2x2 7.77 ms, 3 along x 7.50 ms, 2x3x3 8.55 ms).
unsigned int bins_yz(const abs_gpu_ctx* c) {
  if (c->cfg.model == ABS_MODEL_SIR || brute_env(c)) return 1u;
  const int b = c->cfg.bins_per_box;
  return b <= 0 ? c->auto_bins : static_cast<unsigned int>(std::min(b, 4));
}
unsigned int bins_x(const abs_gpu_ctx* c) {  // auto: 3 along x with 2x2 in y/z (c4 sweep)
  if (c->cfg.model == ABS_MODEL_SIR || brute_env(c)) return 1u;
  const int b = c->cfg.bins_per_box_x;
  return b <= 0 ? (c->auto_bins == 2u ? 3u : c->auto_bins) : static_cast<unsigned int>(std::min(b, 4));
}

// The fp32 copy `pf` is written by the re-bin only when the force kernel's
// fp32-classified walk will read it (sub-binned grids; not SIR, not box mode).
bool uses_f32_walk(const abs_gpu_ctx* c) {
  return c->cfg.model != ABS_MODEL_SIR && !(bins_x(c) == 1u && bins_yz(c) == 1u);
}

void launch_commit(abs_gpu_ctx* c);

constexpr unsigned long long kSortChunk = 4096;

// Radix-sort scratch of the Morton sort and the kd-tree build, sized by the capacity.
int ensure_sort_scratch(abs_gpu_ctx* c) {
  if (c->sort_cap == c->cap) return ABS_OK;
  for (int b = 0; b < 2; ++b) {
    cudaFree(c->sort_k[b]);
    cudaFree(c->sort_i[b]);
    c->sort_k[b] = nullptr;
    c->sort_i[b] = nullptr;
  }
  cudaFree(c->sort_hist); cudaFree(c->sort_tiles); cudaFree(c->sort_hlen);
  c->sort_hist = nullptr;
  c->sort_tiles = nullptr;
  c->sort_hlen = nullptr;
  c->sort_cap = 0;
  const unsigned long long blocks = (c->cap + kSortChunk - 1) / kSortChunk;
  for (int b = 0; b < 2; ++b) {
    CK(dalloc(&c->sort_k[b], c->cap));
    CK(dalloc(&c->sort_i[b], c->cap));
  }
  const unsigned long long hlen = 256ull * blocks;
  CK(dalloc(&c->sort_hist, hlen + 1));
  CK(dalloc(&c->sort_tiles, hlen / kScanTile + 2));
  CK(dalloc(&c->sort_hlen, 1));
  k_set_u64<<<1, 1, 0, c->stream>>>(c->sort_hlen, hlen);  // a kernel: capturable in a graph
  c->sort_cap = c->cap;
  return ABS_OK;
}

#include "kdtree.cuh"

// Environment::update: reduce, size, bin, scan, scatter into S[cur^1].
void launch_env_update(abs_gpu_ctx* c, unsigned long long iteration, int may_add, bool in_step = false,
                       int list_mode = 0, double skin = 0.0) {
  const int nb = agent_blocks(c);
  const unsigned long long* nbins_dev = &c->g->nbins;
  static const bool fused = env_flag("ABSIM_FUSED_FINALIZE", true);
  if (c->grid_valid && !fused) {  // previous cell table still holds scanned offsets
    k_zero_u32<<<grid_blocks(c, c->bins_cap), kThreads, 0, c->stream>>>(c->start, nbins_dev, 1, &c->g->err, c->bins_cap + 1);
    sync_check(c, "k_zero_u32");
    ++c->launches;
  }
  const Pd* pos = cur_pos(c);
  const FinArgs fa{c->cfg.fixed_box_length, brute_env(c), bins_x(c), bins_yz(c), row_block_shift(),
                   c->bins_cap, c->cap, c->uid_cap, may_add, iteration, list_mode, skin, in_step ? 1 : 0};
  if (fused) {
    k_reduce_finalize<<<nb, kThreads, 0, c->stream>>>(pos, c->g, fa, c->grid_valid ? c->start : nullptr);
    sync_check(c, "k_reduce_finalize");
  } else {
    k_reduce<<<nb, kThreads, 0, c->stream>>>(pos, c->g);
    sync_check(c, "k_reduce");
    k_finalize<<<1, 32, 0, c->stream>>>(c->g, fa);
    sync_check(c, "k_finalize");
    ++c->launches;
  }
  k_key<<<nb, kThreads, 0, c->stream>>>(pos, c->g, c->start, c->key, c->rank);
  sync_check(c, "k_key");
  c->launches += 2;
  launch_scan_cells(c, nbins_dev, c->bins_cap, &c->g->err);
  const int nxt = c->cur ^ 1;
  // inside an iteration without static detection (and not SIR, whose
  // partners hold infection times) k_force rewrites every agent's partners
  const bool carry_partners = !in_step || c->cfg.detect_static_agents || c->cfg.model == ABS_MODEL_SIR;
  // static detection inside an iteration: the scatter also lists the agents whose neighbours k_mark
  // marks (c->holes is free during the iteration; the kd gather would re-order the slots, so not there)
  c->marks_listed = in_step && c->cfg.detect_static_agents && iteration > 0 && !kd_env(c);
  auto scatter = [&](auto kernel) {
    kernel<<<nb, kThreads, 0, c->stream>>>(pos, c->S[c->cur], c->S[nxt], c->pf, c->start, c->key, c->rank, c->g, c->cap,
                                           c->cfg.model == ABS_MODEL_PROLIFERATION, c->cfg.record_forces,
                                           uses_f32_walk(c) || list_mode == 2, -1, uses_ext(c->cfg),
                                           carry_partners ? 1 : 0, c->cfg.model != ABS_MODEL_NONE ? 1 : 0, c->holes,
                                           &c->g->mark_n);
  };
  if (c->marks_listed) scatter(k_scatter<true>);
  else scatter(k_scatter<false>);
                                        sync_check(c, "k_scatter");
  ++c->launches;
  c->cur = nxt;
  c->pos_in_new = false;
  c->grid_valid = true;
  c->list_valid = false;  // storage re-ordered (a list build follows in list mode 2)
  if (kd_env(c) && kd_build(c) != ABS_OK) {  // KdTreeEnvironment::update on top of the single box
    c->kd_valid = false;
    c->kd_failed = true;  // reported by the caller (an empty tree would silently find no neighbours)
  }
}


// ABSIM_STATIC_PREPASS=0: static agents settled inside the force sweep (A/B)
bool static_prepass() {
  static const bool v = env_flag("ABSIM_STATIC_PREPASS", true);
  return v;
}

constexpr int kForceSmemBox = kMaxContacts * kForceThreads * 4;  // contact lists only
constexpr int kForceSmemF32 = (kMaxRows + kMaxRows / 2 + kMaxContacts) * kForceThreads * 4;
static_assert(kMaxRows % 2 == 0, "16-bit bound array packs two rows per word");

template <int MODEL, bool STATIC, bool RECORD, int WALK>
void launch_gather_f(abs_gpu_ctx* c, Soa& S, const StepArgs& a) {
  static int blocks = 0;  // per template instance
  constexpr int smem = WALK >= 2 ? kForceSmemBox : kForceSmemF32;
  if (!blocks) {
    cudaFuncSetAttribute(k_force<MODEL, STATIC, RECORD, WALK>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    blocks = force_blocks(c, k_force<MODEL, STATIC, RECORD, WALK>, smem);
  }
  const unsigned int* work = nullptr;
  if (STATIC && a.iteration != 0 && static_prepass()) {  // iteration 0: nobody is static (simulation.cpp:335-349)
    // c->rank is free after k_mark (it listed the marking agents there)
    k_static_pass<<<agent_blocks(c), kThreads, 0, c->stream>>>(S, c->newpd, c->g, c->nv, c->nn,
                                                                       MODEL != ABS_MODEL_NONE, c->rank);
                                                                   sync_check(c, "k_static_pass");
    ++c->launches;
    work = c->rank;
  }
  k_force<MODEL, STATIC, RECORD, WALK><<<blocks, kForceThreads, smem, c->stream>>>(
      S, c->pf, c->newpd, c->g, c->g, c->start, c->nv, c->nn, a, c->cap, c->st_parent, c->st_pd, c->st_vol, c->div_mark,
      c->st_tag, work, c->rmark, kd_view(c));
  sync_check(c, "k_force");
}

template <int MODEL, bool STATIC, bool RECORD>
void launch_gather(abs_gpu_ctx* c, Soa& S, const StepArgs& a) {
  if (kd_env(c)) launch_gather_f<MODEL, STATIC, RECORD, 3>(c, S, a);
  else if (bins_x(c) == 1u && bins_yz(c) == 1u) launch_gather_f<MODEL, STATIC, RECORD, 2>(c, S, a);
  else launch_gather_f<MODEL, STATIC, RECORD, 1>(c, S, a);
}

template <int MODEL, bool STATIC>
void launch_force_t(abs_gpu_ctx* c, int, Soa& S, const StepArgs& a) {
  const bool box_mode = bins_x(c) == 1u && bins_yz(c) == 1u;
  if (MODEL == ABS_MODEL_COHERE) {  // its behaviour query lives in the gather kernel
    if (c->cfg.record_forces) launch_gather<MODEL, STATIC, true>(c, S, a);
    else launch_gather<MODEL, STATIC, false>(c, S, a);
    return;
  }
  if (c->cfg.record_forces) launch_gather<MODEL, STATIC, true>(c, S, a);
  else launch_gather<MODEL, STATIC, false>(c, S, a);
}

template <int MODEL>
void launch_force_m(abs_gpu_ctx* c, int nb, Soa& S, const StepArgs& a) {
  if (c->cfg.detect_static_agents) launch_force_t<MODEL, true>(c, nb, S, a);
  else launch_force_t<MODEL, false>(c, nb, S, a);
}

void launch_force(abs_gpu_ctx* c, int nb, Soa& S, const StepArgs& a) {
  switch (c->cfg.model) {
    case ABS_MODEL_PROLIFERATION: launch_force_m<ABS_MODEL_PROLIFERATION>(c, nb, S, a); break;
    case ABS_MODEL_DRIVE: launch_force_m<ABS_MODEL_DRIVE>(c, nb, S, a); break;
    case ABS_MODEL_GROW: launch_force_m<ABS_MODEL_GROW>(c, nb, S, a); break;
    case ABS_MODEL_GROW_DIVIDE: launch_force_m<ABS_MODEL_GROW_DIVIDE>(c, nb, S, a); break;
    case ABS_MODEL_COHERE: launch_force_m<ABS_MODEL_COHERE>(c, nb, S, a); break;
    case ABS_MODEL_GROW_DIVIDE_DIE: launch_force_m<ABS_MODEL_GROW_DIVIDE_DIE>(c, nb, S, a); break;
    default: launch_force_m<ABS_MODEL_NONE>(c, nb, S, a); break;
  }
}

void phase_mark(abs_gpu_ctx* c) {
  if (!c->timing) return;
  if (c->pev_used + 1 > c->pev.size()) {
    for (int q = 0; q < 320; ++q) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      c->pev.push_back(e);
    }
  }
  cudaEventRecord(c->pev[c->pev_used++], c->stream);
}

// Neighbour lists serve the mechanical step when the
// diameters are constant and one context owns the whole population: no
// behaviours, no static detection, no ghosts or grid override, the grid
// environment. ABSIM_NLIST=0 turns them off (A/B switch).
bool list_mode_ok(const abs_gpu_ctx* c) {
  static const bool on = env_flag("ABSIM_NLIST", true);
  return on && !c->list_off && c->cfg.neighbor_list >= 0 && c->cfg.model == ABS_MODEL_NONE &&
         !c->cfg.detect_static_agents && !brute_env(c) && !c->defer_commit && c->ghosts == 0 && !c->ov_on;
}

double list_skin(const abs_gpu_ctx* c) {
  if (c->cfg.neighbor_skin > 0.0) return c->cfg.neighbor_skin;
  return 0.2 * (c->host_dmax > 0.0 ? c->host_dmax : 1.0);
}

constexpr unsigned int kListKmaxInit = 64;
// A build must serve >= this many steps (the build iteration included) to pay
// off. c4 at 2^26 (ncu launch list, profiles/r2_*): build iteration 46.6 ms
// (re-bin 3.3 + k_list_build 28 + list step), list step 15.5 ms, re-bin + walk
// 29.3 ms: two steps lose (31 ms/step), three win (25.9), four 23.3.
// ABSIM_LIST_MIN_STEPS overrides (A/B switch).
double list_min_steps() {
  static const double v = [] {
    const char* e = std::getenv("ABSIM_LIST_MIN_STEPS");
    const double x = e ? std::atof(e) : 0.0;
    return x > 0.0 ? x : 3.0;
  }();
  return v;
}
constexpr unsigned int kListKmaxMax = 254;  // u8 counts (255 = overflow sentinel)

// List storage for the current population: [kmax][stride] u32 + u8 counts.
int ensure_lists(abs_gpu_ctx* c, unsigned int kmax) {
  const unsigned long long stride = std::max<unsigned long long>(32, (c->n + 31) / 32 * 32);
  if (c->pf2_cap < c->cap) {
    CK(cudaStreamSynchronize(c->stream));
    cudaFree(c->pf2);
    c->pf2 = nullptr;
    c->pf2_cap = 0;
    c->list_valid = false;
    CK(dalloc(&c->pf2, c->cap));
    c->pf2_cap = c->cap;
  }
  if (c->nl && stride <= c->nl_stride && kmax <= c->nl_kmax) return ABS_OK;
  const unsigned long long ns = std::max(stride, c->nl_stride);
  const unsigned int kk = std::max(kmax, c->nl_kmax);
  CK(cudaStreamSynchronize(c->stream));
  cudaFree(c->nl);
  cudaFree(c->nl_cnt);
  cudaFree(c->nl_ct);
  cudaFree(c->nl_nct);
  c->nl = nullptr;
  c->nl_cnt = nullptr;
  c->nl_ct = nullptr;
  c->nl_nct = nullptr;
  c->nl_stride = 0;
  c->nl_kmax = 0;
  c->list_valid = false;
  CK(dalloc(&c->nl, ns * kk));
  CK(dalloc(&c->nl_cnt, ns));
  CK(dalloc(&c->nl_ct, ns * kListContacts));
  CK(dalloc(&c->nl_nct, ns));
  c->nl_stride = ns;
  c->nl_kmax = kk;
  return ABS_OK;
}

cudaEvent_t* event_pair(abs_gpu_ctx* c, std::vector<cudaEvent_t>& v, size_t& used) {
  if (used + 2 > v.size()) {
    for (int q = 0; q < 256; ++q) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      v.push_back(e);
    }
  }
  used += 2;
  return &v[used - 2];
}

// One list iteration. kind 2: re-bin (the environment update), build the
// lists, force sweep over them; kind 1: bounds reduction + grid sizing +
// coverage check (finalize_grid), force sweep over the existing lists.
// Positions and their fp32 copies travel in pairs: (S[cur].pd, pf) and
// (newpd, pf2).
void launch_list_iteration(abs_gpu_ctx* c, unsigned long long iteration, int kind) {
  sync_check(c, "before list iteration");
  const StepArgs a = step_args(c, iteration);
  const double skin = list_skin(c);
  Pd* pin;
  Pd* pout;
  float4* fin;
  float4* fout;
  if (kind == 2) {
    launch_env_update(c, iteration, 0, true, 2, skin);
    static int blocks = 0;
    if (!blocks) {
      cudaFuncSetAttribute(k_list_build, cudaFuncAttributeMaxDynamicSharedMemorySize, kListSmem);
      blocks = force_blocks(c, k_list_build, kListSmem);
    }
    cudaEvent_t* ev = c->timing ? event_pair(c, c->bev, c->bev_used) : nullptr;
    if (ev) cudaEventRecord(ev[0], c->stream);
    k_list_build<<<blocks, kForceThreads, kListSmem, c->stream>>>(c->pf, c->g, c->start, c->nl, c->nl_cnt,
                                                                  c->nl_kmax, skin);
    if (ev) cudaEventRecord(ev[1], c->stream);
    sync_check(c, "k_list_build");
    ++c->launches;
    c->list_valid = true;
    pin = c->S[c->cur].pd;
    fin = c->pf;
    pout = c->newpd;
    fout = c->pf2;
    c->pos_in_new = true;
  } else {
    const FinArgs fa{c->cfg.fixed_box_length, brute_env(c), bins_x(c), bins_yz(c), row_block_shift(),
                     c->bins_cap, c->cap, c->uid_cap, 0, iteration, 1, skin, 1};
    const bool from_new = c->pos_in_new;
    pin = from_new ? c->newpd : c->S[c->cur].pd;
    fin = from_new ? c->pf2 : c->pf;
    pout = from_new ? c->S[c->cur].pd : c->newpd;
    fout = from_new ? c->pf : c->pf2;
    k_reduce_finalize<<<agent_blocks(c, 4), kThreads, 0, c->stream>>>(pin, c->g, fa,
                                                                          c->grid_valid ? c->start : nullptr);
    sync_check(c, "k_reduce_finalize(list)");
    ++c->launches;
    c->grid_valid = false;
    c->pos_in_new = !from_new;
  }
  phase_mark(c);  // after environment update
  static int scan_blocks = 0;
  if (!scan_blocks) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_list_scan, kThreads, 0);
    scan_blocks = c->sms * std::max(per_sm, 1);
  }
  cudaEvent_t* ev = c->timing ? event_pair(c, c->ev, c->ev_used) : nullptr;
  if (ev) cudaEventRecord(ev[0], c->stream);
  k_list_scan<<<scan_blocks, kThreads, 0, c->stream>>>(pin, fin, c->g, c->nl, c->nl_cnt, c->nl_kmax, c->nl_ct,
                                                       c->nl_nct, a.evc, c->start);
  sync_check(c, "k_list_scan");
  const int nb = agent_blocks(c);
  auto forces = [&](auto kernel) {
    kernel<<<nb, kThreads, 0, c->stream>>>(pin, pout, fout, c->S[c->cur], c->g, c->nl, c->nl_cnt, c->nl_kmax,
                                           c->nl_ct, c->nl_nct, a, c->cap, c->start);
  };
  if (c->cfg.record_forces) forces(k_list_forces<true>);
  else forces(k_list_forces<false>);
  if (ev) cudaEventRecord(ev[1], c->stream);
  sync_check(c, "k_list_forces");
  c->launches += 2;
  phase_mark(c);  // after agent ops
  phase_mark(c);  // no commit
}

#ifdef ABS_DEBUG
// Debug builds (direct launches, ABSIM_GRAPHS=0): the storage keys of a
// single-domain context are a permutation of [0, n).
void check_keys(abs_gpu_ctx* c, const char* where, unsigned long long iteration) {
  static const bool on = env_flag("ABSIM_CHECK_KEYS", false);
  if (!on) return;
  DevGrid h{};
  cudaStreamSynchronize(c->stream);
  cudaMemcpy(&h, c->g, sizeof h, cudaMemcpyDeviceToHost);
  if (h.err || h.nkeys != h.n) return;
  std::vector<unsigned int> k(h.n);
  if (h.n) cudaMemcpy(k.data(), c->S[c->cur].skey, h.n * 4, cudaMemcpyDeviceToHost);
  std::vector<char> seen(h.n, 0);
  for (unsigned long long i = 0; i < h.n; ++i) {
    if (k[i] >= h.n || seen[k[i]]) {
      std::fprintf(stderr, "absim: bad storage key %u at slot %llu of %llu (%s, iteration %llu, dup %d)\n", k[i], i,
                   h.n, where, iteration, k[i] < h.n);
      std::abort();
    }
    seen[k[i]] = 1;
  }
}
#else
inline void check_keys(abs_gpu_ctx*, const char*, unsigned long long) {}
#endif

void launch_iteration(abs_gpu_ctx* c, unsigned long long iteration, int kind = 0) {
  sync_check(c, "before iteration");
  if (c->rec_evals && c->evc) {  // static / ghost agents evaluate nothing this iteration
    cudaMemsetAsync(c->evc, 0, c->evc_cap * sizeof(unsigned int), c->stream);
  }
  if (kind == 1 || kind == 2) {
    launch_list_iteration(c, iteration, kind);
    return;
  }
  c->track_now = kind == 3;  // re-binning step whose displacement the list policy tracks
  check_keys(c, "iteration start (after the sort)", iteration);
  launch_env_update(c, iteration, adds_agents(c->cfg), true, kind == 3 ? 3 : 0);
  check_keys(c, "after the re-bin", iteration);
  phase_mark(c);  // after environment update
  if (c->cfg.model == ABS_MODEL_SIR) {
    const int nb = agent_blocks(c);
    const StepArgs a = step_args(c, iteration);
    Soa& S = c->S[c->cur];
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (c->timing) {  // the dominant kernel of config 5
      if (c->ev_used + 2 > c->ev.size()) {
        for (int q = 0; q < 256; ++q) {
          cudaEvent_t e;
          cudaEventCreate(&e);
          c->ev.push_back(e);
        }
      }
      e0 = c->ev[c->ev_used++];
      e1 = c->ev[c->ev_used++];
      cudaEventRecord(e0, c->stream);
    }
    k_sir<<<nb, kThreads, 0, c->stream>>>(S, c->newpd, c->g, c->start, c->nv, c->key, a);
    if (c->timing) cudaEventRecord(e1, c->stream);
    k_sir_commit<<<nb, kThreads, 0, c->stream>>>(S, c->g, c->nv, c->key);
    c->launches += 2;
    c->pos_in_new = true;
    phase_mark(c);  // after agent ops
    phase_mark(c);  // no commit
    return;
  }
  const int nb = agent_blocks(c);
  const StepArgs a = step_args(c, iteration);
  Soa& S = c->S[c->cur];
  if (c->cfg.detect_static_agents && iteration > 0) {
    // c->rank is free between the re-bin's scatter and the next k_key
    if (c->marks_listed) {  // listed by the re-bin's scatter
      k_mark<<<nb, kThreads, 0, c->stream>>>(S, c->g, c->start, c->nv, c->nn, c->holes);
      c->launches += 1;
    } else {
      k_mark_list<<<nb, kThreads, 0, c->stream>>>(S, c->g, c->rank);
      k_mark<<<nb, kThreads, 0, c->stream>>>(S, c->g, c->start, c->nv, c->nn, c->rank);
      c->launches += 2;
    }
  }
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (c->timing) {
    if (c->ev_used + 2 > c->ev.size()) {
      for (int q = 0; q < 256; ++q) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        c->ev.push_back(e);
      }
    }
    e0 = c->ev[c->ev_used++];
    e1 = c->ev[c->ev_used++];
    cudaEventRecord(e0, c->stream);
  }
  launch_force(c, nb, S, a);
  ++c->launches;
  if (c->timing) cudaEventRecord(e1, c->stream);
  c->pos_in_new = true;
  phase_mark(c);  // after agent ops (staticness marking, behaviours, forces, integration)
  if (adds_agents(c->cfg)) {
    if (c->cfg.detect_static_agents) {
      k_mark_new<<<nb, kThreads, 0, c->stream>>>(S, c->newpd, c->g, c->start, c->st_pd);
      ++c->launches;
    }
    if (!c->defer_commit) launch_commit(c);
    check_keys(c, "after the commit", iteration);
  }
  phase_mark(c);  // after commit
}

// CommitBuffer::commit for additions (commit.cpp:186-222): daughter uids
// uid_count + rank of the parent uid among all dividing parents (the
// single-thread creation order), appended in that order. Deferred commit
// (multi-domain): div_mark_g holds every rank's dividers (the caller summed
// the ranks' div_mark into it), giving global uid ranks, while this rank's
// own div_mark gives the local append slots.
// The removal half of CommitBuffer::commit (removals before additions,
// commit.cpp:164-185) for agents the loop staged (ABS_FLAG_REMOVED + key marks).
void launch_removals(abs_gpu_ctx* c, bool keys_in_list_order = false) {
  const int nb = agent_blocks(c);
  Soa& S = c->S[c->cur];
  unsigned int* tiles = reinterpret_cast<unsigned int*>(c->tiles64);
  launch_scan<unsigned int>(c, c->rmark, &c->g->nkeys, c->uid_cap, tiles, &c->g->err);
  if (!keys_in_list_order) {
    k_rem_holes<<<grid_blocks(c, c->uid_cap), kThreads, 0, c->stream>>>(c->rmark, c->g, c->hole_at);
    ++c->launches;
  }
  k_rem_rekey<<<nb, kThreads, 0, c->stream>>>(S, c->g, c->rmark, c->hole_at, c->key, c->rank);
  launch_scan<unsigned int>(c, c->rank, &c->g->n, c->cap, c->ctiles, &c->g->err);
  k_hole_list_d<<<nb, kThreads, 0, c->stream>>>(c->key, c->rank, c->g, c->holes);
  k_swap_move_d<<<nb, kThreads, 0, c->stream>>>(cur_pos(c), S, c->key, c->rank, c->holes, c->g, c->cap);
  k_rem_fin<<<1, 32, 0, c->stream>>>(c->g, c->rank, c->rmark);
  k_zero_marks<<<grid_blocks(c, c->uid_cap), kThreads, 0, c->stream>>>(c->rmark, c->g);
  c->launches += 5;
}

void launch_commit(abs_gpu_ctx* c) {
  if (removes_agents(c->cfg)) launch_removals(c);
  const int nb = agent_blocks(c);
  Soa& S = c->S[c->cur];
  const unsigned long long* uc = &c->g->uid_count;
  unsigned int* tiles = reinterpret_cast<unsigned int*>(c->tiles64);
  launch_scan<unsigned int>(c, c->div_mark, uc, c->uid_cap, tiles, &c->g->err);
  if (c->defer_commit) launch_scan<unsigned int>(c, c->div_mark_g, uc, c->uid_cap, tiles, &c->g->err);
  const unsigned int* grank = c->defer_commit ? c->div_mark_g : c->div_mark;
  k_append<<<nb, kThreads, 0, c->stream>>>(S, c->newpd, c->g, c->st_parent, c->st_pd, c->st_vol, c->st_tag,
                                           c->div_mark, grank, c->cap, c->cfg.record_forces);
  // counts first (reads the scan total grank[uid_count]), then clear the
  // marks over the grown range [0, uid_count]
  k_commit_fin<<<1, 32, 0, c->stream>>>(c->g, grank);
  k_zero_marks<<<grid_blocks(c, c->uid_cap), kThreads, 0, c->stream>>>(c->div_mark, c->g);
  if (c->defer_commit) k_zero_marks<<<grid_blocks(c, c->uid_cap), kThreads, 0, c->stream>>>(c->div_mark_g, c->g);
  c->launches += c->defer_commit ? 4 : 3;
}

int read_grid(abs_gpu_ctx* c, DevGrid* h) {
  if (c->hgrid) {  // mapped mirror: no copy-engine work (see k_grid_out)
    k_grid_out<<<1, 64, 0, c->stream>>>(c->g, c->hgrid);
    ++c->launches;
    CK(cudaStreamSynchronize(c->stream));
    std::memcpy(h, c->hgrid, sizeof(DevGrid));
  } else {
    CK(cudaMemcpyAsync(h, c->g, sizeof(DevGrid), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  }
  c->n = h->n;
  return ABS_OK;
}

int dzero(abs_gpu_ctx* c, void* p, unsigned long long bytes) {
  if (!bytes) return ABS_OK;
  k_zero_bytes<<<grid_blocks(c, (bytes + 15) / 16), kThreads, 0, c->stream>>>(static_cast<unsigned char*>(p), bytes);
  ++c->launches;
  return ABS_OK;
}

int map_dev_err(abs_gpu_ctx* c, const DevGrid& h) {
  switch (h.err) {
    case kErrNone: return ABS_OK;
    case kErrNonFinite:
      return set_err(c, ABS_ERR_NONFINITE, "operation 'environment update' failed at iteration " +
                                               std::to_string(h.failed_iteration) + ": agent positions are not finite");
    case kErrFixedBox:
      return set_err(c, ABS_ERR_FIXED_BOX, "operation 'environment update' failed at iteration " +
                                               std::to_string(h.failed_iteration) +
                                               ": fixed box length is smaller than the largest agent diameter");
    case kErrSlabs:
      return set_err(c, ABS_ERR_STATE, "slab decomposition at iteration " + std::to_string(h.failed_iteration) +
                                           ": fewer than 2 z box layers per rank");
    case kErrQueryRadius:
      return set_err(c, ABS_ERR_INVALID_ARGUMENT, "operation 'behaviours' failed at iteration " +
                                                      std::to_string(h.failed_iteration) +
                                                      ": query radius exceeds the grid box length");
    case kErrBoxBudget:
      return set_err(c, ABS_ERR_BOX_BUDGET, "operation 'environment update' failed at iteration " +
                                                std::to_string(h.failed_iteration) + ": grid would exceed the box budget");
    default: return set_err(c, ABS_ERR_STATE, "internal retry state leaked");
  }
}

int clear_dev_err(abs_gpu_ctx* c) {
  CK(cudaMemsetAsync(&c->g->err, 0, sizeof(int), c->stream));
  return ABS_OK;
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

void abs_gpu_default_config(abs_gpu_config* cfg) {
  std::memset(cfg, 0, sizeof(*cfg));
  cfg->seed = 42;
  cfg->simulation_time_step = 0.1;
  cfg->repulsion_coefficient = 2.0;
  cfg->max_displacement = 3.0;
  cfg->force_threshold = 0.0;
  cfg->fixed_box_length = 0.0;
  cfg->record_forces = 1;
  cfg->bins_per_box = 0;
}

const char* abs_gpu_last_error(const abs_gpu_ctx* c) { return c ? c->err.c_str() : g_create_err.c_str(); }

int abs_gpu_create(const abs_gpu_config* cfg, int device, abs_gpu_ctx** out) {
  abs_gpu_ctx* c = nullptr;
  if (!cfg || !out) return set_err(nullptr, ABS_ERR_INVALID_ARGUMENT, "null argument");
  // SimulationParams::validate (params.cpp:44-72), hot-path fields
  if (cfg->fixed_box_length < 0.0) return set_err(nullptr, ABS_ERR_INVALID_ARGUMENT, "fixed_box_length must be >= 0");
  if (!(cfg->simulation_time_step > 0.0))
    return set_err(nullptr, ABS_ERR_INVALID_ARGUMENT, "simulation_time_step must be > 0");
  if (cfg->repulsion_coefficient < 0.0)
    return set_err(nullptr, ABS_ERR_INVALID_ARGUMENT, "repulsion_coefficient must be >= 0");
  if (!(cfg->max_displacement > 0.0)) return set_err(nullptr, ABS_ERR_INVALID_ARGUMENT, "max_displacement must be > 0");
  if (cfg->force_threshold < 0.0) return set_err(nullptr, ABS_ERR_INVALID_ARGUMENT, "force_threshold must be >= 0");
  if (cfg->model < 0 || cfg->model > 7) return set_err(nullptr, ABS_ERR_INVALID_ARGUMENT, "unknown model");
  if (cfg->environment != ABS_ENV_UNIFORM_GRID && cfg->environment != ABS_ENV_BRUTE_FORCE &&
      cfg->environment != ABS_ENV_KD_TREE)
    return set_err(nullptr, ABS_ERR_INVALID_ARGUMENT, "unknown environment kind");
  // params.cpp:52-55
  if (cfg->sorting_frequency > 0 && cfg->environment != ABS_ENV_UNIFORM_GRID)
    return set_err(nullptr, ABS_ERR_INVALID_ARGUMENT, "sorting requires the uniform_grid environment");
  if (cfg->model == ABS_MODEL_SIR && cfg->environment != ABS_ENV_UNIFORM_GRID)
    return set_err(nullptr, ABS_ERR_INVALID_ARGUMENT, "the periodic SIR model runs on the uniform grid");
  if (cfg->model == ABS_MODEL_GROW_DIVIDE && !(cfg->model_params[2] > 0.0))
    return set_err(nullptr, ABS_ERR_INVALID_ARGUMENT, "GrowDivide needs an initial diameter > 0");
  if (cfg->model == ABS_MODEL_COHERE && !(cfg->model_params[0] > 0.0))
    return set_err(nullptr, ABS_ERR_INVALID_ARGUMENT, "Cohere needs an attraction radius > 0");
  if (cfg->model == ABS_MODEL_SIR && !(cfg->model_params[0] > 0.0 && cfg->model_params[1] > 0.0 &&
                                       cfg->model_params[0] >= 3.0 * cfg->model_params[1]))
    return set_err(nullptr, ABS_ERR_INVALID_ARGUMENT, "SIR needs L >= 3 r > 0");
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
    return set_err(nullptr, ABS_ERR_NO_DEVICE, "no CUDA device available");
  if (device < 0 || device >= count) return set_err(nullptr, ABS_ERR_INVALID_ARGUMENT, "bad device index");
  if (cudaSetDevice(device) != cudaSuccess) return set_err(nullptr, ABS_ERR_CUDA, "cudaSetDevice failed");
  c = new abs_gpu_ctx();
  c->cfg = *cfg;
  c->device = device;
  cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device);
  CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  c->own_stream = true;
  CK(cudaMalloc(&c->g, sizeof(DevGrid)));
  DevGrid h{};
  h.red[0] = h.red[1] = h.red[2] = kInfOrdLo;
  h.red[3] = h.red[4] = h.red[5] = kInfOrdHi;
  h.red[6] = kZeroOrd;
  h.dims[0] = h.dims[1] = h.dims[2] = 1;
  h.B[0] = h.B[1] = h.B[2] = 1;
  CK(cudaMemcpy(c->g, &h, sizeof h, cudaMemcpyHostToDevice));
  // small host-visible results (grid record, ingest partials) through mapped
  // page-locked memory; on failure read_grid falls back to cudaMemcpy
  if (cudaHostAlloc(reinterpret_cast<void**>(&c->hgrid), sizeof(DevGrid), cudaHostAllocMapped) != cudaSuccess) {
    c->hgrid = nullptr;
    cudaGetLastError();
  }
  CK(cudaHostAlloc(reinterpret_cast<void**>(&c->ingest_part), (2ull * c->sms * 8 + 2) * sizeof(double),
                   cudaHostAllocMapped));
  int rc = ensure_capacity(c, std::max<unsigned long long>(cfg->capacity, 1024), 0);
  if (!rc) rc = ensure_uid_space(c, 1024);
  if (rc) { abs_gpu_destroy(c); return set_err(nullptr, rc, "allocation failed"); }
  rc = ensure_bins(c, 1 << 16);
  if (rc) { abs_gpu_destroy(c); return set_err(nullptr, rc, "allocation failed"); }
  if (cfg->model == ABS_MODEL_SIR) {  // periodic cube [0, L)^3 in boxes of L / floor(L / r)
    const double L = cfg->model_params[0], r = cfg->model_params[1];
    unsigned int D = static_cast<unsigned int>(std::floor(L / r));
    if (D < 3) D = 3;
    const double grid[5] = {0.0, 0.0, 0.0, L / static_cast<double>(D), r};
    const unsigned int dims[3] = {D, D, D};
    rc = abs_gpu_set_grid_override(c, grid, dims);
    if (rc) { abs_gpu_destroy(c); return set_err(nullptr, rc, "grid setup failed"); }
  }
  *out = c;
  return ABS_OK;
}

static void free_sort_scratch(abs_gpu_ctx* c);
void decomp_destroy(abs_gpu_ctx* c);  // decomp.cuh

int abs_gpu_destroy(abs_gpu_ctx* c) {
  if (!c) return ABS_OK;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  free_soa(c->S[0]);
  free_soa(c->S[1]);
  cudaFree(c->newpd); cudaFree(c->pf); cudaFree(c->g); cudaFree(c->start); cudaFree(c->key); cudaFree(c->rank);
  cudaFree(c->tiles); cudaFree(c->tiles64); cudaFree(c->scan_state); cudaFree(c->nv); cudaFree(c->nn);
  cudaFree(c->xcounts); cudaFree(c->holes); cudaFree(c->nl); cudaFree(c->nl_cnt); cudaFree(c->evc);
  cudaFree(c->pf2); cudaFree(c->nl_ct); cudaFree(c->nl_nct); cudaFree(c->ctiles);
  cudaFree(c->kd_axis); cudaFree(c->kd_lmax); cudaFree(c->kd_rmin); cudaFree(c->kd_bbox);
  if (c->hxcounts) cudaFreeHost(c->hxcounts);
  cudaFree(c->st_parent);
  cudaFree(c->st_pd); cudaFree(c->st_vol); cudaFree(c->st_tag); cudaFree(c->div_mark); cudaFree(c->div_mark_g);
  cudaFree(c->rmark); cudaFree(c->hole_at);
  if (c->ingest_part) cudaFreeHost(c->ingest_part);
  if (c->hgrid) cudaFreeHost(c->hgrid);
  for (int b = 0; b < 2; ++b) {
    cudaFree(c->fin[b]);
    cudaFree(c->fout[b]);
    for (cudaEvent_t e : {c->in_ready[b], c->in_free[b], c->out_ready[b], c->out_free[b]})
      if (e) cudaEventDestroy(e);
  }
  for (cudaGraphExec_t e : c->gexec)
    if (e) cudaGraphExecDestroy(e);
  if (c->h2d) cudaStreamDestroy(c->h2d);
  if (c->d2h) cudaStreamDestroy(c->d2h);
  free_sort_scratch(c);
  for (cudaEvent_t e : c->ev) cudaEventDestroy(e);
  for (cudaEvent_t e : c->pev) cudaEventDestroy(e);
  for (cudaEvent_t e : c->bev) cudaEventDestroy(e);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  decomp_destroy(c);
  delete c;
  return ABS_OK;
}

// Upload, stage 1: everything stream-ordered (no host synchronisation).
// Host coordinate arrays are DMA'd into the staging area; device arrays
// (kind == cudaMemcpyDeviceToDevice) are read in place by k_ingest. Only
// kernels touch the compute stream besides the caller's own host copies, so a
// frame upload never waits behind another stream's bulk DMA.
static int upload_enqueue(abs_gpu_ctx* c, unsigned long long n, unsigned long long uid_count,
                          cudaMemcpyKind kind, const uint64_t* uid, const double* x, const double* y,
                          const double* z, const double* d, const uint8_t* mask, const double* volume,
                          const uint8_t* flags, const uint32_t* partners, int* blocks_out) {
  if (!c) return ABS_ERR_INVALID_ARGUMENT;
  if (n && (!x || !y || !z || !d)) return set_err(c, ABS_ERR_INVALID_ARGUMENT, "null coordinate array");
  if (n >= 0xFFFFFFF0ull) return set_err(c, ABS_ERR_INVALID_ARGUMENT, "too many agents");
  cudaSetDevice(c->device);
  const bool host = kind == cudaMemcpyHostToDevice;
  // uid_count == 0 with explicit uids: derive it (host scan); otherwise the
  // device checks every uid < uid_count during ingest
  const unsigned long long uid_limit = (uid && uid_count) ? uid_count : 0;
  if (uid && host && !uid_count) {
    for (unsigned long long i = 0; i < n; ++i) uid_count = std::max<unsigned long long>(uid_count, uid[i] + 1);
  }
  if (uid && !host && !uid_count) return set_err(c, ABS_ERR_INVALID_ARGUMENT, "device upload with uids needs uid_count");
  uid_count = std::max<unsigned long long>(uid_count, n);
  int rc = ensure_capacity(c, std::max<unsigned long long>(c->cap, 2 * n + 1024), 0);
  if (rc) return rc;
  if (adds_agents(c->cfg)) {  // uid-indexed division marks: uids cannot outgrow
    // uid_count + capacity before a capacity retry, so no uid-space retry either
    rc = ensure_uid_space(c, std::max<unsigned long long>(2 * uid_count, uid_count + c->cap) + 1024);
    if (rc) return rc;
  }
  c->pending_commit = false;
  Soa& S = c->S[c->cur];
  const double *dx = x, *dy = y, *dz = z, *dd = d;
  const unsigned char* dmask = mask;
  if (host && n) {  // contiguous H2D into the staging area, interleaved on the device
    double* st = reinterpret_cast<double*>(c->st_pd);
    CK(cudaMemcpyAsync(st, x, n * 8, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(st + n, y, n * 8, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(st + 2 * n, z, n * 8, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(st + 3 * n, d, n * 8, cudaMemcpyHostToDevice, c->stream));
    dx = st; dy = st + n; dz = st + 2 * n; dd = st + 3 * n;
    if (mask) {
      CK(cudaMemcpyAsync(c->key, mask, n, cudaMemcpyHostToDevice, c->stream));
      dmask = reinterpret_cast<const unsigned char*>(c->key);
    }
  }
  if (uid) CK(cudaMemcpyAsync(S.uid, uid, n * 8, kind, c->stream));
  if (volume) CK(cudaMemcpyAsync(S.vol, volume, n * 8, kind, c->stream));
  if (flags) CK(cudaMemcpyAsync(S.flags, flags, n, kind, c->stream));
  else dzero(c, S.flags, n);
  if (partners) CK(cudaMemcpyAsync(S.partners, partners, n * 4, kind, c->stream));
  else dzero(c, S.partners, n * 4);
  if (c->cfg.record_forces) dzero(c, S.force, 3 * c->cap * 8);
  k_grid_reset<<<1, 64, 0, c->stream>>>(c->g, n, uid_count);
  ++c->launches;
  const int ib = grid_blocks(c, n);
  if (n) {
    k_ingest<<<ib, kThreads, 0, c->stream>>>(dx, dy, dz, dd, dmask, n, uid == nullptr, volume == nullptr,
                                             c->cfg.model != ABS_MODEL_NONE, c->newpd, S, c->g,
                                             c->cfg.model == ABS_MODEL_SIR, c->cfg.seed, c->ingest_part, uid_limit);
    ++c->launches;
  }
  // the cell table is a counter array between iterations: always start clean
  dzero(c, c->start, (c->bins_cap + 1) * 4);
  c->pos_in_new = true;
  c->grid_valid = false;
  c->iteration = 0;
  c->ghosts = flags ? n : 0;  // uploaded flags may carry ABS_FLAG_GHOST
  c->n = n;
  *blocks_out = ib;
  return ABS_OK;
}

// Upload, stage 2: wait for the ingest, check the inputs, pick the sub-bins.
static int upload_finish(abs_gpu_ctx* c, unsigned long long n, int ib) {
  DevGrid h{};
  int rc = read_grid(c, &h);  // synchronises the stream
  if (rc) return rc;
  const unsigned int bad = h.bad_input;
  if (n && !bad) {  // Sub-bins: bins == boxes when the typical radius is close to the box (see bins_yz)
    double sum = 0.0, mx = 0.0;
    for (int b = 0; b < ib; ++b) {
      sum += c->ingest_part[2 * b];
      mx = c->ingest_part[2 * b + 1] > mx ? c->ingest_part[2 * b + 1] : mx;
    }
    c->auto_bins = (mx > 0.0 && sum / static_cast<double>(n) > 0.75 * mx) ? 1u : 2u;
    c->host_dmax = mx;
  }
  c->list_valid = false;
  if (bad) {
    c->n = 0;
    CK(cudaMemsetAsync(&c->g->n, 0, 8, c->stream));
    CK(cudaMemsetAsync(&c->g->bad_input, 0, 4, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return set_err(c, ABS_ERR_INVALID_ARGUMENT, (bad & 1u) ? "diameter must be > 0" : "uid >= uid_count");
  }
  c->n = n;
  return ABS_OK;
}

static int upload_common(abs_gpu_ctx* c, unsigned long long n, unsigned long long uid_count,
                         cudaMemcpyKind kind, const uint64_t* uid, const double* x, const double* y,
                         const double* z, const double* d, const uint8_t* mask, const double* volume,
                         const uint8_t* flags, const uint32_t* partners) {
  int ib = 0;
  int rc = upload_enqueue(c, n, uid_count, kind, uid, x, y, z, d, mask, volume, flags, partners, &ib);
  if (rc) return rc;
  return upload_finish(c, n, ib);
}

int abs_gpu_upload(abs_gpu_ctx* c, uint64_t n, const uint64_t* uid, const double* x, const double* y,
                   const double* z, const double* d, const uint8_t* mask, const double* volume,
                   const uint8_t* flags, const uint32_t* partners, uint64_t uid_count) {
  return upload_common(c, n, uid_count, cudaMemcpyHostToDevice, uid, x, y, z, d, mask, volume, flags, partners);
}

int abs_gpu_upload_device(abs_gpu_ctx* c, uint64_t n, const uint64_t* uid, const double* x, const double* y,
                          const double* z, const double* d, const uint8_t* mask, uint64_t uid_count) {
  return upload_common(c, n, uid_count, cudaMemcpyDeviceToDevice, uid, x, y, z, d, mask, nullptr, nullptr,
                       nullptr);
}

static void free_sort_scratch(abs_gpu_ctx* c) {
  for (int b = 0; b < 2; ++b) {
    cudaFree(c->sort_k[b]);
    cudaFree(c->sort_i[b]);
    c->sort_k[b] = nullptr;
    c->sort_i[b] = nullptr;
  }
  cudaFree(c->sort_hist); cudaFree(c->sort_tiles); cudaFree(c->sort_hlen);
  c->sort_hist = nullptr;
  c->sort_tiles = nullptr;
  c->sort_hlen = nullptr;
  c->sort_cap = 0;
}

// sort_and_balance (sort_balance.cpp:22-148) on the device, stream-ordered and
// without host synchronisation: grid of the current state (no re-binning),
// Morton-code keys in descending index order, 8 8-bit LSD pass slots of which
// the device runs sort_passes, gather into the other state buffer. Callable
// inside the iteration loop (sorting_frequency, simulation.cpp:246-247).
static int launch_sort(abs_gpu_ctx* c, unsigned long long iteration, bool exact_order) {
  if (c) c->list_valid = false;  // storage order changes (neighbour lists index it)
  {
    const int rc = ensure_sort_scratch(c);
    if (rc) return rc;
  }
  const Pd* pos = cur_pos(c);
  sync_check(c, "k_set_u64");
  if (c->grid_valid) {  // the sort leaves no valid cell table behind
    k_zero_u32<<<grid_blocks(c, c->bins_cap), kThreads, 0, c->stream>>>(c->start, &c->g->nbins, 1, &c->g->err, c->bins_cap + 1);
    sync_check(c, "k_zero_u32");
    ++c->launches;
    c->grid_valid = false;
  }
  k_reduce<<<agent_blocks(c, 4), kThreads, 0, c->stream>>>(pos, c->g);
  sync_check(c, "k_reduce");
  k_finalize<<<1, 32, 0, c->stream>>>(c->g, FinArgs{c->cfg.fixed_box_length, 0, 1, 1, row_block_shift(), ~0ull,
                                                     ~0ull, ~0ull, 0, iteration});
                                                 sync_check(c, "k_finalize");
  // Path choice: the counting sort needs the Morton code space of this grid
  // to fit the cell table. The host guesses from the last grid it read (dims
  // change slowly) and launches only that path; the device checks the guess
  // (k_sort_mode) and a wrong counting guess rolls the iteration back to be
  // re-run with the exact path (kErrSortRetry). Without a guess both paths
  // are launched and the device picks.
  int mode_arg = exact_order ? 0 : 1;
  bool launch_counting = !exact_order, launch_radix = true;
  if (!exact_order && c->sort_guess_dims[0]) {
    unsigned int maxdim = std::max(c->sort_guess_dims[0], std::max(c->sort_guess_dims[1], c->sort_guess_dims[2]));
    unsigned int axis_bits = 0;
    while ((1u << axis_bits) < maxdim) ++axis_bits;
    const unsigned int code_bits = (c->sort_guess_dims[2] == 1 ? 2u : 3u) * (axis_bits + 1);  // one bit of slack
    static const bool force_counting = env_flag("ABSIM_SORT_GUESS_COUNTING", false);  // test hook: always guess counting
    const bool guess = (force_counting || (code_bits < 40 && (1ull << code_bits) <= c->bins_cap)) &&
                       iteration != c->sort_radix_iteration;
    mode_arg = guess ? 2 : 0;
    launch_counting = guess;
    launch_radix = !guess;
  }
  k_sort_mode<<<1, 1, 0, c->stream>>>(c->g, c->bins_cap, mode_arg, iteration);
  sync_check(c, "k_sort_mode");
  c->launches += 1;
  const int nxt = c->cur ^ 1;
  if (launch_counting) {  // Morton key + atomic slot, scan, scatter
    k_mkey<<<agent_blocks(c), kThreads, 0, c->stream>>>(pos, c->g, c->start, c->key, c->rank);
    sync_check(c, "k_mkey");
    launch_scan_cells(c, &c->g->sort_len, c->bins_cap, &c->g->err);
    k_scatter<false><<<agent_blocks(c), kThreads, 0, c->stream>>>(pos, c->S[c->cur], c->S[nxt], c->pf, c->start,
                                                                 c->key, c->rank, c->g, c->cap,
                                                                 c->cfg.model == ABS_MODEL_PROLIFERATION,
                                                                 c->cfg.record_forces, 0, 1, uses_ext(c->cfg));
                                                             sync_check(c, "k_scatter");
    k_zero_u32<<<grid_blocks(c, c->bins_cap), kThreads, 0, c->stream>>>(c->start, &c->g->sort_len, 1, &c->g->err, c->bins_cap + 1);
    sync_check(c, "k_zero_u32");
    c->launches += 3;
  }
  if (!launch_radix) {
    c->cur = nxt;
    c->pos_in_new = false;
    return ABS_OK;
  }
  // exact path (device-selected otherwise): radix passes + gather
  const unsigned int blocks = static_cast<unsigned int>((c->cap + kSortChunk - 1) / kSortChunk);
  unsigned long long* k1 = c->sort_k[0];
  unsigned long long* k2 = c->sort_k[1];
  unsigned int* i1 = c->sort_i[0];
  unsigned int* i2 = c->sort_i[1];
  k_sort_keys<<<agent_blocks(c), kThreads, 0, c->stream>>>(pos, c->g, k1, i1, c->S[c->cur].skey,
                                                                 exact_order ? 1 : 0);
  sync_check(c, "k_sort_keys");
  c->launches += 3;
  for (int shift = 0; shift < 64; shift += 8) {
    k_radix_hist<<<blocks, kThreads, 0, c->stream>>>(k1, i1, c->g, shift, c->sort_hist, kSortChunk);
    sync_check(c, "k_radix_hist");
    launch_scan<unsigned int>(c, c->sort_hist, c->sort_hlen, 256ull * blocks, c->sort_tiles, nullptr);
    // one warp per chunk (stable by construction): 32-thread blocks keep the
    // SM full of independent chunk walkers
    k_radix_scatter<<<blocks, 32, 0, c->stream>>>(k1, i1, k2, i2, c->g, shift, c->sort_hist, kSortChunk);
    sync_check(c, "k_radix_scatter");
    c->launches += 2;
    std::swap(k1, k2);
    std::swap(i1, i2);
  }
  k_gather<<<agent_blocks(c), kThreads, 0, c->stream>>>(pos, c->S[c->cur], c->S[nxt], i1, c->g, c->cap,
                                                              c->cfg.model == ABS_MODEL_PROLIFERATION,
                                                              c->cfg.record_forces, 0, uses_ext(c->cfg));
                                                          sync_check(c, "k_gather");
  ++c->launches;
  c->cur = nxt;
  c->pos_in_new = false;
  return ABS_OK;
}

constexpr double kCrowdedAgentsPerBox = 6.0;  // c1 2.9, c3 ~1, c4 ~10 (sub-binned anyway), c2 late ~14

// Graph replay of iterations: ABSIM_GRAPHS=0 disables; never while the
// per-launch timing events are on.
bool use_graphs(const abs_gpu_ctx* c) {
  static const bool on = env_flag("ABSIM_GRAPHS", true);
  return on && !c->graphs_off && !c->timing && !kd_env(c);  // the kd build sizes its launches on the host
}

int abs_gpu_simulate(abs_gpu_ctx* c, uint64_t iterations) {
  if (!c) return ABS_ERR_INVALID_ARGUMENT;
  cudaSetDevice(c->device);
  const bool deferred = c->defer_commit && adds_agents(c->cfg);
  if (deferred && c->pending_commit)
    return set_err(c, ABS_ERR_STATE, "abs_gpu_commit is pending for the previous iteration");
  if (deferred && iterations > 1)
    return set_err(c, ABS_ERR_INVALID_ARGUMENT, "deferred commit runs one iteration per call");
  // Launch in chunks; a chunk whose finalize asked for more bins/capacity is
  // rolled back to the failed iteration (no kernel touched state after it).
  unsigned long long done = 0;
  // (the kd-tree build reads the agent count on the host: one iteration per chunk)
  const unsigned long long chunk = kd_env(c) ? 1 : 32;
  sync_check(c, "simulate entry");
  // neighbour lists: storage for this population, allocated
  // outside any graph capture
  if (list_mode_ok(c) && iterations >= 2) {
    if (ensure_lists(c, c->nl_kmax ? c->nl_kmax : kListKmaxInit) != ABS_OK) {
      cudaGetLastError();
      c->list_off = true;  // no room for the lists: re-bin + walk every iteration
    }
    sync_check(c, "ensure_lists");
  }
  while (done < iterations) {
    // while the list policy is re-binning (a relaxing system's rate decays), re-read the
    // displacement rate every 4 iterations
    // (and while the rate is still unknown, a build + one list step to learn it:
    // a whole chunk scheduled as list steps would be rolled back at the first
    // failed coverage check)
    const bool lists_on = list_mode_ok(c) && c->nl;
    const bool rebinning = lists_on && c->pred_rate > 0.0 && c->cfg.neighbor_list <= 0 &&
                           list_skin(c) < 2.0 * list_min_steps() * c->pred_rate;
    const unsigned long long todo = std::min<unsigned long long>(
        lists_on && c->pred_rate <= 0.0 ? 2 : (rebinning ? 4 : (lists_on && !c->list_valid ? 8 : chunk)),
        iterations - done);
    struct Snap { int cur; bool pos_in_new; bool grid_valid; bool list_valid; };
    std::vector<Snap> snaps;
    snaps.reserve(todo);
    std::vector<int> kinds;
    kinds.reserve(todo);
    for (unsigned long long t = 0; t < todo; ++t) {
      snaps.push_back({c->cur, c->pos_in_new, c->grid_valid, c->list_valid});
      const unsigned long long it = c->iteration + t;
      const bool sorts =
          c->cfg.sorting_frequency > 0 && it % static_cast<unsigned long long>(c->cfg.sorting_frequency) == 0;
      // iteration kind: 0 re-bin + cell-table walk, 1 list step, 2 list
      // rebuild (a build pays off only if at least one more iteration of
      // this call can use the lists; a sort re-orders storage)
      const unsigned long long remaining = iterations - done - t;
      // The host predicts the device's coverage check from the last observed
      // displacement rate and schedules the rebuild itself, so a rejected list
      // step (rolled back with the rest of its chunk) stays the exception.
      // A build pays off only if the lists then serve several steps: at the
      // current rate a fresh list lasts skin / (2 rate) steps; below
      // list_min_steps() the iteration re-bins and walks (tracking the rate).
      int kind = 0;
      if (list_mode_ok(c) && c->nl) {
        const double skin = list_skin(c);
        const bool usable = c->list_valid && !sorts;
        // life of a list built now: until the displacement check fails or the next Morton sort
        // (builds at iterations 8 or 9 of a 10-iteration sort period do not pay: walk instead)
        double life = c->pred_rate > 0.0 ? skin / (2.0 * c->pred_rate) : 1e18;
        if (c->cfg.sorting_frequency > 0) {
          const unsigned long long sf = static_cast<unsigned long long>(c->cfg.sorting_frequency);
          life = std::min(life, static_cast<double>(sf - it % sf));
        }
        const bool pays = c->cfg.neighbor_list > 0 || c->pred_rate <= 0.0 || life >= list_min_steps();
        if (usable && (2.0 * c->pred_acc <= skin || remaining < 2)) {
          kind = 1;
          c->pred_acc += c->pred_rate;
        } else if (remaining >= 2 && pays) {
          kind = 2;
          c->pred_acc = c->pred_rate;
        } else {
          kind = 3;
          c->list_valid = false;
        }
      }
      kinds.push_back(kind);
      auto enqueue = [&]() -> int {
        phase_mark(c);  // iteration start
        if (sorts) {
          const int rc = launch_sort(c, it, keys_exact(c->cfg));
          if (rc) return rc;
        }
        phase_mark(c);  // after sort
        launch_iteration(c, it, kind);
        return ABS_OK;
      };
      // One CUDA graph per iteration (cached executable, parameters updated in
      // place): the launch-bound small configs lose the inter-kernel gaps.
      // Any capture problem (e.g. a first-use allocation) falls back to
      // direct launches for this iteration.
      if (use_graphs(c)) {
        const Snap sn = snaps.back();
        const unsigned long long launches0 = c->launches;
        const unsigned int epoch0 = c->scan_epoch;
        bool ok = cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeRelaxed) == cudaSuccess;
        int rc = ok ? enqueue() : ABS_OK;
        cudaGraph_t graph = nullptr;
        if (ok) ok = cudaStreamEndCapture(c->stream, &graph) == cudaSuccess && graph && rc == ABS_OK;
        if (ok) {
          const int slot = (sorts ? 1 : 0) + 2 * kind;
          if (c->gexec[slot]) {
            cudaGraphExecUpdateResultInfo info;
            if (cudaGraphExecUpdate(c->gexec[slot], graph, &info) != cudaSuccess) {
              cudaGetLastError();
              cudaGraphExecDestroy(c->gexec[slot]);
              c->gexec[slot] = nullptr;
            }
          }
          if (!c->gexec[slot] && cudaGraphInstantiate(&c->gexec[slot], graph, 0) != cudaSuccess) {
            c->gexec[slot] = nullptr;
            ok = false;
          }
          if (ok) ok = cudaGraphLaunch(c->gexec[slot], c->stream) == cudaSuccess;
        }
        if (graph) cudaGraphDestroy(graph);
        if (ok) continue;
        cudaGetLastError();  // clear the capture error; replay this iteration directly
        c->cur = sn.cur;
        c->pos_in_new = sn.pos_in_new;
        c->grid_valid = sn.grid_valid;
        c->list_valid = sn.list_valid;
        c->launches = launches0;
        c->scan_epoch = epoch0;
        if (++c->graph_failures >= 4) c->graphs_off = true;
        if (rc) return rc;
      }
      const int rc = enqueue();
      if (rc) return rc;
    }
    cudaError_t le = cudaGetLastError();
    if (le != cudaSuccess) return set_err(c, ABS_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(le));
    if (c->kd_failed) {
      c->kd_failed = false;
      cudaStreamSynchronize(c->stream);
      return set_err(c, ABS_ERR_CAPACITY, "kd-tree environment: the tree build failed (device memory)");
    }
    DevGrid h{};
    int rc = read_grid(c, &h);
    if (rc) return rc;
    static const bool trace = env_flag("ABSIM_LIST_TRACE", false);
    if (trace) {  // debugging: the chunk's iteration kinds and the device's coverage numbers
      float rate = 0.0f;
      std::memcpy(&rate, &h.step_disp, sizeof rate);
      std::fprintf(stderr, "absim: it %llu kinds", c->iteration);
      for (int k : kinds) std::fprintf(stderr, " %d", k);
      std::fprintf(stderr, " | err %d failed_it %llu rate %.4f acc %.4f pred_rate %.4f pred_acc %.4f need %u\n", h.err,
                   h.failed_iteration, rate, h.list_acc, c->pred_rate, c->pred_acc, h.list_need);
    }
    {  // the prediction restarts from the device's own numbers
      float rate = 0.0f;
      std::memcpy(&rate, &h.step_disp, sizeof rate);
      const double margin = h.margin + 1e-12;
      c->pred_acc = h.list_acc + static_cast<double>(rate) + margin;
      if (rate > 0.0f) c->pred_rate = static_cast<double>(rate) + margin;
    }
    auto count_kinds = [&](unsigned long long upto) {
      for (unsigned long long q = 0; q < upto && q < kinds.size(); ++q) {
        c->list_builds += kinds[q] == 2;
        c->list_steps += kinds[q] == 1 || kinds[q] == 2;
      }
    };
    if (h.err == kErrNone) {
      count_kinds(todo);
      if (h.list_incomplete && c->list_valid) {  // the last build overflowed: grow, rebuild next
        c->list_valid = false;
        const unsigned int need = h.list_need;
        if (need > kListKmaxMax || ensure_lists(c, std::min(kListKmaxMax, need + need / 4 + 8)) != ABS_OK) {
          cudaGetLastError();
          c->list_off = true;
        }
      }
      if (h.n) std::memcpy(c->sort_guess_dims, h.dims, sizeof c->sort_guess_dims);
      // Auto sub-bins (bins_yz): a crowded grid (config 2 once its cells have
      // grown: ~14 agents per box, 106 evaluations per agent) needs the row
      // culling of sub-bins even when diameters are uniform; from the next
      // chunk on (c2 after 150 iterations: 2.2e8 -> 2.8e8 agent-it/s).
      if (h.n && c->auto_bins == 1u && c->cfg.model != ABS_MODEL_SIR && !brute_env(c)) {
        const double boxes = static_cast<double>(h.dims[0]) * h.dims[1] * h.dims[2];
        if (static_cast<double>(h.n) > kCrowdedAgentsPerBox * boxes) c->auto_bins = 2u;
      }
      c->iteration += todo;
      done += todo;
      if (deferred && todo) c->pending_commit = true;
      continue;
    }
    const unsigned long long fi = h.failed_iteration;
    const unsigned long long off = fi - c->iteration;
    if (fi < c->iteration || off >= todo) return set_err(c, ABS_ERR_STATE, "bad failed iteration");
    c->cur = snaps[off].cur;
    c->pos_in_new = snaps[off].pos_in_new;
    c->grid_valid = false;  // finalize may have left a partially filled count table
    c->list_valid = snaps[off].list_valid;
    count_kinds(off);
    c->iteration = fi;
    done += off;
    if (h.err == kErrBinsRetry) {
      CK(cudaMemsetAsync(c->start, 0, (c->bins_cap + 1) * 4, c->stream));
      rc = ensure_bins(c, h.needed_bins);
      if (rc) return rc;
      CK(cudaMemsetAsync(c->start, 0, (c->bins_cap + 1) * 4, c->stream));
      rc = clear_dev_err(c);
      if (rc) return rc;
    } else if (h.err == kErrSortRetry) {  // re-run that iteration's sort on the exact path
      c->sort_radix_iteration = fi;
      if (env_flag("ABSIM_SORT_GUESS_COUNTING", false)) std::fprintf(stderr, "absim: sort retry at iteration %llu\n", fi);
      CK(cudaMemsetAsync(c->start, 0, (c->bins_cap + 1) * 4, c->stream));
      rc = clear_dev_err(c);
      if (rc) return rc;
    } else if (h.err == kErrListRebuild) {  // the lists no longer cover r: rebuild at this iteration
      c->list_valid = false;
      const unsigned int need = h.list_need;
      if (h.list_incomplete) {  // the last build overflowed: grow the lists first
        if (need > kListKmaxMax || ensure_lists(c, std::min(kListKmaxMax, need + need / 4 + 8)) != ABS_OK) {
          cudaGetLastError();
          c->list_off = true;
        }
      }
      rc = clear_dev_err(c);
      if (rc) return rc;
    } else if (h.err == kErrCapRetry) {
      CK(cudaMemsetAsync(c->start, 0, (c->bins_cap + 1) * 4, c->stream));
      if (2 * h.n > c->cap) rc = ensure_capacity(c, 2 * c->cap, h.n);
      if (rc) return rc;
      rc = ensure_uid_space(c, std::max<unsigned long long>(2 * (h.uid_count + h.n), h.uid_count + c->cap) + 1024);
      if (rc) return rc;
      rc = clear_dev_err(c);
      if (rc) return rc;
    } else {
      rc = map_dev_err(c, h);
      clear_dev_err(c);
      CK(cudaMemsetAsync(c->start, 0, (c->bins_cap + 1) * 4, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      return rc;
    }
  }
  return ABS_OK;
}

int abs_gpu_set_agent_ext(abs_gpu_ctx* c, const uint32_t* tags, const uint64_t* rng_counters) {
  if (!c) return ABS_ERR_INVALID_ARGUMENT;
  cudaSetDevice(c->device);
  DevGrid h{};
  int rc = read_grid(c, &h);
  if (rc) return rc;
  Soa& S = c->S[c->cur];
  if (h.n && tags) CK(cudaMemcpyAsync(S.tag, tags, h.n * 4, cudaMemcpyHostToDevice, c->stream));
  if (h.n && rng_counters) CK(cudaMemcpyAsync(S.rngc, rng_counters, h.n * 8, cudaMemcpyHostToDevice, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return ABS_OK;
}

int abs_gpu_download_ext(abs_gpu_ctx* c, uint32_t* tags, uint64_t* rng_counters) {
  if (!c) return ABS_ERR_INVALID_ARGUMENT;
  cudaSetDevice(c->device);
  DevGrid h{};
  int rc = read_grid(c, &h);
  if (rc) return rc;
  Soa& S = c->S[c->cur];
  if (h.n && tags) CK(cudaMemcpyAsync(tags, S.tag, h.n * 4, cudaMemcpyDeviceToHost, c->stream));
  if (h.n && rng_counters) CK(cudaMemcpyAsync(rng_counters, S.rngc, h.n * 8, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return ABS_OK;
}

int abs_gpu_set_defer_commit(abs_gpu_ctx* c, int defer) {
  if (!c) return ABS_ERR_INVALID_ARGUMENT;
  if (c->pending_commit) return set_err(c, ABS_ERR_STATE, "abs_gpu_commit is pending");
  if (defer && adds_agents(c->cfg) && c->cfg.detect_static_agents)
    return set_err(c, ABS_ERR_INVALID_ARGUMENT,
                   "static detection with multi-domain additions is not supported (new-neighbour marks stay local)");
  cudaSetDevice(c->device);
  c->defer_commit = defer != 0;
  return ensure_uid_space(c, c->uid_cap);
}

int abs_gpu_division_marks(abs_gpu_ctx* c, uint32_t* out, uint64_t cap, uint64_t* len) {
  if (!c || !len) return ABS_ERR_INVALID_ARGUMENT;
  cudaSetDevice(c->device);
  DevGrid h{};
  int rc = read_grid(c, &h);
  if (rc) return rc;
  *len = h.uid_count;
  if (!c->pending_commit) return set_err(c, ABS_ERR_STATE, "no deferred iteration to commit");
  if (!out || cap < h.uid_count) return set_err(c, ABS_ERR_CAPACITY, "division mark buffer too small");
  if (h.uid_count) CK(cudaMemcpyAsync(out, c->div_mark, h.uid_count * 4, cudaMemcpyDeviceToDevice, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return ABS_OK;
}

int abs_gpu_commit(abs_gpu_ctx* c, const uint32_t* global_marks, uint64_t len) {
  if (!c) return ABS_ERR_INVALID_ARGUMENT;
  if (!c->pending_commit) return ABS_OK;
  cudaSetDevice(c->device);
  DevGrid h{};
  int rc = read_grid(c, &h);
  if (rc) return rc;
  if (global_marks) {
    if (len != h.uid_count) return set_err(c, ABS_ERR_INVALID_ARGUMENT, "division marks length != uid_count");
    if (len) CK(cudaMemcpyAsync(c->div_mark_g, global_marks, len * 4, cudaMemcpyDeviceToDevice, c->stream));
  } else if (h.uid_count) {  // single domain: this rank's marks are everyone's
    CK(cudaMemcpyAsync(c->div_mark_g, c->div_mark, h.uid_count * 4, cudaMemcpyDeviceToDevice, c->stream));
  }
  launch_commit(c);
  c->pending_commit = false;
  CK(cudaGetLastError());
  rc = read_grid(c, &h);
  if (rc) return rc;
  if (h.err) {
    rc = map_dev_err(c, h);
    clear_dev_err(c);
    return rc;
  }
  return ABS_OK;
}

int abs_gpu_set_grid_override(abs_gpu_ctx* c, const double* grid, const uint32_t* dims) {
  if (!c) return ABS_ERR_INVALID_ARGUMENT;
  struct { int on; int pad; double g[5]; unsigned int d[3]; } ov{};
  ov.on = grid != nullptr;
  if (grid) {
    if (!dims) return set_err(c, ABS_ERR_INVALID_ARGUMENT, "grid override needs dims");
    for (int k = 0; k < 5; ++k) ov.g[k] = grid[k];
    for (int k = 0; k < 3; ++k) ov.d[k] = dims[k];
    if (!(grid[3] > 0.0) || !dims[0] || !dims[1] || !dims[2])
      return set_err(c, ABS_ERR_INVALID_ARGUMENT, "bad grid override");
  }
  c->ov_on = ov.on != 0;
  CK(cudaMemcpyAsync(&c->g->ov_on, &ov.on, sizeof(int), cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(c->g->ov_grid, ov.g, sizeof ov.g, cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(c->g->ov_dims, ov.d, sizeof ov.d, cudaMemcpyHostToDevice, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return ABS_OK;
}

int abs_gpu_local_bounds(abs_gpu_ctx* c, double* out7) {
  if (!c || !out7) return ABS_ERR_INVALID_ARGUMENT;
  cudaSetDevice(c->device);
  k_reduce<<<agent_blocks(c, 4), kThreads, 0, c->stream>>>(cur_pos(c), c->g);
  ++c->launches;
  DevGrid h{};
  int rc = read_grid(c, &h);
  if (rc) return rc;
  for (int k = 0; k < 7; ++k) {
    const unsigned long long o = h.red[k];
    const unsigned long long b = (o >> 63) ? (o & 0x7fffffffffffffffull) : ~o;
    std::memcpy(&out7[k], &b, 8);
  }
  k_reset_reduction<<<1, 1, 0, c->stream>>>(c->g);  // a kernel: no pageable copy
  ++c->launches;
  if (h.nonfinite) return set_err(c, ABS_ERR_NONFINITE, "agent positions are not finite");
  return ABS_OK;
}

// Keep only agents with keep[i] (already filled for the current population).
static int compact_population(abs_gpu_ctx* c, unsigned long long n) {
  if (c) c->list_valid = false;  // storage order changes (neighbour lists index it)
  unsigned int* keep = c->rank;  // scratch: rank[] is rewritten by the next k_key
  unsigned int* idx = c->key;
  CK(cudaMemcpyAsync(idx, keep, n * 4, cudaMemcpyDeviceToDevice, c->stream));
  if (!c->xcounts) {
    CK(dalloc(&c->xcounts, 2));
    CK(cudaHostAlloc(reinterpret_cast<void**>(&c->hxcounts), 16, cudaHostAllocDefault));
  }
  unsigned long long* len = c->xcounts + 1;  // persistent scratch (no allocation per call)
  k_set_u64<<<1, 1, 0, c->stream>>>(len, n);
  // ctiles holds cap / kScanTile + 2 u32 tile sums: room for any n <= cap
  launch_scan<unsigned int>(c, idx, len, n, c->ctiles, nullptr);  // idx[n] = survivors
  CK(cudaMemcpyAsync(c->hxcounts, idx + n, 4, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  const unsigned long long nn = *reinterpret_cast<const unsigned int*>(c->hxcounts);
  if (nn < n) {
    if (c->holes_cap < c->cap) {
      cudaFree(c->holes);
      c->holes = nullptr;
      c->holes_cap = 0;
      CK(dalloc(&c->holes, c->cap));
      c->holes_cap = c->cap;
    }
    k_hole_list<<<grid_blocks(c, nn), kThreads, 0, c->stream>>>(keep, idx, nn, c->holes);
    k_swap_move<<<grid_blocks(c, n - nn), kThreads, 0, c->stream>>>(cur_pos(c), c->S[c->cur], keep,
                                                                     idx, c->holes, nn, n, c->cap);
    c->launches += 2;
  }
  k_set_u64<<<1, 1, 0, c->stream>>>(&c->g->n, nn);
  if (c->grid_valid) dzero(c, c->start, (c->bins_cap + 1) * 4);
  CK(cudaStreamSynchronize(c->stream));
  c->grid_valid = false;
  c->n = nn;
  return ABS_OK;
}

int abs_gpu_export_layers(abs_gpu_ctx* c, const double* grid, const uint32_t* dims, int64_t lo, int64_t hi, int mode,
                          void* out_lo, void* out_hi, uint64_t cap, uint64_t* n_lo, uint64_t* n_hi) {
  if (!c || !grid || !dims || mode < 0 || mode > 3) return ABS_ERR_INVALID_ARGUMENT;
  const int halo = mode & 1, periodic = (mode >> 1) & 1;
  cudaSetDevice(c->device);
  DevGrid h{};
  int rc = read_grid(c, &h);
  if (rc) return rc;
  const unsigned long long n = h.n;
  if (!c->xcounts) {  // persistent: no allocation (and its device sync) per exchange
    CK(dalloc(&c->xcounts, 2));
    CK(cudaHostAlloc(reinterpret_cast<void**>(&c->hxcounts), 16, cudaHostAllocDefault));
  }
  unsigned long long* counts = c->xcounts;
  k_zero_bytes<<<1, 32, 0, c->stream>>>(reinterpret_cast<unsigned char*>(counts), 16);
  if (n) {
    k_export<<<grid_blocks(c, n), kThreads, 0, c->stream>>>(
        cur_pos(c), c->S[c->cur], c->cap, n, grid[2], grid[3], dims[2], lo, hi, halo, periodic,
        static_cast<Rec*>(out_lo), static_cast<Rec*>(out_hi), cap, counts, halo == 0 ? c->rank : nullptr);
    ++c->launches;
  }
  CK(cudaMemcpyAsync(c->hxcounts, counts, 16, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  const unsigned long long hc[2] = {c->hxcounts[0], c->hxcounts[1]};
  if (n_lo) *n_lo = hc[0];
  if (n_hi) *n_hi = hc[1];
  if (hc[0] > cap || hc[1] > cap) return set_err(c, ABS_ERR_CAPACITY, "export buffer too small");
  if (halo == 0 && (hc[0] || hc[1])) return compact_population(c, n);
  return ABS_OK;
}

int abs_gpu_import(abs_gpu_ctx* c, const void* records, uint64_t count, int as_ghost) {
  if (c) c->list_valid = false;  // storage order changes (neighbour lists index it)
  if (!c || (count && !records)) return ABS_ERR_INVALID_ARGUMENT;
  if (!count) return ABS_OK;
  cudaSetDevice(c->device);
  DevGrid h{};
  int rc = read_grid(c, &h);
  if (rc) return rc;
  const unsigned long long n = h.n;
  rc = ensure_capacity(c, std::max<unsigned long long>(c->cap, 2 * (n + count) + 1024), n);
  if (rc) return rc;
  k_import<<<grid_blocks(c, count), kThreads, 0, c->stream>>>(static_cast<const Rec*>(records), count, n, cur_pos(c),
                                                              c->S[c->cur], c->cap, as_ghost);
  ++c->launches;
  const unsigned long long nn = n + count;
  CK(cudaMemcpyAsync(&c->g->n, &nn, 8, cudaMemcpyHostToDevice, c->stream));
  if (c->grid_valid) CK(cudaMemsetAsync(c->start, 0, (c->bins_cap + 1) * 4, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  c->grid_valid = false;
  c->n = nn;
  if (as_ghost) c->ghosts += count;
  return ABS_OK;
}

int abs_gpu_drop_ghosts(abs_gpu_ctx* c) {
  if (!c) return ABS_ERR_INVALID_ARGUMENT;
  if (!c->ghosts) return ABS_OK;  // nothing imported as ghost since the last drop
  cudaSetDevice(c->device);
  DevGrid h{};
  int rc = read_grid(c, &h);
  if (rc) return rc;
  if (!h.n) return ABS_OK;
  k_keep_ghostless<<<grid_blocks(c, h.n), kThreads, 0, c->stream>>>(c->S[c->cur], h.n, c->rank);
  ++c->launches;
  rc = compact_population(c, h.n);
  if (rc == ABS_OK) c->ghosts = 0;
  return rc;
}

int abs_gpu_sir_counts(abs_gpu_ctx* c, uint64_t* out3) {
  if (!c || !out3) return ABS_ERR_INVALID_ARGUMENT;
  DevGrid h{};
  int rc = read_grid(c, &h);
  if (rc) return rc;
  for (int q = 0; q < 3; ++q) out3[q] = h.sir[q];
  return ABS_OK;
}

int abs_gpu_sir_state(abs_gpu_ctx* c, uint8_t* state, uint32_t* t_infected) {
  if (!c) return ABS_ERR_INVALID_ARGUMENT;
  DevGrid h{};
  int rc = read_grid(c, &h);
  if (rc) return rc;
  Soa& S = c->S[c->cur];
  if (state) CK(cudaMemcpy(state, S.beh, h.n, cudaMemcpyDeviceToHost));
  if (t_infected) CK(cudaMemcpy(t_infected, S.partners, h.n * 4, cudaMemcpyDeviceToHost));
  return ABS_OK;
}

int abs_gpu_set_iteration(abs_gpu_ctx* c, uint64_t iteration) {
  if (!c) return ABS_ERR_INVALID_ARGUMENT;
  c->iteration = iteration;
  return ABS_OK;
}

int abs_gpu_synchronize(abs_gpu_ctx* c) {
  CK(cudaStreamSynchronize(c->stream));
  return ABS_OK;
}

int abs_gpu_stats(abs_gpu_ctx* c, abs_step_stats* out) {
  if (!c || !out) return ABS_ERR_INVALID_ARGUMENT;
  DevGrid h{};
  int rc = read_grid(c, &h);
  if (rc) return rc;
  out->agents = h.n;
  out->uid_count = h.uid_count;
  out->iterations = c->iteration;
  out->force_evaluations = h.evals;
  out->force_skips = h.skips;
  out->agents_added = h.added;
  out->agents_removed = h.removed;
  out->kernel_launches = c->launches;
  out->agent_iterations = h.agent_its;
  return ABS_OK;
}

int abs_gpu_download(abs_gpu_ctx* c, uint64_t* n_out, uint64_t* uid, double* x, double* y, double* z, double* d,
                     double* fx, double* fy, double* fz, uint32_t* partners, uint8_t* flags, double* volume) {
  if (!c) return ABS_ERR_INVALID_ARGUMENT;
  DevGrid h{};
  int rc = read_grid(c, &h);
  if (rc) return rc;
  const unsigned long long n = h.n;
  if (n_out) *n_out = n;
  Soa& S = c->S[c->cur];
  // Components are split on the device into the staging area and copied
  // straight into the caller's arrays (page-locked arrays: plain DMA).
  if (n && (x || y || z || d)) {
    double* st = reinterpret_cast<double*>(c->st_pd);
    k_split_pd<<<grid_blocks(c, n), kThreads, 0, c->stream>>>(cur_pos(c), c->g, st, n);
    ++c->launches;
    double* dst[4] = {x, y, z, d};
    for (int q = 0; q < 4; ++q)
      if (dst[q]) CK(cudaMemcpyAsync(dst[q], st + q * n, n * 8, cudaMemcpyDeviceToHost, c->stream));
  }
  if (n && uid) CK(cudaMemcpyAsync(uid, S.uid, n * 8, cudaMemcpyDeviceToHost, c->stream));
  double* fdst[3] = {fx, fy, fz};
  for (int q = 0; q < 3; ++q) {
    if (!n || !fdst[q]) continue;
    if (c->cfg.record_forces) CK(cudaMemcpyAsync(fdst[q], S.force + q * c->cap, n * 8, cudaMemcpyDeviceToHost, c->stream));
    else std::fill(fdst[q], fdst[q] + n, 0.0);  // last_force is not kept (record_forces == 0)
  }
  if (n && partners) CK(cudaMemcpyAsync(partners, S.partners, n * 4, cudaMemcpyDeviceToHost, c->stream));
  if (n && flags) {
    unsigned char* fb = reinterpret_cast<unsigned char*>(c->key);
    k_mask_flags<<<grid_blocks(c, n), kThreads, 0, c->stream>>>(S.flags, fb, c->g);
    ++c->launches;
    CK(cudaMemcpyAsync(flags, fb, n, cudaMemcpyDeviceToHost, c->stream));
  }
  if (n && volume) {
    if (c->cfg.model == ABS_MODEL_PROLIFERATION)
      CK(cudaMemcpyAsync(volume, S.vol, n * 8, cudaMemcpyDeviceToHost, c->stream));
    else
      std::fill(volume, volume + n, 0.0);
  }
  CK(cudaStreamSynchronize(c->stream));
  return ABS_OK;
}

// Host-boundary pipeline. Per frame: H2D of the frame's x|y|z|d into device
// staging slot f%2 (stream h2d), ingest + `iterations` iterations (compute
// stream), positions split into output slot f%2 and D2H into the frame's
// host arrays (stream d2h). Events order the slots: the H2D of frame f+1 is
// issued before frame f computes, so it overlaps frame f's iterations, and
// the D2H of frame f overlaps frame f+1. Each frame is exactly
// abs_gpu_upload (uids 0..n-1) + abs_gpu_set_iteration + abs_gpu_simulate +
// abs_gpu_download (x, y, z).
static int run_frames_impl(abs_gpu_ctx* c, const abs_frame* frames, uint64_t count, uint64_t iterations,
                           uint64_t first_iteration);

int abs_gpu_run_frames(abs_gpu_ctx* c, const abs_frame* frames, uint64_t count, uint64_t iterations,
                       uint64_t first_iteration) {
  const int rc = run_frames_impl(c, frames, count, iterations, first_iteration);
  if (rc && c) {  // never return with copies into or out of caller memory still in flight
    if (c->h2d) cudaStreamSynchronize(c->h2d);
    if (c->d2h) cudaStreamSynchronize(c->d2h);
    if (c->stream) cudaStreamSynchronize(c->stream);
  }
  return rc;
}

static int run_frames_impl(abs_gpu_ctx* c, const abs_frame* frames, uint64_t count, uint64_t iterations,
                           uint64_t first_iteration) {
  if (!c) return ABS_ERR_INVALID_ARGUMENT;
  if (count && !frames) return set_err(c, ABS_ERR_INVALID_ARGUMENT, "null frames");
  if (c->defer_commit && adds_agents(c->cfg))
    return set_err(c, ABS_ERR_STATE, "frames need the commit inside the iteration (defer_commit is set)");
  if (c->cfg.model == ABS_MODEL_SIR) return set_err(c, ABS_ERR_INVALID_ARGUMENT, "frames carry no SIR state");
  unsigned long long mx = 0;
  for (uint64_t f = 0; f < count; ++f) {
    const abs_frame& F = frames[f];
    if (F.n && (!F.x || !F.y || !F.z || !F.d || !F.out_x || !F.out_y || !F.out_z))
      return set_err(c, ABS_ERR_INVALID_ARGUMENT, "null frame array");
    mx = std::max<unsigned long long>(mx, F.n);
  }
  if (!count) return ABS_OK;
  cudaSetDevice(c->device);
  if (!c->h2d) {
    CK(cudaStreamCreateWithFlags(&c->h2d, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&c->d2h, cudaStreamNonBlocking));
    for (int b = 0; b < 2; ++b)
      for (cudaEvent_t* e : {&c->in_ready[b], &c->in_free[b], &c->out_ready[b], &c->out_free[b]})
        CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  }
  if (mx > c->fcap) {
    for (int b = 0; b < 2; ++b) {
      cudaFree(c->fin[b]);
      c->fin[b] = nullptr;
    }
    c->fcap = 0;
    for (int b = 0; b < 2; ++b) CK(dalloc(&c->fin[b], 4 * mx));
    c->fcap = mx;
  }
  if (mx > c->fout_cap) {
    for (int b = 0; b < 2; ++b) {
      cudaFree(c->fout[b]);
      c->fout[b] = nullptr;
    }
    c->fout_cap = 0;
    for (int b = 0; b < 2; ++b) CK(dalloc(&c->fout[b], 4 * mx));
    c->fout_cap = mx;
  }
  // capacity for the largest frame up front (allocation synchronises)
  int rc = ensure_capacity(c, std::max<unsigned long long>(c->cap, 2 * mx + 1024), 0);
  if (rc) return rc;
  CK(cudaStreamSynchronize(c->stream));
  for (int b = 0; b < 2; ++b) {  // slots start free
    CK(cudaEventRecord(c->in_free[b], c->stream));
    CK(cudaEventRecord(c->out_free[b], c->d2h));
  }
  auto stage_in = [&](uint64_t f) -> int {
    const abs_frame& F = frames[f];
    const int b = static_cast<int>(f & 1);
    double* st = c->fin[b];
    CK(cudaStreamWaitEvent(c->h2d, c->in_free[b], 0));
    const double* src[4] = {F.x, F.y, F.z, F.d};
    for (int q = 0; q < 4; ++q)
      if (F.n) CK(cudaMemcpyAsync(st + q * F.n, src[q], F.n * 8, cudaMemcpyHostToDevice, c->h2d));
    CK(cudaEventRecord(c->in_ready[b], c->h2d));
    return ABS_OK;
  };
  rc = stage_in(0);
  if (rc) return rc;
  for (uint64_t f = 0; f < count; ++f) {
    const abs_frame& F = frames[f];
    const int b = static_cast<int>(f & 1);
    if (f + 1 < count) {
      rc = stage_in(f + 1);  // overlaps this frame's iterations
      if (rc) return rc;
    }
    CK(cudaStreamWaitEvent(c->stream, c->in_ready[b], 0));
    const double* st = c->fin[b];
    int ib = 0;
    rc = upload_enqueue(c, F.n, 0, cudaMemcpyDeviceToDevice, nullptr, st, st + F.n, st + 2 * F.n, st + 3 * F.n,
                        nullptr, nullptr, nullptr, nullptr, &ib);
    if (rc) return rc;
    CK(cudaEventRecord(c->in_free[b], c->stream));  // k_ingest has consumed the slot
    rc = upload_finish(c, F.n, ib);
    if (rc) return rc;
    c->iteration = first_iteration + f * iterations;
    rc = abs_gpu_simulate(c, iterations);
    if (rc) return rc;
    // positions -> output slot (after the slot's previous D2H), then D2H
    if (c->n > c->fout_cap) {  // a model added agents beyond the output staging: regrow it
      CK(cudaStreamSynchronize(c->d2h));
      c->fout_cap = 0;
      for (int q = 0; q < 2; ++q) {
        cudaFree(c->fout[q]);
        c->fout[q] = nullptr;
      }
      for (int q = 0; q < 2; ++q) CK(dalloc(&c->fout[q], 4 * c->n));
      c->fout_cap = c->n;
    }
    CK(cudaStreamWaitEvent(c->stream, c->out_free[b], 0));
    if (c->n) {
      k_split_xyz<<<grid_blocks(c, c->n), kThreads, 0, c->stream>>>(cur_pos(c), F.out_uid ? c->S[c->cur].uid : nullptr,
                                                                      c->g, c->fout[b], c->n);
      ++c->launches;
    }
    CK(cudaEventRecord(c->out_ready[b], c->stream));
    CK(cudaStreamWaitEvent(c->d2h, c->out_ready[b], 0));
    double* dst[3] = {F.out_x, F.out_y, F.out_z};
    const unsigned long long m = c->n;
    if (F.n_out) *F.n_out = m;
    if (m > F.out_cap) {
      cudaStreamSynchronize(c->d2h);
      cudaStreamSynchronize(c->h2d);
      return set_err(c, ABS_ERR_CAPACITY, "frame " + std::to_string(f) + ": " + std::to_string(m) +
                                              " agents exceed out_cap " + std::to_string(F.out_cap));
    }
    for (int q = 0; q < 3; ++q)
      if (m) CK(cudaMemcpyAsync(dst[q], c->fout[b] + q * m, m * 8, cudaMemcpyDeviceToHost, c->d2h));
    if (m && F.out_uid) CK(cudaMemcpyAsync(F.out_uid, c->fout[b] + 3 * m, m * 8, cudaMemcpyDeviceToHost, c->d2h));
    CK(cudaEventRecord(c->out_free[b], c->d2h));
  }
  CK(cudaStreamSynchronize(c->d2h));
  CK(cudaStreamSynchronize(c->h2d));
  return ABS_OK;
}

int abs_gpu_env_update(abs_gpu_ctx* c) {
  if (!c) return ABS_ERR_INVALID_ARGUMENT;
  cudaSetDevice(c->device);
  for (int attempt = 0; attempt < 4; ++attempt) {
    const int cur0 = c->cur;
    const bool pin0 = c->pos_in_new;
    launch_env_update(c, c->iteration, 0);
    if (c->kd_failed) {
      c->kd_failed = false;
      cudaStreamSynchronize(c->stream);
      return set_err(c, ABS_ERR_CAPACITY, "kd-tree environment: the tree build failed (device memory)");
    }
    DevGrid h{};
    int rc = read_grid(c, &h);
    if (rc) return rc;
    if (h.err == kErrNone) return ABS_OK;
    c->cur = cur0;  // the scatter did not run
    c->pos_in_new = pin0;
    c->grid_valid = false;
    CK(cudaMemsetAsync(c->start, 0, (c->bins_cap + 1) * 4, c->stream));
    if (h.err == kErrBinsRetry) {
      rc = ensure_bins(c, h.needed_bins);
      if (rc) return rc;
      rc = clear_dev_err(c);
      if (rc) return rc;
      continue;
    }
    rc = map_dev_err(c, h);
    clear_dev_err(c);
    CK(cudaStreamSynchronize(c->stream));
    return rc;
  }
  return set_err(c, ABS_ERR_STATE, "environment update did not converge");
}

int abs_gpu_grid_info(abs_gpu_ctx* c, double* grid, uint32_t* dims) {
  if (!c) return ABS_ERR_INVALID_ARGUMENT;
  DevGrid h{};
  int rc = read_grid(c, &h);
  if (rc) return rc;
  if (grid) {
    grid[0] = h.origin[0]; grid[1] = h.origin[1]; grid[2] = h.origin[2];
    grid[3] = h.box; grid[4] = h.dmax;
  }
  if (dims) { dims[0] = h.dims[0]; dims[1] = h.dims[1]; dims[2] = h.dims[2]; }
  return ABS_OK;
}

int abs_gpu_cell_ids(abs_gpu_ctx* c, uint64_t* out) {
  if (c && brute_env(c)) return set_err(c, ABS_ERR_STATE, "the brute_force and kd_tree environments have no cells");
  if (!c || !out) return ABS_ERR_INVALID_ARGUMENT;
  if (!c->grid_valid) return set_err(c, ABS_ERR_STATE, "cell ids require abs_gpu_env_update");
  DevGrid h{};
  int rc = read_grid(c, &h);
  if (rc) return rc;
  unsigned long long* d_out = nullptr;
  CK(dalloc(&d_out, h.n));
  k_cell_ids<<<grid_blocks(c, h.n), kThreads, 0, c->stream>>>(cur_pos(c), c->g, d_out);
  ++c->launches;
  CK(cudaMemcpyAsync(out, d_out, h.n * 8, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  cudaFree(d_out);
  return ABS_OK;
}

int abs_gpu_neighbors(abs_gpu_ctx* c, uint64_t* offsets, uint64_t* uids, uint64_t cap, uint64_t* total) {
  if (!c || !offsets) return ABS_ERR_INVALID_ARGUMENT;
  if (!c->grid_valid) return set_err(c, ABS_ERR_STATE, "neighbour queries require abs_gpu_env_update");
  DevGrid h{};
  int rc = read_grid(c, &h);
  if (rc) return rc;
  const unsigned long long n = h.n;
  unsigned long long *cnt = nullptr, *len = nullptr, *t64 = nullptr, *out = nullptr;
  CK(dalloc(&cnt, n + 1));
  CK(dalloc(&len, 1));
  CK(dalloc(&t64, (n + 1) / kScanTile + 2));
  CK(cudaMemcpyAsync(len, &n, 8, cudaMemcpyHostToDevice, c->stream));
  const Pd* pd = c->S[c->cur].pd;
  k_nbr_count<<<grid_blocks(c, n), kThreads, 0, c->stream>>>(pd, c->g, c->start, cnt, kd_view(c));
  ++c->launches;
  launch_scan<unsigned long long>(c, cnt, len, n + 1, t64, nullptr);
  CK(cudaMemcpyAsync(offsets, cnt, (n + 1) * 8, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  const unsigned long long tot = offsets[n];
  if (total) *total = tot;
  if (!uids || tot > cap) {
    cudaFree(cnt); cudaFree(len); cudaFree(t64);
    return uids ? set_err(c, ABS_ERR_CAPACITY, "neighbour buffer too small") : ABS_OK;
  }
  CK(dalloc(&out, tot));
  k_nbr_fill<<<grid_blocks(c, n), kThreads, 0, c->stream>>>(pd, c->S[c->cur].uid, c->g, c->start, cnt, out,
                                                           kd_view(c));
  ++c->launches;
  CK(cudaMemcpyAsync(uids, out, tot * 8, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  cudaFree(cnt); cudaFree(len); cudaFree(t64); cudaFree(out);
  return ABS_OK;
}

int abs_gpu_sort(abs_gpu_ctx* c) {
  if (!c) return ABS_ERR_INVALID_ARGUMENT;
  cudaSetDevice(c->device);
  DevGrid h{};
  int rc = read_grid(c, &h);
  if (rc) return rc;
  if (h.n == 0) return ABS_OK;
  rc = launch_sort(c, c->iteration, true);
  if (rc) return rc;
  CK(cudaGetLastError());
  rc = read_grid(c, &h);
  if (rc) return rc;
  if (h.err) {
    rc = map_dev_err(c, h);
    clear_dev_err(c);
    return rc;
  }
  return ABS_OK;
}

int abs_gpu_remove(abs_gpu_ctx* c, const uint64_t* uids, uint64_t r) {
  if (c) c->list_valid = false;  // storage order changes (neighbour lists index it)
  if (!c) return ABS_ERR_INVALID_ARGUMENT;
  if (r == 0) return ABS_OK;
  cudaSetDevice(c->device);
  DevGrid h{};
  int rc = read_grid(c, &h);
  if (rc) return rc;
  const unsigned long long n = h.n;
  if (r > n) return set_err(c, ABS_ERR_INVALID_ARGUMENT, "more removals than agents");
  if (h.nkeys != n) return set_err(c, ABS_ERR_STATE, "removals need the whole population in one context");
  // key-indexed removal marks and hole table (sized at upload only for models that add agents)
  rc = ensure_uid_space(c, h.nkeys + 1);
  if (rc) return rc;
  Soa& S = c->S[c->cur];
  // the removal list sorted on the host (O(r log r)) for the uid lookup;
  // duplicates are the reference's double-staging error (agent.hpp:136-141)
  std::vector<unsigned long long> perm(r);
  for (unsigned long long k = 0; k < r; ++k) perm[k] = k;
  std::sort(perm.begin(), perm.end(), [&](unsigned long long a, unsigned long long b) { return uids[a] < uids[b]; });
  std::vector<unsigned long long> su(r);
  for (unsigned long long k = 0; k < r; ++k) su[k] = uids[perm[k]];
  for (unsigned long long k = 1; k < r; ++k)
    if (su[k] == su[k - 1]) return set_err(c, ABS_ERR_STATE, "agent staged for removal twice");
  unsigned long long *d_su, *d_perm, *d_found, *d_slots, *len;
  unsigned int *to_right, *key_of, *hrank, *tiles;
  CK(dalloc(&d_su, r)); CK(dalloc(&d_perm, r)); CK(dalloc(&d_found, 1)); CK(dalloc(&d_slots, r));
  CK(dalloc(&len, 1)); CK(dalloc(&to_right, r + 1)); CK(dalloc(&key_of, r + 1)); CK(dalloc(&hrank, r + 1));
  CK(dalloc(&tiles, r / kScanTile + 2));
  auto release = [&] {
    cudaFree(d_su); cudaFree(d_perm); cudaFree(d_found); cudaFree(d_slots); cudaFree(len);
    cudaFree(to_right); cudaFree(key_of); cudaFree(hrank); cudaFree(tiles);
  };
  CK(cudaMemcpyAsync(d_su, su.data(), r * 8, cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(d_perm, perm.data(), r * 8, cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemsetAsync(d_found, 0, 8, c->stream));
  k_find_slots<<<grid_blocks(c, n), kThreads, 0, c->stream>>>(S.uid, c->g, d_su, d_perm, r, d_slots, d_found);
  ++c->launches;
  unsigned long long found = 0;
  CK(cudaMemcpyAsync(&found, d_found, 8, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (found != r) {
    release();
    return set_err(c, ABS_ERR_INVALID_ARGUMENT, "unknown uid");
  }
  // holes in the caller's list order (the reference's removal vector), movers
  // by key, then the same re-key + compaction as the loop-staged removals
  const unsigned long long new_size = n - r;
  const int nb = grid_blocks(c, r);
  k_api_mark<<<nb, kThreads, 0, c->stream>>>(S, d_slots, r, new_size, c->rmark, to_right, key_of);
  CK(cudaMemcpyAsync(hrank, to_right, r * 4, cudaMemcpyDeviceToDevice, c->stream));
  CK(cudaMemcpyAsync(len, &r, 8, cudaMemcpyHostToDevice, c->stream));
  launch_scan<unsigned int>(c, hrank, len, r, tiles, nullptr);
  k_api_holes<<<nb, kThreads, 0, c->stream>>>(to_right, hrank, key_of, r, c->hole_at);
  c->launches += 2;
  launch_removals(c, true);
  CK(cudaStreamSynchronize(c->stream));
  release();
  if (c->grid_valid) {
    CK(cudaMemsetAsync(c->start, 0, (c->bins_cap + 1) * 4, c->stream));
    c->grid_valid = false;
  }
  rc = read_grid(c, &h);
  if (rc) return rc;
  return ABS_OK;
}

void* abs_gpu_stream(abs_gpu_ctx* c) { return c ? c->stream : nullptr; }

int abs_gpu_set_stream(abs_gpu_ctx* c, void* stream) {
  if (!c || !stream) return ABS_ERR_INVALID_ARGUMENT;
  CK(cudaStreamSynchronize(c->stream));
  if (c->own_stream) cudaStreamDestroy(c->stream);
  c->stream = static_cast<cudaStream_t>(stream);
  c->own_stream = false;
  return ABS_OK;
}

int abs_gpu_force_kernel_time(abs_gpu_ctx* c, double* total_ms, uint64_t* launches) {
  if (!c) return ABS_ERR_INVALID_ARGUMENT;
  CK(cudaStreamSynchronize(c->stream));
  for (size_t q = 0; q + 1 < c->ev_used; q += 2) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, c->ev[q], c->ev[q + 1]));
    c->force_ms += ms;
    ++c->force_launches;
  }
  c->ev_used = 0;
  if (total_ms) *total_ms = c->force_ms;
  if (launches) *launches = c->force_launches;
  return ABS_OK;
}

int abs_gpu_phase_times(abs_gpu_ctx* c, double* out4, double* per_iteration_ms, uint64_t cap, uint64_t* n) {
  if (!c) return ABS_ERR_INVALID_ARGUMENT;
  CK(cudaStreamSynchronize(c->stream));
  for (size_t q = 0; q + 4 < c->pev_used; q += 5) {
    float t[4];
    for (int k = 0; k < 4; ++k) CK(cudaEventElapsedTime(&t[k], c->pev[q + k], c->pev[q + k + 1]));
    c->phase_ms[1] += t[0];  // sorting
    c->phase_ms[0] += t[1];  // environment update
    c->phase_ms[2] += t[2];  // agent ops
    c->phase_ms[3] += t[3];  // setup/teardown
    c->iter_ms.push_back(static_cast<double>(t[0]) + t[1] + t[2] + t[3]);
  }
  c->pev_used = 0;
  if (out4)
    for (int k = 0; k < 4; ++k) out4[k] = c->phase_ms[k];
  if (per_iteration_ms)
    for (size_t k = 0; k < c->iter_ms.size() && k < cap; ++k) per_iteration_ms[k] = c->iter_ms[k];
  if (n) *n = c->iter_ms.size();
  return ABS_OK;
}

int abs_gpu_record_evaluations(abs_gpu_ctx* c, int enable) {
  if (!c) return ABS_ERR_INVALID_ARGUMENT;
  c->rec_evals = enable != 0;
  if (c->rec_evals && c->evc_cap < c->cap) {
    CK(cudaStreamSynchronize(c->stream));
    cudaFree(c->evc);
    c->evc = nullptr;
    c->evc_cap = 0;
    CK(dalloc(&c->evc, c->cap));
    CK(cudaMemsetAsync(c->evc, 0, c->cap * sizeof(unsigned int), c->stream));
    c->evc_cap = c->cap;
  }
  return ABS_OK;
}

int abs_gpu_download_evaluations(abs_gpu_ctx* c, uint32_t* out, uint64_t cap) {
  if (!c || !out) return ABS_ERR_INVALID_ARGUMENT;
  if (!c->evc) return set_err(c, ABS_ERR_STATE, "evaluation recording is off (abs_gpu_record_evaluations)");
  DevGrid h{};
  int rc = read_grid(c, &h);
  if (rc) return rc;
  if (cap < h.n) return set_err(c, ABS_ERR_CAPACITY, "output holds fewer entries than agents");
  CK(cudaMemcpy(out, c->evc, h.n * sizeof(unsigned int), cudaMemcpyDeviceToHost));
  return ABS_OK;
}

int abs_gpu_download_storage_keys(abs_gpu_ctx* c, uint32_t* out, uint64_t cap) {
  if (!c || !out) return ABS_ERR_INVALID_ARGUMENT;
  cudaSetDevice(c->device);
  DevGrid h{};
  int rc = read_grid(c, &h);
  if (rc) return rc;
  if (cap < h.n) return set_err(c, ABS_ERR_CAPACITY, "output holds fewer entries than agents");
  if (h.n) CK(cudaMemcpy(out, c->S[c->cur].skey, h.n * sizeof(unsigned int), cudaMemcpyDeviceToHost));
  return ABS_OK;
}

int abs_gpu_list_stats(abs_gpu_ctx* c, uint64_t* out4, double* build_ms) {
  if (!c) return ABS_ERR_INVALID_ARGUMENT;
  CK(cudaStreamSynchronize(c->stream));
  for (size_t q = 0; q + 1 < c->bev_used; q += 2) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, c->bev[q], c->bev[q + 1]));
    c->build_ms += ms;
    ++c->build_launches;
  }
  c->bev_used = 0;
  unsigned int need = 0;
  CK(cudaMemcpy(&need, &c->g->list_need, sizeof need, cudaMemcpyDeviceToHost));
  if (out4) {
    out4[0] = c->list_builds;
    out4[1] = c->list_steps;
    out4[2] = c->build_launches;
    out4[3] = need;
  }
  if (build_ms) *build_ms = c->build_ms;
  return ABS_OK;
}

int abs_gpu_reset_timers(abs_gpu_ctx* c, int enable) {
  if (!c) return ABS_ERR_INVALID_ARGUMENT;
  CK(cudaStreamSynchronize(c->stream));
  c->ev_used = 0;
  c->bev_used = 0;
  c->build_ms = 0.0;
  c->build_launches = 0;
  c->force_ms = 0.0;
  c->force_launches = 0;
  c->pev_used = 0;
  for (double& v : c->phase_ms) v = 0.0;
  c->iter_ms.clear();
  c->timing = enable != 0;
  return ABS_OK;
}

}  // extern "C"

#include "decomp.cuh"
