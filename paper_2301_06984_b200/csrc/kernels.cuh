// kernels.cuh — sm_100a kernels of the mechanical step.
//
// Compiled with --fmad=false: every floating-point decision (d2 <= r2,
// overlap <= 0, floor((p-o)/box), clamp) and every force/integration term is
// evaluated with the same IEEE operations, in the same order, as the
// reference's g++ -O2 build (which contains no FMA). See DESIGN.md §Parity.
//
// HBM layout (per context, capacity C agents):
//   pd    : Pd[C]      {x, y, z, d} fp64, 32 B, cell order (ping-pong A/B)
//   newpd : Pd[C]      positions/diameters after integration (same order as pd)
//   uid   : u64[C]     flags: u8[C]   partners: u32[C]   vol: f64[C]  beh: u8[C]
//   force : f64[3C]    last_force (only when record_forces)
//   key/rank : u32[C]  bin of each agent / its slot inside the bin
//   start : u32[bins+1] exclusive scan of per-bin counts (the cell table)
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "absim_models.h"

#ifdef ABS_DEBUG
#include <cassert>
#define ABS_ASSERT(c) assert(c)
#else
#define ABS_ASSERT(c) ((void)0)
#endif

namespace absgpu {

constexpr int kThreads = 256;
constexpr int kScanTile = 2048;  // 256 threads x 8 values
#ifndef ABS_UNROLL
#define ABS_UNROLL 1
#endif
constexpr int kUnroll = ABS_UNROLL;  // candidate loads in flight per lane

struct __align__(32) Pd {
  double x, y, z, d;
};

enum DevErr : int {
  kErrNone = 0,
  kErrNonFinite = 1,
  kErrFixedBox = 2,
  kErrBoxBudget = 3,
  kErrBinsRetry = 4,  // internal: grow the bin table and re-run the iteration
  kErrCapRetry = 5,   // internal: grow agent capacity and re-run the iteration
  kErrQueryRadius = 6,  // a behaviour's query radius exceeds the box (uniform_grid.cpp:176-181)
  kErrSortRetry = 7,    // internal: the host's counting-sort guess did not fit; re-run with the exact path
  kErrListRebuild = 8,  // internal: the neighbour lists no longer cover the query radius; re-run as a rebuild
  kErrSlabs = 9,        // slab decomposition: fewer than 3 z-layers per rank
};

// Grid + bookkeeping living in device memory (one per context).
struct DevGrid {
  unsigned long long red[7];  // ordered-int min(x,y,z), max(x,y,z), max(d)
  unsigned int nonfinite;
  int err;
  unsigned int bad_input;  // set by k_ingest on a diameter <= 0
  unsigned long long work;  // chunk counter of the persistent force kernel (reset by k_finalize)
  unsigned long long failed_iteration;
  double origin[3];
  double box;
  double dmax;
  double s[3];    // internal bin edge per axis = box / B[k]
  double margin;  // conservative culling slack (absolute)
  unsigned int dims[3];
  unsigned int bd[3];  // bins per axis = B[k] * dims[k]
  unsigned int B[3];   // sub-bins per box edge per axis (x, y, z)
  unsigned int sort_passes;  // 8-bit radix passes the last k_sort_keys needs (even)
  unsigned int ysh;   // bin rows are stored in y-blocks of 2^ysh rows (row_of)
  unsigned int bd1p;  // bd[1] padded to a multiple of 2^ysh
  unsigned long long nbins;
  unsigned long long needed_bins;
  unsigned long long n;
  unsigned long long uid_count;
  unsigned long long staged;
  unsigned long long evals;
  unsigned long long skips;
  unsigned long long added;
  unsigned long long removed;
  unsigned long long sir[3];  // S/I/R counts after the last SIR iteration
  unsigned long long mark_n;  // staticness phase 1: listed disturbers / fresh agents
  unsigned long long fin_count;  // k_reduce_finalize: blocks done (last one sizes the grid)
  unsigned long long work_n;     // static detection: agents listed for the force sweep (k_static_pass)
  unsigned long long agent_its;  // sum over completed iterations of the agents at iteration start
  unsigned long long nkeys;      // size of the reference's storage (the key space): keys are 0..nkeys-1
  unsigned long long removed_now;  // removals staged this iteration (device-initiated)
  // --- kept across uploads (abs_gpu_upload copies everything above) ---
  int ov_on;               // multi-domain: use the global grid below
  int pad1;
  double ov_grid[5];       // origin[3], box, dmax over all ranks
  unsigned int ov_dims[3];
  unsigned int pad2;
  // --- in-loop Morton sort (set by k_sort_mode each sort) ---
  unsigned long long sort_len;  // counting mode: Morton code space (cell-table entries used)
  unsigned int sort_mode;       // 1 counting sort by code (in-box order free), 0 exact radix path
  unsigned int pad3;
  // --- neighbour lists ---
  double list_acc;              // sum over steps since the last build of the largest displacement (+ margin)
  double list_dmax;             // largest diameter when the lists were built
  unsigned int step_disp;       // float bits of this step's largest displacement (atomicMax)
  unsigned int list_need;       // largest candidate count seen by the last build
  double lorigin[3];            // grid origin at the build: list steps classify in fp32 relative to it
  float lslack;                 // fp32 classification slack of the list steps (build extent + skin)
  unsigned int list_incomplete; // the last build met more candidates than a list holds (those agents walk)
};

struct StepArgs {
  unsigned long long seed;
  unsigned long long iteration;
  double dt, k, max_disp, threshold2;
  double mp[8];
  int model;
  int detect_static;
  int record_forces;
  int brute;  // BruteForceEnvironment: no maximum query radius
  unsigned int* evc;  // per-agent force evaluations of the step (parity hook; nullptr = off)
  int track_disp;     // fold the step's largest displacement into DevGrid::step_disp (list policy)
};

// Order-preserving double <-> u64 map for atomicMin/atomicMax.
__device__ __forceinline__ unsigned long long ord_enc(double v) {
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double ord_dec(unsigned long long o) {
  const unsigned long long b = (o >> 63) ? (o & 0x7fffffffffffffffull) : ~o;
  return __longlong_as_double(static_cast<long long>(b));
}

// One 256-bit read-only load per record (sm_100: LDG.E.ENL2.256): half the
// L1 requests of two 128-bit loads on the gather-bound neighbour walks.
__device__ __forceinline__ Pd load_pd(const Pd* __restrict__ p) {
  Pd r;
  asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
               : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.d)
               : "l"(p));
  return r;
}

__device__ __forceinline__ int clamp_bin(double v, double s, unsigned int nb) {
  double t = floor(v / s);
  t = t < 0.0 ? 0.0 : t;
  const double hi = static_cast<double>(nb) - 1.0;
  t = t > hi ? hi : t;
  return static_cast<int>(t);
}

// Reference box coordinate (uniform_grid.cpp:28-37): floor((p-o)/box) clamped.
__device__ __forceinline__ unsigned int box_coord(double p, double o, double box, unsigned int dim) {
  const double rel = (p - o) / box;
  long long i = static_cast<long long>(floor(rel));
  i = i < 0 ? 0 : i;
  i = i > static_cast<long long>(dim) - 1 ? static_cast<long long>(dim) - 1 : i;
  return static_cast<unsigned int>(i);
}

// Internal bin along one axis: sub-bins nest exactly inside reference boxes.
__device__ __forceinline__ unsigned int bin_coord(double p, double o, const DevGrid& g, int k) {
  const unsigned int c = box_coord(p, o, g.box, g.dims[k]);
  if (g.B[k] == 1) return c;
  const double t = (p - o) - static_cast<double>(c) * g.box;
  return c * g.B[k] + static_cast<unsigned int>(clamp_bin(t, g.s[k], g.B[k]));
}

// Culling geometry of the current grid, in fp32 relative to the origin.
// Only used to choose WHICH bins to scan; every neighbour decision is the
// exact fp64 test. `slack` bounds the fp32 rounding of coordinates and bin
// edges, so the scanned set is a superset of the true neighbour set.
struct QGrid {
  double ox, oy, oz;
  double box;
  float inv_s[3];
  float s[3];
  float slack;
  unsigned int bd[3];
  unsigned int B[3];
  unsigned int dims[3];
  unsigned int ysh;
};

// Storage position of bin row (by, bz): rows are x-contiguous runs of the
// cell-ordered arrays, ordered by (y-block, z, y within the block). A
// front-to-back sweep over storage then walks one y-block column along z, so
// the rows its neighbour queries touch span (2^ysh + a few) x (a few) rows
// instead of whole z-layers: the candidate working set stays in L2 at any
// population size (bin index = x + bd[0] * row_of(...)).
__device__ __forceinline__ unsigned int row_of(unsigned int by, unsigned int bz, unsigned int ysh,
                                               unsigned int bd2) {
  return (((by >> ysh) * bd2 + bz) << ysh) + (by & ((1u << ysh) - 1u));
}

__device__ __forceinline__ QGrid make_qgrid(const DevGrid& g) {
  QGrid q;
  q.ox = g.origin[0];
  q.oy = g.origin[1];
  q.oz = g.origin[2];
  q.box = g.box;
  float ext = 1.0f;
  for (int k = 0; k < 3; ++k) {
    q.s[k] = static_cast<float>(g.s[k]);
    q.inv_s[k] = 1.0f / q.s[k];
    q.bd[k] = g.bd[k];
    q.B[k] = g.B[k];
    q.dims[k] = g.dims[k];
    ext = fmaxf(ext, static_cast<float>(g.s[k] * g.bd[k]));
  }
  q.ysh = g.ysh;
  q.slack = 16.0f * ext * 5.96046448e-8f + 1e-5f;
  return q;
}

__device__ __forceinline__ int fbin(float v, float inv_s, unsigned int nb) {
  const int i = __float2int_rd(v * inv_s);
  return min(max(i, 0), static_cast<int>(nb) - 1);
}

// Row chord half-width for culling: MUFU sqrt (relative error < 2^-22)
// inflated outward, so the chosen x range stays a superset.
__device__ __forceinline__ float cull_sqrt(float v) {
  float r;
  asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r * 1.000001f;
}

// Unclamped floor bin: callers clamp to the reference box range [lo, hi],
// which already lies inside [0, nb).
__device__ __forceinline__ int fbin_raw(float v, float inv_s) { return __float2int_rd(v * inv_s); }

// Bin range (inclusive) of the 3x3x3 reference boxes around the box holding
// c (uniform_grid.cpp:185-201): the reference never looks further, so
// neither do we — this keeps the candidate universe identical to the
// reference's even for agents that land exactly on a box boundary.
__device__ __forceinline__ void box_bin_range(const QGrid& g, double cx, double cy, double cz, int lo[3],
                                              int hi[3]) {
  const double c[3] = {cx, cy, cz};
  const double o[3] = {g.ox, g.oy, g.oz};
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int b = static_cast<int>(box_coord(c[k], o[k], g.box, g.dims[k]));
    lo[k] = (b > 0 ? b - 1 : 0) * static_cast<int>(g.B[k]);
    hi[k] = min(b + 2, static_cast<int>(g.dims[k])) * static_cast<int>(g.B[k]) - 1;
  }
}

// Visits every agent j != self whose exact fp64 squared distance to c is
// <= r2 (inclusive, vec3.hpp:44 evaluation order). Bins are culled
// conservatively row by row: for each (z, y) bin row the x extent is trimmed
// to the sphere's cross-section, and a row is one contiguous range of the
// cell-ordered arrays.
template <class F>
__device__ __forceinline__ void for_each_neighbor(const QGrid& g, const Pd* __restrict__ pd,
                                                  const unsigned int* __restrict__ start,
                                                  unsigned int self, double cx, double cy,
                                                  double cz, double r, double r2, F&& visit) {
  const float fx = static_cast<float>(cx - g.ox);
  const float fy = static_cast<float>(cy - g.oy);
  const float fz = static_cast<float>(cz - g.oz);
  const float rf = static_cast<float>(r) * 1.000001f + g.slack;
  const float rf2 = rf * rf;
  int bl[3], bh[3];
  box_bin_range(g, cx, cy, cz, bl, bh);
  const int z0 = max(fbin(fz - rf, g.inv_s[2], g.bd[2]), bl[2]), z1 = min(fbin(fz + rf, g.inv_s[2], g.bd[2]), bh[2]);
  const int y0 = max(fbin(fy - rf, g.inv_s[1], g.bd[1]), bl[1]), y1 = min(fbin(fy + rf, g.inv_s[1], g.bd[1]), bh[1]);
  for (int bz = z0; bz <= z1; ++bz) {
    const float zl = static_cast<float>(bz) * g.s[2];
    const float gz = fmaxf(fmaxf(zl - fz, fz - (zl + g.s[2])), 0.0f);
    for (int by = y0; by <= y1; ++by) {
      const float yl = static_cast<float>(by) * g.s[1];
      const float gy = fmaxf(fmaxf(yl - fy, fy - (yl + g.s[1])), 0.0f);
      const float rem = rf2 - (gy * gy + gz * gz);
      if (rem < 0.0f) continue;
      const float w = cull_sqrt(rem);
      const int x0 = max(fbin(fx - w, g.inv_s[0], g.bd[0]), bl[0]);
      const int x1 = min(fbin(fx + w, g.inv_s[0], g.bd[0]), bh[0]);
      const unsigned int row = g.bd[0] * row_of(static_cast<unsigned int>(by), static_cast<unsigned int>(bz), g.ysh, g.bd[2]);
      const unsigned int j1 = __ldg(start + row + x1 + 1);
      for (unsigned int j = __ldg(start + row + x0); j < j1; ++j) {
        if (j == self) continue;
        const Pd q = load_pd(pd + j);
        const double dx = cx - q.x, dy = cy - q.y, dz = cz - q.z;
        const double d2 = (dx * dx + dy * dy) + dz * dz;
        if (d2 <= r2) visit(j, q, dx, dy, dz, d2);
      }
    }
  }
}

// Flat-stream variant used by the force kernel. Phase 1 computes this
// lane's non-empty row windows (their `start` loads are independent, so they
// are all in flight together) into shared memory laid out [row][thread];
// phase 2 walks all windows as ONE candidate stream with a one-ahead
// prefetch, so a warp costs max(total candidates) rather than the sum over
// rows of the longest window. Rows beyond kMaxRows fall back to the nested
// walk. Visits exactly the same set as for_each_neighbor.
#ifndef ABS_MAX_ROWS
#define ABS_MAX_ROWS 32
#endif
#ifndef ABS_MAX_CONTACTS
#define ABS_MAX_CONTACTS 16
#endif
constexpr int kMaxRows = ABS_MAX_ROWS;
constexpr int kMaxContacts = ABS_MAX_CONTACTS;  // recorded possible contacts per agent (pass B)
#ifndef ABS_SPILL_CONTACTS
#define ABS_SPILL_CONTACTS 48
#endif
constexpr int kSpillContacts = ABS_SPILL_CONTACTS;  // further contacts kept per thread before a second walk
constexpr int kForceThreads = 128;
#ifndef ABS_BATCH
#define ABS_BATCH 4
#endif
constexpr int kBatch = ABS_BATCH;

// Box-lockstep variant (requires bins == reference boxes). Every lane walks
// the 3x3x3 reference boxes around ITS box as 9 contiguous x-runs
// (uniform_grid.cpp:198-200 without the per-lane trimming), so the lanes of a
// warp whose agents share a box fetch the same candidate at the same time:
// their loads coalesce into one broadcast instead of one L1 line per lane.
template <class F>
__device__ __forceinline__ void for_each_neighbor_box(const QGrid& g, const Pd* __restrict__ pd,
                                                      const unsigned int* __restrict__ start, unsigned int self,
                                                      double cx, double cy, double cz, double r2, F&& visit) {
  const int bx = static_cast<int>(box_coord(cx, g.ox, g.box, g.dims[0]));
  const int by = static_cast<int>(box_coord(cy, g.oy, g.box, g.dims[1]));
  const int bz = static_cast<int>(box_coord(cz, g.oz, g.box, g.dims[2]));
  const int x0 = max(bx - 1, 0), x1 = min(bx + 1, static_cast<int>(g.dims[0]) - 1);
  const int y0 = max(by - 1, 0), y1 = min(by + 1, static_cast<int>(g.dims[1]) - 1);
  const int z0 = max(bz - 1, 0), z1 = min(bz + 1, static_cast<int>(g.dims[2]) - 1);
  for (int z = z0; z <= z1; ++z)
    for (int y = y0; y <= y1; ++y) {
      const unsigned int row =
          g.dims[0] * row_of(static_cast<unsigned int>(y), static_cast<unsigned int>(z), g.ysh, g.dims[2]);
      const unsigned int j0 = __ldg(start + row + x0), j1 = __ldg(start + row + x1 + 1);
      for (unsigned int j = j0; j < j1; j += kBatch) {
        Pd q[kBatch];
#pragma unroll
        for (int u = 0; u < kBatch; ++u) q[u] = load_pd(pd + min(j + u, j1 - 1));
#pragma unroll
        for (int u = 0; u < kBatch; ++u) {
          const unsigned int jj = j + u;
          const double dx = cx - q[u].x, dy = cy - q[u].y, dz = cz - q[u].z;
          const double d2 = (dx * dx + dy * dy) + dz * dz;
          if (jj < j1 && jj != self && d2 <= r2) visit(jj, q[u], dx, dy, dz, d2);
        }
      }
    }
}


// ------------------------------------------------------------ kd-tree environment
// KdTreeEnvironment (kdtree_env.cpp:8-86) on the device: a balanced kd-tree
// over the agent array itself. The array is permuted so that every node owns
// a contiguous range [begin, end), split at its midpoint index along the
// widest axis of the range's bounding box (kdtree_env.cpp:31-50); ranges are
// implicit (they follow from n by the midpoint rule), nodes are addressed in
// heap order (children 2 id + 1, 2 id + 2) and store their split axis and the
// two bounds left_max >= every left coordinate, right_min <= every right
// coordinate. A range of <= kKdLeaf agents is a leaf (kLeafSize). The query
// (kdtree_env.cpp:55-84) descends with an explicit stack and applies the
// exact fp64 d2 <= r^2 to every agent of a reached leaf — the brute-force
// query contract, no maximum radius.
constexpr unsigned int kKdLeaf = 32;
struct KdView {
  const unsigned char* axis;
  const double* lmax;
  const double* rmin;
  unsigned int n;  // 0: no tree
};

template <class F>
__device__ __forceinline__ void for_each_neighbor_kd(const KdView& t, const Pd* __restrict__ pd, unsigned int self,
                                                     double cx, double cy, double cz, double r, double r2,
                                                     F&& visit) {
  if (t.n == 0) return;
  unsigned int sid[40], sb[40], se[40];
  int top = 1;
  sid[0] = 0;
  sb[0] = 0;
  se[0] = t.n;
  const double rr = r * (1.0 + 1e-12);  // pruning is conservative; membership is decided by d2 <= r2
  while (top > 0) {
    --top;
    const unsigned int id = sid[top], b = sb[top], e = se[top];
    if (e - b <= kKdLeaf) {
      for (unsigned int j = b; j < e; j += kBatch) {
        Pd q[kBatch];
#pragma unroll
        for (int u = 0; u < kBatch; ++u) q[u] = load_pd(pd + min(j + u, e - 1));
#pragma unroll
        for (int u = 0; u < kBatch; ++u) {
          const unsigned int jj = j + u;
          const double dx = cx - q[u].x, dy = cy - q[u].y, dz = cz - q[u].z;
          const double d2 = (dx * dx + dy * dy) + dz * dz;
          if (jj < e && jj != self && d2 <= r2) visit(jj, q[u], dx, dy, dz, d2);
        }
      }
      continue;
    }
    const unsigned int mid = b + (e - b) / 2;
    const unsigned int ax = t.axis[id];
    const double c = ax == 0 ? cx : (ax == 1 ? cy : cz);
    if (__ldg(t.rmin + id) - c <= rr) {  // right child (kdtree_env.cpp:82)
      sid[top] = 2 * id + 2;
      sb[top] = mid;
      se[top] = e;
      ++top;
    }
    if (c - __ldg(t.lmax + id) <= rr) {  // left child (kdtree_env.cpp:81)
      sid[top] = 2 * id + 1;
      sb[top] = b;
      se[top] = mid;
      ++top;
    }
  }
}

// Flat-stream, fp32-classified walk used by the force kernel. Candidates are read
// from `pf` (float4 {x, y, z, d} relative to the grid origin, 16 B) and
// classified against the exact fp64 test with a proven margin: the fp32
// distance differs from the fp64 one by less than `g.slack` (rounding of two
// relative coordinates of magnitude <= grid extent, their difference and the
// fp32 norm: < 7 ext 2^-24; slack = 16 ext 2^-24 + 1e-5). So
//   df2 <= (r - slack)^2  => the reference's d2 <= r^2 holds   (visit)
//   df2 >  (r + slack)^2  => it fails                           (skip)
// and only the thin band between re-reads the exact fp64 record and applies
// the reference's own test. The visited set is identical to
// for_each_neighbor's; visit(j, df2, qd) gets the fp32 squared distance and
// diameter (for the caller's conservative contact test).
template <class F>
__device__ __forceinline__ void for_each_neighbor_flat32(const QGrid& g, const Pd* __restrict__ pd,
                                                         const float4* __restrict__ pf,
                                                         const unsigned int* __restrict__ start,
                                                         unsigned int (*wj0)[kForceThreads],
                                                         unsigned short (*wj1)[kForceThreads],
                                                         unsigned int self, double cx, double cy,
                                                         double cz, double r, double r2, F&& visit) {
  const int t = threadIdx.x;
  const float fx = static_cast<float>(cx - g.ox);
  const float fy = static_cast<float>(cy - g.oy);
  const float fz = static_cast<float>(cz - g.oz);
  const float rf = static_cast<float>(r) * 1.000001f + g.slack;
  const float rf2 = rf * rf;
  const double sl = static_cast<double>(g.slack);
  const double rin = r - sl;
  const float rin2 = rin > 0.0 ? __double2float_rd(rin * rin * (1.0 - 0x1.0p-40)) : -1.0f;
  const float rout2 = __double2float_ru((r + sl) * (r + sl) * (1.0 + 0x1.0p-40));
  int bl[3], bh[3];
  box_bin_range(g, cx, cy, cz, bl, bh);
  const int z0 = max(fbin_raw(fz - rf, g.inv_s[2]), bl[2]), z1 = min(fbin_raw(fz + rf, g.inv_s[2]), bh[2]);
  const int y0 = max(fbin_raw(fy - rf, g.inv_s[1]), bl[1]), y1 = min(fbin_raw(fy + rf, g.inv_s[1]), bh[1]);
  // Classification of one candidate: `in` is exactly the reference's
  // j != self && fp64 d2 <= r2 (fp32 decides outside the margin band, fp64
  // inside it). Branch-free apart from the rare band reload; the visitor is
  // called for every slot with the decision (visit(j, df2, qd, in)).
  auto test = [&](unsigned int j, const float4& qf, bool valid) {
    const float ex = fx - qf.x, ey = fy - qf.y, ez = fz - qf.z;
    // fused: fewer roundings than the unfused sum, inside the same slack bound
    const float df2 = __fmaf_rn(ex, ex, __fmaf_rn(ey, ey, ez * ez));
    bool in = valid && j != self && df2 <= rout2;
    if (in && df2 > rin2) {  // margin band: the reference's exact fp64 test
      const Pd q = load_pd(pd + j);
      const double dx = cx - q.x, dy = cy - q.y, dz = cz - q.z;
      in = (dx * dx + dy * dy) + dz * dz <= r2;
    }
    visit(j, df2, qf.w, in);
  };
  // Phase 1a: row geometry only — the cell-table slots of each row's x range
  // [start[a0], start[a1]) go to the window arrays, no loads yet.
  int nr = 0;
  for (int bz = z0; bz <= z1; ++bz) {
    const float zl = static_cast<float>(bz) * g.s[2];
    const float gz = fmaxf(fmaxf(zl - fz, fz - (zl + g.s[2])), 0.0f);
    for (int by = y0; by <= y1; ++by) {
      const float yl = static_cast<float>(by) * g.s[1];
      const float gy = fmaxf(fmaxf(yl - fy, fy - (yl + g.s[1])), 0.0f);
      const float rem = rf2 - (gy * gy + gz * gz);
      if (rem < 0.0f) continue;
      const float w = cull_sqrt(rem);
      const int x0 = max(fbin_raw(fx - w, g.inv_s[0]), bl[0]);
      const int x1 = min(fbin_raw(fx + w, g.inv_s[0]), bh[0]);
      const unsigned int row = g.bd[0] * row_of(static_cast<unsigned int>(by), static_cast<unsigned int>(bz), g.ysh, g.bd[2]);
      if (nr < kMaxRows) {  // first bin and bin count of the row window
        wj0[nr][t] = row + x0;
        wj1[nr][t] = static_cast<unsigned short>(x1 + 1 - x0);
        ++nr;
      } else {  // overflow rows: nested walk
        const unsigned int j1 = __ldg(start + row + x1 + 1);
        for (unsigned int j = __ldg(start + row + x0); j < j1; ++j) test(j, __ldg(pf + j), true);
      }
    }
  }
  // Phase 1b: the cell-table loads, kRowBatch rows in flight at a time. Empty
  // windows are compacted out in place (write index <= read index) and the
  // rest are stored as one flat stream: window k covers flat positions
  // [P_k, P_{k+1}) and candidate index = flat position + off_k, with
  // off_k = start_k - P_k in wj0 and the bound P_{k+1} in wj1 (16 bits: a
  // window that would push the stream past 65535 candidates is walked
  // directly instead).
#ifndef ABS_ROW_BATCH
#define ABS_ROW_BATCH 4
#endif
  constexpr int kRowBatch = ABS_ROW_BATCH;
  int nw = 0;
  unsigned int total = 0;
  for (int r0 = 0; r0 < nr; r0 += kRowBatch) {
    unsigned int lo[kRowBatch], hi[kRowBatch];
#pragma unroll
    for (int u = 0; u < kRowBatch; ++u) {
      const int q = min(r0 + u, nr - 1);
      const unsigned int b0 = wj0[q][t];
      lo[u] = __ldg(start + b0);
      hi[u] = __ldg(start + b0 + wj1[q][t]);
    }
#pragma unroll
    for (int u = 0; u < kRowBatch; ++u) {
      if (r0 + u < nr && hi[u] > lo[u]) {
        if (total + (hi[u] - lo[u]) > 0xFFFFu) {  // stream bound would not fit 16 bits
          for (unsigned int j = lo[u]; j < hi[u]; ++j) test(j, __ldg(pf + j), true);
          continue;
        }
        wj0[nw][t] = lo[u] - total;
        total += hi[u] - lo[u];
        wj1[nw][t] = static_cast<unsigned short>(total);
        ++nw;
      }
    }
  }
#if defined(ABS_ABLATE) && ABS_ABLATE == 1
  if (nw > 1000) visit(self, 0.0f, 0.0f, true);  // timing ablation: rows only
  return;
#endif
  if (nw == 0) return;
  // Phase 2: the flat stream, kBatch candidates per step. Advancing a window
  // is a predicated reload (windows are non-empty), no per-candidate branch.
  int k = 0;
  unsigned int off = wj0[0][t], bnd = wj1[0][t];
  for (unsigned int p = 0; p < total;) {
    unsigned int idx[kBatch];
    bool val[kBatch];
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      val[u] = p < total;
      idx[u] = val[u] ? p + off : self;
      ++p;
      if (p == bnd) {
        k = min(k + 1, nw - 1);
        off = wj0[k][t];
        bnd = wj1[k][t];
      }
    }
    float4 qf[kBatch];
#pragma unroll
    for (int u = 0; u < kBatch; ++u) qf[u] = __ldg(pf + idx[u]);
#ifndef ABS_BAND_BATCH
#define ABS_BAND_BATCH 0  // c4 @ 2^26: 25.8 ms per-candidate vs 26.9 batched (2^24: 5.63 vs 5.50)
#endif
#if !ABS_BAND_BATCH
#pragma unroll
    for (int u = 0; u < kBatch; ++u) test(idx[u], qf[u], val[u]);
    continue;
#endif
    // classify the batch; one branch covers the (rare) margin-band reloads
    float df2[kBatch];
    bool in[kBatch];
    bool band = false;
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const float ex = fx - qf[u].x, ey = fy - qf[u].y, ez = fz - qf[u].z;
      df2[u] = __fmaf_rn(ex, ex, __fmaf_rn(ey, ey, ez * ez));
      in[u] = val[u] && idx[u] != self && df2[u] <= rout2;
      band |= in[u] && df2[u] > rin2;
    }
    if (band) {
#pragma unroll
      for (int u = 0; u < kBatch; ++u) {
        if (in[u] && df2[u] > rin2) {  // the reference's exact fp64 test
          const Pd q = load_pd(pd + idx[u]);
          const double dx = cx - q.x, dy = cy - q.y, dz = cz - q.z;
          in[u] = (dx * dx + dy * dy) + dz * dz <= r2;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kBatch; ++u) visit(idx[u], df2[u], qf[u].w, in[u]);
  }
}

// Candidate walk of the neighbour-list build: every agent j != self whose
// fp32 squared distance (relative coordinates from `pf`) is <= rf2 — a
// conservative superset of the exact fp64 ball of radius R when
// rf >= R * (1 + 1e-6) + slack. Rows cover the whole ball, clamped to the
// grid only (NOT to the reference's 3x3x3 boxes: R = r + skin may exceed the
// box, and the list must hold every agent that can come within r before the
// next rebuild). Same two-phase row windows as for_each_neighbor_flat32.
template <class F>
__device__ __forceinline__ void for_each_candidate32(const QGrid& g, const float4* __restrict__ pf,
                                                     const unsigned int* __restrict__ start,
                                                     unsigned int (*wj0)[kForceThreads],
                                                     unsigned short (*wj1)[kForceThreads], unsigned int self,
                                                     float fx, float fy, float fz, float rf, F&& visit) {
  const int t = threadIdx.x;
  const float rf2 = rf * rf;
  const int z0 = fbin(fz - rf, g.inv_s[2], g.bd[2]), z1 = fbin(fz + rf, g.inv_s[2], g.bd[2]);
  const int y0 = fbin(fy - rf, g.inv_s[1], g.bd[1]), y1 = fbin(fy + rf, g.inv_s[1], g.bd[1]);
  auto test = [&](unsigned int j, const float4& qf, bool valid) {
    const float ex = fx - qf.x, ey = fy - qf.y, ez = fz - qf.z;
    const float df2 = __fmaf_rn(ex, ex, __fmaf_rn(ey, ey, ez * ez));
    if (valid && j != self && df2 <= rf2) visit(j);
  };
  int nr = 0;
  for (int bz = z0; bz <= z1; ++bz) {
    const float zl = static_cast<float>(bz) * g.s[2];
    const float gz = fmaxf(fmaxf(zl - fz, fz - (zl + g.s[2])), 0.0f);
    for (int by = y0; by <= y1; ++by) {
      const float yl = static_cast<float>(by) * g.s[1];
      const float gy = fmaxf(fmaxf(yl - fy, fy - (yl + g.s[1])), 0.0f);
      const float rem = rf2 - (gy * gy + gz * gz);
      if (rem < 0.0f) continue;
      const float w = cull_sqrt(rem);
      const int x0 = fbin(fx - w, g.inv_s[0], g.bd[0]);
      const int x1 = fbin(fx + w, g.inv_s[0], g.bd[0]);
      const unsigned int row = g.bd[0] * row_of(static_cast<unsigned int>(by), static_cast<unsigned int>(bz), g.ysh, g.bd[2]);
      if (nr < kMaxRows) {
        wj0[nr][t] = row + x0;
        wj1[nr][t] = static_cast<unsigned short>(x1 + 1 - x0);
        ++nr;
      } else {  // overflow rows: direct walk
        const unsigned int j1 = __ldg(start + row + x1 + 1);
        for (unsigned int j = __ldg(start + row + x0); j < j1; ++j) test(j, __ldg(pf + j), true);
      }
    }
  }
  constexpr int kRowBatch = 4;
  int nw = 0;
  unsigned int total = 0;
  for (int r0 = 0; r0 < nr; r0 += kRowBatch) {
    unsigned int lo[kRowBatch], hi[kRowBatch];
#pragma unroll
    for (int u = 0; u < kRowBatch; ++u) {
      const int q = min(r0 + u, nr - 1);
      const unsigned int b0 = wj0[q][t];
      lo[u] = __ldg(start + b0);
      hi[u] = __ldg(start + b0 + wj1[q][t]);
    }
#pragma unroll
    for (int u = 0; u < kRowBatch; ++u) {
      if (r0 + u < nr && hi[u] > lo[u]) {
        if (total + (hi[u] - lo[u]) > 0xFFFFu) {
          for (unsigned int j = lo[u]; j < hi[u]; ++j) test(j, __ldg(pf + j), true);
          continue;
        }
        wj0[nw][t] = lo[u] - total;
        total += hi[u] - lo[u];
        wj1[nw][t] = static_cast<unsigned short>(total);
        ++nw;
      }
    }
  }
  if (nw == 0) return;
  int k = 0;
  unsigned int off = wj0[0][t], bnd = wj1[0][t];
  for (unsigned int p = 0; p < total;) {
    unsigned int idx[kBatch];
    bool val[kBatch];
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      val[u] = p < total;
      idx[u] = val[u] ? p + off : self;
      ++p;
      if (p == bnd) {
        k = min(k + 1, nw - 1);
        off = wj0[k][t];
        bnd = wj1[k][t];
      }
    }
    float4 qf[kBatch];
#pragma unroll
    for (int u = 0; u < kBatch; ++u) qf[u] = __ldg(pf + idx[u]);
#pragma unroll
    for (int u = 0; u < kBatch; ++u) test(idx[u], qf[u], val[u]);
  }
}

}  // namespace absgpu
