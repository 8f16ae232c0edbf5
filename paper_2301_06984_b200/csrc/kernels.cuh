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

namespace absgpu {

constexpr int kThreads = 256;
constexpr int kScanTile = 2048;  // 256 threads x 8 values

struct __align__(16) Pd {
  double x, y, z, d;
};

enum DevErr : int {
  kErrNone = 0,
  kErrNonFinite = 1,
  kErrFixedBox = 2,
  kErrBoxBudget = 3,
  kErrBinsRetry = 4,  // internal: grow the bin table and re-run the iteration
  kErrCapRetry = 5,   // internal: grow agent capacity and re-run the iteration
};

// Grid + bookkeeping living in device memory (one per context).
struct DevGrid {
  unsigned long long red[7];  // ordered-int min(x,y,z), max(x,y,z), max(d)
  unsigned int nonfinite;
  int err;
  unsigned long long failed_iteration;
  double origin[3];
  double box;
  double dmax;
  double s;       // internal bin edge = box / B
  double margin;  // conservative culling slack (absolute)
  unsigned int dims[3];
  unsigned int bd[3];  // bins per axis = B * dims
  unsigned int B;
  unsigned int pad;
  unsigned long long nbins;
  unsigned long long needed_bins;
  unsigned long long n;
  unsigned long long uid_count;
  unsigned long long staged;
  unsigned long long evals;
  unsigned long long skips;
  unsigned long long added;
  unsigned long long removed;
};

struct StepArgs {
  unsigned long long seed;
  unsigned long long iteration;
  double dt, k, max_disp, threshold2;
  double mp[8];
  int model;
  int detect_static;
  int record_forces;
  int pad;
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

__device__ __forceinline__ Pd load_pd(const Pd* __restrict__ p) {
  const double2 a = __ldg(reinterpret_cast<const double2*>(p));
  const double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
  return Pd{a.x, a.y, b.x, b.y};
}

__device__ __forceinline__ int clamp_bin(double v, double s, unsigned int nb) {
  double t = floor(v / s);
  t = t < 0.0 ? 0.0 : t;
  const double hi = static_cast<double>(nb) - 1.0;
  t = t > hi ? hi : t;
  return static_cast<int>(t);
}

// Reference box coordinate (uniform_grid.cpp:124-133): floor((p-o)/box) clamped.
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
  if (g.B == 1) return c;
  const double t = (p - o) - static_cast<double>(c) * g.box;
  return c * g.B + static_cast<unsigned int>(clamp_bin(t, g.s, g.B));
}

// Visits every agent j != self whose exact fp64 squared distance to c is
// <= r2 (inclusive, vec3.hpp:44 evaluation order). Bins are culled
// conservatively (margin) row by row: for each (z, y) bin row the x extent
// is trimmed to the sphere's cross-section, and a row is one contiguous
// range of the cell-ordered arrays.
template <class F>
__device__ __forceinline__ void for_each_neighbor(const DevGrid& g, const Pd* __restrict__ pd,
                                                  const unsigned int* __restrict__ start,
                                                  unsigned int self, double cx, double cy,
                                                  double cz, double r, double r2, F&& visit) {
  const double rm = r + g.margin;
  const double rm2 = rm * rm;
  const double s = g.s;
  const int z0 = clamp_bin(cz - rm - g.origin[2], s, g.bd[2]);
  const int z1 = clamp_bin(cz + rm - g.origin[2], s, g.bd[2]);
  const int y0 = clamp_bin(cy - rm - g.origin[1], s, g.bd[1]);
  const int y1 = clamp_bin(cy + rm - g.origin[1], s, g.bd[1]);
  for (int bz = z0; bz <= z1; ++bz) {
    const double zl = g.origin[2] + bz * s;
    const double gz = cz < zl ? zl - cz : (cz > zl + s ? cz - (zl + s) : 0.0);
    for (int by = y0; by <= y1; ++by) {
      const double yl = g.origin[1] + by * s;
      const double gy = cy < yl ? yl - cy : (cy > yl + s ? cy - (yl + s) : 0.0);
      const double rem = rm2 - (gy * gy + gz * gz);
      if (rem < 0.0) continue;
      const double w = sqrt(rem);
      const int x0 = clamp_bin(cx - w - g.origin[0], s, g.bd[0]);
      const int x1 = clamp_bin(cx + w - g.origin[0], s, g.bd[0]);
      const unsigned int row = g.bd[0] * (static_cast<unsigned int>(by) + g.bd[1] * static_cast<unsigned int>(bz));
      const unsigned int j0 = __ldg(start + row + x0);
      const unsigned int j1 = __ldg(start + row + x1 + 1);
      for (unsigned int j = j0; j < j1; ++j) {
        if (j == self) continue;
        const Pd q = load_pd(pd + j);
        const double dx = cx - q.x, dy = cy - q.y, dz = cz - q.z;
        const double d2 = (dx * dx + dy * dy) + dz * dz;
        if (d2 <= r2) visit(j, q, dx, dy, dz, d2);
      }
    }
  }
}

}  // namespace absgpu
