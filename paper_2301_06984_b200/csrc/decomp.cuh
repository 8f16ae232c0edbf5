// decomp.cuh — multi-GPU slab decomposition driven from inside the library
// (included at the end of absim_gpu.cu).
//
// One process (context) per GPU owns the agents whose reference-box z-layer
// lies in its slab [L[r], L[r+1]). Per iteration, on the context's stream:
//   1. local bounds {-lo, hi, dmax} (k_reduce) -> all-reduce(MAX) on the
//      device -> k_global_grid: the single-domain grid of all ranks
//      (uniform_grid.cpp:59-141, same IEEE operations) forced as the grid
//      override, so box geometry and cell ids equal the one-process run;
//   2. z-layer histogram of the owned agents -> all-reduce(SUM) ->
//      k_layer_bounds: slab edges with equal agent counts (the analogue of
//      the box-aligned domain shares of sort_balance.cpp:61-77), at least
//      kMinLayers layers thick, identical on every rank;
//   3. k_export_slab, ONE pass and ONE exchange per iteration: emigrants go
//      to the neighbouring slab as owned records, the two boundary layers as
//      ghost records; an emigrant that lands in the layer next to this slab
//      stays here as a ghost (its new owner's boundary layer), the others
//      leave. Slabs >= 2 layers and steps <= max_displacement (<= one box)
//      guarantee no agent crosses a whole slab (checked on the device);
//   4. the records are imported (owned or ghost), the iteration runs with
//      ghosts as candidates only (ABS_FLAG_GHOST), additions are committed
//      with daughter uids ranked over all ranks (division marks all-reduced,
//      commit.cpp:186-222), and the ghosts are dropped.
// Host synchronisations per iteration: the export counts (one mapped read)
// and the transport's count exchange; the all-reduces stay on the device.
//
// Transports: the built-in NCCL one (abs_gpu_comm_init, NCCL loaded with
// dlopen so the library does not depend on it) or caller callbacks
// (abs_gpu_comm_set_transport; the tests use torch.distributed gloo).
#pragma once

#include <dlfcn.h>
#include <nccl.h>

namespace {

constexpr int kHistBins = 4096;   // layer histogram bins (layers are coarsened beyond)
constexpr int kMinLayers = 2;     // slab thickness floor (the device checks that no agent crosses a slab)

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

// NCCL is resolved at run time: the process's already-loaded libnccl.so.2
// (e.g. torch's) if any, else the system one.
const NcclApi* nccl_api(std::string* why) {
  static NcclApi api;
  static bool tried = false;
  static std::string err;
  if (!tried) {
    tried = true;
    api.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!api.h) {
      err = std::string("libnccl.so.2 not found: ") + dlerror();
    } else {
      auto sym = [&](const char* n) { return dlsym(api.h, n); };
      api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
      api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
      api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
      api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
      api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
      api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
      api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
      api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
      api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
      if (!api.GetUniqueId || !api.CommInitRank || !api.AllReduce || !api.Send || !api.Recv || !api.GroupStart ||
          !api.GroupEnd || !api.CommDestroy) {
        err = "libnccl.so.2 lacks a required symbol";
        api.h = nullptr;
      }
    }
  }
  if (!api.h) {
    if (why) *why = err;
    return nullptr;
  }
  return &api;
}

// ---------------------------------------------------------------- kernels
// Local bounds from the reduction record as {-lo, hi, dmax} (one all-reduce
// with MAX yields the global bounds), then reset for the next reduction.
__global__ void k_bounds_out(DevGrid* g, double* __restrict__ b7) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  for (int k = 0; k < 7; ++k) {
    const double v = ord_dec(g->red[k]);
    b7[k] = k < 3 ? -v : v;
  }
  if (g->nonfinite) b7[6] = NAN;  // propagates through MAX as a non-finite bound
  reset_reduction(g);
}

// UniformGrid::update sizing (uniform_grid.cpp:112-141) on the all-reduced
// bounds; the result becomes the grid override of this context.
__global__ void k_global_grid(DevGrid* g, const double* __restrict__ b7, double fixed_box,
                              unsigned long long iteration) {
  if (threadIdx.x != 0 || blockIdx.x != 0 || g->err) return;
  double lo[3], hi[3];
  for (int k = 0; k < 3; ++k) {
    lo[k] = -b7[k];
    hi[k] = b7[3 + k];
  }
  const double dm = b7[6];
  int err = kErrNone;
  for (int k = 0; k < 3; ++k)
    if (!isfinite(lo[k]) || !isfinite(hi[k])) err = kErrNonFinite;
  if (!(dm == dm)) err = kErrNonFinite;
  double box = dm;
  if (err == kErrNone && fixed_box > 0.0) {
    if (dm > fixed_box) err = kErrFixedBox;
    box = fixed_box;
  }
  unsigned long long needed = 1;
  unsigned int dims[3] = {1, 1, 1};
  if (err == kErrNone) {
    for (int k = 0; k < 3; ++k) {
      const unsigned long long nk = static_cast<unsigned long long>(floor((hi[k] - lo[k]) / box)) + 1ull;
      dims[k] = static_cast<unsigned int>(nk < 1 ? 1 : nk);
      needed *= dims[k];
    }
    if (needed > (1ull << 31)) err = kErrBoxBudget;
  }
  if (err != kErrNone) {
    g->err = err;
    g->failed_iteration = iteration;
    return;
  }
  g->ov_on = 1;
  for (int k = 0; k < 3; ++k) {
    g->ov_grid[k] = lo[k];
    g->ov_dims[k] = dims[k];
  }
  g->ov_grid[3] = box;
  g->ov_grid[4] = dm;
}

__device__ __forceinline__ unsigned int layer_coarsening(unsigned int D) {
  return (D + kHistBins - 1) / kHistBins;
}

// Owned agents per (coarsened) z-layer of the override grid. Storage is
// cell-ordered, so neighbouring agents share a layer: counts gather in a
// shared-memory histogram per block (warp-aggregated increments), and only
// the non-zero bins reach global memory.
__global__ void __launch_bounds__(kThreads) k_layer_hist(const Pd* __restrict__ pos,
                                                         const unsigned char* __restrict__ flags, const DevGrid* g,
                                                         unsigned long long n, unsigned long long* __restrict__ hist) {
  __shared__ unsigned int sh[kHistBins];
  for (int b = threadIdx.x; b < kHistBins; b += blockDim.x) sh[b] = 0u;
  __syncthreads();
  const bool ok = !g->err;
  const unsigned int D = g->ov_dims[2];
  const unsigned int cz = layer_coarsening(D);
  const double oz = g->ov_grid[2], box = g->ov_grid[3];
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  for (unsigned long long b0 = blockIdx.x * (unsigned long long)blockDim.x; ok && b0 < n; b0 += stride) {
    const unsigned long long i = b0 + threadIdx.x;  // warp-uniform trip count
    int bin = -1;
    if (i < n && !(flags[i] & ABS_FLAG_GHOST)) bin = static_cast<int>(box_coord(pos[i].z, oz, box, D) / cz);
    const unsigned int peers = __match_any_sync(0xffffffffu, bin);
    if (bin >= 0 && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&sh[bin], __popc(peers));
  }
  __syncthreads();
  for (int b = threadIdx.x; b < kHistBins; b += blockDim.x)
    if (sh[b]) atomicAdd(hist + b, static_cast<unsigned long long>(sh[b]));
}

// Slab edges L[0..W] (layer indices): equal shares of the agents, snapped to
// (coarsened) layer edges, every slab >= kMinLayers thick. Deterministic
// from the all-reduced histogram, so every rank computes the same edges.
__global__ void k_layer_bounds(DevGrid* g, const unsigned long long* __restrict__ hist, int world,
                               long long* __restrict__ lb, int periodic, unsigned long long iteration) {
  if (threadIdx.x != 0 || blockIdx.x != 0 || g->err) return;
  const long long D = g->ov_dims[2];
  const long long cz = layer_coarsening(static_cast<unsigned int>(D));
  const long long nb = (D + cz - 1) / cz;
  if (D < static_cast<long long>(world) * kMinLayers) {
    g->err = kErrSlabs;
    g->failed_iteration = iteration;
    return;
  }
  unsigned long long total = 0;
  for (long long b = 0; b < nb; ++b) total += hist[b];
  lb[0] = 0;
  lb[world] = D;
  unsigned long long run = 0;
  long long b = 0;
  for (int r = 1; r < world; ++r) {
    const unsigned long long target = (total * static_cast<unsigned long long>(r)) / world;
    while (b < nb && run + hist[b] <= target) run += hist[b++];
    long long e = b * cz;  // first layer of the first bin past the target
    if (total == 0) e = (D * r) / world;
    const long long lo_ok = lb[r - 1] + kMinLayers;
    const long long hi_ok = D - static_cast<long long>(world - r) * kMinLayers;
    lb[r] = e < lo_ok ? lo_ok : (e > hi_ok ? hi_ok : e);
  }
  (void)periodic;
}

// One export pass (see the file header). Records carry the owned / ghost
// role in pad0. counts: [0] records to lo, [1] records to hi, [2] agents
// leaving this context, [3] agents that skipped a slab (error), [4] agents
// turned into local ghosts (k_import_slab adds the imported ghosts in [5]).
__global__ void k_export_slab(Pd* pos, Soa S, unsigned long long cap, unsigned long long n, const DevGrid* g,
                              const long long* __restrict__ lb, int rank, int world, int periodic,
                              Rec* __restrict__ out_lo, Rec* __restrict__ out_hi, unsigned long long out_cap,
                              unsigned long long* __restrict__ counts, unsigned int* __restrict__ keep) {
  if (g->err) return;
  const long long D = g->ov_dims[2];
  const double oz = g->ov_grid[2], box = g->ov_grid[3];
  const long long lo = lb[rank], hi = lb[rank + 1];
  const bool has_lo = periodic ? world > 1 : rank > 0;
  const bool has_hi = periodic ? world > 1 : rank < world - 1;
  const long long lo2 = periodic ? lb[(rank - 1 + world) % world] : (rank > 0 ? lb[rank - 1] : 0);
  const long long hi2 = periodic ? lb[(rank + 1) % world + 1] : (rank < world - 1 ? lb[rank + 2] : D);
  auto emit = [&](int dest, unsigned long long i, const Pd& p, unsigned char fl, bool owned) {
    const unsigned long long slot = atomicAdd(counts + dest, 1ull);
    if (slot >= out_cap) return;  // the host sees count > cap and fails
    Rec r;
    r.x = p.x; r.y = p.y; r.z = p.z; r.d = p.d;
    r.vol = S.vol[i];
    r.fx = S.force[i]; r.fy = S.force[cap + i]; r.fz = S.force[2 * cap + i];
    r.uid = S.uid[i];
    r.partners = S.partners[i];
    r.flags = static_cast<unsigned char>(fl & ~ABS_FLAG_GHOST);
    r.beh = S.beh[i];
    r.pad0 = owned ? 1 : 0;
    r.pad1 = 0;
    r.rngc = S.rngc[i];
    r.tag = S.tag[i];
    r.pad3 = S.skey[i];
    (dest ? out_hi : out_lo)[slot] = r;
  };
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    keep[i] = 1u;
    const unsigned char fl = S.flags[i];
    if (fl & ABS_FLAG_GHOST) continue;
    const Pd p = load_pd(pos + i);
    const long long layer = static_cast<long long>(box_coord(p.z, oz, box, static_cast<unsigned int>(D)));
    if (layer >= lo && layer < hi) {  // stays owned; boundary layers go out as ghosts
      if (has_lo && layer == lo) emit(0, i, p, fl, false);
      if (has_hi && layer == hi - 1) emit(1, i, p, fl, false);
      continue;
    }
    // emigrant: to the neighbour whose slab holds its layer
    int dest;
    bool adjacent;
    if (periodic) {
      const long long dlo = (lo - layer + D) % D, dhi = (layer - (hi - 1) + D) % D;
      dest = dlo <= dhi ? 0 : 1;
      const bool in_lo = ((layer - lo2 + D) % D) < ((lo - lo2 + D) % D ? (lo - lo2 + D) % D : D);
      const bool in_hi = ((layer - hi + D) % D) < ((hi2 - hi + D) % D ? (hi2 - hi + D) % D : D);
      if (!(dest == 0 ? in_lo : in_hi)) atomicAdd(counts + 3, 1ull);
      adjacent = dest == 0 ? layer == (lo - 1 + D) % D : layer == hi % D;
    } else {
      dest = layer < lo ? 0 : 1;
      if ((dest == 0 && (!has_lo || layer < lo2)) || (dest == 1 && (!has_hi || layer >= hi2)))
        atomicAdd(counts + 3, 1ull);
      adjacent = dest == 0 ? layer == lo - 1 : layer == hi;
    }
    emit(dest, i, p, fl, true);
    if (adjacent) {
      S.flags[i] = fl | ABS_FLAG_GHOST;  // its new owner's boundary layer: a candidate here
      atomicAdd(counts + 4, 1ull);
    } else {
      keep[i] = 0u;
      atomicAdd(counts + 2, 1ull);
    }
  }
}

// Append records at `base`: owned ones as agents of this context, the rest as ghosts.
__global__ void k_import_slab(const Rec* __restrict__ in, unsigned long long count, unsigned long long base,
                              Pd* __restrict__ pos, Soa S, unsigned long long cap,
                              unsigned long long* __restrict__ ghosts) {
  for (unsigned long long k = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; k < count;
       k += (unsigned long long)gridDim.x * blockDim.x) {
    const Rec r = in[k];
    const unsigned long long j = base + k;
    pos[j] = Pd{r.x, r.y, r.z, r.d};
    S.vol[j] = r.vol;
    S.force[j] = r.fx; S.force[cap + j] = r.fy; S.force[2 * cap + j] = r.fz;
    S.uid[j] = r.uid;
    S.partners[j] = r.partners;
    S.flags[j] = r.pad0 ? static_cast<unsigned char>(r.flags & ~ABS_FLAG_GHOST)
                        : static_cast<unsigned char>(r.flags | ABS_FLAG_GHOST);
    if (!r.pad0) atomicAdd(ghosts, 1ull);
    S.beh[j] = r.beh;
    S.tag[j] = r.tag;
    S.rngc[j] = r.rngc;
    S.skey[j] = r.pad3;  // the global storage key travels with the agent (k_export_slab)
  }
}

// Multi-domain additions rank daughters by reference storage key over ALL
// ranks; with no removals or sorts the reference's order is creation = uid
// order, so the global keys are the uids.
__global__ void k_keys_from_uids(Soa S, DevGrid* g) {
  const unsigned long long n = g->n;
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x)
    S.skey[i] = static_cast<unsigned int>(S.uid[i]);
  if (blockIdx.x == 0 && threadIdx.x == 0) g->nkeys = g->uid_count;
}

__global__ void k_clear_ghosts(unsigned char* __restrict__ flags, unsigned long long n) {
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x)
    flags[i] &= static_cast<unsigned char>(~ABS_FLAG_GHOST);
}

__global__ void k_count_owned(const unsigned char* __restrict__ flags, unsigned long long n,
                              unsigned long long* __restrict__ out) {
  unsigned long long c = 0;
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x)
    c += !(flags[i] & ABS_FLAG_GHOST);
  for (int off = 16; off; off >>= 1) c += __shfl_xor_sync(0xffffffffu, c, off);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

}  // namespace

// ---------------------------------------------------------------- host side
struct abs_gpu_decomp {
  int rank = 0, world = 1;
  bool periodic = false;
  abs_gpu_transport tr{};
  bool nccl = false;
  ncclComm_t comm = nullptr;
  double* b7 = nullptr;                 // device [7]
  unsigned long long* hist = nullptr;   // device [kHistBins]
  long long* lb = nullptr;              // device [world + 1]
  long long* hlb = nullptr;             // mapped host copy of lb
  unsigned long long* xc = nullptr;     // device [4] export counters
  unsigned long long* hxc = nullptr;    // mapped host copy
  unsigned long long* rcnt = nullptr;   // device [2] received counts (NCCL transport)
  unsigned long long* owned = nullptr;  // device [1]
  Rec* send[2] = {nullptr, nullptr};
  Rec* recv[2] = {nullptr, nullptr};
  unsigned long long rec_cap = 0;
  unsigned int* marks = nullptr;        // all-reduced division marks
  unsigned long long marks_cap = 0;
  int lo_peer = -1, hi_peer = -1;
};

namespace {

void decomp_free(abs_gpu_decomp* d) {
  if (!d) return;
  if (d->nccl && d->comm) {
    if (const NcclApi* api = nccl_api(nullptr)) api->CommDestroy(d->comm);
  }
  cudaFree(d->b7); cudaFree(d->hist); cudaFree(d->lb); cudaFree(d->xc); cudaFree(d->rcnt); cudaFree(d->owned);
  if (d->hlb) cudaFreeHost(d->hlb);
  if (d->hxc) cudaFreeHost(d->hxc);
  for (int k = 0; k < 2; ++k) {
    cudaFree(d->send[k]);
    cudaFree(d->recv[k]);
  }
  cudaFree(d->marks);
  delete d;
}

int decomp_records(abs_gpu_ctx* c, unsigned long long want) {
  abs_gpu_decomp* d = c->decomp;
  if (want <= d->rec_cap) return ABS_OK;
  const unsigned long long cap = std::max<unsigned long long>(want + want / 2, 1 << 16);
  CK(cudaStreamSynchronize(c->stream));
  for (int k = 0; k < 2; ++k) {
    cudaFree(d->send[k]);
    cudaFree(d->recv[k]);
    d->send[k] = d->recv[k] = nullptr;
  }
  d->rec_cap = 0;
  for (int k = 0; k < 2; ++k) {
    CK(dalloc(&d->send[k], cap));
    CK(dalloc(&d->recv[k], cap));
  }
  d->rec_cap = cap;
  return ABS_OK;
}

int decomp_setup(abs_gpu_ctx* c, int rank, int world) {
  if (world < 1 || rank < 0 || rank >= world) return set_err(c, ABS_ERR_INVALID_ARGUMENT, "bad rank / world size");
  abs_gpu_decomp* d = c->decomp;
  d->rank = rank;
  d->world = world;
  d->periodic = c->cfg.model == ABS_MODEL_SIR;
  if (world > 1) {
    d->lo_peer = d->periodic ? (rank - 1 + world) % world : (rank > 0 ? rank - 1 : -1);
    d->hi_peer = d->periodic ? (rank + 1) % world : (rank < world - 1 ? rank + 1 : -1);
  }
  CK(dalloc(&d->b7, 7));
  CK(dalloc(&d->hist, kHistBins));
  CK(dalloc(&d->lb, world + 1));
  CK(dalloc(&d->xc, 6));
  CK(dalloc(&d->rcnt, 2));
  CK(dalloc(&d->owned, 1));
  CK(cudaHostAlloc(reinterpret_cast<void**>(&d->hlb), (world + 1) * sizeof(long long), cudaHostAllocDefault));
  CK(cudaHostAlloc(reinterpret_cast<void**>(&d->hxc), 6 * sizeof(unsigned long long), cudaHostAllocDefault));
  if (removes_agents(c->cfg))
    return set_err(c, ABS_ERR_INVALID_ARGUMENT, "models that remove agents run in one domain");
  if (c->cfg.environment != ABS_ENV_UNIFORM_GRID)
    return set_err(c, ABS_ERR_INVALID_ARGUMENT, "the slab decomposition needs the uniform_grid environment");
  if (c->cfg.sorting_frequency > 0 && adds_agents(c->cfg))
    return set_err(c, ABS_ERR_INVALID_ARGUMENT,
                   "multi-domain additions with Morton sorting: the reference's global storage order is not tracked");
  if (adds_agents(c->cfg)) {
    int rc = abs_gpu_set_defer_commit(c, 1);
    if (rc) return rc;
    k_keys_from_uids<<<agent_blocks(c), kThreads, 0, c->stream>>>(c->S[c->cur], c->g);
    ++c->launches;
  }
  return decomp_records(c, 1 << 16);
}

// ---- the built-in NCCL transport ---------------------------------------------
int nccl_allreduce(void* user, void* dev, uint64_t count, int dtype, void* stream) {
  abs_gpu_decomp* d = static_cast<abs_gpu_decomp*>(user);
  const NcclApi* api = nccl_api(nullptr);
  const ncclDataType_t t = dtype == ABS_DT_F64_MAX ? ncclFloat64 : (dtype == ABS_DT_U64_SUM ? ncclUint64 : ncclUint32);
  const ncclRedOp_t op = dtype == ABS_DT_F64_MAX ? ncclMax : ncclSum;
  return api->AllReduce(dev, dev, count, t, op, d->comm, static_cast<cudaStream_t>(stream)) == ncclSuccess ? 0 : 1;
}

// Counts (device words, one host read), then the payload. Messages to one
// peer go lo-side first and are received hi-side first on every rank, so on
// a two-rank ring (both peers the same rank) NCCL's in-order matching pairs
// each message with the right buffer.
int nccl_counts(void* user, uint64_t n_lo, uint64_t n_hi, uint64_t* got_lo, uint64_t* got_hi, void* stream) {
  abs_gpu_decomp* d = static_cast<abs_gpu_decomp*>(user);
  const NcclApi* api = nccl_api(nullptr);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  unsigned long long* scnt = d->xc;  // xc[0..1] hold the send counts (k_export_slab)
  (void)n_lo;
  (void)n_hi;
  if (api->GroupStart() != ncclSuccess) return 1;
  if (d->lo_peer >= 0) api->Send(scnt + 0, 1, ncclUint64, d->lo_peer, d->comm, s);
  if (d->hi_peer >= 0) api->Send(scnt + 1, 1, ncclUint64, d->hi_peer, d->comm, s);
  if (d->hi_peer >= 0) api->Recv(d->rcnt + 1, 1, ncclUint64, d->hi_peer, d->comm, s);
  if (d->lo_peer >= 0) api->Recv(d->rcnt + 0, 1, ncclUint64, d->lo_peer, d->comm, s);
  if (api->GroupEnd() != ncclSuccess) return 1;
  unsigned long long r[2] = {0, 0};
  if (cudaMemcpyAsync(r, d->rcnt, 16, cudaMemcpyDeviceToHost, s) != cudaSuccess) return 1;
  if (cudaStreamSynchronize(s) != cudaSuccess) return 1;
  *got_lo = d->lo_peer >= 0 ? r[0] : 0;
  *got_hi = d->hi_peer >= 0 ? r[1] : 0;
  return 0;
}

int nccl_records(void* user, const void* send_lo, uint64_t n_lo, const void* send_hi, uint64_t n_hi, void* recv_lo,
                 uint64_t got_lo, void* recv_hi, uint64_t got_hi, void* stream) {
  abs_gpu_decomp* d = static_cast<abs_gpu_decomp*>(user);
  const NcclApi* api = nccl_api(nullptr);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (api->GroupStart() != ncclSuccess) return 1;
  if (d->lo_peer >= 0 && n_lo) api->Send(send_lo, n_lo * sizeof(Rec), ncclUint8, d->lo_peer, d->comm, s);
  if (d->hi_peer >= 0 && n_hi) api->Send(send_hi, n_hi * sizeof(Rec), ncclUint8, d->hi_peer, d->comm, s);
  if (d->hi_peer >= 0 && got_hi) api->Recv(recv_hi, got_hi * sizeof(Rec), ncclUint8, d->hi_peer, d->comm, s);
  if (d->lo_peer >= 0 && got_lo) api->Recv(recv_lo, got_lo * sizeof(Rec), ncclUint8, d->lo_peer, d->comm, s);
  return api->GroupEnd() == ncclSuccess ? 0 : 1;
}

int tr_fail(abs_gpu_ctx* c, const char* what) {
  return set_err(c, ABS_ERR_CUDA, std::string("decomposition transport failed in ") + what);
}

// One decomposed iteration (see the file header).
int decomp_step(abs_gpu_ctx* c) {
  abs_gpu_decomp* d = c->decomp;
  const int W = d->world;
  void* stream = c->stream;
  DevGrid h{};
  int rc = ABS_OK;
  unsigned long long n = c->n;  // host mirror, current after every call that changes it
  if (!d->periodic) {  // 1. global grid (config 5 keeps its fixed periodic grid)
    k_reduce<<<agent_blocks(c, 4), kThreads, 0, c->stream>>>(cur_pos(c), c->g);
    k_bounds_out<<<1, 1, 0, c->stream>>>(c->g, d->b7);
    c->launches += 2;
    if (W > 1 && d->tr.allreduce(d->tr.user, d->b7, 7, ABS_DT_F64_MAX, stream)) return tr_fail(c, "bounds all-reduce");
    k_global_grid<<<1, 1, 0, c->stream>>>(c->g, d->b7, c->cfg.fixed_box_length, c->iteration);
    ++c->launches;
    c->ov_on = true;
  }
  if (W == 1) {  // one slab: no neighbours, nothing to export or import
    rc = abs_gpu_simulate(c, 1);
    if (rc) return rc;
    if (c->defer_commit && adds_agents(c->cfg)) return abs_gpu_commit(c, nullptr, 0);
    return ABS_OK;
  }
  // 2. equal-count slab edges
  CK(cudaMemsetAsync(d->hist, 0, kHistBins * sizeof(unsigned long long), c->stream));
  if (n) k_layer_hist<<<grid_blocks(c, n), kThreads, 0, c->stream>>>(cur_pos(c), c->S[c->cur].flags, c->g, n, d->hist);
  if (W > 1 && d->tr.allreduce(d->tr.user, d->hist, kHistBins, ABS_DT_U64_SUM, stream))
    return tr_fail(c, "layer histogram all-reduce");
  k_layer_bounds<<<1, 1, 0, c->stream>>>(c->g, d->hist, W, d->lb, d->periodic ? 1 : 0, c->iteration);
  c->launches += 2;
  // 3. one export pass
  CK(cudaMemsetAsync(d->xc, 0, 6 * sizeof(unsigned long long), c->stream));
  if (n) {
    k_export_slab<<<grid_blocks(c, n), kThreads, 0, c->stream>>>(cur_pos(c), c->S[c->cur], c->cap, n, c->g, d->lb,
                                                                 d->rank, W, d->periodic ? 1 : 0, d->send[0],
                                                                 d->send[1], d->rec_cap, d->xc, c->rank);
    ++c->launches;
  }
  CK(cudaMemcpyAsync(d->hxc, d->xc, 5 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(d->hlb, d->lb, (W + 1) * sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
  rc = read_grid(c, &h);  // synchronises the stream
  if (rc) return rc;
  if (h.err) {
    rc = map_dev_err(c, h);
    clear_dev_err(c);
    return rc;
  }
  const unsigned long long n_lo = d->hxc[0], n_hi = d->hxc[1], leaving = d->hxc[2];
  if (d->hxc[3]) return set_err(c, ABS_ERR_STATE, "an agent crossed a whole slab in one iteration");
  if (n_lo > d->rec_cap || n_hi > d->rec_cap) {
    // records beyond the buffers were dropped: undo this export's ghost
    // marks (there are no other ghosts between iterations), grow, export again
    k_clear_ghosts<<<grid_blocks(c, n), kThreads, 0, c->stream>>>(c->S[c->cur].flags, n);
    ++c->launches;
    rc = decomp_records(c, std::max(n_lo, n_hi));
    if (rc) return rc;
    return decomp_step(c);
  }
  uint64_t got_lo = 0, got_hi = 0;
  if (W > 1) {
    if (d->tr.counts(d->tr.user, n_lo, n_hi, &got_lo, &got_hi, stream)) return tr_fail(c, "count exchange");
    rc = decomp_records(c, std::max<unsigned long long>(got_lo, got_hi));  // every rank posts its receive: grow here
    if (rc) return rc;
    if (d->tr.records(d->tr.user, d->send[0], n_lo, d->send[1], n_hi, d->recv[0], got_lo, d->recv[1], got_hi,
                      stream))
      return tr_fail(c, "record exchange");
  }
  // keep the buffers ahead of the traffic (no regrowth on the next iteration)
  rc = decomp_records(c, 2 * std::max<unsigned long long>(std::max(n_lo, n_hi), std::max<unsigned long long>(got_lo, got_hi)));
  if (rc) return rc;
  // 4. leave, arrive
  if (leaving) {
    rc = compact_population(c, n);
    if (rc) return rc;
    n = c->n;
  }
  const unsigned long long arrive = got_lo + got_hi;
  if (arrive) {
    rc = ensure_capacity(c, std::max<unsigned long long>(c->cap, 2 * (n + arrive) + 1024), n);
    if (rc) return rc;
    if (got_lo) k_import_slab<<<grid_blocks(c, got_lo), kThreads, 0, c->stream>>>(d->recv[0], got_lo, n, cur_pos(c),
                                                                                  c->S[c->cur], c->cap, d->xc + 5);
    if (got_hi) k_import_slab<<<grid_blocks(c, got_hi), kThreads, 0, c->stream>>>(d->recv[1], got_hi, n + got_lo,
                                                                                  cur_pos(c), c->S[c->cur], c->cap,
                                                                                  d->xc + 5);
    c->launches += 2;
    const unsigned long long nn = n + arrive;
    k_set_u64<<<1, 1, 0, c->stream>>>(&c->g->n, nn);
    ++c->launches;
    n = nn;
    c->n = nn;
    c->list_valid = false;
    if (c->grid_valid) dzero(c, c->start, (c->bins_cap + 1) * 4);
    c->grid_valid = false;
  }
  c->ghosts = n;  // upper bound (abs_gpu_drop_ghosts' no-op test); refined below
  rc = abs_gpu_simulate(c, 1);
  if (rc) return rc;
  CK(cudaMemcpyAsync(d->hxc + 5, d->xc + 5, sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  c->ghosts = d->hxc[4] + d->hxc[5];  // local ghost conversions + imported ghosts
  if (c->defer_commit && adds_agents(c->cfg)) {  // daughters: uids ranked over all ranks
    unsigned long long len = 0;
    DevGrid hh{};
    rc = read_grid(c, &hh);
    if (rc) return rc;
    len = hh.uid_count;
    if (len + 1 > d->marks_cap) {
      cudaFree(d->marks);
      d->marks = nullptr;
      d->marks_cap = 0;
      CK(dalloc(&d->marks, len + len / 2 + 1024));
      d->marks_cap = len + len / 2 + 1024;
    }
    if (len) CK(cudaMemcpyAsync(d->marks, c->div_mark, len * 4, cudaMemcpyDeviceToDevice, c->stream));
    if (W > 1 && len && d->tr.allreduce(d->tr.user, d->marks, len, ABS_DT_U32_SUM, stream))
      return tr_fail(c, "division marks all-reduce");
    rc = abs_gpu_commit(c, d->marks, len);
    if (rc) return rc;
  }
  return abs_gpu_drop_ghosts(c);
}

}  // namespace

void decomp_destroy(abs_gpu_ctx* c) {
  if (c && c->decomp) {
    decomp_free(c->decomp);
    c->decomp = nullptr;
  }
}

extern "C" {

int abs_gpu_nccl_unique_id(void* id) {
  std::string why;
  const NcclApi* api = nccl_api(&why);
  if (!api) return set_err(nullptr, ABS_ERR_NO_DEVICE, why);
  if (!id) return set_err(nullptr, ABS_ERR_INVALID_ARGUMENT, "null id");
  ncclUniqueId u;
  if (api->GetUniqueId(&u) != ncclSuccess) return set_err(nullptr, ABS_ERR_CUDA, "ncclGetUniqueId failed");
  std::memcpy(id, &u, sizeof u);
  return ABS_OK;
}

int abs_gpu_comm_init(abs_gpu_ctx* c, const void* nccl_id, int rank, int nranks) {
  if (!c || !nccl_id) return ABS_ERR_INVALID_ARGUMENT;
  std::string why;
  const NcclApi* api = nccl_api(&why);
  if (!api) return set_err(c, ABS_ERR_NO_DEVICE, why);
  cudaSetDevice(c->device);
  if (c->decomp) decomp_free(c->decomp);
  c->decomp = new abs_gpu_decomp();
  abs_gpu_decomp* d = c->decomp;
  ncclUniqueId u;
  std::memcpy(&u, nccl_id, sizeof u);
  if (api->CommInitRank(&d->comm, nranks, u, rank) != ncclSuccess) {
    delete d;
    c->decomp = nullptr;
    return set_err(c, ABS_ERR_CUDA, "ncclCommInitRank failed");
  }
  d->nccl = true;
  d->tr.user = d;
  d->tr.allreduce = nccl_allreduce;
  d->tr.counts = nccl_counts;
  d->tr.records = nccl_records;
  return decomp_setup(c, rank, nranks);
}

int abs_gpu_comm_set_transport(abs_gpu_ctx* c, const abs_gpu_transport* t, int rank, int nranks) {
  if (!c || !t || !t->allreduce || !t->counts || !t->records) return ABS_ERR_INVALID_ARGUMENT;
  cudaSetDevice(c->device);
  if (c->decomp) decomp_free(c->decomp);
  c->decomp = new abs_gpu_decomp();
  c->decomp->tr = *t;
  return decomp_setup(c, rank, nranks);
}

int abs_gpu_comm_reserve(abs_gpu_ctx* c, uint64_t records) {
  if (!c || !c->decomp) return set_err(c, ABS_ERR_STATE, "no communicator (abs_gpu_comm_init)");
  cudaSetDevice(c->device);
  return decomp_records(c, records);
}

int abs_gpu_simulate_decomposed(abs_gpu_ctx* c, uint64_t iterations) {
  if (!c) return ABS_ERR_INVALID_ARGUMENT;
  if (!c->decomp) return set_err(c, ABS_ERR_STATE, "no communicator (abs_gpu_comm_init)");
  cudaSetDevice(c->device);
  for (uint64_t k = 0; k < iterations; ++k) {
    const int rc = decomp_step(c);
    if (rc) return rc;
  }
  return ABS_OK;
}

int abs_gpu_memcpy(void* dst, const void* src, uint64_t bytes, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, s) != cudaSuccess) return ABS_ERR_CUDA;
  return cudaStreamSynchronize(s) == cudaSuccess ? ABS_OK : ABS_ERR_CUDA;
}

int abs_gpu_decomp_info(abs_gpu_ctx* c, int64_t* layer_bounds, uint64_t* owned) {
  if (!c || !c->decomp) return set_err(c, ABS_ERR_STATE, "no communicator (abs_gpu_comm_init)");
  abs_gpu_decomp* d = c->decomp;
  cudaSetDevice(c->device);
  DevGrid h{};
  int rc = read_grid(c, &h);
  if (rc) return rc;
  if (d->world == 1) {  // one slab: every layer
    d->hlb[0] = 0;
    d->hlb[1] = h.ov_on ? h.ov_dims[2] : h.dims[2];
  }
  if (layer_bounds)
    for (int r = 0; r <= d->world; ++r) layer_bounds[r] = d->hlb[r];
  if (owned) {
    CK(cudaMemsetAsync(d->owned, 0, 8, c->stream));
    if (h.n) k_count_owned<<<grid_blocks(c, h.n), kThreads, 0, c->stream>>>(c->S[c->cur].flags, h.n, d->owned);
    CK(cudaMemcpyAsync(owned, d->owned, 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  }
  return ABS_OK;
}

}  // extern "C"
