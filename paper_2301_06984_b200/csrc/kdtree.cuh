// kdtree.cuh — build of the device kd-tree environment (DESIGN.md §1 f4;
// included by absim_gpu.cu after the radix-sort kernels and host helpers).
// Traversal: for_each_neighbor_kd (kernels.cuh).
//
// KdTreeEnvironment::update (kdtree_env.cpp:8-52) partitions recursively with
// nth_element. On the device every level of the tree is built at once: the
// ranges of a level are contiguous and implicit (midpoint rule), so one pass
// finds each range's bounding box (its widest axis is the split axis,
// kdtree_env.cpp:31-44), one stable radix sort on (node id, coordinate along
// that axis) orders every range — a full sort where the reference only
// partitions around the median, which yields the same kind of tree — and one
// pass records the split bounds. log2(n / kKdLeaf) levels, then ONE gather
// moves the agent state into tree order.
#pragma once
// (included inside absim_gpu.cu's anonymous namespace)

// Order-preserving float -> u32 map.
__device__ __forceinline__ unsigned int ordf32(float v) {
  const unsigned int b = __float_as_uint(v);
  return (b >> 31) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float ordf32_dec(unsigned int o) {
  return __uint_as_float((o >> 31) ? (o & 0x7fffffffu) : ~o);
}

// The level-`level` node (heap id, range) that array position p falls in;
// a range of <= kKdLeaf positions is a leaf and is not split further.
__device__ __forceinline__ unsigned int kd_node_of(unsigned int p, unsigned int n, int level, unsigned int* b_out,
                                                   unsigned int* e_out) {
  unsigned int id = 0, b = 0, e = n;
  for (int l = 0; l < level && e - b > kKdLeaf; ++l) {
    const unsigned int mid = b + (e - b) / 2;
    if (p < mid) {
      e = mid;
      id = 2 * id + 1;
    } else {
      b = mid;
      id = 2 * id + 2;
    }
  }
  *b_out = b;
  *e_out = e;
  return id;
}

// Bounding box of every internal node of the level (ordered-u64 atomics,
// one set per warp when the warp's positions share a node).
__global__ void __launch_bounds__(kThreads) k_kd_bbox(const Pd* __restrict__ pos, const unsigned int* __restrict__ perm,
                                                      unsigned int n, int level, unsigned long long* __restrict__ bbox) {
  for (unsigned int p0 = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); p0 < n; p0 += gridDim.x * blockDim.x) {
    const unsigned int p = p0 + (threadIdx.x & 31);
    const bool live = p < n;
    unsigned int b = 0, e = 0;
    const unsigned int id = live ? kd_node_of(p, n, level, &b, &e) : 0xFFFFFFFFu;
    const bool internal = live && e - b > kKdLeaf;
    double v[3] = {0.0, 0.0, 0.0};
    if (internal) {
      const Pd q = load_pd(pos + perm[p]);
      v[0] = q.x;
      v[1] = q.y;
      v[2] = q.z;
    }
    const unsigned int first = __shfl_sync(0xffffffffu, id, 0);
    const bool uniform = __all_sync(0xffffffffu, id == first && internal);
    if (uniform) {
      double lo[3] = {v[0], v[1], v[2]}, hi[3] = {v[0], v[1], v[2]};
      for (int off = 16; off; off >>= 1)
        for (int k = 0; k < 3; ++k) {
          const double a = __shfl_xor_sync(0xffffffffu, lo[k], off), c = __shfl_xor_sync(0xffffffffu, hi[k], off);
          lo[k] = a < lo[k] ? a : lo[k];
          hi[k] = hi[k] < c ? c : hi[k];
        }
      if ((threadIdx.x & 31) == 0)
        for (int k = 0; k < 3; ++k) {
          atomicMin(bbox + 6ull * id + k, ord_enc(lo[k]));
          atomicMax(bbox + 6ull * id + 3 + k, ord_enc(hi[k]));
        }
    } else if (internal) {
      for (int k = 0; k < 3; ++k) {
        atomicMin(bbox + 6ull * id + k, ord_enc(v[k]));
        atomicMax(bbox + 6ull * id + 3 + k, ord_enc(v[k]));
      }
    }
  }
}

__global__ void k_kd_bbox_reset(unsigned long long* __restrict__ bbox, unsigned long long nodes) {
  for (unsigned long long q = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; q < nodes;
       q += (unsigned long long)gridDim.x * blockDim.x)
    for (int k = 0; k < 3; ++k) {
      bbox[6 * q + k] = ord_enc(INFINITY);
      bbox[6 * q + 3 + k] = ord_enc(-INFINITY);
    }
}

// Sort keys of the level: node id in the high word; below it the coordinate
// along the node's widest axis (kdtree_env.cpp:36-44: the first axis wins
// ties), rounded to fp32 and order-mapped — the rounding is monotone, and the
// split bounds recorded below absorb it — or, in a leaf, the position itself
// (leaves stay as they are).
__global__ void __launch_bounds__(kThreads) k_kd_keys(const Pd* __restrict__ pos, const unsigned int* __restrict__ perm,
                                                      unsigned int n, int level,
                                                      const unsigned long long* __restrict__ bbox,
                                                      unsigned char* __restrict__ axis,
                                                      unsigned long long* __restrict__ key,
                                                      unsigned int* __restrict__ idx) {
  for (unsigned int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
    unsigned int b, e;
    const unsigned int id = kd_node_of(p, n, level, &b, &e);
    const unsigned int i = perm[p];
    unsigned int low;
    if (e - b > kKdLeaf) {
      int ax = 0;
      double widest = ord_dec(bbox[6ull * id + 3]) - ord_dec(bbox[6ull * id]);
      for (int k = 1; k < 3; ++k) {
        const double w = ord_dec(bbox[6ull * id + 3 + k]) - ord_dec(bbox[6ull * id + k]);
        if (w > widest) {
          widest = w;
          ax = k;
        }
      }
      if (p == b) axis[id] = static_cast<unsigned char>(ax);
      const Pd q = load_pd(pos + i);
      low = ordf32(static_cast<float>(ax == 0 ? q.x : (ax == 1 ? q.y : q.z)));
    } else {
      low = p - b;
    }
    key[p] = (static_cast<unsigned long long>(id) << 32) | low;
    idx[p] = i;
  }
}

// Split bounds of the level's internal nodes from the sorted keys: every left
// key <= key[mid - 1] and fp32 rounding is to nearest, so the next float above
// bounds every left coordinate; likewise below key[mid] on the right.
__global__ void k_kd_split(const unsigned long long* __restrict__ key, unsigned int n, int level,
                           double* __restrict__ lmax, double* __restrict__ rmin) {
  const unsigned long long count = 1ull << level;
  for (unsigned long long q = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; q < count;
       q += (unsigned long long)gridDim.x * blockDim.x) {
    unsigned int id = 0, b = 0, e = n;
    bool internal = true;
    for (int l = 0; l < level; ++l) {
      if (e - b <= kKdLeaf) {
        internal = false;  // an ancestor is already a leaf: this path has no node here
        break;
      }
      const unsigned int mid = b + (e - b) / 2;
      if ((q >> (level - 1 - l)) & 1ull) {
        b = mid;
        id = 2 * id + 2;
      } else {
        e = mid;
        id = 2 * id + 1;
      }
    }
    if (!internal || e - b <= kKdLeaf) continue;
    const unsigned int mid = b + (e - b) / 2;
    const float kl = ordf32_dec(static_cast<unsigned int>(key[mid - 1]));
    const float kr = ordf32_dec(static_cast<unsigned int>(key[mid]));
    lmax[id] = static_cast<double>(nextafterf(kl, INFINITY));
    rmin[id] = static_cast<double>(nextafterf(kr, -INFINITY));
  }
}

__global__ void k_kd_iota(unsigned int* __restrict__ perm, unsigned int n) {
  for (unsigned int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) perm[p] = p;
}

__global__ void k_kd_set_passes(DevGrid* g, unsigned int passes) { g->sort_passes = passes; }

// KdTreeEnvironment::update for the current state (S[cur], n = the host's
// agent count): builds the tree and gathers the state into tree order.
int kd_build(abs_gpu_ctx* c) {
  const unsigned long long n = c->n;
  c->kd_valid = false;
  c->kd_n = n;
  if (n == 0) {
    c->kd_valid = true;
    return ABS_OK;
  }
  int levels = 0;
  while (((n + (1ull << levels) - 1) >> levels) > kKdLeaf) ++levels;  // deepest internal level + 1
  const unsigned long long nodes = 1ull << (levels + 1);
  if (nodes > c->kd_nodes_cap) {
    CK(cudaStreamSynchronize(c->stream));
    cudaFree(c->kd_axis); cudaFree(c->kd_lmax); cudaFree(c->kd_rmin); cudaFree(c->kd_bbox);
    c->kd_axis = nullptr; c->kd_lmax = nullptr; c->kd_rmin = nullptr; c->kd_bbox = nullptr;
    c->kd_nodes_cap = 0;
    CK(dalloc(&c->kd_axis, nodes));
    CK(dalloc(&c->kd_lmax, nodes));
    CK(dalloc(&c->kd_rmin, nodes));
    CK(dalloc(&c->kd_bbox, 6 * nodes));
    c->kd_nodes_cap = nodes;
  }
  int rc = ensure_sort_scratch(c);
  if (rc) return rc;
  const Pd* pos = cur_pos(c);
  const unsigned int un = static_cast<unsigned int>(n);
  const int nb = grid_blocks(c, n);
  const unsigned int blocks = static_cast<unsigned int>((c->cap + kSortChunk - 1) / kSortChunk);
  unsigned long long* k1 = c->sort_k[0];
  unsigned long long* k2 = c->sort_k[1];
  unsigned int* perm = c->sort_i[0];   // current permutation (position -> agent slot)
  unsigned int* i2 = c->sort_i[1];
  unsigned int* itmp = c->key;         // key/idx pairs of the level being sorted
  k_kd_iota<<<nb, kThreads, 0, c->stream>>>(perm, un);
  k_kd_bbox_reset<<<grid_blocks(c, nodes), kThreads, 0, c->stream>>>(c->kd_bbox, nodes);
  c->launches += 2;
  for (int level = 0; level < levels; ++level) {
    k_kd_bbox<<<nb, kThreads, 0, c->stream>>>(pos, perm, un, level, c->kd_bbox);
    k_kd_keys<<<nb, kThreads, 0, c->stream>>>(pos, perm, un, level, c->kd_bbox, c->kd_axis, k1, itmp);
    // stable LSD radix sort on the used key bits: 32 coordinate bits + node ids < 2^(level + 1)
    const unsigned int passes = (32u + static_cast<unsigned int>(level) + 1u + 7u) / 8u;
    k_kd_set_passes<<<1, 1, 0, c->stream>>>(c->g, passes);
    c->launches += 3;
    unsigned int* ia = itmp;
    unsigned int* ib = i2;
    for (unsigned int ps = 0; ps < passes; ++ps) {
      const int shift = static_cast<int>(8 * ps);
      k_radix_hist<<<blocks, kThreads, 0, c->stream>>>(k1, ia, c->g, shift, c->sort_hist, kSortChunk);
      launch_scan<unsigned int>(c, c->sort_hist, c->sort_hlen, 256ull * blocks, c->sort_tiles, nullptr);
      k_radix_scatter<<<blocks, 32, 0, c->stream>>>(k1, ia, k2, ib, c->g, shift, c->sort_hist, kSortChunk);
      c->launches += 2;
      std::swap(k1, k2);
      std::swap(ia, ib);
    }
    // ia now holds the level's sorted agent slots: the next permutation
    k_kd_split<<<grid_blocks(c, 1ull << level), kThreads, 0, c->stream>>>(k1, un, level, c->kd_lmax, c->kd_rmin);
    ++c->launches;
    CK(cudaMemcpyAsync(perm, ia, n * sizeof(unsigned int), cudaMemcpyDeviceToDevice, c->stream));
  }
  // the agent state in tree order (storage keys travel, they are not renumbered)
  const int nxt = c->cur ^ 1;
  k_gather<<<nb, kThreads, 0, c->stream>>>(pos, c->S[c->cur], c->S[nxt], perm, c->g, c->cap,
                                           c->cfg.model == ABS_MODEL_PROLIFERATION, c->cfg.record_forces, -1,
                                           uses_ext(c->cfg), 0);
  ++c->launches;
  c->cur = nxt;
  c->pos_in_new = false;
  c->kd_valid = true;
  return ABS_OK;
}
