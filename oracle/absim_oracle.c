/* absim_oracle.c — TEST INFRASTRUCTURE ONLY: CPU restatement of the
 * reference hot path, used solely as the checker by tests/, smoke() and
 * bench.py's cpu_baseline leg. Never linked into the product.
 *
 * Pinned against (a) the unmodified reference compiled by oracle/Makefile
 * (oracle/_ref/libabsim_ref.so; tests/test_oracle.py compares
 * every output bit-for-bit) and (b) the golden fixtures in tests/golden/.
 *
 * Semantics follow the reference with ONE worker and ONE domain (the only
 * bitwise-deterministic mode, test_scheduler.cpp:196-212):
 *   grid build        uniform_grid.cpp:59-170 (pass 1, sizing, LIFO chains)
 *   box_index_of      uniform_grid.cpp:28-37
 *   for_each_neighbor uniform_grid.cpp:172-230 (z,y,x boxes; chain order)
 *   pairwise force    mechanics.cpp:10-27
 *   run_forces        simulation.cpp:463-489
 *   integration       agent.hpp:115-133, simulation.cpp:491-500
 *   staticness        simulation.cpp:334-386, flags agent.hpp:61-101
 *   commit            commit.cpp:14-106 (5-step removal), :236-297 (appends),
 *                     mark_new_agent_neighbors simulation.cpp:510-530
 *   morton / offsets  morton.cpp:11-186
 *   sort_and_balance  sort_balance.cpp:22-148 (single domain)
 *   prefix sum        prefix_sum.cpp:11-51
 *   schedule          simulation.cpp:222-322
 * Model behaviours come from include/absim_models.h (shared definitions).
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "absim_models.h"

#define ORC_NIL UINT64_MAX
#define F_STATIC 1u
#define F_MOVED 2u
#define F_GREW 4u
#define F_NEWLY_ADDED 8u
#define F_NVIOL 16u
#define F_NNEW 32u
#define F_SELF_FORCE 64u
#define F_GHOST 128u /* halo copy owned by another rank: candidate only */

static char g_err[512];
const char* orc_last_error(void) { return g_err; }
static int fail(const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return -1;
}

typedef struct {
  uint64_t seed;
  int32_t threads, domains; /* ignored: always one worker, one domain */
  double dt, k, max_disp, threshold, fixed_box;
  uint64_t sorting_frequency;
  int32_t detect_static;
  int32_t model; /* 0 none, 1 volume grow/divide, 2 drive, 3 grow, 4 SIR,
                    5 models::GrowDivide, 6 models::Cohere */
  double mp[8];
  int32_t env; /* EnvironmentKind; the port restates the uniform grid only (0) */
  int32_t pad;
} orc_params;

typedef struct {
  orc_params p;
  uint64_t n, cap;
  uint64_t* uid;
  double *x, *y, *z, *d;
  double *tx, *ty, *tz, *tg; /* pending translation / growth */
  double *fx, *fy, *fz;
  uint32_t* partners;
  uint8_t* flags;
  uint8_t* beh;
  double* vol;
  uint32_t* tag;   /* Agent::tag (agent.hpp:35-36) */
  uint64_t* rngc;  /* Agent::rng_counter (agent.hpp:145, 188) */
  uint64_t uid_counter, iteration;
  uint64_t evals, skips, added, removed, sorted;
  /* grid */
  double origin[3], box, dmax;
  uint32_t dims[3];
  uint64_t indexed, nboxes, box_cap;
  uint64_t* head;
  uint64_t* succ;
  uint32_t* count;
  int grid_override;
  double ov_grid[5];
  uint32_t ov_dims[3];
  /* staged additions */
  uint64_t nstage, stage_cap;
  uint64_t* s_uid;
  double *s_x, *s_y, *s_z, *s_d, *s_vol;
  uint8_t* s_beh;
  uint32_t* s_tag;
  /* staged removals (AgentContext::remove_self, simulation.cpp:64-66): slots in loop order */
  uint32_t* rem;
  uint64_t nrem, rem_cap;
} orc_sim;

static void* xrealloc(void* p, size_t n) {
  void* q = realloc(p, n ? n : 1);
  if (!q) abort();
  return q;
}

static void reserve(orc_sim* s, uint64_t want) {
  if (want <= s->cap) return;
  uint64_t c = s->cap ? s->cap : 16;
  while (c < want) c *= 2;
#define GROW(f) s->f = xrealloc(s->f, c * sizeof(*s->f))
  GROW(uid); GROW(x); GROW(y); GROW(z); GROW(d); GROW(tx); GROW(ty); GROW(tz);
  GROW(tg); GROW(fx); GROW(fy); GROW(fz); GROW(partners); GROW(flags); GROW(beh);
  GROW(vol); GROW(succ); GROW(tag); GROW(rngc);
#undef GROW
  s->cap = c;
}

static void init_slot(orc_sim* s, uint64_t i, uint64_t uid, double x, double y, double z,
                      double d, uint8_t beh, double vol, uint8_t flags) {
  s->uid[i] = uid;
  s->x[i] = x; s->y[i] = y; s->z[i] = z; s->d[i] = d;
  s->tx[i] = s->ty[i] = s->tz[i] = s->tg[i] = 0.0;
  s->fx[i] = s->fy[i] = s->fz[i] = 0.0;
  s->partners[i] = 0;
  s->flags[i] = flags;
  s->beh[i] = beh;
  s->vol[i] = vol;
  s->tag[i] = 0;
  s->rngc[i] = 0;
}

orc_sim* orc_create(const orc_params* p, uint64_t n, const double* x, const double* y,
                    const double* z, const double* d, const uint8_t* mask) {
  if (p->env != 0) {
    fail("the port restates the uniform grid environment only");
    return NULL;
  }
  orc_sim* s = calloc(1, sizeof *s);
  s->p = *p;
  reserve(s, n);
  for (uint64_t i = 0; i < n; ++i) {
    if (!(d[i] > 0.0)) { /* agent.hpp:25 */
      free(s);
      fail("diameter must be > 0");
      return NULL;
    }
    uint8_t b = (mask == NULL || mask[i]) && p->model != 0;
    if (p->model == 4)  /* SIR: beh holds the state (absim_models.h) */
      b = abs_u01(abs_rng_word(p->seed, i, ABS_RNG_SIR_INIT)) < 0.01 ? ABS_SIR_I : ABS_SIR_S;
    init_slot(s, i, i, x[i], y[i], z[i], d[i], b,
              p->model == 1 ? abs_volume_of_diameter(d[i]) : 0.0, 0);
  }
  s->n = n;
  s->uid_counter = n;
  s->dims[0] = s->dims[1] = s->dims[2] = 1;
  return s;
}

/* Replace the population with a full state (uids, flags incl. F_GHOST,
 * partners, volume, behaviour mask) — teacher forcing and multi-domain. */
int orc_load(orc_sim* s, uint64_t n, const uint64_t* uid, const double* x, const double* y,
             const double* z, const double* d, const uint8_t* flags, const uint32_t* partners,
             const double* vol, const uint8_t* beh, uint64_t uid_count, uint64_t iteration) {
  reserve(s, n);
  for (uint64_t i = 0; i < n; ++i) {
    if (!(d[i] > 0.0)) return fail("diameter must be > 0");
    init_slot(s, i, uid[i], x[i], y[i], z[i], d[i], beh ? beh[i] : 0, vol ? vol[i] : 0.0,
              flags ? flags[i] : 0);
    if (partners) s->partners[i] = partners[i];
  }
  s->n = n;
  s->uid_counter = uid_count;
  s->iteration = iteration;
  s->indexed = 0;
  s->nstage = 0;
  return 0;
}

void orc_destroy(orc_sim* s) {
  if (!s) return;
  free(s->uid); free(s->x); free(s->y); free(s->z); free(s->d); free(s->tx);
  free(s->ty); free(s->tz); free(s->tg); free(s->fx); free(s->fy); free(s->fz);
  free(s->partners); free(s->flags); free(s->beh); free(s->vol); free(s->succ);
  free(s->tag); free(s->rngc);
  free(s->head); free(s->count); free(s->s_uid); free(s->s_x); free(s->s_y);
  free(s->s_z); free(s->s_d); free(s->s_vol); free(s->s_beh); free(s->s_tag); free(s->rem);
  free(s);
}

/* ---- uniform grid ------------------------------------------------------ */

/* uniform_grid.cpp:28-37 */
static uint64_t box_index_of(const orc_sim* s, double px, double py, double pz) {
  const double p[3] = {px, py, pz};
  uint64_t c[3];
  for (int k = 0; k < 3; ++k) {
    const double rel = (p[k] - s->origin[k]) / s->box;
    int64_t i = (int64_t)floor(rel);
    if (i < 0) i = 0;
    if (i > (int64_t)s->dims[k] - 1) i = (int64_t)s->dims[k] - 1;
    c[k] = (uint64_t)i;
  }
  return c[0] + s->dims[0] * (c[1] + (uint64_t)s->dims[1] * c[2]);
}

/* std::min / std::max argument order (b < a ? b : a), uniform_grid.cpp:95-96, 106-107 */
static double smin(double a, double b) { return b < a ? b : a; }
static double smax(double a, double b) { return a < b ? b : a; }

/* Multi-domain support: force the global grid (origin[3], box, dmax) and
 * dims computed over all ranks; grid == NULL clears it. */
int orc_set_grid_override(orc_sim* s, const double* grid, const uint32_t* dims) {
  s->grid_override = grid != NULL;
  if (grid) {
    for (int k = 0; k < 5; ++k) s->ov_grid[k] = grid[k];
    for (int k = 0; k < 3; ++k) s->ov_dims[k] = dims[k];
  }
  return 0;
}

/* uniform_grid.cpp:59-170 with one worker */
int orc_env_update(orc_sim* s, double* grid, uint32_t* dims, uint64_t* indexed) {
  s->indexed = s->n;
  if (s->n == 0) {
    s->dims[0] = s->dims[1] = s->dims[2] = 1;
    s->origin[0] = s->origin[1] = s->origin[2] = 0.0;
    s->box = s->p.fixed_box > 0.0 ? s->p.fixed_box : 1.0;
    s->dmax = 0.0;
    s->nboxes = 1;
  } else {
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    double dm = 0.0;
    for (uint64_t i = 0; i < s->n; ++i) {
      const double p[3] = {s->x[i], s->y[i], s->z[i]};
      for (int k = 0; k < 3; ++k) {
        lo[k] = smin(lo[k], p[k]);
        hi[k] = smax(hi[k], p[k]);
      }
      dm = smax(dm, s->d[i]);
    }
    for (int k = 0; k < 3; ++k)
      if (!isfinite(lo[k]) || !isfinite(hi[k])) return fail("agent positions are not finite");
    if (s->grid_override) { /* multi-domain: the global grid of all ranks */
      for (int k = 0; k < 3; ++k) {
        lo[k] = s->ov_grid[k];
        s->dims[k] = s->ov_dims[k];
      }
      dm = s->ov_grid[4];
    }
    s->dmax = dm;
    if (s->grid_override) {
      s->box = s->ov_grid[3];
    } else if (s->p.fixed_box > 0.0) {
      if (dm > s->p.fixed_box) return fail("fixed box length is smaller than the largest agent diameter");
      s->box = s->p.fixed_box;
    } else {
      s->box = dm;
    }
    uint64_t needed = 1;
    for (int k = 0; k < 3; ++k) {
      s->origin[k] = lo[k];
      if (!s->grid_override) {
        uint64_t nk = (uint64_t)floor((hi[k] - lo[k]) / s->box) + 1;
        s->dims[k] = (uint32_t)(nk < 1 ? 1 : nk);
      }
      needed *= s->dims[k];
    }
    if (needed > (1ull << 31)) return fail("grid would exceed the box budget");
    s->nboxes = needed;
  }
  if (s->nboxes > s->box_cap) {
    s->head = xrealloc(s->head, s->nboxes * sizeof *s->head);
    s->count = xrealloc(s->count, s->nboxes * sizeof *s->count);
    s->box_cap = s->nboxes;
  }
  for (uint64_t b = 0; b < s->nboxes; ++b) {
    s->head[b] = ORC_NIL;
    s->count[b] = 0;
  }
  if (s->n) {
    for (uint64_t i = 0; i < s->n; ++i) { /* :249-265, LIFO chains */
      const uint64_t b = box_index_of(s, s->x[i], s->y[i], s->z[i]);
      s->succ[i] = s->head[b];
      s->head[b] = i;
      s->count[b]++;
    }
  }
  if (grid) {
    grid[0] = s->origin[0]; grid[1] = s->origin[1]; grid[2] = s->origin[2];
    grid[3] = s->box; grid[4] = s->dmax;
  }
  if (dims) { dims[0] = s->dims[0]; dims[1] = s->dims[1]; dims[2] = s->dims[2]; }
  if (indexed) *indexed = s->indexed;
  return 0;
}

typedef void (*visit_fn)(orc_sim* s, void* ctx, uint64_t j, double d2);

/* uniform_grid.cpp:172-230; query == ORC_NIL means no exclusion */
static int for_each_neighbor(orc_sim* s, uint64_t query, double cx, double cy, double cz,
                             double r2, visit_fn fn, void* ctx) {
  if (s->indexed == 0) return 0;
  if (r2 > s->box * s->box * (1.0 + 1e-12)) return fail("query radius exceeds the grid box length");
  const double radius = sqrt(r2);
  const double c[3] = {cx, cy, cz};
  int64_t lo[3], hi[3];
  for (int k = 0; k < 3; ++k) {
    int64_t a = (int64_t)floor((c[k] - radius - s->origin[k]) / s->box);
    int64_t b = (int64_t)floor((c[k] + radius - s->origin[k]) / s->box);
    lo[k] = a > 0 ? a : 0;
    hi[k] = b < (int64_t)s->dims[k] - 1 ? b : (int64_t)s->dims[k] - 1;
  }
  const double cull = r2 * (1.0 + 1e-12);
  for (int64_t z = lo[2]; z <= hi[2]; ++z)
    for (int64_t y = lo[1]; y <= hi[1]; ++y)
      for (int64_t x = lo[0]; x <= hi[0]; ++x) {
        double min_d2 = 0.0;
        const int64_t at[3] = {x, y, z};
        for (int k = 0; k < 3; ++k) {
          const double b0 = s->origin[k] + (double)at[k] * s->box;
          const double b1 = b0 + s->box;
          const double gap = c[k] < b0 ? b0 - c[k] : (c[k] > b1 ? c[k] - b1 : 0.0);
          min_d2 += gap * gap;
        }
        if (min_d2 > cull) continue;
        uint64_t j = s->head[(uint64_t)x + s->dims[0] * ((uint64_t)y + (uint64_t)s->dims[1] * (uint64_t)z)];
        while (j != ORC_NIL) {
          if (j != query) {
            const double dx = cx - s->x[j], dy = cy - s->y[j], dz = cz - s->z[j];
            const double d2 = (dx * dx + dy * dy) + dz * dz; /* vec3.hpp:44 */
            if (d2 <= r2) fn(s, ctx, j, d2);
          }
          j = s->succ[j];
        }
      }
  return 0;
}

int orc_cell_ids(const orc_sim* s, uint64_t* out) {
  for (uint64_t i = 0; i < s->n; ++i) out[i] = box_index_of(s, s->x[i], s->y[i], s->z[i]);
  return 0;
}

typedef struct {
  uint64_t* buf;
  uint64_t n, cap;
} uidvec;
static void collect_uid(orc_sim* s, void* ctx, uint64_t j, double d2) {
  (void)d2;
  uidvec* v = ctx;
  if (v->n == v->cap) {
    v->cap = v->cap ? v->cap * 2 : 64;
    v->buf = xrealloc(v->buf, v->cap * sizeof *v->buf);
  }
  v->buf[v->n++] = s->uid[j];
}
static int cmp_u64(const void* a, const void* b) {
  const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : x > y;
}

/* Sorted force-query neighbour uids per agent (simulation.cpp:469). */
int64_t orc_neighbors(orc_sim* s, uint64_t* offsets, uint64_t* uids, uint64_t cap) {
  uidvec v = {0};
  uint64_t pos = 0;
  for (uint64_t i = 0; i < s->n; ++i) {
    v.n = 0;
    const double r = 0.5 * (s->d[i] + s->dmax);
    if (for_each_neighbor(s, i, s->x[i], s->y[i], s->z[i], r * r, collect_uid, &v)) {
      free(v.buf);
      return -1;
    }
    qsort(v.buf, v.n, sizeof(uint64_t), cmp_u64);
    offsets[i] = pos;
    for (uint64_t k = 0; k < v.n; ++k, ++pos)
      if (pos < cap) uids[pos] = v.buf[k];
  }
  offsets[s->n] = pos;
  free(v.buf);
  return pos > cap ? -2 : (int64_t)pos;
}

/* ---- mechanics ----------------------------------------------------------- */

/* random.hpp:47-52 unit_vector via RandomStream(seed=lo uid, stream=hi uid, counter 0) */
static void coincident_dir(uint64_t lo, uint64_t hi, double out[3]) {
  const double u0 = abs_u01(abs_rng_word(lo, hi, 0));
  const double u1 = abs_u01(abs_rng_word(lo, hi, 1));
  const double zz = -1.0 + (1.0 - -1.0) * u0;
  const double phi = 0.0 + (2.0 * ABS_PI - 0.0) * u1;
  const double r = sqrt(smax(0.0, 1.0 - zz * zz));
  out[0] = r * cos(phi);
  out[1] = r * sin(phi);
  out[2] = zz;
}

/* mechanics.cpp:10-27 */
static void pairwise_repulsion(const orc_sim* s, uint64_t a, uint64_t b, double k, double f[3]) {
  const double dx = s->x[a] - s->x[b], dy = s->y[a] - s->y[b], dz = s->z[a] - s->z[b];
  const double dist = sqrt((dx * dx + dy * dy) + dz * dz);
  const double overlap = 0.5 * (s->d[a] + s->d[b]) - dist;
  f[0] = f[1] = f[2] = 0.0;
  if (overlap <= 0.0) return;
  if (dist > 0.0) {
    const double sc = k * overlap / dist;
    f[0] = dx * sc; f[1] = dy * sc; f[2] = dz * sc;
    return;
  }
  const uint64_t lo = s->uid[a] < s->uid[b] ? s->uid[a] : s->uid[b];
  const uint64_t hi = s->uid[a] < s->uid[b] ? s->uid[b] : s->uid[a];
  double dir[3];
  coincident_dir(lo, hi, dir);
  if (s->uid[a] != lo) { dir[0] *= -1.0; dir[1] *= -1.0; dir[2] *= -1.0; }
  const double m = k * overlap;
  f[0] = dir[0] * m; f[1] = dir[1] * m; f[2] = dir[2] * m;
}

typedef struct {
  uint64_t a, evals;
  uint32_t contributors;
  double t[3];
} force_ctx;
static void force_visit(orc_sim* s, void* vctx, uint64_t j, double d2) {
  (void)d2;
  force_ctx* c = vctx;
  c->evals++;
  double f[3];
  pairwise_repulsion(s, c->a, j, s->p.k, f);
  if ((f[0] * f[0] + f[1] * f[1]) + f[2] * f[2] > 0.0) {
    c->contributors++;
    c->t[0] += f[0]; c->t[1] += f[1]; c->t[2] += f[2];
  }
}

/* simulation.cpp:463-489 */
static int run_forces(orc_sim* s, uint64_t i) {
  if (s->flags[i] & F_GHOST) return 0;
  if (s->p.detect_static && (s->flags[i] & F_STATIC)) {
    s->skips++;
    return 0;
  }
  const double r = 0.5 * (s->d[i] + s->dmax);
  force_ctx c = {i, 0, 0, {0.0, 0.0, 0.0}};
  if (for_each_neighbor(s, i, s->x[i], s->y[i], s->z[i], r * r, force_visit, &c)) return -1;
  s->evals += c.evals;
  s->fx[i] = c.t[0]; s->fy[i] = c.t[1]; s->fz[i] = c.t[2];
  s->partners[i] = c.contributors;
  const double n2 = (c.t[0] * c.t[0] + c.t[1] * c.t[1]) + c.t[2] * c.t[2];
  if (n2 > s->p.threshold * s->p.threshold) {
    s->tx[i] += c.t[0] * s->p.dt;
    s->ty[i] += c.t[1] * s->p.dt;
    s->tz[i] += c.t[2] * s->p.dt;
  }
  return 0;
}

/* agent.hpp:115-133 */
static void apply_pending(orc_sim* s, uint64_t i) {
  if (s->flags[i] & F_GHOST) return;
  double tx = s->tx[i], ty = s->ty[i], tz = s->tz[i];
  const double disp = sqrt((tx * tx + ty * ty) + tz * tz);
  if (disp > 0.0) {
    if (disp > s->p.max_disp) {
      const double sc = s->p.max_disp / disp;
      tx *= sc; ty *= sc; tz *= sc;
    }
    s->x[i] += tx; s->y[i] += ty; s->z[i] += tz;
    s->flags[i] |= F_MOVED;
  }
  if (s->tg[i] != 0.0) {
    const double dd = s->d[i] + s->tg[i];
    s->d[i] = dd > 1e-9 ? dd : 1e-9;
    if (s->tg[i] > 0.0) s->flags[i] |= F_GREW;
  }
  s->tx[i] = s->ty[i] = s->tz[i] = s->tg[i] = 0.0;
}

/* ---- staticness (simulation.cpp:334-386) ------------------------------- */
typedef struct {
  uint8_t set;
} mark_ctx;
static void mark_visit(orc_sim* s, void* vctx, uint64_t j, double d2) {
  (void)d2;
  s->flags[j] |= ((mark_ctx*)vctx)->set;
}

static int run_staticness(orc_sim* s) {
  const uint8_t reset = F_MOVED | F_GREW | F_SELF_FORCE | F_NEWLY_ADDED | F_NVIOL | F_NNEW;
  if (s->iteration == 0) {
    for (uint64_t i = 0; i < s->n; ++i)
      if (!(s->flags[i] & F_GHOST)) s->flags[i] &= (uint8_t)~(reset | F_STATIC);
    return 0;
  }
  for (uint64_t i = 0; i < s->n; ++i) {
    const int disturbs = (s->flags[i] & (F_MOVED | F_GREW)) != 0;
    const int fresh = (s->flags[i] & F_NEWLY_ADDED) != 0;
    if (!disturbs && !fresh) continue;
    const double r = 0.5 * (s->d[i] + s->dmax);
    mark_ctx m = {(uint8_t)((disturbs ? F_NVIOL : 0) | (fresh ? F_NNEW : 0))};
    if (for_each_neighbor(s, i, s->x[i], s->y[i], s->z[i], r * r, mark_visit, &m)) return -1;
  }
  for (uint64_t i = 0; i < s->n; ++i) {
    if (s->flags[i] & F_GHOST) continue;
    const int skip = !(s->flags[i] & (F_MOVED | F_GREW | F_SELF_FORCE | F_NEWLY_ADDED | F_NVIOL | F_NNEW)) &&
                     s->partners[i] <= 1;
    s->flags[i] = (uint8_t)((s->flags[i] & ~(reset | F_STATIC)) | (skip ? F_STATIC : 0));
  }
  return 0;
}

/* ---- behaviours (absim_models.h / models.hpp:69-83) -------------------- */
static void stage_daughter_tag(orc_sim* s, double x, double y, double z, double d, double vol, uint32_t tag);
static void stage_daughter(orc_sim* s, double x, double y, double z, double d, double vol) {
  stage_daughter_tag(s, x, y, z, d, vol, 0);
}

static void stage_daughter_tag(orc_sim* s, double x, double y, double z, double d, double vol, uint32_t tag) {
  if (s->nstage == s->stage_cap) {
    s->stage_cap = s->stage_cap ? 2 * s->stage_cap : 64;
    s->s_uid = xrealloc(s->s_uid, s->stage_cap * sizeof *s->s_uid);
    s->s_x = xrealloc(s->s_x, s->stage_cap * sizeof *s->s_x);
    s->s_y = xrealloc(s->s_y, s->stage_cap * sizeof *s->s_y);
    s->s_z = xrealloc(s->s_z, s->stage_cap * sizeof *s->s_z);
    s->s_d = xrealloc(s->s_d, s->stage_cap * sizeof *s->s_d);
    s->s_vol = xrealloc(s->s_vol, s->stage_cap * sizeof *s->s_vol);
    s->s_beh = xrealloc(s->s_beh, s->stage_cap * sizeof *s->s_beh);
    s->s_tag = xrealloc(s->s_tag, s->stage_cap * sizeof *s->s_tag);
  }
  const uint64_t k = s->nstage++;
  s->s_uid[k] = s->uid_counter++; /* resource_manager.hpp:44-46 at creation */
  s->s_x[k] = x; s->s_y[k] = y; s->s_z[k] = z; s->s_d[k] = d;
  s->s_vol[k] = vol;
  s->s_beh[k] = 1;
  s->s_tag[k] = tag;
}

/* RandomStream::unit_vector (random.hpp:47-52) on the agent's own stream:
 * two draws at the agent's counter (advanced), cos/sin from libm. */
static void orc_unit_vector(uint64_t seed, uint64_t uid, uint64_t* counter, double out[3]) {
  const double u1 = abs_u01(abs_rng_word(seed, uid, (*counter)++));
  const double zz = -1.0 + (1.0 - -1.0) * u1;
  const double two_pi = 2.0 * 3.14159265358979323846;
  const double u2 = abs_u01(abs_rng_word(seed, uid, (*counter)++));
  const double phi = 0.0 + (two_pi - 0.0) * u2;
  const double r = sqrt(smax(0.0, 1.0 - zz * zz));
  out[0] = r * cos(phi);
  out[1] = r * sin(phi);
  out[2] = zz;
}

typedef struct {
  double sx, sy, sz;
  uint64_t count;
  uint32_t tag;
} cohere_ctx;

static void cohere_visit(orc_sim* s, void* vctx, uint64_t j, double d2) {
  (void)d2;
  cohere_ctx* c = (cohere_ctx*)vctx;
  if (s->tag[j] != c->tag) return;
  c->sx += s->x[j]; c->sy += s->y[j]; c->sz += s->z[j];
  ++c->count;
}

static int run_behaviour(orc_sim* s, uint64_t i) {
  if (!s->beh[i] || (s->flags[i] & F_GHOST)) return 0;
  const orc_params* p = &s->p;
  if (p->model == 1) {
    s->vol[i] += p->mp[0];
    if (s->vol[i] > p->mp[1]) {
      s->vol[i] *= 0.5;
      double dir[3];
      abs_unit_vector(p->seed, s->uid[i], ABS_RNG_DIVISION_BASE(s->iteration), dir);
      const double half = 0.5 * s->d[i];
      const double dd = abs_diameter_of_volume(s->vol[i]);
      if (!(dd > 0.0)) return fail("diameter must be > 0");
      stage_daughter(s, s->x[i] + dir[0] * half, s->y[i] + dir[1] * half,
                     s->z[i] + dir[2] * half, dd, s->vol[i]);
    }
    s->tg[i] += abs_diameter_of_volume(s->vol[i]) - s->d[i];
  } else if (p->model == 2) {
    double dl[3];
    abs_drive_delta(s->x[i], s->y[i], s->z[i], p->mp[0], p->mp[1], p->mp[2], p->mp[3],
                    p->seed, s->uid[i], s->iteration, dl);
    s->tx[i] += dl[0]; s->ty[i] += dl[1]; s->tz[i] += dl[2];
  } else if (p->model == 3) { /* models::Grow (models.hpp:69-83) */
    const double cap = p->mp[1];
    if (s->d[i] < cap) {
      const double rem = cap - s->d[i];
      s->tg[i] += rem < p->mp[0] ? rem : p->mp[0];
    }
  } else if (p->model == 7 &&
             abs_u01(abs_rng_word(p->seed, s->uid[i], ABS_RNG_DEATH(s->iteration))) < p->mp[3]) {
    /* GrowDivide + remove_self (absim_gpu.h ABS_MODEL_GROW_DIVIDE_DIE): staged in loop order */
    if (s->nrem == s->rem_cap) {
      s->rem_cap = s->rem_cap ? 2 * s->rem_cap : 64;
      s->rem = xrealloc(s->rem, s->rem_cap * sizeof *s->rem);
    }
    s->rem[s->nrem++] = (uint32_t)i;
  } else if (p->model == 5 || p->model == 7) { /* models::GrowDivide (models.hpp:15-37): mp rate, threshold, initial d */
    if (s->d[i] >= p->mp[1]) {
      double dir[3];
      orc_unit_vector(p->seed, s->uid[i], &s->rngc[i], dir); /* ctx.random(), random.hpp:47-52 */
      const double half = 0.5 * s->d[i];
      stage_daughter_tag(s, s->x[i] + dir[0] * half, s->y[i] + dir[1] * half, s->z[i] + dir[2] * half,
                         p->mp[2], 0.0, s->tag[i]);
      s->tg[i] += p->mp[2] - s->d[i];
    } else {
      s->tg[i] += p->mp[0];
    }
  } else if (p->model == 6) { /* models::Cohere (models.hpp:42-64): mp attraction radius, speed */
    cohere_ctx cc = {0.0, 0.0, 0.0, 0, s->tag[i]};
    if (for_each_neighbor(s, i, s->x[i], s->y[i], s->z[i], p->mp[0] * p->mp[0], cohere_visit, &cc)) return -1;
    if (cc.count == 0) return 0;
    const double inv = 1.0 / (double)cc.count;
    const double tx = cc.sx * inv - s->x[i], ty = cc.sy * inv - s->y[i], tz = cc.sz * inv - s->z[i];
    const double dist = sqrt((tx * tx + ty * ty) + tz * tz);
    if (dist > 0.0) {
      const double f = p->mp[1] / dist;
      s->tx[i] += tx * f; s->ty[i] += ty * f; s->tz[i] += tz * f;
    }
  }
  return 0;
}

/* ---- commit ---------------------------------------------------------------- */

static void nn_visit(orc_sim* s, void* vctx, uint64_t j, double d2) {
  (void)vctx; (void)d2;
  s->flags[j] |= F_NNEW;
}

/* simulation.cpp:510-530: start-of-step grid, live positions, no exclusion */
static int mark_new_agent_neighbors(orc_sim* s) {
  for (uint64_t k = 0; k < s->nstage; ++k) {
    const double r = 0.5 * (s->s_d[k] + s->dmax);
    if (r <= s->box) {
      if (for_each_neighbor(s, ORC_NIL, s->s_x[k], s->s_y[k], s->s_z[k], r * r, nn_visit, NULL)) return -1;
    } else {
      for (uint64_t j = 0; j < s->n; ++j) {
        const double dx = s->s_x[k] - s->x[j], dy = s->s_y[k] - s->y[j], dz = s->s_z[k] - s->z[j];
        if ((dx * dx + dy * dy) + dz * dz <= r * r) s->flags[j] |= F_NNEW;
      }
    }
  }
  return 0;
}

static void move_slot(orc_sim* s, uint64_t dst, uint64_t src) {
  s->uid[dst] = s->uid[src];
  s->x[dst] = s->x[src]; s->y[dst] = s->y[src]; s->z[dst] = s->z[src]; s->d[dst] = s->d[src];
  s->tx[dst] = s->tx[src]; s->ty[dst] = s->ty[src]; s->tz[dst] = s->tz[src]; s->tg[dst] = s->tg[src];
  s->fx[dst] = s->fx[src]; s->fy[dst] = s->fy[src]; s->fz[dst] = s->fz[src];
  s->partners[dst] = s->partners[src];
  s->flags[dst] = s->flags[src];
  s->beh[dst] = s->beh[src];
  s->vol[dst] = s->vol[src];
  s->tag[dst] = s->tag[src];
  s->rngc[dst] = s->rngc[src];
}

/* Agent::tag / rng_counter in storage order (models.hpp, agent.hpp:35-36, 145) */
int orc_set_tags(orc_sim* s, const uint32_t* tags) {
  for (uint64_t i = 0; i < s->n; ++i) s->tag[i] = tags[i];
  return 0;
}
int orc_tags(const orc_sim* s, uint32_t* out) {
  for (uint64_t i = 0; i < s->n; ++i) out[i] = s->tag[i];
  return 0;
}
int orc_set_rng_counters(orc_sim* s, const uint64_t* c) {
  for (uint64_t i = 0; i < s->n; ++i) s->rngc[i] = c[i];
  return 0;
}
int orc_rng_counters(const orc_sim* s, uint64_t* out) {
  for (uint64_t i = 0; i < s->n; ++i) out[i] = s->rngc[i];
  return 0;
}

/* commit.cpp:14-106 (five steps, slot semantics independent of workers) */
int orc_remove(orc_sim* s, const uint32_t* removed, uint32_t r) {
  if (r == 0) return 0;
  if (r > s->n) return fail("more removals than agents");
  const uint64_t new_size = s->n - r;
  uint32_t* to_right = malloc(r * sizeof *to_right);
  uint32_t* tail = calloc(r, sizeof *tail);
  for (uint32_t k = 0; k < r; ++k) {
    to_right[k] = UINT32_MAX;
    if (removed[k] < new_size) to_right[k] = removed[k];
    else tail[removed[k] - new_size] = 1;
  }
  uint32_t holes = 0, movers = 0;
  for (uint32_t k = 0; k < r; ++k) {
    if (to_right[k] != UINT32_MAX) to_right[holes++] = to_right[k];
    if (tail[k] == 0) tail[movers++] = (uint32_t)(k + new_size);
  }
  if (holes != movers) {
    free(to_right); free(tail);
    return fail("removal bookkeeping out of balance");
  }
  for (uint32_t k = 0; k < holes; ++k) move_slot(s, to_right[k], tail[k]);
  s->n = new_size;
  s->removed += r;
  free(to_right); free(tail);
  return 0;
}

/* commit.cpp:164-225 with one staging slot: removals first (remove_agents_parallel
 * over the slots in staging order), then the additions appended in creation order */
static int run_commit(orc_sim* s) {
  if (s->nrem == 0 && s->nstage == 0) return 0;
  /* simulation.cpp:502-508: new-agent marking sees the pre-commit storage */
  if (s->nstage && s->p.detect_static && mark_new_agent_neighbors(s)) return -1;
  if (s->nrem) {
    const uint64_t r = s->nrem;
    s->nrem = 0;
    if (orc_remove(s, s->rem, (uint32_t)r)) return -1;
  }
  if (s->nstage == 0) return 0;
  reserve(s, s->n + s->nstage);
  for (uint64_t k = 0; k < s->nstage; ++k) {
    init_slot(s, s->n + k, s->s_uid[k], s->s_x[k], s->s_y[k], s->s_z[k], s->s_d[k],
              s->s_beh[k], s->s_vol[k], F_NEWLY_ADDED);
    s->tag[s->n + k] = s->s_tag[k]; /* daughter.set_tag(a.tag()), models.hpp:27 */
  }
  s->n += s->nstage;
  s->added += s->nstage;
  s->nstage = 0;
  return 0;
}

/* ---- morton (morton.cpp:11-186) ---------------------------------------- */
static uint64_t spread3(uint64_t v) {
  uint64_t out = 0;
  for (int i = 0; i < 21; ++i) out |= ((v >> i) & 1ull) << (3 * i);
  return out;
}
static uint64_t compact3(uint64_t v) {
  uint64_t out = 0;
  for (int i = 0; i < 21; ++i) out |= ((v >> (3 * i)) & 1ull) << i;
  return out;
}
int orc_morton_encode3(uint32_t x, uint32_t y, uint32_t z, uint64_t* out) {
  if (x >= (1u << 21) || y >= (1u << 21) || z >= (1u << 21)) return fail("3D coordinates limited to 21 bits");
  *out = spread3(x) | spread3(y) << 1 | spread3(z) << 2;
  return 0;
}
void orc_morton_decode3(uint64_t c, uint32_t* out) {
  out[0] = (uint32_t)compact3(c);
  out[1] = (uint32_t)compact3(c >> 1);
  out[2] = (uint32_t)compact3(c >> 2);
}

typedef struct {
  uint32_t dims[3];
  int d;
  uint64_t counter, offset;
  int found_gap;
  uint64_t* start;
  uint64_t* off;
  uint64_t n, cap;
} tbuild;

static void tvisit(tbuild* b, int level, uint32_t x, uint32_t y, uint32_t z) {
  const uint64_t side = 1ull << level;
  const uint64_t leaves = 1ull << (level * b->d);
  if (x >= b->dims[0] || y >= b->dims[1] || (b->d == 3 && z >= b->dims[2])) {
    b->offset += leaves;
    b->found_gap = 1;
    return;
  }
  if (x + side <= b->dims[0] && y + side <= b->dims[1] && (b->d == 2 || z + side <= b->dims[2])) {
    if (b->found_gap) {
      if (b->n < b->cap) { b->start[b->n] = b->counter; b->off[b->n] = b->offset; }
      b->n++;
      b->found_gap = 0;
    }
    b->counter += leaves;
    return;
  }
  const uint32_t half = (uint32_t)(side / 2);
  for (int c = 0; c < (1 << b->d); ++c)
    tvisit(b, level - 1, x + ((c & 1) ? half : 0), y + ((c & 2) ? half : 0), z + ((c & 4) ? half : 0));
}

/* OffsetsTable::build (morton.cpp:124-143); returns the number of runs */
int64_t orc_offsets_table(const uint32_t* dims, uint64_t* start, uint64_t* off, uint64_t cap) {
  if (!dims[0] || !dims[1] || !dims[2]) return fail("grid dimensions must be positive");
  tbuild b = {{dims[0], dims[1], dims[2]}, dims[2] == 1 ? 2 : 3, 0, 0, 1, start, off, 0, cap};
  uint32_t m = dims[0] > dims[1] ? dims[0] : dims[1];
  if (b.d == 3 && dims[2] > m) m = dims[2];
  int level = 0;
  while ((1ull << level) < m) ++level;
  tvisit(&b, level, 0, 0, 0);
  return (int64_t)b.n;
}

/* prefix_sum.cpp:11-19 */
uint64_t orc_exclusive_scan(uint64_t* v, uint64_t n) {
  uint64_t acc = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t next = acc + v[i];
    v[i] = acc;
    acc = next;
  }
  return acc;
}

/* sort_balance.cpp:22-148 with one domain: boxes in Morton-rank order, chain
 * order inside a box. Requires a current grid. */
int orc_sort(orc_sim* s, uint64_t* moved) {
  if (moved) *moved = 0;
  if (s->indexed != s->n) return fail("sort requires a grid updated for the current agents");
  if (s->n == 0) return 0;
  uint64_t cap = 64;
  uint64_t *st = NULL, *of = NULL;
  int64_t runs;
  for (;;) {
    st = xrealloc(st, cap * sizeof *st);
    of = xrealloc(of, cap * sizeof *of);
    runs = orc_offsets_table(s->dims, st, of, cap);
    if (runs < 0) { free(st); free(of); return -1; }
    if ((uint64_t)runs <= cap) break;
    cap = (uint64_t)runs;
  }
  uint64_t* order = malloc(s->n * sizeof *order);
  uint64_t w = 0, e = 0;
  for (uint64_t rank = 0; rank < s->nboxes; ++rank) {
    while (e + 1 < (uint64_t)runs && st[e + 1] <= rank) ++e;
    uint32_t c[3];
    orc_morton_decode3(rank + of[e], c);
    if (s->dims[2] == 1) { /* 2D table: (x, y) interleave */
      uint64_t code = rank + of[e], xx = 0, yy = 0;
      for (int i = 0; i < 31; ++i) {
        xx |= ((code >> (2 * i)) & 1ull) << i;
        yy |= ((code >> (2 * i + 1)) & 1ull) << i;
      }
      c[0] = (uint32_t)xx; c[1] = (uint32_t)yy; c[2] = 0;
    }
    const uint64_t box = c[0] + (uint64_t)s->dims[0] * (c[1] + (uint64_t)s->dims[1] * c[2]);
    for (uint64_t j = s->head[box]; j != ORC_NIL; j = s->succ[j]) order[w++] = j;
  }
  free(st); free(of);
  if (w != s->n) { free(order); return fail("grid population changed during sort"); }
  orc_sim tmp = *s;
  tmp.cap = 0;
  tmp.uid = NULL; tmp.x = tmp.y = tmp.z = tmp.d = NULL; tmp.tx = tmp.ty = tmp.tz = tmp.tg = NULL;
  tmp.fx = tmp.fy = tmp.fz = NULL; tmp.partners = NULL; tmp.flags = NULL; tmp.beh = NULL;
  tmp.vol = NULL; tmp.succ = NULL; tmp.tag = NULL; tmp.rngc = NULL;
  reserve(&tmp, s->n);
  for (uint64_t i = 0; i < s->n; ++i) {
    const uint64_t j = order[i];
    tmp.uid[i] = s->uid[j];
    tmp.x[i] = s->x[j]; tmp.y[i] = s->y[j]; tmp.z[i] = s->z[j]; tmp.d[i] = s->d[j];
    tmp.tx[i] = s->tx[j]; tmp.ty[i] = s->ty[j]; tmp.tz[i] = s->tz[j]; tmp.tg[i] = s->tg[j];
    tmp.fx[i] = s->fx[j]; tmp.fy[i] = s->fy[j]; tmp.fz[i] = s->fz[j];
    tmp.partners[i] = s->partners[j]; tmp.flags[i] = s->flags[j]; tmp.beh[i] = s->beh[j];
    tmp.vol[i] = s->vol[j];
    tmp.tag[i] = s->tag[j];
    tmp.rngc[i] = s->rngc[j];
  }
  free(order);
#define SWAPF(f) do { void* t_ = s->f; s->f = tmp.f; tmp.f = t_; } while (0)
  SWAPF(uid); SWAPF(x); SWAPF(y); SWAPF(z); SWAPF(d); SWAPF(tx); SWAPF(ty); SWAPF(tz);
  SWAPF(tg); SWAPF(fx); SWAPF(fy); SWAPF(fz); SWAPF(partners); SWAPF(flags); SWAPF(beh);
  SWAPF(vol); SWAPF(succ); SWAPF(tag); SWAPF(rngc);
#undef SWAPF
  const uint64_t c2 = s->cap;
  s->cap = tmp.cap;
  tmp.cap = c2;
  free(tmp.uid); free(tmp.x); free(tmp.y); free(tmp.z); free(tmp.d); free(tmp.tx); free(tmp.ty);
  free(tmp.tz); free(tmp.tg); free(tmp.fx); free(tmp.fy); free(tmp.fz); free(tmp.partners);
  free(tmp.flags); free(tmp.beh); free(tmp.vol); free(tmp.succ); free(tmp.tag); free(tmp.rngc);
  s->sorted += 0; /* one domain: nothing migrates (agents_moved counts domain changes) */
  return 0;
}

/* ---- config 5: SIR on a periodic cube (absim_models.h) -------------------
 * States live in beh (0 S, 1 I, 2 R), infection iteration in partners.
 * All decisions read start-of-iteration states and positions. */
static uint64_t sir_counts[3];
int orc_sir_counts(const orc_sim* s, uint64_t* out) {
  (void)s;
  out[0] = sir_counts[0]; out[1] = sir_counts[1]; out[2] = sir_counts[2];
  return 0;
}

static int sir_step(orc_sim* s) {
  const double L = s->p.mp[0], r = s->p.mp[1], step = s->p.mp[2], prob = s->p.mp[4];
  const uint64_t rec = (uint64_t)s->p.mp[3];
  uint32_t dims = (uint32_t)floor(L / r);
  if (dims < 3) dims = 3;
  const double box = L / (double)dims;
  const uint64_t nb = (uint64_t)dims * dims * dims;
  if (nb > s->box_cap) {
    s->head = xrealloc(s->head, nb * sizeof *s->head);
    s->count = xrealloc(s->count, nb * sizeof *s->count);
    s->box_cap = nb;
  }
  for (uint64_t b = 0; b < nb; ++b) s->head[b] = ORC_NIL;
  uint32_t* cb = malloc(3 * s->n * sizeof *cb + 1);
  for (uint64_t i = 0; i < s->n; ++i) {
    const double p[3] = {s->x[i], s->y[i], s->z[i]};
    for (int k = 0; k < 3; ++k) {
      int64_t c = (int64_t)floor(p[k] / box);
      if (c < 0) c = 0;
      if (c > (int64_t)dims - 1) c = dims - 1;
      cb[3 * i + k] = (uint32_t)c;
    }
    const uint64_t b = cb[3 * i] + (uint64_t)dims * (cb[3 * i + 1] + (uint64_t)dims * cb[3 * i + 2]);
    s->succ[i] = s->head[b];
    s->head[b] = i;
  }
  uint8_t* ns = malloc(s->n + 1);
  uint32_t* nt = malloc((s->n + 1) * sizeof *nt);
  const double r2 = r * r;
  for (uint64_t i = 0; i < s->n; ++i) {
    uint8_t st = s->beh[i];
    uint32_t ti = s->partners[i];
    if (st == ABS_SIR_I && s->iteration - ti >= rec) st = ABS_SIR_R;
    if (st == ABS_SIR_S) {
      unsigned int k = 0;
      for (int dz = -1; dz <= 1; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
          for (int dx = -1; dx <= 1; ++dx) {
            const uint64_t bx = (cb[3 * i] + dims + dx) % dims, by = (cb[3 * i + 1] + dims + dy) % dims,
                           bz = (cb[3 * i + 2] + dims + dz) % dims;
            for (uint64_t j = s->head[bx + dims * (by + (uint64_t)dims * bz)]; j != ORC_NIL; j = s->succ[j]) {
              if (j == i || s->beh[j] != ABS_SIR_I) continue;
              const double ddx = abs_min_image(s->x[i] - s->x[j], L);
              const double ddy = abs_min_image(s->y[i] - s->y[j], L);
              const double ddz = abs_min_image(s->z[i] - s->z[j], L);
              if ((ddx * ddx + ddy * ddy) + ddz * ddz <= r2) ++k;
            }
          }
      if (k > 0 && abs_rng_word(s->p.seed, s->uid[i], ABS_RNG_SIR_INFECT(s->iteration)) < abs_sir_threshold(prob, k)) {
        st = ABS_SIR_I;
        ti = (uint32_t)s->iteration;
      }
    }
    ns[i] = st;
    nt[i] = ti;
  }
  sir_counts[0] = sir_counts[1] = sir_counts[2] = 0;
  for (uint64_t i = 0; i < s->n; ++i) {
    double dir[3];
    abs_unit_vector(s->p.seed, s->uid[i], ABS_RNG_SIR_WALK(s->iteration), dir);
    s->x[i] = abs_wrap(s->x[i] + dir[0] * step, L);
    s->y[i] = abs_wrap(s->y[i] + dir[1] * step, L);
    s->z[i] = abs_wrap(s->z[i] + dir[2] * step, L);
    s->beh[i] = ns[i];
    s->partners[i] = nt[i];
    sir_counts[ns[i]]++;
  }
  free(cb); free(ns); free(nt);
  return 0;
}

/* ---- schedule (simulation.cpp:222-322) --------------------------------- */
int orc_simulate(orc_sim* s, uint64_t iterations) {
  if (s->p.model == 4) {
    for (uint64_t it = 0; it < iterations; ++it) {
      if (sir_step(s)) return -1;
      s->iteration++;
    }
    return 0;
  }
  for (uint64_t it = 0; it < iterations; ++it) {
    if (orc_env_update(s, NULL, NULL, NULL)) return -1;
    if (s->p.sorting_frequency > 0 && s->iteration % s->p.sorting_frequency == 0) {
      if (orc_sort(s, NULL)) return -1;
      if (orc_env_update(s, NULL, NULL, NULL)) return -1;
    }
    if (s->p.detect_static && run_staticness(s)) return -1;
    /* agent phase: behaviours then forces per agent block; neither reads
     * state the other writes, so whole-population order is equivalent */
    const uint64_t n = s->n;
    for (uint64_t i = 0; i < n; ++i)
      if (run_behaviour(s, i)) return -1;
    for (uint64_t i = 0; i < n; ++i)
      if (run_forces(s, i)) return -1;
    for (uint64_t i = 0; i < n; ++i) apply_pending(s, i);
    if (run_commit(s)) return -1;
    s->iteration++;
  }
  return 0;
}

int orc_counts(const orc_sim* s, uint64_t* out) {
  out[0] = s->n; out[1] = s->uid_counter; out[2] = s->iteration; out[3] = s->evals;
  out[4] = s->skips; out[5] = s->added; out[6] = s->removed; out[7] = s->sorted;
  return 0;
}

int orc_dump_beh(const orc_sim* s, uint8_t* beh, uint32_t* partners) {
  for (uint64_t i = 0; i < s->n; ++i) {
    beh[i] = s->beh[i];
    partners[i] = s->partners[i];
  }
  return 0;
}

/* same layout as ref_dump (oracle/ref_harness.cpp) */
int orc_dump(const orc_sim* s, uint64_t* uid, double* x, double* y, double* z, double* d,
             double* fx, double* fy, double* fz, uint32_t* partners, uint8_t* flags, double* vol) {
  for (uint64_t i = 0; i < s->n; ++i) {
    if (uid) uid[i] = s->uid[i];
    if (x) x[i] = s->x[i];
    if (y) y[i] = s->y[i];
    if (z) z[i] = s->z[i];
    if (d) d[i] = s->d[i];
    if (fx) fx[i] = s->fx[i];
    if (fy) fy[i] = s->fy[i];
    if (fz) fz[i] = s->fz[i];
    if (partners) partners[i] = s->partners[i];
    if (flags) flags[i] = (uint8_t)(s->flags[i] & (63u | F_GHOST));
    if (vol) vol[i] = s->vol[i];
  }
  return 0;
}
