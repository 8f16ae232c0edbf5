// ref_harness.cpp — TEST INFRASTRUCTURE ONLY (oracle side; never shipped).
//
// A thin extern "C" shim over the UNMODIFIED reference engine (absim, built
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/). It lets
// tests, golden-fixture scripts and bench.py's reference arm drive the
// reference through its own public API:
//   Simulation::add_agent / add_agent_operation / simulate  (simulation.hpp:89-123)
//   Behavior subclasses (behavior.hpp:14-38) for the BASELINE config models
//   Environment::update / for_each_neighbor (environment.hpp:36-51)
//   UniformGrid::box_index_of (uniform_grid.hpp:52)
//   sort_and_balance (sort_balance.hpp:30-31)
// The config behaviours use include/absim_models.h so their stochastic
// decisions are bit-identical to the GPU kernels'.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "absim/models.hpp"
#include "absim/simulation.hpp"
#include "absim/sort_balance.hpp"
#include "absim/uniform_grid.hpp"
#include "absim_models.h"

using namespace absim;

namespace {

thread_local std::string g_error;

struct RefParams {
  std::uint64_t seed;
  std::int32_t threads;
  std::int32_t domains;
  double dt, k, max_disp, threshold, fixed_box;
  std::uint64_t sorting_frequency;
  std::int32_t detect_static;
  std::int32_t model;  // 0 none, 1 volume grow/divide (c2), 2 drive (c3), 3 grow (ref Grow)
  double mp[8];
  std::int32_t env;  // EnvironmentKind: 0 uniform grid, 1 brute force, 2 kd-tree
  std::int32_t pad;
};

// BASELINE configs[1]: volume growth + division (see absim_models.h).
class VolumeGrowDivide final : public BehaviorBase<VolumeGrowDivide> {
 public:
  VolumeGrowDivide(double volume, double rate, double v_divide)
      : volume_(volume), rate_(rate), v_divide_(v_divide) {}
  void run(Agent& a, AgentContext& ctx) override {
    volume_ += rate_;
    if (volume_ > v_divide_) {
      volume_ *= 0.5;
      double dir[3];
      abs_unit_vector(ctx.params().seed, a.uid(), ABS_RNG_DIVISION_BASE(ctx.iteration()), dir);
      const double half = 0.5 * a.diameter();
      const Vec3 p{a.position().x + dir[0] * half, a.position().y + dir[1] * half,
                   a.position().z + dir[2] * half};
      Agent& daughter = ctx.add_daughter(p, abs_diameter_of_volume(volume_));
      for (Behavior* b : daughter.behaviors()) {
        if (auto* g = dynamic_cast<VolumeGrowDivide*>(b)) g->volume_ = volume_;
      }
    }
    a.grow(abs_diameter_of_volume(volume_) - a.diameter());
  }
  double volume() const { return volume_; }

 private:
  double volume_, rate_, v_divide_;
};

// BASELINE configs[2]: outward drive of the outer shells.
class Drive final : public BehaviorBase<Drive> {
 public:
  Drive(double cx, double cy, double cz, double vmax) : c_{cx, cy, cz}, vmax_(vmax) {}
  void run(Agent& a, AgentContext& ctx) override {
    double d[3];
    abs_drive_delta(a.position().x, a.position().y, a.position().z, c_[0], c_[1], c_[2],
                    vmax_, ctx.params().seed, a.uid(), ctx.iteration(), d);
    a.translate({d[0], d[1], d[2]});
  }

 private:
  double c_[3];
  double vmax_;
};

// ABS_MODEL_GROW_DIVIDE_DIE (absim_gpu.h): the reference's own
// models::GrowDivide, preceded by a removal draw that calls
// AgentContext::remove_self (simulation.cpp:64-66).
class GrowDivideDie final : public BehaviorBase<GrowDivideDie> {
 public:
  GrowDivideDie(double rate, double threshold, double initial, double p_remove)
      : inner_(rate, threshold, initial), p_remove_(p_remove) {}
  void run(Agent& a, AgentContext& ctx) override {
    if (abs_u01(abs_rng_word(ctx.params().seed, a.uid(), ABS_RNG_DEATH(ctx.iteration()))) < p_remove_) {
      ctx.remove_self();
      return;
    }
    inner_.run(a, ctx);
  }

 private:
  models::GrowDivide inner_;
  double p_remove_;
};

struct Ref {
  std::unique_ptr<Simulation> sim;
  RefParams p;
};

SimulationParams to_params(const RefParams& r) {
  SimulationParams p;
  p.seed = r.seed;
  p.thread_count = r.threads;
  p.domain_count = r.domains;
  p.simulation_time_step = r.dt;
  p.repulsion_coefficient = r.k;
  p.max_displacement = r.max_disp;
  p.force_threshold = r.threshold;
  p.fixed_box_length = r.fixed_box;
  p.sorting_frequency = r.sorting_frequency;
  p.detect_static_agents = r.detect_static != 0;
  p.environment_kind = r.env == 1 ? EnvironmentKind::kBruteForce
                                  : (r.env == 2 ? EnvironmentKind::kKdTree : EnvironmentKind::kUniformGrid);
  return p;
}

std::vector<Agent*> storage_order(ResourceManager& rm) {
  std::vector<Agent*> out;
  rm.for_each_agent([&](Agent& a, AgentHandle) { out.push_back(&a); });
  return out;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_error = e.what();
  } catch (...) {
    g_error = "unknown error";
  }
  return -1;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_error.c_str(); }

// Agents get uids 0..n-1 in array order; storage order = array order for
// one domain (simulation.cpp:131-141).
void* ref_create(const RefParams* rp, std::uint64_t n, const double* x, const double* y,
                 const double* z, const double* d, const std::uint8_t* behaviour_mask) {
  Ref* r = nullptr;
  const int rc = guarded([&] {
    auto h = std::make_unique<Ref>();
    h->p = *rp;
    h->sim = std::make_unique<Simulation>(to_params(*rp));
    ResourceManager& rm = h->sim->resource_manager();
    for (std::uint64_t i = 0; i < n; ++i) {
      Agent& a = h->sim->add_agent({x[i], y[i], z[i]}, d[i]);
      const int dom = static_cast<int>(rm.handle_of_uid(a.uid()).domain);
      const bool on = behaviour_mask == nullptr || behaviour_mask[i] != 0;
      if (!on) continue;
      if (rp->model == 1) {
        VolumeGrowDivide proto(abs_volume_of_diameter(d[i]), rp->mp[0], rp->mp[1]);
        a.add_behavior(rm.clone_behavior(proto, dom));
      } else if (rp->model == 2) {
        Drive proto(rp->mp[0], rp->mp[1], rp->mp[2], rp->mp[3]);
        a.add_behavior(rm.clone_behavior(proto, dom));
      } else if (rp->model == 3) {
        models::Grow proto(rp->mp[0], rp->mp[1]);
        a.add_behavior(rm.clone_behavior(proto, dom));
      } else if (rp->model == 5) {  // the reference's own models (models.hpp:15-64)
        models::GrowDivide proto(rp->mp[0], rp->mp[1], rp->mp[2]);
        a.add_behavior(rm.clone_behavior(proto, dom));
      } else if (rp->model == 6) {
        models::Cohere proto(rp->mp[0], rp->mp[1]);
        a.add_behavior(rm.clone_behavior(proto, dom));
      } else if (rp->model == 7) {
        GrowDivideDie proto(rp->mp[0], rp->mp[1], rp->mp[2], rp->mp[3]);
        a.add_behavior(rm.clone_behavior(proto, dom));
      }
    }
    r = h.release();
  });
  return rc == 0 ? r : nullptr;
}

// The reference's own population builders (models.cpp), for known answers.
void* ref_create_builtin(const RefParams* rp, const char* name, std::uint64_t n) {
  Ref* r = nullptr;
  const int rc = guarded([&] {
    auto h = std::make_unique<Ref>();
    h->p = *rp;
    SimulationParams p = to_params(*rp);
    const std::string which(name);
    if (which == "clustering") models::tune_clustering_params(p);
    h->sim = std::make_unique<Simulation>(p);
    if (which == "static_front") {
      models::build_static_front(*h->sim, n);
    } else if (which == "static_front_nogrowth") {
      models::StaticFrontConfig cfg;
      cfg.growth = false;
      models::build_static_front(*h->sim, n, cfg);
    } else if (which == "clustering") {
      models::build_clustering(*h->sim, n);
    } else if (which == "proliferation") {
      models::build_proliferation(*h->sim, n);
    } else {
      throw std::invalid_argument("unknown builtin population: " + which);
    }
    r = h.release();
  });
  return rc == 0 ? r : nullptr;
}

void ref_destroy(void* h) { delete static_cast<Ref*>(h); }

int ref_simulate(void* h, std::uint64_t iterations) {
  return guarded([&] { static_cast<Ref*>(h)->sim->simulate(iterations); });
}

// out[0..7] = agents, uid_count, iterations, force_evaluations, force_skips,
// agents_added, agents_removed, agents_sorted; wall = report.total_wall_ms.
int ref_counts(void* h, std::uint64_t* out, double* wall_ms) {
  return guarded([&] {
    Simulation& s = *static_cast<Ref*>(h)->sim;
    const SimulationReport& r = s.report();
    out[0] = s.resource_manager().total_agents();
    out[1] = s.resource_manager().uid_count();
    out[2] = s.iteration();
    out[3] = r.force_evaluations;
    out[4] = r.force_skips;
    out[5] = r.agents_added;
    out[6] = r.agents_removed;
    out[7] = r.agents_sorted;
    if (wall_ms) *wall_ms = r.total_wall_ms;
  });
}

// Storage order (domain-major). flags: bit0 static, 1 moved, 2 grew,
// 3 newly_added, 4 neighbor_violation, 5 new_neighbor. Any pointer may be null.
int ref_dump(void* h, std::uint64_t* uid, double* x, double* y, double* z, double* d,
             double* fx, double* fy, double* fz, std::uint32_t* partners,
             std::uint8_t* flags, double* volume) {
  return guarded([&] {
    Simulation& s = *static_cast<Ref*>(h)->sim;
    const auto agents = storage_order(s.resource_manager());
    for (std::size_t i = 0; i < agents.size(); ++i) {
      const Agent& a = *agents[i];
      if (uid) uid[i] = a.uid();
      if (x) x[i] = a.position().x;
      if (y) y[i] = a.position().y;
      if (z) z[i] = a.position().z;
      if (d) d[i] = a.diameter();
      if (fx) fx[i] = a.last_force().x;
      if (fy) fy[i] = a.last_force().y;
      if (fz) fz[i] = a.last_force().z;
      if (partners) partners[i] = a.nonzero_force_partners();
      if (flags) {
        flags[i] = (a.is_static() ? 1 : 0) | (a.moved_this_iteration() ? 2 : 0) |
                   (a.grew_this_iteration() ? 4 : 0) | (a.newly_added() ? 8 : 0) |
                   (a.neighbor_violation() ? 16 : 0) | (a.new_neighbor() ? 32 : 0);
      }
      if (volume) {
        volume[i] = 0.0;
        for (Behavior* b : a.behaviors()) {
          if (auto* g = dynamic_cast<VolumeGrowDivide*>(b)) volume[i] = g->volume();
        }
      }
    }
  });
}

// Agent::tag and rng_counter in storage order (agent.hpp:35-36, 145).
int ref_set_tags(void* h, const std::uint32_t* tags) {
  return guarded([&] {
    const auto agents = storage_order(static_cast<Ref*>(h)->sim->resource_manager());
    for (std::size_t i = 0; i < agents.size(); ++i) agents[i]->set_tag(tags[i]);
  });
}

int ref_tags(void* h, std::uint32_t* out) {
  return guarded([&] {
    const auto agents = storage_order(static_cast<Ref*>(h)->sim->resource_manager());
    for (std::size_t i = 0; i < agents.size(); ++i) out[i] = agents[i]->tag();
  });
}

int ref_rng_counters(void* h, std::uint64_t* out) {
  return guarded([&] {
    const auto agents = storage_order(static_cast<Ref*>(h)->sim->resource_manager());
    for (std::size_t i = 0; i < agents.size(); ++i) out[i] = *agents[i]->rng_counter();
  });
}

// Environment::update on the current state; grid = origin[3], box, dmax.
int ref_env_update(void* h, double* grid, std::uint32_t* dims, std::uint64_t* indexed) {
  return guarded([&] {
    Simulation& s = *static_cast<Ref*>(h)->sim;
    s.environment().update();
    auto* gp = dynamic_cast<UniformGrid*>(&s.environment());
    if (!gp) {  // brute-force / kd-tree: no grid tuple, only the largest diameter
      grid[0] = grid[1] = grid[2] = grid[3] = 0.0;
      grid[4] = s.environment().largest_agent_diameter();
      dims[0] = dims[1] = dims[2] = 0;
      if (indexed) *indexed = 0;
      return;
    }
    auto& g = *gp;
    grid[0] = g.origin().x;
    grid[1] = g.origin().y;
    grid[2] = g.origin().z;
    grid[3] = g.box_length();
    grid[4] = g.largest_agent_diameter();
    dims[0] = g.dims()[0];
    dims[1] = g.dims()[1];
    dims[2] = g.dims()[2];
    if (indexed) *indexed = g.total_agents_indexed();
  });
}

// UniformGrid::box_index_of per agent (storage order); call after ref_env_update.
int ref_cell_ids(void* h, std::uint64_t* out) {
  return guarded([&] {
    Simulation& s = *static_cast<Ref*>(h)->sim;
    auto& g = dynamic_cast<UniformGrid&>(s.environment());
    const auto agents = storage_order(s.resource_manager());
    for (std::size_t i = 0; i < agents.size(); ++i) out[i] = g.box_index_of(agents[i]->position());
  });
}

// Force-query neighbour sets (simulation.cpp:469): for each agent in storage
// order the sorted uids within r = 0.5 (d + dmax) through for_each_neighbor.
// offsets has n+1 entries; returns the total (or -1; -2 if cap too small).
std::int64_t ref_neighbors(void* h, std::uint64_t* offsets, std::uint64_t* uids,
                           std::uint64_t cap) {
  std::int64_t total = -1;
  const int rc = guarded([&] {
    Simulation& s = *static_cast<Ref*>(h)->sim;
    Environment& env = s.environment();
    ResourceManager& rm = s.resource_manager();
    const double dmax = env.largest_agent_diameter();
    std::uint64_t pos = 0;
    std::uint64_t i = 0;
    std::vector<AgentUid> tmp;
    rm.for_each_agent([&](Agent& a, AgentHandle hd) {
      tmp.clear();
      LambdaVisitor v([&](Agent& b, double) { tmp.push_back(b.uid()); });
      const double r = 0.5 * (a.diameter() + dmax);
      env.for_each_neighbor(hd, a.position(), r * r, v);
      std::sort(tmp.begin(), tmp.end());
      offsets[i++] = pos;
      for (AgentUid u : tmp) {
        if (pos < cap) uids[pos] = u;
        ++pos;
      }
    });
    offsets[i] = pos;
    total = pos > cap ? -2 : static_cast<std::int64_t>(pos);
  });
  return rc == 0 ? total : -1;
}

// Force-query neighbour COUNTS per agent (storage order), i.e. the force
// evaluations run_forces performs for a non-static agent (simulation.cpp:469-
// 475), for populations too large for ref_neighbors' uid lists. Queries run
// concurrently on `threads` std::threads, as the reference's own workers do
// (for_each_neighbor is read-only between updates).
int ref_neighbor_counts(void* h, std::uint32_t* counts, int threads) {
  return guarded([&] {
    Simulation& s = *static_cast<Ref*>(h)->sim;
    Environment& env = s.environment();
    const double dmax = env.largest_agent_diameter();
    std::vector<std::pair<Agent*, AgentHandle>> all;
    s.resource_manager().for_each_agent([&](Agent& a, AgentHandle hd) { all.push_back({&a, hd}); });
    const std::size_t n = all.size();
    const int T = std::max(1, threads);
    std::vector<std::thread> pool;
    for (int t = 0; t < T; ++t) {
      pool.emplace_back([&, t] {
        for (std::size_t i = t; i < n; i += T) {
          std::uint32_t c = 0;
          LambdaVisitor v([&](Agent&, double) { ++c; });
          const double r = 0.5 * (all[i].first->diameter() + dmax);
          env.for_each_neighbor(all[i].second, all[i].first->position(), r * r, v);
          counts[i] = c;
        }
      });
    }
    for (auto& th : pool) th.join();
  });
}

// env update + sort_and_balance (sort_balance.cpp:22-148) on the current state.
int ref_sort(void* h, std::uint64_t* moved) {
  return guarded([&] {
    Simulation& s = *static_cast<Ref*>(h)->sim;
    s.environment().update();
    auto& g = dynamic_cast<UniformGrid&>(s.environment());
    const SortOutcome o = sort_and_balance(s.resource_manager(), g, s.worker_pool(), true);
    if (moved) *moved = o.agents_moved;
  });
}

// ---- config 5 (SIR on a periodic cube) through the reference engine -------
// The reference has no periodic boundaries, so the periodic
// cube is realised with ghost images: before every iteration each agent
// within r (+ margin) of a face gets translated copies (x +- L per axis, up
// to 7 per corner agent) as extra agents of the reference Simulation. The
// reference's own grid and AgentContext::for_each_neighbor (inclusive
// d2 <= r^2, simulation.hpp:41-44) then find every neighbour the
// minimum-image convention of absim_models.h finds (L > 4 r: one image of a
// pair at most is within r). Everything else runs through public hooks:
//   agent op "sir"    (add_agent_operation, simulation.hpp:111): real agents
//                     update their state from the START-of-iteration states
//                     (double-buffered in the harness, keyed by uid) and
//                     translate by the random-walk step; ghosts remove_self
//   repulsion k = 0   the engine's forces op still runs, contributing nothing
//   post ops          (add_standalone_operation, Phase::kPost, after the
//                     commit removed the old ghosts): wrap positions into
//                     [0, L) with Agent::set_position, publish the new
//                     states, count S/I/R, add the next iteration's ghosts.
// Decisions and draws use absim_models.h (the shared definitions), so the
// result is comparable bit for bit with the C port and the kernels; the only
// arithmetic difference is the ghost position x + L (computed here) against
// the port's wrapped difference (x_i - x_j) - L, which can move d2 by an ulp
// (a decision flips only if d2 is within ~1e-15 of r^2).
struct RefSir {
  std::unique_ptr<Simulation> sim;
  double L, r, step, prob;
  std::uint64_t rec;
  std::uint64_t seed;
  std::uint64_t n_real;
  std::vector<std::int64_t> ghost_of;  // by uid: real uid of a ghost, -1 for a real agent
  std::vector<std::uint8_t> st_old, st_new;
  std::vector<std::uint32_t> t_old, t_new;
  std::vector<std::uint64_t> counts;  // 3 per completed iteration

  void ensure(std::uint64_t uid) {
    if (uid >= ghost_of.size()) {
      const std::size_t m = std::max<std::size_t>(uid + 1, ghost_of.size() * 2);
      ghost_of.resize(m, -1);
      st_old.resize(m, 0);
      st_new.resize(m, 0);
      t_old.resize(m, 0);
      t_new.resize(m, 0);
    }
  }

  void add_ghosts() {
    std::vector<std::pair<Vec3, std::uint64_t>> img;
    const double m = r * 1.01 + 1e-9;  // superset: a spare image is never within r
    sim->resource_manager().for_each_agent([&](Agent& a, AgentHandle) {
      if (ghost_of[a.uid()] >= 0) return;
      const double p[3] = {a.position().x, a.position().y, a.position().z};
      int lo[3], hi[3];
      for (int k = 0; k < 3; ++k) {
        lo[k] = p[k] >= L - m ? -1 : 0;
        hi[k] = p[k] < m ? 1 : 0;
      }
      for (int ox = lo[0]; ox <= hi[0]; ++ox)
        for (int oy = lo[1]; oy <= hi[1]; ++oy)
          for (int oz = lo[2]; oz <= hi[2]; ++oz) {
            if (!ox && !oy && !oz) continue;
            const Vec3 q{ox ? p[0] + ox * L : p[0], oy ? p[1] + oy * L : p[1], oz ? p[2] + oz * L : p[2]};
            img.push_back({q, a.uid()});
          }
    });
    for (auto& [q, real] : img) {
      Agent& g = sim->add_agent(q, 1.0);
      ensure(g.uid());
      ghost_of[g.uid()] = static_cast<std::int64_t>(real);
    }
  }
};

void* ref_sir_create(const RefParams* rp, std::uint64_t n, const double* x, const double* y, const double* z) {
  RefSir* r = nullptr;
  const int rc = guarded([&] {
    auto h = std::make_unique<RefSir>();
    h->L = rp->mp[0];
    h->r = rp->mp[1];
    h->step = rp->mp[2];
    h->rec = static_cast<std::uint64_t>(rp->mp[3]);
    h->prob = rp->mp[4];
    h->seed = rp->seed;
    h->n_real = n;
    if (!(h->L > 4.0 * h->r)) throw std::invalid_argument("ghost images need L > 4 r");
    RefParams q = *rp;
    q.k = 0.0;           // no mechanics: the forces op contributes nothing
    q.fixed_box = h->r;  // boxes of the infection radius (point agents, d = 1 <= r)
    q.sorting_frequency = 0;
    q.detect_static = 0;
    h->sim = std::make_unique<Simulation>(to_params(q));
    h->ensure(n);
    for (std::uint64_t i = 0; i < n; ++i) {
      Agent& a = h->sim->add_agent({x[i], y[i], z[i]}, 1.0);
      const std::uint64_t u = a.uid();
      h->ensure(u);
      h->st_old[u] = abs_u01(abs_rng_word(rp->seed, u, ABS_RNG_SIR_INIT)) < 0.01 ? ABS_SIR_I : ABS_SIR_S;
      h->t_old[u] = 0;
    }
    RefSir* self = h.get();
    self->add_ghosts();
    self->sim->add_agent_operation("sir", 1, [self](Agent& a, AgentContext& ctx) {
      const std::uint64_t u = a.uid();
      if (self->ghost_of[u] >= 0) {  // an image of the previous iteration
        ctx.remove_self();
        return;
      }
      std::uint8_t st = self->st_old[u];
      std::uint32_t ti = self->t_old[u];
      const std::uint64_t it = ctx.iteration();
      if (st == ABS_SIR_I && it - ti >= self->rec) st = ABS_SIR_R;
      if (st == ABS_SIR_S) {
        unsigned int k = 0;
        ctx.for_each_neighbor(self->r, [&](Agent& b, double) {
          const std::int64_t g = self->ghost_of[b.uid()];
          const std::uint64_t real = g >= 0 ? static_cast<std::uint64_t>(g) : b.uid();
          if (self->st_old[real] == ABS_SIR_I) ++k;
        });
        if (k > 0 && abs_rng_word(self->seed, u, ABS_RNG_SIR_INFECT(it)) < abs_sir_threshold(self->prob, k)) {
          st = ABS_SIR_I;
          ti = static_cast<std::uint32_t>(it);
        }
      }
      self->st_new[u] = st;
      self->t_new[u] = ti;
      double dir[3];
      abs_unit_vector(self->seed, u, ABS_RNG_SIR_WALK(it), dir);
      a.translate({dir[0] * self->step, dir[1] * self->step, dir[2] * self->step});
    });
    self->sim->add_standalone_operation("sir_publish", Phase::kPost, 1, [self](Simulation& s) {
      std::uint64_t c[3] = {0, 0, 0};
      s.resource_manager().for_each_agent([&](Agent& a, AgentHandle) {
        const std::uint64_t u = a.uid();
        if (self->ghost_of[u] >= 0) return;
        const Vec3& p = a.position();
        a.set_position({abs_wrap(p.x, self->L), abs_wrap(p.y, self->L), abs_wrap(p.z, self->L)});
        self->st_old[u] = self->st_new[u];
        self->t_old[u] = self->t_new[u];
        ++c[self->st_old[u]];
      });
      self->counts.insert(self->counts.end(), c, c + 3);
      self->add_ghosts();
    });
    r = h.release();
  });
  return rc == 0 ? r : nullptr;
}

void ref_sir_destroy(void* h) { delete static_cast<RefSir*>(h); }

int ref_sir_simulate(void* h, std::uint64_t iterations) {
  return guarded([&] { static_cast<RefSir*>(h)->sim->simulate(iterations); });
}

// S/I/R counts after each completed iteration: out[3 * t + s], t < cap.
std::int64_t ref_sir_counts(void* h, std::uint64_t* out, std::uint64_t cap) {
  const RefSir& r = *static_cast<RefSir*>(h);
  const std::uint64_t its = r.counts.size() / 3;
  for (std::uint64_t t = 0; t < its && t < cap; ++t)
    for (int k = 0; k < 3; ++k) out[3 * t + k] = r.counts[3 * t + k];
  return static_cast<std::int64_t>(its);
}

// Real agents (ghosts excluded) in storage order: uid, position, state, infection iteration.
int ref_sir_dump(void* h, std::uint64_t* uid, double* x, double* y, double* z, std::uint8_t* state,
                 std::uint32_t* t_inf) {
  return guarded([&] {
    RefSir& r = *static_cast<RefSir*>(h);
    std::uint64_t i = 0;
    r.sim->resource_manager().for_each_agent([&](Agent& a, AgentHandle) {
      const std::uint64_t u = a.uid();
      if (r.ghost_of[u] >= 0) return;
      uid[i] = u;
      x[i] = a.position().x;
      y[i] = a.position().y;
      z[i] = a.position().z;
      state[i] = r.st_old[u];
      t_inf[i] = r.t_old[u];
      ++i;
    });
  });
}

std::uint64_t ref_sir_agents(void* h) { return static_cast<RefSir*>(h)->n_real; }

}  // extern "C"
