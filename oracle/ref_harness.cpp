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

}  // extern "C"
