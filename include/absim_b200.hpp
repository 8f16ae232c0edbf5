// absim_b200.hpp — C++17 host API over the C ABI (absim_gpu.h).
//
// Keeps the reference's call shapes for the hot path so a reference user can
// switch with minimal edits:
//   absim::SimulationParams      -> absim_b200::SimulationParams  (params.hpp:17-52)
//   absim::Simulation            -> absim_b200::Simulation        (simulation.hpp:89-123)
//     add_agent(pos, d) / simulate(n) / report() / environment() / iteration()
//   absim::Environment / UniformGrid -> absim_b200::UniformGrid    (environment.hpp:36-51,
//     update(), largest_agent_diameter(), max_query_radius(), name(),   uniform_grid.hpp:26-94)
//     box_length(), origin(), dims(), box_index_of (batched: cell_ids()),
//     for_each_neighbor (batched: for_each_neighbor_pair / neighbor_lists())
//   absim::SimulationReport      -> absim_b200::SimulationReport  (report.hpp:18-41)
// Errors surface as the reference's exception types: std::invalid_argument
// for bad arguments (params.cpp:44-72), absim_b200::Error (a
// std::runtime_error) otherwise, with the reference's "operation '...' failed
// at iteration N" wording for step failures (simulation.cpp:194-205).
// Everything runs in the sm_100a kernels behind libabsim_gpu.so.
#pragma once

#include <array>
#include <limits>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "absim_gpu.h"

namespace absim_b200 {

struct Vec3 {
  double x = 0.0, y = 0.0, z = 0.0;
};

class Error : public std::runtime_error {
 public:
  Error(int code, const std::string& what) : std::runtime_error(what), code_(code) {}
  int code() const { return code_; }

 private:
  int code_;
};

inline void check(int rc, const abs_gpu_ctx* ctx) {
  if (rc == ABS_OK) return;
  const std::string msg = abs_gpu_last_error(ctx);
  if (rc == ABS_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  throw Error(rc, msg);
}

struct SimulationParams {
  std::uint64_t seed = 42;
  double simulation_time_step = 0.1;
  double repulsion_coefficient = 2.0;
  double max_displacement = 3.0;
  double force_threshold = 0.0;
  double fixed_box_length = 0.0;
  std::uint64_t sorting_frequency = 0;
  bool detect_static_agents = false;
  // device behaviour model (ABS_MODEL_*) with its parameters
  int model = ABS_MODEL_NONE;
  std::array<double, 8> model_params{};
  bool record_forces = true;
  // EnvironmentKind (params.hpp:9): ABS_ENV_UNIFORM_GRID, ABS_ENV_BRUTE_FORCE or ABS_ENV_KD_TREE
  int environment_kind = ABS_ENV_UNIFORM_GRID;

  // SimulationParams::validate (params.cpp:44-72), hot-path fields
  void validate() const {
    auto fail = [](const char* what) { throw std::invalid_argument(what); };
    if (fixed_box_length < 0.0) fail("fixed_box_length must be >= 0");
    if (sorting_frequency > 0 && environment_kind != ABS_ENV_UNIFORM_GRID)
      fail("sorting requires the uniform_grid environment");
    if (!(simulation_time_step > 0.0)) fail("simulation_time_step must be > 0");
    if (repulsion_coefficient < 0.0) fail("repulsion_coefficient must be >= 0");
    if (!(max_displacement > 0.0)) fail("max_displacement must be > 0");
    if (force_threshold < 0.0) fail("force_threshold must be >= 0");
  }
};

struct SimulationReport {
  std::uint64_t iterations = 0;
  std::uint64_t final_agent_count = 0;
  std::uint64_t force_evaluations = 0;
  std::uint64_t force_skips = 0;
  std::uint64_t agents_added = 0;
  std::uint64_t agents_removed = 0;
};

struct AgentState {
  std::uint64_t uid;
  Vec3 position;
  double diameter;
  Vec3 last_force;
  std::uint32_t nonzero_force_partners;
  std::uint8_t flags;  // ABS_FLAG_*
  bool is_static() const { return flags & ABS_FLAG_STATIC; }
};

class Simulation;

class UniformGrid {
 public:
  explicit UniformGrid(Simulation& sim) : sim_(sim) {}
  void update();
  double largest_agent_diameter() const { return info().first[4]; }
  double max_query_radius() const;  // unbounded for the brute-force environment
  double box_length() const { return info().first[3]; }
  Vec3 origin() const {
    const auto g = info().first;
    return {g[0], g[1], g[2]};
  }
  std::array<std::uint32_t, 3> dims() const { return info().second; }
  const char* name() const;
  // box_index_of for every agent (storage order of agents())
  std::vector<std::uint64_t> cell_ids();
  // for_each_neighbor at the force radius 0.5 (d + dmax) for every agent,
  // batched: fn(query_uid, neighbour_uid) in ascending neighbour uid order.
  template <class F>
  void for_each_neighbor_pair(F&& fn);

 private:
  std::pair<std::array<double, 5>, std::array<std::uint32_t, 3>> info() const;
  Simulation& sim_;
};

class Simulation {
 public:
  explicit Simulation(SimulationParams params, int device = 0) : params_(std::move(params)), env_(*this) {
    params_.validate();
    abs_gpu_config cfg;
    abs_gpu_default_config(&cfg);
    cfg.seed = params_.seed;
    cfg.simulation_time_step = params_.simulation_time_step;
    cfg.repulsion_coefficient = params_.repulsion_coefficient;
    cfg.max_displacement = params_.max_displacement;
    cfg.force_threshold = params_.force_threshold;
    cfg.fixed_box_length = params_.fixed_box_length;
    cfg.sorting_frequency = params_.sorting_frequency;
    cfg.detect_static_agents = params_.detect_static_agents ? 1 : 0;
    cfg.model = params_.model;
    for (int i = 0; i < 8; ++i) cfg.model_params[i] = params_.model_params[i];
    cfg.record_forces = params_.record_forces ? 1 : 0;
    cfg.environment = params_.environment_kind;
    check(abs_gpu_create(&cfg, device, &ctx_), nullptr);
  }
  ~Simulation() { abs_gpu_destroy(ctx_); }
  Simulation(const Simulation&) = delete;
  Simulation& operator=(const Simulation&) = delete;

  const SimulationParams& params() const { return params_; }
  abs_gpu_ctx* native() { return ctx_; }

  // Simulation::add_agent (simulation.cpp:131-141): uids in call order. Agents
  // are staged on the host and uploaded before the next device call.
  std::uint64_t add_agent(const Vec3& p, double diameter, bool behaviour = true) {
    if (!(diameter > 0.0)) throw std::invalid_argument("diameter must be > 0");
    if (uploaded_) throw std::logic_error("add_agent after the population was uploaded");
    x_.push_back(p.x);
    y_.push_back(p.y);
    z_.push_back(p.z);
    d_.push_back(diameter);
    mask_.push_back(behaviour ? 1 : 0);
    return x_.size() - 1;
  }

  void simulate(std::uint64_t iterations) {
    flush();
    check(abs_gpu_simulate(ctx_, iterations), ctx_);
  }

  SimulationReport report() {
    flush();
    abs_step_stats s{};
    check(abs_gpu_stats(ctx_, &s), ctx_);
    SimulationReport r;
    r.iterations = s.iterations;
    r.final_agent_count = s.agents;
    r.force_evaluations = s.force_evaluations;
    r.force_skips = s.force_skips;
    r.agents_added = s.agents_added;
    r.agents_removed = s.agents_removed;
    return r;
  }

  std::uint64_t iteration() { return report().iterations; }
  UniformGrid& environment() { return env_; }

  std::vector<AgentState> agents() {
    flush();
    abs_step_stats s{};
    check(abs_gpu_stats(ctx_, &s), ctx_);
    const std::size_t n = s.agents;
    std::vector<std::uint64_t> uid(n);
    std::vector<double> x(n), y(n), z(n), d(n), fx(n), fy(n), fz(n);
    std::vector<std::uint32_t> partners(n);
    std::vector<std::uint8_t> flags(n);
    std::uint64_t got = 0;
    check(abs_gpu_download(ctx_, &got, uid.data(), x.data(), y.data(), z.data(), d.data(), fx.data(), fy.data(),
                           fz.data(), partners.data(), flags.data(), nullptr),
          ctx_);
    std::vector<AgentState> out(got);
    for (std::size_t i = 0; i < got; ++i)
      out[i] = AgentState{uid[i], {x[i], y[i], z[i]}, d[i], {fx[i], fy[i], fz[i]}, partners[i], flags[i]};
    return out;
  }

  // Host-boundary pipeline (abs_gpu_run_frames): independent host frames, each
  // = add the frame's agents -> simulate(iterations) -> read positions back,
  // with the next frame's upload and the previous frame's download overlapping
  // the current frame on the device. Replaces the staged population.
  struct Frame {
    const double *x, *y, *z, *d;  // n agents (page-locked memory: plain DMA)
    std::uint64_t n;
    double *out_x, *out_y, *out_z;  // out_cap entries each
    std::uint64_t out_cap;
    std::uint64_t* out_uid = nullptr;  // optional
    std::uint64_t n_out = 0;           // filled: agents after the iterations
  };
  void run_frames(std::vector<Frame>& frames, std::uint64_t iterations, std::uint64_t first_iteration = 0) {
    std::vector<abs_frame> f(frames.size());
    for (std::size_t i = 0; i < frames.size(); ++i) {
      const Frame& F = frames[i];
      f[i] = abs_frame{F.n, F.x, F.y, F.z, F.d, F.out_x, F.out_y, F.out_z, F.out_cap, &frames[i].n_out, F.out_uid};
    }
    uploaded_ = true;  // the frames replace any staged population
    check(abs_gpu_run_frames(ctx_, f.data(), f.size(), iterations, first_iteration), ctx_);
  }

  void flush() {
    if (uploaded_) return;
    uploaded_ = true;
    check(abs_gpu_upload(ctx_, x_.size(), nullptr, x_.data(), y_.data(), z_.data(), d_.data(), mask_.data(), nullptr,
                         nullptr, nullptr, 0),
          ctx_);
  }

 private:
  SimulationParams params_;
  abs_gpu_ctx* ctx_ = nullptr;
  UniformGrid env_;
  bool uploaded_ = false;
  std::vector<double> x_, y_, z_, d_;
  std::vector<std::uint8_t> mask_;
};

inline void UniformGrid::update() {
  sim_.flush();
  check(abs_gpu_env_update(sim_.native()), sim_.native());
}

inline double UniformGrid::max_query_radius() const {
  return sim_.params().environment_kind != ABS_ENV_UNIFORM_GRID ? std::numeric_limits<double>::infinity()
                                                                : box_length();
}

inline const char* UniformGrid::name() const {
  const int k = sim_.params().environment_kind;
  return k == ABS_ENV_BRUTE_FORCE ? "brute_force" : (k == ABS_ENV_KD_TREE ? "kdtree" : "uniform_grid");
}

inline std::pair<std::array<double, 5>, std::array<std::uint32_t, 3>> UniformGrid::info() const {
  std::array<double, 5> g{};
  std::array<std::uint32_t, 3> d{};
  check(abs_gpu_grid_info(sim_.native(), g.data(), d.data()), sim_.native());
  return {g, d};
}

inline std::vector<std::uint64_t> UniformGrid::cell_ids() {
  const std::size_t n = sim_.report().final_agent_count;
  std::vector<std::uint64_t> out(n);
  check(abs_gpu_cell_ids(sim_.native(), out.data()), sim_.native());
  return out;
}

template <class F>
void UniformGrid::for_each_neighbor_pair(F&& fn) {
  const auto agents = sim_.agents();
  std::vector<std::uint64_t> off(agents.size() + 1);
  std::uint64_t total = 0;
  check(abs_gpu_neighbors(sim_.native(), off.data(), nullptr, 0, &total), sim_.native());
  std::vector<std::uint64_t> uids(total ? total : 1);
  check(abs_gpu_neighbors(sim_.native(), off.data(), uids.data(), total, &total), sim_.native());
  for (std::size_t i = 0; i < agents.size(); ++i)
    for (std::uint64_t k = off[i]; k < off[i + 1]; ++k) fn(agents[i].uid, uids[k]);
}

}  // namespace absim_b200
