// integration/gpu_step.hpp — the reference-side bridge.
//
// What a maintainer of the reference adds to make its own absim::Simulation
// run the hot path on the B200: GpuStep packs the Simulation's agents
// (ResourceManager::for_each_agent, resource_manager.hpp:19-101) into the
// C ABI's SoA arrays (include/absim_gpu.h), runs whole iterations there —
// UniformGrid::update, the behaviour as a compiled device model, run_forces,
// run_integration, run_commit and the Morton sort cadence
// (simulation.cpp:222-322) — and writes the resulting agent state back into
// the same Agent objects by uid (position, diameter, tag, RandomStream
// counter, last force, partners, staticness flags). Daughters created on the
// device are added through Simulation::add_agent in uid order, which
// reproduces the reference's uid assignment (resource_manager.hpp:44-46).
// Compiled against the reference's public headers only; no reference source
// is modified. tests/cpp/gpu_step_clustering.cpp runs the reference's own
// build_clustering population through it and against the pure reference.
#pragma once

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "absim/simulation.hpp"
#include "absim_gpu.h"

namespace absim_gpu_bridge {

// The behaviour attached to the population, as a compiled device model
// (absim_gpu.h ABS_MODEL_*; e.g. models::Cohere(r, v) -> {ABS_MODEL_COHERE, {r, v}}).
struct DeviceModel {
  int model = ABS_MODEL_NONE;
  double params[8] = {0, 0, 0, 0, 0, 0, 0, 0};
};

class GpuStep {
 public:
  GpuStep(const absim::SimulationParams& p, const DeviceModel& m = {}, int device = 0) {
    abs_gpu_config c;
    abs_gpu_default_config(&c);
    c.seed = p.seed;
    c.simulation_time_step = p.simulation_time_step;
    c.repulsion_coefficient = p.repulsion_coefficient;
    c.max_displacement = p.max_displacement;
    c.force_threshold = p.force_threshold;
    c.fixed_box_length = p.fixed_box_length;
    c.sorting_frequency = p.sorting_frequency;  // Morton sort cadence, simulation.cpp:246-247
    c.detect_static_agents = p.detect_static_agents ? 1 : 0;
    c.environment = p.environment_kind == absim::EnvironmentKind::kBruteForce
                        ? ABS_ENV_BRUTE_FORCE
                        : (p.environment_kind == absim::EnvironmentKind::kKdTree ? ABS_ENV_KD_TREE : ABS_ENV_UNIFORM_GRID);
    c.model = m.model;
    for (int q = 0; q < 8; ++q) c.model_params[q] = m.params[q];
    c.record_forces = 1;
    if (abs_gpu_create(&c, device, &ctx_) != ABS_OK) throw std::runtime_error(abs_gpu_last_error(nullptr));
  }
  ~GpuStep() { abs_gpu_destroy(ctx_); }
  GpuStep(const GpuStep&) = delete;
  GpuStep& operator=(const GpuStep&) = delete;

  // Runs iterations [first_iteration, first_iteration + iterations) of sim's
  // population on the device and writes the state back into sim's agents.
  void run(absim::Simulation& sim, std::uint64_t first_iteration, std::uint64_t iterations) {
    absim::ResourceManager& rm = sim.resource_manager();
    std::vector<std::uint64_t> uid;
    std::vector<double> x, y, z, d;
    std::vector<std::uint32_t> tag;
    std::vector<std::uint64_t> rngc;
    rm.for_each_agent([&](absim::Agent& a, absim::AgentHandle) {
      uid.push_back(a.uid());
      x.push_back(a.position().x);
      y.push_back(a.position().y);
      z.push_back(a.position().z);
      d.push_back(a.diameter());
      tag.push_back(a.tag());
      rngc.push_back(*a.rng_counter());
    });
    const std::uint64_t n = uid.size();
    check(abs_gpu_upload(ctx_, n, uid.data(), x.data(), y.data(), z.data(), d.data(), nullptr, nullptr, nullptr,
                         nullptr, rm.uid_count()));
    check(abs_gpu_set_agent_ext(ctx_, tag.data(), rngc.data()));
    check(abs_gpu_set_iteration(ctx_, first_iteration));
    check(abs_gpu_simulate(ctx_, iterations));
    abs_step_stats st{};
    check(abs_gpu_stats(ctx_, &st));
    const std::uint64_t m = st.agents;
    uid.assign(m, 0);
    x.assign(m, 0.0), y.assign(m, 0.0), z.assign(m, 0.0), d.assign(m, 0.0);
    std::vector<double> fx(m), fy(m), fz(m), vol(m);
    std::vector<std::uint32_t> partners(m);
    std::vector<std::uint8_t> flags(m);
    tag.assign(m, 0);
    rngc.assign(m, 0);
    std::uint64_t got = 0;
    check(abs_gpu_download(ctx_, &got, uid.data(), x.data(), y.data(), z.data(), d.data(), fx.data(), fy.data(),
                           fz.data(), partners.data(), flags.data(), vol.data()));
    check(abs_gpu_download_ext(ctx_, tag.data(), rngc.data()));
    // removals are not part of the device models; daughters get uids
    // uid_count.. in creation order, which Simulation::add_agent reproduces
    std::vector<std::uint64_t> order(m);
    for (std::uint64_t i = 0; i < m; ++i) order[i] = i;
    std::sort(order.begin(), order.end(), [&](std::uint64_t a, std::uint64_t b) { return uid[a] < uid[b]; });
    for (std::uint64_t i : order) {
      absim::Agent* a = nullptr;
      if (uid[i] < rm.uid_count()) {
        a = &rm.agent(rm.handle_of_uid(uid[i]));
      } else {
        a = &sim.add_agent({x[i], y[i], z[i]}, d[i]);
        if (a->uid() != uid[i]) throw std::logic_error("daughter uid mismatch");
      }
      a->set_position({x[i], y[i], z[i]});
      a->set_diameter(d[i]);
      a->set_tag(tag[i]);
      *a->rng_counter() = rngc[i];
      a->set_last_force({fx[i], fy[i], fz[i]});
      a->set_nonzero_force_partners(partners[i]);
      a->set_static((flags[i] & ABS_FLAG_STATIC) != 0);
    }
  }

  abs_gpu_ctx* native() { return ctx_; }

 private:
  void check(int rc) {
    if (rc != ABS_OK) throw std::runtime_error(std::string("absim_gpu: ") + abs_gpu_last_error(ctx_));
  }
  abs_gpu_ctx* ctx_ = nullptr;
};

}  // namespace absim_gpu_bridge
