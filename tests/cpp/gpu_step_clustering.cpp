// gpu_step_clustering.cpp — the reference's own clustering benchmark
// population (models::build_clustering, models.cpp:40-61; Cohere(30, 1),
// box pinned by tune_clustering_params) advanced K iterations twice: by the
// unmodified reference Simulation on the CPU, and by the same kind of
// Simulation whose hot path is forwarded to the B200 through
// integration/gpu_step.hpp. Agent state is compared per uid with the parity
// bars of SURVEY.md §8c (positions within 1e-9 relative, tags / stream
// counters / partners exact). Exit status = failures; prints PASSED.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <map>

#include "absim/models.hpp"
#include "gpu_step.hpp"

using namespace absim;

struct State {
  double x, y, z, d;
  std::uint32_t tag, partners;
  std::uint64_t rngc;
};

static std::map<std::uint64_t, State> snapshot(Simulation& s) {
  std::map<std::uint64_t, State> out;
  s.resource_manager().for_each_agent([&](Agent& a, AgentHandle) {
    out[a.uid()] = {a.position().x, a.position().y, a.position().z, a.diameter(), a.tag(),
                    a.nonzero_force_partners(), *a.rng_counter()};
  });
  return out;
}

int main(int argc, char** argv) {
  const std::uint64_t n = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 20000;
  const std::uint64_t iters = argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 20;
  SimulationParams p;
  p.thread_count = 1;
  p.domain_count = 1;
  models::ClusteringConfig cfg;
  models::tune_clustering_params(p, cfg);
  Simulation cpu(p), gpu(p);
  models::build_clustering(cpu, n, cfg);
  models::build_clustering(gpu, n, cfg);

  cpu.simulate(iters);  // the reference, unmodified
  absim_gpu_bridge::DeviceModel m;
  m.model = ABS_MODEL_COHERE;
  m.params[0] = cfg.attraction_radius;
  m.params[1] = cfg.speed;
  absim_gpu_bridge::GpuStep step(p, m);
  step.run(gpu, 0, iters);

  const auto a = snapshot(cpu), b = snapshot(gpu);
  int failures = 0;
  double worst = 0.0;
  if (a.size() != b.size()) ++failures;
  for (const auto& [uid, s] : a) {
    const auto it = b.find(uid);
    if (it == b.end()) {
      ++failures;
      continue;
    }
    const State& g = it->second;
    for (const auto& [o, v] : {std::pair{s.x, g.x}, std::pair{s.y, g.y}, std::pair{s.z, g.z}, std::pair{s.d, g.d}}) {
      const double e = std::fabs(o - v) / std::fmax(std::fabs(o), 1.0);
      worst = std::fmax(worst, e);
      if (e > 1e-9) ++failures;
    }
    if (s.tag != g.tag || s.partners != g.partners || s.rngc != g.rngc) ++failures;
  }
  std::printf("clustering n=%llu iterations=%llu agents=%zu worst position error %.3e, failures %d\n",
              static_cast<unsigned long long>(n), static_cast<unsigned long long>(iters), a.size(), worst, failures);
  if (!failures) std::printf("PASSED\n");
  return failures;
}
