// host_known_answers.cpp — the reference's own known-answer tests, re-run
// through the C++ host API (include/absim_b200.hpp) on the B200 kernels.
// Each case cites the reference test it restates. Exit status = failures.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <set>
#include <string>
#include <vector>

#include "absim_b200.hpp"

using namespace absim_b200;

static int failures = 0;
#define CHECK(cond)                                                        \
  do {                                                                     \
    if (!(cond)) {                                                         \
      std::printf("  FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);         \
      ++failures;                                                          \
    }                                                                      \
  } while (0)

static std::set<std::uint64_t> static_uids(Simulation& sim) {
  std::set<std::uint64_t> s;
  for (const AgentState& a : sim.agents())
    if (a.is_static()) s.insert(a.uid);
  return s;
}

static void lattice(Simulation& sim, int side, double spacing, bool grow_column) {
  for (int x = 0; x < side; ++x)
    for (int y = 0; y < side; ++y)
      for (int z = 0; z < side; ++z)
        sim.add_agent({x * spacing, y * spacing, z * spacing}, 10.0, grow_column && x == 0 && y == side / 2);
}

int main() {
  {  // test_scheduler.cpp:464-488 — settled lattice
    std::printf("settled lattice\n");
    SimulationParams p;
    p.detect_static_agents = true;
    Simulation sim(p);
    lattice(sim, 3, 10.0, false);
    sim.simulate(1);
    CHECK(sim.report().force_evaluations == 108 && sim.report().force_skips == 0);
    sim.simulate(1);
    CHECK(sim.report().force_evaluations == 108 && sim.report().force_skips == 27);
    sim.simulate(1);
    CHECK(sim.report().force_skips == 54);
    CHECK(static_uids(sim).size() == 27);
  }
  {  // test_scheduler.cpp:490-519 — cancelling triple
    std::printf("cancelling triple\n");
    SimulationParams p;
    p.detect_static_agents = true;
    p.force_threshold = 10.0;
    Simulation sim(p);
    sim.add_agent({0, 0, 0}, 12.0);
    sim.add_agent({10, 0, 0}, 12.0);
    sim.add_agent({20, 0, 0}, 12.0);
    sim.simulate(1);
    CHECK(sim.report().force_evaluations == 4 && sim.report().force_skips == 0);
    sim.simulate(2);
    CHECK(sim.report().force_evaluations == 8 && sim.report().force_skips == 4);
    CHECK((static_uids(sim) == std::set<std::uint64_t>{0, 2}));
    for (const AgentState& a : sim.agents()) CHECK(a.position.x == 10.0 * static_cast<double>(a.uid));
  }
  {  // test_scheduler.cpp:521-534 — growth wakes shells (models::Grow)
    std::printf("static front\n");
    SimulationParams p;
    p.detect_static_agents = true;
    p.model = ABS_MODEL_GROW;
    p.model_params[0] = 0.5;
    p.model_params[1] = 20.0;
    Simulation sim(p);
    lattice(sim, 3, 10.0, true);
    sim.simulate(3);
    CHECK((static_uids(sim) == std::set<std::uint64_t>{18, 19, 20, 24, 25, 26}));
    CHECK(sim.report().force_skips > 0);
  }
  {  // test_mechanics.cpp:20-31 — overlap 2, k 2 -> force 4 along +x
    std::printf("pairwise repulsion\n");
    SimulationParams p;
    Simulation sim(p);
    sim.add_agent({8, 0, 0}, 10.0);
    sim.add_agent({0, 0, 0}, 10.0);
    sim.simulate(1);
    for (const AgentState& a : sim.agents()) {
      const double expect = a.uid == 0 ? 4.0 : -4.0;
      CHECK(std::fabs(a.last_force.x - expect) <= 1e-12 && a.last_force.y == 0.0 && a.last_force.z == 0.0);
    }
  }
  {  // test_grid.cpp:68-86, :108-120 — floor/clamp, inclusive radius
    std::printf("grid\n");
    SimulationParams p;
    p.fixed_box_length = 20.0;
    Simulation sim(p);
    sim.add_agent({0, 0, 0}, 10.0);
    sim.add_agent({100, 100, 100}, 10.0);
    sim.add_agent({19.999, 20.0, 39.9}, 10.0);
    sim.environment().update();
    CHECK((sim.environment().dims() == std::array<std::uint32_t, 3>{6, 6, 6}));
    const auto ids = sim.environment().cell_ids();
    const auto ag = sim.agents();
    for (std::size_t i = 0; i < ag.size(); ++i) {
      if (ag[i].uid == 2) CHECK(ids[i] == 0 + 6 * (1 + 6 * 1));
      if (ag[i].uid == 1) CHECK(ids[i] == 215);
    }
    SimulationParams q;
    Simulation two(q);
    two.add_agent({0, 0, 0}, 15.0);
    two.add_agent({15, 0, 0}, 15.0);
    two.environment().update();
    int pairs = 0;
    two.environment().for_each_neighbor_pair([&](std::uint64_t a, std::uint64_t b) {
      CHECK(a != b);
      ++pairs;
    });
    CHECK(pairs == 2);
    CHECK(std::string(two.environment().name()) == "uniform_grid");
  }
  {  // errors: params.cpp:44-72, uniform_grid.cpp:118-125
    std::printf("errors\n");
    SimulationParams p;
    p.simulation_time_step = 0.0;
    bool threw = false;
    try {
      Simulation bad(p);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    CHECK(threw);
    SimulationParams q;
    q.fixed_box_length = 5.0;
    Simulation sim(q);
    sim.add_agent({0, 0, 0}, 10.0);
    threw = false;
    try {
      sim.simulate(1);
    } catch (const Error& e) {
      threw = std::string(e.what()).find("failed at iteration 0") != std::string::npos;
    }
    CHECK(threw);
  }
  {  // test_scheduler.cpp:50-66 — empty simulation runs the schedule
    std::printf("empty\n");
    SimulationParams p;
    p.detect_static_agents = true;
    Simulation sim(p);
    sim.simulate(10);
    CHECK(sim.report().iterations == 10 && sim.report().final_agent_count == 0);
  }
  {  // mechanics.cpp:10-27 through the frame pipeline: each frame is a pair at
     // distance 8 with diameters 10 -> overlap 2, |F| = 4 (test_mechanics.cpp:11-30),
     // displaced by F dt; frames are independent populations
    std::printf("frames\n");
    SimulationParams p;
    p.simulation_time_step = 0.01;
    Simulation sim(p);
    std::vector<double> x = {0.0, 8.0}, y = {0.0, 0.0}, z = {0.0, 0.0}, d = {10.0, 10.0};
    std::vector<double> x2 = {100.0, 108.0};
    std::vector<std::vector<double>> ox(2, std::vector<double>(2)), oy = ox, oz = ox;
    std::vector<std::vector<std::uint64_t>> ou(2, std::vector<std::uint64_t>(2));
    std::vector<Simulation::Frame> fr(2);
    for (int f = 0; f < 2; ++f)
      fr[f] = Simulation::Frame{f ? x2.data() : x.data(), y.data(), z.data(), d.data(), 2,
                                ox[f].data(), oy[f].data(), oz[f].data(), 2, ou[f].data()};
    sim.run_frames(fr, 1);
    for (int f = 0; f < 2; ++f) {
      CHECK(fr[f].n_out == 2);
      const double base = f ? 100.0 : 0.0;
      for (int i = 0; i < 2; ++i) {
        const double want = base + (ou[f][i] == 0 ? -0.04 : 8.04);  // F dt = 4 * 0.01
        CHECK(std::fabs(ox[f][i] - want) < 1e-12);
      }
    }
  }
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "PASSED", failures);
  return failures;
}
