// Drop-in check of include/tmpc_b200/planner.hpp: a program written against
// the reference library's own headers (tmpc/*.hpp) calls solve_ocp /
// plan_step and gets the B200 planner.  Built by __graft_entry__.build() when
// the reference headers are present; run by tests/test_cpp_api.py.
//   ./test_planner_api        -> host-side checks (no GPU needed)
//   ./test_planner_api gpu    -> one solve on cuda:0
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "tmpc_b200/planner.hpp"

using namespace tmpc;

static int fails = 0;
#define CHECK(c)                                                   \
  do {                                                             \
    if (!(c)) {                                                    \
      std::fprintf(stderr, "CHECK failed: %s (line %d)\n", #c, __LINE__); \
      ++fails;                                                     \
    }                                                              \
  } while (0)

int main(int argc, char** argv) {
  const bool gpu = argc > 1 && std::strcmp(argv[1], "gpu") == 0;
  // flat terrain via the reference's own generator (terrain.hpp:281-332)
  SynthSpec spec;
  spec.kind = TerrainKind::kFlat;
  spec.grid = GridSpec{-20.0, -40.0, 0.2, 400, 400};
  const Heightmap hm = synth_terrain(spec);
  const SignedDistanceMap sd = build_sdist_map(hm.grid, {});  // no features
  VehicleParams vp;
  SrbState s0;
  s0.z = vp.h + vp.R;
  s0.v_bx = 5.0;
  Goal goal{15.0, 0.0, 2.5};
  PlannerConfig cfg;
  cfg.n_samples = 256;
  cfg.n_steps = 20;
  cfg.dt_zoh = 0.05;
  cfg.seed = 7;

  // validation happens before any device work (constraints.hpp:51-57)
  ConstraintConfig bad;
  bad.sigma = 0.0;
  bool threw = false;
  try {
    solve_ocp(s0, hm, sd, goal, cfg, CostWeights{}, bad);
  } catch (const ConfigError& e) {
    threw = std::string(e.what()).find("sigma") != std::string::npos;
  }
  CHECK(threw);
  PlannerConfig bad_dt = cfg;
  bad_dt.dt_int = 0.003;  // dynamics.hpp:477-481
  threw = false;
  try {
    solve_ocp(s0, hm, sd, goal, bad_dt);
  } catch (const ConfigError&) {
    threw = true;
  }
  CHECK(threw);

  if (!gpu) {
    threw = false;
    try {
      solve_ocp(s0, hm, sd, goal, cfg);
    } catch (const ConfigError&) {
    } catch (const std::runtime_error& e) {
      threw = std::string(e.what()).find("CUDA") != std::string::npos;
    }
    CHECK(threw);
    std::printf(fails ? "FAIL\n" : "host checks ok\n");
    return fails ? 1 : 0;
  }

  const SolveOutput out = solve_ocp(s0, hm, sd, goal, cfg);
  CHECK(out.best.entries.size() == 20u);
  CHECK(out.result.index >= 0 && out.result.index < 256);
  CHECK(out.result.feasible);
  CHECK(out.stats.n_samples == 256);
  CHECK(out.stats.n_diverged == 0);
  CHECK(out.stats.min_cost == out.result.cost);
  for (const Control& c : out.best.entries) CHECK(std::fabs(c.delta_rate) <= vp.delta_rate_max);
  Planner pl(cfg);
  pl.set_terrain(hm, sd);
  const Control u = plan_step(pl, s0, goal);
  CHECK(u.delta_rate == out.best.entries[0].delta_rate);  // SPEC.md:395 contract
  // the other formulations through the same drop-in: Scheme::kRk4 and EstModel
  for (int variant = 0; variant < 3; ++variant) {
    PlannerConfig c2 = cfg;
    c2.rk4 = variant != 1;
    c2.est_model = variant >= 1;
    const SolveOutput o2 = solve_ocp(s0, hm, sd, goal, c2);
    CHECK(o2.stats.n_diverged == 0);
    CHECK(o2.result.feasible);
    CHECK(std::isfinite(o2.result.cost) && o2.result.cost > 0.0);
    // flat ground: RK4 and Euler agree to integration error on the same candidates
    if (variant == 0) CHECK(std::fabs(o2.result.cost - out.result.cost) < 1e-2 * out.result.cost);
  }
  // one solve_ocp over several GPUs (here two shards on cuda:0): the same
  // winner, cost and counts as the one-GPU solve
  {
    PlannerConfig cm = cfg;
    cm.devices = {0, 0};
    const SolveOutput om = solve_ocp(s0, hm, sd, goal, cm);
    CHECK(om.result.index == out.result.index);
    CHECK(om.result.cost == out.result.cost);
    CHECK(om.stats.n_feasible == out.stats.n_feasible);
    CHECK(om.stats.mean_cost == out.stats.mean_cost);
    CHECK(om.best.entries[0].delta_rate == out.best.entries[0].delta_rate);
  }
  // device terrain preprocessing == the reference functions, bit for bit
  {
    SynthSpec bumps;
    bumps.kind = TerrainKind::kBumpField;
    bumps.grid = GridSpec{-10.0, -10.0, 0.1, 200, 180};
    bumps.amplitude = 0.5;
    bumps.n_bumps = 12;
    bumps.seed = 3;
    const Heightmap hb = synth_terrain(bumps);
    const Heightmap a = b200::gaussian_smooth(hb, 0.3), b = gaussian_smooth(hb, 0.3);
    CHECK(a.heights == b.heights);
    Perimeter box;
    box.vertices = {{1.0, 1.0}, {3.0, 1.0}, {3.0, 2.5}, {1.0, 2.5}};
    Perimeter lane;
    lane.kind = PerimeterKind::kPathBoundary;
    lane.vertices = {{-9.0, -5.0}, {9.0, -5.0}, {9.0, 5.0}, {-9.0, 5.0}};
    const SignedDistanceMap s1 = b200::build_sdist_map(bumps.grid, {box, lane});
    const SignedDistanceMap s2 = build_sdist_map(bumps.grid, {box, lane});
    CHECK(s1.values == s2.values);
  }
  std::printf("best %lld cost %.6f  %s\n", static_cast<long long>(out.result.index),
              out.result.cost, fails ? "FAIL" : "gpu checks ok");
  return fails ? 1 : 0;
}
