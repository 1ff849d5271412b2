// tmpc_b200/planner.hpp — drop-in C++ planner API over libtmpc_b200.so.
//
// A user of the reference library keeps including its headers (tmpc/*.hpp,
// /root/reference/proj/include) for VehicleParams, TireParams, SrbState,
// Control, ControlSequence, Heightmap, SignedDistanceMap and ConstraintConfig
// (dynamics.hpp:20-183, terrain.hpp:20-239, constraints.hpp:42-58), and gets
// from this header the SPEC planner types and entry points the reference
// leaves unimplemented: CostWeights, Goal, PlannerConfig,
// RolloutResult, SolverStats, solve_ocp, plan_step — evaluated by the sm_100a
// kernels behind the C ABI (tmpc_b200.h).  Link with -ltmpc_b200.
//
// Error mapping (errors.hpp:8-27): TMPC_ERR_CONFIG ->
// ConfigError, TMPC_ERR_NUMERIC -> NumericError, TMPC_ERR_RUNTIME ->
// std::runtime_error.
#pragma once

#include <algorithm>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "tmpc/constraints.hpp"
#include "tmpc/dynamics.hpp"
#include "tmpc/errors.hpp"
#include "tmpc/terrain.hpp"
#include "tmpc_b200.h"

namespace tmpc {

// SPEC.md:349 (PAPER.md:880-883 defaults)
struct CostWeights {
  double w_t = 5.0;
  double w_c = 8.0;
  double w_g = 15.0;
};

// SPEC.md:357
struct Goal {
  double x_g = 0.0;
  double y_g = 0.0;
  double r_g = 2.5;
};

enum class SamplerKind { kUniform = TMPC_SAMPLE_UNIFORM, kRandomWalk = TMPC_SAMPLE_RANDOM_WALK,
                         kWarmGauss = TMPC_SAMPLE_WARM_GAUSS };

// SPEC.md:360-363 + the sampler / selection / device knobs of the B200 build.
struct PlannerConfig {
  int64_t n_samples = 1024;
  std::uint64_t seed = 0;
  int n_steps = 16;
  double dt_zoh = 0.25;
  double dt_int = 0.005;
  SamplerKind sampler = SamplerKind::kUniform;
  double vdot_max = 0.0;
  double walk_step = 0.25;
  double warm_sigma_frac = 0.10;
  bool feasible_first = true;  // arg-min key (infeasible, J, k); false = (J, k)
  bool est_model = false;      // EST formulation (dynamics.hpp:230-275) instead of SRB
  bool rk4 = false;            // Scheme::kRk4 substeps (dynamics.hpp:453-462) instead of Euler
  int device = 0;
  // GPUs driven by this one planner (one process):
  // the candidates of every solve are split over them and the per-GPU
  // arg-min records folded in order; empty = {device}.  An ordinal may repeat.
  std::vector<int> devices;
  bool fp64 = false;  // TMPC_PRECISION_FP64 certification mode
};

// SPEC.md:365-367
struct RolloutResult {
  double cost = 0.0;
  bool feasible = false;
  float margin = 0.0f;
  int64_t index = -1;
};

// SPEC.md:386,414
struct SolverStats {
  double best_cost = 0.0, min_cost = 0.0, mean_cost = 0.0;
  int64_t n_samples = 0, n_feasible = 0, n_diverged = 0, n_goal = 0, substeps = 0;
  double kernel_ms = 0.0, cycle_ms = 0.0;
  double rollouts_per_s() const { return cycle_ms > 0 ? n_samples / (cycle_ms * 1e-3) : 0.0; }
};

struct SolveOutput {
  ControlSequence best;
  RolloutResult result;
  SolverStats stats;
};

namespace b200 {

inline void check(int rc, const tmpc_ctx* ctx) {
  if (rc == TMPC_OK) return;
  const std::string msg = tmpc_last_error(ctx);
  if (rc == TMPC_ERR_CONFIG) throw ConfigError(msg);
  if (rc == TMPC_ERR_NUMERIC) throw NumericError(msg);
  throw std::runtime_error(msg);
}

inline tmpc_params to_params(const VehicleParams& vp, const TireParams& tp,
                             const ConstraintConfig& cc, const CostWeights& w, const Goal& g,
                             const PlannerConfig& cfg) {
  tmpc_params p{};
  p.M = vp.M; p.J_xx = vp.J_xx; p.J_yy = vp.J_yy; p.J_zz = vp.J_zz; p.L_f = vp.L_f;
  p.L_r = vp.L_r; p.e = vp.e; p.h = vp.h; p.R = vp.R; p.k_f = vp.k_f; p.k_r = vp.k_r;
  p.b_f = vp.b_f; p.b_r = vp.b_r; p.delta_max = vp.delta_max;
  p.delta_rate_max = vp.delta_rate_max; p.g = vp.g;
  p.C = tp.C; p.mu = tp.mu;
  p.a_by_bar = cc.a_by_bar;
  // esm_nominal defaults to 0 in the reference (constraints.hpp:44), which
  // would make eps_ESM zero; fill it from esm_normalization
  p.esm_nominal = cc.esm_nominal > 0.0 ? cc.esm_nominal : esm_normalization(vp);
  p.eps_dist = cc.eps_dist; p.sigma = cc.sigma; p.safety_factor = cc.safety_factor;
  p.enable_dist = cc.enable_dist; p.enable_rollover = cc.enable_rollover;
  p.w_t = w.w_t; p.w_c = w.w_c; p.w_g = w.w_g;
  p.goal_x = g.x_g; p.goal_y = g.y_g; p.goal_r = g.r_g;
  p.dt_zoh = cfg.dt_zoh; p.dt_int = cfg.dt_int; p.n_steps = cfg.n_steps;
  p.selection = cfg.feasible_first ? TMPC_SELECT_FEASIBLE_FIRST : TMPC_SELECT_PLAIN;
  p.model = cfg.est_model ? TMPC_MODEL_EST : TMPC_MODEL_SRB;
  p.scheme = cfg.rk4 ? TMPC_SCHEME_RK4 : TMPC_SCHEME_EULER;
  return p;
}

// Device terrain preprocessing, bit-identical to the reference functions of
// the same name (terrain.hpp:102-138, 241-260).
inline Heightmap gaussian_smooth(const Heightmap& m, double sigma_m, int device = 0) {
  Heightmap out = m;
  check(tmpc_gaussian_smooth(device, m.heights.data(), m.grid.nx, m.grid.ny, m.grid.resolution,
                             sigma_m, out.heights.data()),
        nullptr);
  return out;
}

inline SignedDistanceMap build_sdist_map(const GridSpec& grid,
                                         const std::vector<Perimeter>& perimeters,
                                         int device = 0) {
  std::vector<int32_t> off{0}, kinds;
  std::vector<double> verts;
  for (const Perimeter& p : perimeters) {
    for (const auto& v : p.vertices) {
      verts.push_back(v.x());
      verts.push_back(v.y());
    }
    off.push_back(static_cast<int32_t>(verts.size() / 2));
    kinds.push_back(p.kind == PerimeterKind::kPathBoundary ? 1 : 0);
  }
  SignedDistanceMap map;
  map.grid = grid;
  map.has_features = !perimeters.empty();
  map.values.resize(static_cast<size_t>(grid.nx) * grid.ny);
  check(tmpc_build_sdist_map_gpu(device, grid.nx, grid.ny, grid.origin_x, grid.origin_y,
                                 grid.resolution, static_cast<int32_t>(perimeters.size()),
                                 off.data(), verts.data(), kinds.data(), map.values.data()),
        nullptr);
  return map;
}

}  // namespace b200

// One planning problem resident on one GPU, or on the GPUs of
// PlannerConfig::devices (terrain uploaded once per GPU).
class Planner {
 public:
  explicit Planner(const PlannerConfig& cfg, int rank = 0, int world_size = 1,
                   const void* nccl_id = nullptr)
      : cfg_(cfg) {
    tmpc_opts o{};
    o.device = cfg.device;
    o.rank = rank;
    o.world_size = world_size;
    o.k_max = cfg.n_samples;
    o.n_steps_max = cfg.n_steps;
    o.precision = cfg.fp64 ? TMPC_PRECISION_FP64 : TMPC_PRECISION_FP32;
    o.nccl_id = nccl_id;
    std::vector<int32_t> devs(cfg.devices.begin(), cfg.devices.end());
    if (!devs.empty()) {
      o.n_devices = static_cast<int32_t>(devs.size());
      o.devices = devs.data();
    }
    tmpc_ctx* c = nullptr;
    b200::check(tmpc_ctx_create(&o, &c), nullptr);
    ctx_.reset(c);
  }

  void set_terrain(const Heightmap& hm, const SignedDistanceMap& sd) {
    tmpc_terrain t{};
    t.heights = hm.heights.data();
    t.sdist = sd.has_features ? sd.values.data() : nullptr;
    t.nx = hm.grid.nx;
    t.ny = hm.grid.ny;
    t.origin_x = hm.grid.origin_x;
    t.origin_y = hm.grid.origin_y;
    t.resolution = hm.grid.resolution;
    if (sd.has_features && (sd.grid.nx != hm.grid.nx || sd.grid.ny != hm.grid.ny))
      throw ConfigError("sdist grid must match the heightmap grid");
    b200::check(tmpc_set_terrain(ctx_.get(), &t), ctx_.get());
  }

  // solve_ocp for candidates [k_begin, k_begin + k_count)
  // of cfg.n_samples (shard of this rank).
  SolveOutput solve(const SrbState& s0, const Goal& goal, const CostWeights& w = {},
                    const ConstraintConfig& cc = {}, const VehicleParams& vp = {},
                    const TireParams& tp = {}, const ControlSequence* warm = nullptr,
                    int64_t k_begin = 0, int64_t k_count = -1) {
    const tmpc_params p = b200::to_params(vp, tp, cc, w, goal, cfg_);
    b200::check(tmpc_set_params(ctx_.get(), &p), ctx_.get());
    std::vector<double> warm_seq;
    tmpc_sampling smp{};
    smp.kind = static_cast<int32_t>(cfg_.sampler);
    smp.seed = cfg_.seed;
    smp.vdot_max = cfg_.vdot_max;
    smp.walk_step = cfg_.walk_step;
    smp.warm_sigma_frac = cfg_.warm_sigma_frac;
    if (warm) {
      for (int t = 0; t < cfg_.n_steps; ++t) {
        const Control& c = warm->entries.at(static_cast<size_t>(t));
        warm_seq.push_back(c.delta_rate);
        warm_seq.push_back(c.v_bx_rate);
      }
      smp.warm_seq = warm_seq.data();
    }
    smp.k_begin = k_begin;
    smp.k_count = k_count < 0 ? cfg_.n_samples : k_count;
    smp.k_total = std::max<int64_t>(cfg_.n_samples, smp.k_begin + smp.k_count);
    const auto a = s0.as_array();
    tmpc_result r{};
    std::vector<double> ctrl(2 * static_cast<size_t>(cfg_.n_steps));
    b200::check(tmpc_solve(ctx_.get(), a.data(), &smp, &r, ctrl.data()), ctx_.get());
    SolveOutput out;
    out.best.dt_zoh = cfg_.dt_zoh;
    for (int t = 0; t < cfg_.n_steps; ++t) out.best.entries.push_back({ctrl[2 * t], ctrl[2 * t + 1]});
    out.result = {r.best_cost, r.best_feasible != 0, r.best_margin, r.best_index};
    out.stats.best_cost = r.best_cost;
    out.stats.min_cost = r.min_cost;
    out.stats.mean_cost = r.mean_cost;
    out.stats.n_samples = r.n_candidates;
    out.stats.n_feasible = r.n_feasible;
    out.stats.n_diverged = r.n_diverged;
    out.stats.n_goal = r.n_goal;
    out.stats.substeps = r.substeps_executed;
    out.stats.kernel_ms = r.kernel_ms;
    out.stats.cycle_ms = r.cycle_ms;
    return out;
  }

  const PlannerConfig& config() const { return cfg_; }

 private:
  struct Del {
    void operator()(tmpc_ctx* c) const { tmpc_ctx_destroy(c); }
  };
  PlannerConfig cfg_;
  std::unique_ptr<tmpc_ctx, Del> ctx_;
};

// One-shot solve_ocp.  Parameters are validated (same rules
// as the reference validate() methods) before any device work.
inline SolveOutput solve_ocp(const SrbState& s0, const Heightmap& hm, const SignedDistanceMap& sd,
                             const Goal& goal, const PlannerConfig& cfg,
                             const CostWeights& w = {}, const ConstraintConfig& cc = {},
                             const VehicleParams& vp = {}, const TireParams& tp = {}) {
  const tmpc_params p = b200::to_params(vp, tp, cc, w, goal, cfg);
  char msg[256] = {0};
  if (tmpc_validate_params(&p, msg, sizeof msg) != TMPC_OK) throw ConfigError(msg);
  Planner pl(cfg);
  pl.set_terrain(hm, sd);
  return pl.solve(s0, goal, w, cc, vp, tp);
}

// plan_step: the first ZOH control of the best sequence.
inline Control plan_step(Planner& pl, const SrbState& s, const Goal& goal,
                         const CostWeights& w = {}, const ConstraintConfig& cc = {},
                         const VehicleParams& vp = {}, const TireParams& tp = {}) {
  return pl.solve(s, goal, w, cc, vp, tp).best.entries.at(0);
}

}  // namespace tmpc
