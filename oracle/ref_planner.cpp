// oracle/_ref — the SPEC planner over the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY (checker + CPU baseline arm of bench.py).  Never
// linked into, or called by, the product library.
//
// Built by oracle/Makefile from /root/reference/proj/include/tmpc/*.hpp (not
// copied) plus oracle/shim/Eigen/Dense.  The reference ships no planner: the
// SPEC defines trajectory_cost / sample_controls / solve_ocp
// and this file writes exactly that loop on top of the
// reference's own integrate_step<SrbModel> (dynamics.hpp:446-468),
// constraint_set_cost (constraints.hpp:87-100), esm (constraints.hpp:16-23),
// wheel_footprint (constraints.hpp:104-113), SignedDistanceMap::value_at
// (terrain.hpp:235-238) and RngStream/substream (rng.hpp:10-48).  The
// decisions the reference leaves open (goal test order, feasibility, margin,
// samplers) follow SURVEY.md App. A and DESIGN.md §3, identically to the
// restatement in oracle/tmpc_oracle.cpp and to the CUDA kernel.
#include <pthread.h>
#include <sched.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <limits>
#include <stdexcept>
#include <thread>
#include <vector>

#include "tmpc/constraints.hpp"
#include "tmpc/dynamics.hpp"
#include "tmpc/rng.hpp"
#include "tmpc/terrain.hpp"
#include "tmpc_b200.h"

namespace {

using namespace tmpc;

struct Problem {
  VehicleParams vp;
  TireParams tp;
  ConstraintConfig cc;
  Heightmap hm;
  SignedDistanceMap sd;
  const tmpc_params* p;
  const tmpc_sampling* smp;
};

Problem make_problem(const tmpc_params* p, const tmpc_sampling* smp, const tmpc_terrain* t) {
  Problem pr;
  VehicleParams& vp = pr.vp;
  vp.M = p->M; vp.J_xx = p->J_xx; vp.J_yy = p->J_yy; vp.J_zz = p->J_zz;
  vp.L_f = p->L_f; vp.L_r = p->L_r; vp.e = p->e; vp.h = p->h; vp.R = p->R;
  vp.k_f = p->k_f; vp.k_r = p->k_r; vp.b_f = p->b_f; vp.b_r = p->b_r;
  vp.delta_max = p->delta_max; vp.delta_rate_max = p->delta_rate_max; vp.g = p->g;
  pr.tp.C = p->C;
  pr.tp.mu = p->mu;
  ConstraintConfig& cc = pr.cc;
  cc.a_by_bar = p->a_by_bar; cc.esm_nominal = p->esm_nominal; cc.eps_dist = p->eps_dist;
  cc.sigma = p->sigma; cc.safety_factor = p->safety_factor;
  cc.enable_dist = p->enable_dist != 0; cc.enable_rollover = p->enable_rollover != 0;
  vp.validate();
  pr.tp.validate();
  cc.validate();
  pr.hm.grid = GridSpec{t->origin_x, t->origin_y, t->resolution, t->nx, t->ny};
  pr.hm.heights.assign(t->heights, t->heights + static_cast<size_t>(t->nx) * t->ny);
  pr.hm.validate();
  pr.sd.grid = pr.hm.grid;
  pr.sd.has_features = t->sdist != nullptr;
  if (t->sdist) pr.sd.values.assign(t->sdist, t->sdist + static_cast<size_t>(t->nx) * t->ny);
  pr.p = p;
  pr.smp = smp;
  return pr;
}

// sample_controls driven sequentially through the
// reference RngStream — this pins the random-access draw formula the device
// uses.
std::vector<Control> sample_controls(const Problem& pr, int64_t k) {
  const tmpc_params& p = *pr.p;
  const tmpc_sampling& s = *pr.smp;
  const int nch = s.vdot_max > 0.0 ? 2 : 1;
  const double bound[2] = {p.delta_rate_max, s.vdot_max};
  RngStream rng(substream(s.seed, static_cast<uint64_t>(k)));
  std::vector<Control> out(p.n_steps);
  double prev[2] = {0.0, 0.0};
  for (int t = 0; t < p.n_steps; ++t) {
    double v[2] = {0.0, 0.0};
    for (int c = 0; c < nch; ++c) {
      const double b = bound[c];
      if (s.kind == TMPC_SAMPLE_UNIFORM) {
        v[c] = rng.uniform(-b, b);
      } else if (s.kind == TMPC_SAMPLE_RANDOM_WALK) {
        const double a = c == 0 ? s.walk_step : s.walk_step * s.vdot_max / p.delta_rate_max;
        v[c] = std::clamp(prev[c] + rng.uniform(-a, a), -b, b);
        prev[c] = v[c];
      } else {
        const double u1 = rng.next_double();
        const double u2 = rng.next_double();
        const double base = s.warm_seq ? s.warm_seq[2 * t + c] : 0.0;
        const double z = std::sqrt(-2.0 * std::log(1.0 - u1)) * std::cos(2.0 * M_PI * u2);
        const double sigma = s.warm_sigma_frac * 2.0 * b;
        v[c] = std::clamp(k == 0 ? base : base + sigma * z, -b, b);
      }
    }
    out[t].delta_rate = v[0];
    out[t].v_bx_rate = v[1];
  }
  return out;
}

struct CandOut {
  double cost;
  uint8_t flags;
  float margin;
  int64_t substeps;
  double jrun;  // running cost accumulated when the rollout stopped (diverged or not)
};

// trajectory_cost over integrate_step, per the per-candidate
// algorithm of SURVEY §8a / DESIGN.md §3.
CandOut rollout(const Problem& pr, const double* s0a, int64_t k) {
  const tmpc_params& p = *pr.p;
  const std::vector<Control> u = sample_controls(pr, k);
  std::array<double, SrbState::kDim> a{};
  for (int i = 0; i < SrbState::kDim; ++i) a[i] = s0a[i];
  SrbState s = SrbState::from_array(a);
  const int S = static_cast<int>(std::lround(p.dt_zoh / p.dt_int));
  const double inf = std::numeric_limits<double>::infinity();
  double J = 0.0;
  bool feasible = true, diverged = false, goal = false;
  double margin = inf;
  int64_t n = 0;
  const double eps_esm = esm_epsilon(pr.cc);
  for (int t = 0; t < p.n_steps && !goal && !diverged; ++t) {
    for (int q = 0; q < S; ++q) {
      const double dx = s.x - p.goal_x, dy = s.y - p.goal_y;
      if (dx * dx + dy * dy <= p.goal_r * p.goal_r) {
        goal = true;
        break;
      }
      ConstraintMeasures m;
      const auto fp = wheel_footprint(s.x, s.y, s.psi, pr.vp);
      for (int i = 0; i < 4; ++i) m.wheel_sdist[i] = pr.sd.value_at(fp[i].x(), fp[i].y());
      const double U = esm(s.phi, s.theta, pr.vp);
      m.rollover_pi = -U;
      m.rollover_epsilon = eps_esm;
      const double L = p.w_t + p.w_c * u[t].delta_rate * u[t].delta_rate +
                       constraint_set_cost(m, pr.cc);
      J += p.dt_int * L;
      if (pr.cc.enable_rollover) {
        if (!(U > 0.0)) feasible = false;
        margin = std::min(margin, U / p.esm_nominal);
      }
      if (pr.cc.enable_dist && pr.sd.has_features) {
        for (int i = 0; i < 4; ++i) {
          if (!(m.wheel_sdist[i] > 0.0)) feasible = false;
          margin = std::min(margin, m.wheel_sdist[i] / p.eps_dist);
        }
      }
      try {
        s = integrate_step<SrbModel>(s, u[t], pr.hm, pr.vp, pr.tp, p.dt_int, p.scheme == TMPC_SCHEME_RK4 ? Scheme::kRk4 : Scheme::kEuler);
      } catch (const std::domain_error&) {  // gimbal guard dynamics.hpp:311-312
        diverged = true;
        break;
      }
      ++n;
      bool fin = true;
      for (double v : s.as_array()) fin = fin && std::isfinite(v);
      if (!fin) {  // integrate() would throw IntegrationError, dynamics.hpp:491-492
        diverged = true;
        break;
      }
    }
  }
  CandOut o;
  o.substeps = n;
  o.jrun = J;
  if (diverged) {
    o.cost = inf;
    o.flags = TMPC_FLAG_DIVERGED;
    o.margin = -inf;
    return o;
  }
  const double dx = s.x - p.goal_x, dy = s.y - p.goal_y;
  o.cost = J + p.w_g * std::sqrt(dx * dx + dy * dy);
  o.flags = static_cast<uint8_t>((feasible ? TMPC_FLAG_FEASIBLE : 0) | (goal ? TMPC_FLAG_GOAL : 0));
  o.margin = static_cast<float>(margin);
  return o;
}

// The EST formulation (model = TMPC_MODEL_EST): the reference EstModel
// (est_derivative dynamics.hpp:230-275 over est_plane_attitude 213-219), the
// lateral-acceleration rollover constraint (lateral_accel_violation
// constraints.hpp:62-65, eps = aby_epsilon 78-80, a_by from EstDiagnostics
// 265) in place of the ESM, the same distance constraints and cost.  The EST
// state lives in the SrbState slots x, y, psi, v_by, omega_bz, delta, v_bx.
CandOut rollout_est(const Problem& pr, const double* s0a, int64_t k) {
  const tmpc_params& p = *pr.p;
  const std::vector<Control> u = sample_controls(pr, k);
  EstState s{s0a[0], s0a[1], s0a[3], s0a[7], s0a[11], s0a[12], s0a[6]};
  const int S = static_cast<int>(std::lround(p.dt_zoh / p.dt_int));
  const double inf = std::numeric_limits<double>::infinity();
  double J = 0.0, margin = inf;
  bool feasible = true, diverged = false, goal = false;
  int64_t n = 0;
  for (int t = 0; t < p.n_steps && !goal && !diverged; ++t) {
    for (int q = 0; q < S; ++q) {
      const double dx = s.x - p.goal_x, dy = s.y - p.goal_y;
      if (dx * dx + dy * dy <= p.goal_r * p.goal_r) {
        goal = true;
        break;
      }
      EstDiagnostics dg;
      (void)est_derivative(s, u[t], pr.hm, pr.vp, pr.tp, &dg);
      ConstraintMeasures m;
      const auto fp = wheel_footprint(s.x, s.y, s.psi, pr.vp);
      for (int i = 0; i < 4; ++i) m.wheel_sdist[i] = pr.sd.value_at(fp[i].x(), fp[i].y());
      const double pi_aby = lateral_accel_violation(dg.a_by, dg.g_by, pr.cc);
      m.rollover_pi = pi_aby;
      m.rollover_epsilon = aby_epsilon(pr.cc);
      const double L = p.w_t + p.w_c * u[t].delta_rate * u[t].delta_rate +
                       constraint_set_cost(m, pr.cc);
      J += p.dt_int * L;
      if (pr.cc.enable_rollover) {
        if (!(pi_aby < 0.0)) feasible = false;
        margin = std::min(margin, -pi_aby / p.a_by_bar);
      }
      if (pr.cc.enable_dist && pr.sd.has_features) {
        for (int i = 0; i < 4; ++i) {
          if (!(m.wheel_sdist[i] > 0.0)) feasible = false;
          margin = std::min(margin, m.wheel_sdist[i] / p.eps_dist);
        }
      }
      s = integrate_step<EstModel>(s, u[t], pr.hm, pr.vp, pr.tp, p.dt_int, p.scheme == TMPC_SCHEME_RK4 ? Scheme::kRk4 : Scheme::kEuler);
      ++n;
      bool fin = true;
      for (double v : s.as_array()) fin = fin && std::isfinite(v);
      if (!fin) {
        diverged = true;
        break;
      }
    }
  }
  CandOut o;
  o.substeps = n;
  o.jrun = J;
  if (diverged) {
    o.cost = inf;
    o.flags = TMPC_FLAG_DIVERGED;
    o.margin = -inf;
    return o;
  }
  const double dx = s.x - p.goal_x, dy = s.y - p.goal_y;
  o.cost = J + p.w_g * std::sqrt(dx * dx + dy * dy);
  o.flags = static_cast<uint8_t>((feasible ? TMPC_FLAG_FEASIBLE : 0) | (goal ? TMPC_FLAG_GOAL : 0));
  o.margin = static_cast<float>(margin);
  return o;
}

}  // namespace

extern "C" {

// solve_ocp over candidates [k_begin, k_begin+k_count):
// per-candidate outputs + arg-min with the selection order of p->selection.
// Returns 0 ok, 1 all diverged, 2 config error (message in err).
int ref_solve(const tmpc_params* p, const tmpc_sampling* smp, const tmpc_terrain* t,
              const double* s0, double* cost, uint8_t* flags, float* margin,
              int64_t* substeps, int n_threads, tmpc_result* res, char* err, size_t err_len) {
  try {
    const Problem pr = make_problem(p, smp, t);
    const int64_t K = smp->k_count;
    std::atomic<int64_t> next{0};
    // TMPC_REF_PIN=1 (bench.py's CPU baseline): worker i runs on the i-th CPU
    // of the process's affinity set (one thread per physical core)
    const bool pin = std::getenv("TMPC_REF_PIN") && std::atoi(std::getenv("TMPC_REF_PIN")) != 0;
    cpu_set_t allowed;
    CPU_ZERO(&allowed);
    if (pin) sched_getaffinity(0, sizeof(allowed), &allowed);
    auto worker = [&](int idx) {
      if (pin) {
        int seen = 0;
        for (int cpu = 0; cpu < CPU_SETSIZE; ++cpu)
          if (CPU_ISSET(cpu, &allowed) && seen++ == idx) {
            cpu_set_t one;
            CPU_ZERO(&one);
            CPU_SET(cpu, &one);
            pthread_setaffinity_np(pthread_self(), sizeof(one), &one);
            break;
          }
      }
      for (;;) {
        const int64_t i0 = next.fetch_add(16);
        if (i0 >= K) break;
        const int64_t i1 = std::min<int64_t>(K, i0 + 16);
        for (int64_t i = i0; i < i1; ++i) {
          const CandOut o = p->model == TMPC_MODEL_EST ? rollout_est(pr, s0, smp->k_begin + i)
                                                       : rollout(pr, s0, smp->k_begin + i);
          if (cost) cost[i] = o.cost;
          if (flags) flags[i] = o.flags;
          if (margin) margin[i] = o.margin;
          if (substeps) substeps[i] = o.substeps;
        }
      }
    };
    const int nt = std::max(1, n_threads);
    std::vector<std::thread> th;
    for (int i = 1; i < nt; ++i) th.emplace_back(worker, i);
    worker(0);
    for (auto& x : th) x.join();
    if (pin) pthread_setaffinity_np(pthread_self(), sizeof(allowed), &allowed);
    if (res && cost && flags) {
      std::memset(res, 0, sizeof(*res));
      int64_t best = -1;
      double sum = 0.0, mn = std::numeric_limits<double>::infinity();
      int64_t nfin = 0;
      for (int64_t i = 0; i < K; ++i) {
        const bool inf_i = (flags[i] & TMPC_FLAG_FEASIBLE) == 0 && p->selection == TMPC_SELECT_FEASIBLE_FIRST;
        if (flags[i] & TMPC_FLAG_FEASIBLE) res->n_feasible++;
        if (flags[i] & TMPC_FLAG_DIVERGED) res->n_diverged++;
        if (flags[i] & TMPC_FLAG_GOAL) res->n_goal++;
        if (std::isfinite(cost[i])) {
          sum += cost[i];
          ++nfin;
          mn = std::min(mn, cost[i]);
        }
        if (best < 0) {
          best = i;
          continue;
        }
        const bool inf_b = (flags[best] & TMPC_FLAG_FEASIBLE) == 0 && p->selection == TMPC_SELECT_FEASIBLE_FIRST;
        if (inf_i < inf_b || (inf_i == inf_b && cost[i] < cost[best])) best = i;
      }
      res->n_candidates = K;
      res->best_index = smp->k_begin + best;
      res->best_cost = cost[best];
      res->best_feasible = (flags[best] & TMPC_FLAG_FEASIBLE) ? 1 : 0;
      res->best_margin = margin ? margin[best] : 0.0f;
      res->min_cost = mn;
      res->mean_cost = nfin ? sum / nfin : std::numeric_limits<double>::infinity();
      if (substeps)
        for (int64_t i = 0; i < K; ++i) res->substeps_executed += substeps[i];
      if (res->n_diverged == K) {
        std::snprintf(err, err_len, "solve_ocp: all %lld rollouts diverged", (long long)K);
        return 1;
      }
    }
    return 0;
  } catch (const ConfigError& e) {
    std::snprintf(err, err_len, "%s", e.what());
    return 2;
  } catch (const std::exception& e) {
    std::snprintf(err, err_len, "%s", e.what());
    return 3;
  }
}

// Candidates at arbitrary GLOBAL indices idx[0..n) (the c5 shadow check of
// bench.py: a strided sample plus the device's best few, every cycle, on the
// same plant state; the conditioning spread of the parity tests).  Outputs
// per listed candidate; substeps / jrun (the running cost when the rollout
// stopped, defined for diverged candidates too) may be NULL.  Returns 0 / 2 / 3.
int ref_solve_indices(const tmpc_params* p, const tmpc_sampling* smp, const tmpc_terrain* t,
                      const double* s0, const int64_t* idx, int64_t n, double* cost,
                      uint8_t* flags, float* margin, int64_t* substeps, double* jrun,
                      int n_threads, char* err, size_t err_len) {
  try {
    const Problem pr = make_problem(p, smp, t);
    std::atomic<int64_t> next{0};
    auto worker = [&]() {
      for (;;) {
        const int64_t i = next.fetch_add(1);
        if (i >= n) break;
        const CandOut o = p->model == TMPC_MODEL_EST ? rollout_est(pr, s0, idx[i])
                                                     : rollout(pr, s0, idx[i]);
        cost[i] = o.cost;
        flags[i] = o.flags;
        margin[i] = o.margin;
        if (substeps) substeps[i] = o.substeps;
        if (jrun) jrun[i] = o.jrun;
      }
    };
    std::vector<std::thread> th;
    for (int i = 1; i < std::max(1, n_threads); ++i) th.emplace_back(worker);
    worker();
    for (auto& x : th) x.join();
    return 0;
  } catch (const ConfigError& e) {
    std::snprintf(err, err_len, "%s", e.what());
    return 2;
  } catch (const std::exception& e) {
    std::snprintf(err, err_len, "%s", e.what());
    return 3;
  }
}

// open_loop_errors over the reference
// functions: per trajectory the plant = integrate_step<SrbModel> with kRk4 at
// plant_dt (the harness plant) and the model =
// integrate_step<SrbModel | EstModel> with p->scheme at dt_int, from the same
// initial state under the same ZOH controls; the time averages over the
// horizon of |(x^, y^) - (x, y)| and |U^_ESM - U_ESM| sampled at every model
// substep start (EST: esm of est_plane_attitude, SPEC.md design decision).
// The plant integrates over plant_t (its LOD) when given, else over t.
// flags: 1 model diverged, 2 plant diverged (errors NaN).
int ref_open_loop_errors(const tmpc_params* p, const tmpc_terrain* t, const tmpc_terrain* plant_t,
                         int model, const double* s0, const double* ctrl, int64_t n,
                         double plant_dt, double* loc, double* esm_err, uint8_t* flags,
                         int n_threads, char* err, size_t err_len) {
  const tmpc_sampling smp{};
  try {
    const Problem pr = make_problem(p, &smp, t);
    const Problem prp = make_problem(p, &smp, plant_t ? plant_t : t);  // the plant's LOD
    const int S = static_cast<int>(std::lround(p->dt_zoh / p->dt_int));
    const int sub = static_cast<int>(std::lround(p->dt_int / plant_dt));
    const Scheme scheme = p->scheme == TMPC_SCHEME_RK4 ? Scheme::kRk4 : Scheme::kEuler;
    const double T = p->n_steps * S * p->dt_int;
    std::atomic<int64_t> next{0};
    auto worker = [&]() {
      for (;;) {
        const int64_t i = next.fetch_add(1);
        if (i >= n) break;
        std::array<double, SrbState::kDim> a{};
        for (int j = 0; j < SrbState::kDim; ++j) a[j] = s0[13 * i + j];
        SrbState pl = SrbState::from_array(a), ms = pl;
        EstState es{a[0], a[1], a[3], a[7], a[11], a[12], a[6]};
        double L = 0.0, E = 0.0;
        uint8_t fl = 0;
        for (int j = 0; j < p->n_steps && !fl; ++j) {
          const Control u{ctrl[2 * (i * p->n_steps + j)], ctrl[2 * (i * p->n_steps + j) + 1]};
          for (int q = 0; q < S && !fl; ++q) {
            double mx, my, mU;
            if (model == TMPC_MODEL_EST) {
              const PlaneAttitude att = est_plane_attitude(pr.hm, es.x, es.y);
              mx = es.x;
              my = es.y;
              mU = esm(att.phi, att.theta, pr.vp);
            } else {
              mx = ms.x;
              my = ms.y;
              mU = esm(ms.phi, ms.theta, pr.vp);
            }
            L += p->dt_int * std::hypot(mx - pl.x, my - pl.y);
            E += p->dt_int * std::fabs(mU - esm(pl.phi, pl.theta, pr.vp));
            try {
              if (model == TMPC_MODEL_EST) {
                es = integrate_step<EstModel>(es, u, pr.hm, pr.vp, pr.tp, p->dt_int, scheme);
                for (double v : es.as_array()) if (!std::isfinite(v)) fl |= 1;
              } else {
                ms = integrate_step<SrbModel>(ms, u, pr.hm, pr.vp, pr.tp, p->dt_int, scheme);
                for (double v : ms.as_array()) if (!std::isfinite(v)) fl |= 1;
              }
            } catch (const std::domain_error&) {
              fl |= 1;
            }
            for (int r = 0; r < sub && !(fl & 2); ++r) {
              try {
                pl = integrate_step<SrbModel>(pl, u, prp.hm, pr.vp, pr.tp, plant_dt, Scheme::kRk4);
                for (double v : pl.as_array()) if (!std::isfinite(v)) fl |= 2;
              } catch (const std::domain_error&) {
                fl |= 2;
              }
            }
          }
        }
        const double nan = std::numeric_limits<double>::quiet_NaN();
        loc[i] = fl ? nan : L / T;
        esm_err[i] = fl ? nan : E / T;
        flags[i] = fl;
      }
    };
    std::vector<std::thread> th;
    for (int i = 1; i < std::max(1, n_threads); ++i) th.emplace_back(worker);
    worker();
    for (auto& x : th) x.join();
    return 0;
  } catch (const ConfigError& e) {
    std::snprintf(err, err_len, "%s", e.what());
    return 2;
  } catch (const std::exception& e) {
    std::snprintf(err, err_len, "%s", e.what());
    return 3;
  }
}

// The control sequence ref_solve uses for global candidate k (n_steps x 2).
int ref_sample_controls(const tmpc_params* p, const tmpc_sampling* smp, int64_t k, double* out) {
  Problem pr;
  pr.p = p;
  pr.smp = smp;
  const auto u = sample_controls(pr, k);
  for (int t = 0; t < p->n_steps; ++t) {
    out[2 * t] = u[t].delta_rate;
    out[2 * t + 1] = u[t].v_bx_rate;
  }
  return 0;
}

// srb_derivative (dynamics.hpp:308-398) for KATs; returns 1 on the gimbal
// guard.  diag (nullable): chi[4], chi_dot[4], f_z[4], f_y[4], slip[4], g_b[3].
int ref_srb_derivative(const tmpc_params* p, const tmpc_terrain* t, const double* s13,
                       const double* u2, double* d13, double* diag) {
  const tmpc_sampling smp{};
  try {
    const Problem pr = make_problem(p, &smp, t);
    std::array<double, SrbState::kDim> a{};
    for (int i = 0; i < SrbState::kDim; ++i) a[i] = s13[i];
    const Control u{u2[0], u2[1]};
    SrbDiagnostics dg;
    const SrbState d = srb_derivative(SrbState::from_array(a), u, pr.hm, pr.vp, pr.tp, &dg);
    const auto da = d.as_array();
    for (int i = 0; i < SrbState::kDim; ++i) d13[i] = da[i];
    if (diag) {
      for (int i = 0; i < 4; ++i) {
        diag[i] = dg.chi[i];
        diag[4 + i] = dg.chi_dot[i];
        diag[8 + i] = dg.f_z[i];
        diag[12 + i] = dg.f_y[i];
        diag[16 + i] = dg.slip_angle[i];
      }
      diag[20] = dg.g_b.x();
      diag[21] = dg.g_b.y();
      diag[22] = dg.g_b.z();
    }
    return 0;
  } catch (const std::domain_error&) {
    return 1;
  } catch (const std::exception&) {
    return 2;
  }
}

// One integrate_step<SrbModel> (dynamics.hpp:446-468); scheme 0 Euler, 1 RK4.
int ref_integrate_step(const tmpc_params* p, const tmpc_terrain* t, const double* s13,
                       const double* u2, double dt, int scheme, double* out13) {
  const tmpc_sampling smp{};
  try {
    const Problem pr = make_problem(p, &smp, t);
    std::array<double, SrbState::kDim> a{};
    for (int i = 0; i < SrbState::kDim; ++i) a[i] = s13[i];
    const Control u{u2[0], u2[1]};
    const SrbState o = integrate_step<SrbModel>(SrbState::from_array(a), u, pr.hm, pr.vp, pr.tp,
                                                dt, scheme ? Scheme::kRk4 : Scheme::kEuler);
    const auto oa = o.as_array();
    for (int i = 0; i < SrbState::kDim; ++i) out13[i] = oa[i];
    return 0;
  } catch (const std::domain_error&) {
    return 1;
  } catch (const std::exception&) {
    return 2;
  }
}

// height_at / gradient_at / SignedDistanceMap::value_at (terrain.hpp:79-93,235-238)
// at n points.  out: n x 4 (h, fx, fy, sd).
int ref_terrain_query(const tmpc_terrain* t, const double* xy, int64_t n, double* out) {
  Heightmap hm;
  hm.grid = GridSpec{t->origin_x, t->origin_y, t->resolution, t->nx, t->ny};
  hm.heights.assign(t->heights, t->heights + static_cast<size_t>(t->nx) * t->ny);
  SignedDistanceMap sd;
  sd.grid = hm.grid;
  sd.has_features = t->sdist != nullptr;
  if (t->sdist) sd.values.assign(t->sdist, t->sdist + static_cast<size_t>(t->nx) * t->ny);
  for (int64_t i = 0; i < n; ++i) {
    const double x = xy[2 * i], y = xy[2 * i + 1];
    const Slope s = gradient_at(hm, x, y);
    out[4 * i] = height_at(hm, x, y);
    out[4 * i + 1] = s.fx;
    out[4 * i + 2] = s.fy;
    out[4 * i + 3] = sd.value_at(x, y);
  }
  return 0;
}

// build_sdist_map (terrain.hpp:241-260) over polygon perimeters.
// poly_off: n_poly+1 offsets into verts (x,y pairs); kinds: 0 obstacle, 1 path boundary.
int ref_build_sdist_map(int nx, int ny, double ox, double oy, double res, int n_poly,
                        const int* poly_off, const double* verts, const int* kinds,
                        double* out) {
  try {
    std::vector<Perimeter> per(n_poly);
    for (int k = 0; k < n_poly; ++k) {
      per[k].kind = kinds[k] ? PerimeterKind::kPathBoundary : PerimeterKind::kObstacle;
      for (int v = poly_off[k]; v < poly_off[k + 1]; ++v)
        per[k].vertices.emplace_back(verts[2 * v], verts[2 * v + 1]);
      per[k].validate();
    }
    const SignedDistanceMap m = build_sdist_map(GridSpec{ox, oy, res, nx, ny}, per);
    std::copy(m.values.begin(), m.values.end(), out);
    return 0;
  } catch (const std::exception&) {
    return 2;
  }
}

// gaussian_smooth (terrain.hpp:102-138) of a heightmap; 2 on ConfigError.
int ref_gaussian_smooth(const tmpc_terrain* t, double sigma_m, double* out) {
  try {
    Heightmap hm;
    hm.grid = GridSpec{t->origin_x, t->origin_y, t->resolution, t->nx, t->ny};
    hm.heights.assign(t->heights, t->heights + static_cast<size_t>(t->nx) * t->ny);
    const Heightmap s = gaussian_smooth(hm, sigma_m);
    std::copy(s.heights.begin(), s.heights.end(), out);
    return 0;
  } catch (const std::exception&) {
    return 2;
  }
}

// Scalar KAT hooks.
double ref_esm(const tmpc_params* p, double phi, double theta) {
  VehicleParams vp;
  vp.M = p->M; vp.e = p->e; vp.h = p->h; vp.R = p->R; vp.g = p->g;
  return esm(phi, theta, vp);
}
double ref_tire_lateral_force(double alpha, double f_z, double C, double mu) {
  TireParams tp;
  tp.C = C;
  tp.mu = mu;
  return tire_lateral_force(alpha, f_z, tp);
}
double ref_soft_cost_rate(double pi, double eps, double sigma) {
  return soft_cost_rate(pi, SoftConstraintParams{eps, sigma});
}
uint64_t ref_substream(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) {
  return substream(seed, a, b, c);
}
// Draw j (0-based) of RngStream(seed_state) via the sequential API.
uint64_t ref_rng_draw(uint64_t stream_seed, int64_t j) {
  RngStream r(stream_seed);
  uint64_t v = 0;
  for (int64_t i = 0; i <= j; ++i) v = r.next_u64();
  return v;
}

}  // extern "C"
