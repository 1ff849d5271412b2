// Host side of libtmpc_b200: the C ABI (include/tmpc_b200.h), parameter
// validation mirroring the reference validate() methods, the terrain store
// upload (padded node fields, one replica per GPU), the
// per-cycle launch (a CUDA graph per GPU, replayed with new arguments), and
// the cross-GPU arg-min: per-GPU reduction records folded on
// the host in device / rank order, gathered across processes with one
// ncclAllGather under a watchdog.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvtx3/nvToolsExt.h>
#include <time.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "launch.cuh"
#include "nccl.h"
#include "rollout.cuh"
#include "tmpc_b200.h"
#include "tmpc_common.h"

namespace tmpcb {
cudaError_t launch_cycle(const KParams& P, const TerrainDev& td, const double* warm, double* cost,
                         uint8_t* flags, float* margin, DevStats* st, int lanes,
                         cudaStream_t stream);
cudaError_t reset_stats(DevStats* st, cudaStream_t stream);
int pick_lanes(int64_t k, int sms);
size_t order_scratch_bytes(int64_t n);
cudaError_t configure_rollout_f32();
cudaError_t configure_rollout_est_f32();
cudaError_t configure_rollout_rk4_f32();
size_t order_hist_bytes();
cudaError_t launch_order(const KParams& P, const double* warm, void* scratch,
                         const int32_t** order_out, cudaStream_t stream);
cudaError_t launch_open_loop(const KParams& P, const TerrainDev& td, const TerrainDev& tdp,
                             int model, const double* s0, const double* ctrl, int64_t n,
                             double plant_dt, int plant_sub, double* loc, double* esm,
                             uint8_t* flags, cudaStream_t stream);

std::vector<LaunchRec>*& launch_recorder() {
  static thread_local std::vector<LaunchRec>* rec = nullptr;
  return rec;
}
}  // namespace tmpcb

using namespace tmpcb;

// The public record is the device block plus the shard: same layout.
static_assert(sizeof(tmpc_rank_record) == sizeof(RankRecord), "record layout");
static_assert(offsetof(tmpc_rank_record, key_hi) == offsetof(DevStats, key_hi), "record layout");
static_assert(offsetof(tmpc_rank_record, cost_limb) == offsetof(DevStats, cost_limb), "record layout");
static_assert(offsetof(tmpc_rank_record, best_flags) == offsetof(DevStats, best_flags), "record layout");
static_assert(offsetof(tmpc_rank_record, k_begin) == offsetof(RankRecord, k_begin), "record layout");

namespace {

constexpr double kPi = 3.14159265358979323846;
constexpr double kGimbalMargin = 1e-3;  // dynamics.hpp:16

thread_local std::string g_last_error;

// ---- NCCL, loaded lazily (only multi-process contexts need it) ------------
struct Nccl {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRankConfig)(ncclComm_t*, int, ncclUniqueId, int, ncclConfig_t*) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool load(std::string& err) {
    if (h) return true;
    const char* cands[] = {
        "libnccl.so.2",
        "/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/lib/libnccl.so.2"};
    for (const char* c : cands)
      if ((h = dlopen(c, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!h) {
      err = "NCCL: cannot dlopen libnccl.so.2";
      return false;
    }
    const auto sym = [&](auto& f, const char* n) { f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(h, n)); };
    sym(GetUniqueId, "ncclGetUniqueId");
    sym(CommInitRankConfig, "ncclCommInitRankConfig");
    sym(AllGather, "ncclAllGather");
    sym(CommDestroy, "ncclCommDestroy");
    sym(CommAbort, "ncclCommAbort");
    sym(CommGetAsyncError, "ncclCommGetAsyncError");
    sym(GetErrorString, "ncclGetErrorString");
    if (!GetUniqueId || !CommInitRankConfig || !AllGather || !CommDestroy || !CommAbort ||
        !CommGetAsyncError || !GetErrorString) {
      err = "NCCL: missing symbols";
      return false;
    }
    return true;
  }
};
Nccl g_nccl;

// NVTX range (tracing): tmpc_stage / tmpc_launch / tmpc_finish
struct Range {
  explicit Range(const char* n) { nvtxRangePushA(n); }
  ~Range() { nvtxRangePop(); }
};

}  // namespace

// One cycle's kernels on one GPU as a CUDA graph (launch.cuh records them).
struct CycleGraph {
  std::vector<LaunchRec> recs;  // the launches the exec was built from
  std::vector<cudaGraphNode_t> nodes;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  void reset() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    exec = nullptr;
    graph = nullptr;
    nodes.clear();
    recs.clear();
  }
};

// One GPU of a context: its stream, terrain replica, output buffers and
// reduction record.  Several slots may name the same ordinal.
struct DevSlot {
  int device = 0;
  int sms = 148;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  void* d_hg = nullptr;
  void* d_sd = nullptr;
  size_t terrain_bytes = 0;
  TerrainDev td{};
  cudaTextureObject_t sd_tex = 0, hq_tex = 0;  // texture views of the fp32 records
  double* d_warm = nullptr;
  double* d_cost = nullptr;
  uint8_t* d_flags = nullptr;
  float* d_margin = nullptr;
  void* d_order = nullptr;       // ordering pass scratch (order.cu)
  RankRecord* d_rec = nullptr;   // this GPU's record (the kernels reduce into d_rec->s)
  RankRecord* d_gather = nullptr;  // world_size records (NCCL mode)
  RankRecord* h_rec = nullptr;   // pinned + mapped: max(1, world_size) records
  RankRecord* h_rec_dev = nullptr;  // its device address (one-process mode: the kernel writes it)
  bool stats_clean = false;      // d_rec->s is reset (one-process mode leaves it so)
  long long* h_shard = nullptr;  // pinned: this GPU's (k_begin, k_count)
  int64_t cap_k = 0;
  int cap_n = 0;
  KParams kp{};          // this GPU's shard of the staged cycle
  int lanes = 1;
  bool use_order = false;
  int kernels = 0;       // kernels the staged cycle launches here
  CycleGraph cg;
};

struct tmpc_ctx {
  tmpc_opts opts{};
  std::string err;
  std::vector<DevSlot> dev;
  bool have_params = false, have_terrain = false, staged = false, launched = false;
  tmpc_params p{};
  tmpc_sampling smp{};
  std::vector<double> warm_host;
  KParams kp{};  // shared part of every slot's KParams
  tmpc_terrain terr{};  // host copy of the last set_terrain
  std::vector<double> terr_h, terr_sd;
  int terr_pad = 0;  // replicated cells per side on the device
  bool l2_prefetch = true;  // TMPC_L2_PREFETCH=0 disables (A/B timing)
  bool graphs = true;
  // plant LOD of the open-loop analysis (tmpc_set_plant_terrain), fp64
  // padded fields on the first GPU; same grid as the terrain
  HG64* d_plant_hg = nullptr;
  tmpc_terrain plant_grid{};
  bool have_plant = false;
  ncclComm_t comm = nullptr;
  bool comm_dead = false;
  // peer-memory exchange (TMPC_EXCHANGE_PEER): this rank's mailbox, the
  // device array of every rank's mailbox (opened IPC mappings), the cycle
  // sequence number
  bool peer = false, peer_dead = false;
  Mailbox* d_mb = nullptr;
  Mailbox** d_peers = nullptr;
  std::vector<void*> opened;
  int xn = 0;
  unsigned long long xseq = 0;
  unsigned long long* h_err = nullptr;  // pinned
  int timeout_ms = 60000;
  std::vector<tmpc_rank_record> fold_buf;
};

namespace {

// One process, no collective: each GPU's record goes straight to the host
// (KParams::xn < 0), the cycle is one kernel per GPU.
bool one_process(const tmpc_ctx* c) { return !c->comm && !(c->peer && c->xn > 0); }

int fail(tmpc_ctx* ctx, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (ctx) ctx->err = buf;
  g_last_error = buf;
  return code;
}

#define CUDA_TRY(ctx, expr)                                                                   \
  do {                                                                                        \
    const cudaError_t e_ = (expr);                                                            \
    if (e_ != cudaSuccess)                                                                    \
      return fail(ctx, TMPC_ERR_RUNTIME, "CUDA error %s at %s:%d (%s)", cudaGetErrorString(e_), \
                  __FILE__, __LINE__, #expr);                                                 \
  } while (0)


int write_msg(char* msg, size_t len, const std::string& s) {
  if (msg && len) std::snprintf(msg, len, "%s", s.c_str());
  return TMPC_ERR_CONFIG;
}

// VehicleParams::validate (dynamics.hpp:38-47), TireParams::validate (54-57),
// ConstraintConfig::validate (constraints.hpp:51-57) + the planner's own
// preconditions (esm_nominal > 0 per App. A D10).
int validate_params(const tmpc_params* p, std::string& why) {
  if (!p) return why = "params: null", TMPC_ERR_CONFIG;
  const struct { double v; const char* n; } pos[] = {
      {p->M, "M"}, {p->J_xx, "J_xx"}, {p->J_yy, "J_yy"}, {p->J_zz, "J_zz"}, {p->L_f, "L_f"},
      {p->L_r, "L_r"}, {p->e, "e"}, {p->h, "h"}, {p->R, "R"}, {p->k_f, "k_f"}, {p->k_r, "k_r"},
      {p->b_f, "b_f"}, {p->b_r, "b_r"}, {p->delta_max, "delta_max"},
      {p->delta_rate_max, "delta_rate_max"}, {p->g, "g"}};
  for (const auto& q : pos)
    if (!(q.v > 0.0)) return why = std::string("vehicle: ") + q.n + " must be > 0", TMPC_ERR_CONFIG;
  if (p->delta_max >= kPi / 2) return why = "vehicle: delta_max must be < pi/2", TMPC_ERR_CONFIG;
  if (!(p->C > 0.0)) return why = "tire: C must be > 0", TMPC_ERR_CONFIG;
  if (!(p->mu > 0.0 && p->mu <= 2.0)) return why = "tire: mu must be in (0, 2]", TMPC_ERR_CONFIG;
  if (!(p->a_by_bar > 0.0)) return why = "constraints: a_by_bar must be > 0", TMPC_ERR_CONFIG;
  if (!(p->eps_dist > 0.0)) return why = "constraints: eps_dist must be > 0", TMPC_ERR_CONFIG;
  if (!(p->sigma > 0.0)) return why = "constraints: sigma must be > 0", TMPC_ERR_CONFIG;
  if (!(p->safety_factor > 0.0))
    return why = "constraints: safety_factor must be > 0", TMPC_ERR_CONFIG;
  if (!(p->esm_nominal > 0.0))
    return why = "constraints: esm_nominal must be > 0 (set it from esm_normalization)",
           TMPC_ERR_CONFIG;
  if (!(p->w_t >= 0.0 && p->w_c >= 0.0 && p->w_g >= 0.0))
    return why = "cost weights must be >= 0", TMPC_ERR_CONFIG;
  if (!(p->goal_r > 0.0)) return why = "goal: r_g must be > 0", TMPC_ERR_CONFIG;
  if (!std::isfinite(p->goal_x) || !std::isfinite(p->goal_y))
    return why = "goal: position must be finite", TMPC_ERR_CONFIG;
  if (p->n_steps < 1) return why = "planner: n_steps must be >= 1", TMPC_ERR_CONFIG;
  if (!(p->dt_int > 0.0) || !(p->dt_zoh > 0.0))
    return why = "planner: dt_int and dt_zoh must be > 0", TMPC_ERR_CONFIG;
  const int S = static_cast<int>(std::lround(p->dt_zoh / p->dt_int));
  if (S < 1 || std::fabs(S * p->dt_int - p->dt_zoh) > 1e-9)  // dynamics.hpp:477-481
    return why = "integrate: dt_int must divide the ZOH period", TMPC_ERR_CONFIG;
  if (p->selection != TMPC_SELECT_FEASIBLE_FIRST && p->selection != TMPC_SELECT_PLAIN)
    return why = "planner: unknown selection order", TMPC_ERR_CONFIG;
  if (p->model != TMPC_MODEL_SRB && p->model != TMPC_MODEL_EST)
    return why = "planner: unknown vehicle model", TMPC_ERR_CONFIG;
  if (p->scheme != TMPC_SCHEME_EULER && p->scheme != TMPC_SCHEME_RK4)
    return why = "planner: unknown integration scheme", TMPC_ERR_CONFIG;
  return TMPC_OK;
}

// Heightmap::validate (terrain.hpp:65-75) + SDF shape.
int validate_terrain(const tmpc_terrain* t, std::string& why) {
  if (!t || !t->heights) return why = "heightmap: null", TMPC_ERR_CONFIG;
  if (t->nx < 2 || t->ny < 2) return why = "heightmap: grid must be at least 2x2", TMPC_ERR_CONFIG;
  if (!(t->resolution > 0.0)) return why = "heightmap: resolution must be positive", TMPC_ERR_CONFIG;
  if (!std::isfinite(t->origin_x) || !std::isfinite(t->origin_y))
    return why = "heightmap: origin must be finite", TMPC_ERR_CONFIG;
  const size_t n = static_cast<size_t>(t->nx) * t->ny;
  for (size_t i = 0; i < n; ++i)
    if (!std::isfinite(t->heights[i])) return why = "heightmap: non-finite height", TMPC_ERR_CONFIG;
  if (t->sdist)
    for (size_t i = 0; i < n; ++i)
      if (std::isnan(t->sdist[i]) || std::isinf(t->sdist[i]))
        return why = "sdist: values must be finite when has_features", TMPC_ERR_CONFIG;
  return TMPC_OK;
}

int validate_sampling(const tmpc_params& p, const tmpc_sampling* s, std::string& why) {
  if (!s) return why = "sampling: null", TMPC_ERR_CONFIG;
  if (s->kind < TMPC_SAMPLE_UNIFORM || s->kind > TMPC_SAMPLE_WARM_GAUSS)
    return why = "sampling: unknown kind", TMPC_ERR_CONFIG;
  if (s->vdot_max < 0.0 || !std::isfinite(s->vdot_max))
    return why = "sampling: vdot_max must be >= 0", TMPC_ERR_CONFIG;
  if (s->kind == TMPC_SAMPLE_RANDOM_WALK && !(s->walk_step > 0.0))
    return why = "sampling: walk_step must be > 0", TMPC_ERR_CONFIG;
  if (s->kind == TMPC_SAMPLE_WARM_GAUSS && !(s->warm_sigma_frac >= 0.0))
    return why = "sampling: warm_sigma_frac must be >= 0", TMPC_ERR_CONFIG;
  if (s->k_count < 1) return why = "sampling: k_count must be >= 1", TMPC_ERR_CONFIG;
  if (s->k_begin < 0 || s->k_begin + s->k_count > 0x7FFFFFFFLL)
    return why = "sampling: global candidate index must fit 31 bits", TMPC_ERR_CONFIG;
  if (s->k_total != 0 && s->k_total < s->k_begin + s->k_count)
    return why = "sampling: k_total must cover [k_begin, k_begin + k_count) (or be 0)", TMPC_ERR_CONFIG;
  (void)p;
  return TMPC_OK;
}

template <typename T>
void fill_consts(KConsts<T>& k, const tmpc_params& p) {
  const double L = p.L_f + p.L_r;
  const double Kzz[2] = {p.M * p.L_r / L, p.M * p.L_f / L};  // dynamics.hpp:67-71
  k.g = static_cast<T>(p.g);
  k.half_M = static_cast<T>(0.5 * p.M);
  k.inv_M = static_cast<T>(1.0 / p.M);
  k.cJx = static_cast<T>(p.J_yy - p.J_zz);
  k.cJy = static_cast<T>(p.J_xx - p.J_zz);
  k.cJz = static_cast<T>(p.J_xx - p.J_yy);
  k.inv_Jxx = static_cast<T>(1.0 / p.J_xx);
  k.inv_Jyy = static_cast<T>(1.0 / p.J_yy);
  k.inv_Jzz = static_cast<T>(1.0 / p.J_zz);
  const double zo = -(p.h + p.R);
  const double rx[4] = {p.L_f, p.L_f, -p.L_r, -p.L_r};
  const double ry[4] = {p.e / 2, -p.e / 2, p.e / 2, -p.e / 2};
  for (int i = 0; i < 4; ++i) {
    k.rho[i][0] = static_cast<T>(rx[i]);
    k.rho[i][1] = static_cast<T>(ry[i]);
    k.rho[i][2] = static_cast<T>(zo);
    k.k_i[i] = static_cast<T>(i < 2 ? p.k_f : p.k_r);
    k.b_i[i] = static_cast<T>(i < 2 ? p.b_f : p.b_r);
    k.fs_i[i] = static_cast<T>(0.5 * p.g * Kzz[i < 2 ? 0 : 1]);
  }
  k.C = static_cast<T>(p.C);
  k.mu = static_cast<T>(p.mu);
  k.mu2 = static_cast<T>(p.mu * p.mu);
  k.delta_max = static_cast<T>(p.delta_max);
  k.vbx_floor = static_cast<T>(0.1);   // kVbxFloor, dynamics.hpp:15
  k.tau_floor = static_cast<T>(1e-6);  // dynamics.hpp:341
  const double r_bar = std::hypot(p.h + p.R, p.e / 2.0);  // constraints.hpp:17-18
  const double phi_bar = std::atan(2.0 * (p.h + p.R) / p.e);
  k.esm_r_bar = static_cast<T>(r_bar);
  k.esm_c_pb = static_cast<T>(std::cos(phi_bar));
  k.esm_s_pb = static_cast<T>(std::sin(phi_bar));
  k.esm_Mg = static_cast<T>(p.M * p.g);
  k.esm_phi_lim = static_cast<T>(kPi / 2.0 - phi_bar);
  k.inv_eps_esm = static_cast<T>(1.0 / (p.safety_factor * p.esm_nominal));
  k.inv_esm_nominal = static_cast<T>(1.0 / p.esm_nominal);
  k.sigma = static_cast<T>(p.sigma);
  k.inv_eps_dist = static_cast<T>(1.0 / p.eps_dist);
  k.dt = static_cast<T>(p.dt_int);
  k.kzzf = static_cast<T>(Kzz[0]);
  k.kzzr = static_cast<T>(Kzz[1]);
  k.kzx = static_cast<T>(p.M * (p.h + p.R) / L);
  k.L_f = static_cast<T>(p.L_f);
  k.L_r = static_cast<T>(p.L_r);
  k.a_by_bar = static_cast<T>(p.a_by_bar);
  k.inv_a_by_bar = static_cast<T>(1.0 / p.a_by_bar);
  k.inv_eps_aby = static_cast<T>(1.0 / (p.safety_factor * p.a_by_bar));
  k.esm_phi_bar = static_cast<T>(phi_bar);
}

void fill_kparams(KParams& k, const tmpc_params& p) {
  fill_consts(k.cf, p);
  fill_consts(k.cd, p);
  k.enable_dist = p.enable_dist != 0;
  k.enable_rollover = p.enable_rollover != 0;
  k.w_t = p.w_t;
  k.w_c = p.w_c;
  k.w_g = p.w_g;
  k.goal_x = p.goal_x;
  k.goal_y = p.goal_y;
  k.goal_r2 = p.goal_r * p.goal_r;
  k.dt = p.dt_int;
  k.n_steps = p.n_steps;
  k.S = static_cast<int>(std::lround(p.dt_zoh / p.dt_int));
  k.gimbal_lim = kPi / 2 - kGimbalMargin;
  k.selection = p.selection;
}

void free_buffers(DevSlot& d) {
  cudaFree(d.d_warm);
  cudaFree(d.d_cost);
  cudaFree(d.d_flags);
  cudaFree(d.d_margin);
  cudaFree(d.d_order);
  d.d_order = nullptr;
  d.d_warm = nullptr;
  d.d_cost = nullptr;
  d.d_flags = nullptr;
  d.d_margin = nullptr;
  d.cap_k = 0;
  d.cap_n = 0;
}

int ensure_capacity(tmpc_ctx* c, DevSlot& d, int64_t K, int N) {
  K = std::max<int64_t>(K, 1);
  N = std::max(N, 1);
  if (K <= d.cap_k && N <= d.cap_n) return TMPC_OK;
  const int64_t ck = std::max(K, d.cap_k);
  const int cn = std::max(N, d.cap_n);
  free_buffers(d);
  d.cg.reset();  // the graph's kernels point at the old buffers
  d.cap_k = ck;
  d.cap_n = cn;
  CUDA_TRY(c, cudaMalloc(&d.d_cost, sizeof(double) * d.cap_k));
  CUDA_TRY(c, cudaMalloc(&d.d_flags, d.cap_k));
  CUDA_TRY(c, cudaMalloc(&d.d_margin, sizeof(float) * d.cap_k));
  CUDA_TRY(c, cudaMalloc(&d.d_warm, sizeof(double) * 2 * d.cap_n));
  CUDA_TRY(c, cudaMalloc(&d.d_order, order_scratch_bytes(d.cap_k)));
  CUDA_TRY(c, cudaMemset(d.d_order, 0, order_hist_bytes()));
  return TMPC_OK;
}

// Fold records in order (tmpc_fold_records): the arg-min pair's MIN, integer
// sums, the MIN of the least cost, and the winner's fields from the record
// that owns it.  Pure integer / MIN arithmetic: the result is the same for
// any split of the candidates into records.
int fold(const tmpc_rank_record* r, int n, tmpc_result* out, std::string& why) {
  std::memset(out, 0, sizeof(*out));
  uint64_t khi = kKeyNone, klo = kKeyNone, minb = 0x7ff0000000000000ULL;
  uint64_t limb[3] = {0, 0, 0};
  int owner = -1;
  for (int i = 0; i < n; ++i) {
    const tmpc_rank_record& q = r[i];
    if (q.key_hi != kKeyNone && key_less(q.key_hi, q.key_lo, khi, klo)) {
      khi = q.key_hi;
      klo = q.key_lo;
      owner = i;
    }
    out->n_candidates += q.k_count;
    out->n_feasible += static_cast<int64_t>(q.n_feasible);
    out->n_diverged += static_cast<int64_t>(q.n_diverged);
    out->n_goal += static_cast<int64_t>(q.n_goal);
    out->substeps_executed += static_cast<int64_t>(q.substeps);
    minb = std::min<uint64_t>(minb, q.min_cost_bits);
    for (int j = 0; j < 3; ++j) limb[j] += q.cost_limb[j];
  }
  uint64_t n_fin = 0;
  for (int i = 0; i < n; ++i) n_fin += r[i].n_finite;
  out->min_cost = n_fin ? __builtin_bit_cast(double, minb) : std::numeric_limits<double>::infinity();
  out->mean_cost = n_fin ? limbs_value(limb) / static_cast<double>(n_fin)
                         : std::numeric_limits<double>::infinity();
  if (owner < 0) {
    out->best_index = -1;
    why = "solve_ocp: no candidates";
    return TMPC_ERR_NUMERIC;
  }
  out->best_index = static_cast<int64_t>(klo);
  out->best_cost = r[owner].best_cost;
  out->best_margin = r[owner].best_margin;
  out->best_feasible = (r[owner].best_flags & TMPC_FLAG_FEASIBLE) ? 1 : 0;
  if (out->n_diverged == out->n_candidates) {
    char b[96];
    std::snprintf(b, sizeof b, "solve_ocp: all %lld rollouts diverged",
                  static_cast<long long>(out->n_candidates));
    why = b;
    return TMPC_ERR_NUMERIC;
  }
  return TMPC_OK;
}

// Poll a non-blocking communicator until its pending operation (init or an
// enqueue) settles; ncclInProgress after timeout_ms.
ncclResult_t nccl_settle(tmpc_ctx* c) {
  const auto t0 = std::chrono::steady_clock::now();
  for (long spins = 0;; ++spins) {
    ncclResult_t ae = ncclInProgress;
    const ncclResult_t q = g_nccl.CommGetAsyncError(c->comm, &ae);
    if (q != ncclSuccess) return q;
    if (ae != ncclInProgress) return ae;
    const double ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (ms > c->timeout_ms) return ncclInProgress;
    if (spins > 1000) {
      const timespec ts{0, 50000};
      nanosleep(&ts, nullptr);
    }
  }
}

void destroy_slot(DevSlot& d) {
  cudaSetDevice(d.device);
  if (d.stream) cudaStreamSynchronize(d.stream);
  d.cg.reset();
  free_buffers(d);
  if (d.sd_tex) cudaDestroyTextureObject(d.sd_tex);
  if (d.hq_tex) cudaDestroyTextureObject(d.hq_tex);
  cudaFree(d.d_hg);
  cudaFree(d.d_sd);
  cudaFree(d.d_rec);
  cudaFree(d.d_gather);
  cudaFreeHost(d.h_rec);
  cudaFreeHost(d.h_shard);
  if (d.ev0) cudaEventDestroy(d.ev0);
  if (d.ev1) cudaEventDestroy(d.ev1);
  if (d.stream) cudaStreamDestroy(d.stream);
  d = DevSlot{};
}

}  // namespace

extern "C" {

const char* tmpc_last_error(const tmpc_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_last_error.c_str();
}

const char* tmpc_build_info(void) {
  return "tmpc_b200 " __DATE__ " sm_100a rollout_kernel(thread-per-candidate, fp32 math, fp64 "
         "position/cost accumulators; multi-GPU: per-GPU records folded in order)";
}

int tmpc_validate_params(const tmpc_params* p, char* msg, size_t msg_len) {
  std::string why;
  const int rc = validate_params(p, why);
  if (rc) write_msg(msg, msg_len, why);
  return rc;
}

int tmpc_validate_terrain(const tmpc_terrain* t, char* msg, size_t msg_len) {
  std::string why;
  const int rc = validate_terrain(t, why);
  if (rc) write_msg(msg, msg_len, why);
  return rc;
}

int tmpc_peer_export(tmpc_ctx* c, void* handle64) {
  if (!c || !handle64) return fail(c, TMPC_ERR_CONFIG, "peer_export: null argument");
  if (!c->peer) return fail(c, TMPC_ERR_CONFIG, "peer_export: the context's exchange is not PEER");
  CUDA_TRY(c, cudaSetDevice(c->dev[0].device));
  cudaIpcMemHandle_t h;
  CUDA_TRY(c, cudaIpcGetMemHandle(&h, c->d_mb));
  static_assert(sizeof(h) == 64, "CUDA IPC handle size");
  std::memcpy(handle64, &h, sizeof(h));
  return TMPC_OK;
}

int tmpc_peer_connect(tmpc_ctx* c, const void* handles, int32_t n) {
  if (!c || !handles) return fail(c, TMPC_ERR_CONFIG, "peer_connect: null argument");
  if (!c->peer) return fail(c, TMPC_ERR_CONFIG, "peer_connect: the context's exchange is not PEER");
  if (n != c->opts.world_size)
    return fail(c, TMPC_ERR_CONFIG, "peer_connect: %d handles for world_size %d", n,
                c->opts.world_size);
  CUDA_TRY(c, cudaSetDevice(c->dev[0].device));
  for (void* p : c->opened) cudaIpcCloseMemHandle(p);
  c->opened.clear();
  c->xn = 0;
  std::vector<Mailbox*> ptrs(n);
  for (int g = 0; g < n; ++g) {
    if (g == c->opts.rank) {  // our own mailbox (a process cannot open its own handle)
      ptrs[g] = c->d_mb;
      continue;
    }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, static_cast<const char*>(handles) + 64 * static_cast<size_t>(g), sizeof(h));
    void* p = nullptr;
    CUDA_TRY(c, cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    c->opened.push_back(p);
    ptrs[g] = static_cast<Mailbox*>(p);
    // every rank's kernel waits for the others' records: ranks sharing a GPU
    // could wait on launches that never run concurrently
    cudaPointerAttributes at{};
    CUDA_TRY(c, cudaPointerGetAttributes(&at, p));
    const char* allow = std::getenv("TMPC_PEER_ALLOW_SHARED_GPU");
    if (at.device == c->dev[0].device && !(allow && allow[0] == '1')) {
      for (void* q : c->opened) cudaIpcCloseMemHandle(q);
      c->opened.clear();
      return fail(c, TMPC_ERR_CONFIG,
                  "peer_connect: ranks %d and %d share GPU %d; the peer exchange needs one GPU per "
                  "rank (use one process with a devices list, or the NCCL exchange)",
                  c->opts.rank, g, at.device);
    }
  }
  CUDA_TRY(c, cudaMemcpy(c->d_peers, ptrs.data(), sizeof(Mailbox*) * n, cudaMemcpyHostToDevice));
  for (DevSlot& d : c->dev) d.cg.reset();
  c->xn = n;
  return TMPC_OK;
}

int tmpc_peer_inspect(tmpc_ctx* c, int32_t src, uint64_t seq, tmpc_rank_record* out,
                      uint64_t* published) {
  if (!c || !out || !published) return fail(c, TMPC_ERR_CONFIG, "peer_inspect: null argument");
  if (!c->peer) return fail(c, TMPC_ERR_CONFIG, "peer_inspect: the context's exchange is not PEER");
  if (src < 0 || src >= kMaxRanks || src >= c->opts.world_size)
    return fail(c, TMPC_ERR_CONFIG, "peer_inspect: rank %d out of range", src);
  CUDA_TRY(c, cudaSetDevice(c->dev[0].device));
  RankRecord r;
  CUDA_TRY(c, cudaMemcpy(&r, &c->d_mb->rec[seq & 1][src], sizeof(r), cudaMemcpyDeviceToHost));
  CUDA_TRY(c, cudaMemcpy(published, &c->d_mb->seq[src], sizeof(*published), cudaMemcpyDeviceToHost));
  std::memcpy(out, &r, sizeof(*out));
  return TMPC_OK;
}

int tmpc_nccl_unique_id(void* out128) {
  std::string err;
  if (!g_nccl.load(err)) return fail(nullptr, TMPC_ERR_RUNTIME, "%s", err.c_str());
  ncclUniqueId id;
  const ncclResult_t r = g_nccl.GetUniqueId(&id);
  if (r != ncclSuccess) return fail(nullptr, TMPC_ERR_RUNTIME, "ncclGetUniqueId failed");
  std::memcpy(out128, &id, sizeof(id));
  return TMPC_OK;
}

int tmpc_ctx_create(const tmpc_opts* opts, tmpc_ctx** out) {
  if (!opts || !out) return fail(nullptr, TMPC_ERR_CONFIG, "ctx_create: null argument");
  if (opts->world_size < 1 || opts->rank < 0 || opts->rank >= opts->world_size)
    return fail(nullptr, TMPC_ERR_CONFIG, "ctx_create: bad rank/world_size");
  if (opts->world_size > 1 && !opts->nccl_id && opts->exchange != TMPC_EXCHANGE_PEER)
    return fail(nullptr, TMPC_ERR_CONFIG,
                "ctx_create: world_size > 1 needs an NCCL unique id (or the PEER exchange)");
  if (opts->lanes != 0 && opts->lanes != 1 && opts->lanes != 2 && opts->lanes != 4)
    return fail(nullptr, TMPC_ERR_CONFIG, "ctx_create: lanes must be 0 (auto), 1, 2 or 4");
  if (opts->precision != TMPC_PRECISION_FP32 && opts->precision != TMPC_PRECISION_FP64)
    return fail(nullptr, TMPC_ERR_CONFIG, "ctx_create: unknown precision");
  if (opts->ordering != TMPC_ORDER_AUTO && opts->ordering != TMPC_ORDER_OFF &&
      opts->ordering != TMPC_ORDER_ON)
    return fail(nullptr, TMPC_ERR_CONFIG, "ctx_create: unknown ordering mode");
  if (opts->graphs != TMPC_GRAPHS_AUTO && opts->graphs != TMPC_GRAPHS_OFF)
    return fail(nullptr, TMPC_ERR_CONFIG, "ctx_create: unknown graphs mode");
  if (opts->n_devices < 0 || opts->n_devices > 64 || (opts->n_devices > 1 && !opts->devices))
    return fail(nullptr, TMPC_ERR_CONFIG, "ctx_create: n_devices > 1 needs a devices[] list (<= 64)");
  if (opts->timeout_ms < 0) return fail(nullptr, TMPC_ERR_CONFIG, "ctx_create: timeout_ms must be >= 0");
  if (opts->exchange != TMPC_EXCHANGE_NCCL && opts->exchange != TMPC_EXCHANGE_PEER)
    return fail(nullptr, TMPC_ERR_CONFIG, "ctx_create: unknown exchange mode");
  if (opts->exchange == TMPC_EXCHANGE_PEER && opts->world_size > kMaxRanks)
    return fail(nullptr, TMPC_ERR_CONFIG, "ctx_create: the peer exchange takes <= %d ranks", kMaxRanks);
  std::vector<int> ords;
  if (opts->devices && opts->n_devices > 0) ords.assign(opts->devices, opts->devices + opts->n_devices);
  else ords.push_back(opts->device);
  if (ords.size() > 1 && (opts->world_size > 1 || opts->nccl_id ||
                          opts->exchange == TMPC_EXCHANGE_PEER))
    return fail(nullptr, TMPC_ERR_CONFIG,
                "ctx_create: use either several devices in one process or one process per GPU "
                "(rank / world_size), not both");
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0)
    return fail(nullptr, TMPC_ERR_RUNTIME, "ctx_create: no CUDA device (%s)", cudaGetErrorString(e));
  for (int o : ords)
    if (o < 0 || o >= ndev)
      return fail(nullptr, TMPC_ERR_CONFIG, "ctx_create: device %d out of range (%d visible)", o, ndev);
  auto* c = new tmpc_ctx();
  c->opts = *opts;
  c->opts.nccl_id = nullptr;
  c->opts.devices = nullptr;
  c->graphs = opts->graphs == TMPC_GRAPHS_AUTO;
  if (const char* g = std::getenv("TMPC_GRAPHS")) c->graphs = c->graphs && std::atoi(g) != 0;
  c->timeout_ms = opts->timeout_ms ? opts->timeout_ms : 60000;
  auto bail = [&](int rc) {
    g_last_error = c->err;
    tmpc_ctx_destroy(c);
    return rc;
  };
  if (const char* ev = std::getenv("TMPC_L2_PREFETCH")) c->l2_prefetch = std::atoi(ev) != 0;
  const int nrec = std::max(1, opts->world_size);
  c->dev.resize(ords.size());
  for (size_t i = 0; i < ords.size(); ++i) {
    DevSlot& d = c->dev[i];
    d.device = ords[i];
    if (cudaSetDevice(d.device) != cudaSuccess)
      return bail(fail(c, TMPC_ERR_RUNTIME, "cudaSetDevice(%d) failed", d.device));
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, d.device);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, d.device);
    cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, d.device);
    if (major != 10 || minor != 0)
      return bail(fail(c, TMPC_ERR_RUNTIME, "ctx_create: built for sm_100a, device %d is sm_%d%d",
                       d.device, major, minor));
    if (configure_rollout_f32() != cudaSuccess || configure_rollout_est_f32() != cudaSuccess ||
        configure_rollout_rk4_f32() != cudaSuccess)
      return bail(fail(c, TMPC_ERR_RUNTIME, "ctx_create: kernel attribute setup failed"));
    if (cudaStreamCreateWithFlags(&d.stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreate(&d.ev0) != cudaSuccess || cudaEventCreate(&d.ev1) != cudaSuccess ||
        cudaMalloc(&d.d_rec, sizeof(RankRecord)) != cudaSuccess ||
        cudaMalloc(&d.d_gather, sizeof(RankRecord) * nrec) != cudaSuccess ||
        cudaHostAlloc(&d.h_rec, sizeof(RankRecord) * nrec,
                      cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess ||
        cudaHostGetDevicePointer(&d.h_rec_dev, d.h_rec, 0) != cudaSuccess ||
        cudaMallocHost(&d.h_shard, 2 * sizeof(long long)) != cudaSuccess)
      return bail(fail(c, TMPC_ERR_RUNTIME, "ctx_create: CUDA allocation failed"));
    if (opts->k_max > 0 || opts->n_steps_max > 0) {
      const int64_t share = (std::max<int64_t>(1, opts->k_max) + ords.size() - 1) / ords.size();
      const int rc = ensure_capacity(c, d, share, std::max(1, opts->n_steps_max));
      if (rc) return bail(rc);
    }
  }
  if (opts->exchange == TMPC_EXCHANGE_PEER) {
    c->peer = true;
    cudaSetDevice(c->dev[0].device);
    if (cudaMalloc(&c->d_mb, sizeof(Mailbox)) != cudaSuccess ||
        cudaMemset(c->d_mb, 0, sizeof(Mailbox)) != cudaSuccess ||
        cudaMalloc(&c->d_peers, sizeof(Mailbox*) * kMaxRanks) != cudaSuccess ||
        cudaMallocHost(&c->h_err, sizeof(unsigned long long)) != cudaSuccess ||
        cudaDeviceSynchronize() != cudaSuccess)
      return bail(fail(c, TMPC_ERR_RUNTIME, "ctx_create: mailbox allocation failed"));
  }
  // NCCL communicator for world_size > 1; with world_size == 1 an explicit id
  // still builds a 1-rank communicator (exercises the collective path on one GPU)
  if (!c->peer && (opts->world_size > 1 || opts->nccl_id)) {
    std::string err;
    if (!g_nccl.load(err)) return bail(fail(c, TMPC_ERR_RUNTIME, "%s", err.c_str()));
    cudaSetDevice(c->dev[0].device);
    ncclUniqueId id;
    std::memcpy(&id, opts->nccl_id, sizeof(id));
    // non-blocking communicator: the init (which needs every rank) and the
    // collectives are polled under the watchdog, so a rank that never shows
    // up fails this call after timeout_ms instead of hanging it
    ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
    cfg.blocking = 0;
    ncclResult_t r = g_nccl.CommInitRankConfig(&c->comm, opts->world_size, id, opts->rank, &cfg);
    if (r == ncclInProgress || r == ncclSuccess) r = nccl_settle(c);
    if (r != ncclSuccess) {
      if (c->comm) g_nccl.CommAbort(c->comm);
      c->comm = nullptr;
      return bail(fail(c, TMPC_ERR_RUNTIME, "ncclCommInitRankConfig: %s (rank %d of %d)",
                       r == ncclInProgress ? "timed out waiting for the other ranks"
                                           : g_nccl.GetErrorString(r),
                       opts->rank, opts->world_size));
    }
  }
  *out = c;
  return TMPC_OK;
}

void tmpc_ctx_destroy(tmpc_ctx* c) {
  if (!c) return;
  if (c->comm) {
    if (c->comm_dead) g_nccl.CommAbort(c->comm);
    else g_nccl.CommDestroy(c->comm);
  }
  if (c->d_plant_hg) {
    cudaSetDevice(c->dev[0].device);
    cudaFree(c->d_plant_hg);
  }
  if (c->peer) {
    cudaSetDevice(c->dev[0].device);
    if (!c->dev.empty() && c->dev[0].stream) cudaStreamSynchronize(c->dev[0].stream);
    for (void* p : c->opened) cudaIpcCloseMemHandle(p);
    cudaFree(c->d_mb);
    cudaFree(c->d_peers);
    cudaFreeHost(c->h_err);
  }
  for (DevSlot& d : c->dev) destroy_slot(d);
  delete c;
}

static int terrain_pad(const tmpc_ctx* c);
static int upload_terrain(tmpc_ctx* c, int Q);

int tmpc_set_params(tmpc_ctx* c, const tmpc_params* p) {
  if (!c) return fail(nullptr, TMPC_ERR_CONFIG, "null ctx");
  std::string why;
  if (validate_params(p, why)) return fail(c, TMPC_ERR_CONFIG, "%s", why.c_str());
  c->p = *p;
  fill_kparams(c->kp, *p);
  c->kp.precision = c->opts.precision;
  c->kp.model = p->model;
  c->kp.scheme = p->scheme;
  c->have_params = true;
  c->staged = false;
  // a vehicle reaching further than the terrain's pad covers: widen it
  if (c->have_terrain && terrain_pad(c) > c->terr_pad) return upload_terrain(c, terrain_pad(c));
  return TMPC_OK;
}

// Replicated cells per side of the fp32 terrain layout.  The SRB kernels
// clamp the CoM to the reference's window widened by m = E0 + 1 cells and add
// the wheel offsets unclamped, E0 = the largest planar wheel / footprint
// offset in cells (|R rho| <= |rho|, wheel_offsets dynamics.hpp:188-192), so
// every lookup stays inside [0, n + 2Q - 1] for Q = 2 E0 + 3.
static int terrain_pad(const tmpc_ctx* c) {
  if (c->opts.precision == TMPC_PRECISION_FP64) return 2;
  double rho = 3.0;  // m, before set_params: a generous vehicle
  if (c->have_params) {
    const tmpc_params& p = c->p;
    rho = std::sqrt(std::max(p.L_f, p.L_r) * std::max(p.L_f, p.L_r) + 0.25 * p.e * p.e +
                    (p.h + p.R) * (p.h + p.R));
  }
  const int e0 = static_cast<int>(std::ceil(rho * (1.0 + 1e-6) / c->terr.resolution)) + 1;
  return 2 * e0 + 3;
}

// One GPU's replica of the terrain store from the host-built records.
static int upload_slot(tmpc_ctx* c, DevSlot& d, const void* hg, size_t hg_bytes, const void* sd,
                       size_t sd_bytes, bool f64) {
  CUDA_TRY(c, cudaSetDevice(d.device));
  if (hg_bytes + sd_bytes != d.terrain_bytes) {
    cudaFree(d.d_hg);
    cudaFree(d.d_sd);
    d.d_hg = nullptr;
    d.d_sd = nullptr;
    d.terrain_bytes = 0;
    CUDA_TRY(c, cudaMalloc(&d.d_hg, hg_bytes));
    CUDA_TRY(c, cudaMalloc(&d.d_sd, sd_bytes));
    d.terrain_bytes = hg_bytes + sd_bytes;
  }
  d.cg.reset();  // the graph's kernels carry the old terrain pointers
  CUDA_TRY(c, cudaMemcpy(d.d_hg, hg, hg_bytes, cudaMemcpyHostToDevice));
  CUDA_TRY(c, cudaMemcpy(d.d_sd, sd, sd_bytes, cudaMemcpyHostToDevice));
  d.td = TerrainDev{};
  if (d.sd_tex) cudaDestroyTextureObject(d.sd_tex);
  if (d.hq_tex) cudaDestroyTextureObject(d.hq_tex);
  d.sd_tex = d.hq_tex = 0;
  if (f64) {
    d.td.hg64 = static_cast<const HG64*>(d.d_hg);
    d.td.sd64 = static_cast<const double*>(d.d_sd);
    return TMPC_OK;
  }
  d.td.hq32 = static_cast<const float4*>(d.d_hg);
  d.td.sdq32 = static_cast<const float4*>(d.d_sd);
  // the fp32 kernels also gather the records through the texture pipe: the
  // linear texture must cover them (set_terrain checked the width)
  cudaResourceDesc rd{};
  rd.resType = cudaResourceTypeLinear;
  rd.res.linear.devPtr = d.d_sd;
  rd.res.linear.desc = cudaCreateChannelDesc<float4>();
  rd.res.linear.sizeInBytes = sd_bytes;
  cudaTextureDesc tdsc{};
  tdsc.readMode = cudaReadModeElementType;
  tdsc.filterMode = cudaFilterModePoint;
  tdsc.addressMode[0] = cudaAddressModeClamp;
  CUDA_TRY(c, cudaCreateTextureObject(&d.sd_tex, &rd, &tdsc, nullptr));
  d.td.sd_tex = d.sd_tex;
  rd.res.linear.devPtr = d.d_hg;
  rd.res.linear.sizeInBytes = hg_bytes;
  CUDA_TRY(c, cudaCreateTextureObject(&d.hq_tex, &rd, &tdsc, nullptr));
  d.td.hq_tex = d.hq_tex;
  return TMPC_OK;
}

// Upload the cached host terrain (c->terr) with Q replicated cells per side
// to every GPU of the context.  fp64 mode: Q = 2 (the gradient stencil's
// reach).  fp32 mode: Q = terrain_pad() so that the SRB kernels clamp only the
// CoM per substep and look the wheel points up unclamped
// (rollout_srb_frame.cuh): beyond the reference's clamp window the replicated
// fields are constant along the clamped axis, so every record there has
// c1 = c3 = 0 (x) or c2 = c3 = 0 (y) exactly and returns the clamped lookup's
// value bit for bit.
// Sliding-window minimum of v[0], v[stride], ... (n values) over [i - w, i + w]
// (clamped to the array): monotone deque, O(n).
static void window_min(const double* v, double* out, int n, size_t stride, int w,
                       std::vector<int>& dq) {
  dq.assign(static_cast<size_t>(n), 0);
  int head = 0, tail = 0;
  for (int i = 0, r = 0; i < n; ++i) {
    for (; r < n && r <= i + w; ++r) {
      while (tail > head && v[dq[tail - 1] * stride] >= v[r * stride]) --tail;
      dq[tail++] = r;
    }
    while (dq[head] < i - w) ++head;
    out[i * stride] = v[dq[head] * stride];
  }
}

// Footprint clearance of every padded cell (the fp32 Euler kernel's skip
// test, rollout_f32.cu): the minimum SDF node over the square window of
// half-width e0 + kClearWindowMove + 2 cells around it, e0 = (Q - 3) / 2
// bounding every planar footprint offset in cells (terrain_pad; the pad only
// widens with set_params, so the window covers every vehicle the store
// serves).  A bilinear SDF value is a convex combination of its 4 nodes, so
// every footprint point of a CoM in the cell, or within kClearWindowMove
// cells of it, reads at least this minimum; the slack covers the fp32
// records' rounding (c0..c3 rounded once, 3 FMAs).  Rounded down to fp32.
static std::vector<float> footprint_clearance(const std::vector<double>& SD, int px, int py,
                                              int Q) {
  const int w = (Q - 3) / 2 + kClearWindowMove + 2;
  std::vector<double> a(SD.size()), b(SD.size());
  std::vector<int> dq;
  double vmax = 0.0;
  for (double v : SD) vmax = std::max(vmax, std::fabs(v));
  for (int j = 0; j < py; ++j)
    window_min(SD.data() + static_cast<size_t>(j) * px, a.data() + static_cast<size_t>(j) * px, px,
               1, w, dq);
  for (int i = 0; i < px; ++i) window_min(a.data() + i, b.data() + i, py, px, w, dq);
  const double slack = 1e-3 + 1e-5 * vmax;
  std::vector<float> out(SD.size());
  for (size_t o = 0; o < SD.size(); ++o) {
    const double v = b[o] - slack;
    float f = static_cast<float>(v);
    if (static_cast<double>(f) > v) f = std::nextafter(f, -INFINITY);
    out[o] = f;
  }
  return out;
}

static int upload_terrain(tmpc_ctx* c, int Q) {
  const tmpc_terrain* t = &c->terr;
  const int nx = t->nx, ny = t->ny, px = nx + 2 * Q, py = ny + 2 * Q;
  const size_t n = static_cast<size_t>(px) * py;
  const bool f64 = c->opts.precision == TMPC_PRECISION_FP64;
  if (!f64) {
    // the hq32 records (4 float4 texels per padded cell) are also read as a
    // 1-D linear texture, whose width the device bounds
    int maxw = 0;
    cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxTexture1DLinearWidth, c->dev[0].device);
    if (maxw > 0 && 4.0 * static_cast<double>(n) > static_cast<double>(maxw))
      return fail(c, TMPC_ERR_CONFIG,
                  "heightmap: %d x %d cells (+%d padding per side) exceed the fp32 terrain "
                  "store's texture limit of %d texels (4 per cell); use the fp64 precision mode "
                  "or a coarser grid", nx, ny, Q, maxw);
  }
  // padded fp64 copies (Q replicated cells per side) -> node fields
  std::vector<double> H(n);
  for (int j = 0; j < py; ++j) {
    const int sj = std::clamp(j - Q, 0, ny - 1);
    for (int i = 0; i < px; ++i)
      H[static_cast<size_t>(j) * px + i] = t->heights[static_cast<size_t>(sj) * nx + std::clamp(i - Q, 0, nx - 1)];
  }
  // node central differences of the padded field (gradient_at identity, §8a T2)
  std::vector<double> Dx(n, 0.0), Dy(n, 0.0), SD(n, 0.0);
  const double inv2r = 1.0 / (2.0 * t->resolution);
  for (int j = 0; j < py; ++j)
    for (int i = 0; i < px; ++i) {
      const size_t o = static_cast<size_t>(j) * px + i;
      if (i >= 1 && i < px - 1) Dx[o] = (H[o + 1] - H[o - 1]) * inv2r;
      if (j >= 1 && j < py - 1) Dy[o] = (H[o + px] - H[o - px]) * inv2r;
    }
  if (t->sdist)
    for (int j = 0; j < py; ++j) {
      const int sj = std::clamp(j - Q, 0, ny - 1);
      for (int i = 0; i < px; ++i)
        SD[static_cast<size_t>(j) * px + i] = t->sdist[static_cast<size_t>(sj) * nx + std::clamp(i - Q, 0, nx - 1)];
    }
  if (f64) {
    std::vector<HG64> hg(n);
    for (size_t o = 0; o < n; ++o) hg[o] = HG64{make_double2(H[o], Dx[o]), make_double2(Dy[o], 0.0)};
    for (DevSlot& d : c->dev) {
      const int rc = upload_slot(c, d, hg.data(), n * sizeof(HG64), SD.data(), n * sizeof(double), true);
      if (rc) return rc;
    }
  } else {
    // cell records: the bilinear coefficients {v00, v10 - v00, v01 - v00,
    // v11 - v10 - v01 + v00} (fp64, rounded once) of H, Dx, Dy (+ pad) and of
    // the SDF, for the cell whose lower-left node is o (lookups never start on
    // the last padded row/column: i0, j0 <= n+2)
    std::vector<float4> hq(4 * n), sdq(n);
    const std::vector<float> clear = t->sdist ? footprint_clearance(SD, px, py, Q)
                                              : std::vector<float>();
    for (int j = 0; j < py; ++j)
      for (int i = 0; i < px; ++i) {
        const size_t o = static_cast<size_t>(j) * px + i;
        const int i1 = std::min(i + 1, px - 1), j1 = std::min(j + 1, py - 1);
        const auto quad = [&](const std::vector<double>& v) {
          const auto at = [&](int a, int b) { return v[static_cast<size_t>(b) * px + a]; };
          const double v00 = at(i, j), v10 = at(i1, j), v01 = at(i, j1), v11 = at(i1, j1);
          return make_float4(static_cast<float>(v00), static_cast<float>(v10 - v00),
                             static_cast<float>(v01 - v00),
                             static_cast<float>((v11 - v10) - (v01 - v00)));
        };
        hq[4 * o + 0] = quad(H);
        hq[4 * o + 1] = quad(Dx);
        hq[4 * o + 2] = quad(Dy);
        hq[4 * o + 3] = make_float4(clear.empty() ? 0.f : clear[o], 0.f, 0.f, 0.f);
        sdq[o] = quad(SD);
      }
    for (DevSlot& d : c->dev) {
      const int rc = upload_slot(c, d, hq.data(), 4 * n * sizeof(float4), sdq.data(),
                                 n * sizeof(float4), false);
      if (rc) return rc;
    }
  }
  KParams& k = c->kp;
  const double inv = 1.0 / t->resolution;
  k.gx_scale = inv;
  k.gx_off = Q - t->origin_x * inv;
  k.gy_scale = inv;
  k.gy_off = Q - t->origin_y * inv;
  k.cf.inv_res = static_cast<float>(inv);
  k.cd.inv_res = inv;
  k.nx = nx;
  k.ny = ny;
  k.pitch = px;
  k.pad = Q;
  k.cell_bias = static_cast<unsigned>(-0x4B400000LL * (px + 1));
  k.last_cell = static_cast<unsigned>(n - 1);
  k.cmargin = Q == 2 ? 0 : (Q - 3) / 2 + 1;
  k.has_sdist = t->sdist != nullptr;
  c->terr_pad = Q;
  c->staged = false;
  return TMPC_OK;
}

int tmpc_set_terrain(tmpc_ctx* c, const tmpc_terrain* t) {
  if (!c) return fail(nullptr, TMPC_ERR_CONFIG, "null ctx");
  std::string why;
  if (validate_terrain(t, why)) return fail(c, TMPC_ERR_CONFIG, "%s", why.c_str());
  // the library copies (ownership): the host copy is kept so a
  // later set_params that needs a wider pad can re-upload
  const size_t n = static_cast<size_t>(t->nx) * t->ny;
  c->terr_h.assign(t->heights, t->heights + n);
  if (t->sdist) c->terr_sd.assign(t->sdist, t->sdist + n);
  else c->terr_sd.clear();
  c->terr = *t;
  c->terr.heights = c->terr_h.data();
  c->terr.sdist = t->sdist ? c->terr_sd.data() : nullptr;
  c->have_terrain = false;
  const int rc = upload_terrain(c, terrain_pad(c));
  if (rc) return rc;
  c->have_terrain = true;
  return TMPC_OK;
}

// The terrain window a cycle can reach, for the kernels' L2 bulk prefetch
// (rollout_dev.cuh l2_prefetch_terrain).  The body-x speed is exactly
// |v0| + integral of v_bx_rate (d v_bx = v_bx_rate in both models,
// dynamics.hpp:376 / 258), so the planar reach over the horizon T is at most
// (|v0| + vdot_max T) T plus the lateral velocity's share (10%) and the wheel
// offsets + bilinear footprint (3 m).  Capped at 48 MB of records (a third of
// the 126 MB L2), shrinking the window around the start.
void set_prefetch_window(tmpc_ctx* c, const double* s0, const tmpc_sampling& smp) {
  KParams& k = c->kp;
  k.pf_i0 = k.pf_j0 = 0;
  k.pf_i1 = k.pf_j1 = -1;
  if (!c->l2_prefetch) return;
  const double T = c->p.n_steps * c->p.dt_zoh;
  const double v = std::hypot(s0[6], s0[7]) + std::fabs(smp.vdot_max) * T;
  double reach = 1.1 * v * T + 3.0;
  const double cell_bytes = c->opts.precision == TMPC_PRECISION_FP64 ? 40.0 : 80.0;
  const double cap = 48.0 * (1 << 20);
  const double sx = k.gx_scale * reach, sy = k.gy_scale * reach;  // half-widths in cells
  const double bytes = (2 * sx + 2) * (2 * sy + 2) * cell_bytes;
  if (bytes > cap) reach *= std::sqrt(cap / bytes);
  const double gx = s0[0] * k.gx_scale + k.gx_off, gy = s0[1] * k.gy_scale + k.gy_off;
  const auto clampi = [](double v, int lo, int hi) {
    return static_cast<int>(std::max<double>(lo, std::min<double>(hi, std::floor(v))));
  };
  const int hi_x = k.pitch - 1, hi_y = k.ny + 2 * k.pad - 1;  // padded index range
  k.pf_i0 = clampi(gx - k.gx_scale * reach, 0, hi_x);
  k.pf_i1 = clampi(gx + k.gx_scale * reach + 1, 0, hi_x);
  k.pf_j0 = clampi(gy - k.gy_scale * reach, 0, hi_y);
  k.pf_j1 = clampi(gy + k.gy_scale * reach + 1, 0, hi_y);
}

static void shard_of(int64_t n, int r, int g, int64_t& begin, int64_t& count) {
  const int64_t base = n / g, rem = n % g;
  begin = r * base + std::min<int64_t>(r, rem);
  count = base + (r < rem ? 1 : 0);
}

int tmpc_stage_cycle(tmpc_ctx* c, const double* s0, const tmpc_sampling* smp) {
  Range nv("tmpc_stage");
  if (!c) return fail(nullptr, TMPC_ERR_CONFIG, "null ctx");
  if (!c->have_params || !c->have_terrain)
    return fail(c, TMPC_ERR_CONFIG, "solve: set_params and set_terrain first");
  if (!s0) return fail(c, TMPC_ERR_CONFIG, "solve: null state");
  for (int i = 0; i < TMPC_STATE_DIM; ++i)
    if (!std::isfinite(s0[i])) return fail(c, TMPC_ERR_CONFIG, "solve: non-finite initial state");
  {
    // the fp32 kernel anchors positions in grid cells (int); keep them sane
    const KParams& k = c->kp;
    const double lim0 = 1 << 19, limg = 1 << 30;
    if (std::fabs(s0[0] * k.gx_scale + k.gx_off) > lim0 || std::fabs(s0[1] * k.gy_scale + k.gy_off) > lim0)
      return fail(c, TMPC_ERR_CONFIG, "solve: initial position more than 2^19 cells off the terrain grid");
    if (std::fabs(c->p.goal_x * k.gx_scale + k.gx_off) > limg ||
        std::fabs(c->p.goal_y * k.gy_scale + k.gy_off) > limg)
      return fail(c, TMPC_ERR_CONFIG, "solve: goal more than 2^30 cells off the terrain grid");
  }
  std::string why;
  if (validate_sampling(c->p, smp, why)) return fail(c, TMPC_ERR_CONFIG, "%s", why.c_str());
  if (c->comm_dead)
    return fail(c, TMPC_ERR_RUNTIME, "solve: the NCCL communicator was aborted after a timeout");
  if (c->peer_dead)
    return fail(c, TMPC_ERR_RUNTIME, "solve: the peer exchange timed out in an earlier cycle");
  if (c->peer && c->opts.world_size > 1 && c->xn == 0)
    return fail(c, TMPC_ERR_CONFIG, "solve: peer exchange: tmpc_peer_connect the ranks first");
  c->smp = *smp;
  c->smp.warm_seq = nullptr;
  c->warm_host.clear();
  if (smp->kind == TMPC_SAMPLE_WARM_GAUSS && smp->warm_seq)
    c->warm_host.assign(smp->warm_seq, smp->warm_seq + 2 * c->p.n_steps);
  KParams& k = c->kp;
  k.smp = make_sampler(c->p, *smp);
  k.seed = smp->seed;
  // lanes per candidate from the WHOLE problem's size, so every shard of a
  // G-GPU solve runs the layout a one-GPU solve would: bitwise identical
  // per-candidate results for any G
  const int64_t k_layout = smp->k_total > 0 ? smp->k_total : smp->k_count;
  k.k_layout = k_layout;
  for (int i = 0; i < TMPC_STATE_DIM; ++i) k.s0[i] = s0[i];
  set_prefetch_window(c, s0, *smp);
  // path ordering serves the fp32 Euler SRB kernel (the others are not
  // gather-latency bound); auto enables it from K = 64 K per GPU, where the
  // measured gain exceeds the pass's cost (c4: -16% at 256 K, -26% at 128 K,
  // -6.5% at 64 K, even at 32 K; c3 -1% at 64 K; round 2, tools/ab.py), except
  // for the warm-started Gaussian batch, which already hugs one path (c5:
  // +4% at 128 K, +5 / +12 / +19% at 64 / 32 / 16 K with it)
  const bool fast_kernel = c->opts.precision == TMPC_PRECISION_FP32 &&
                           c->p.model == TMPC_MODEL_SRB && c->p.scheme == TMPC_SCHEME_EULER;
  const int G = static_cast<int>(c->dev.size());
  for (int g = 0; g < G; ++g) {
    DevSlot& d = c->dev[g];
    int64_t b, n;
    shard_of(smp->k_count, g, G, b, n);
    CUDA_TRY(c, cudaSetDevice(d.device));
    int rc = ensure_capacity(c, d, n, c->p.n_steps);
    if (rc) return rc;
    if (!c->warm_host.empty())
      CUDA_TRY(c, cudaMemcpyAsync(d.d_warm, c->warm_host.data(), sizeof(double) * 2 * c->p.n_steps,
                                  cudaMemcpyHostToDevice, d.stream));
    d.kp = k;
    d.kp.k_begin = smp->k_begin + b;
    d.kp.k_count = n;
    d.kp.xpeers = c->d_peers;
    d.kp.xn = c->xn;
    d.kp.xrank = c->opts.rank;
    d.kp.xtimeout_ns = static_cast<unsigned long long>(c->timeout_ms) * 1000000ULL;
    if (one_process(c)) {
      // the last block writes the record into the mapped host record itself
      d.kp.xn = -1;
      d.kp.xhost = d.h_rec_dev;
    }
    d.lanes = c->opts.lanes > 0 ? c->opts.lanes : pick_lanes(k_layout, d.sms);
    d.use_order = fast_kernel && n > 0 &&
                  (c->opts.ordering == TMPC_ORDER_ON ||
                   (c->opts.ordering == TMPC_ORDER_AUTO && n >= 65536 &&
                    smp->kind != TMPC_SAMPLE_WARM_GAUSS));
  }
  c->staged = true;
  return TMPC_OK;
}

// Enqueue one GPU's kernels: directly, or by replaying its cycle graph with
// the new arguments (the graph is rebuilt when the launch shape changes).
static int enqueue_kernels(tmpc_ctx* c, DevSlot& d) {
  const double* warm = c->warm_host.empty() ? nullptr : d.d_warm;
  DevStats* st = &d.d_rec->s;
  std::vector<LaunchRec> recs;
  // one-process mode: the previous cycle's last block left the reduction
  // block reset; after a failed or first cycle it is reset here
  int extra = 0;
  if (d.kp.xn < 0 && !d.stats_clean) {
    CUDA_TRY(c, reset_stats(st, d.stream));
    extra = 1;
  }
  d.stats_clean = false;  // until this cycle completes (tmpc_finish_cycle)
  if (c->graphs) launch_recorder() = &recs;
  d.kp.order = nullptr;
  cudaError_t e = cudaSuccess;
  if (d.use_order) e = launch_order(d.kp, warm, d.d_order, &d.kp.order, d.stream);
  if (e == cudaSuccess)
    e = launch_cycle(d.kp, d.td, warm, d.d_cost, d.d_flags, d.d_margin, st, d.lanes, d.stream);
  launch_recorder() = nullptr;
  CUDA_TRY(c, e);
  if (!c->graphs) {
    d.kernels = (d.use_order ? 4 : 1) + (d.kp.xn >= 0 ? 1 : 0) + extra;
    return TMPC_OK;
  }
  d.kernels = static_cast<int>(recs.size()) + extra;
  CycleGraph& g = d.cg;
  bool same = g.exec && g.recs.size() == recs.size();
  for (size_t i = 0; same && i < recs.size(); ++i)
    same = recs[i].func == g.recs[i].func && recs[i].grid.x == g.recs[i].grid.x &&
           recs[i].grid.y == g.recs[i].grid.y && recs[i].block.x == g.recs[i].block.x;
  if (same) {
    for (size_t i = 0; i < recs.size(); ++i) {
      cudaKernelNodeParams np{};
      np.func = const_cast<void*>(recs[i].func);
      np.gridDim = recs[i].grid;
      np.blockDim = recs[i].block;
      np.kernelParams = recs[i].args.data();
      CUDA_TRY(c, cudaGraphExecKernelNodeSetParams(g.exec, g.nodes[i], &np));
    }
  } else {
    g.reset();
    CUDA_TRY(c, cudaGraphCreate(&g.graph, 0));
    cudaGraphNode_t prev = nullptr;
    for (LaunchRec& r : recs) {
      cudaKernelNodeParams np{};
      np.func = const_cast<void*>(r.func);
      np.gridDim = r.grid;
      np.blockDim = r.block;
      np.kernelParams = r.args.data();
      cudaGraphNode_t node;
      CUDA_TRY(c, cudaGraphAddKernelNode(&node, g.graph, prev ? &prev : nullptr, prev ? 1 : 0, &np));
      g.nodes.push_back(node);
      prev = node;
    }
    CUDA_TRY(c, cudaGraphInstantiate(&g.exec, g.graph, 0));
  }
  g.recs = std::move(recs);
  CUDA_TRY(c, cudaGraphLaunch(g.exec, d.stream));
  return TMPC_OK;
}

int tmpc_launch_cycle(tmpc_ctx* c) {
  Range nv("tmpc_launch");
  if (!c || !c->staged) return fail(c, TMPC_ERR_CONFIG, "launch: stage a cycle first");
  if (c->peer && c->xn > 0) c->dev[0].kp.xseq = ++c->xseq;
  for (DevSlot& d : c->dev) {
    CUDA_TRY(c, cudaSetDevice(d.device));
    CUDA_TRY(c, cudaEventRecord(d.ev0, d.stream));
    if (d.kp.k_count > 0) {
      const int rc = enqueue_kernels(c, d);
      if (rc) return rc;
    } else {
      // an idle GPU (fewer candidates than GPUs) contributes an empty record
      d.kernels = 0;
      RankRecord empty{};
      empty.s.key_lo = empty.s.key_hi = kKeyNone;
      empty.s.min_cost_bits = 0x7ff0000000000000ULL;
      *d.h_rec = empty;
      if (d.kp.xn >= 0)
        CUDA_TRY(c, cudaMemcpyAsync(d.d_rec, d.h_rec, sizeof(RankRecord), cudaMemcpyHostToDevice,
                                    d.stream));
    }
    CUDA_TRY(c, cudaEventRecord(d.ev1, d.stream));
  }
  for (DevSlot& d : c->dev) {
    CUDA_TRY(c, cudaSetDevice(d.device));
    if (c->peer && c->xn > 0) {
      // the kernel exchanged the records itself: bring this cycle's buffer
      // of the local mailbox (every rank's record, rank order) and the flag
      const int par = static_cast<int>(c->xseq & 1);
      CUDA_TRY(c, cudaMemcpyAsync(d.h_rec, &c->d_mb->rec[par][0], sizeof(RankRecord) * c->xn,
                                  cudaMemcpyDeviceToHost, d.stream));
    } else if (c->comm) {
      // one collective per cycle: every rank's record (the shard is written
      // next to the kernel's block) gathered in rank order
      d.h_shard[0] = d.kp.k_begin;
      d.h_shard[1] = d.kp.k_count;
      CUDA_TRY(c, cudaMemcpyAsync(&d.d_rec->k_begin, d.h_shard, 2 * sizeof(long long),
                                  cudaMemcpyHostToDevice, d.stream));
      ncclResult_t r = g_nccl.AllGather(d.d_rec, d.d_gather, sizeof(RankRecord), ncclUint8,
                                        c->comm, d.stream);
      if (r == ncclInProgress) r = nccl_settle(c);  // non-blocking communicator
      if (r != ncclSuccess) {
        g_nccl.CommAbort(c->comm);
        c->comm = nullptr;
        c->comm_dead = true;
        return fail(c, TMPC_ERR_RUNTIME, "ncclAllGather: %s (communicator aborted)",
                    r == ncclInProgress ? "enqueue timed out" : g_nccl.GetErrorString(r));
      }
      CUDA_TRY(c, cudaMemcpyAsync(d.h_rec, d.d_gather, sizeof(RankRecord) * c->opts.world_size,
                                  cudaMemcpyDeviceToHost, d.stream));
    } else if (d.kp.xn >= 0) {
      CUDA_TRY(c, cudaMemcpyAsync(d.h_rec, d.d_rec, offsetof(RankRecord, k_begin),
                                  cudaMemcpyDeviceToHost, d.stream));
    }  // else: one-process mode, the kernel wrote d.h_rec itself
  }
  c->launched = true;
  return TMPC_OK;
}

// Wait for the cycle.  With an NCCL communicator the wait is a watchdog: a
// peer rank that failed before the collective would otherwise block this
// rank forever; past timeout_ms the communicator is aborted (which releases
// the collective's kernel) and the call fails.
static int wait_cycle(tmpc_ctx* c) {
  if (!c->comm) {
    for (DevSlot& d : c->dev) {
      CUDA_TRY(c, cudaSetDevice(d.device));
      CUDA_TRY(c, cudaStreamSynchronize(d.stream));
    }
    return TMPC_OK;
  }
  DevSlot& d = c->dev[0];
  CUDA_TRY(c, cudaSetDevice(d.device));
  const auto t0 = std::chrono::steady_clock::now();
  for (long spins = 0;; ++spins) {
    const cudaError_t q = cudaStreamQuery(d.stream);
    if (q == cudaSuccess) return TMPC_OK;
    if (q != cudaErrorNotReady) CUDA_TRY(c, q);
    ncclResult_t ae = ncclSuccess;
    g_nccl.CommGetAsyncError(c->comm, &ae);
    const double ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if ((ae != ncclSuccess && ae != ncclInProgress) || ms > c->timeout_ms) {
      g_nccl.CommAbort(c->comm);
      c->comm = nullptr;
      c->comm_dead = true;
      c->launched = false;
      if (ae != ncclSuccess && ae != ncclInProgress)
        return fail(c, TMPC_ERR_RUNTIME, "NCCL asynchronous error: %s (communicator aborted)",
                    g_nccl.GetErrorString(ae));
      return fail(c, TMPC_ERR_RUNTIME,
                  "NCCL all-gather did not complete within %d ms (a peer rank failed before the "
                  "collective?); communicator aborted",
                  c->timeout_ms);
    }
    if (spins > 20000) {
      const timespec ts{0, 20000};
      nanosleep(&ts, nullptr);
    }
  }
}

int tmpc_finish_cycle(tmpc_ctx* c, tmpc_result* out) {
  Range nv("tmpc_finish");
  if (!c || !c->launched) return fail(c, TMPC_ERR_CONFIG, "finish: launch a cycle first");
  if (!out) return fail(c, TMPC_ERR_CONFIG, "finish: null result");
  const int wrc = wait_cycle(c);
  if (wrc) return wrc;
  c->launched = false;
  // a one-process kernel that ran to its last block left its reduction block
  // reset; the other modes reset it at the start of every cycle
  for (DevSlot& d : c->dev)
    if (d.kp.k_count > 0) d.stats_clean = d.kp.xn < 0;
  // records in device / rank order
  c->fold_buf.clear();
  if (c->peer && c->xn > 0) {
    bool missing = false;
    for (int i = 0; i < c->xn; ++i) missing = missing || c->dev[0].h_rec[i].k_begin < 0;
    if (missing) {
      c->peer_dead = true;
      return fail(c, TMPC_ERR_RUNTIME,
                  "peer exchange: a rank's record did not arrive within %d ms (a peer failed "
                  "before its cycle?)",
                  c->timeout_ms);
    }
    for (int i = 0; i < c->xn; ++i) {
      tmpc_rank_record q;
      std::memcpy(&q, &c->dev[0].h_rec[i], sizeof(q));
      c->fold_buf.push_back(q);
    }
  } else if (c->comm) {
    const RankRecord* r = c->dev[0].h_rec;
    for (int i = 0; i < c->opts.world_size; ++i) {
      tmpc_rank_record q;
      std::memcpy(&q, &r[i], sizeof(q));
      c->fold_buf.push_back(q);
    }
  } else {
    for (DevSlot& d : c->dev) {
      d.h_rec->k_begin = d.kp.k_begin;
      d.h_rec->k_count = d.kp.k_count;
      tmpc_rank_record q;
      std::memcpy(&q, d.h_rec, sizeof(q));
      c->fold_buf.push_back(q);
    }
  }
  std::string why;
  const int rc = fold(c->fold_buf.data(), static_cast<int>(c->fold_buf.size()), out, why);
  float kms = 0.f;
  for (DevSlot& d : c->dev) {
    float m = 0.f;
    cudaSetDevice(d.device);
    cudaEventElapsedTime(&m, d.ev0, d.ev1);
    kms = std::max(kms, m);
  }
  out->kernel_ms = kms;
  if (rc) return fail(c, rc, "%s", why.c_str());
  return TMPC_OK;
}

int tmpc_sample_controls(const tmpc_params* p, const tmpc_sampling* smp, int64_t k, double* out) {
  std::string why;
  if (validate_params(p, why)) return fail(nullptr, TMPC_ERR_CONFIG, "%s", why.c_str());
  if (!smp || !out) return fail(nullptr, TMPC_ERR_CONFIG, "sample_controls: null argument");
  const Sampler z = make_sampler(*p, *smp);
  const uint64_t base = mix64(substream(smp->seed, static_cast<uint64_t>(k)));
  double prev[2] = {0.0, 0.0};
  for (int t = 0; t < p->n_steps; ++t)
    sample_step(z, base, k == 0, t, smp->kind == TMPC_SAMPLE_WARM_GAUSS ? smp->warm_seq : nullptr,
                prev, out + 2 * t);
  return TMPC_OK;
}

int tmpc_solve(tmpc_ctx* c, const double* s0, const tmpc_sampling* smp, tmpc_result* out,
               double* best_controls) {
  const auto t0 = std::chrono::steady_clock::now();
  if (!out) return fail(c, TMPC_ERR_CONFIG, "solve: null result");
  int rc = tmpc_stage_cycle(c, s0, smp);
  if (rc) return rc;
  rc = tmpc_launch_cycle(c);
  if (rc) return rc;
  rc = tmpc_finish_cycle(c, out);
  if (rc == TMPC_OK && best_controls) {
    tmpc_sampling s = c->smp;
    s.warm_seq = c->warm_host.empty() ? nullptr : c->warm_host.data();
    rc = tmpc_sample_controls(&c->p, &s, out->best_index, best_controls);
  }
  out->cycle_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return rc;
}

int tmpc_get_costs(tmpc_ctx* c, double* cost, uint8_t* flags, float* margin) {
  if (!c || !c->staged) return fail(c, TMPC_ERR_CONFIG, "get_costs: no cycle");
  int64_t off = 0;
  for (DevSlot& d : c->dev) {
    const int64_t K = d.kp.k_count;
    if (K > 0) {
      CUDA_TRY(c, cudaSetDevice(d.device));
      if (cost)
        CUDA_TRY(c, cudaMemcpyAsync(cost + off, d.d_cost, sizeof(double) * K, cudaMemcpyDeviceToHost, d.stream));
      if (flags)
        CUDA_TRY(c, cudaMemcpyAsync(flags + off, d.d_flags, K, cudaMemcpyDeviceToHost, d.stream));
      if (margin)
        CUDA_TRY(c, cudaMemcpyAsync(margin + off, d.d_margin, sizeof(float) * K, cudaMemcpyDeviceToHost, d.stream));
    }
    off += K;
  }
  for (DevSlot& d : c->dev) {
    CUDA_TRY(c, cudaSetDevice(d.device));
    CUDA_TRY(c, cudaStreamSynchronize(d.stream));
  }
  return TMPC_OK;
}

void* tmpc_get_stream(tmpc_ctx* c) {
  return c && !c->dev.empty() ? static_cast<void*>(c->dev[0].stream) : nullptr;
}
int tmpc_num_devices(const tmpc_ctx* c) { return c ? static_cast<int>(c->dev.size()) : 0; }
void* tmpc_get_device_stream(tmpc_ctx* c, int32_t i) {
  return c && i >= 0 && i < static_cast<int>(c->dev.size()) ? static_cast<void*>(c->dev[i].stream)
                                                             : nullptr;
}
int tmpc_get_device_ordinal(const tmpc_ctx* c, int32_t i) {
  return c && i >= 0 && i < static_cast<int>(c->dev.size()) ? c->dev[i].device : -1;
}
int tmpc_kernels_per_cycle(const tmpc_ctx* c) {
  if (!c) return 0;
  int n = 0;
  for (const DevSlot& d : c->dev) n += d.kernels;
  return n;
}

int tmpc_set_plant_terrain(tmpc_ctx* c, const tmpc_terrain* t) {
  if (!c) return fail(nullptr, TMPC_ERR_CONFIG, "null ctx");
  if (!t) {  // back to the planning terrain
    c->have_plant = false;
    return TMPC_OK;
  }
  std::string why;
  if (validate_terrain(t, why)) return fail(c, TMPC_ERR_CONFIG, "%s", why.c_str());
  if (c->opts.precision != TMPC_PRECISION_FP64)
    return fail(c, TMPC_ERR_CONFIG, "set_plant_terrain: needs a TMPC_PRECISION_FP64 context");
  // the fp64 store's layout (Q = 2 replicated cells, node central differences)
  const int Q = 2, nx = t->nx, ny = t->ny, px = nx + 2 * Q, py = ny + 2 * Q;
  const size_t n = static_cast<size_t>(px) * py;
  std::vector<double> H(n);
  for (int j = 0; j < py; ++j)
    for (int i = 0; i < px; ++i)
      H[static_cast<size_t>(j) * px + i] =
          t->heights[static_cast<size_t>(std::clamp(j - Q, 0, ny - 1)) * nx + std::clamp(i - Q, 0, nx - 1)];
  const double inv2r = 1.0 / (2.0 * t->resolution);
  std::vector<HG64> hg(n);
  for (int j = 0; j < py; ++j)
    for (int i = 0; i < px; ++i) {
      const size_t o = static_cast<size_t>(j) * px + i;
      const double dx = (i >= 1 && i < px - 1) ? (H[o + 1] - H[o - 1]) * inv2r : 0.0;
      const double dy = (j >= 1 && j < py - 1) ? (H[o + px] - H[o - px]) * inv2r : 0.0;
      hg[o] = HG64{make_double2(H[o], dx), make_double2(dy, 0.0)};
    }
  DevSlot& d = c->dev[0];
  CUDA_TRY(c, cudaSetDevice(d.device));
  cudaFree(c->d_plant_hg);
  c->d_plant_hg = nullptr;
  c->have_plant = false;
  CUDA_TRY(c, cudaMalloc(&c->d_plant_hg, n * sizeof(HG64)));
  CUDA_TRY(c, cudaMemcpy(c->d_plant_hg, hg.data(), n * sizeof(HG64), cudaMemcpyHostToDevice));
  c->plant_grid = *t;
  c->plant_grid.heights = nullptr;
  c->plant_grid.sdist = nullptr;
  c->have_plant = true;
  return TMPC_OK;
}

int tmpc_open_loop_errors(tmpc_ctx* c, int32_t model, const double* s0, const double* controls,
                          int64_t n_traj, double plant_dt, double* loc_err, double* esm_err,
                          uint8_t* flags) {
  Range nv("tmpc_open_loop_errors");
  if (!c) return fail(nullptr, TMPC_ERR_CONFIG, "null ctx");
  if (!c->have_params || !c->have_terrain)
    return fail(c, TMPC_ERR_CONFIG, "open_loop_errors: set_params and set_terrain first");
  if (c->opts.precision != TMPC_PRECISION_FP64)
    return fail(c, TMPC_ERR_CONFIG, "open_loop_errors: needs a TMPC_PRECISION_FP64 context");
  if (model != TMPC_MODEL_SRB && model != TMPC_MODEL_EST)
    return fail(c, TMPC_ERR_CONFIG, "open_loop_errors: unknown model");
  if (n_traj < 0 || (n_traj > 0 && (!s0 || !controls || !loc_err || !esm_err || !flags)))
    return fail(c, TMPC_ERR_CONFIG, "open_loop_errors: bad arguments");
  const int sub = static_cast<int>(std::lround(c->p.dt_int / plant_dt));
  if (!(plant_dt > 0.0) || sub < 1 || std::fabs(sub * plant_dt - c->p.dt_int) > 1e-12)
    return fail(c, TMPC_ERR_CONFIG, "open_loop_errors: plant_dt must divide dt_int");
  if (n_traj == 0) return TMPC_OK;
  for (int64_t i = 0; i < 13 * n_traj; ++i)
    if (!std::isfinite(s0[i])) return fail(c, TMPC_ERR_CONFIG, "open_loop_errors: non-finite state");
  DevSlot& d = c->dev[0];
  CUDA_TRY(c, cudaSetDevice(d.device));
  const size_t ns = sizeof(double) * 13 * n_traj, nc = sizeof(double) * 2 * c->p.n_steps * n_traj;
  const size_t no = sizeof(double) * n_traj;
  char* buf = nullptr;
  CUDA_TRY(c, cudaMalloc(&buf, ns + nc + 2 * no + n_traj));
  double* d_s0 = reinterpret_cast<double*>(buf);
  double* d_u = reinterpret_cast<double*>(buf + ns);
  double* d_loc = reinterpret_cast<double*>(buf + ns + nc);
  double* d_esm = reinterpret_cast<double*>(buf + ns + nc + no);
  uint8_t* d_fl = reinterpret_cast<uint8_t*>(buf + ns + nc + 2 * no);
  KParams kp = c->kp;
  kp.k_count = n_traj;
  TerrainDev tdp = d.td;
  if (c->have_plant) {
    const tmpc_terrain& g = c->plant_grid;
    if (g.nx != c->terr.nx || g.ny != c->terr.ny || g.origin_x != c->terr.origin_x ||
        g.origin_y != c->terr.origin_y || g.resolution != c->terr.resolution) {
      cudaFree(buf);
      return fail(c, TMPC_ERR_CONFIG, "open_loop_errors: the plant terrain's grid differs from the "
                                      "terrain's (set both on the same GridSpec)");
    }
    tdp.hg64 = c->d_plant_hg;
  }
  cudaError_t e = cudaMemcpyAsync(d_s0, s0, ns, cudaMemcpyHostToDevice, d.stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_u, controls, nc, cudaMemcpyHostToDevice, d.stream);
  if (e == cudaSuccess)
    e = launch_open_loop(kp, d.td, tdp, model, d_s0, d_u, n_traj, plant_dt, sub, d_loc, d_esm,
                         d_fl, d.stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(loc_err, d_loc, no, cudaMemcpyDeviceToHost, d.stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(esm_err, d_esm, no, cudaMemcpyDeviceToHost, d.stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(flags, d_fl, n_traj, cudaMemcpyDeviceToHost, d.stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(d.stream);
  cudaFree(buf);
  CUDA_TRY(c, e);
  return TMPC_OK;
}

uint64_t tmpc_key_hi(double cost, int feasible, int selection) {
  return key_hi(cost, selection == TMPC_SELECT_FEASIBLE_FIRST && !feasible);
}

int tmpc_make_record(const double* cost, const uint8_t* flags, const float* margin,
                     const int64_t* substeps, int64_t k_begin, int64_t k_count, int selection,
                     tmpc_rank_record* out) {
  if (!out || (k_count > 0 && (!cost || !flags || !margin)) || k_count < 0)
    return fail(nullptr, TMPC_ERR_CONFIG, "make_record: bad arguments");
  std::memset(out, 0, sizeof(*out));
  out->key_lo = out->key_hi = kKeyNone;
  out->min_cost_bits = 0x7ff0000000000000ULL;
  out->best_cost = std::numeric_limits<double>::infinity();
  out->k_begin = k_begin;
  out->k_count = k_count;
  int64_t w = -1;
  for (int64_t i = 0; i < k_count; ++i) {
    const bool feas = flags[i] & TMPC_FLAG_FEASIBLE, div = flags[i] & TMPC_FLAG_DIVERGED;
    const uint64_t hi = key_hi(cost[i], selection == TMPC_SELECT_FEASIBLE_FIRST && !feas);
    const uint64_t lo = static_cast<uint64_t>(k_begin + i);
    if (key_less(hi, lo, out->key_hi, out->key_lo)) {
      out->key_hi = hi;
      out->key_lo = lo;
      w = i;
    }
    out->n_feasible += feas;
    out->n_diverged += div;
    out->n_goal += (flags[i] & TMPC_FLAG_GOAL) != 0;
    if (substeps) out->substeps += static_cast<uint64_t>(substeps[i]);
    if (!div) {
      out->n_finite += 1;
      uint64_t l[3];
      cost_limbs(cost[i], l);
      for (int j = 0; j < 3; ++j) out->cost_limb[j] += l[j];
      out->min_cost_bits = std::min<uint64_t>(out->min_cost_bits, dbits(cost[i]));
    }
  }
  if (w >= 0) {
    out->best_cost = cost[w];
    out->best_flags = flags[w];
    out->best_margin = margin[w];
  }
  return TMPC_OK;
}

int tmpc_fold_records(const tmpc_rank_record* recs, int32_t n, tmpc_result* out) {
  if (!recs || n < 1 || !out) return fail(nullptr, TMPC_ERR_CONFIG, "fold_records: bad arguments");
  std::string why;
  const int rc = fold(recs, n, out, why);
  if (rc) return fail(nullptr, rc, "%s", why.c_str());
  return TMPC_OK;
}

}  // extern "C"

namespace tmpcb {
// Context-free entry points (terrain_prep.cu) report through tmpc_last_error(NULL).
int set_global_error(int code, const char* msg) {
  g_last_error = msg;
  return code;
}
}  // namespace tmpcb
