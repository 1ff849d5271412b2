// Host side of libtmpc_b200: the C ABI (include/tmpc_b200.h), parameter
// validation mirroring the reference validate() methods, the terrain store
// upload (padded node fields), the per-cycle launch and the
// cross-GPU arg-min through NCCL.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "nccl.h"
#include "rollout.cuh"
#include "tmpc_b200.h"
#include "tmpc_common.h"

namespace tmpcb {
cudaError_t launch_cycle(const KParams& P, const TerrainDev& td, const double* warm, double* cost,
                         uint8_t* flags, float* margin, DevStats* st, int lanes,
                         cudaStream_t stream);
int pick_lanes(int64_t k, int sms);
size_t order_scratch_bytes(int64_t n);
cudaError_t configure_rollout_f32();
cudaError_t configure_rollout_est_f32();
cudaError_t configure_rollout_rk4_f32();
size_t order_hist_bytes();
cudaError_t launch_order(const KParams& P, const double* warm, void* scratch,
                         const int32_t** order_out, cudaStream_t stream);
cudaError_t launch_winner_pack(const DevStats* st, double* red, int64_t k_begin, int64_t k_count,
                               cudaStream_t stream);
}  // namespace tmpcb

using namespace tmpcb;

namespace {

constexpr double kPi = 3.14159265358979323846;
constexpr double kGimbalMargin = 1e-3;  // dynamics.hpp:16

thread_local std::string g_last_error;

// ---- NCCL, loaded lazily (only world_size > 1 needs it) -------------------
struct Nccl {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
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
    GetUniqueId = reinterpret_cast<decltype(GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    CommInitRank = reinterpret_cast<decltype(CommInitRank)>(dlsym(h, "ncclCommInitRank"));
    AllReduce = reinterpret_cast<decltype(AllReduce)>(dlsym(h, "ncclAllReduce"));
    CommDestroy = reinterpret_cast<decltype(CommDestroy)>(dlsym(h, "ncclCommDestroy"));
    GetErrorString = reinterpret_cast<decltype(GetErrorString)>(dlsym(h, "ncclGetErrorString"));
    if (!GetUniqueId || !CommInitRank || !AllReduce || !CommDestroy || !GetErrorString) {
      err = "NCCL: missing symbols";
      return false;
    }
    return true;
  }
};
Nccl g_nccl;

}  // namespace

struct tmpc_ctx {
  tmpc_opts opts{};
  std::string err;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // params / terrain / sampler
  bool have_params = false, have_terrain = false, staged = false, launched = false;
  tmpc_params p{};
  tmpc_sampling smp{};
  std::vector<double> warm_host;
  KParams kp{};
  // device buffers (terrain store in the precision of the context)
  void* d_hg = nullptr;
  void* d_sd = nullptr;
  size_t terrain_bytes = 0;
  TerrainDev td{};
  cudaTextureObject_t sd_tex = 0, hq_tex = 0;  // texture views of the fp32 records
  tmpc_terrain terr{};                   // host copy of the last set_terrain
  std::vector<double> terr_h, terr_sd;
  int terr_pad = 0;                      // replicated cells per side on the device
  double* d_warm = nullptr;
  double* d_cost = nullptr;
  uint8_t* d_flags = nullptr;
  float* d_margin = nullptr;
  DevStats* d_stats = nullptr;
  void* d_order = nullptr;  // ordering pass scratch (order.cu)
  bool use_order = false;   // ordering pass in the staged cycle
  bool l2_prefetch = true;  // TMPC_L2_PREFETCH=0 disables (A/B timing)
  double* d_red = nullptr;  // multi-GPU SUM buffer
  DevStats* h_stats = nullptr;  // pinned
  double* h_red = nullptr;      // pinned
  int sms = 148;
  int lanes = 1;  // lanes per candidate of the staged cycle (fp32 kernel)
  int64_t cap_k = 0;
  int cap_n = 0;
  ncclComm_t comm = nullptr;
  int kernels_per_cycle = 2;
};

namespace {

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

#define NCCL_TRY(ctx, expr)                                                                  \
  do {                                                                                       \
    const ncclResult_t r_ = (expr);                                                          \
    if (r_ != ncclSuccess)                                                                   \
      return fail(ctx, TMPC_ERR_RUNTIME, "NCCL error %s at %s:%d", g_nccl.GetErrorString(r_), \
                  __FILE__, __LINE__);                                                       \
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

void free_buffers(tmpc_ctx* c) {
  cudaFree(c->d_warm);
  cudaFree(c->d_cost);
  cudaFree(c->d_flags);
  cudaFree(c->d_margin);
  cudaFree(c->d_order);
  c->d_order = nullptr;
  c->d_warm = nullptr;
  c->d_cost = nullptr;
  c->d_flags = nullptr;
  c->d_margin = nullptr;
}

int ensure_capacity(tmpc_ctx* c, int64_t K, int N) {
  if (K <= c->cap_k && N <= c->cap_n) return TMPC_OK;
  free_buffers(c);
  c->cap_k = std::max(K, c->cap_k);
  c->cap_n = std::max(N, c->cap_n);
  CUDA_TRY(c, cudaMalloc(&c->d_cost, sizeof(double) * c->cap_k));
  CUDA_TRY(c, cudaMalloc(&c->d_flags, c->cap_k));
  CUDA_TRY(c, cudaMalloc(&c->d_margin, sizeof(float) * c->cap_k));
  CUDA_TRY(c, cudaMalloc(&c->d_warm, sizeof(double) * 2 * c->cap_n));
  CUDA_TRY(c, cudaMalloc(&c->d_order, order_scratch_bytes(c->cap_k)));
  CUDA_TRY(c, cudaMemset(c->d_order, 0, order_hist_bytes()));
  return TMPC_OK;
}

}  // namespace

extern "C" {

const char* tmpc_last_error(const tmpc_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_last_error.c_str();
}

const char* tmpc_build_info(void) {
  return "tmpc_b200 " __DATE__ " sm_100a rollout_kernel(thread-per-candidate, fp32 math, fp64 "
         "position/cost accumulators)";
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
  if (opts->world_size > 1 && !opts->nccl_id)
    return fail(nullptr, TMPC_ERR_CONFIG, "ctx_create: world_size > 1 needs an NCCL unique id");
  if (opts->lanes != 0 && opts->lanes != 1 && opts->lanes != 2 && opts->lanes != 4)
    return fail(nullptr, TMPC_ERR_CONFIG, "ctx_create: lanes must be 0 (auto), 1, 2 or 4");
  if (opts->precision != TMPC_PRECISION_FP32 && opts->precision != TMPC_PRECISION_FP64)
    return fail(nullptr, TMPC_ERR_CONFIG, "ctx_create: unknown precision");
  if (opts->ordering != TMPC_ORDER_AUTO && opts->ordering != TMPC_ORDER_OFF &&
      opts->ordering != TMPC_ORDER_ON)
    return fail(nullptr, TMPC_ERR_CONFIG, "ctx_create: unknown ordering mode");
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0)
    return fail(nullptr, TMPC_ERR_RUNTIME, "ctx_create: no CUDA device (%s)", cudaGetErrorString(e));
  if (opts->device < 0 || opts->device >= ndev)
    return fail(nullptr, TMPC_ERR_CONFIG, "ctx_create: device %d out of range", opts->device);
  auto* c = new tmpc_ctx();
  c->opts = *opts;
  c->opts.nccl_id = nullptr;
  auto bail = [&](int rc) {
    g_last_error = c->err;
    tmpc_ctx_destroy(c);
    return rc;
  };
  if (cudaSetDevice(opts->device) != cudaSuccess) return bail(fail(c, TMPC_ERR_RUNTIME, "cudaSetDevice failed"));
  int major = 0, minor = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, opts->device);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, opts->device);
  cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, opts->device);
  if (major != 10 || minor != 0)
    return bail(fail(c, TMPC_ERR_RUNTIME, "ctx_create: built for sm_100a, device is sm_%d%d", major, minor));
  if (const char* e = std::getenv("TMPC_L2_PREFETCH")) c->l2_prefetch = std::atoi(e) != 0;
  if (configure_rollout_f32() != cudaSuccess || configure_rollout_est_f32() != cudaSuccess ||
      configure_rollout_rk4_f32() != cudaSuccess)
    return bail(fail(c, TMPC_ERR_RUNTIME, "ctx_create: kernel attribute setup failed"));
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreate(&c->ev0) != cudaSuccess || cudaEventCreate(&c->ev1) != cudaSuccess ||
      cudaMalloc(&c->d_stats, sizeof(DevStats)) != cudaSuccess ||
      cudaMalloc(&c->d_red, sizeof(double) * 16) != cudaSuccess ||
      cudaMallocHost(&c->h_stats, sizeof(DevStats)) != cudaSuccess ||
      cudaMallocHost(&c->h_red, sizeof(double) * 16) != cudaSuccess)
    return bail(fail(c, TMPC_ERR_RUNTIME, "ctx_create: CUDA allocation failed"));
  if (opts->k_max > 0 || opts->n_steps_max > 0) {
    const int rc = ensure_capacity(c, std::max<int64_t>(1, opts->k_max), std::max(1, opts->n_steps_max));
    if (rc) return bail(rc);
  }
  // NCCL communicator for world_size > 1; with world_size == 1 an explicit id
  // still builds a 1-rank communicator (exercises the collective path on one GPU)
  if (opts->world_size > 1 || opts->nccl_id) {
    std::string err;
    if (!g_nccl.load(err)) return bail(fail(c, TMPC_ERR_RUNTIME, "%s", err.c_str()));
    ncclUniqueId id;
    std::memcpy(&id, opts->nccl_id, sizeof(id));
    const ncclResult_t r = g_nccl.CommInitRank(&c->comm, opts->world_size, id, opts->rank);
    if (r != ncclSuccess)
      return bail(fail(c, TMPC_ERR_RUNTIME, "ncclCommInitRank: %s", g_nccl.GetErrorString(r)));
  }
  *out = c;
  return TMPC_OK;
}

void tmpc_ctx_destroy(tmpc_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->opts.device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->comm) g_nccl.CommDestroy(c->comm);
  free_buffers(c);
  if (c->sd_tex) cudaDestroyTextureObject(c->sd_tex);
  if (c->hq_tex) cudaDestroyTextureObject(c->hq_tex);
  cudaFree(c->d_hg);
  cudaFree(c->d_sd);
  cudaFree(c->d_stats);
  cudaFree(c->d_red);
  cudaFreeHost(c->h_stats);
  cudaFreeHost(c->h_red);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  if (c->stream) cudaStreamDestroy(c->stream);
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

// Upload the cached host terrain (c->terr) with Q replicated cells per side.
// fp64 mode: Q = 2 (the gradient stencil's reach).  fp32 mode: Q = terrain_pad()
// so that the SRB kernels clamp only the CoM per substep and look the wheel
// points up unclamped (rollout_srb_frame.cuh): beyond the reference's clamp
// window the replicated fields are constant along the clamped axis, so every
// record there has c1 = c3 = 0 (x) or c2 = c3 = 0 (y) exactly and returns the
// clamped lookup's value bit for bit.
static int upload_terrain(tmpc_ctx* c, int Q) {
  const tmpc_terrain* t = &c->terr;
  CUDA_TRY(c, cudaSetDevice(c->opts.device));
  const int nx = t->nx, ny = t->ny, px = nx + 2 * Q, py = ny + 2 * Q;
  const size_t n = static_cast<size_t>(px) * py;
  // padded fp64 copies (Q replicated cells per side) -> fp32 node fields
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
  const bool f64 = c->opts.precision == TMPC_PRECISION_FP64;
  const size_t hg_bytes = n * (f64 ? sizeof(HG64) : 4 * sizeof(float4));
  const size_t sd_bytes = n * (f64 ? sizeof(double) : sizeof(float4));
  if (hg_bytes + sd_bytes != c->terrain_bytes) {
    cudaFree(c->d_hg);
    cudaFree(c->d_sd);
    c->d_hg = nullptr;
    c->d_sd = nullptr;
    CUDA_TRY(c, cudaMalloc(&c->d_hg, hg_bytes));
    CUDA_TRY(c, cudaMalloc(&c->d_sd, sd_bytes));
    c->terrain_bytes = hg_bytes + sd_bytes;
  }
  c->td = TerrainDev{};
  if (f64) {
    std::vector<HG64> hg(n);
    for (size_t o = 0; o < n; ++o) hg[o] = HG64{make_double2(H[o], Dx[o]), make_double2(Dy[o], 0.0)};
    CUDA_TRY(c, cudaMemcpy(c->d_hg, hg.data(), hg_bytes, cudaMemcpyHostToDevice));
    CUDA_TRY(c, cudaMemcpy(c->d_sd, SD.data(), sd_bytes, cudaMemcpyHostToDevice));
    c->td.hg64 = static_cast<const HG64*>(c->d_hg);
    c->td.sd64 = static_cast<const double*>(c->d_sd);
  } else {
    // cell records: the bilinear coefficients {v00, v10 - v00, v01 - v00,
    // v11 - v10 - v01 + v00} (fp64, rounded once) of H, Dx, Dy (+ pad) and of
    // the SDF, for the cell whose lower-left node is o (lookups never start on
    // the last padded row/column: i0, j0 <= n+2)
    std::vector<float4> hq(4 * n), sdq(n);
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
        hq[4 * o + 3] = make_float4(0.f, 0.f, 0.f, 0.f);
        sdq[o] = quad(SD);
      }
    CUDA_TRY(c, cudaMemcpy(c->d_hg, hq.data(), hg_bytes, cudaMemcpyHostToDevice));
    CUDA_TRY(c, cudaMemcpy(c->d_sd, sdq.data(), sd_bytes, cudaMemcpyHostToDevice));
    c->td.hq32 = static_cast<const float4*>(c->d_hg);
    c->td.sdq32 = static_cast<const float4*>(c->d_sd);
    if (c->sd_tex) cudaDestroyTextureObject(c->sd_tex);
    c->sd_tex = 0;
    cudaResourceDesc rd{};
    rd.resType = cudaResourceTypeLinear;
    rd.res.linear.devPtr = c->d_sd;
    rd.res.linear.desc = cudaCreateChannelDesc<float4>();
    rd.res.linear.sizeInBytes = sd_bytes;
    cudaTextureDesc tdsc{};
    tdsc.readMode = cudaReadModeElementType;
    tdsc.filterMode = cudaFilterModePoint;
    tdsc.addressMode[0] = cudaAddressModeClamp;
    CUDA_TRY(c, cudaCreateTextureObject(&c->sd_tex, &rd, &tdsc, nullptr));
    c->td.sd_tex = c->sd_tex;
    if (c->hq_tex) cudaDestroyTextureObject(c->hq_tex);
    c->hq_tex = 0;
    rd.res.linear.devPtr = c->d_hg;
    rd.res.linear.sizeInBytes = hg_bytes;
    CUDA_TRY(c, cudaCreateTextureObject(&c->hq_tex, &rd, &tdsc, nullptr));
    c->td.hq_tex = c->hq_tex;
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

int tmpc_stage_cycle(tmpc_ctx* c, const double* s0, const tmpc_sampling* smp) {
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
  CUDA_TRY(c, cudaSetDevice(c->opts.device));
  int rc = ensure_capacity(c, smp->k_count, c->p.n_steps);
  if (rc) return rc;
  c->smp = *smp;
  c->smp.warm_seq = nullptr;
  c->warm_host.clear();
  if (smp->kind == TMPC_SAMPLE_WARM_GAUSS && smp->warm_seq) {
    c->warm_host.assign(smp->warm_seq, smp->warm_seq + 2 * c->p.n_steps);
    CUDA_TRY(c, cudaMemcpyAsync(c->d_warm, c->warm_host.data(), sizeof(double) * 2 * c->p.n_steps,
                                cudaMemcpyHostToDevice, c->stream));
  }
  KParams& k = c->kp;
  k.smp = make_sampler(c->p, *smp);
  k.seed = smp->seed;
  k.k_begin = smp->k_begin;
  k.k_count = smp->k_count;
  // lanes per candidate from the WHOLE problem's size, so every shard of a
  // G-GPU solve runs the layout a one-GPU solve would: bitwise identical
  // per-candidate results for any G
  const int64_t k_layout = smp->k_total > 0 ? smp->k_total : smp->k_count;
  k.k_layout = k_layout;
  c->lanes = c->opts.lanes > 0 ? c->opts.lanes : pick_lanes(k_layout, c->sms);
  // path ordering serves the fp32 Euler SRB kernel (the others are not
  // gather-latency bound); auto enables it from K = 128 K, where the
  // measured gain exceeds the pass's cost (c4: -16%; c2 / c3: +0-5%), except
  // for the warm-started Gaussian batch, which already hugs one path (c5:
  // +4% with it)
  const bool fast_kernel = c->opts.precision == TMPC_PRECISION_FP32 &&
                           c->p.model == TMPC_MODEL_SRB && c->p.scheme == TMPC_SCHEME_EULER;
  c->use_order = fast_kernel && (c->opts.ordering == TMPC_ORDER_ON ||
                                 (c->opts.ordering == TMPC_ORDER_AUTO && smp->k_count >= 131072 &&
                                  smp->kind != TMPC_SAMPLE_WARM_GAUSS));
  for (int i = 0; i < TMPC_STATE_DIM; ++i) k.s0[i] = s0[i];
  set_prefetch_window(c, s0, *smp);
  c->staged = true;
  return TMPC_OK;
}

int tmpc_launch_cycle(tmpc_ctx* c) {
  if (!c || !c->staged) return fail(c, TMPC_ERR_CONFIG, "launch: stage a cycle first");
  const double* warm = c->warm_host.empty() ? nullptr : c->d_warm;
  CUDA_TRY(c, cudaEventRecord(c->ev0, c->stream));
  c->kp.order = nullptr;
  if (c->use_order) CUDA_TRY(c, launch_order(c->kp, warm, c->d_order, &c->kp.order, c->stream));
  CUDA_TRY(c, launch_cycle(c->kp, c->td, warm, c->d_cost, c->d_flags, c->d_margin, c->d_stats,
                           c->lanes, c->stream));
  CUDA_TRY(c, cudaEventRecord(c->ev1, c->stream));
  c->kernels_per_cycle = c->use_order ? 5 : 2;
  if (c->comm) {
    // cross-GPU reduction, all on the stream (one host sync per cycle): an
    // in-place ncclMin over (key, min cost bits), the owner-masked pack, one
    // ncclSum of the counts / sums / winner fields
    NCCL_TRY(c, g_nccl.AllReduce(&c->d_stats->key, &c->d_stats->key, 2, ncclInt64, ncclMin,
                                 c->comm, c->stream));
    CUDA_TRY(c, launch_winner_pack(c->d_stats, c->d_red, c->kp.k_begin, c->kp.k_count, c->stream));
    NCCL_TRY(c, g_nccl.AllReduce(c->d_red, c->d_red, 10, ncclFloat64, ncclSum, c->comm, c->stream));
    CUDA_TRY(c, cudaMemcpyAsync(c->h_red, c->d_red, sizeof(double) * 10, cudaMemcpyDeviceToHost,
                                c->stream));
    c->kernels_per_cycle += 1;
  }
  CUDA_TRY(c, cudaMemcpyAsync(c->h_stats, c->d_stats, sizeof(DevStats), cudaMemcpyDeviceToHost, c->stream));
  c->launched = true;
  return TMPC_OK;
}

int tmpc_finish_cycle(tmpc_ctx* c, tmpc_result* out) {
  if (!c || !c->launched) return fail(c, TMPC_ERR_CONFIG, "finish: launch a cycle first");
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  c->launched = false;
  const DevStats& s = *c->h_stats;
  double red[8] = {static_cast<double>(s.n_feasible), static_cast<double>(s.n_diverged),
                   static_cast<double>(s.n_goal),     static_cast<double>(s.n_finite),
                   static_cast<double>(s.substeps),   s.sum_cost,
                   s.best_cost,                        static_cast<double>(s.best_margin)};
  double best_flags = s.best_flags;
  double n_total = static_cast<double>(c->kp.k_count);
  if (c->comm) {  // global sums (the key and min cost bits in s are global already)
    const double* h = c->h_red;
    for (int i = 0; i < 8; ++i) red[i] = h[i];
    best_flags = h[8];
    n_total = h[9];
  }
  const double min_cost = red[3] > 0 ? __builtin_bit_cast(double, s.min_cost_bits)
                                     : std::numeric_limits<double>::infinity();
  float kms = 0.f;
  cudaEventElapsedTime(&kms, c->ev0, c->ev1);
  std::memset(out, 0, sizeof(*out));
  out->best_index = key_index(s.key);
  out->best_cost = red[6];
  out->best_margin = static_cast<float>(red[7]);
  out->best_feasible = (static_cast<int>(best_flags) & TMPC_FLAG_FEASIBLE) ? 1 : 0;
  out->n_candidates = static_cast<int64_t>(n_total);
  out->n_feasible = static_cast<int64_t>(red[0]);
  out->n_diverged = static_cast<int64_t>(red[1]);
  out->n_goal = static_cast<int64_t>(red[2]);
  const double n_fin = red[3];
  out->substeps_executed = static_cast<int64_t>(red[4]);
  out->min_cost = min_cost;
  out->mean_cost = n_fin > 0 ? red[5] / n_fin : std::numeric_limits<double>::infinity();
  out->kernel_ms = kms;
  if (s.key == kKeyNone || out->n_diverged == out->n_candidates)
    return fail(c, TMPC_ERR_NUMERIC, "solve_ocp: all %lld rollouts diverged",
                static_cast<long long>(out->n_candidates));
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
  CUDA_TRY(c, cudaSetDevice(c->opts.device));
  const int64_t K = c->kp.k_count;
  if (cost) CUDA_TRY(c, cudaMemcpyAsync(cost, c->d_cost, sizeof(double) * K, cudaMemcpyDeviceToHost, c->stream));
  if (flags) CUDA_TRY(c, cudaMemcpyAsync(flags, c->d_flags, K, cudaMemcpyDeviceToHost, c->stream));
  if (margin) CUDA_TRY(c, cudaMemcpyAsync(margin, c->d_margin, sizeof(float) * K, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return TMPC_OK;
}

void* tmpc_get_stream(tmpc_ctx* c) { return c ? static_cast<void*>(c->stream) : nullptr; }
int tmpc_kernels_per_cycle(const tmpc_ctx* c) { return c ? c->kernels_per_cycle : 0; }

int64_t tmpc_pack_key(double cost, int feasible, int64_t index, int selection) {
  const bool infeasible = selection == TMPC_SELECT_FEASIBLE_FIRST && !feasible;
  return pack_key(static_cast<float>(cost), infeasible, index);
}
int64_t tmpc_key_index(int64_t key) { return key_index(key); }

}  // extern "C"

namespace tmpcb {
// Context-free entry points (terrain_prep.cu) report through tmpc_last_error(NULL).
int set_global_error(int code, const char* msg) {
  g_last_error = msg;
  return code;
}
}  // namespace tmpcb
