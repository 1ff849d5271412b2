// Device terrain preprocessing: the reference's
// gaussian_smooth (terrain.hpp:102-138, the planner / plant LODs) and
// build_sdist_map (terrain.hpp:241-260, per-cell minimum of signed_distance
// 186-224) on the GPU, bit-identical to the reference fp64 code.
//
// Exactness: every fp64 operation is an explicit round-to-nearest intrinsic
// (no FMA contraction), in the reference's operation order; the Gaussian
// taps are computed on the host exactly like the reference (std::exp, then
// renormalised) and only the convolutions run on the device.  The SDF build
// evaluates, per cell, every path boundary and every obstacle that its
// bounding circle cannot exclude; skipping a polygon whose signed distance is
// provably >= the running minimum leaves the minimum unchanged, so the result
// equals the all-polygon minimum bit for bit.
//
// Layout: one thread per cell, 32 x 8 cells per CTA (row-major grid, x
// fastest, so the row reads of the x-pass and the column reads of the y-pass
// are both coalesced across a warp); the polygon table (vertices, bounding
// circles) is staged once per CTA in shared memory when it fits.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <limits>
#include <vector>

#include "tmpc_b200.h"

namespace tmpcb {
int set_global_error(int code, const char* msg);  // ctx.cu
}

namespace {

using tmpcb::set_global_error;

constexpr int kTx = 32, kTy = 8;

__device__ __forceinline__ double dsub(double a, double b) { return __dadd_rn(a, -b); }

// ---- gaussian_smooth --------------------------------------------------------
// acc = sum_k w[k] * src(clamp(i + k)) in k order (terrain.hpp:121-124 / 129-132)
template <bool AlongX>
__global__ void __launch_bounds__(kTx * kTy) gauss_pass(const double* __restrict__ src,
                                                        double* __restrict__ dst, int nx, int ny,
                                                        const double* __restrict__ w,
                                                        int radius) {
  const int i = blockIdx.x * kTx + threadIdx.x, j = blockIdx.y * kTy + threadIdx.y;
  if (i >= nx || j >= ny) return;
  double acc = 0.0;
  for (int k = -radius; k <= radius; ++k) {
    double v;
    if (AlongX) {
      v = __ldg(src + static_cast<size_t>(j) * nx + min(max(i + k, 0), nx - 1));
    } else {
      v = __ldg(src + static_cast<size_t>(min(max(j + k, 0), ny - 1)) * nx + i);
    }
    acc = __dadd_rn(acc, __dmul_rn(__ldg(w + k + radius), v));
  }
  dst[static_cast<size_t>(j) * nx + i] = acc;
}

// ---- build_sdist_map --------------------------------------------------------
// point_segment_distance (terrain.hpp:186-194)
__device__ __forceinline__ double seg_dist(double px, double py, double ax, double ay, double bx,
                                           double by) {
  const double abx = dsub(bx, ax), aby = dsub(by, ay);
  const double len2 = __dadd_rn(__dmul_rn(abx, abx), __dmul_rn(aby, aby));
  if (len2 == 0.0) {
    const double dx = dsub(px, ax), dy = dsub(py, ay);
    return __dsqrt_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)));
  }
  const double dot = __dadd_rn(__dmul_rn(dsub(px, ax), abx), __dmul_rn(dsub(py, ay), aby));
  const double t = fmin(fmax(__ddiv_rn(dot, len2), 0.0), 1.0);
  const double qx = dsub(px, __dadd_rn(ax, __dmul_rn(abx, t)));
  const double qy = dsub(py, __dadd_rn(ay, __dmul_rn(aby, t)));
  return __dsqrt_rn(__dadd_rn(__dmul_rn(qx, qx), __dmul_rn(qy, qy)));
}

// signed_distance (terrain.hpp:215-224) with point_in_polygon (196-209)
__device__ double signed_dist(double px, double py, const double2* v, int n, int kind) {
  double d = __longlong_as_double(0x7ff0000000000000LL);
  bool inside = false;
  for (int i = 0, j = n - 1; i < n; j = i++) {
    const double2 a = v[i], b = v[i + 1 == n ? 0 : i + 1], c = v[j];
    d = fmin(d, seg_dist(px, py, a.x, a.y, b.x, b.y));
    if ((a.y > py) != (c.y > py)) {
      const double x_at =
          __dadd_rn(c.x, __dmul_rn(__ddiv_rn(dsub(py, c.y), dsub(a.y, c.y)), dsub(a.x, c.x)));
      if (px < x_at) inside = !inside;
    }
  }
  const bool violating = kind == 0 ? inside : !inside;
  return violating ? -d : d;
}

struct __align__(16) Circ {
  double x, y, z, pad;  // bounding circle centre (x, y), radius z
};

struct PolyTable {
  const int* off;       // n_poly + 1 vertex offsets
  const double2* vert;  // vertices
  const int* kind;      // 0 obstacle, 1 path boundary
  const Circ* circ;     // bounding circles
  int n_poly, n_vert;
};

__global__ void __launch_bounds__(kTx * kTy) sdist_kernel(PolyTable T, int nx, int ny, double ox,
                                                          double oy, double res, int use_smem,
                                                          double* __restrict__ out) {
  extern __shared__ Circ smem[];
  const double2* vert = T.vert;
  const Circ* circ = T.circ;
  if (use_smem) {  // stage the polygon table: every cell of the CTA reads all of it
    Circ* sc = smem;
    double2* sv = reinterpret_cast<double2*>(smem + T.n_poly);
    const int tid = threadIdx.y * kTx + threadIdx.x;
    for (int q = tid; q < T.n_poly; q += kTx * kTy) sc[q] = T.circ[q];
    for (int q = tid; q < T.n_vert; q += kTx * kTy) sv[q] = T.vert[q];
    __syncthreads();
    vert = sv;
    circ = sc;
  }
  const int i = blockIdx.x * kTx + threadIdx.x, j = blockIdx.y * kTy + threadIdx.y;
  if (i >= nx || j >= ny) return;
  // cell centre exactly as the reference: origin + resolution * index
  const double x = __dadd_rn(ox, __dmul_rn(res, static_cast<double>(i)));
  const double y = __dadd_rn(oy, __dmul_rn(res, static_cast<double>(j)));
  double d = __longlong_as_double(0x7ff0000000000000LL);
  for (int k = 0; k < T.n_poly; ++k) {
    const int kind = T.kind ? __ldg(T.kind + k) : 0;
    if (kind == 0) {
      // obstacle: outside its bounding circle the signed distance is
      // positive and >= |p - c| - r; skip when that provably exceeds d
      const Circ c = circ[k];
      const double dx = x - c.x, dy = y - c.y;
      const double thr = fmax(d, 0.0) + c.z + 1e-9;
      if (dx * dx + dy * dy > thr * thr * (1.0 + 1e-12)) continue;
    }
    const int o = __ldg(T.off + k);
    d = fmin(d, signed_dist(x, y, vert + o, __ldg(T.off + k + 1) - o, kind));
  }
  out[static_cast<size_t>(j) * nx + i] = d;
}

struct DevBuf {
  void* p = nullptr;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

int cuda_fail(cudaError_t e, const char* what) {
  char buf[256];
  std::snprintf(buf, sizeof buf, "%s: %s", what, cudaGetErrorString(e));
  return set_global_error(TMPC_ERR_RUNTIME, buf);
}

#define PREP_TRY(expr, what)                 \
  do {                                       \
    const cudaError_t e_ = (expr);           \
    if (e_ != cudaSuccess) return cuda_fail(e_, what); \
  } while (0)

}  // namespace

extern "C" {

int tmpc_gaussian_smooth(int32_t device, const double* heights, int32_t nx, int32_t ny,
                         double resolution, double sigma_m, double* out) {
  if (!heights || !out || nx < 1 || ny < 1 || !(resolution > 0.0))
    return set_global_error(TMPC_ERR_CONFIG, "gaussian_smooth: bad grid");
  if (sigma_m < 0.0) return set_global_error(TMPC_ERR_CONFIG, "gaussian_smooth: sigma must be >= 0");
  const size_t n = static_cast<size_t>(nx) * ny;
  if (sigma_m == 0.0) {  // terrain.hpp:106
    std::copy(heights, heights + n, out);
    return TMPC_OK;
  }
  // taps exactly as terrain.hpp:108-116 (host fp64, no contraction)
  const double sigma_c = sigma_m / resolution;
  const int radius = static_cast<int>(std::ceil(3.0 * sigma_c));
  if (radius > (1 << 20)) return set_global_error(TMPC_ERR_CONFIG, "gaussian_smooth: sigma too large");
  std::vector<double> w(2 * static_cast<size_t>(radius) + 1);
  double sum = 0.0;
  for (int k = -radius; k <= radius; ++k) {
    w[k + radius] = std::exp(-0.5 * (k * k) / (sigma_c * sigma_c));
    sum += w[k + radius];
  }
  for (double& v : w) v /= sum;
  PREP_TRY(cudaSetDevice(device), "gaussian_smooth: cudaSetDevice");
  DevBuf a, b, dw;
  PREP_TRY(cudaMalloc(&a.p, n * sizeof(double)), "gaussian_smooth: cudaMalloc");
  PREP_TRY(cudaMalloc(&b.p, n * sizeof(double)), "gaussian_smooth: cudaMalloc");
  PREP_TRY(cudaMalloc(&dw.p, w.size() * sizeof(double)), "gaussian_smooth: cudaMalloc");
  PREP_TRY(cudaMemcpy(a.p, heights, n * sizeof(double), cudaMemcpyHostToDevice), "gaussian_smooth: H2D");
  PREP_TRY(cudaMemcpy(dw.p, w.data(), w.size() * sizeof(double), cudaMemcpyHostToDevice),
           "gaussian_smooth: H2D");
  const dim3 blk(kTx, kTy), grd((nx + kTx - 1) / kTx, (ny + kTy - 1) / kTy);
  gauss_pass<true><<<grd, blk>>>(a.as<double>(), b.as<double>(), nx, ny, dw.as<double>(), radius);
  gauss_pass<false><<<grd, blk>>>(b.as<double>(), a.as<double>(), nx, ny, dw.as<double>(), radius);
  PREP_TRY(cudaGetLastError(), "gaussian_smooth: launch");
  PREP_TRY(cudaMemcpy(out, a.p, n * sizeof(double), cudaMemcpyDeviceToHost), "gaussian_smooth: D2H");
  return TMPC_OK;
}

int tmpc_build_sdist_map_gpu(int32_t device, int32_t nx, int32_t ny, double origin_x,
                             double origin_y, double resolution, int32_t n_poly,
                             const int32_t* poly_off, const double* verts, const int32_t* kinds,
                             double* out) {
  if (nx < 1 || ny < 1 || !(resolution > 0.0) || n_poly < 0 || !out)
    return set_global_error(TMPC_ERR_CONFIG, "build_sdist_map: bad grid");
  const size_t n = static_cast<size_t>(nx) * ny;
  if (n_poly == 0) {  // has_features == false: every cell +inf (terrain.hpp:252-254)
    std::fill(out, out + n, std::numeric_limits<double>::infinity());
    return TMPC_OK;
  }
  if (!poly_off || !verts) return set_global_error(TMPC_ERR_CONFIG, "build_sdist_map: no polygons");
  const int n_vert = poly_off[n_poly];
  // bounding circles about the vertex centroid (host, tiny)
  std::vector<double> circ(4 * static_cast<size_t>(n_poly), 0.0);
  for (int k = 0; k < n_poly; ++k) {
    const int nv = poly_off[k + 1] - poly_off[k];
    if (nv < 3 || poly_off[k] < 0 || poly_off[k + 1] > n_vert)
      return set_global_error(TMPC_ERR_CONFIG, "perimeter: needs at least 3 vertices");
    const double* v = verts + 2 * poly_off[k];
    double sx = 0, sy = 0;
    for (int q = 0; q < nv; ++q) {
      sx += v[2 * q];
      sy += v[2 * q + 1];
    }
    const double cx = sx / nv, cy = sy / nv;
    double rr = 0;
    for (int q = 0; q < nv; ++q) rr = std::max(rr, std::hypot(v[2 * q] - cx, v[2 * q + 1] - cy));
    circ[4 * k] = cx;
    circ[4 * k + 1] = cy;
    circ[4 * k + 2] = rr * (1.0 + 1e-12) + 1e-12;
  }
  PREP_TRY(cudaSetDevice(device), "build_sdist_map: cudaSetDevice");
  DevBuf doff, dvert, dkind, dcirc, dout;
  PREP_TRY(cudaMalloc(&doff.p, (n_poly + 1) * sizeof(int)), "build_sdist_map: cudaMalloc");
  PREP_TRY(cudaMalloc(&dvert.p, 2 * static_cast<size_t>(n_vert) * sizeof(double)),
           "build_sdist_map: cudaMalloc");
  PREP_TRY(cudaMalloc(&dcirc.p, circ.size() * sizeof(double)), "build_sdist_map: cudaMalloc");
  PREP_TRY(cudaMalloc(&dout.p, n * sizeof(double)), "build_sdist_map: cudaMalloc");
  PREP_TRY(cudaMemcpy(doff.p, poly_off, (n_poly + 1) * sizeof(int), cudaMemcpyHostToDevice),
           "build_sdist_map: H2D");
  PREP_TRY(cudaMemcpy(dvert.p, verts, 2 * static_cast<size_t>(n_vert) * sizeof(double),
                      cudaMemcpyHostToDevice),
           "build_sdist_map: H2D");
  PREP_TRY(cudaMemcpy(dcirc.p, circ.data(), circ.size() * sizeof(double), cudaMemcpyHostToDevice),
           "build_sdist_map: H2D");
  if (kinds) {
    PREP_TRY(cudaMalloc(&dkind.p, n_poly * sizeof(int)), "build_sdist_map: cudaMalloc");
    PREP_TRY(cudaMemcpy(dkind.p, kinds, n_poly * sizeof(int), cudaMemcpyHostToDevice),
             "build_sdist_map: H2D");
  }
  PolyTable T{doff.as<int>(), dvert.as<double2>(), dkind.as<int>(), dcirc.as<Circ>(), n_poly,
              n_vert};
  const size_t smem = static_cast<size_t>(n_poly) * sizeof(Circ) +
                      static_cast<size_t>(n_vert) * sizeof(double2);
  const int use_smem = smem <= 200 * 1024;
  if (use_smem)
    PREP_TRY(cudaFuncSetAttribute(sdist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)),
             "build_sdist_map: smem attribute");
  const dim3 blk(kTx, kTy), grd((nx + kTx - 1) / kTx, (ny + kTy - 1) / kTy);
  sdist_kernel<<<grd, blk, use_smem ? smem : 0>>>(T, nx, ny, origin_x, origin_y, resolution,
                                                   use_smem, dout.as<double>());
  PREP_TRY(cudaGetLastError(), "build_sdist_map: launch");
  PREP_TRY(cudaMemcpy(out, dout.p, n * sizeof(double), cudaMemcpyDeviceToHost),
           "build_sdist_map: D2H");
  return TMPC_OK;
}

}  // extern "C"
