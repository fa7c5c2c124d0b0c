// ehmg_solver.cu -- host runtime of the B200 multigrid path and its C ABI.
//
// C++ host code drives hand-written sm_100a kernels (ehmg_kernels.cuh,
// ehmg_stencil3d.cuh) on one CUDA stream per handle:
//   * OpHandle      -- operator.hpp:40 OpData on HBM (packed cell media)
//   * VankaHandle   -- vanka.hpp:27 VankaSmoother (device factor cache)
//   * MgHandle      -- multigrid.hpp:70 Multigrid (re-discretised levels,
//                      V/W/K cycles, exact coarsest solve via an LU-derived
//                      inverse resident in HBM)
//   * Fgmres        -- krylov.hpp:65 fgmres on device vectors with host
//                      Givens/Hessenberg bookkeeping
// Everything the reference does per cycle runs on the GPU; the host only
// sequences launches and makes the Krylov control decisions.

#include <cuda_runtime.h>
#include <cublas_v2.h>
#include <cusolverDn.h>

#include <algorithm>
#include <cmath>
#include <complex>
#include <random>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/ehmg_b200.h"
#include "ehmg_comm.cuh"
#include "ehmg_kernels.cuh"
#include "ehmg_media.cuh"
#include "ehmg_stencil2d.cuh"
#include "ehmg_stencil3d.cuh"
#include "ehmg_stencil3d_rr.cuh"
#include "ehmg_stencil3d_sp.cuh"

namespace ehmg {

// ------------------------------------------------------------------ errors
struct Err : std::runtime_error {
  int code;
  Err(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
static thread_local std::string g_last_error;

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess)                                                                 \
      throw Err(EHMG_ECUDA, std::string("cuda: ") + cudaGetErrorString(e_) + " at " #x);  \
  } while (0)
#define CKS(x)                                                                         \
  do {                                                                                 \
    cusolverStatus_t e_ = (x);                                                         \
    if (e_ != CUSOLVER_STATUS_SUCCESS)                                                 \
      throw Err(EHMG_ECUDA, "cusolver status " + std::to_string((int)e_) + " at " #x); \
  } while (0)

template <class F>
static int guard(F&& f) {
  try {
    f();
    return EHMG_OK;
  } catch (const Err& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return EHMG_ERUNTIME;
  }
}

// --------------------------------------------------------------- profiling
// Optional per-launch CUDA-event timing (bench roofline): events recorded on
// the launching stream around every kernel of the cycle, tagged with the
// kernel name and the multigrid level.
struct ProfRec {
  const char* name;
  int level;
  cudaEvent_t a, b;
};
static bool g_prof = false;
static thread_local int g_level = -1;
static std::vector<ProfRec> g_recs;
struct Prof {
  ProfRec r{};
  cudaStream_t s;
  bool on;
  Prof(const char* name, cudaStream_t s_) : s(s_), on(g_prof) {
    if (!on) return;
    r.name = name;
    r.level = g_level;
    cudaEventCreate(&r.a);
    cudaEventCreate(&r.b);
    cudaEventRecord(r.a, s);
  }
  ~Prof() {
    if (!on) return;
    cudaEventRecord(r.b, s);
    g_recs.push_back(r);
  }
};

// ----------------------------------------------------------------- memory
template <class T>
struct DBuf {
  T* p = nullptr;
  int64_t n = 0;
  DBuf() = default;
  explicit DBuf(int64_t n_) { alloc(n_); }
  void alloc(int64_t n_) {
    release();
    n = n_;
    if (n > 0) CK(cudaMalloc(&p, sizeof(T) * n));
  }
  void zero(cudaStream_t s) {
    if (n) CK(cudaMemsetAsync(p, 0, sizeof(T) * n, s));
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  ~DBuf() { release(); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
};

static void validate_grid(int nd, const int* dims, double h) {
  if (nd != 2 && nd != 3) throw Err(EHMG_EINVAL, "grid: 2D or 3D only");
  if (!(h > 0)) throw Err(EHMG_EINVAL, "grid: h must be positive");
  for (int a = 0; a < nd; ++a)
    if (dims[a] < 2) throw Err(EHMG_EINVAL, "grid: need >= 2 cells per axis");
}

// media.hpp:27 MediaModel::validate
static void validate_media(int64_t n, const double* lam, const double* mu, const double* rho,
                           const double* gam) {
  for (int64_t i = 0; i < n; ++i) {
    if (!(rho[i] > 0)) throw Err(EHMG_EINVAL, "media: rho must be positive");
    if (!(mu[i] > 0)) throw Err(EHMG_EINVAL, "media: mu must be positive");
    if (!(lam[i] + mu[i] > 0)) throw Err(EHMG_EINVAL, "media: lambda+mu must be positive");
    if (!(gam[i] >= 0)) throw Err(EHMG_EINVAL, "media: gamma must be nonnegative");
  }
}

// Cell media views: packed {mu, rho, gamma, 1/(lambda+mu)} per cell for the
// generic kernels, and the same four fields as consecutive arrays (SoA) for
// the TMA-staged 3D stencil.
struct MediaRef {
  const Cell* packed;
  const double* soa;
  const float* soaf;  // float copy of soa (single-precision hierarchy), or null
};

__global__ void k_d2f(int64_t n, const double* __restrict__ in, float* __restrict__ out) {
  GRID_STRIDE(i, n) out[i] = (float)in[i];
}

__global__ void k_media_soa(int64_t n, const Cell* __restrict__ in, double* __restrict__ out) {
  GRID_STRIDE(i, n) {
    const Cell c = in[i];
    out[i] = c.x;
    out[n + i] = c.y;
    out[2 * n + i] = c.z;
    out[3 * n + i] = c.w;
  }
}

// Raw cell media on the device (lambda, mu, rho, gamma) + packed forms.
struct DevMedia {
  DBuf<double> raw[4];
  DBuf<Cell> packed;
  DBuf<double> soa;
  DBuf<float> soaf;
  MediaRef ref() const { return MediaRef{packed.p, soa.p, soaf.p}; }
  // float SoA for the complex64 stencil (the double SoA is released)
  void make_float(int64_t n, cudaStream_t s) {
    soaf.alloc(4 * n);
    k_d2f<<<grid_for(4 * n), kThreads, 0, s>>>(4 * n, soa.p, soaf.p);
    CK(cudaGetLastError());
  }
  void upload(int64_t n, const double* const* f, cudaStream_t s) {
    for (int q = 0; q < 4; ++q) {
      raw[q].alloc(n);
      CK(cudaMemcpyAsync(raw[q].p, f[q], sizeof(double) * n, cudaMemcpyHostToDevice, s));
    }
    pack(n, s);
  }
  void pack(int64_t n, cudaStream_t s) {
    packed.alloc(n);
    k_pack_media<<<grid_for(n), kThreads, 0, s>>>(n, raw[0].p, raw[1].p, raw[2].p, raw[3].p,
                                                   packed.p);
    CK(cudaGetLastError());
    soa.alloc(4 * n);
    k_media_soa<<<grid_for(n), kThreads, 0, s>>>(n, packed.p, soa.p);
    CK(cudaGetLastError());
  }
  void coarsen_into(const Geo& gf, DevMedia& out, const Geo& gc, cudaStream_t s) const {
    for (int q = 0; q < 4; ++q) out.raw[q].alloc(gc.ncells);
    k_coarsen_media<<<grid_for(gc.ncells), kThreads, 0, s>>>(
        gf.nd, gf.n[0], gf.n[1], gf.n[2], gc.ncells, raw[0].p, raw[1].p, raw[2].p, raw[3].p,
        out.raw[0].p, out.raw[1].p, out.raw[2].p, out.raw[3].p);
    CK(cudaGetLastError());
    out.pack(gc.ncells, s);
  }
  void drop_raw() {
    for (auto& r : raw) r.release();
  }
  // raw arrays copied from another (global) media set, then packed
  void copy_from(const DevMedia& o, int64_t n, cudaStream_t s) {
    for (int q = 0; q < 4; ++q) {
      raw[q].alloc(n);
      CK(cudaMemcpyAsync(raw[q].p, o.raw[q].p, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    }
    pack(n, s);
  }
  // the cell-plane window [z0, z1) of a global media set (packed + SoA)
  void window_of(const DevMedia& o, const Geo& gg, int z0, int z1, cudaStream_t s) {
    const int64_t plane = (int64_t)gg.n[0] * gg.n[1], n = plane * (z1 - z0);
    packed.alloc(n);
    CK(cudaMemcpyAsync(packed.p, o.packed.p + plane * z0, sizeof(Cell) * n, cudaMemcpyDeviceToDevice, s));
    soa.alloc(4 * n);
    k_media_soa<<<grid_for(n), kThreads, 0, s>>>(n, packed.p, soa.p);
    CK(cudaGetLastError());
  }
};

// ----------------------------------------------------------- level kernels
// r = b - A x (b != null) or y = A x.
// Rows of output planes [z_lo, z_hi) only (TMA path; the generic kernels
// always write every row, a correct superset).
static void launch_residual(const Geo& g, const OpPar& P, const MediaRef& mr, const cplx* x,
                            const cplx* b, cplx* y, cudaStream_t s, int z_lo = 0, int z_hi = -1) {
  Prof pf(b ? "residual" : "apply", s);
  const Cell* m = mr.packed;
  if (g.nd == 3 && stencil3d_supported(g)) {
    launch_stencil3d(g, P, mr.soa, x, b, y, s, z_lo, z_hi);
  } else if (g.nd == 3) {
    k_apply_generic<3><<<grid_for(g.ndofs, 148 * 64), kThreads, 0, s>>>(g, P, m, x, b, y);
  } else {
    launch_stencil2d<cplx>(g, P, m, x, b, y, s);
  }
  CK(cudaGetLastError());
}
// complex64 fields: the 3D stencil computes in float; the generic rows
// evaluate in double and store complex64.
static void launch_residual(const Geo& g, const OpPar& P, const MediaRef& mr, const cplxf* x,
                            const cplxf* b, cplxf* y, cudaStream_t s, int z_lo = 0, int z_hi = -1) {
  Prof pf(b ? "residual" : "apply", s);
  const Cell* m = mr.packed;
  if (g.nd == 3 && g.n[0] % 2 == 0 && mr.soaf) {
    launch_stencil3d(g, P, mr.soaf, x, b, y, s, z_lo, z_hi);
  } else if (g.nd == 3) {
    k_apply_generic<3, cplxf><<<grid_for(g.ndofs, 148 * 64), kThreads, 0, s>>>(g, P, m, x, b, y);
  } else {
    launch_stencil2d<cplxf>(g, P, m, x, b, y, s);
  }
  CK(cudaGetLastError());
}

template <class V>
static void launch_transfer(const Geo& gf, const Geo& gc, bool restricting, const V* in, V* out,
                            bool accumulate, cudaStream_t s) {
  const Geo& gto = restricting ? gc : gf;
  Prof pf(restricting ? "restrict" : "prolong_add", s);
  if (gf.nd == 3) {
    const dim3 blk(32, 8);
    for (int c = 0; c < 4; ++c) {
      const int d0 = gto.n[0] + (c == 0), d1 = gto.n[1] + (c == 1), d2 = gto.n[2] + (c == 2);
      // prolongation: zc fine planes per thread (fewer on small levels, to keep the SMs busy)
      const int zc = d2 >= 128 ? 16 : 4;
      const dim3 grd((d0 + 31) / 32, (d1 + 7) / 8, restricting ? d2 : (d2 + zc - 1) / zc);
      if (restricting) {
        if (c == 0) k_restrict3<0, V><<<grd, blk, 0, s>>>(gf, gc, in, out);
        else if (c == 1) k_restrict3<1, V><<<grd, blk, 0, s>>>(gf, gc, in, out);
        else if (c == 2) k_restrict3<2, V><<<grd, blk, 0, s>>>(gf, gc, in, out);
        else k_restrict3<3, V><<<grd, blk, 0, s>>>(gf, gc, in, out);
      } else {
        if (c == 0) k_prolong3<0, V><<<grd, blk, 0, s>>>(gf, gc, in, out, accumulate, zc);
        else if (c == 1) k_prolong3<1, V><<<grd, blk, 0, s>>>(gf, gc, in, out, accumulate, zc);
        else if (c == 2) k_prolong3<2, V><<<grd, blk, 0, s>>>(gf, gc, in, out, accumulate, zc);
        else k_prolong3<3, V><<<grd, blk, 0, s>>>(gf, gc, in, out, accumulate, zc);
      }
    }
  } else {
    k_transfer<2, V><<<grid_for(gto.ndofs, 148 * 64), kThreads, 0, s>>>(gf, gc, restricting, in, out,
                                                                        accumulate);
  }
  CK(cudaGetLastError());
}

static Geo coarse_geo(const Geo& g) {
  int d[3];
  for (int a = 0; a < g.nd; ++a) d[a] = g.n[a] / 2;
  return make_geo(g.nd, d, 2.0 * g.h);
}

// Vanka factor cache + red-black / lexicographic sweeps on one level.
// Red-black colour = fused residual kernel (stencil) + coalesced local
// solve/update kernel reading the colour-major SoA factor cache.
struct Smoother {
  int full = 1, stride = 0;  // stride: reference (vanka.hpp:35) entries per cell
  VkPar vk;
  DBuf<cplx> soa, res;
  DBuf<cplxf> soaf, resf;  // complex64 cache / residual (single-precision hierarchy)
  // stiffness cache (k_vanka_update_k): 3D full Vanka on complex128 levels / z-windows
  DBuf<double> ksoa;
  const double* mrho = nullptr;
  const double* mgam = nullptr;
  bool kpath = false;
  // factor dictionary (complex128): id per colour cell + table of the distinct entry sets
  DBuf<unsigned> didx;
  DBuf<cplx> dtab;
  DBuf<cplxf> dtabf;  // complex64 hierarchy
  const cplx* dict_table(const cplx*) const { return dtab.p; }
  const cplxf* dict_table(const cplxf*) const { return dtabf.p; }
  bool dict = false;
  int dict_sets = 0;
  // Deduplicate the compact cache when the level has few distinct entry sets
  // (homogeneous regions, sponge depth classes): exact, see k_vkd_*.
  void build_dictionary(const Geo& g, cudaStream_t s) {
    dict = false;
    dict_sets = 0;
    const char* ev = getenv("EHMG_VANKA_DICT");
    if (ev && ev[0] == '0') return;
    const int64_t nt = colour_threads(g);
    const int cs = g.nd * (full ? 4 : 2) + 1;
    if (2 * nt < 8192 || 2 * nt >= ((int64_t)1 << 32)) return;
    // at least 8 cells per set on average, and a table of at most 32 MB (L2-resident)
    const int64_t umax = std::min<int64_t>(2 * nt / 8, ((int64_t)32 << 20) / (cs * (int64_t)sizeof(cplx)));
    if (umax < 1) return;
    unsigned M = 1024;
    while ((int64_t)M < 8 * umax) M <<= 1;
    DBuf<unsigned long long> keys(M);
    DBuf<unsigned> rep(M), dense(M), slot(2 * nt);
    DBuf<int> flags(2), next(1);
    CK(cudaMemsetAsync(keys.p, 0, sizeof(unsigned long long) * M, s));
    CK(cudaMemsetAsync(rep.p, 0xff, sizeof(unsigned) * M, s));
    CK(cudaMemsetAsync(flags.p, 0, sizeof(int) * 2, s));
    CK(cudaMemsetAsync(next.p, 0, sizeof(int), s));
    VkDict D{keys.p, rep.p, dense.p, slot.p, nullptr, flags.p, M, (unsigned)umax};
    k_vkd_insert<<<grid_for(2 * nt, 148 * 64), kThreads, 0, s>>>(nt, cs, soa.p, D);
    k_vkd_verify<<<grid_for(2 * nt, 148 * 64), kThreads, 0, s>>>(nt, cs, soa.p, D, next.p);
    CK(cudaGetLastError());
    int hf[2] = {0, 0};
    CK(cudaMemcpyAsync(hf, flags.p, sizeof(hf), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (hf[0] || hf[1] < 1 || hf[1] > umax) return;
    didx.alloc(2 * nt);
    D.idx = didx.p;
    dtab.alloc((int64_t)hf[1] * cs);
    k_vkd_fill<<<grid_for(2 * nt, 148 * 64), kThreads, 0, s>>>(nt, cs, soa.p, D, dtab.p);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(s));
    dict = true;
    dict_sets = hf[1];
    if (getenv("EHMG_DEBUG"))
      fprintf(stderr, "ehmg: factor dictionary %d x %d x %d: %d entry sets for %lld cells (%.1f MB table)\n", g.n[0],
              g.n[1], g.n[2], dict_sets, (long long)(2 * nt), dict_sets * cs * 16.0 / 1048576.0);
  }
  // switch this smoother to complex64 storage (the double cache is released)
  void make_float(const Geo& g, cudaStream_t s) {
    soaf.alloc(soa.n);
    k_convert<cplxf, cplx><<<grid_for(soa.n, 148 * 64), kThreads, 0, s>>>(soa.n, soa.p, soaf.p);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(s));
    soa.release();
    res.release();
    ksoa.release();
    kpath = false;
    if (dict) {  // the dictionary follows: the table rounded like the per-cell entries, same ids
      dtabf.alloc(dtab.n);
      k_convert<cplxf, cplx><<<grid_for(dtab.n, 148 * 64), kThreads, 0, s>>>(dtab.n, dtab.p, dtabf.p);
      CK(cudaGetLastError());
      CK(cudaStreamSynchronize(s));
    }
    dtab.release();
    resf.alloc(g.ndofs);
  }
  const cplx* cache(const cplx*) const { return soa.p; }
  const cplxf* cache(const cplxf*) const { return soaf.p; }
  cplx* resbuf(const cplx*) { return res.p; }
  cplxf* resbuf(const cplxf*) { return resf.p; }
  // Cache for the cells of `gg` (global grid, global packed media m), or of
  // its z-window [z0, z1) when z1 >= 0; sweeps then run on the window geometry.
  void build(const Geo& gg, const OpPar& P, const Cell* m, int full_, cudaStream_t s, int z0 = 0,
             int z1 = -1, const double* media_soa = nullptr) {
    full = full_;
    stride = gg.nd * ((full ? 4 : 2) + 4) + 1;
    const Geo g = z1 < 0 ? gg : make_window(gg, z0, z1);
    const int nz = z1 < 0 ? gg.n[2] : z1 - z0;
    {
      // factorise in z-chunks of <= 8M cells: the reference-layout scratch
      // (25 complex per 3D cell) never exceeds ~3.4 GB, so 513^3 builds fit
      const int64_t plane = (int64_t)g.n[0] * g.n[1];
      const int cz_max = g.nd == 3 ? (int)std::max<int64_t>(1, ((int64_t)8 << 20) / plane) : 1;
      const int nzc = g.nd == 3 ? nz : 1;
      DBuf<cplx> aos(plane * std::min(cz_max, nzc) * stride);
      DBuf<int> bad(1);
      bad.zero(s);
      const int64_t nt = colour_threads(g);
      vk = make_vkpar(g, P);
      soa.alloc(2 * nt * (g.nd * (full ? 4 : 2) + 1));
      for (int c0 = 0; c0 < nzc; c0 += cz_max) {
        const int cz = std::min(cz_max, nzc - c0);
        if (g.nd == 3) {
          k_vanka_build<3><<<grid_for(plane * cz, 148 * 64), kThreads, 0, s>>>(gg, P, m, full, aos.p, bad.p,
                                                                             z0 + c0, cz);
          k_vanka_to_soa<3><<<grid_for(2 * (nt / g.n[2]) * cz, 148 * 64), kThreads, 0, s>>>(g, full, aos.p, soa.p,
                                                                                          c0, cz);
        } else {
          k_vanka_build<2><<<grid_for(g.ncells, 148 * 64), kThreads, 0, s>>>(gg, P, m, full, aos.p, bad.p, 0, 1);
          k_vanka_to_soa<2><<<grid_for(2 * nt, 148 * 64), kThreads, 0, s>>>(g, full, aos.p, soa.p, 0, 1);
        }
        CK(cudaGetLastError());
      }
      int hb = 0;
      CK(cudaMemcpyAsync(&hb, bad.p, sizeof(int), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      if (hb) throw Err(EHMG_ERUNTIME, "vanka: singular local cell system");
      build_dictionary(g, s);
      // optional stiffness cache for the colour updates (EHMG_VANKA_KCACHE=1): 12% fewer HBM bytes
      // per update, measured time-neutral (+2% at 256^3, -1% at 512^3 under the power cap), so off
      const char* ev = getenv("EHMG_VANKA_KCACHE");
      kpath = false;
      if (g.nd == 3 && full && media_soa && g.n[0] % 2 == 0 && ev && ev[0] == '1') {
        ksoa.alloc(2 * nt * kVkK);
        mrho = media_soa + g.ncells;
        mgam = media_soa + 2 * g.ncells;
        k_vanka_kcache<<<grid_for(2 * nt, 148 * 64), kThreads, 0, s>>>(g, vk, mrho, mgam, soa.p, ksoa.p);
        CK(cudaGetLastError());
        kpath = true;
      }
    }
    res.alloc(g.ndofs);
  }
  // reference (AoS, vanka.hpp:72) layout of the cache, for inspection
  void cache_aos(const Geo& g, cplx* out, cudaStream_t s) const {
    const int64_t nt = colour_threads(g);
    if (g.nd == 3) k_vanka_expand<3><<<grid_for(2 * nt, 148 * 64), kThreads, 0, s>>>(g, vk, full, soa.p, out);
    else k_vanka_expand<2><<<grid_for(2 * nt, 148 * 64), kThreads, 0, s>>>(g, vk, full, soa.p, out);
    CK(cudaGetLastError());
  }
  // xzero: x is zero on entry, so the first colour's residual is b itself
  // (b - H*0 == b exactly) and its operator apply is skipped.
  template <class V>
  void sweep(const Geo& g, const OpPar& P, const MediaRef& mr, const V* b, V* x, double w, int order,
             cudaStream_t s, bool xzero = false) {
    const Cell* m = mr.packed;
    if (order == 0) {
      if constexpr (sizeof(V) == sizeof(cplx)) {
        if (g.nd == 3) k_vanka_lex<3><<<1, 1, 0, s>>>(g, P, vk, m, full, soa.p, b, x, w);
        else k_vanka_lex<2><<<1, 1, 0, s>>>(g, P, vk, m, full, soa.p, b, x, w);
        CK(cudaGetLastError());
        return;
      } else {
        throw Err(EHMG_EINVAL, "mixed precision: lexicographic Vanka sweeps are not supported");
      }
    }
    for (int color = 0; color < 2; ++color) colour_phase(g, P, mr, b, x, w, color, s, xzero && color == 0);
  }
  // colour 0 of a sweep from a zero iterate can also write x's zeros itself
  // (no memset) when every cell's x-partner has the other colour
  static bool zero_fill_ok(const Geo& g) { return g.n[0] % 2 == 0 && g.zoff == 0; }
  // One red-black colour (global parity `color`; windows shift the local parity).
  template <class V>
  void colour_phase(const Geo& g, const OpPar& P, const MediaRef& mr, const V* b, V* x, double w, int color,
                    cudaStream_t s, bool xzero = false) {
    V* rb = resbuf(b);
    const V* r = xzero ? b : rb;
    if (!xzero) launch_residual(g, P, mr, x, b, rb, s);
    update(g, r, x, w, color, s, xzero && zero_fill_ok(g));
  }
  // Vanka update of one colour from a precomputed residual r.
  template <class V>
  void update(const Geo& g, const V* r, V* x, double w, int color, cudaStream_t s, bool xzero = false) {
    const int64_t nt = colour_threads(g);
    const int lc = color ^ (g.zoff & 1);
    const V* cq = cache(r);
    Prof pf("vanka_update", s);
    if constexpr (sizeof(V) == sizeof(cplx)) {
      if (kpath && g.nd == 3) {
        (xzero ? k_vanka_update_k<true> : k_vanka_update_k<false>)<<<(int)std::min<int64_t>((nt + kVkkThreads - 1) / kVkkThreads, 148 * 64), kVkkThreads, 0, s>>>(
            g, vk, ksoa.p, mrho, mgam, r, lc, w, x);
        CK(cudaGetLastError());
        return;
      }
    }
    constexpr int nth = vk_threads<V>();
    const int nblk = (int)std::min<int64_t>((nt + nth - 1) / nth, 148 * 64);
    if (dict) {
#ifndef EHMG_VKD_BLOCKS_PER_SM
#define EHMG_VKD_BLOCKS_PER_SM 2
#endif
      // blocks resident per SM x EHMG_VKD_BLOCKS_PER_SM (complex128: one 384-thread block per SM)
      const int nblk = (int)std::min<int64_t>((nt + nth - 1) / nth,
                                              148 * EHMG_VKD_BLOCKS_PER_SM * (sizeof(V) == sizeof(cplx) ? 1 : 2));
      const V* tab = dict_table(r);
      // (an L2 access-policy window pinning the table was measured: 0.81 vs 0.56 ms, so not used)
      if (g.nd == 3)
        (xzero ? k_vanka_update<3, V, true, true> : k_vanka_update<3, V, false, true>)<<<nblk, nth, 0, s>>>(
            g, vk, full, cq, r, lc, w, x, didx.p, tab);
      else
        (xzero ? k_vanka_update<2, V, true, true> : k_vanka_update<2, V, false, true>)<<<nblk, nth, 0, s>>>(
            g, vk, full, cq, r, lc, w, x, didx.p, tab);
      CK(cudaGetLastError());
      return;
    }
    if (g.nd == 3)
      (xzero ? k_vanka_update<3, V, true> : k_vanka_update<3, V, false>)<<<nblk, nth, 0, s>>>(
          g, vk, full, cq, r, lc, w, x, (const unsigned*)nullptr, (const V*)nullptr);
    else
      (xzero ? k_vanka_update<2, V, true> : k_vanka_update<2, V, false>)<<<nblk, nth, 0, s>>>(
          g, vk, full, cq, r, lc, w, x, (const unsigned*)nullptr, (const V*)nullptr);
    CK(cudaGetLastError());
  }
};

// --------------------------------------------------------------- BLAS-1
struct Blas {
  cudaStream_t s = nullptr;
  DBuf<double2> partial;
  DBuf<unsigned> counter;
  DBuf<double> scal;  // [0..1] last result, [2..3] coef, [4..] hessenberg column
  DBuf<double> partial3;
  DBuf<double> partialN;  // classical Gram-Schmidt passes: 2 kGsMax + 1 per block
  DBuf<double> corr;      // re-orthogonalisation corrections of one Arnoldi step
  void init(cudaStream_t s_, int ncol) {
    s = s_;
    partial.alloc(kRedBlocks);
    partial3.alloc(3 * kRedBlocks);
    partialN.alloc((2 * kGsMax + 1) * kRedBlocks);
    corr.alloc(2 * kGsMax);
    counter.alloc(1);
    counter.zero(s);
    scal.alloc(8 + 2 * (ncol + 2));
    scal.zero(s);
  }
  double* res() { return scal.p; }
  double* coef() { return scal.p + 2; }
  double* wpre() { return scal.p + 4; }
  double* wn() { return scal.p + 6; }
  double* hcol(int i) { return scal.p + 8 + 2 * i; }
  // Distributed vectors (z-slab windows): reductions cover only the owned
  // index ranges and are summed across ranks in rank order (deterministic).
  NodeComm* comm = nullptr;
  std::vector<std::pair<int64_t, int64_t>> owned;
  DBuf<double> tmp;
  void reduce(int mode, int64_t n, const cplx* x, const cplx* y, double* out, double* coef_,
              double* hacc) {
    if (owned.empty()) {
      k_reduce<<<kRedBlocks, kThreads, 0, s>>>(mode, n, x, y, partial.p, counter.p, out, coef_, hacc);
      CK(cudaGetLastError());
      return;
    }
    if (!tmp.n) tmp.alloc(2);
    double h[2] = {0, 0};
    for (auto& rg : owned) {
      k_reduce<<<kRedBlocks, kThreads, 0, s>>>(mode, rg.second - rg.first, x + rg.first, y ? y + rg.first : nullptr,
                                               partial.p, counter.p, tmp.p, nullptr, nullptr);
      CK(cudaGetLastError());
      double part[2];
      CK(cudaMemcpyAsync(part, tmp.p, sizeof(part), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      h[0] += part[0];
      h[1] += part[1];
    }
    if (comm) comm->allreduce(h, 2);
    CK(cudaMemcpyAsync(out, h, sizeof(h), cudaMemcpyHostToDevice, s));
    if (coef_) {
      const double c[2] = {-h[0], -h[1]};
      CK(cudaMemcpyAsync(coef_, c, sizeof(c), cudaMemcpyHostToDevice, s));
    }
    if (hacc) {
      double a[2];
      CK(cudaMemcpyAsync(a, hacc, sizeof(a), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      a[0] += h[0];
      a[1] += h[1];
      CK(cudaMemcpyAsync(hacc, a, sizeof(a), cudaMemcpyHostToDevice, s));
    }
    CK(cudaStreamSynchronize(s));
  }
  double norm_host(int64_t n, const cplx* x) {
    reduce(1, n, x, nullptr, res(), nullptr, nullptr);
    double h[2];
    CK(cudaMemcpyAsync(h, res(), sizeof(h), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return std::sqrt(h[0]);
  }
  void axpy(int64_t n, cplx a, const double* ap, const cplx* x, cplx* y) {
    k_axpy<<<grid_for(n, 148 * 16), kThreads, 0, s>>>(n, a.x, a.y, ap, x, y);
    CK(cudaGetLastError());
  }
  void scale_copy(int64_t n, double sc, const cplx* x, cplx* y) {
    k_scale_copy<<<grid_for(n, 148 * 16), kThreads, 0, s>>>(n, sc, nullptr, 0, x, y);
    CK(cudaGetLastError());
  }
  void sub(int64_t n, const cplx* b, const cplx* t, cplx* r) {
    k_sub<<<grid_for(n, 148 * 16), kThreads, 0, s>>>(n, b, t, r);
    CK(cudaGetLastError());
  }
};

// ----------------------------------------------------------------- FGMRES
// krylov.hpp:65, restated on device vectors. The preconditioned vectors
// are stored (flexible variant); Arnoldi uses modified Gram-Schmidt with one
// optional re-orthogonalisation pass; Givens rotations on the host.
struct Fgmres {
  int64_t n = 0;
  int m = 0;
  std::vector<std::unique_ptr<DBuf<cplx>>> V, Z;
  DBuf<cplx> r, w;
  Blas blas;

  void init(int64_t n_, int m_, cudaStream_t s) {
    if (n == n_ && m == m_) return;
    // marked initialised only once every buffer exists: a failed cudaMalloc
    // part-way (2m+3 level-0 vectors) leaves n = m = 0, so the next call
    // allocates again instead of indexing missing buffers
    n = 0;
    m = 0;
    V.clear();
    Z.clear();
    for (int i = 0; i <= m_; ++i) V.emplace_back(new DBuf<cplx>(n_));
    for (int i = 0; i < m_; ++i) Z.emplace_back(new DBuf<cplx>(n_));
    r.alloc(n_);
    w.alloc(n_);
    blas.init(s, m_ + 1);
    n = n_;
    m = m_;
  }

  using Fn = std::function<void(const cplx*, cplx*)>;

  ehmg_krylov_result run(const Fn& A, const Fn& M, const cplx* b, cplx* x,
                         const ehmg_krylov_options& opt, std::vector<double>& hist) {
    cudaStream_t s = blas.s;
    ehmg_krylov_result res{1, 0, 1.0, 0};
    const double bnorm = blas.norm_host(n, b);
    if (bnorm == 0.0) {
      CK(cudaMemsetAsync(x, 0, sizeof(cplx) * n, s));
      res.status = 0;
      res.relres = 0.0;
      return res;
    }
    const double target = opt.rtol * bnorm;
    A(x, w.p);
    blas.sub(n, b, w.p, r.p);
    double beta = blas.norm_host(n, r.p);
    hist.push_back(beta / bnorm);
    res.relres = beta / bnorm;
    if (beta <= target) {
      res.status = 0;
      return res;
    }
    std::vector<cplx> H((size_t)(m + 1) * m, mk(0, 0));
    auto HH = [&](int i, int j) -> cplx& { return H[(size_t)i * m + j]; };
    std::vector<double> gc(m, 0.0);
    std::vector<cplx> gs(m, mk(0, 0)), g(m + 1, mk(0, 0)), y(m, mk(0, 0));
    std::vector<double> hbuf(8 + 2 * (m + 2)), hcorr(2 * kGsMax);
    double prev_cycle = beta;
    int stall = 0;
    while (res.iterations < opt.max_iterations) {
      blas.scale_copy(n, 1.0 / beta, r.p, V[0]->p);
      for (auto& q : g) q = mk(0, 0);
      g[0] = mk(beta, 0);
      bool broke = false;
      int j = 0;
      while (j < m && res.iterations < opt.max_iterations) {
        M(V[j]->p, Z[j]->p);
        A(Z[j]->p, w.p);
        const bool cgs = blas.owned.empty() && opt.orthogonalization == 0 && j + 1 <= kGsMax;
        GsVecs gv{};
        if (cgs) {
          // classical passes: all <V[i], w> and |w|^2 in one pass, then
          // w -= sum_i h_i V[i] and |w|^2. (Taking the projections of the
          // updated w in the same pass -- mode 2 -- saves the first pass of a
          // re-orthogonalisation but slows every update pass 0.98 -> 1.10 ms
          // at 256^3 under ncu, and the test rarely fires: not used.)
          for (int i = 0; i <= j; ++i) gv.v[i] = V[i]->p;
          gs_launch<1>(0, j + 1, n, gv, w.p, nullptr, blas.partialN.p, blas.counter.p, blas.wpre(),
                       blas.hcol(0), nullptr, s);
          CK(cudaGetLastError());
          gs_launch<1>(1, j + 1, n, gv, w.p, blas.hcol(0), blas.partialN.p, blas.counter.p, blas.wn(),
                       nullptr, nullptr, s);
          CK(cudaGetLastError());
        } else if (blas.owned.empty()) {
          // pipelined MGS: pass i applies the projection on V[i-1] and takes <V[i], w>
          double* cf[2] = {blas.coef(), blas.res()};
          for (int i = 0; i <= j + 1; ++i) {
            k_mgs<<<kRedBlocks, kThreads, 0, s>>>(n, i > 0 ? cf[(i - 1) & 1] : nullptr,
                                                  i > 0 ? V[i - 1]->p : nullptr, w.p,
                                                  i <= j ? V[i]->p : nullptr, i == 0 || i == j + 1,
                                                  blas.partial3.p, blas.counter.p,
                                                  i == 0 ? blas.wpre() : (i == j + 1 ? blas.wn() : nullptr),
                                                  i <= j ? blas.hcol(i) : nullptr, i <= j ? cf[i & 1] : nullptr);
            CK(cudaGetLastError());
          }
        } else {
          blas.reduce(1, n, w.p, nullptr, blas.wpre(), nullptr, nullptr);
          for (int i = 0; i <= j; ++i) {
            blas.reduce(0, n, V[i]->p, w.p, blas.hcol(i), blas.coef(), nullptr);
            blas.axpy(n, mk(0, 0), blas.coef(), V[i]->p, w.p);
          }
          blas.reduce(1, n, w.p, nullptr, blas.wn(), nullptr, nullptr);
        }
        CK(cudaMemcpyAsync(hbuf.data(), blas.scal.p, sizeof(double) * (8 + 2 * (j + 1)),
                           cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        const double wpre = std::sqrt(hbuf[4]);
        double wn = std::sqrt(hbuf[6]);
        if (wn < 0.70710678 * wpre) {  // one re-orthogonalisation pass
          if (cgs) {
            // corrections c_i = <V[i], w> in one pass, w -= sum_i c_i V[i]
            // (H += c on the host below)
            gs_launch<1>(0, j + 1, n, gv, w.p, nullptr, blas.partialN.p, blas.counter.p, nullptr, blas.corr.p,
                         nullptr, s);
            CK(cudaGetLastError());
            gs_launch<1>(1, j + 1, n, gv, w.p, blas.corr.p, blas.partialN.p, blas.counter.p, blas.wn(), nullptr,
                         nullptr, s);
            CK(cudaGetLastError());
            CK(cudaMemcpyAsync(hcorr.data(), blas.corr.p, sizeof(double) * 2 * (j + 1), cudaMemcpyDeviceToHost, s));
          } else if (blas.owned.empty()) {
            // pipelined like the first pass; the corrections accumulate into H
            double* cf[2] = {blas.coef(), blas.res()};
            for (int i = 0; i <= j + 1; ++i) {
              k_mgs<<<kRedBlocks, kThreads, 0, s>>>(n, i > 0 ? cf[(i - 1) & 1] : nullptr,
                                                    i > 0 ? V[i - 1]->p : nullptr, w.p,
                                                    i <= j ? V[i]->p : nullptr, i == j + 1, blas.partial3.p,
                                                    blas.counter.p, i == j + 1 ? blas.wn() : nullptr,
                                                    i <= j ? blas.hcol(m + 1) : nullptr, i <= j ? cf[i & 1] : nullptr,
                                                    i <= j ? blas.hcol(i) : nullptr);
              CK(cudaGetLastError());
            }
          } else {
            for (int i = 0; i <= j; ++i) {
              blas.reduce(0, n, V[i]->p, w.p, blas.res(), blas.coef(), blas.hcol(i));
              blas.axpy(n, mk(0, 0), blas.coef(), V[i]->p, w.p);
            }
            blas.reduce(1, n, w.p, nullptr, blas.wn(), nullptr, nullptr);
          }
          CK(cudaMemcpyAsync(hbuf.data(), blas.scal.p, sizeof(double) * (8 + 2 * (j + 1)),
                             cudaMemcpyDeviceToHost, s));
          CK(cudaStreamSynchronize(s));
          wn = std::sqrt(hbuf[6]);
          if (cgs)  // H += c, the addition the device-side accumulation performed
            for (int i = 0; i < 2 * (j + 1); ++i) hbuf[8 + i] += hcorr[i];
        }
        for (int i = 0; i <= j; ++i) HH(i, j) = mk(hbuf[8 + 2 * i], hbuf[9 + 2 * i]);
        HH(j + 1, j) = mk(wn, 0);
        ++res.iterations;
        if (!(wn > 1e-14 * (wpre > 0 ? wpre : 1.0))) {
          broke = true;
        } else {
          blas.scale_copy(n, 1.0 / wn, w.p, V[j + 1]->p);
        }
        for (int i = 0; i < j; ++i) {
          const cplx a = HH(i, j), bb = HH(i + 1, j);
          HH(i, j) = gc[i] * a + gs[i] * bb;
          HH(i + 1, j) = -(conj(gs[i]) * a) + gc[i] * bb;
        }
        const cplx h1 = HH(j, j), h2 = HH(j + 1, j);
        const double t = std::sqrt(abs2(h1) + abs2(h2));
        const double ah1 = std::hypot(h1.x, h1.y);
        if (t == 0.0) {
          gc[j] = 1.0;
          gs[j] = mk(0, 0);
        } else if (ah1 == 0.0) {
          gc[j] = 0.0;
          gs[j] = mk(1, 0);
        } else {
          gc[j] = ah1 / t;
          gs[j] = (mk(h1.x / ah1, h1.y / ah1) * conj(h2)) * (1.0 / t);
        }
        HH(j, j) = gc[j] * h1 + gs[j] * h2;
        HH(j + 1, j) = mk(0, 0);
        const cplx gj = g[j];
        g[j] = gc[j] * gj;
        g[j + 1] = -(conj(gs[j]) * gj);
        const double est = std::hypot(g[j + 1].x, g[j + 1].y);
        hist.push_back(est / bnorm);
        ++j;
        if (broke || est <= target) break;
      }
      for (int i = j - 1; i >= 0; --i) {
        cplx v = g[i];
        for (int l = i + 1; l < j; ++l) v -= HH(i, l) * y[l];
        if (std::hypot(HH(i, i).x, HH(i, i).y) == 0.0) {
          res.status = 2;
          return res;
        }
        y[i] = cdiv(v, HH(i, i));
      }
      if (j <= 16) {
        MultiAxpy ma;
        ma.m = j;
        for (int i = 0; i < j; ++i) {
          ma.c[2 * i] = y[i].x;
          ma.c[2 * i + 1] = y[i].y;
          ma.z[i] = Z[i]->p;
        }
        k_multi_axpy<<<grid_for(n, 148 * 16), kThreads, 0, s>>>(n, ma, x);
        CK(cudaGetLastError());
      } else {
        for (int i = 0; i < j; ++i) blas.axpy(n, y[i], nullptr, Z[i]->p, x);
      }
      A(x, w.p);
      blas.sub(n, b, w.p, r.p);
      beta = blas.norm_host(n, r.p);
      res.relres = beta / bnorm;
      if (beta <= target) {
        res.status = 0;
        return res;
      }
      if (broke) {
        res.status = 2;
        return res;
      }
      if (beta > opt.stall_factor * prev_cycle) {
        if (++stall >= opt.stall_cycles) {
          res.status = 3;
          return res;
        }
      } else {
        stall = 0;
      }
      prev_cycle = beta;
    }
    res.status = 1;
    return res;
  }
};

}  // namespace ehmg

using namespace ehmg;

// ------------------------------------------------------------- handles
struct ehmg_op_s {
  int dev = 0;
  cudaStream_t s = nullptr;
  Geo g;
  OpPar P;
  DevMedia media;
  DBuf<cplx> hx, hy, hb;  // staging for EHMG_HOST calls
  ~ehmg_op_s() {
    if (s) cudaStreamDestroy(s);
  }
};

struct ehmg_vanka_s {
  ehmg_op op;
  Smoother sm;
};

struct Level {
  Geo g;
  OpPar P;
  DevMedia media;
  Smoother sm;
  DBuf<cplx> r, bc, ec;
  DBuf<cplxf> rf, bcf, ecf;  // complex64 level vectors (single-precision hierarchy)
  Fgmres inner;              // K-cycle acceleration on this level
};
// level vectors by element type
template <class V> struct LB;
template <> struct LB<cplx> {
  static cplx* r(Level& L) { return L.r.p; }
  static cplx* bc(Level& L) { return L.bc.p; }
  static cplx* ec(Level& L) { return L.ec.p; }
};
template <> struct LB<cplxf> {
  static cplxf* r(Level& L) { return L.rf.p; }
  static cplxf* bc(Level& L) { return L.bcf.p; }
  static cplxf* ec(Level& L) { return L.ecf.p; }
};

struct ehmg_mg_s {
  int dev = 0;
  cudaStream_t s = nullptr;
  ehmg_mg_options opt;
  std::vector<std::unique_ptr<Level>> L;
  // Coarsest solve with the pressure eliminated (ehmg_kernels.cuh k_schur_*):
  // ainv = row-major S^-1 of the displacement Schur complement (ncu rows),
  // plus the gradient / divergence entries and 1/Dpp of the assembled matrix.
  DBuf<cplx> ainv;
  int64_t nco = 0, ncu = 0;
  DBuf<int> s_gcol, s_dcnt, s_dcol;
  DBuf<cplx> s_gval, s_dval, s_rdp, s_bu;
  DBuf<cplxf> s_buf;
  cplx* schur_scratch(const cplx*) { return s_bu.p; }
  cplxf* schur_scratch(const cplxf*) { return s_buf.p; }
  // FGMRES workspace of solves preconditioned by this hierarchy (2m+3
  // level-0 vectors), kept between solves so the basis buffers -- and the
  // CUDA graphs of the cycle, keyed by (r, z) -- are reused; released with
  // the handle
  std::unique_ptr<Fgmres> solve_ws;
  DBuf<cplx> hx, hy;
  // precision 1: the hierarchy holds complex64 fields, caches and coarsest
  // inverse (experiments.hpp:241 MixedPrecondition); r and z stay complex128.
  int prec = 0;
  DBuf<cplxf> ainvf, rin, zout;
  const cplx* coarse_inv(const cplx*) const { return ainv.p; }
  const cplxf* coarse_inv(const cplxf*) const { return ainvf.p; }
  // Row-partitioned coarsest solve (one z-slab per process): this rank keeps
  // rows [c_r0, c_r1) of S^-1, computes those rows of u and all-gathers u
  // (coarse_gather pushes the block into every rank's x, then a barrier).
  int64_t c_r0 = 0, c_r1 = -1;
  std::function<void(void* x, size_t esize)> coarse_gather;
  void split_coarse(int64_t r0, int64_t r1, cudaStream_t st) {
    const int64_t rows = r1 - r0;
    if (prec == 0) {
      DBuf<cplx> blk(rows * ncu);
      CK(cudaMemcpyAsync(blk.p, ainv.p + r0 * ncu, sizeof(cplx) * rows * ncu, cudaMemcpyDeviceToDevice, st));
      CK(cudaStreamSynchronize(st));
      std::swap(ainv.p, blk.p);
      std::swap(ainv.n, blk.n);
    } else {
      DBuf<cplxf> blk(rows * ncu);
      CK(cudaMemcpyAsync(blk.p, ainvf.p + r0 * ncu, sizeof(cplxf) * rows * ncu, cudaMemcpyDeviceToDevice, st));
      CK(cudaStreamSynchronize(st));
      std::swap(ainvf.p, blk.p);
      std::swap(ainvf.n, blk.n);
    }
    c_r0 = r0;
    c_r1 = r1;
  }
  // CUDA graphs of whole preconditioner applications, one per (r, z) pair:
  // a V(2,2) cycle is ~75 launches, many of them short on the coarse levels.
  struct GraphEntry {
    const cplx* r;
    cplx* z;
    int uses;
    cudaGraphExec_t exec;
  };
  std::vector<GraphEntry> graphs;
  // precondition_many: host<->device copy streams, staging pairs, events
  cudaStream_t s_in = nullptr, s_out = nullptr;
  DBuf<cplx> rst[2], zst[2];
  cudaEvent_t ev_in[2] = {nullptr, nullptr}, ev_comp[2] = {nullptr, nullptr}, ev_out[2] = {nullptr, nullptr};
  ~ehmg_mg_s() {
    for (auto& e : graphs)
      if (e.exec) cudaGraphExecDestroy(e.exec);
    L.clear();
    for (int k = 0; k < 2; ++k)
      for (cudaEvent_t e : {ev_in[k], ev_comp[k], ev_out[k]})
        if (e) cudaEventDestroy(e);
    if (s_in) cudaStreamDestroy(s_in);
    if (s_out) cudaStreamDestroy(s_out);
    if (s) cudaStreamDestroy(s);
  }

  // xzero: x is known to be zero on entry (precondition, coarse corrections)
  template <class V>
  void cycle_t(int l, const V* b, V* x, bool xzero);
  void cycle_at(int l, const cplx* b, cplx* x, bool xzero = false) { cycle_t<cplx>(l, b, x, xzero); }
  // K-cycle coarse correction on this hierarchy's level 0 (the cycle_t
  // K branch one level up): inner FGMRES with A_0 and M = cycle_at(0, ...).
  // The z-slab mode calls it for its first agglomerated level.
  void kcycle_top(const cplx* b, cplx* x) {
    Level& lv = *L[0];
    // inner K-cycle solves keep the reference's MGS order (few, small vectors)
    ehmg_krylov_options ko{opt.k_inner_iterations, opt.k_inner_iterations, opt.k_inner_rtol, 0.99, 2, 1};
    lv.inner.init(lv.g.ndofs, opt.k_inner_iterations, s);
    CK(cudaMemsetAsync(x, 0, sizeof(cplx) * lv.g.ndofs, s));
    std::vector<double> hist;
    Fgmres::Fn A = [&](const cplx* in, cplx* out) {
      launch_residual(lv.g, lv.P, lv.media.ref(), in, nullptr, out, s);
    };
    Fgmres::Fn M = [&](const cplx* in, cplx* out) { cycle_at(0, in, out, true); };
    lv.inner.run(A, M, b, x, ko, hist);
  }
  void precondition_direct(const cplx* r, cplx* z) {
    const int64_t n = L[0]->g.ndofs;
    if (prec == 0) {
      cycle_at(0, r, z, true);  // cycle_t clears z where the first sweep does not
      return;
    }
    // multigrid.hpp:310 convert_field in, float cycle, convert out
    k_convert<cplxf, cplx><<<grid_for(n, 148 * 64), kThreads, 0, s>>>(n, r, rin.p);
    CK(cudaGetLastError());
    cycle_t<cplxf>(0, rin.p, zout.p, true);
    k_convert<cplx, cplxf><<<grid_for(n, 148 * 64), kThreads, 0, s>>>(n, zout.p, z);
    CK(cudaGetLastError());
  }
  static bool graphs_enabled() {
    static int on = -1;
    if (on < 0) {
      const char* e = getenv("EHMG_GRAPHS");
      on = (e && atoi(e) == 0) ? 0 : 1;
    }
    return on == 1;
  }
  // The K-cycle's inner Krylov makes host decisions (not capturable); the
  // per-launch profiler records events between kernels. Both run direct.
  void precondition(const cplx* r, cplx* z) {
    if (g_prof || opt.cycle == 3 || !graphs_enabled()) {
      precondition_direct(r, z);
      return;
    }
    GraphEntry* e = nullptr;
    for (auto& q : graphs)
      if (q.r == r && q.z == z) e = &q;
    if (!e) {
      if (graphs.size() >= 32) {
        if (graphs.front().exec) cudaGraphExecDestroy(graphs.front().exec);
        graphs.erase(graphs.begin());
      }
      graphs.push_back({r, z, 0, nullptr});
      e = &graphs.back();
    }
    if (++e->uses == 1) {  // first use runs direct (lazy per-kernel setup happens outside capture)
      precondition_direct(r, z);
      return;
    }
    if (!e->exec) {
      cudaGraph_t gph;
      CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
      try {
        precondition_direct(r, z);
      } catch (...) {
        cudaGraph_t dead = nullptr;
        cudaStreamEndCapture(s, &dead);
        if (dead) cudaGraphDestroy(dead);
        throw;
      }
      CK(cudaStreamEndCapture(s, &gph));
      CK(cudaGraphInstantiate(&e->exec, gph, 0));
      CK(cudaGraphDestroy(gph));
    }
    CK(cudaGraphLaunch(e->exec, s));
  }
};

// multigrid.hpp:217 cycle_at
template <class V>
void ehmg_mg_s::cycle_t(int l, const V* b, V* x, bool xzero) {
  const int nl = (int)L.size();
  g_level = l;
  if (l + 1 == nl) {
    Prof pf("coarse_solve", s);
    V* bu = schur_scratch(b);
    k_schur_rhs<V><<<grid_for(ncu, 148 * 8), kThreads, 0, s>>>(ncu, b, s_gcol.p, s_gval.p, s_rdp.p, bu);
    CK(cudaGetLastError());
    if (c_r1 < 0) {
      k_gemv_rows<V><<<grid_for(ncu * 32, 148 * 64), kThreads, 0, s>>>(ncu, coarse_inv(b), bu, x, ncu);
      CK(cudaGetLastError());
    } else {
      const int64_t rows = c_r1 - c_r0;
      if (rows > 0)
        k_gemv_rows<V><<<grid_for(rows * 32, 148 * 64), kThreads, 0, s>>>(ncu, coarse_inv(b), bu, x + c_r0, rows);
      CK(cudaGetLastError());
      coarse_gather(x, sizeof(V));  // every rank holds all of u
    }
    k_schur_p<V><<<grid_for((nco - ncu) * 32, 148 * 8), kThreads, 0, s>>>(ncu, nco - ncu, b, s_dcnt.p, s_dcol.p,
                                                                        s_dval.p, s_rdp.p, x);
    CK(cudaGetLastError());
    return;
  }
  Level& lev = *L[l];
  Level& nxt = *L[l + 1];
  // xzero: x holds zero or nothing yet; the first red-black colour writes
  // every DOF itself where it can, otherwise x is cleared here
  if (xzero && (opt.sweep == 0 || opt.nu1 == 0 || !Smoother::zero_fill_ok(lev.g)))
    CK(cudaMemsetAsync(x, 0, sizeof(V) * lev.g.ndofs, s));
  for (int q = 0; q < opt.nu1; ++q)
    lev.sm.sweep(lev.g, lev.P, lev.media.ref(), b, x, opt.damping, opt.sweep, s, xzero && q == 0);
  V* const lr = LB<V>::r(lev);
  V* const nbc = LB<V>::bc(nxt);
  V* const nec = LB<V>::ec(nxt);
  launch_residual(lev.g, lev.P, lev.media.ref(), x, b, lr, s);
  launch_transfer(lev.g, nxt.g, true, (const V*)lr, nbc, false, s);
  const bool next_coarsest = (l + 2 == nl);
  switch (opt.cycle) {
    case 0:
    case 1:
      cycle_t<V>(l + 1, nbc, nec, true);
      break;
    case 2:
      cycle_t<V>(l + 1, nbc, nec, true);
      if (!next_coarsest) cycle_t<V>(l + 1, nbc, nec, false);
      break;
    default:
      if (next_coarsest) {
        cycle_t<V>(l + 1, nbc, nec, true);
      } else if constexpr (sizeof(V) != sizeof(cplx)) {
        throw Err(EHMG_EINVAL, "mixed precision: K-cycles are not supported");
      } else {
        ehmg_krylov_options ko{opt.k_inner_iterations, opt.k_inner_iterations, opt.k_inner_rtol,
                               0.99, 2, 1};
        nxt.inner.init(nxt.g.ndofs, opt.k_inner_iterations, s);
        CK(cudaMemsetAsync(nec, 0, sizeof(V) * nxt.g.ndofs, s));  // the inner solve's initial guess
        std::vector<double> hist;
        Fgmres::Fn A = [&](const cplx* in, cplx* out) {
          launch_residual(nxt.g, nxt.P, nxt.media.ref(), in, nullptr, out, s);
        };
        Fgmres::Fn M = [&](const cplx* in, cplx* out) { cycle_at(l + 1, in, out, true); };
        nxt.inner.run(A, M, nxt.bc.p, nxt.ec.p, ko, hist);
      }
      break;
  }
  g_level = l;
  launch_transfer(lev.g, nxt.g, false, (const V*)nec, x, true, s);
  for (int q = 0; q < opt.nu2; ++q) lev.sm.sweep(lev.g, lev.P, lev.media.ref(), b, x, opt.damping, opt.sweep, s);
}

// ------------------------------------------------------------ helpers
static int64_t ndofs_of(int nd, const int* dims) {
  int d[3] = {dims[0], dims[1], nd == 3 ? dims[2] : 1};
  return make_geo(nd, d, 1.0).ndofs;
}

static void to_dev(const double* src, DBuf<cplx>& stage, int64_t n, int where, cudaStream_t s,
                   const cplx** out) {
  if (where == EHMG_DEVICE) {
    *out = reinterpret_cast<const cplx*>(src);
    return;
  }
  if (stage.n < n) stage.alloc(n);
  CK(cudaMemcpyAsync(stage.p, src, sizeof(cplx) * n, cudaMemcpyHostToDevice, s));
  *out = stage.p;
}

static cplx* out_dev(double* dst, DBuf<cplx>& stage, int64_t n, int where) {
  if (where == EHMG_DEVICE) return reinterpret_cast<cplx*>(dst);
  if (stage.n < n) stage.alloc(n);
  return stage.p;
}

static void from_dev(double* dst, const cplx* dev, int64_t n, int where, cudaStream_t s) {
  if (where == EHMG_DEVICE) {
    CK(cudaStreamSynchronize(s));
    return;
  }
  CK(cudaMemcpyAsync(dst, dev, sizeof(cplx) * n, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
}

static void check_device() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
    throw Err(EHMG_ECUDA, "no CUDA device: the B200 path has no CPU fallback");
}

// Exact coarsest solve: assemble A row-major (== A^T column-major), take the
// gradient / divergence entries and 1/Dpp, form S^T = Auu^T - Apu^T Dpp^-1
// Aup^T in place (cuBLAS ZGEMM on the column-major view), LU it with
// cuSOLVER and solve against the identity, leaving S^-1 row-major (ncu^2).
static void build_coarse_inverse(const Geo& g, const OpPar& P, const Cell* m, ehmg_mg_s& mg, cudaStream_t s) {
  const int64_t N = g.ndofs, Nu = g.off[g.nd], Np = N - Nu;
  // The coarsest operator is dense in HBM during the build (N^2 + Np Nu +
  // Nu^2 complex): allow it while that fits in 80% of free memory (N ~ 60000
  // on an idle B200), the reference's SparseLU budget aside.
  size_t free_b = 0, total_b = 0;
  CK(cudaMemGetInfo(&free_b, &total_b));
  const double need = ((double)N * N + (double)Np * Nu + (double)Nu * Nu) * sizeof(cplx) + 64.0 * N * sizeof(cplx);
  if (need > 0.8 * (double)free_b)
    throw Err(EHMG_ERANGE, "assemble_sparse: coarsest grid of " + std::to_string(N) +
                               " DOFs exceeds the dense-LU memory budget");
  DBuf<cplx> A(N * N);
  A.zero(s);
  const int nwin = g.nd == 3 ? 125 : 25;
  const int64_t total = N * (g.nd + 1) * nwin;
  if (g.nd == 3) k_coarse_matrix<3><<<grid_for(total, 148 * 64), kThreads, 0, s>>>(g, P, m, A.p);
  else k_coarse_matrix<2><<<grid_for(total, 148 * 64), kThreads, 0, s>>>(g, P, m, A.p);
  CK(cudaGetLastError());
  mg.nco = N;
  mg.ncu = Nu;
  mg.s_gcol.alloc(2 * Nu);
  mg.s_gval.alloc(2 * Nu);
  mg.s_dcnt.alloc(Np);
  mg.s_dcol.alloc(Np * kSchurDiv);
  mg.s_dval.alloc(Np * kSchurDiv);
  mg.s_rdp.alloc(Np);
  DBuf<int> err(1);
  err.zero(s);
  k_schur_extract_grad<<<grid_for(Nu * 32, 148 * 32), kThreads, 0, s>>>(N, Nu, A.p, mg.s_gcol.p, mg.s_gval.p, err.p);
  k_schur_extract_div<<<grid_for(Np * 32, 148 * 32), kThreads, 0, s>>>(N, Nu, A.p, mg.s_dcnt.p, mg.s_dcol.p,
                                                                      mg.s_dval.p, mg.s_rdp.p, err.p);
  CK(cudaGetLastError());
  int herr = 0;
  CK(cudaMemcpyAsync(&herr, err.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (herr != 0) throw Err(EHMG_ERUNTIME, "multigrid: unexpected coarsest-operator structure (pressure block)");
  {
    DBuf<cplx> Y(Np * Nu);
    k_schur_scale_rows<<<grid_for(Np * Nu, 148 * 64), kThreads, 0, s>>>(N, Nu, A.p, mg.s_rdp.p, Y.p);
    CK(cudaGetLastError());
    cublasHandle_t hb;
    if (cublasCreate(&hb) != CUBLAS_STATUS_SUCCESS) throw Err(EHMG_ECUDA, "cublas: create failed");
    cublasSetStream(hb, s);
    const cuDoubleComplex mone = make_cuDoubleComplex(-1.0, 0.0), one = make_cuDoubleComplex(1.0, 0.0);
    const cublasStatus_t st =
        cublasZgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, (int)Nu, (int)Nu, (int)Np, &mone,
                    (const cuDoubleComplex*)(A.p + Nu * N), (int)N, (const cuDoubleComplex*)Y.p, (int)Np, &one,
                    (cuDoubleComplex*)A.p, (int)N);
    CK(cudaStreamSynchronize(s));
    cublasDestroy(hb);
    if (st != CUBLAS_STATUS_SUCCESS) throw Err(EHMG_ECUDA, "cublas: zgemm failed");
  }
  DBuf<cplx>& ainv = mg.ainv;
  ainv.alloc(Nu * Nu);
  k_identity<<<grid_for(Nu * Nu, 148 * 64), kThreads, 0, s>>>(Nu, ainv.p);
  CK(cudaGetLastError());
  cusolverDnHandle_t h;
  CKS(cusolverDnCreate(&h));
  CKS(cusolverDnSetStream(h, s));
  int lwork = 0;
  CKS(cusolverDnZgetrf_bufferSize(h, (int)Nu, (int)Nu, (cuDoubleComplex*)A.p, (int)N, &lwork));
  DBuf<cplx> work(lwork > 0 ? lwork : 1);
  DBuf<int> ipiv(Nu), info(1);
  CKS(cusolverDnZgetrf(h, (int)Nu, (int)Nu, (cuDoubleComplex*)A.p, (int)N, (cuDoubleComplex*)work.p, ipiv.p,
                       info.p));
  int hinfo = 0;
  CK(cudaMemcpyAsync(&hinfo, info.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (hinfo != 0) {
    cusolverDnDestroy(h);
    throw Err(EHMG_ERUNTIME, "multigrid: coarsest LU factorization failed");
  }
  CKS(cusolverDnZgetrs(h, CUBLAS_OP_N, (int)Nu, (int)Nu, (cuDoubleComplex*)A.p, (int)N, ipiv.p,
                       (cuDoubleComplex*)ainv.p, (int)Nu, info.p));
  CK(cudaStreamSynchronize(s));
  cusolverDnDestroy(h);
  mg.s_bu.alloc(Nu);
}

// Build a hierarchy of `nlevels` levels below grid g from host media (host)
// or from a device media set with raw arrays (src).
static std::unique_ptr<ehmg_mg_s> build_mg(const Geo& g, const double* const* host, const DevMedia* src,
                                           const OpPar& P, const ehmg_mg_options& opt, int nlevels) {
  auto mg = std::make_unique<ehmg_mg_s>();
  mg->opt = opt;
  mg->opt.n_levels = nlevels;
  CK(cudaGetDevice(&mg->dev));
  CK(cudaStreamCreateWithFlags(&mg->s, cudaStreamNonBlocking));
  cudaStream_t s = mg->s;
  const bool mixed = opt.precision == 1;
  if (opt.precision != 0 && opt.precision != 1) throw Err(EHMG_EINVAL, "multigrid: precision must be 0 or 1");
  if (mixed && opt.cycle == 3) throw Err(EHMG_EINVAL, "mixed precision: K-cycles are not supported");
  if (mixed && opt.sweep == 0)
    throw Err(EHMG_EINVAL, "mixed precision: lexicographic Vanka sweeps are not supported");
  mg->prec = mixed ? 1 : 0;
  for (int l = 0; l < nlevels; ++l) {
    auto lev = std::make_unique<Level>();
    lev->g = l == 0 ? g : coarse_geo(mg->L[l - 1]->g);
    lev->P = P;
    if (l == 0) {
      if (host) lev->media.upload(g.ncells, host, s);
      else lev->media.copy_from(*src, g.ncells, s);
    } else {
      mg->L[l - 1]->media.coarsen_into(mg->L[l - 1]->g, lev->media, lev->g, s);
    }
    const bool coarsest = (l + 1 == nlevels);
    if (!coarsest) {
      lev->sm.build(lev->g, P, lev->media.packed.p, opt.vanka_mode == 0 ? 1 : 0, s, 0, -1, lev->media.soa.p);
      if (mixed) {
        lev->sm.make_float(lev->g, s);
        lev->rf.alloc(lev->g.ndofs);
      } else {
        lev->r.alloc(lev->g.ndofs);
      }
    }
    if (l > 0) {
      if (mixed) {
        lev->bcf.alloc(lev->g.ndofs);
        lev->ecf.alloc(lev->g.ndofs);
      } else {
        lev->bc.alloc(lev->g.ndofs);
        lev->ec.alloc(lev->g.ndofs);
      }
    }
    mg->L.push_back(std::move(lev));
  }
  for (auto& lev : mg->L) lev->media.drop_raw();
  if (mixed)
    for (auto& lev : mg->L) {
      lev->media.make_float(lev->g.ncells, s);
      lev->media.soa.release();
    }
  Level& cl = *mg->L.back();
  build_coarse_inverse(cl.g, P, cl.media.packed.p, *mg, s);
  if (mixed) {
    mg->s_buf.alloc(mg->ncu);
    const int64_t nn = mg->ncu * mg->ncu;
    mg->ainvf.alloc(nn);
    k_convert<cplxf, cplx><<<grid_for(nn, 148 * 64), kThreads, 0, s>>>(nn, mg->ainv.p, mg->ainvf.p);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(s));
    mg->ainv.release();
    mg->rin.alloc(g.ndofs);
    mg->zout.alloc(g.ndofs);
  }
  CK(cudaStreamSynchronize(s));
  return mg;
}

#include "ehmg_slab.cuh"

// multigrid.hpp:143 measure_convergence_factor: stationary cycles on the
// homogeneous problem from a seeded random start (the reference's
// std::mt19937_64 / uniform(-1, 1) draws, re and im per value in component
// order), residual norm ||H x|| of the level-0 (shifted) operator.
template <class V>
static void measure_t(ehmg_mg_s& mg, uint64_t seed, const ehmg_measure_options& mo, ehmg_measure_result* res,
                      double* history, int cap) {
  typedef typename VT<V>::R Real;
  typedef std::complex<Real> C;
  Level& fl = *mg.L[0];
  const int64_t n = fl.g.ndofs;
  cudaStream_t s = mg.s;
  std::vector<C> hx((size_t)n);
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> dist(-1.0, 1.0);
  for (auto& v : hx) v = C(Real(dist(rng)), Real(dist(rng)));  // same expression as the reference
  DBuf<V> x(n), zero(n), t(n);
  DBuf<double2> partial(kRedBlocks);
  DBuf<unsigned> counter(1);
  DBuf<double> out(2);
  counter.zero(s);
  zero.zero(s);
  CK(cudaMemcpyAsync(x.p, hx.data(), sizeof(V) * n, cudaMemcpyHostToDevice, s));
  auto rnorm = [&]() {
    launch_residual(fl.g, fl.P, fl.media.ref(), (const V*)x.p, (const V*)nullptr, t.p, s);
    k_reduce<V><<<kRedBlocks, kThreads, 0, s>>>(1, n, t.p, nullptr, partial.p, counter.p, out.p, nullptr, nullptr);
    CK(cudaGetLastError());
    double h2[2];
    CK(cudaMemcpyAsync(h2, out.p, sizeof(h2), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return std::sqrt(h2[0]);
  };
  for (int i = 0; i < mo.warmup; ++i) mg.cycle_t<V>(0, zero.p, x.p, false);
  const double r0 = rnorm();
  res->factor = 0.0;
  res->cycles = 0;
  res->diverged = 0;
  res->n_history = 0;
  if (r0 == 0.0) return;
  const Real sc = Real(1.0 / r0);
  k_scale_real<V><<<grid_for(n, 148 * 64), kThreads, 0, s>>>(n, sc, x.p);
  CK(cudaGetLastError());
  std::vector<double> hist;
  double prev = 1.0;
  int growths = 0;
  while (res->cycles < mo.max_cycles) {
    mg.cycle_t<V>(0, zero.p, x.p, false);
    ++res->cycles;
    const double rn = rnorm();
    hist.push_back(rn);
    if (rn > prev) {
      if (++growths >= mo.growth_limit) {
        res->diverged = 1;
        break;
      }
    } else {
      growths = 0;
    }
    prev = rn;
    if (rn < mo.tol) break;
    if (!std::isfinite(rn) || rn > 1e12) {
      res->diverged = 1;
      break;
    }
  }
  res->factor = std::pow(hist.empty() ? 1.0 : hist.back(), 1.0 / std::max(1, res->cycles));
  res->n_history = (int)hist.size();
  for (int i = 0; i < std::min(cap, (int)hist.size()); ++i) history[i] = hist[(size_t)i];
}

// ------------------------------------------------------------------ C ABI
// krylov.hpp:45 KrylovOptions sanity: a restart of 0 would never grow the
// iteration count (the outer loop would spin), so it is rejected up front.
static void check_krylov_args(const ehmg_krylov_options* opt, const ehmg_krylov_result* res) {
  if (!opt || !res) throw Err(EHMG_EINVAL, "fgmres: null options or result");
  if (opt->restart < 1) throw Err(EHMG_EINVAL, "fgmres: restart must be >= 1");
  if (opt->max_iterations < 0) throw Err(EHMG_EINVAL, "fgmres: max_iterations must be >= 0");
  if (opt->orthogonalization != 0 && opt->orthogonalization != 1)
    throw Err(EHMG_EINVAL, "krylov: unknown orthogonalization");
}

extern "C" {

const char* ehmg_last_error(void) { return g_last_error.c_str(); }
const char* ehmg_version(void) { return "ehmg_b200 0.1 (sm_100a)"; }

int ehmg_set_device(int device) {
  return guard([&] {
    check_device();
    CK(cudaSetDevice(device));
  });
}

int ehmg_op_create(int nd, const int* dims, double h, const double* lambda, const double* mu,
                   const double* rho, const double* gamma, double beta, double omega,
                   double alpha, ehmg_op* out) {
  return guard([&] {
    validate_grid(nd, dims, h);
    check_device();
    int d[3] = {dims[0], dims[1], nd == 3 ? dims[2] : 1};
    auto op = std::make_unique<ehmg_op_s>();
    CK(cudaGetDevice(&op->dev));
    CK(cudaStreamCreateWithFlags(&op->s, cudaStreamNonBlocking));
    op->g = make_geo(nd, d, h);
    validate_media(op->g.ncells, lambda, mu, rho, gamma);
    op->P = OpPar{beta, omega * omega, alpha};
    const double* f[4] = {lambda, mu, rho, gamma};
    op->media.upload(op->g.ncells, f, op->s);
    op->media.drop_raw();
    CK(cudaStreamSynchronize(op->s));
    *out = op.release();
  });
}

int ehmg_op_destroy(ehmg_op op) {
  return guard([&] { delete op; });
}

int64_t ehmg_op_n_dofs(ehmg_op op) { return op ? op->g.ndofs : -1; }
uint64_t ehmg_op_stream(ehmg_op op) { return op ? (uint64_t)(uintptr_t)op->s : 0; }

int ehmg_apply_mixed_operator(ehmg_op op, const double* x, double* y, int where) {
  return guard([&] {
    const int64_t n = op->g.ndofs;
    const cplx* dx;
    to_dev(x, op->hx, n, where, op->s, &dx);
    cplx* dy = out_dev(y, op->hy, n, where);
    launch_residual(op->g, op->P, op->media.ref(), dx, nullptr, dy, op->s);
    from_dev(y, dy, n, where, op->s);
  });
}

int ehmg_residual(ehmg_op op, const double* b, const double* x, double* r, int where) {
  return guard([&] {
    const int64_t n = op->g.ndofs;
    const cplx *dx, *db;
    to_dev(x, op->hx, n, where, op->s, &dx);
    to_dev(b, op->hb, n, where, op->s, &db);
    cplx* dr = out_dev(r, op->hy, n, where);
    launch_residual(op->g, op->P, op->media.ref(), dx, db, dr, op->s);
    from_dev(r, dr, n, where, op->s);
  });
}

int ehmg_vanka_create(ehmg_op op, int mode, ehmg_vanka* out) {
  return guard([&] {
    auto v = std::make_unique<ehmg_vanka_s>();
    v->op = op;
    v->sm.build(op->g, op->P, op->media.packed.p, mode == 0 ? 1 : 0, op->s, 0, -1, op->media.soa.p);
    *out = v.release();
  });
}

int ehmg_vanka_destroy(ehmg_vanka v) {
  return guard([&] { delete v; });
}

int ehmg_vanka_per_cell_complex_count(ehmg_vanka v) { return v ? v->sm.stride : -1; }

int ehmg_vanka_cache(ehmg_vanka v, double* out) {
  return guard([&] {
    const Geo& g = v->op->g;
    DBuf<cplx> aos(g.ncells * v->sm.stride);
    v->sm.cache_aos(g, aos.p, v->op->s);
    CK(cudaMemcpyAsync(out, aos.p, sizeof(cplx) * aos.n, cudaMemcpyDeviceToHost, v->op->s));
    CK(cudaStreamSynchronize(v->op->s));
  });
}

int ehmg_vanka_sweep(ehmg_vanka v, const double* b, double* x, double w, int order, int nsweeps,
                     int where) {
  return guard([&] {
    ehmg_op op = v->op;
    const int64_t n = op->g.ndofs;
    const cplx* db;
    to_dev(b, op->hb, n, where, op->s, &db);
    cplx* dx;
    if (where == EHMG_DEVICE) {
      dx = reinterpret_cast<cplx*>(x);
    } else {
      if (op->hx.n < n) op->hx.alloc(n);
      CK(cudaMemcpyAsync(op->hx.p, x, sizeof(cplx) * n, cudaMemcpyHostToDevice, op->s));
      dx = op->hx.p;
    }
    for (int q = 0; q < nsweeps; ++q) v->sm.sweep(op->g, op->P, op->media.ref(), db, dx, w, order, op->s);
    from_dev(x, dx, n, where, op->s);
  });
}

static int transfer_abi(int nd, const int* dims_f, const double* in, double* out, int where,
                        bool restricting) {
  return guard([&] {
    validate_grid(nd, dims_f, 1.0);
    for (int a = 0; a < nd; ++a)
      if (dims_f[a] % 2 != 0 || dims_f[a] / 2 < 2)
        throw Err(EHMG_EINVAL, "coarsen_grid: dims must be even and >= 4");
    check_device();
    int d[3] = {dims_f[0], dims_f[1], nd == 3 ? dims_f[2] : 1};
    Geo gf = make_geo(nd, d, 1.0), gc = coarse_geo(gf);
    const int64_t nin = restricting ? gf.ndofs : gc.ndofs, nout = restricting ? gc.ndofs : gf.ndofs;
    cudaStream_t s = 0;
    DBuf<cplx> si, so;
    const cplx* di;
    to_dev(in, si, nin, where, s, &di);
    cplx* dout = out_dev(out, so, nout, where);
    launch_transfer(gf, gc, restricting, di, dout, false, s);
    from_dev(out, dout, nout, where, s);
  });
}

int ehmg_restrict_field(int nd, const int* dims_f, const double* xf, double* xc, int where) {
  return transfer_abi(nd, dims_f, xf, xc, where, true);
}
int ehmg_prolong_field(int nd, const int* dims_f, const double* xc, double* xf, int where) {
  return transfer_abi(nd, dims_f, xc, xf, where, false);
}

int ehmg_coarsen_media(int nd, const int* dims_f, const double* fine, double* coarse) {
  return guard([&] {
    validate_grid(nd, dims_f, 1.0);
    for (int a = 0; a < nd; ++a)
      if (dims_f[a] % 2 != 0 || dims_f[a] / 2 < 2)
        throw Err(EHMG_EINVAL, "coarsen_grid: dims must be even and >= 4");
    check_device();
    int d[3] = {dims_f[0], dims_f[1], nd == 3 ? dims_f[2] : 1};
    Geo gf = make_geo(nd, d, 1.0), gc = coarse_geo(gf);
    DBuf<double> in(gf.ncells), o(gc.ncells);
    CK(cudaMemcpy(in.p, fine, sizeof(double) * gf.ncells, cudaMemcpyHostToDevice));
    k_coarsen_media<<<grid_for(gc.ncells), kThreads>>>(nd, gf.n[0], gf.n[1], gf.n[2], gc.ncells,
                                                       in.p, in.p, in.p, in.p, o.p, o.p, o.p, o.p);
    CK(cudaGetLastError());
    CK(cudaMemcpy(coarse, o.p, sizeof(double) * gc.ncells, cudaMemcpyDeviceToHost));
  });
}

// media.hpp:95 (host-side media preparation; not on the per-cycle path)
// experiments.hpp:78 layered_media: the same std::mt19937_64 stream and the
// same <random> distributions, drawn in the reference's order, so one seed
// gives the reference's layers bit for bit (same C++ standard library).
int ehmg_layered_media(int nd, const int* dims, double gamma_phys, uint64_t seed, double* lambda,
                       double* mu, double* rho, double* gamma) {
  return guard([&] {
    if (nd != 2 && nd != 3) throw Err(EHMG_EINVAL, "layered_media: ndim must be 2 or 3");
    int d[3] = {dims[0], dims[1], nd == 3 ? dims[2] : 1};
    for (int a = 0; a < nd; ++a)
      if (d[a] < 1) throw Err(EHMG_EINVAL, "layered_media: dims must be positive");
    std::mt19937_64 rng(seed);
    const int depth_n = d[nd - 1];
    const int nl = std::min(std::uniform_int_distribution<int>(5, 10)(rng), depth_n);
    std::vector<int> tops{0};
    std::uniform_int_distribution<int> depth(1, depth_n - 1);
    while ((int)tops.size() < nl) {
      const int t = depth(rng);
      if (std::find(tops.begin(), tops.end(), t) == tops.end()) tops.push_back(t);
    }
    std::sort(tops.begin(), tops.end());
    std::uniform_real_distribution<double> vs(0.5, 2.0), dens(1.5, 3.0), ratio(2.0, 20.0);
    std::vector<double> lr, ll, lm;
    for (int l = 0; l < nl; ++l) {
      const double v = vs(rng), r = dens(rng), q = ratio(rng);
      const double m = r * v * v;
      lr.push_back(r);
      ll.push_back(q * m);
      lm.push_back(m);
    }
    const int64_t plane = nd == 3 ? (int64_t)d[0] * d[1] : d[0];
    for (int64_t i = 0; i < plane * depth_n; ++i) {
      const int z = (int)(i / plane);
      const int j = (int)(std::upper_bound(tops.begin(), tops.end(), z) - tops.begin()) - 1;
      rho[i] = lr[j];
      lambda[i] = ll[j];
      mu[i] = lm[j];
      gamma[i] = gamma_phys;
    }
  });
}

int ehmg_layered_grf_media(int nd, const int* dims, int n_layers, const double* ranges, double perturb,
                           double corr_cells, double gamma_phys, uint64_t seed, double* lambda, double* mu,
                           double* rho, double* gamma) {
  return guard([&] {
    if (nd != 2 && nd != 3) throw Err(EHMG_EINVAL, "layered_grf_media: ndim must be 2 or 3");
    int d[3] = {dims[0], dims[1], nd == 3 ? dims[2] : 1};
    for (int a = 0; a < nd; ++a)
      if (d[a] < 2) throw Err(EHMG_EINVAL, "layered_grf_media: need >= 2 cells per axis");
    if (n_layers < 1 || n_layers > 64) throw Err(EHMG_EINVAL, "layered_grf_media: 1..64 layers");
    for (int k = 0; k < 3; ++k)
      if (!(ranges[2 * k] > 0 && ranges[2 * k + 1] >= ranges[2 * k]))
        throw Err(EHMG_EINVAL, "layered_grf_media: ranges must be positive and ordered");
    if (!(ranges[2] * (1 - perturb) > 1.4142135623730951))
      throw Err(EHMG_EINVAL, "layered_grf_media: cp/cs must stay above sqrt(2) (lambda > 0)");
    if (!(perturb >= 0 && perturb < 1)) throw Err(EHMG_EINVAL, "layered_grf_media: perturb in [0, 1)");
    if (!(corr_cells > 0 && corr_cells <= 40)) throw Err(EHMG_EINVAL, "layered_grf_media: corr in (0, 40] cells");
    check_device();
    const LayerTable L = grf_layers(d[nd - 1], n_layers, ranges, seed);
    const GrfTaps T = grf_taps(corr_cells);
    const int R = T.R;
    const int E0 = d[0] + 2 * R, E1 = d[1] + 2 * R, E2 = nd == 3 ? d[2] + 2 * R : 1;
    const int64_t nc = (int64_t)d[0] * d[1] * d[2];
    cudaStream_t s = nullptr;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    struct SG {
      cudaStream_t s;
      ~SG() { cudaStreamDestroy(s); }
    } sg{s};
    DBuf<double> noise((int64_t)E0 * E1 * E2), t1((int64_t)d[0] * E1 * E2),
        t2(nd == 3 ? (int64_t)d[0] * d[1] * E2 : 0);
    DBuf<double> g[3] = {DBuf<double>(nc), DBuf<double>(nc), DBuf<double>(nc)};
    const int gb = 148 * 16;
    for (int f = 0; f < 3; ++f) {
      k_grf_noise<<<gb, 256, 0, s>>>((int64_t)E0 * E1 * E2, seed ^ grf_salt(f), noise.p);
      k_grf_filter<<<gb, 256, 0, s>>>(T, 0, E0, E1, E2, noise.p, t1.p);
      if (nd == 2) {
        k_grf_filter<<<gb, 256, 0, s>>>(T, 1, d[0], E1, 1, t1.p, g[f].p);
      } else {
        k_grf_filter<<<gb, 256, 0, s>>>(T, 1, d[0], E1, E2, t1.p, t2.p);
        k_grf_filter<<<gb, 256, 0, s>>>(T, 2, d[0], d[1], E2, t2.p, g[f].p);
      }
      CK(cudaGetLastError());
    }
    DBuf<double> out[4] = {DBuf<double>(nc), DBuf<double>(nc), DBuf<double>(nc), DBuf<double>(nc)};
    const int64_t plane = nd == 3 ? (int64_t)d[0] * d[1] : d[0];
    k_compose_media<<<gb, 256, 0, s>>>(L, nc, plane, perturb, gamma_phys, g[0].p, g[1].p, g[2].p, out[0].p,
                                       out[1].p, out[2].p, out[3].p);
    CK(cudaGetLastError());
    double* dst[4] = {lambda, mu, rho, gamma};
    for (int k = 0; k < 4; ++k)
      CK(cudaMemcpyAsync(dst[k], out[k].p, sizeof(double) * nc, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  });
}

int ehmg_attenuation_profile(int nd, const int* dims, double gamma_phys, int L, double gamma_max,
                             int absorb_top, double* out) {
  return guard([&] {
    if (L < 0) throw Err(EHMG_EINVAL, "sponge: negative layer width");
    if (L > 0)
      for (int a = 0; a < nd; ++a)
        if (2 * L >= dims[a]) throw Err(EHMG_EINVAL, "sponge: 2*layer_width must be < dims on every axis");
    int d[3] = {dims[0], dims[1], nd == 3 ? dims[2] : 1};
    for (int64_t c2 = 0; c2 < d[2]; ++c2)
      for (int64_t c1 = 0; c1 < d[1]; ++c1)
        for (int64_t c0 = 0; c0 < d[0]; ++c0) {
          int c[3] = {(int)c0, (int)c1, (int)c2};
          double ramp = 0;
          if (L > 0)
            for (int a = 0; a < nd; ++a) {
              int dist_lo = c[a], dist_hi = d[a] - 1 - c[a];
              bool skip_lo = absorb_top ? false : (a == nd - 1);
              if (!skip_lo && dist_lo < L) {
                double q = double(L - dist_lo) / L;
                ramp = std::max(ramp, q * q);
              }
              if (dist_hi < L) {
                double q = double(L - dist_hi) / L;
                ramp = std::max(ramp, q * q);
              }
            }
          out[c0 + d[0] * (c1 + d[1] * c2)] = L == 0 ? gamma_phys : gamma_phys + gamma_max * ramp;
        }
  });
}

// multigrid.hpp:40-50 coarsest-solver options. automatic and lu take the
// exact solve (the reference's automatic picks Kaczmarz-FGMRES in 3D,
// multigrid.hpp:93-95, a strictly sequential row-projection sweep with no
// B200 counterpart: DESIGN.md "Coarsest solve"); kaczmarz is rejected. The
// reference's lu_dof_budget is honoured with its own length_error text
// (assemble.hpp:209-211); 0 means the reference default of 4M DOFs.
static void check_coarse_options(const Geo& fine, const ehmg_mg_options* opt) {
  if (opt->coarse == 2)
    throw Err(EHMG_EINVAL,
              "multigrid: coarse solver 'kaczmarz' is not on the B200 path (use 'lu' or 'automatic')");
  if (opt->coarse != 0 && opt->coarse != 1) throw Err(EHMG_EINVAL, "config: unknown coarse solver");
  if (opt->lu_dof_budget < 0) throw Err(EHMG_EINVAL, "multigrid: lu_dof_budget must be >= 0");
  const int64_t budget = opt->lu_dof_budget > 0 ? opt->lu_dof_budget : (int64_t)4000000;
  Geo t = fine;
  for (int l = 0; l + 1 < opt->n_levels; ++l) t = coarse_geo(t);
  if (t.ndofs > budget)
    throw Err(EHMG_ERANGE, "assemble_sparse: grid exceeds DOF budget of " + std::to_string(budget));
}

int ehmg_multigrid_create(int nd, const int* dims, double h, const double* lambda,
                          const double* mu, const double* rho, const double* gamma, double beta,
                          double omega, double alpha, const ehmg_mg_options* opt, ehmg_mg* out) {
  return guard([&] {
    if (opt->n_levels < 2) throw Err(EHMG_EINVAL, "multigrid: need at least 2 levels");
    if (opt->cycle == 0 && opt->n_levels != 2)
      throw Err(EHMG_EINVAL, "multigrid: two_grid cycle requires exactly 2 levels");
    validate_grid(nd, dims, h);
    int d[3] = {dims[0], dims[1], nd == 3 ? dims[2] : 1};
    Geo g = make_geo(nd, d, h);
    validate_media(g.ncells, lambda, mu, rho, gamma);
    // every level but the last must coarsen (transfer.hpp:25 can_coarsen)
    {
      Geo t = g;
      for (int l = 0; l + 1 < opt->n_levels; ++l) {
        for (int a = 0; a < nd; ++a)
          if (t.n[a] % 2 != 0 || t.n[a] / 2 < 2)
            throw Err(EHMG_EINVAL, "multigrid: grid cannot support requested levels");
        t = coarse_geo(t);
      }
    }
    check_coarse_options(g, opt);
    check_device();
    const OpPar P{beta, omega * omega, alpha};
    const double* f[4] = {lambda, mu, rho, gamma};
    *out = build_mg(g, f, nullptr, P, *opt, opt->n_levels).release();
  });
}

// ---- z-slab decomposition (ehmg_slab.cuh) -------------------------------
int ehmg_slab_plan(int n2, int n_levels, int nslabs, int agg_n2, int* la, int* z0) {
  return guard([&] {
    SlabPlan p = make_slab_plan(n2, n_levels, nslabs, agg_n2);
    *la = p.La;
    for (int q = 0; q <= nslabs; ++q) z0[q] = p.z0[q];
  });
}

int ehmg_slab_multigrid_create(int nd, const int* dims, double h, const double* lambda,
                               const double* mu, const double* rho, const double* gamma,
                               double beta, double omega, double alpha,
                               const ehmg_mg_options* opt, int nslabs, int agg_n2,
                               ehmg_slab_mg* out) {
  return guard([&] {
    if (opt->n_levels < 2) throw Err(EHMG_EINVAL, "multigrid: need at least 2 levels");
    validate_grid(nd, dims, h);
    check_device();
    int d[3] = {dims[0], dims[1], nd == 3 ? dims[2] : 1};
    Geo g = make_geo(nd, d, h);
    validate_media(g.ncells, lambda, mu, rho, gamma);
    {
      Geo t = g;
      for (int l = 0; l + 1 < opt->n_levels; ++l) {
        for (int a = 0; a < nd; ++a)
          if (t.n[a] % 2 != 0 || t.n[a] / 2 < 2)
            throw Err(EHMG_EINVAL, "multigrid: grid cannot support requested levels");
        t = coarse_geo(t);
      }
    }
    check_coarse_options(g, opt);
    const OpPar P{beta, omega * omega, alpha};
    const double* f[4] = {lambda, mu, rho, gamma};
    *out = build_slab_mg(g, f, P, *opt, nslabs, agg_n2, nullptr).release();
  });
}

int ehmg_slab_multigrid_destroy(ehmg_slab_mg mg) {
  return guard([&] { delete mg; });
}

int ehmg_slab_multigrid_levels(ehmg_slab_mg mg, int* distributed, int* total) {
  return guard([&] {
    *distributed = mg->plan.La;
    *total = mg->plan.nl;
  });
}

int ehmg_slab_multigrid_precondition(ehmg_slab_mg mg, const double* r, double* z, int where) {
  return guard([&] {
    const int64_t n = mg->G[0].ndofs;
    DBuf<cplx> sr, sz;
    const cplx* dr;
    to_dev(r, sr, n, where, mg->s, &dr);
    cplx* dz = out_dev(z, sz, n, where);
    mg->exchanged_bytes = 0;
    mg->precondition(dr, dz);
    from_dev(z, dz, n, where, mg->s);
  });
}

int64_t ehmg_slab_multigrid_exchanged_bytes(ehmg_slab_mg mg) { return mg ? mg->exchanged_bytes : -1; }

}  // extern "C"

// ---- one slab per process (NodeComm + CUDA IPC) ---------------------------
struct ehmg_dist_s {
  NodeComm comm;
  std::unique_ptr<ehmg_slab_mg_s> mg;
  OpPar P0;  // unshifted operator (alpha = 0) for the Krylov level
  ~ehmg_dist_s() {
    // every rank drains its streams and meets the others before the IPC
    // events and inboxes its neighbours' streams may still reference go away
    if (mg) {
      if (mg->s) cudaStreamSynchronize(mg->s);
      if (mg->sx) cudaStreamSynchronize(mg->sx);
    }
    if (comm.shm && !comm.shm->failed.load()) {
      try {
        comm.barrier();
      } catch (...) {
      }
    }
    mg.reset();
    comm.close();
  }
  SlabLevel& me() { return *mg->L[0][comm.rank]; }
  // host full array <-> this rank's level-0 window (window planes / owned planes)
  void load_window(const double* full, cplx* w) {
    const SlabGeo& sg = me().sg;
    const Geo& G0 = mg->G[0];
    for (int k = 0; k < 4; ++k) {
      const int64_t ps = slab_plane(sg.g, k);
      CK(cudaMemcpyAsync(w + sg.g.off[k], reinterpret_cast<const cplx*>(full) + G0.off[k] + (int64_t)sg.g.zoff * ps,
                         sizeof(cplx) * ps * (sg.g.n[2] + (k == 2)), cudaMemcpyHostToDevice, mg->s));
    }
  }
  void store_owned(const cplx* w, double* full) {
    const SlabGeo& sg = me().sg;
    const Geo& G0 = mg->G[0];
    const bool last = comm.rank + 1 == comm.n;
    for (int k = 0; k < 4; ++k) {
      const int64_t ps = slab_plane(sg.g, k);
      const int b = (k == 2 && last) ? sg.Z1 + 1 : sg.Z1;
      CK(cudaMemcpyAsync(reinterpret_cast<cplx*>(full) + G0.off[k] + (int64_t)sg.Z0 * ps,
                         w + sg.g.off[k] + (sg.Z0 - sg.g.zoff) * ps, sizeof(cplx) * ps * (b - sg.Z0),
                         cudaMemcpyDeviceToHost, mg->s));
    }
    CK(cudaStreamSynchronize(mg->s));
  }
  std::vector<std::pair<int64_t, int64_t>> owned_ranges() {
    const SlabGeo& sg = me().sg;
    const bool last = comm.rank + 1 == comm.n;
    std::vector<std::pair<int64_t, int64_t>> o;
    for (int k = 0; k < 4; ++k) {
      const int64_t ps = slab_plane(sg.g, k);
      const int b = (k == 2 && last) ? sg.Z1 + 1 : sg.Z1;
      o.push_back({sg.g.off[k] + (sg.Z0 - sg.g.zoff) * ps, sg.g.off[k] + (b - sg.g.zoff) * ps});
    }
    return o;
  }
};

extern "C" {

int ehmg_dist_create(const char* job, int rank, int nranks, int device, int nd, const int* dims, double h,
                     const double* lambda, const double* mu, const double* rho, const double* gamma,
                     double beta, double omega, double alpha, const ehmg_mg_options* opt, int agg_n2,
                     ehmg_dist* out) {
  return guard([&] {
    if (opt->n_levels < 2) throw Err(EHMG_EINVAL, "multigrid: need at least 2 levels");
    validate_grid(nd, dims, h);
    check_device();
    CK(cudaSetDevice(device));
    int d[3] = {dims[0], dims[1], nd == 3 ? dims[2] : 1};
    Geo g = make_geo(nd, d, h);
    validate_media(g.ncells, lambda, mu, rho, gamma);
    {
      Geo t = g;
      for (int l = 0; l + 1 < opt->n_levels; ++l) {
        for (int a = 0; a < nd; ++a)
          if (t.n[a] % 2 != 0 || t.n[a] / 2 < 2)
            throw Err(EHMG_EINVAL, "multigrid: grid cannot support requested levels");
        t = coarse_geo(t);
      }
    }
    check_coarse_options(g, opt);
    auto dd = std::make_unique<ehmg_dist_s>();
    dd->comm.open(job, rank, nranks);
    const OpPar P{beta, omega * omega, alpha};
    dd->P0 = OpPar{beta, omega * omega, 0.0};
    const double* f[4] = {lambda, mu, rho, gamma};
    try {
      dd->mg = build_slab_mg(g, f, P, *opt, nranks, agg_n2, &dd->comm);
    } catch (...) {
      dd->comm.fail();  // peers' barriers throw; no teardown barrier pairs with theirs
      throw;
    }
    *out = dd.release();
  });
}

int ehmg_dist_destroy(ehmg_dist d) {
  return guard([&] { delete d; });
}

int ehmg_dist_window(ehmg_dist d, int* z0, int* z1, int* w0, int* w1) {
  return guard([&] {
    const SlabGeo& sg = d->me().sg;
    *z0 = sg.Z0;
    *z1 = sg.Z1;
    *w0 = sg.W0();
    *w1 = sg.W1();
  });
}

int ehmg_dist_precondition(ehmg_dist d, const double* r, double* z) {
  return guard([&] {
    ehmg_slab_mg_s& mg = *d->mg;
    const int q = d->comm.rank;
    std::vector<cplx*> B(mg.P_(), nullptr), X(mg.P_(), nullptr);
    B[q] = mg.bw[0]->p;
    X[q] = mg.xw[0]->p;
    d->load_window(r, B[q]);
    mg.precondition_windows(B, X);
    d->store_owned(X[q], z);
  });
}

// CUDA-event time of `count` distributed preconditioner applications on the
// resident level-0 window (exchanges and barriers included).
int ehmg_dist_time_precondition(ehmg_dist d, const double* r, int count, double* ms) {
  return guard([&] {
    ehmg_slab_mg_s& mg = *d->mg;
    const int q = d->comm.rank;
    std::vector<cplx*> B(mg.P_(), nullptr), X(mg.P_(), nullptr);
    B[q] = mg.bw[0]->p;
    X[q] = mg.xw[0]->p;
    d->load_window(r, B[q]);
    CK(cudaStreamSynchronize(mg.s));
    d->comm.barrier();
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    CK(cudaEventRecord(a, mg.s));
    for (int i = 0; i < count; ++i) mg.precondition_windows(B, X);
    CK(cudaEventRecord(b, mg.s));
    CK(cudaEventSynchronize(b));
    float f = 0;
    CK(cudaEventElapsedTime(&f, a, b));
    *ms = f;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  });
}

int64_t ehmg_dist_exchanged_bytes(ehmg_dist d) { return d ? d->mg->exchanged_bytes : -1; }

int ehmg_dist_solve(ehmg_dist d, const double* b, double* x, const ehmg_krylov_options* opt,
                    ehmg_krylov_result* res, double* history, int history_cap) {
  return guard([&] {
    check_krylov_args(opt, res);
    if (!d) throw Err(EHMG_EINVAL, "fgmres: null distributed handle");
    ehmg_slab_mg_s& mg = *d->mg;
    const int q = d->comm.rank;
    SlabLevel& me = d->me();
    const int64_t n = me.sg.g.ndofs;
    cudaStream_t s = mg.s;
    DBuf<cplx> db(n), dx(n);
    d->load_window(b, db.p);
    dx.zero(s);
    Fgmres fg;
    fg.init(n, opt->restart, s);
    fg.blas.comm = &d->comm;
    fg.blas.owned = d->owned_ranges();
    std::vector<cplx*> V(mg.P_(), nullptr), W(mg.P_(), nullptr);
    Fgmres::Fn Af = [&](const cplx* in, cplx* out) {
      V[q] = const_cast<cplx*>(in);  // ghost planes are scratch
      mg.exchange(0, V);
      launch_residual(me.sg.g, d->P0, me.media.ref(), in, nullptr, out, s);
    };
    Fgmres::Fn Mf = [&](const cplx* in, cplx* out) {
      V[q] = const_cast<cplx*>(in);
      W[q] = out;
      mg.precondition_windows(V, W);
    };
    std::vector<double> hist;
    *res = fg.run(Af, Mf, db.p, dx.p, *opt, hist);
    res->n_history = (int)hist.size();
    if (history)
      for (int i = 0; i < (int)hist.size() && i < history_cap; ++i) history[i] = hist[i];
    d->store_owned(dx.p, x);
  });
}

int ehmg_multigrid_destroy(ehmg_mg mg) {
  return guard([&] { delete mg; });
}
int ehmg_multigrid_n_levels(ehmg_mg mg) { return mg ? (int)mg->L.size() : -1; }
int ehmg_multigrid_factor_sets(ehmg_mg mg, int level) {
  if (!mg || level < 0 || level >= (int)mg->L.size()) return -1;
  const Smoother& sm = mg->L[level]->sm;
  return sm.dict ? sm.dict_sets : 0;
}
uint64_t ehmg_multigrid_stream(ehmg_mg mg) { return mg ? (uint64_t)(uintptr_t)mg->s : 0; }

int ehmg_multigrid_cycle(ehmg_mg mg, const double* b, double* x, int where) {
  return guard([&] {
    const int64_t n = mg->L[0]->g.ndofs;
    const cplx* db;
    to_dev(b, mg->hy, n, where, mg->s, &db);
    cplx* dx;
    if (where == EHMG_DEVICE) {
      dx = reinterpret_cast<cplx*>(x);
    } else {
      if (mg->hx.n < n) mg->hx.alloc(n);
      CK(cudaMemcpyAsync(mg->hx.p, x, sizeof(cplx) * n, cudaMemcpyHostToDevice, mg->s));
      dx = mg->hx.p;
    }
    if (mg->prec == 0) {
      mg->cycle_at(0, db, dx);
    } else {
      cudaStream_t s = mg->s;
      k_convert<cplxf, cplx><<<grid_for(n, 148 * 64), kThreads, 0, s>>>(n, db, mg->rin.p);
      k_convert<cplxf, cplx><<<grid_for(n, 148 * 64), kThreads, 0, s>>>(n, dx, mg->zout.p);
      CK(cudaGetLastError());
      mg->cycle_t<cplxf>(0, mg->rin.p, mg->zout.p, false);
      k_convert<cplx, cplxf><<<grid_for(n, 148 * 64), kThreads, 0, s>>>(n, mg->zout.p, dx);
      CK(cudaGetLastError());
    }
    from_dev(x, dx, n, where, mg->s);
  });
}

int ehmg_multigrid_precondition(ehmg_mg mg, const double* r, double* z, int where) {
  return guard([&] {
    const int64_t n = mg->L[0]->g.ndofs;
    const cplx* dr;
    to_dev(r, mg->hy, n, where, mg->s, &dr);
    cplx* dz = out_dev(z, mg->hx, n, where);
    mg->precondition(dr, dz);
    from_dev(z, dz, n, where, mg->s);
  });
}

// Three-stage pipeline over right-hand sides i = 0..count-1, staging pair
// k = i & 1: s_in copies r[i] into rst[k] once the cycle of i-2 released it;
// the solver stream runs the cycle rst[k] -> zst[k] once that copy landed
// and the copy-out of i-2 released zst[k]; s_out copies zst[k] to z[i].
int ehmg_multigrid_precondition_many(ehmg_mg mg, int count, const double* const* r, double* const* z) {
  return guard([&] {
    if (count < 0 || (count > 0 && (!r || !z))) throw Err(EHMG_EINVAL, "precondition_many: bad batch");
    if (count == 0) return;
    CK(cudaSetDevice(mg->dev));
    const int64_t n = mg->L[0]->g.ndofs;
    if (!mg->s_in) {
      CK(cudaStreamCreateWithFlags(&mg->s_in, cudaStreamNonBlocking));
      CK(cudaStreamCreateWithFlags(&mg->s_out, cudaStreamNonBlocking));
      for (int k = 0; k < 2; ++k) {
        CK(cudaEventCreateWithFlags(&mg->ev_in[k], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&mg->ev_comp[k], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&mg->ev_out[k], cudaEventDisableTiming));
      }
    }
    for (int k = 0; k < 2; ++k) {
      if (mg->rst[k].n < n) mg->rst[k].alloc(n);
      if (mg->zst[k].n < n) mg->zst[k].alloc(n);
    }
    // nothing in flight from an earlier call may still use the staging pairs
    CK(cudaEventRecord(mg->ev_comp[0], mg->s));
    CK(cudaStreamWaitEvent(mg->s_in, mg->ev_comp[0], 0));
    CK(cudaStreamWaitEvent(mg->s_out, mg->ev_comp[0], 0));
    for (int i = 0; i < count; ++i) {
      if (!r[i] || !z[i]) throw Err(EHMG_EINVAL, "precondition_many: null buffer");
      const int k = i & 1;
      if (i >= 2) CK(cudaStreamWaitEvent(mg->s_in, mg->ev_comp[k], 0));
      CK(cudaMemcpyAsync(mg->rst[k].p, r[i], sizeof(cplx) * n, cudaMemcpyHostToDevice, mg->s_in));
      CK(cudaEventRecord(mg->ev_in[k], mg->s_in));
      CK(cudaStreamWaitEvent(mg->s, mg->ev_in[k], 0));
      if (i >= 2) CK(cudaStreamWaitEvent(mg->s, mg->ev_out[k], 0));
      mg->precondition(mg->rst[k].p, mg->zst[k].p);
      CK(cudaEventRecord(mg->ev_comp[k], mg->s));
      CK(cudaStreamWaitEvent(mg->s_out, mg->ev_comp[k], 0));
      CK(cudaMemcpyAsync(z[i], mg->zst[k].p, sizeof(cplx) * n, cudaMemcpyDeviceToHost, mg->s_out));
      CK(cudaEventRecord(mg->ev_out[k], mg->s_out));
    }
    CK(cudaStreamSynchronize(mg->s_out));
    CK(cudaStreamSynchronize(mg->s));
  });
}

int ehmg_multigrid_measure_convergence(ehmg_mg mg, uint64_t seed, const ehmg_measure_options* mo,
                                       ehmg_measure_result* res, double* history, int cap) {
  return guard([&] {
    if (!mo || !res) throw Err(EHMG_EINVAL, "measure: null options or result");
    if (mg->prec == 0) measure_t<cplx>(*mg, seed, *mo, res, history, cap);
    else measure_t<cplxf>(*mg, seed, *mo, res, history, cap);
  });
}

int ehmg_multigrid_time_precondition(ehmg_mg mg, const double* r_dev, double* z_dev, int count,
                                     double* ms) {
  return guard([&] {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    CK(cudaEventRecord(a, mg->s));
    for (int i = 0; i < count; ++i)
      mg->precondition(reinterpret_cast<const cplx*>(r_dev), reinterpret_cast<cplx*>(z_dev));
    CK(cudaEventRecord(b, mg->s));
    CK(cudaEventSynchronize(b));
    float f = 0;
    CK(cudaEventElapsedTime(&f, a, b));
    *ms = f;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  });
}

int ehmg_profile_enable(int on) {
  return guard([&] {
    g_prof = on != 0;
    for (auto& r : g_recs) {
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    }
    g_recs.clear();
  });
}

// Aggregate recorded launches: one line "name level count total_ms" per
// (kernel, level) into buf (newline separated).
int ehmg_profile_report(char* buf, int cap) {
  return guard([&] {
    struct Agg {
      std::string name;
      int level;
      int count;
      double ms;
    };
    std::vector<Agg> agg;
    for (auto& r : g_recs) {
      CK(cudaEventSynchronize(r.b));
      float f = 0;
      CK(cudaEventElapsedTime(&f, r.a, r.b));
      bool found = false;
      for (auto& a : agg)
        if (a.name == r.name && a.level == r.level) {
          a.count++;
          a.ms += f;
          found = true;
        }
      if (!found) agg.push_back({r.name, r.level, 1, (double)f});
    }
    std::string out;
    for (auto& a : agg)
      out += a.name + " " + std::to_string(a.level) + " " + std::to_string(a.count) + " " +
             std::to_string(a.ms) + "\n";
    std::snprintf(buf, (size_t)cap, "%s", out.c_str());
  });
}

int ehmg_fgmres_solve(ehmg_op A, ehmg_mg M, const double* b, double* x, int where,
                      const ehmg_krylov_options* opt, ehmg_krylov_result* res, double* history,
                      int history_cap) {
  return guard([&] {
    check_krylov_args(opt, res);
    if (!A) throw Err(EHMG_EINVAL, "fgmres: null operator");
    const int64_t n = A->g.ndofs;
    if (M && M->L[0]->g.ndofs != n) throw Err(EHMG_EINVAL, "fgmres: operator/preconditioner size mismatch");
    cudaStream_t s = M ? M->s : A->s;
    // keep the operator on the solver stream
    const cplx* db;
    DBuf<cplx> sb, sx;
    to_dev(b, sb, n, where, s, &db);
    cplx* dx;
    if (where == EHMG_DEVICE) {
      dx = reinterpret_cast<cplx*>(x);
    } else {
      sx.alloc(n);
      CK(cudaMemcpyAsync(sx.p, x, sizeof(cplx) * n, cudaMemcpyHostToDevice, s));
      dx = sx.p;
    }
    Fgmres local;
    if (M && !M->solve_ws) M->solve_ws.reset(new Fgmres());
    Fgmres& fg = M ? *M->solve_ws : local;
    fg.init(n, opt->restart, s);
    Fgmres::Fn Af = [&](const cplx* in, cplx* out) {
      launch_residual(A->g, A->P, A->media.ref(), in, nullptr, out, s);
    };
    Fgmres::Fn Mf = [&](const cplx* in, cplx* out) {
      if (M) M->precondition(in, out);
      else CK(cudaMemcpyAsync(out, in, sizeof(cplx) * n, cudaMemcpyDeviceToDevice, s));
    };
    std::vector<double> hist;
    *res = fg.run(Af, Mf, db, dx, *opt, hist);
    res->n_history = (int)hist.size();
    if (history)
      for (int i = 0; i < (int)hist.size() && i < history_cap; ++i) history[i] = hist[i];
    from_dev(x, dx, n, where, s);
  });
}

int ehmg_field_dot(int64_t n, const double* x, const double* y, double* out) {
  return guard([&] {
    Blas b;
    b.init(0, 1);
    b.reduce(0, n, (const cplx*)x, (const cplx*)y, b.res(), nullptr, nullptr);
    CK(cudaMemcpy(out, b.res(), 2 * sizeof(double), cudaMemcpyDeviceToHost));
  });
}
int ehmg_field_norm(int64_t n, const double* x, double* out) {
  return guard([&] {
    Blas b;
    b.init(0, 1);
    *out = b.norm_host(n, (const cplx*)x);
  });
}
int ehmg_field_axpy(int64_t n, double ar, double ai, const double* x, double* y) {
  return guard([&] {
    Blas b;
    b.init(0, 1);
    b.axpy(n, mk(ar, ai), nullptr, (const cplx*)x, (cplx*)y);
    CK(cudaDeviceSynchronize());
  });
}

int ehmg_device_alloc(int64_t bytes, void** out) {
  return guard([&] {
    check_device();
    CK(cudaMalloc(out, (size_t)bytes));
  });
}
int ehmg_device_free(void* p) {
  return guard([&] { CK(cudaFree(p)); });
}
int ehmg_memcpy(void* dst, const void* src, int64_t bytes, int kind) {
  return guard([&] {
    cudaMemcpyKind k = kind == 0 ? cudaMemcpyHostToDevice
                                 : (kind == 1 ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice);
    CK(cudaMemcpy(dst, src, (size_t)bytes, k));
  });
}

}  // extern "C"
