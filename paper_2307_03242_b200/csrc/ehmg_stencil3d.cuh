// ehmg_stencil3d.cuh -- shared 3D-stencil machinery (tensor-map encoder,
// TMA/mbarrier helpers, boundary-renormalisation tables, z-chunk planning)
// and the 11/20-warp shared-memory kernel k_stencil3d.
//
// y = H x  or  r = b - H x  for the staggered mixed elastic-Helmholtz
// operator (operator.hpp:389-421), all four components in one launch.
// Production kernels live in ehmg_stencil3d_rr.cuh (k_stencil3d_rr); the
// kernel below now serves only the complex64 hierarchy on widths with
// n0 % 4 != 0 (its cp.async path), and documents the previous design:
//
// Design (B200, complex128 and complex64):
//  * 2.5D tiling. A CTA owns a 33x8 tile of the (i,j) index plane plus a
//    one-cell flux halo (35x10 = 350 positions, one thread each, 11 warps)
//    and marches a z-chunk (persistent CTAs stride over tile x chunk items).
//  * TMA. u0,u1,u2 (planes z, z+1), p (z-1, z) and the SoA cell media
//    (z-1..z+1) sit in shared-memory rings filled by cp.async.bulk.tensor
//    3D box loads issued by one thread and tracked by an mbarrier; the
//    hardware's out-of-bounds zero fill supplies exactly the reference's zero
//    ghosts (operator.hpp:172 GhostAcc). The next plane streams in while the
//    current one is computed.
//  * Separable spread derivatives. The 9-tap transverse (1,2,1)x(1,2,1)
//    spread of every first derivative (operator.hpp:267 / :306) is split
//    into an in-plane 3-tap row sum and a z-direction 3-tap combination; the
//    row sums of the previous two planes are carried in registers. The three
//    purely in-plane families (F22, F02, F12) filter a shared difference field.
//  * Flux sharing. Each flux is evaluated once and shared through shared
//    memory by the two rows that use it; z-neighbour fluxes and mass
//    products are carried in registers.
//  * Exactness. Boundary renormalisations (1/wsum, mass 1/wsum) come from
//    tables built on the host in the reference's accumulation order; edge /
//    face media averages divide by 1, 2 or 4, applied as exact reciprocal
//    multiplies. Results match the reference to rounding (<= 1e-13 rel).
#pragma once

#include <cuda.h>  // CUtensorMap (types only; the encoder is fetched at run time)

#include <mutex>
#include <vector>

#include "ehmg_core.cuh"

namespace ehmg {

// 33 columns: the n0+1 u0 faces of a power-of-two level (257, 129, 65, 33)
// split into whole tiles with no one-column remainder tile.
constexpr int S3_TX = 33, S3_TY = 8;
constexpr int S3_UX = S3_TX + 4, S3_UY = S3_TY + 4, S3_UN = S3_UX * S3_UY;  // origin (i0-2, j0-2)
constexpr int S3_US = (S3_UN + 15) / 16 * 16;  // ring-slot stride: TMA destinations stay 128-byte aligned
// media boxes: TMA inner box extents and start offsets are 16-byte multiples,
// so the float64 media planes start at an even column and use an even pitch
// (UX + 1 columns: one spare column on the left or the right of the tile)
constexpr int S3_MX = (S3_UX + 1) / 2 * 2, S3_MN = S3_MX * S3_UY, S3_MS = (S3_MN + 15) / 16 * 16;
static_assert(S3_MX >= S3_UX + 1, "media pitch needs the spare column");
constexpr int S3_FX = S3_TX + 2, S3_FY = S3_TY + 2, S3_FN = S3_FX * S3_FY;  // origin (i0-1, j0-1)
constexpr int S3_THREADS = ((S3_FN + 31) / 32) * 32;                         // 352
constexpr int S3_ZCHUNK = 32;
constexpr unsigned S3_CBYTES = S3_UN * 16, S3_DBYTES = S3_MN * 8;  // one complex / double box

// Tile height per element type: complex128 fits a 33x8 tile (11 warps at the
// 168-register limit); complex64 halves the rings and the register file per
// value, so a 33x16 tile (20 warps, 96 registers) runs with less halo work.
template <class V> struct S3Cfg;
template <> struct S3Cfg<cplx> {
  static constexpr int TY = S3_TY, UY = S3_UY, UN = S3_UN, US = S3_US, MN = S3_MN, MS = S3_MS, FY = S3_FY,
                       FN = S3_FN, THREADS = S3_THREADS;
};
template <> struct S3Cfg<cplxf> {
  static constexpr int TY = 16, UY = TY + 4, UN = S3_UX * UY, US = (UN + 15) / 16 * 16, MN = S3_MX * UY,
                       MS = (MN + 15) / 16 * 16, FY = TY + 2, FN = S3_FX * FY, THREADS = ((FN + 31) / 32) * 32;
};

struct S3Params {
  Geo g;
  double beta, omega2, alpha, w;  // w = (1-beta)/16
  double inv_wsum[16];            // 1/wsum by transverse validity bits (lo1,hi1,lo2,hi2)
  double wn;                      // (1-beta)/6
  double inv_msum[7];             // 1/(beta + k*wn), k valid mass neighbours
  int nchunks, ntiles_x, ntiles_y;
  int itx, ity;  // k_stencil3d_sp: tile columns 1..itx / rows 1..ity lie strictly inside the box
  int z_lo, z_hi;  // output planes [z_lo, z_hi); z_hi = n2 + 1 includes the top u2 faces
  float inv_wsum_f[16], inv_msum_f[7];  // the same tables accumulated in float (complex64 kernel)
  double inv_wsum_h[16];                // inv_wsum * inv_h (k_stencil3d_sp)
  // k_stencil3d_sp, tiles strictly inside the box: the z-dependent constants by
  // plane class lz | hz0 << 1 | hz1 << 2 | (z >= 0) << 3, with c = inv_wsum_h[.]:
  // {beta c, w c} for c at [3|zA], [zB|12], [3|zC]; inv_msum[4+lz+hz0], inv_msum[4+lz+hz1], izp, izp*omega2
  double zt[16][10];
  double bw_in[2];  // {beta c, w c} for c = inv_wsum_h[15] (in-plane families inside the box)
};

// Source arrays of the complex64 kernel (loaded with cp.async: complex64
// rows of n0+1 faces are not 16-byte multiples, which tensor maps require).
struct S3Src {
  const cplxf* u[3];
  const cplxf* p;
  const float *mu, *rho, *gam, *ilm;
};

struct S3Maps {
  CUtensorMap u[3], p, mu, rho, gam, ilm;
};

template <class V>
struct __align__(128) S3SmemT {
  typedef typename VT<V>::R R;
  typedef S3Cfg<V> K;
  V u[3][3][K::US];  // [plane % 3][component]
  V p[3][K::US];     // [plane % 3]
  R mu[4][K::MS], rho[4][K::MS], gam[4][K::MS], ilm[4][K::MS];  // [plane % 4], pitch S3_MX
  V f[6][K::FN];     // z-family fluxes at plane z: F00 F11 F01 F10 F20 F21
  V di[3][K::FN];    // in-plane difference fields: d22 (cell z), d02, d12 (edge z+1)
  V q[2][3][K::FN];  // mass products md*u [plane & 1][component]
  unsigned long long bar[2];
};
typedef S3SmemT<cplx> S3Smem;

__device__ __forceinline__ unsigned s3_saddr(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void s3_tma(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                       unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(s3_saddr(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(s3_saddr(bar))
      : "memory");
}
__device__ __forceinline__ void s3_expect(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(s3_saddr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void s3_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred P1;\n"
      "WAIT%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @!P1 bra WAIT%=;\n}\n" ::"r"(s3_saddr(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ int s3_mod3(int z) { return ((z % 3) + 3) % 3; }

// One load group: u planes zu (each listed), media planes zm, p planes zp.
__device__ __forceinline__ void s3_issue(S3Smem& S, const S3Maps& M, int i0, int j0, const int* zu, int nu,
                                         const int* zm, int nm, const int* zp, int np,
                                         unsigned long long* bar) {
  s3_expect(bar, (unsigned)(nu * 3 * S3_CBYTES + nm * 4 * S3_DBYTES + np * S3_CBYTES));
  const int cx = 2 * (i0 - 2), cy = j0 - 2;
  for (int q = 0; q < nu; ++q) {
    const int sl = s3_mod3(zu[q]);
    s3_tma(S.u[sl][0], &M.u[0], cx, cy, zu[q], bar);
    s3_tma(S.u[sl][1], &M.u[1], cx, cy, zu[q], bar);
    s3_tma(S.u[sl][2], &M.u[2], cx, cy, zu[q], bar);
  }
  for (int q = 0; q < nm; ++q) {
    const int sl = zm[q] & 3;
    const int mx = (i0 - 2) & ~1;
    s3_tma(S.mu[sl], &M.mu, mx, cy, zm[q], bar);
    s3_tma(S.rho[sl], &M.rho, mx, cy, zm[q], bar);
    s3_tma(S.gam[sl], &M.gam, mx, cy, zm[q], bar);
    s3_tma(S.ilm[sl], &M.ilm, mx, cy, zm[q], bar);
  }
  for (int q = 0; q < np; ++q) s3_tma(S.p[s3_mod3(zp[q])], &M.p, cx, cy, zp[q], bar);
}

template <class R>
__device__ __forceinline__ R s3_inv(int c) {  // 1/c for c in {0,1,2}
  return c == 2 ? R(0.5) : (c == 1 ? R(1) : R(0));
}
template <class R> __device__ __forceinline__ R s3_iw(const S3Params& P, int i);
template <> __device__ __forceinline__ double s3_iw<double>(const S3Params& P, int i) { return P.inv_wsum[i]; }
template <> __device__ __forceinline__ float s3_iw<float>(const S3Params& P, int i) { return P.inv_wsum_f[i]; }
template <class R> __device__ __forceinline__ R s3_im(const S3Params& P, int i);
template <> __device__ __forceinline__ double s3_im<double>(const S3Params& P, int i) { return P.inv_msum[i]; }
template <> __device__ __forceinline__ float s3_im<float>(const S3Params& P, int i) { return P.inv_msum_f[i]; }

// complex64 loads: every thread copies its share of each box with cp.async
// (zero outside the array, like the tensor maps' out-of-bounds fill).
__device__ __forceinline__ void s3_cp8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s3_saddr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void s3_cp4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s3_saddr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void s3_cp_commit_wait() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}
__device__ __forceinline__ void s3_cplane(cplxf* dst, const cplxf* base, int d0, int d1, int d2, int x0, int y0,
                                          int z) {
  const bool zin = z >= 0 && z < d2;
  for (int e = threadIdx.x; e < S3Cfg<cplxf>::UN; e += blockDim.x) {
    const int r = e / S3_UX, j = e - r * S3_UX, x = x0 + j, y = y0 + r;
    if (zin && x >= 0 && x < d0 && y >= 0 && y < d1)
      s3_cp8(&dst[e], base + ((int64_t)z * d1 + y) * d0 + x);
    else
      dst[e] = mkf(0.f, 0.f);
  }
}
__device__ __forceinline__ void s3_mplane(float* dst, const float* base, int d0, int d1, int d2, int x0, int y0,
                                          int z) {
  const bool zin = z >= 0 && z < d2;
  for (int e = threadIdx.x; e < S3Cfg<cplxf>::MN; e += blockDim.x) {
    const int r = e / S3_MX, j = e - r * S3_MX, x = x0 + j, y = y0 + r;
    if (zin && x >= 0 && x < d0 && y >= 0 && y < d1)
      s3_cp4(&dst[e], base + ((int64_t)z * d1 + y) * d0 + x);
    else
      dst[e] = 0.f;
  }
}
__device__ __forceinline__ void s3_issue_ca(S3SmemT<cplxf>& S, const S3Src& M, const Geo& g, int i0, int j0,
                                            const int* zu, int nu, const int* zm, int nm, const int* zp, int np) {
  const int n0 = g.n[0], n1 = g.n[1], n2 = g.n[2];
  const int cx = i0 - 2, cy = j0 - 2, mx = (i0 - 2) & ~1;
  for (int q = 0; q < nu; ++q) {
    const int sl = s3_mod3(zu[q]);
    s3_cplane(S.u[sl][0], M.u[0], n0 + 1, n1, n2, cx, cy, zu[q]);
    s3_cplane(S.u[sl][1], M.u[1], n0, n1 + 1, n2, cx, cy, zu[q]);
    s3_cplane(S.u[sl][2], M.u[2], n0, n1, n2 + 1, cx, cy, zu[q]);
  }
  for (int q = 0; q < nm; ++q) {
    const int sl = zm[q] & 3;
    s3_mplane(S.mu[sl], M.mu, n0, n1, n2, mx, cy, zm[q]);
    s3_mplane(S.rho[sl], M.rho, n0, n1, n2, mx, cy, zm[q]);
    s3_mplane(S.gam[sl], M.gam, n0, n1, n2, mx, cy, zm[q]);
    s3_mplane(S.ilm[sl], M.ilm, n0, n1, n2, mx, cy, zm[q]);
  }
  for (int q = 0; q < np; ++q) s3_cplane(S.p[s3_mod3(zp[q])], M.p, n0, n1, n2, cx, cy, zp[q]);
}

// ----------------------------------------------------------------- kernel
// 11 warps = 3 per SM sub-partition: 16K registers / 96 threads caps this at 168
// V = C: complex128, planes by TMA. V = cplxf: complex64 arithmetic (the
// single-precision hierarchy), planes by cp.async from `src`.
template <class V>
__global__ void __launch_bounds__(S3Cfg<V>::THREADS, 1)
    k_stencil3d(const __grid_constant__ S3Maps maps, const __grid_constant__ S3Src src, const S3Params P,
                const V* __restrict__ b, V* __restrict__ y) {
  typedef V C;
  constexpr int S3_FN_ = S3Cfg<V>::FN, S3_TY_ = S3Cfg<V>::TY, S3_FY_ = S3Cfg<V>::FY;
  typedef typename VT<V>::R R;
  constexpr bool kTma = sizeof(R) == 8;
  const C zc = VT<V>::mk(0, 0);
  extern __shared__ __align__(1024) unsigned char s3_raw[];
  S3SmemT<V>& S = *reinterpret_cast<S3SmemT<V>*>(s3_raw);
  const Geo& g = P.g;
  const int t = threadIdx.x;
  const bool act = t < S3_FN_;
  const int fx = act ? t % S3_FX : 1, fy = act ? t / S3_FX : 1;
  const int ui = (fx + 1) + S3_UX * (fy + 1);  // own U-local index
  const bool interior = act && fx >= 1 && fx <= S3_TX && fy >= 1 && fy <= S3_TY_;
  const R beta = (R)P.beta, w = (R)P.w, ih = (R)g.inv_h, wn = (R)P.wn;
  const int n0 = g.n[0], n1 = g.n[1], n2 = g.n[2];  // local storage extents
  const int zoff = g.zoff, n2g = g.gn2;               // global z semantics (slab windows)

  if (kTma && t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(s3_saddr(&S.bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(s3_saddr(&S.bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  unsigned seq = 0;  // load groups issued so far (uniform)

  const int items = P.ntiles_x * P.ntiles_y * P.nchunks;
  for (int item = blockIdx.x; item < items; item += gridDim.x) {
    const int tile = item % (P.ntiles_x * P.ntiles_y);
    const int chunk = item / (P.ntiles_x * P.ntiles_y);
    const int i0 = (tile % P.ntiles_x) * S3_TX, j0 = (tile / P.ntiles_x) * S3_TY_;
    const int zspan = P.z_hi - P.z_lo;
    const int zb = P.z_lo + (int)(((int64_t)chunk * zspan) / P.nchunks);
    const int zend = P.z_lo + (int)(((int64_t)(chunk + 1) * zspan) / P.nchunks);

    // ---- per-item constants of this thread's position
    // media boxes start at an even column (16-byte aligned TMA start): i0-2 or i0-3
    const int um = (fx + 1 + (i0 & 1)) + S3_MX * (fy + 1);  // own media-local index
    const int xg = i0 - 1 + fx, yg = j0 - 1 + fy;
    const int lx = xg >= 1, hx0 = xg + 1 < n0, hx1 = xg < n0;
    const int ly = yg >= 1, hy0 = yg + 1 < n1, hy1 = yg < n1;
    const R ix = s3_inv<R>(lx + hx1), iy = s3_inv<R>(ly + hy1);
    const int fl00 = ly | (hy0 << 1), fl11 = (lx << 2) | (hx0 << 3);
    const int fl01 = (lx << 2) | (hx1 << 3), fl10 = (ly << 2) | (hy1 << 3);
    const int fl20 = ly | (hy0 << 1), fl21 = lx | (hx0 << 1);
    const R c22 = s3_iw<R>(P, lx | (hx0 << 1) | (ly << 2) | (hy0 << 3)) * ih;
    const R c02 = s3_iw<R>(P, ly | (hy0 << 1) | (lx << 2) | (hx1 << 3)) * ih;
    const R c12 = s3_iw<R>(P, lx | (hx0 << 1) | (ly << 2) | (hy1 << 3)) * ih;
    const R mu01s = ix * iy;
    const int mc0 = (lx + (xg + 1 < n0 + 1)) + (ly + hy0), mc1 = (lx + hx0) + (ly + (yg + 1 < n1 + 1)),
              mc2 = (lx + hx0) + (ly + hy0);
    const bool v0 = interior && xg >= 0 && xg <= n0 && yg >= 0 && yg < n1;
    const bool v1 = interior && xg >= 0 && xg < n0 && yg >= 0 && yg <= n1;
    const bool v2 = interior && xg >= 0 && xg < n0 && yg >= 0 && yg < n1;
    const bool q0ok = xg >= 0 && xg <= n0 && yg >= 0 && yg < n1;
    const bool q1ok = xg >= 0 && xg < n0 && yg >= 0 && yg <= n1;
    const bool q2ok = xg >= 0 && xg < n0 && yg >= 0 && yg < n1;
    const int64_t o0 = g.off[0] + xg + (int64_t)(n0 + 1) * yg, s0 = (int64_t)(n0 + 1) * n1;
    const int64_t o1 = g.off[1] + xg + (int64_t)n0 * yg, s1 = (int64_t)n0 * (n1 + 1);
    const int64_t o2 = g.off[2] + xg + (int64_t)n0 * yg, s2 = (int64_t)n0 * n1;
    const int64_t o3 = g.off[3] + xg + (int64_t)n0 * yg;

    // ---- prologue load group for the first (warm-up) step z = zb-2
    {
      const int zu[2] = {zb - 2, zb - 1}, zm[3] = {zb - 3, zb - 2, zb - 1}, zp[2] = {zb - 3, zb - 2};
      if constexpr (kTma) {
        if (t == 0) {
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          s3_issue(S, maps, i0, j0, zu, 2, zm, 3, zp, 2, &S.bar[seq & 1]);
        }
      } else {
        s3_issue_ca(S, src, g, i0, j0, zu, 2, zm, 3, zp, 2);
      }
    }

    C r00m = zc, r00c = zc, r11m = zc, r11c = zc;
    C r01m = zc, r01c = zc, r10m = zc, r10c = zc;
    C r20m = zc, r20c = zc, r21m = zc, r21c = zc;
    C f02c = zc, f12c = zc, f22m = zc;
    C qm0 = zc, qm1 = zc, qm2 = zc;
    int su0 = s3_mod3(zb - 2), pm = s3_mod3(zb - 3);  // ring slots of u plane z, p plane z-1

    for (int z = zb - 2; z < zend; ++z) {
      if constexpr (kTma) s3_wait(&S.bar[seq & 1], (seq >> 1) & 1);
      else s3_cp_commit_wait();
      ++seq;
      __syncthreads();  // all of step z-1 done: its slots may be refilled
      {
        const int zu[1] = {z + 2}, zm[1] = {z + 2}, zp[1] = {z + 1};
        if constexpr (kTma) {
          if (t == 0) {
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            s3_issue(S, maps, i0, j0, zu, 1, zm, 1, zp, 1, &S.bar[seq & 1]);
          }
        } else {
          s3_issue_ca(S, src, g, i0, j0, zu, 1, zm, 1, zp, 1);
        }
      }
      const int su1 = su0 == 2 ? 0 : su0 + 1;
      const int pc_ = pm == 2 ? 0 : pm + 1;
      const C* U0 = S.u[su0][0];
      const C* U1 = S.u[su0][1];
      const C* U2 = S.u[su0][2];
      const C* V0 = S.u[su1][0];
      const C* V1 = S.u[su1][1];
      const C* V2 = S.u[su1][2];
      const R* MUm = S.mu[(z - 1) & 3];
      const R* MUc = S.mu[z & 3];
      const R* MUp = S.mu[(z + 1) & 3];
      // uniform z quantities (global plane index zg decides the boundary rules)
      const int zg = z + zoff;
      const int lz = zg >= 1, hz0 = zg + 1 < n2g, hz1 = zg + 1 < n2g + 1;
      const R izc = s3_inv<R>(lz + (zg < n2g)), izp = s3_inv<R>((zg + 1 >= 1) + (zg + 1 < n2g));
      const int zA = (lz << 2) | (hz0 << 3), zB = lz | (hz0 << 1), zC = (lz << 2) | (hz1 << 3);
      C d00 = zc, d11 = zc;

      if (act) {
        // Every shared-memory value this position needs is loaded once into
        // registers (grouped per component to bound register pressure).
        const R al = (R)P.alpha, w2 = (R)P.omega2;
        const R mc00 = MUc[um], mc_l = MUc[um - 1], mc_b = MUc[um - S3_MX], mc_lb = MUc[um - 1 - S3_MX];
        const R mm00 = MUm[um], mm_l = MUm[um - 1], mm_b = MUm[um - S3_MX];
        // mu on the edges (operator.hpp:108 order: first axis outer, second inner)
        const R mu01 = (mc_lb + mc_l + mc_b + mc00) * mu01s;
        const R mu02 = (mm_l + mc_l + mm00 + mc00) * (ix * izc);
        const R mu12 = (mm_b + mc_b + mm00 + mc00) * (iy * izc);
        const R* RHc = S.rho[z & 3];
        const R* RHp = S.rho[(z + 1) & 3];
        const R* GAc = S.gam[z & 3];
        const R* GAp = S.gam[(z + 1) & 3];
        const R rp00 = RHp[um], gp00 = GAp[um];
        auto md = [&](R sr, R sg, R ic) {
          const R rho_f = sr * ic, gam_f = sg * ic + al;
          return VT<V>::mk(w2 * rho_f, -w2 * gam_f * rho_f);
        };
        const bool zin = zg + 1 >= 0 && zg + 1 < n2g;
        const int qb = (z + 1) & 1;
        // ---- component 0: F00 (cell, +x pair, in-plane y), F01 (edge01, -y pair, in-plane x)
        {
          const C vmm = V0[ui - S3_UX - 1], vm0 = V0[ui - S3_UX], vmp = V0[ui - S3_UX + 1];
          const C v0m = V0[ui - 1], v00 = V0[ui], v0p = V0[ui + 1];
          const C vp0 = V0[ui + S3_UX], vpp = V0[ui + S3_UX + 1];
          const C u00 = U0[ui], u0p = U0[ui + 1], um0 = U0[ui - S3_UX];
          const C rn0 = (vmp - vm0) + (vpp - vp0) + R(2) * (v0p - v00);
          const C sz0 = r00m + rn0 + R(2) * r00c;
          d00 = (beta * (u0p - u00) + w * sz0) * (s3_iw<R>(P, fl00 | zA) * ih);
          S.f[0][t] = mc00 * d00;
          r00m = r00c;
          r00c = rn0;
          const C rn1 = (v0m - vmm) + (v0p - vmp) + R(2) * (v00 - vm0);
          const C sz1 = r01m + rn1 + R(2) * r01c;
          S.f[2][t] = mu01 * ((beta * (u00 - um0) + w * sz1) * (s3_iw<R>(P, zB | fl01) * ih));
          r01m = r01c;
          r01c = rn1;
          S.di[1][t] = v00 - u00;  // d02 at edge (q, z+1)
          S.q[qb][0][t] = (zin && q0ok) ? md(RHp[um - 1] + rp00, GAp[um - 1] + gp00, ix) * v00 : zc;
        }
        // ---- component 1: F11 (cell, +y pair, in-plane x), F10 (edge01, -x pair, in-plane y)
        {
          const C vmm = V1[ui - S3_UX - 1], vm0 = V1[ui - S3_UX];
          const C v0m = V1[ui - 1], v00 = V1[ui], v0p = V1[ui + 1];
          const C vpm = V1[ui + S3_UX - 1], vp0 = V1[ui + S3_UX], vpp = V1[ui + S3_UX + 1];
          const C u00 = U1[ui], up0 = U1[ui + S3_UX], u0m = U1[ui - 1];
          const C rn0 = (vpm - v0m) + (vpp - v0p) + R(2) * (vp0 - v00);
          const C sz0 = r11m + rn0 + R(2) * r11c;
          d11 = (beta * (up0 - u00) + w * sz0) * (s3_iw<R>(P, zB | fl11) * ih);
          S.f[1][t] = mc00 * d11;
          r11m = r11c;
          r11c = rn0;
          const C rn1 = (vm0 - vmm) + (vp0 - vpm) + R(2) * (v00 - v0m);
          const C sz1 = r10m + rn1 + R(2) * r10c;
          S.f[3][t] = mu01 * ((beta * (u00 - u0m) + w * sz1) * (s3_iw<R>(P, zB | fl10) * ih));
          r10m = r10c;
          r10c = rn1;
          S.di[2][t] = v00 - u00;  // d12 at edge (q, z+1)
          S.q[qb][1][t] =
              (zin && q1ok) ? md(RHp[um - S3_MX] + rp00, GAp[um - S3_MX] + gp00, iy) * v00 : zc;
        }
        // ---- component 2: F20 (edge02, -x pair, in-plane y), F21 (edge12, -y pair, in-plane x)
        {
          const C vmm = V2[ui - S3_UX - 1], vm0 = V2[ui - S3_UX], vmp = V2[ui - S3_UX + 1];
          const C v0m = V2[ui - 1], v00 = V2[ui], v0p = V2[ui + 1];
          const C vpm = V2[ui + S3_UX - 1], vp0 = V2[ui + S3_UX];
          const C u00 = U2[ui], u0m = U2[ui - 1], um0 = U2[ui - S3_UX];
          const C rn0 = (vm0 - vmm) + (vp0 - vpm) + R(2) * (v00 - v0m);
          const C sz0 = r20m + rn0 + R(2) * r20c;
          S.f[4][t] = mu02 * ((beta * (u00 - u0m) + w * sz0) * (s3_iw<R>(P, fl20 | zC) * ih));
          r20m = r20c;
          r20c = rn0;
          const C rn1 = (v0m - vmm) + (v0p - vmp) + R(2) * (v00 - vm0);
          const C sz1 = r21m + rn1 + R(2) * r21c;
          S.f[5][t] = mu12 * ((beta * (u00 - um0) + w * sz1) * (s3_iw<R>(P, fl21 | zC) * ih));
          r21m = r21c;
          r21c = rn1;
          S.di[0][t] = v00 - u00;  // d22 at cell (q, z)
          S.q[qb][2][t] = (zg + 1 >= 0 && zg + 1 <= n2g && q2ok)
                              ? md(RHc[um] + rp00, GAc[um] + gp00, izp) * v00
                              : zc;
        }
      }
      __syncthreads();

      if (interior) {
        // residual mode: fetch b for this plane's rows early (latency overlap)
        C bb0 = zc, bb1 = zc, bb2 = zc, bb3 = zc;
        if (b && z >= zb) {
          if (v0 && z < n2) bb0 = __ldg(&b[o0 + s0 * z]);
          if (v1 && z < n2) bb1 = __ldg(&b[o1 + s1 * z]);
          if (v2) bb2 = __ldg(&b[o2 + s2 * z]);
          if (v2 && z < n2) bb3 = __ldg(&b[o3 + s2 * z]);
        }
        auto filt = [&](const C* D) {
          const C a = D[t - 1 - S3_FX] + D[t + 1 - S3_FX] + R(2) * D[t - S3_FX];
          const C c = D[t - 1 + S3_FX] + D[t + 1 + S3_FX] + R(2) * D[t + S3_FX];
          const C m_ = D[t - 1] + D[t + 1] + R(2) * D[t];
          return a + c + R(2) * m_;
        };
        const C d22 = (beta * S.di[0][t] + w * filt(S.di[0])) * c22;
        const C f22 = MUc[um] * d22;  // zero-filled mu masks cells outside the box
        const R mu02p = (MUc[um - 1] + MUp[um - 1] + MUc[um] + MUp[um]) * (ix * izp);
        const C f02p = mu02p * ((beta * S.di[1][t] + w * filt(S.di[1])) * c02);
        const R mu12p = (MUc[um - S3_MX] + MUp[um - S3_MX] + MUc[um] + MUp[um]) * (iy * izp);
        const C f12p = mu12p * ((beta * S.di[2][t] + w * filt(S.di[2])) * c12);
        const C(*Q)[S3_FN_] = S.q[z & 1];
        const C qc0 = Q[0][t], qc1 = Q[1][t], qc2 = Q[2][t];

        if (z >= zb) {
          const C(*QN)[S3_FN_] = S.q[(z + 1) & 1];
          const C* Pc = S.p[pc_];
          const C pc = Pc[ui];
          auto mass = [&](int k, C qc, C qm, int cnt) -> C {
            C v = beta * qc;
            v += wn * Q[k][t - 1];
            v += wn * Q[k][t + 1];
            v += wn * Q[k][t - S3_FX];
            v += wn * Q[k][t + S3_FX];
            v += wn * qm;
            v += wn * QN[k][t];
            return v * s3_im<R>(P, cnt);
          };
          const int czz = lz + hz0;
          // all four rows evaluated unconditionally (one basic block: the
          // scheduler overlaps their shared-memory loads); stores predicated
          C o0v = (S.f[0][t - 1] - S.f[0][t]) * ih;
          o0v += (S.f[2][t] - S.f[2][t + S3_FX]) * ih;
          o0v += (f02c - f02p) * ih;
          o0v -= mass(0, qc0, qm0, mc0 + czz);
          o0v += (pc - Pc[ui - 1]) * ih;
          C o1v = (S.f[3][t] - S.f[3][t + 1]) * ih;
          o1v += (S.f[1][t - S3_FX] - S.f[1][t]) * ih;
          o1v += (f12c - f12p) * ih;
          o1v -= mass(1, qc1, qm1, mc1 + czz);
          o1v += (pc - Pc[ui - S3_UX]) * ih;
          C o2v = (S.f[4][t] - S.f[4][t + 1]) * ih;
          o2v += (S.f[5][t] - S.f[5][t + S3_FX]) * ih;
          o2v += (f22m - f22) * ih;
          o2v -= mass(2, qc2, qm2, mc2 + lz + hz1);
          o2v += (pc - S.p[pm][ui]) * ih;
          C o3v = d00;
          o3v += d11;
          o3v += d22;
          o3v += S.ilm[z & 3][um] * pc;
          if (v0 && z < n2) y[o0 + s0 * z] = b ? bb0 - o0v : o0v;
          if (v1 && z < n2) y[o1 + s1 * z] = b ? bb1 - o1v : o1v;
          if (v2) y[o2 + s2 * z] = b ? bb2 - o2v : o2v;
          if (v2 && z < n2) y[o3 + s2 * z] = b ? bb3 - o3v : o3v;
        }
        f02c = f02p;
        f12c = f12p;
        f22m = f22;
        qm0 = qc0;
        qm1 = qc1;
        qm2 = qc2;
      }
      su0 = su1;
      pm = pc_;
    }
    // drain the group issued by the last step before the next item reuses smem
    if constexpr (kTma) s3_wait(&S.bar[seq & 1], (seq >> 1) & 1);
    else s3_cp_commit_wait();
    ++seq;
    __syncthreads();
  }
}

inline S3Params make_s3params(const Geo& g, const OpPar& P, int nsm = 148, int z_lo = 0, int z_hi = -1,
                               int ty = S3_TY, int tx = S3_TX) {
  S3Params s;
  s.g = g;
  s.beta = P.beta;
  s.omega2 = P.omega2;
  s.alpha = P.alpha;
  const double w = (1.0 - P.beta) / 16.0;
  s.w = w;
  // wsum in the reference's accumulation order (operator.hpp:289-296)
  for (int f = 0; f < 16; ++f) {
    const bool lo1 = f & 1, hi1 = f & 2, lo2 = f & 4, hi2 = f & 8;
    double wsum = P.beta;
    if (P.beta != 1.0)
      for (int s1 = -1; s1 <= 1; ++s1)
        for (int s2 = -1; s2 <= 1; ++s2) {
          if ((s1 == -1 && !lo1) || (s1 == 1 && !hi1) || (s2 == -1 && !lo2) || (s2 == 1 && !hi2)) continue;
          wsum += w * (double)((s1 == 0 ? 2 : 1) * (s2 == 0 ? 2 : 1));
        }
    s.inv_wsum[f] = P.beta != 1.0 ? 1.0 / wsum : 1.0;
    // operator.hpp:288 with Real = float
    const float wf = (float)((1.0 - P.beta) / 16.0);
    float wsf = (float)P.beta;
    if (P.beta != 1.0)
      for (int s1 = -1; s1 <= 1; ++s1)
        for (int s2 = -1; s2 <= 1; ++s2) {
          if ((s1 == -1 && !lo1) || (s1 == 1 && !hi1) || (s2 == -1 && !lo2) || (s2 == 1 && !hi2)) continue;
          wsf += wf * (float)((s1 == 0 ? 2 : 1) * (s2 == 0 ? 2 : 1));
        }
    s.inv_wsum_f[f] = P.beta != 1.0 ? 1.0f / wsf : 1.0f;
    s.inv_wsum_h[f] = s.inv_wsum[f] * g.inv_h;
  }
  s.wn = (1.0 - P.beta) / 6.0;
  for (int c = 0; c <= 6; ++c) {
    double wsum = P.beta;
    for (int q = 0; q < c; ++q) wsum += s.wn;
    s.inv_msum[c] = P.beta != 1.0 ? 1.0 / wsum : 1.0;
    float wsf = (float)P.beta;
    for (int q = 0; q < c; ++q) wsf += (float)s.wn;
    s.inv_msum_f[c] = P.beta != 1.0 ? 1.0f / wsf : 1.0f;
  }
  for (int c = 0; c < 16; ++c) {
    const int lz = c & 1, hz0 = (c >> 1) & 1, hz1 = (c >> 2) & 1, z0 = (c >> 3) & 1;
    const int zA = (lz << 2) | (hz0 << 3), zB = lz | (hz0 << 1), zC = (lz << 2) | (hz1 << 3);
    const double cA = s.inv_wsum_h[3 | zA], cB = s.inv_wsum_h[zB | 12], cC = s.inv_wsum_h[3 | zC];
    s.zt[c][0] = P.beta * cA, s.zt[c][1] = w * cA;
    s.zt[c][2] = P.beta * cB, s.zt[c][3] = w * cB;
    s.zt[c][4] = P.beta * cC, s.zt[c][5] = w * cC;
    s.zt[c][6] = s.inv_msum[4 + lz + hz0];
    s.zt[c][7] = s.inv_msum[4 + lz + hz1];
    const int cnt = z0 + hz0;
    s.zt[c][8] = cnt == 2 ? 0.5 : (cnt == 1 ? 1.0 : 0.0);
    s.zt[c][9] = s.zt[c][8] * P.omega2;
  }
  s.bw_in[0] = P.beta * s.inv_wsum_h[15], s.bw_in[1] = w * s.inv_wsum_h[15];
  s.ntiles_x = (g.n[0] + 1 + tx - 1) / tx;
  s.ntiles_y = (g.n[1] + 1 + ty - 1) / ty;
  s.itx = s.ity = 0;
  // z-chunks: minimise (rounds of persistent CTAs) x (planes per chunk + 2
  // warm-up planes) over chunk counts with >= 4 planes per chunk, so that
  // the tile x chunk items fill whole waves of the 148 SMs.
  const int tiles = s.ntiles_x * s.ntiles_y;
  s.z_lo = z_lo;
  s.z_hi = z_hi < 0 ? g.n[2] + 1 : z_hi;
  const int n2 = s.z_hi - s.z_lo;  // planes to emit
  int best = 1;
  double best_cost = 1e300;
  for (int nch = 1; nch <= (n2 / 4 > 0 ? n2 / 4 : 1); ++nch) {
    const int64_t items = (int64_t)tiles * nch;
    const int64_t rounds = (items + nsm - 1) / nsm;
    const double cost = (double)rounds * ((n2 + nch - 1) / nch + 2);
    if (cost < best_cost * 0.999) {
      best_cost = cost;
      best = nch;
    }
  }
  s.nchunks = best;
  return s;
}

// ------------------------------------------------------- tensor-map setup
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn s3_encoder() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// 3D float64 map over a (d0*mult, d1, d2) array, box (box0, S3_UY, 1).
inline bool s3_encode(CUtensorMap* map, const void* base, int64_t d0, int64_t d1, int64_t d2, int box0) {
  EncodeTiledFn enc = s3_encoder();
  if (!enc) return false;
  const cuuint64_t dim[3] = {(cuuint64_t)d0, (cuuint64_t)d1, (cuuint64_t)d2};
  const cuuint64_t str[2] = {(cuuint64_t)(d0 * 8), (cuuint64_t)(d0 * d1 * 8)};
  const cuuint32_t box[3] = {(cuuint32_t)box0, (cuuint32_t)S3_UY, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(base), dim, str, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// TMA needs 16-byte global strides: the SoA media rows (n0 doubles) need n0 even.
inline bool stencil3d_supported(const Geo& g) {
  return g.nd == 3 && g.n[0] >= 2 && g.n[1] >= 2 && g.n[0] % 2 == 0 && s3_encoder() != nullptr;
}

// Per-device one-time setup (the shared-memory opt-in is a per-device
// function attribute); returns the SM count of the current device.
inline int s3_device_init() {
  static std::mutex mu;
  static int nsm_of[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  std::lock_guard<std::mutex> lock(mu);
  if (!nsm_of[dev]) {
    cudaFuncSetAttribute(k_stencil3d<cplxf>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(S3SmemT<cplxf>));
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    nsm_of[dev] = nsm > 0 ? nsm : 148;
  }
  return nsm_of[dev];
}

// complex64 variant (single-precision hierarchy): media_soa holds the four
// float cell arrays; planes are loaded with cp.async, so no tensor maps.
// Fallback for n0 % 4 != 0 (ehmg_stencil3d_rr.cuh dispatches).
inline void launch_stencil3d_ca(const Geo& g, const OpPar& P, const float* media_soa, const cplxf* x,
                                const cplxf* b, cplxf* y, cudaStream_t s, int z_lo = 0, int z_hi = -1) {
  const int nsm = s3_device_init();
  const int64_t nc = g.ncells;
  S3Src src;
  for (int k = 0; k < 3; ++k) src.u[k] = x + g.off[k];
  src.p = x + g.off[3];
  src.mu = media_soa;
  src.rho = media_soa + nc;
  src.gam = media_soa + 2 * nc;
  src.ilm = media_soa + 3 * nc;
  const S3Params sp = make_s3params(g, P, nsm, z_lo, z_hi, S3Cfg<cplxf>::TY);
  if (sp.z_hi <= sp.z_lo) return;
  const int items = sp.ntiles_x * sp.ntiles_y * sp.nchunks;
  const int grid = items < nsm ? items : nsm;
  k_stencil3d<cplxf><<<grid, S3Cfg<cplxf>::THREADS, sizeof(S3SmemT<cplxf>), s>>>(S3Maps{}, src, sp, b, y);
}

}  // namespace ehmg
