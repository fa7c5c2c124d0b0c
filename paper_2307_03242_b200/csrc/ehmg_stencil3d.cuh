// ehmg_stencil3d.cuh -- bandwidth-tuned 3D operator / residual kernel.
//
// y = H x  or  r = b - H x  for the staggered mixed elastic-Helmholtz
// operator (operator.hpp:389-421), all four components in one launch.
//
// Design (B200, complex128, HBM-bound):
//  * 2.5D tiling. A CTA owns a 32x8 tile of the (i,j) index plane plus a
//    one-cell flux halo (34x10 = 340 positions, one thread each, 11 warps)
//    and marches a z-chunk. u0,u1,u2 (planes z, z+1), p (z-1, z) and the
//    cell media (z-1..z+1) sit in shared-memory rings; the next plane is
//    fetched with cp.async 16-byte copies, zero-filled outside each
//    component's box (= the reference's zero ghosts), while the current
//    plane is computed.
//  * Separable spread derivatives. The 9-tap transverse (1,2,1)x(1,2,1)
//    spread of every first derivative (operator.hpp:267 / :306) is split
//    into an in-plane 3-tap row sum and a z-direction 3-tap combination; the
//    row sums of the previous two planes are carried in registers, so each
//    flux costs one row sum per plane. The three purely in-plane families
//    (F22, F02, F12) filter a shared-memory difference field.
//  * Flux sharing. Each flux is evaluated once and shared through shared
//    memory by the two rows that use it; z-neighbour fluxes and mass
//    products are carried in registers.
//  * Exactness. Boundary renormalisations (1/wsum, mass 1/wsum) come from
//    tables built on the host in the reference's accumulation order; edge /
//    face media averages divide by 1, 2 or 4, applied as exact reciprocal
//    multiplies. Results match the reference to rounding (<= 1e-13 rel).
#pragma once

#include "ehmg_core.cuh"

namespace ehmg {

constexpr int S3_TX = 32, S3_TY = 8;
constexpr int S3_UX = S3_TX + 4, S3_UY = S3_TY + 4, S3_UN = S3_UX * S3_UY;  // origin (i0-2, j0-2)
constexpr int S3_FX = S3_TX + 2, S3_FY = S3_TY + 2, S3_FN = S3_FX * S3_FY;  // origin (i0-1, j0-1)
constexpr int S3_THREADS = ((S3_FN + 31) / 32) * 32;                         // 352
constexpr int S3_ZCHUNK = 32;

struct S3Params {
  Geo g;
  double beta, omega2, alpha, w;  // w = (1-beta)/16
  double inv_wsum[16];            // 1/wsum by transverse validity bits (lo1,hi1,lo2,hi2)
  double wn;                      // (1-beta)/6
  double inv_msum[7];             // 1/(beta + k*wn), k valid mass neighbours
  int nchunks, ntiles_x, ntiles_y;
};

struct S3Smem {
  cplx u[3][3][S3_UN];   // [plane % 3][component]
  cplx p[3][S3_UN];      // [plane % 3]
  double mu[4][S3_UN], rho[4][S3_UN], gam[4][S3_UN], ilm[4][S3_UN];  // [plane % 4]
  cplx f[6][S3_FN];      // z-family fluxes at plane z: F00 F11 F01 F10 F20 F21
  cplx di[3][S3_FN];     // in-plane difference fields: d22 (cell z), d02, d12 (edge z+1)
  cplx q[2][3][S3_FN];   // mass products md*u [plane & 1][component]
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int bytes = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int bytes = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }

__device__ __forceinline__ int mod3(int z) { return ((z % 3) + 3) % 3; }

// u planes
__device__ __forceinline__ void s3_load_u(S3Smem& S, const Geo& g, const cplx* __restrict__ x, int i0,
                                          int j0, int z) {
  const int sl = mod3(z);
  for (int t = threadIdx.x; t < S3_UN; t += S3_THREADS) {
    const int xg = i0 - 2 + t % S3_UX, yg = j0 - 2 + t / S3_UX;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const int d0 = g.n[0] + (k == 0), d1 = g.n[1] + (k == 1), d2 = g.n[2] + (k == 2);
      const bool ok = xg >= 0 && xg < d0 && yg >= 0 && yg < d1 && z >= 0 && z < d2;
      const cplx* src = ok ? x + g.off[k] + xg + (int64_t)d0 * (yg + (int64_t)d1 * z) : x;
      cp_async16(&S.u[sl][k][t], src, ok);
    }
  }
}
// p plane
__device__ __forceinline__ void s3_load_p(S3Smem& S, const Geo& g, const cplx* __restrict__ x, int i0,
                                          int j0, int z) {
  const int sl = mod3(z);
  for (int t = threadIdx.x; t < S3_UN; t += S3_THREADS) {
    const int xg = i0 - 2 + t % S3_UX, yg = j0 - 2 + t / S3_UX;
    const bool ok = z >= 0 && z < g.n[2] && xg >= 0 && xg < g.n[0] && yg >= 0 && yg < g.n[1];
    const cplx* src = ok ? x + g.off[3] + xg + (int64_t)g.n[0] * (yg + (int64_t)g.n[1] * z) : x;
    cp_async16(&S.p[sl][t], src, ok);
  }
}
// media plane (SoA in shared memory)
__device__ __forceinline__ void s3_load_m(S3Smem& S, const Geo& g, const Cell* __restrict__ m, int i0,
                                          int j0, int z) {
  const int sl = z & 3;
  for (int t = threadIdx.x; t < S3_UN; t += S3_THREADS) {
    const int xg = i0 - 2 + t % S3_UX, yg = j0 - 2 + t / S3_UX;
    const bool ok = z >= 0 && z < g.n[2] && xg >= 0 && xg < g.n[0] && yg >= 0 && yg < g.n[1];
    const double* src =
        reinterpret_cast<const double*>(ok ? m + xg + (int64_t)g.n[0] * (yg + (int64_t)g.n[1] * z) : m);
    cp_async8(&S.mu[sl][t], src + 0, ok);
    cp_async8(&S.rho[sl][t], src + 1, ok);
    cp_async8(&S.gam[sl][t], src + 2, ok);
    cp_async8(&S.ilm[sl][t], src + 3, ok);
  }
}

// transverse validity bits of family (K, J) at global q
template <int K, int J>
__device__ __forceinline__ int s3_vflags(const Geo& g, int x, int y, int z) {
  constexpr int T1 = (J == K) ? (K + 1) % 3 : 3 - K - J;
  constexpr int T2 = (J == K) ? (K + 2) % 3 : K;
  const int q[3] = {x, y, z};
  const int L1 = g.n[T1] + (T1 == K), L2 = g.n[T2] + (T2 == K);
  return (q[T1] >= 1) | ((q[T1] + 1 < L1) << 1) | ((q[T2] >= 1) << 2) | ((q[T2] + 1 < L2) << 3);
}

// 1/count for count in {0,1,2,4} (media averages: exact reciprocal multiply)
__device__ __forceinline__ double inv_cnt(int c) { return c == 4 ? 0.25 : (c == 2 ? 0.5 : (c == 1 ? 1.0 : 0.0)); }

// ----------------------------------------------------------------- kernel
__global__ void __launch_bounds__(S3_THREADS, 1)
    k_stencil3d(S3Params P, const Cell* __restrict__ m, const cplx* __restrict__ x,
                const cplx* __restrict__ b, cplx* __restrict__ y) {
  extern __shared__ __align__(16) unsigned char s3_raw[];
  S3Smem& S = *reinterpret_cast<S3Smem*>(s3_raw);
  const Geo& g = P.g;
  const int t = threadIdx.x;
  const bool act = t < S3_FN;
  const int fx = act ? t % S3_FX : 1, fy = act ? t / S3_FX : 1;
  const int ui = (fx + 1) + S3_UX * (fy + 1);  // own U-local index
  const bool interior = act && fx >= 1 && fx <= S3_TX && fy >= 1 && fy <= S3_TY;
  const double beta = P.beta, w = P.w, ih = g.inv_h;
  const int n0 = g.n[0], n1 = g.n[1], n2 = g.n[2];

  const int items = P.ntiles_x * P.ntiles_y * P.nchunks;
  for (int item = blockIdx.x; item < items; item += gridDim.x) {
    const int tile = item % (P.ntiles_x * P.ntiles_y);
    const int chunk = item / (P.ntiles_x * P.ntiles_y);
    const int i0 = (tile % P.ntiles_x) * S3_TX, j0 = (tile / P.ntiles_x) * S3_TY;
    const int zb = (int)(((int64_t)chunk * n2) / P.nchunks);
    const int zend = (chunk + 1 == P.nchunks) ? n2 + 1 : (int)(((int64_t)(chunk + 1) * n2) / P.nchunks);
    const int xg = i0 - 1 + fx, yg = j0 - 1 + fy;

    __syncthreads();  // previous item fully consumed
    // prologue for the first (warm-up) step z = zb-2
    s3_load_u(S, g, x, i0, j0, zb - 2);
    s3_load_u(S, g, x, i0, j0, zb - 1);
    s3_load_m(S, g, m, i0, j0, zb - 3);
    s3_load_m(S, g, m, i0, j0, zb - 2);
    s3_load_m(S, g, m, i0, j0, zb - 1);
    s3_load_p(S, g, x, i0, j0, zb - 3);
    s3_load_p(S, g, x, i0, j0, zb - 2);
    cp_async_commit();

    // carries (registers)
    cplx r00m = mk(0, 0), r00c = mk(0, 0), r11m = mk(0, 0), r11c = mk(0, 0);
    cplx r01m = mk(0, 0), r01c = mk(0, 0), r10m = mk(0, 0), r10c = mk(0, 0);
    cplx r20m = mk(0, 0), r20c = mk(0, 0), r21m = mk(0, 0), r21c = mk(0, 0);
    cplx f02c = mk(0, 0), f12c = mk(0, 0), f22m = mk(0, 0);
    cplx qm0 = mk(0, 0), qm1 = mk(0, 0), qm2 = mk(0, 0);

    for (int z = zb - 2; z < zend; ++z) {
      cp_async_wait_all();
      __syncthreads();
      s3_load_u(S, g, x, i0, j0, z + 2);
      s3_load_m(S, g, m, i0, j0, z + 2);
      s3_load_p(S, g, x, i0, j0, z + 1);
      cp_async_commit();

      const cplx* U0 = S.u[mod3(z)][0];
      const cplx* U1 = S.u[mod3(z)][1];
      const cplx* U2 = S.u[mod3(z)][2];
      const cplx* V0 = S.u[mod3(z + 1)][0];
      const cplx* V1 = S.u[mod3(z + 1)][1];
      const cplx* V2 = S.u[mod3(z + 1)][2];
      const double* MUm = S.mu[(z - 1) & 3];
      const double* MUc = S.mu[z & 3];
      const double* MUp = S.mu[(z + 1) & 3];
      cplx d00 = mk(0, 0), d11 = mk(0, 0);

      if (act) {
        // ---- z-families: in-plane row sum at z+1, z-combination, flux at z
        // F00: cell, pair +x, in-plane axis y
        {
          auto dn = [&](int o) { return V0[ui + o + 1] - V0[ui + o]; };
          const cplx rn = dn(-S3_UX) + dn(S3_UX) + 2.0 * dn(0);
          const cplx s = r00m + rn + 2.0 * r00c;
          const cplx v = beta * (U0[ui + 1] - U0[ui]) + w * s;
          d00 = v * (P.inv_wsum[s3_vflags<0, 0>(g, xg, yg, z)] * ih);
          S.f[0][t] = MUc[ui] * d00;
          r00m = r00c;
          r00c = rn;
        }
        // F11: cell, pair +y, in-plane axis x
        {
          auto dn = [&](int o) { return V1[ui + o + S3_UX] - V1[ui + o]; };
          const cplx rn = dn(-1) + dn(1) + 2.0 * dn(0);
          const cplx s = r11m + rn + 2.0 * r11c;
          const cplx v = beta * (U1[ui + S3_UX] - U1[ui]) + w * s;
          d11 = v * (P.inv_wsum[s3_vflags<1, 1>(g, xg, yg, z)] * ih);
          S.f[1][t] = MUc[ui] * d11;
          r11m = r11c;
          r11c = rn;
        }
        // mu on the (0,1) edge at plane z (cells x-1..x, y-1..y)
        const double mu01 = (MUc[ui - 1 - S3_UX] + MUc[ui - 1] + MUc[ui - S3_UX] + MUc[ui]) *
                            inv_cnt(((xg >= 1) + (xg < n0)) * ((yg >= 1) + (yg < n1)));
        // F01: edge (0,1), pair u0(b)-u0(b-y), in-plane axis x
        {
          auto dn = [&](int o) { return V0[ui + o] - V0[ui + o - S3_UX]; };
          const cplx rn = dn(-1) + dn(1) + 2.0 * dn(0);
          const cplx s = r01m + rn + 2.0 * r01c;
          const cplx v = beta * (U0[ui] - U0[ui - S3_UX]) + w * s;
          S.f[2][t] = mu01 * (v * (P.inv_wsum[s3_vflags<0, 1>(g, xg, yg, z)] * ih));
          r01m = r01c;
          r01c = rn;
        }
        // F10: edge (0,1), pair u1(b)-u1(b-x), in-plane axis y
        {
          auto dn = [&](int o) { return V1[ui + o] - V1[ui + o - 1]; };
          const cplx rn = dn(-S3_UX) + dn(S3_UX) + 2.0 * dn(0);
          const cplx s = r10m + rn + 2.0 * r10c;
          const cplx v = beta * (U1[ui] - U1[ui - 1]) + w * s;
          S.f[3][t] = mu01 * (v * (P.inv_wsum[s3_vflags<1, 0>(g, xg, yg, z)] * ih));
          r10m = r10c;
          r10c = rn;
        }
        // F20: edge (0,2) at plane z, pair u2(b)-u2(b-x), in-plane axis y
        {
          const double mu02 = (MUm[ui - 1] + MUc[ui - 1] + MUm[ui] + MUc[ui]) *
                              inv_cnt(((xg >= 1) + (xg < n0)) * ((z >= 1) + (z < n2)));
          auto dn = [&](int o) { return V2[ui + o] - V2[ui + o - 1]; };
          const cplx rn = dn(-S3_UX) + dn(S3_UX) + 2.0 * dn(0);
          const cplx s = r20m + rn + 2.0 * r20c;
          const cplx v = beta * (U2[ui] - U2[ui - 1]) + w * s;
          S.f[4][t] = mu02 * (v * (P.inv_wsum[s3_vflags<2, 0>(g, xg, yg, z)] * ih));
          r20m = r20c;
          r20c = rn;
        }
        // F21: edge (1,2) at plane z, pair u2(b)-u2(b-y), in-plane axis x
        {
          const double mu12 = (MUm[ui - S3_UX] + MUc[ui - S3_UX] + MUm[ui] + MUc[ui]) *
                              inv_cnt(((yg >= 1) + (yg < n1)) * ((z >= 1) + (z < n2)));
          auto dn = [&](int o) { return V2[ui + o] - V2[ui + o - S3_UX]; };
          const cplx rn = dn(-1) + dn(1) + 2.0 * dn(0);
          const cplx s = r21m + rn + 2.0 * r21c;
          const cplx v = beta * (U2[ui] - U2[ui - S3_UX]) + w * s;
          S.f[5][t] = mu12 * (v * (P.inv_wsum[s3_vflags<2, 1>(g, xg, yg, z)] * ih));
          r21m = r21c;
          r21c = rn;
        }
        // ---- in-plane difference fields
        S.di[0][t] = V2[ui] - U2[ui];  // d22 at cell (q, z)
        S.di[1][t] = V0[ui] - U0[ui];  // d02 at edge (q, z+1)
        S.di[2][t] = V1[ui] - U1[ui];  // d12 at edge (q, z+1)
        // ---- mass products at plane z+1 (operator.hpp:132, :365)
        {
          const double* RHc = S.rho[z & 3];
          const double* RHp = S.rho[(z + 1) & 3];
          const double* GAc = S.gam[z & 3];
          const double* GAp = S.gam[(z + 1) & 3];
          const int zf = z + 1;
          const double al = P.alpha, w2 = P.omega2;
          auto md = [&](double sr, double sg, int cnt) {
            const double ic = inv_cnt(cnt);
            const double rho_f = sr * ic, gam_f = sg * ic + al;
            return mk(w2 * rho_f, -w2 * gam_f * rho_f);
          };
          const bool zin = zf >= 0 && zf < n2;
          const bool ok0 = zin && yg >= 0 && yg < n1 && xg >= 0 && xg <= n0;
          const bool ok1 = zin && xg >= 0 && xg < n0 && yg >= 0 && yg <= n1;
          const bool ok2 = zf >= 0 && zf <= n2 && xg >= 0 && xg < n0 && yg >= 0 && yg < n1;
          const cplx q0 = ok0 ? md(RHp[ui - 1] + RHp[ui], GAp[ui - 1] + GAp[ui], (xg >= 1) + (xg < n0)) * V0[ui]
                              : mk(0, 0);
          const cplx q1 = ok1 ? md(RHp[ui - S3_UX] + RHp[ui], GAp[ui - S3_UX] + GAp[ui], (yg >= 1) + (yg < n1)) * V1[ui]
                              : mk(0, 0);
          const cplx q2 = ok2 ? md(RHc[ui] + RHp[ui], GAc[ui] + GAp[ui], (zf >= 1) + (zf < n2)) * V2[ui] : mk(0, 0);
          S.q[(z + 1) & 1][0][t] = q0;
          S.q[(z + 1) & 1][1][t] = q1;
          S.q[(z + 1) & 1][2][t] = q2;
        }
      }
      __syncthreads();

      if (interior) {
        // ---- in-plane families (own column)
        auto filt = [&](const cplx* D) {
          const cplx a = D[t - 1 - S3_FX] + D[t + 1 - S3_FX] + 2.0 * D[t - S3_FX];
          const cplx c = D[t - 1 + S3_FX] + D[t + 1 + S3_FX] + 2.0 * D[t + S3_FX];
          const cplx m_ = D[t - 1] + D[t + 1] + 2.0 * D[t];
          return a + c + 2.0 * m_;
        };
        const cplx d22 = (beta * S.di[0][t] + w * filt(S.di[0])) *
                         (P.inv_wsum[s3_vflags<2, 2>(g, xg, yg, z)] * ih);
        const cplx f22 = MUc[ui] * d22;  // zero-filled mu masks cells outside the box
        const double mu02p = (MUc[ui - 1] + MUp[ui - 1] + MUc[ui] + MUp[ui]) *
                             inv_cnt(((xg >= 1) + (xg < n0)) * ((z + 1 >= 1) + (z + 1 < n2)));
        const cplx f02p = mu02p * ((beta * S.di[1][t] + w * filt(S.di[1])) *
                                   (P.inv_wsum[s3_vflags<0, 2>(g, xg, yg, z + 1)] * ih));
        const double mu12p = (MUc[ui - S3_UX] + MUp[ui - S3_UX] + MUc[ui] + MUp[ui]) *
                             inv_cnt(((yg >= 1) + (yg < n1)) * ((z + 1 >= 1) + (z + 1 < n2)));
        const cplx f12p = mu12p * ((beta * S.di[2][t] + w * filt(S.di[2])) *
                                   (P.inv_wsum[s3_vflags<1, 2>(g, xg, yg, z + 1)] * ih));
        const cplx (*Q)[S3_FN] = S.q[z & 1];
        const cplx qc0 = Q[0][t], qc1 = Q[1][t], qc2 = Q[2][t];
        const cplx qn0 = S.q[(z + 1) & 1][0][t], qn1 = S.q[(z + 1) & 1][1][t], qn2 = S.q[(z + 1) & 1][2][t];

        if (z >= zb) {
          const cplx* Pc = S.p[mod3(z)];
          const cplx pc = Pc[ui];
          auto mass = [&](int k, cplx qc, cplx qm, cplx qn, int cnt) -> cplx {
            cplx v = beta * qc;
            v += P.wn * Q[k][t - 1];
            v += P.wn * Q[k][t + 1];
            v += P.wn * Q[k][t - S3_FX];
            v += P.wn * Q[k][t + S3_FX];
            v += P.wn * qm;
            v += P.wn * qn;
            return v * P.inv_msum[cnt];
          };
          const int cx0 = (xg >= 1) + (xg + 1 < n0), cy0 = (yg >= 1) + (yg + 1 < n1), cz0 = (z >= 1) + (z + 1 < n2);
          // u0 row (operator.hpp:389 / :409)
          if (xg <= n0 && yg < n1 && z < n2) {
            cplx out = (S.f[0][t - 1] - S.f[0][t]) * ih;
            out += (S.f[2][t] - S.f[2][t + S3_FX]) * ih;
            out += (f02c - f02p) * ih;
            out -= mass(0, qc0, qm0, qn0, ((xg >= 1) + (xg + 1 < n0 + 1)) + cy0 + cz0);
            out += (pc - Pc[ui - 1]) * ih;
            const int64_t r = g.off[0] + xg + (int64_t)(n0 + 1) * (yg + (int64_t)n1 * z);
            y[r] = b ? b[r] - out : out;
          }
          // u1 row
          if (xg < n0 && yg <= n1 && z < n2) {
            cplx out = (S.f[3][t] - S.f[3][t + 1]) * ih;
            out += (S.f[1][t - S3_FX] - S.f[1][t]) * ih;
            out += (f12c - f12p) * ih;
            out -= mass(1, qc1, qm1, qn1, cx0 + ((yg >= 1) + (yg + 1 < n1 + 1)) + cz0);
            out += (pc - Pc[ui - S3_UX]) * ih;
            const int64_t r = g.off[1] + xg + (int64_t)n0 * (yg + (int64_t)(n1 + 1) * z);
            y[r] = b ? b[r] - out : out;
          }
          // u2 row
          if (xg < n0 && yg < n1 && z <= n2) {
            cplx out = (S.f[4][t] - S.f[4][t + 1]) * ih;
            out += (S.f[5][t] - S.f[5][t + S3_FX]) * ih;
            out += (f22m - f22) * ih;
            out -= mass(2, qc2, qm2, qn2, cx0 + cy0 + ((z >= 1) + (z + 1 < n2 + 1)));
            out += (pc - S.p[mod3(z - 1)][ui]) * ih;
            const int64_t r = g.off[2] + xg + (int64_t)n0 * (yg + (int64_t)n1 * z);
            y[r] = b ? b[r] - out : out;
          }
          // p row (operator.hpp:416)
          if (xg < n0 && yg < n1 && z < n2) {
            cplx out = d00;
            out += d11;
            out += d22;
            out += S.ilm[z & 3][ui] * pc;
            const int64_t r = g.off[3] + xg + (int64_t)n0 * (yg + (int64_t)n1 * z);
            y[r] = b ? b[r] - out : out;
          }
        }
        f02c = f02p;
        f12c = f12p;
        f22m = f22;
        qm0 = qc0;
        qm1 = qc1;
        qm2 = qc2;
      }
    }
    cp_async_wait_all();
  }
}

inline S3Params make_s3params(const Geo& g, const OpPar& P) {
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
  }
  s.wn = (1.0 - P.beta) / 6.0;
  for (int c = 0; c <= 6; ++c) {
    double wsum = P.beta;
    for (int q = 0; q < c; ++q) wsum += s.wn;
    s.inv_msum[c] = P.beta != 1.0 ? 1.0 / wsum : 1.0;
  }
  s.ntiles_x = (g.n[0] + 1 + S3_TX - 1) / S3_TX;
  s.ntiles_y = (g.n[1] + 1 + S3_TY - 1) / S3_TY;
  s.nchunks = (g.n[2] + S3_ZCHUNK / 2) / S3_ZCHUNK;
  if (s.nchunks < 1) s.nchunks = 1;
  return s;
}

inline bool stencil3d_supported(const Geo& g) { return g.nd == 3 && g.n[0] >= 2 && g.n[1] >= 2; }

inline void launch_stencil3d(const Geo& g, const OpPar& P, const Cell* m, const cplx* x, const cplx* b,
                             cplx* y, cudaStream_t s) {
  static int nsm = 0;
  const size_t smem = sizeof(S3Smem);
  if (!nsm) {
    cudaFuncSetAttribute(k_stencil3d, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (nsm <= 0) nsm = 148;
  }
  const S3Params sp = make_s3params(g, P);
  const int items = sp.ntiles_x * sp.ntiles_y * sp.nchunks;
  const int grid = items < nsm ? items : nsm;
  k_stencil3d<<<grid, S3_THREADS, smem, s>>>(sp, m, x, b, y);
}

}  // namespace ehmg
