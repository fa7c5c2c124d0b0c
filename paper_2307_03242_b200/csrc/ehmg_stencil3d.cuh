// ehmg_stencil3d.cuh -- bandwidth-tuned 3D operator / residual kernel.
//
// y = H x  or  r = b - H x  for the staggered mixed elastic-Helmholtz
// operator (operator.hpp:389-421), one launch for all four components.
//
// Design (B200):
//  * 2.5D tiling: a CTA owns a 32x8 column tile of the (n+1)^2 face/cell
//    index plane and marches a z-chunk. u0,u1,u2,p and the packed cell media
//    for planes z-1..z+1 live in a 4-slot shared-memory ring; plane z+2 is
//    fetched with cp.async (16-byte complex128 copies, zero-filled outside
//    each component's box == the reference's zero ghosts) while plane z is
//    computed.
//  * Flux sharing: every spread first-derivative flux F_kj (operator.hpp:344,
//    :350) is evaluated once per plane on the tile + 1-cell halo and shared
//    through shared memory by the two rows that use it; z-neighbour fluxes
//    (F_02, F_12, F_22) and the z-neighbour mass products are carried in
//    registers along the march. The spread derivative keeps the reference's
//    9-tap loop order; its boundary renormalisation 1/wsum, the mass
//    renormalisation and the edge/face media averages are looked up from
//    validity bits (tables built on the host with the reference's own
//    accumulation order), so results agree with the reference to rounding.
#pragma once

#include "ehmg_core.cuh"

namespace ehmg {

constexpr int S3_TX = 32, S3_TY = 8, S3_THREADS = S3_TX * S3_TY;
constexpr int S3_UX = S3_TX + 4, S3_UY = S3_TY + 4, S3_UN = S3_UX * S3_UY;  // origin (i0-2, j0-2)
constexpr int S3_FX = S3_TX + 2, S3_FY = S3_TY + 2, S3_FN = S3_FX * S3_FY;  // origin (i0-1, j0-1)
constexpr int S3_ZCHUNK = 32;

struct S3Params {
  Geo g;
  double beta, omega2, alpha;
  double wt[3];          // (1-beta)/16 * {1, 2, 4}
  double inv_wsum[16];   // 1/wsum by transverse validity bits (lo1,hi1,lo2,hi2)
  double wn;             // (1-beta)/6
  double inv_msum[7];    // 1/(beta + k*wn), k valid mass neighbours
};

struct S3Smem {
  cplx u[4][3][S3_UN];
  cplx p[4][S3_UN];
  Cell m[4][S3_UN];
  cplx d00[S3_FN], d11[S3_FN];                          // cell derivative (no mu)
  cplx f01[S3_FN], f10[S3_FN], f20[S3_FN], f21[S3_FN];  // edge fluxes (mu included)
  cplx q[3][S3_FN];                                      // mass products md*u
};

__device__ __forceinline__ int s3_slot(int z) { return z & 3; }

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int bytes = pred ? 16 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Issue the loads of plane z (u0..u2, p, media) into its ring slot.
__device__ __forceinline__ void s3_load_plane(S3Smem& S, const S3Params& P, const cplx* __restrict__ x,
                                              const Cell* __restrict__ m, int i0, int j0, int z) {
  const Geo& g = P.g;
  const int sl = s3_slot(z);
  const bool zc_ok = z >= 0 && z < g.n[2];
  for (int t = threadIdx.x; t < S3_UN; t += S3_THREADS) {
    const int lx = t % S3_UX, ly = t / S3_UX;
    const int xg = i0 - 2 + lx, yg = j0 - 2 + ly;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const int d0 = g.n[0] + (k == 0), d1 = g.n[1] + (k == 1), d2 = g.n[2] + (k == 2);
      const bool ok = xg >= 0 && xg < d0 && yg >= 0 && yg < d1 && z >= 0 && z < d2;
      const cplx* src = ok ? x + g.off[k] + xg + (int64_t)d0 * (yg + (int64_t)d1 * z) : x;
      cp_async16(&S.u[sl][k][t], src, ok);
    }
    const bool cok = zc_ok && xg >= 0 && xg < g.n[0] && yg >= 0 && yg < g.n[1];
    const int64_t ci = cok ? xg + (int64_t)g.n[0] * (yg + (int64_t)g.n[1] * z) : 0;
    cp_async16(&S.p[sl][t], cok ? x + g.off[3] + ci : x, cok);
    const char* ms = reinterpret_cast<const char*>(m + ci);
    cp_async16(reinterpret_cast<char*>(&S.m[sl][t]), ms, cok);
    cp_async16(reinterpret_cast<char*>(&S.m[sl][t]) + 16, ms + 16, cok);
  }
}

// u_k at U-local (lx, ly) on plane z+dz.
template <int K>
__device__ __forceinline__ cplx s3_u(const S3Smem& S, int z, int lx, int ly, int dz) {
  return S.u[s3_slot(z + dz)][K][lx + S3_UX * ly];
}

// Spread first derivative of u_K along J at U-local (lx, ly), plane z+dz0
// (operator.hpp:267 dspread_cell when J==K, :306 dspread_edge otherwise);
// vflags = transverse validity bits. Returns the value times inv_h.
template <int K, int J>
__device__ __forceinline__ cplx s3_spread(const S3Smem& S, const S3Params& P, int z, int lx, int ly,
                                          int dz0, int vflags) {
  constexpr int T1 = (J == K) ? (K + 1) % 3 : 3 - K - J;
  constexpr int T2 = (J == K) ? (K + 2) % 3 : K;
  auto pair = [&](int ox, int oy, int oz) -> cplx {
    const int x = lx + ox, y = ly + oy, dz = dz0 + oz;
    if (J == K) {
      const int px = x + (K == 0), py = y + (K == 1), pz = dz + (K == 2);
      return s3_u<K>(S, z, px, py, pz) - s3_u<K>(S, z, x, y, dz);
    } else {
      const int mx = x - (J == 0), my = y - (J == 1), mz = dz - (J == 2);
      return s3_u<K>(S, z, x, y, dz) - s3_u<K>(S, z, mx, my, mz);
    }
  };
  cplx v = P.beta * pair(0, 0, 0);
  if (P.beta != 1.0) {
#pragma unroll
    for (int s1 = -1; s1 <= 1; ++s1)
#pragma unroll
      for (int s2 = -1; s2 <= 1; ++s2) {
        const int o[3] = {(T1 == 0 ? s1 : 0) + (T2 == 0 ? s2 : 0), (T1 == 1 ? s1 : 0) + (T2 == 1 ? s2 : 0),
                          (T1 == 2 ? s1 : 0) + (T2 == 2 ? s2 : 0)};
        const double wt = P.wt[(s1 == 0) + (s2 == 0)];
        v += wt * pair(o[0], o[1], o[2]);
      }
    v = v * P.inv_wsum[vflags];
  }
  return v * P.g.inv_h;
}

// Transverse validity bits of flux family (K, J) at global position q.
template <int K, int J>
__device__ __forceinline__ int s3_vflags(const Geo& g, int x, int y, int z) {
  constexpr int T1 = (J == K) ? (K + 1) % 3 : 3 - K - J;
  constexpr int T2 = (J == K) ? (K + 2) % 3 : K;
  const int q[3] = {x, y, z};
  const int L1 = g.n[T1] + (T1 == K), L2 = g.n[T2] + (T2 == K);
  return (q[T1] >= 1) | ((q[T1] + 1 < L1) << 1) | ((q[T2] >= 1) << 2) | ((q[T2] + 1 < L2) << 3);
}

// mu on the edge staggered in (A,B) at global (x,y,z): mean of in-range
// cells (operator.hpp:108); zero-filled staging makes the sum exact.
template <int A, int B>
__device__ __forceinline__ double s3_mu_edge(const S3Smem& S, const Geo& g, int z, int lx, int ly, int dz,
                                             int x, int y, int ze) {
  double s = 0;
#pragma unroll
  for (int da = -1; da <= 0; ++da)
#pragma unroll
    for (int db = -1; db <= 0; ++db) {
      const int ox = (A == 0 ? da : 0) + (B == 0 ? db : 0);
      const int oy = (A == 1 ? da : 0) + (B == 1 ? db : 0);
      const int oz = (A == 2 ? da : 0) + (B == 2 ? db : 0);
      s += S.m[s3_slot(z + dz + oz)][(lx + ox) + S3_UX * (ly + oy)].x;
    }
  const int q[3] = {x, y, ze};
  const int ca = (q[A] >= 1) + (q[A] < g.n[A]);
  const int cb = (q[B] >= 1) + (q[B] < g.n[B]);
  const int cnt = ca * cb;
  return cnt ? s / cnt : 0.0;
}

// Face mass product md_K(f) * u_K(f) (operator.hpp:132, :365).
template <int K>
__device__ __forceinline__ cplx s3_massq(const S3Smem& S, const S3Params& P, int z, int lx, int ly, int dz,
                                         int x, int y, int zf) {
  const Geo& g = P.g;
  const int f[3] = {x, y, zf};
  if (x < 0 || y < 0 || zf < 0 || x >= g.n[0] + (K == 0) || y >= g.n[1] + (K == 1) ||
      zf >= g.n[2] + (K == 2))
    return mk(0, 0);
  const Cell a = S.m[s3_slot(z + dz - (K == 2))][(lx - (K == 0)) + S3_UX * (ly - (K == 1))];
  const Cell b = S.m[s3_slot(z + dz)][lx + S3_UX * ly];
  const double sr = a.y + b.y, sg = a.z + b.z;
  const int cnt = (f[K] >= 1) + (f[K] < g.n[K]);
  const double rho_f = sr / cnt, gam_f = sg / cnt + P.alpha;
  const cplx md = mk(P.omega2 * rho_f, -P.omega2 * gam_f * rho_f);
  return md * s3_u<K>(S, z, lx, ly, dz);
}

template <int K>
__device__ __forceinline__ int s3_mass_count(const Geo& g, int x, int y, int z) {
  const int f[3] = {x, y, z};
  int c = 0;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const int L = g.n[a] + (a == K);
    c += (f[a] >= 1) + (f[a] + 1 < L);
  }
  return c;
}

__global__ void __launch_bounds__(S3_THREADS, 1)
    k_stencil3d(S3Params P, const Cell* __restrict__ m, const cplx* __restrict__ x,
                const cplx* __restrict__ b, cplx* __restrict__ y) {
  extern __shared__ __align__(16) unsigned char s3_raw[];
  S3Smem& S = *reinterpret_cast<S3Smem*>(s3_raw);
  const Geo& g = P.g;
  const int i0 = blockIdx.x * S3_TX, j0 = blockIdx.y * S3_TY;
  const int zb = blockIdx.z * S3_ZCHUNK;
  const int zend = min(zb + S3_ZCHUNK, g.n[2] + 1);
  const int tx = threadIdx.x % S3_TX, ty = threadIdx.x / S3_TX;
  const int xi = i0 + tx, yj = j0 + ty;
  const int ulx = tx + 2, uly = ty + 2;         // own U-local
  const int fpos = (tx + 1) + S3_FX * (ty + 1);  // own F-local

  // prologue: planes zb-2 .. zb; the march starts one warm-up plane early
  s3_load_plane(S, P, x, m, i0, j0, zb - 2);
  s3_load_plane(S, P, x, m, i0, j0, zb - 1);
  s3_load_plane(S, P, x, m, i0, j0, zb);
  cp_async_commit();

  cplx f02c = mk(0, 0), f12c = mk(0, 0), f22m = mk(0, 0);  // carries
  cplx qm[3] = {mk(0, 0), mk(0, 0), mk(0, 0)};

  for (int z = zb - 1; z < zend; ++z) {
    cp_async_wait<0>();
    __syncthreads();
    // planes z-1..z+1 resident; fetch z+2 into the free slot
    s3_load_plane(S, P, x, m, i0, j0, z + 2);
    cp_async_commit();

    // --- fluxes on the tile + halo at plane z -----------------------------
    for (int t = threadIdx.x; t < S3_FN; t += S3_THREADS) {
      const int fx = t % S3_FX, fy = t / S3_FX;
      const int lx = fx + 1, ly = fy + 1;
      const int xg = i0 - 1 + fx, yg = j0 - 1 + fy;
      S.d00[t] = s3_spread<0, 0>(S, P, z, lx, ly, 0, s3_vflags<0, 0>(g, xg, yg, z));
      S.d11[t] = s3_spread<1, 1>(S, P, z, lx, ly, 0, s3_vflags<1, 1>(g, xg, yg, z));
      S.f01[t] = s3_mu_edge<0, 1>(S, g, z, lx, ly, 0, xg, yg, z) *
                 s3_spread<0, 1>(S, P, z, lx, ly, 0, s3_vflags<0, 1>(g, xg, yg, z));
      S.f10[t] = s3_mu_edge<0, 1>(S, g, z, lx, ly, 0, xg, yg, z) *
                 s3_spread<1, 0>(S, P, z, lx, ly, 0, s3_vflags<1, 0>(g, xg, yg, z));
      S.f20[t] = s3_mu_edge<0, 2>(S, g, z, lx, ly, 0, xg, yg, z) *
                 s3_spread<2, 0>(S, P, z, lx, ly, 0, s3_vflags<2, 0>(g, xg, yg, z));
      S.f21[t] = s3_mu_edge<1, 2>(S, g, z, lx, ly, 0, xg, yg, z) *
                 s3_spread<2, 1>(S, P, z, lx, ly, 0, s3_vflags<2, 1>(g, xg, yg, z));
      S.q[0][t] = s3_massq<0>(S, P, z, lx, ly, 0, xg, yg, z);
      S.q[1][t] = s3_massq<1>(S, P, z, lx, ly, 0, xg, yg, z);
      S.q[2][t] = s3_massq<2>(S, P, z, lx, ly, 0, xg, yg, z);
    }
    // --- own-column z-neighbour quantities ---------------------------------
    const cplx f02p = s3_mu_edge<0, 2>(S, g, z, ulx, uly, 1, xi, yj, z + 1) *
                      s3_spread<0, 2>(S, P, z, ulx, uly, 1, s3_vflags<0, 2>(g, xi, yj, z + 1));
    const cplx f12p = s3_mu_edge<1, 2>(S, g, z, ulx, uly, 1, xi, yj, z + 1) *
                      s3_spread<1, 2>(S, P, z, ulx, uly, 1, s3_vflags<1, 2>(g, xi, yj, z + 1));
    const cplx d22 = s3_spread<2, 2>(S, P, z, ulx, uly, 0, s3_vflags<2, 2>(g, xi, yj, z));
    const Cell mc = S.m[s3_slot(z)][ulx + S3_UX * uly];
    const cplx f22 = mc.x * d22;  // zero-filled mu masks cells outside the box
    cplx qp[3];
    qp[0] = s3_massq<0>(S, P, z, ulx, uly, 1, xi, yj, z + 1);
    qp[1] = s3_massq<1>(S, P, z, ulx, uly, 1, xi, yj, z + 1);
    qp[2] = s3_massq<2>(S, P, z, ulx, uly, 1, xi, yj, z + 1);
    __syncthreads();

    cplx qc[3] = {S.q[0][fpos], S.q[1][fpos], S.q[2][fpos]};
    if (z >= zb) {
      const double ih = g.inv_h;
      const cplx pc = S.p[s3_slot(z)][ulx + S3_UX * uly];
      auto mass = [&](int k, int cnt) -> cplx {
        cplx v = P.beta * qc[k];
        if (P.beta == 1.0) return v;
        v += P.wn * S.q[k][fpos - 1];
        v += P.wn * S.q[k][fpos + 1];
        v += P.wn * S.q[k][fpos - S3_FX];
        v += P.wn * S.q[k][fpos + S3_FX];
        v += P.wn * qm[k];
        v += P.wn * qp[k];
        return v * P.inv_msum[cnt];
      };
      // u0 row (operator.hpp:389, :409)
      if (xi <= g.n[0] && yj < g.n[1] && z < g.n[2]) {
        const Cell ml = S.m[s3_slot(z)][(ulx - 1) + S3_UX * uly];
        cplx out = mk(0, 0);
        out += (ml.x * S.d00[fpos - 1] - mc.x * S.d00[fpos]) * ih;
        out += (S.f01[fpos] - S.f01[fpos + S3_FX]) * ih;
        out += (f02c - f02p) * ih;
        out -= mass(0, s3_mass_count<0>(g, xi, yj, z));
        out += (pc - S.p[s3_slot(z)][(ulx - 1) + S3_UX * uly]) * ih;
        const int64_t r = g.off[0] + xi + (int64_t)(g.n[0] + 1) * (yj + (int64_t)g.n[1] * z);
        y[r] = b ? b[r] - out : out;
      }
      // u1 row
      if (xi < g.n[0] && yj <= g.n[1] && z < g.n[2]) {
        const Cell mb = S.m[s3_slot(z)][ulx + S3_UX * (uly - 1)];
        cplx out = mk(0, 0);
        out += (S.f10[fpos] - S.f10[fpos + 1]) * ih;
        out += (mb.x * S.d11[fpos - S3_FX] - mc.x * S.d11[fpos]) * ih;
        out += (f12c - f12p) * ih;
        out -= mass(1, s3_mass_count<1>(g, xi, yj, z));
        out += (pc - S.p[s3_slot(z)][ulx + S3_UX * (uly - 1)]) * ih;
        const int64_t r = g.off[1] + xi + (int64_t)g.n[0] * (yj + (int64_t)(g.n[1] + 1) * z);
        y[r] = b ? b[r] - out : out;
      }
      // u2 row
      if (xi < g.n[0] && yj < g.n[1] && z <= g.n[2]) {
        cplx out = mk(0, 0);
        out += (S.f20[fpos] - S.f20[fpos + 1]) * ih;
        out += (S.f21[fpos] - S.f21[fpos + S3_FX]) * ih;
        out += (f22m - f22) * ih;
        out -= mass(2, s3_mass_count<2>(g, xi, yj, z));
        out += (pc - S.p[s3_slot(z - 1)][ulx + S3_UX * uly]) * ih;
        const int64_t r = g.off[2] + xi + (int64_t)g.n[0] * (yj + (int64_t)g.n[1] * z);
        y[r] = b ? b[r] - out : out;
      }
      // p row (operator.hpp:416)
      if (xi < g.n[0] && yj < g.n[1] && z < g.n[2]) {
        cplx out = mk(0, 0);
        out += S.d00[fpos];
        out += S.d11[fpos];
        out += d22;
        out += mc.w * pc;
        const int64_t r = g.off[3] + xi + (int64_t)g.n[0] * (yj + (int64_t)g.n[1] * z);
        y[r] = b ? b[r] - out : out;
      }
    }
    // carries
    f02c = f02p;
    f12c = f12p;
    f22m = f22;
    qm[0] = qc[0];
    qm[1] = qc[1];
    qm[2] = qc[2];
  }
  cp_async_wait<0>();
}

inline S3Params make_s3params(const Geo& g, const OpPar& P) {
  S3Params s;
  s.g = g;
  s.beta = P.beta;
  s.omega2 = P.omega2;
  s.alpha = P.alpha;
  const double w = (1.0 - P.beta) / 16.0;
  s.wt[0] = w * (double)(1 * 1);  // both transverse offsets nonzero
  s.wt[1] = w * (double)(2 * 1);  // one zero
  s.wt[2] = w * (double)(2 * 2);  // centre
  // wsum in the reference's accumulation order (operator.hpp:289-296)
  for (int f = 0; f < 16; ++f) {
    const bool lo1 = f & 1, hi1 = f & 2, lo2 = f & 4, hi2 = f & 8;
    double wsum = P.beta;
    for (int s1 = -1; s1 <= 1; ++s1)
      for (int s2 = -1; s2 <= 1; ++s2) {
        if ((s1 == -1 && !lo1) || (s1 == 1 && !hi1) || (s2 == -1 && !lo2) || (s2 == 1 && !hi2)) continue;
        wsum += w * (double)((s1 == 0 ? 2 : 1) * (s2 == 0 ? 2 : 1));
      }
    s.inv_wsum[f] = 1.0 / wsum;
  }
  s.wn = (1.0 - P.beta) / 6.0;
  for (int c = 0; c <= 6; ++c) {
    double wsum = P.beta;
    for (int q = 0; q < c; ++q) wsum += s.wn;
    s.inv_msum[c] = 1.0 / wsum;
  }
  return s;
}

inline bool stencil3d_supported(const Geo& g) { return g.nd == 3 && g.n[0] >= 2 && g.n[1] >= 2; }

inline void launch_stencil3d(const Geo& g, const OpPar& P, const Cell* m, const cplx* x, const cplx* b,
                             cplx* y, cudaStream_t s) {
  static bool attr = false;
  const size_t smem = sizeof(S3Smem);
  if (!attr) {
    cudaFuncSetAttribute(k_stencil3d, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  dim3 grid((g.n[0] + 1 + S3_TX - 1) / S3_TX, (g.n[1] + 1 + S3_TY - 1) / S3_TY,
            (g.n[2] + 1 + S3_ZCHUNK - 1) / S3_ZCHUNK);
  k_stencil3d<<<grid, S3_THREADS, smem, s>>>(make_s3params(g, P), m, x, b, y);
}

}  // namespace ehmg
