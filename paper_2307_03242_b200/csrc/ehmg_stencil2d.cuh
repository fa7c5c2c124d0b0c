// ehmg_stencil2d.cuh -- 2D operator / residual kernel.
//
// y = H x or r = b - H x for the 2D staggered mixed operator
// (operator.hpp:267-421 with Dim = 2), all three rows (u0, u1, p) per
// position. u0 / u1 / p and the packed cell media of a block plus halo are
// staged in shared memory with coalesced loads (zero outside the arrays, the
// reference's ghosts); fluxes and face mass products are evaluated once per
// position and shared through shared memory (the generic rows of
// ehmg_core.cuh read global memory per term, which left the 2D configs
// latency-bound). V = cplx (complex128) or cplxf (complex64 storage;
// arithmetic in double).
#pragma once

#include <mutex>

#include "ehmg_core.cuh"

namespace ehmg {


struct S2Params {
  double beta, omega2, alpha, w;  // w = (1 - beta) / 4
  double inv_wsum[4];             // 1/wsum by transverse validity (lo | hi << 1), operator.hpp:276
  double wn, inv_msum[5];         // mass neighbour weight (1 - beta) / 4, 1/(beta + k wn)
};

inline S2Params make_s2params(const OpPar& P) {
  S2Params s;
  s.beta = P.beta;
  s.omega2 = P.omega2;
  s.alpha = P.alpha;
  s.w = (1.0 - P.beta) / 4.0;
  for (int f = 0; f < 4; ++f) {
    double wsum = P.beta;
    for (int st = -1; st <= 1; ++st) {
      if ((st == -1 && !(f & 1)) || (st == 1 && !(f & 2))) continue;
      wsum += s.w * (double)(st == 0 ? 2 : 1);
    }
    s.inv_wsum[f] = P.beta != 1.0 ? 1.0 / wsum : 1.0;
  }
  s.wn = (1.0 - P.beta) / 4.0;
  for (int c = 0; c <= 4; ++c) {
    double wsum = P.beta;
    for (int q = 0; q < c; ++q) wsum += s.wn;
    s.inv_msum[c] = P.beta != 1.0 ? 1.0 / wsum : 1.0;
  }
  return s;
}

// The 32x16 thread grid is the flux window of a 30x14 output block. Each thread evaluates the fluxes
// of its own cell and edge, and the mass products of its own faces, once;
// neighbouring rows read them from shared memory instead of re-evaluating
// them (the term-by-term kernel above evaluated every flux twice and every
// face mass five times). Same per-term operation order as the reference;
// averages divide by 1, 2 or 4 as exact reciprocal multiplies.
constexpr int S2B_FX = 32, S2B_FY = 16, S2B_T = S2B_FX * S2B_FY;
constexpr int S2B_TX = S2B_FX - 2, S2B_TY = S2B_FY - 2;
constexpr int S2B_WX = S2B_FX + 2, S2B_WY = S2B_FY + 2, S2B_WN = S2B_WX * S2B_WY;  // origin (i0-2, j0-2)

__device__ __forceinline__ double s2_inv(int c) { return c == 4 ? 0.25 : (c == 2 ? 0.5 : 1.0); }

struct S2BSmem {
  cplx U0[S2B_WN], U1[S2B_WN], Pp[S2B_WN];
  Cell M[S2B_WN];
  cplx SF0[S2B_T], SF1[S2B_T], SG01[S2B_T], SG10[S2B_T], SQ0[S2B_T], SQ1[S2B_T];
};

template <class V>
__global__ void __launch_bounds__(S2B_T) k_stencil2d_fs(Geo g, S2Params P, const Cell* __restrict__ m,
                                                        const V* __restrict__ x, const V* __restrict__ b,
                                                        V* __restrict__ y) {
  extern __shared__ __align__(16) unsigned char s2b_raw[];
  S2BSmem& SM = *reinterpret_cast<S2BSmem*>(s2b_raw);
  cplx* U0 = SM.U0;
  cplx* U1 = SM.U1;
  cplx* Pp = SM.Pp;
  Cell* M = SM.M;
  cplx* SF0 = SM.SF0;
  cplx* SF1 = SM.SF1;
  cplx* SG01 = SM.SG01;
  cplx* SG10 = SM.SG10;
  cplx* SQ0 = SM.SQ0;
  cplx* SQ1 = SM.SQ1;
  const int n0 = g.n[0], n1 = g.n[1];
  const int i0 = blockIdx.x * S2B_TX, j0 = blockIdx.y * S2B_TY;
  const int t = threadIdx.x + S2B_FX * threadIdx.y;
  const V* X0 = x + g.off[0];
  const V* X1 = x + g.off[1];
  const V* XP = x + g.off[2];
  for (int e = t; e < S2B_WN; e += S2B_T) {
    const int wy = e / S2B_WX, wx = e - wy * S2B_WX;
    const int xx = i0 - 2 + wx, yy = j0 - 2 + wy;
    const bool cy = yy >= 0 && yy < n1, cx = xx >= 0 && xx < n0;
    U0[e] = (xx >= 0 && xx <= n0 && cy) ? wide(X0[xx + (int64_t)(n0 + 1) * yy]) : mk(0, 0);
    U1[e] = (cx && yy >= 0 && yy <= n1) ? wide(X1[xx + (int64_t)n0 * yy]) : mk(0, 0);
    const bool cok = cx && cy;
    Pp[e] = cok ? wide(XP[xx + (int64_t)n0 * yy]) : mk(0, 0);
    M[e] = cok ? m[xx + (int64_t)n0 * yy] : make_double4(0, 0, 0, 0);
  }
  __syncthreads();

  const int px = i0 - 1 + threadIdx.x, py = j0 - 1 + threadIdx.y;  // this thread's position
  const int W = S2B_WX;
  const int c0 = (threadIdx.x + 1) + W * (threadIdx.y + 1);  // window index of (px, py)
  const double beta = P.beta, w = P.w, ih = g.inv_h, wn = P.wn;
  auto cell_ok = [&](int cx, int cy) { return cx >= 0 && cx < n0 && cy >= 0 && cy < n1; };
  // operator.hpp:267 dspread_cell / :306 dspread_edge (as k_stencil2d)
  auto dsc0 = [&](int cy, int ci) {
    cplx v = beta * (U0[ci + 1] - U0[ci]);
    if (beta != 1.0) {
      if (cy - 1 >= 0) v += w * (U0[ci + 1 - W] - U0[ci - W]);
      v += (2.0 * w) * (U0[ci + 1] - U0[ci]);
      if (cy + 1 < n1) v += w * (U0[ci + 1 + W] - U0[ci + W]);
      v = v * P.inv_wsum[(cy - 1 >= 0) | ((cy + 1 < n1) << 1)];
    }
    return v * ih;
  };
  auto dsc1 = [&](int cx, int ci) {
    cplx v = beta * (U1[ci + W] - U1[ci]);
    if (beta != 1.0) {
      if (cx - 1 >= 0) v += w * (U1[ci - 1 + W] - U1[ci - 1]);
      v += (2.0 * w) * (U1[ci + W] - U1[ci]);
      if (cx + 1 < n0) v += w * (U1[ci + 1 + W] - U1[ci + 1]);
      v = v * P.inv_wsum[(cx - 1 >= 0) | ((cx + 1 < n0) << 1)];
    }
    return v * ih;
  };
  auto dse01 = [&](int ex, int ei) {
    cplx v = beta * (U0[ei] - U0[ei - W]);
    if (beta != 1.0) {
      if (ex - 1 >= 0) v += w * (U0[ei - 1] - U0[ei - 1 - W]);
      v += (2.0 * w) * (U0[ei] - U0[ei - W]);
      if (ex + 1 < n0 + 1) v += w * (U0[ei + 1] - U0[ei + 1 - W]);
      v = v * P.inv_wsum[(ex - 1 >= 0) | ((ex + 1 < n0 + 1) << 1)];
    }
    return v * ih;
  };
  auto dse10 = [&](int ey, int ei) {
    cplx v = beta * (U1[ei] - U1[ei - 1]);
    if (beta != 1.0) {
      if (ey - 1 >= 0) v += w * (U1[ei - W] - U1[ei - 1 - W]);
      v += (2.0 * w) * (U1[ei] - U1[ei - 1]);
      if (ey + 1 < n1 + 1) v += w * (U1[ei + W] - U1[ei - 1 + W]);
      v = v * P.inv_wsum[(ey - 1 >= 0) | ((ey + 1 < n1 + 1) << 1)];
    }
    return v * ih;
  };
  // operator.hpp:108 mu on the (0,1) edge (first axis outer; yfirst: u1 rows)
  auto mu_e = [&](int ex, int ey, int ei, bool yfirst) {
    double s = 0;
    int cnt = 0;
    if (cell_ok(ex - 1, ey - 1)) s += M[ei - 1 - W].x, ++cnt;
    if (!yfirst) {
      if (cell_ok(ex - 1, ey)) s += M[ei - 1].x, ++cnt;
      if (cell_ok(ex, ey - 1)) s += M[ei - W].x, ++cnt;
    } else {
      if (cell_ok(ex, ey - 1)) s += M[ei - W].x, ++cnt;
      if (cell_ok(ex - 1, ey)) s += M[ei - 1].x, ++cnt;
    }
    if (cell_ok(ex, ey)) s += M[ei].x, ++cnt;
    return s * s2_inv(cnt);
  };
  // operator.hpp:132 face mass diagonal of a k-face
  auto mdiag = [&](int k, int fx, int fy, int fi) {
    const int st = k == 0 ? 1 : W;
    const int bx = fx - (k == 0), by = fy - (k == 1);
    double sr = 0, sg = 0;
    int cnt = 0;
    if (cell_ok(bx, by)) sr += M[fi - st].y, sg += M[fi - st].z, ++cnt;
    if (cell_ok(px, py)) sr += M[fi].y, sg += M[fi].z, ++cnt;
    const double ic = s2_inv(cnt);
    const double rho_f = sr * ic, gam_f = sg * ic + P.alpha;
    return mk(P.omega2 * rho_f, -P.omega2 * gam_f * rho_f);
  };

  // ---- phase 1: this position's cell fluxes, edge fluxes and face mass products
  const bool cok = cell_ok(px, py);
  const cplx d0 = cok ? dsc0(py, c0) : mk(0, 0);
  const cplx d1 = cok ? dsc1(px, c0) : mk(0, 0);
  const cplx f0 = cok ? M[c0].x * d0 : mk(0, 0);
  const cplx f1 = cok ? M[c0].x * d1 : mk(0, 0);
  const bool eok = px >= 0 && px <= n0 && py >= 0 && py <= n1;
  const cplx g01 = (eok && py < n1 + 1) ? mu_e(px, py, c0, false) * dse01(px, c0) : mk(0, 0);
  const cplx g10 = (eok && px < n0 + 1) ? mu_e(px, py, c0, true) * dse10(py, c0) : mk(0, 0);
  const bool q0ok = px >= 0 && px <= n0 && py >= 0 && py < n1;
  const bool q1ok = px >= 0 && px < n0 && py >= 0 && py <= n1;
  const cplx q0 = q0ok ? mdiag(0, px, py, c0) * U0[c0] : mk(0, 0);
  const cplx q1 = q1ok ? mdiag(1, px, py, c0) * U1[c0] : mk(0, 0);
  SF0[t] = f0;
  SF1[t] = f1;
  SG01[t] = g01;
  SG10[t] = g10;
  SQ0[t] = q0;
  SQ1[t] = q1;
  __syncthreads();

  // ---- phase 2: rows of the interior positions
  const bool inner = threadIdx.x >= 1 && threadIdx.x <= S2B_TX && threadIdx.y >= 1 && threadIdx.y <= S2B_TY;
  if (!inner) return;
  const int xo = px, yo = py;
  // operator.hpp:359 mass_eval from the face products (neighbours outside
  // the face box are skipped, as the reference's loop does)
  auto mass = [&](const cplx* Q, cplx qc, int d0_, int d1_) {
    cplx v = beta * qc;
    if (beta == 1.0) return v;
    int cnt = 0;
    if (xo - 1 >= 0) v += wn * Q[t - 1], ++cnt;
    if (xo + 1 < d0_) v += wn * Q[t + 1], ++cnt;
    if (yo - 1 >= 0) v += wn * Q[t - S2B_FX], ++cnt;
    if (yo + 1 < d1_) v += wn * Q[t + S2B_FX], ++cnt;
    return v * P.inv_msum[cnt];
  };
  if (xo <= n0 && yo < n1) {  // u0 row (operator.hpp:389 / :409)
    cplx out = mk(0, 0);
    out += (SF0[t - 1] - f0) * ih;
    out += (g01 - SG01[t + S2B_FX]) * ih;
    out -= mass(SQ0, q0, n0 + 1, n1);
    out += (Pp[c0] - Pp[c0 - 1]) * ih;
    const int64_t o = g.off[0] + xo + (int64_t)(n0 + 1) * yo;
    y[o] = narrow<V>(b ? wide(b[o]) - out : out);
  }
  if (xo < n0 && yo <= n1) {  // u1 row
    cplx out = mk(0, 0);
    out += (g10 - SG10[t + 1]) * ih;
    out += (SF1[t - S2B_FX] - f1) * ih;
    out -= mass(SQ1, q1, n0, n1 + 1);
    out += (Pp[c0] - Pp[c0 - W]) * ih;
    const int64_t o = g.off[1] + xo + (int64_t)n0 * yo;
    y[o] = narrow<V>(b ? wide(b[o]) - out : out);
  }
  if (xo < n0 && yo < n1) {  // p row (operator.hpp:416)
    cplx out = mk(0, 0);
    out += d0;
    out += d1;
    out += M[c0].w * Pp[c0];
    const int64_t o = g.off[2] + xo + (int64_t)n0 * yo;
    y[o] = narrow<V>(b ? wide(b[o]) - out : out);
  }
}

template <class V>
inline void launch_stencil2d(const Geo& g, const OpPar& P, const Cell* m, const V* x, const V* b, V* y,
                             cudaStream_t s) {
  {  // the dynamic shared-memory opt-in is a per-device function attribute
    static std::mutex mu;
    static bool done[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    std::lock_guard<std::mutex> lock(mu);
    if (!done[dev]) {
      cudaFuncSetAttribute(k_stencil2d_fs<cplx>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(S2BSmem));
      cudaFuncSetAttribute(k_stencil2d_fs<cplxf>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)sizeof(S2BSmem));
      done[dev] = true;
    }
  }
  const dim3 blk(S2B_FX, S2B_FY);
  const dim3 grd((g.n[0] + 1 + S2B_TX - 1) / S2B_TX, (g.n[1] + 1 + S2B_TY - 1) / S2B_TY);
  k_stencil2d_fs<V><<<grd, blk, sizeof(S2BSmem), s>>>(g, make_s2params(P), m, x, b, y);
}

}  // namespace ehmg
