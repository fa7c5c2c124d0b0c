// ehmg_slab.cuh -- z-slab decomposed multigrid (north_star subsystem (6)).
//
// Fine levels are split into z-slabs: slab s owns cell planes [Z0, Z1) (and
// u2 faces [Z0, Z1), plus face n2 on the last slab) and stores the window
// [Z0-3, Z1+2) (ghost planes, clipped to the grid; one extra plane below
// because the u2 mass row of the first ghost face averages rho/gamma one
// cell further down). Kernels run on the
// window with global boundary semantics (Geo::zoff/gn2); values near the
// window edge are scratch. Every operation that changes a field is followed
// by a ghost exchange (owned planes -> neighbour ghosts), which keeps the
// owned region bit-identical to the undecomposed cycle:
//   * a red-black colour updates all window cells; owned DOFs only depend on
//     residuals of owned cells and of the first ghost cell layer below, which
//     only depend on data inside the window;
//   * restriction reads the fine residual one plane beyond the owned range;
//   * prolongation reads coarse ghosts refreshed by the coarse level's last
//     exchange.
// Levels whose z extent is <= agg_n2 are agglomerated: the restricted
// residual is gathered into one full array and every rank runs the remaining
// levels (incl. the exact coarsest solve) redundantly, then prolongs into its
// own window -- no scatter is needed on the way up.
//
// Transport: slabs of one process exchange with device-to-device copies
// (the in-process P-slab mode used by the tests on one GPU); across
// processes the same plane ranges go over NCCL/NVLink (ExchangeFn hook).
#pragma once

struct SlabPlan {
  int nslabs = 1, La = 1, nl = 2;  // distributed levels [0, La), replicated [La, nl)
  std::vector<int> z0;             // level-0 slab boundaries, size nslabs+1
};

constexpr int kSlabGhostLo = 3, kSlabGhostHi = 2;

// Partition n2 planes into nslabs slabs whose boundaries are multiples of
// 2^La, with at least 4 owned planes on every distributed level; levels with
// z extent <= agg_n2 (and always the coarsest) are replicated.
static SlabPlan make_slab_plan(int n2, int nl, int nslabs, int agg_n2) {
  if (nslabs < 1) throw Err(EHMG_EINVAL, "slab: need >= 1 slab");
  SlabPlan p;
  p.nslabs = nslabs;
  p.nl = nl;
  int La = 1;
  while (La < nl - 1 && (n2 >> La) > agg_n2) ++La;
  for (; La >= 1; --La) {
    const int unit = 1 << La;
    if (n2 % unit != 0) continue;
    const int units = n2 / unit;
    if (units < nslabs) continue;
    std::vector<int> z(nslabs + 1);
    for (int s = 0; s <= nslabs; ++s) z[s] = (int)((int64_t)units * s / nslabs) * unit;
    bool ok = true;
    for (int s = 0; s < nslabs; ++s)
      if (((z[s + 1] - z[s]) >> (La - 1)) < 4) ok = false;
    if (!ok) continue;
    p.La = La;
    p.z0 = z;
    return p;
  }
  throw Err(EHMG_EINVAL, "slab: grid too thin for the requested number of slabs");
}

struct SlabLevel {
  Geo g;           // window geometry (local storage, global semantics)
  int Z0, Z1;      // owned cell planes (global)
  DevMedia media;  // window media
  Smoother sm;
  DBuf<cplx> r, bc, ec;
};

struct ehmg_slab_mg_s {
  int dev = 0;
  cudaStream_t s = nullptr;
  ehmg_mg_options opt;
  OpPar P;
  SlabPlan plan;
  std::vector<Geo> G;                                        // global geometry per level
  std::vector<std::vector<std::unique_ptr<SlabLevel>>> L;   // [level < La][slab]
  std::unique_ptr<ehmg_mg_s> rep;                            // replicated levels [La, nl)
  DBuf<cplx> brep, erep;                                     // level-La full rhs / correction
  std::vector<std::unique_ptr<DBuf<cplx>>> bw, xw;          // level-0 windows
  std::vector<std::unique_ptr<DBuf<cplx>>> ctmp;            // restriction staging (level La windows)
  int64_t exchanged_bytes = 0;

  ~ehmg_slab_mg_s() {
    L.clear();
    rep.reset();
    if (s) cudaStreamDestroy(s);
  }

  int P_() const { return plan.nslabs; }

  // bytes per z-plane of component k (faces or cells) on geometry g
  static int64_t plane(const Geo& g, int k) {
    return (int64_t)(g.n[0] + (k == 0)) * (g.n[1] + (k == 1));
  }
  // copy global planes [a, b) of component k between two window/full arrays
  void copy_planes(cplx* dst, const Geo& dg, const cplx* src, const Geo& sg, int k, int a, int b) {
    if (b <= a) return;
    const int64_t ps = plane(dg, k);
    CK(cudaMemcpyAsync(dst + dg.off[k] + (a - dg.zoff) * ps, src + sg.off[k] + (a - sg.zoff) * ps,
                       sizeof(cplx) * ps * (b - a), cudaMemcpyDeviceToDevice, s));
    exchanged_bytes += (int64_t)sizeof(cplx) * ps * (b - a);
  }

  // owned planes -> neighbour ghosts, every slab boundary, all 4 components
  void exchange(int l, const std::vector<cplx*>& V) {
    const int64_t before = exchanged_bytes;
    for (int q = 0; q + 1 < P_(); ++q) {
      SlabLevel& lo = *L[l][q];
      SlabLevel& hi = *L[l][q + 1];
      const int zb = lo.Z1;  // == hi.Z0
      const int lo_top = lo.g.zoff + lo.g.n[2], hi_bot = hi.g.zoff;
      for (int k = 0; k < 4; ++k) {
        const bool face = (k == 2);
        // up: lo's owned top planes -> hi's ghosts below (cells/faces [hi_bot, zb))
        copy_planes(V[q + 1], hi.g, V[q], lo.g, k, hi_bot, zb);
        // down: hi's owned bottom planes -> lo's ghosts above (cells [zb, lo_top), faces [zb, lo_top])
        copy_planes(V[q], lo.g, V[q + 1], hi.g, k, zb, face ? lo_top + 1 : lo_top);
      }
    }
    (void)before;
  }

  void sweep_all(int l, const std::vector<const cplx*>& B, const std::vector<cplx*>& X) {
    for (int color = 0; color < 2; ++color) {
      for (int q = 0; q < P_(); ++q) {
        SlabLevel& sl = *L[l][q];
        sl.sm.colour_phase(sl.g, P, sl.media.ref(), B[q], X[q], opt.damping, color, s);
      }
      exchange(l, X);
    }
  }

  // multigrid.hpp:217 cycle_at on the distributed levels
  void cycle(int l, const std::vector<const cplx*>& B, const std::vector<cplx*>& X) {
    const int La = plan.La, nl = plan.nl;
    for (int q = 0; q < opt.nu1; ++q) sweep_all(l, B, X);
    for (int q = 0; q < P_(); ++q) {
      SlabLevel& sl = *L[l][q];
      launch_residual(sl.g, P, sl.media.ref(), X[q], B[q], sl.r.p, s);
    }
    const bool next_coarsest = (l + 2 == nl);
    const int repeat = (opt.cycle == 2 && !next_coarsest) ? 2 : 1;
    if (l + 1 < La) {
      std::vector<const cplx*> BC(P_());
      std::vector<cplx*> BCw(P_()), EC(P_());
      for (int q = 0; q < P_(); ++q) {
        SlabLevel& f = *L[l][q];
        SlabLevel& c = *L[l + 1][q];
        launch_transfer(f.g, c.g, true, f.r.p, c.bc.p, false, s);
        CK(cudaMemsetAsync(c.ec.p, 0, sizeof(cplx) * c.g.ndofs, s));
        BC[q] = c.bc.p;
        BCw[q] = c.bc.p;
        EC[q] = c.ec.p;
      }
      exchange(l + 1, BCw);
      for (int r = 0; r < repeat; ++r) cycle(l + 1, BC, EC);
      for (int q = 0; q < P_(); ++q)
        launch_transfer(L[l][q]->g, L[l + 1][q]->g, false, L[l + 1][q]->ec.p, X[q], true, s);
    } else {
      // agglomerate: restrict each slab's owned coarse planes into the full array
      const Geo& gc = G[La];
      for (int q = 0; q < P_(); ++q) {
        SlabLevel& f = *L[l][q];
        const int c0 = f.Z0 / 2, c1 = f.Z1 / 2;
        const Geo cw = make_window(gc, c0, c1);
        launch_transfer(f.g, cw, true, f.r.p, ctmp[q]->p, false, s);
        const bool last = (q + 1 == P_());
        for (int k = 0; k < 4; ++k)
          copy_planes(brep.p, gc, ctmp[q]->p, cw, k, c0, (k == 2 && last) ? c1 + 1 : c1);
      }
      CK(cudaMemsetAsync(erep.p, 0, sizeof(cplx) * gc.ndofs, s));
      CK(cudaStreamSynchronize(s));
      for (int r = 0; r < repeat; ++r) rep->cycle_at(0, brep.p, erep.p);
      CK(cudaStreamSynchronize(rep->s));
      for (int q = 0; q < P_(); ++q) launch_transfer(L[l][q]->g, gc, false, erep.p, X[q], true, s);
    }
    for (int q = 0; q < opt.nu2; ++q) sweep_all(l, B, X);
  }

  // Full-array boundary of the in-process mode: scatter r into the level-0
  // windows (ghosts included), cycle, gather the owned planes into z.
  void precondition(const cplx* r, cplx* z) {
    const Geo& g0 = G[0];
    std::vector<const cplx*> B(P_());
    std::vector<cplx*> X(P_());
    for (int q = 0; q < P_(); ++q) {
      const Geo& w = L[0][q]->g;
      for (int k = 0; k < 4; ++k)
        copy_planes(bw[q]->p, w, r, g0, k, w.zoff, w.zoff + w.n[2] + (k == 2));
      CK(cudaMemsetAsync(xw[q]->p, 0, sizeof(cplx) * w.ndofs, s));
      B[q] = bw[q]->p;
      X[q] = xw[q]->p;
    }
    cycle(0, B, X);
    for (int q = 0; q < P_(); ++q) {
      SlabLevel& sl = *L[0][q];
      const bool last = (q + 1 == P_());
      for (int k = 0; k < 4; ++k)
        copy_planes(z, g0, xw[q]->p, sl.g, k, sl.Z0, (k == 2 && last) ? sl.Z1 + 1 : sl.Z1);
    }
    CK(cudaStreamSynchronize(s));
  }
};

static std::unique_ptr<ehmg_slab_mg_s> build_slab_mg(const Geo& g0, const double* const* host, const OpPar& P,
                                                     const ehmg_mg_options& opt, int nslabs, int agg_n2) {
  if (g0.nd != 3) throw Err(EHMG_EINVAL, "slab: z-slab decomposition is 3D only");
  if (opt.cycle == 3) throw Err(EHMG_EINVAL, "slab: K-cycles need a distributed inner Krylov (not supported)");
  if (opt.sweep != 1) throw Err(EHMG_EINVAL, "slab: only red-black sweeps decompose");
  auto sm = std::make_unique<ehmg_slab_mg_s>();
  sm->opt = opt;
  sm->P = P;
  sm->plan = make_slab_plan(g0.n[2], opt.n_levels, nslabs, agg_n2);
  const int La = sm->plan.La, nl = opt.n_levels;
  CK(cudaGetDevice(&sm->dev));
  CK(cudaStreamCreateWithFlags(&sm->s, cudaStreamNonBlocking));
  cudaStream_t s = sm->s;
  if (!stencil3d_supported(g0)) throw Err(EHMG_EINVAL, "slab: needs an even x extent (TMA stencil)");
  // global media per level [0, La]
  std::vector<std::unique_ptr<DevMedia>> gm;
  for (int l = 0; l <= La; ++l) {
    sm->G.push_back(l == 0 ? g0 : coarse_geo(sm->G[l - 1]));
    gm.emplace_back(new DevMedia());
    if (l == 0) gm[0]->upload(g0.ncells, host, s);
    else gm[l - 1]->coarsen_into(sm->G[l - 1], *gm[l], sm->G[l], s);
  }
  sm->L.resize(La);
  for (int l = 0; l < La; ++l) {
    for (int q = 0; q < nslabs; ++q) {
      auto sl = std::make_unique<SlabLevel>();
      sl->Z0 = sm->plan.z0[q] >> l;
      sl->Z1 = sm->plan.z0[q + 1] >> l;
      const int w0 = std::max(0, sl->Z0 - kSlabGhostLo), w1 = std::min(sm->G[l].n[2], sl->Z1 + kSlabGhostHi);
      sl->g = make_window(sm->G[l], w0, w1);
      sl->media.window_of(*gm[l], sm->G[l], w0, w1, s);
      sl->sm.build(sm->G[l], P, gm[l]->packed.p, opt.vanka_mode == 0 ? 1 : 0, s, w0, w1);
      sl->r.alloc(sl->g.ndofs);
      if (l > 0) {
        sl->bc.alloc(sl->g.ndofs);
        sl->ec.alloc(sl->g.ndofs);
      }
      sm->L[l].push_back(std::move(sl));
    }
  }
  for (int q = 0; q < nslabs; ++q) {
    sm->bw.emplace_back(new DBuf<cplx>(sm->L[0][q]->g.ndofs));
    sm->xw.emplace_back(new DBuf<cplx>(sm->L[0][q]->g.ndofs));
    const SlabLevel& f = *sm->L[La - 1][q];
    sm->ctmp.emplace_back(new DBuf<cplx>(make_window(sm->G[La], f.Z0 / 2, f.Z1 / 2).ndofs));
  }
  CK(cudaStreamSynchronize(s));
  sm->rep = build_mg(sm->G[La], nullptr, gm[La].get(), P, opt, nl - La);
  sm->brep.alloc(sm->G[La].ndofs);
  sm->erep.alloc(sm->G[La].ndofs);
  CK(cudaStreamSynchronize(s));
  return sm;
}
