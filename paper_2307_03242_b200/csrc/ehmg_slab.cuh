// ehmg_slab.cuh -- z-slab decomposed multigrid and FGMRES (north_star
// subsystem (6)).
//
// Fine levels are split into z-slabs: slab q owns cell planes [Z0, Z1) (and
// u2 faces [Z0, Z1), plus face n2 on the last slab) and stores the window
// [Z0-3, Z1+2) clipped to the grid (one extra ghost plane below because the
// u2 mass row of the first ghost face averages rho/gamma one cell further
// down). Kernels run on the window with global boundary semantics
// (Geo::zoff/gn2); values near the window edge are scratch. Every operation
// that changes a field is followed by a ghost exchange, which keeps the owned
// region identical to the undecomposed computation:
//   * a red-black colour updates all window cells; owned DOFs only depend on
//     residuals of owned cells and of the first ghost cell layer below, which
//     only depend on data inside the window;
//   * restriction reads the fine residual one plane beyond the owned range;
//   * prolongation reads coarse ghosts refreshed by the coarse level's last
//     exchange.
// Levels whose z extent is <= agg_n2 are agglomerated: every slab pushes its
// restricted owned planes into each rank's full coarse array and every rank
// runs the remaining levels (incl. the exact coarsest solve) redundantly,
// then prolongs into its own window.
//
// Exchange = push owned boundary planes into the neighbour's inbox (device
// copy; a peer pointer over NVLink when the neighbour is another process),
// barrier, pull the inbox into the ghost planes. One code path serves the
// in-process P-slab mode (all slabs in one process on one GPU -- the GPU
// tests) and the one-slab-per-process mode (NodeComm + CUDA IPC).
#pragma once

#include <cstdlib>
#include <cstring>

#include "ehmg_comm.cuh"

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

// planes of component k per z step on geometry g
static inline int64_t slab_plane(const Geo& g, int k) { return (int64_t)(g.n[0] + (k == 0)) * (g.n[1] + (k == 1)); }

struct SlabGeo {
  Geo g;       // window geometry (local storage, global semantics)
  int Z0, Z1;  // owned cell planes (global)
  int W0() const { return g.zoff; }
  int W1() const { return g.zoff + g.n[2]; }
  // ghost planes [a, b) of component k below / above the owned range
  void ghost(int k, bool above, int& a, int& b) const {
    if (!above) {
      a = W0();
      b = Z0;
    } else {
      a = Z1;
      b = W1() + (k == 2 ? 1 : 0);
    }
  }
  // inbox layout: component blocks of the ghost planes, below or above
  int64_t inbox_off(int k, bool above) const {
    int64_t o = 0;
    for (int c = 0; c < k; ++c) {
      int a, b;
      ghost(c, above, a, b);
      o += slab_plane(g, c) * std::max(0, b - a);
    }
    return o;
  }
  int64_t inbox_size(bool above) const { return inbox_off(4, above); }
};

struct SlabLevel {
  SlabGeo sg;
  bool local = false;
  DevMedia media;  // window media (local slabs)
  Smoother sm;
  DBuf<cplx> r, bc, ec, in_lo, in_hi, ctmp;
  cplx* peer_lo = nullptr;  // inbox pointers (own or IPC-mapped)
  cplx* peer_hi = nullptr;
  // complex64 hierarchy (precision 1, experiments.hpp:241)
  DBuf<cplxf> rf, bcf, ecf, in_lof, in_hif, ctmpf;
  cplxf* peer_lof = nullptr;
  cplxf* peer_hif = nullptr;
};
// slab-level vectors by element type
template <class V> struct SB;
template <> struct SB<cplx> {
  static cplx* r(SlabLevel& L) { return L.r.p; }
  static cplx* bc(SlabLevel& L) { return L.bc.p; }
  static cplx* ec(SlabLevel& L) { return L.ec.p; }
  static cplx* ctmp(SlabLevel& L) { return L.ctmp.p; }
  static cplx* in_lo(SlabLevel& L) { return L.in_lo.p; }
  static cplx* in_hi(SlabLevel& L) { return L.in_hi.p; }
  static cplx* peer_lo(const SlabLevel& L) { return L.peer_lo; }
  static cplx* peer_hi(const SlabLevel& L) { return L.peer_hi; }
};
template <> struct SB<cplxf> {
  static cplxf* r(SlabLevel& L) { return L.rf.p; }
  static cplxf* bc(SlabLevel& L) { return L.bcf.p; }
  static cplxf* ec(SlabLevel& L) { return L.ecf.p; }
  static cplxf* ctmp(SlabLevel& L) { return L.ctmpf.p; }
  static cplxf* in_lo(SlabLevel& L) { return L.in_lof.p; }
  static cplxf* in_hi(SlabLevel& L) { return L.in_hif.p; }
  static cplxf* peer_lo(const SlabLevel& L) { return L.peer_lof; }
  static cplxf* peer_hi(const SlabLevel& L) { return L.peer_hif; }
};

struct ehmg_slab_mg_s {
  int dev = 0;
  cudaStream_t s = nullptr;
  ehmg_mg_options opt;
  OpPar P;
  SlabPlan plan;
  int q_lo = 0, q_hi = 0;   // local slabs [q_lo, q_hi)
  NodeComm* comm = nullptr;  // one-slab-per-process mode
  std::vector<Geo> G;        // global geometry per level
  std::vector<std::vector<std::unique_ptr<SlabLevel>>> L;  // [level < La][slab]
  std::unique_ptr<ehmg_mg_s> rep;                           // replicated levels [La, nl)
  DBuf<cplx> brep, erep;                                    // level-La full rhs / correction (this rank)
  std::vector<cplx*> brep_of;                               // every rank's brep (own or IPC-mapped)
  int prec = 0;                                             // 1: complex64 hierarchy
  DBuf<cplxf> brepf, erepf;
  std::vector<cplxf*> brepf_of;
  std::vector<std::unique_ptr<DBuf<cplxf>>> bwf, xwf;      // complex64 level-0 windows
  std::vector<void*> cx_of;  // every rank's coarsest-level solution buffer (row-partitioned solve)
  std::vector<std::unique_ptr<Fgmres>> kin;  // K-cycle inner Krylov per distributed level
  std::vector<void*> mapped;                                // IPC mappings to close
  std::vector<std::unique_ptr<DBuf<cplx>>> bw, xw;         // level-0 windows of local slabs
  int64_t exchanged_bytes = 0;
  const std::vector<cplx*>& rep_of(cplx*) const { return brep_of; }
  const std::vector<cplxf*>& rep_of(cplxf*) const { return brepf_of; }
  cplx* rep_b(cplx*) { return brep.p; }
  cplxf* rep_b(cplxf*) { return brepf.p; }
  cplx* rep_e(cplx*) { return erep.p; }
  cplxf* rep_e(cplxf*) { return erepf.p; }

  // Overlap of the smoothing ghost exchanges with the stencil rows that do not
  // read ghost planes: pushes/pulls run on sx, the interior rows on s.
  cudaStream_t sx = nullptr;
  cudaEvent_t ev_upd = nullptr, ev_x = nullptr;
  // One slab per process: halo exchanges ordered GPU-side through CUDA IPC
  // events (recorded after this rank's pushes, waited on by the neighbours'
  // copy streams) instead of a stream drain + host barrier per exchange.
  // kXEv slots in rotation: a rank re-records slot e % kXEv only after its
  // neighbours published exchange e + kXEv - 1, i.e. after they enqueued
  // their waits for e.
  static constexpr int kXEv = 4;
  bool ev_exchange = false;
  cudaEvent_t xev[kXEv] = {}, xev_lo[kXEv] = {}, xev_hi[kXEv] = {};
  long long xseq = 0;
  std::vector<char> pend;  // per level: the smoothed iterate's ghosts are stale
  std::vector<int> xpar;   // per level: inbox half of the next exchange

  ~ehmg_slab_mg_s() {
    if (sx) cudaStreamSynchronize(sx);
    for (int i = 0; i < kXEv; ++i) {
      if (xev[i]) cudaEventDestroy(xev[i]);
      if (xev_lo[i]) cudaEventDestroy(xev_lo[i]);
      if (xev_hi[i]) cudaEventDestroy(xev_hi[i]);
    }
    for (void* p : mapped) cudaIpcCloseMemHandle(p);
    L.clear();
    rep.reset();
    if (ev_upd) cudaEventDestroy(ev_upd);
    if (ev_x) cudaEventDestroy(ev_x);
    if (sx) cudaStreamDestroy(sx);
    if (s) cudaStreamDestroy(s);
  }

  int P_() const { return plan.nslabs; }
  bool local(int q) const { return q >= q_lo && q < q_hi; }

  void sync_barrier(cudaStream_t st) {
    CK(cudaStreamSynchronize(st));
    if (comm) comm->barrier();
  }
  void sync_barrier() { sync_barrier(s); }
  template <class V>
  void copy(V* dst, const V* src, int64_t n, cudaStream_t st) {
    if (n <= 0) return;
    CK(cudaMemcpyAsync(dst, src, sizeof(V) * n, cudaMemcpyDeviceToDevice, st));
    exchanged_bytes += (int64_t)sizeof(V) * n;
  }
  template <class V>
  void copy(V* dst, const V* src, int64_t n) { copy(dst, src, n, s); }
  // global planes [a, b) of component k between a window array and an inbox block
  template <class V>
  void to_inbox(V* inbox, const SlabGeo& dst, bool above, const V* v, const SlabGeo& src, int k,
                cudaStream_t st) {
    int a, b;
    dst.ghost(k, above, a, b);
    const int64_t ps = slab_plane(src.g, k);
    copy(inbox + dst.inbox_off(k, above), v + src.g.off[k] + (a - src.g.zoff) * ps, ps * (b - a), st);
  }
  template <class V>
  void from_inbox(V* v, const SlabGeo& dst, bool above, const V* inbox, int k, cudaStream_t st) {
    int a, b;
    dst.ghost(k, above, a, b);
    const int64_t ps = slab_plane(dst.g, k);
    copy(v + dst.g.off[k] + (a - dst.g.zoff) * ps, inbox + dst.inbox_off(k, above), ps * (b - a), st);
  }

  // Ghost exchange of one field per local slab (V indexed by slab). Every
  // inbox holds two halves used in turn (parity per level; all ranks make
  // the same exchange calls), and all copies run on sx: a push into parity
  // k can only follow the neighbour's pulls from k two exchanges back, which
  // its stream finished before the previous exchange's barrier. One barrier
  // per exchange: after the pushes, before the pulls.
  // on_sx: the caller already made sx wait for the update (overlap mode) and
  // orders s after the pulls itself.
  template <class V>
  void exchange(int l, const std::vector<V*>& X, bool on_sx = false) {
    if (!on_sx) {
      CK(cudaEventRecord(ev_upd, s));
      CK(cudaStreamWaitEvent(sx, ev_upd, 0));
    }
    const int par = xpar[l];
    xpar[l] ^= 1;
    for (int q = q_lo; q < q_hi; ++q) {
      const SlabLevel& me = *L[l][q];
      if (q + 1 < P_()) {
        const SlabLevel& up = *L[l][q + 1];
        V* box = SB<V>::peer_lo(up) + par * inbox_half(up.sg, false);
        for (int k = 0; k < 4; ++k) to_inbox(box, up.sg, false, (const V*)X[q], me.sg, k, sx);
      }
      if (q > 0) {
        const SlabLevel& dn = *L[l][q - 1];
        V* box = SB<V>::peer_hi(dn) + par * inbox_half(dn.sg, true);
        for (int k = 0; k < 4; ++k) to_inbox(box, dn.sg, true, (const V*)X[q], me.sg, k, sx);
      }
    }
    if (ev_exchange) {
      // GPU-side: the neighbours' pushes into my inboxes are ordered before my
      // pulls by their events; the host only waits for their enqueue progress
      const int slot = (int)(xseq % kXEv);
      CK(cudaEventRecord(xev[slot], sx));
      ++xseq;
      comm->publish(xseq);
      const int q = comm->rank;
      if (q > 0) {
        comm->wait_for(q - 1, xseq);
        CK(cudaStreamWaitEvent(sx, xev_lo[slot], 0));
      }
      if (q + 1 < P_()) {
        comm->wait_for(q + 1, xseq);
        CK(cudaStreamWaitEvent(sx, xev_hi[slot], 0));
      }
    } else {
      sync_barrier(sx);  // all pushes landed
    }
    for (int q = q_lo; q < q_hi; ++q) {
      SlabLevel& me = *L[l][q];
      const V* lo = (const V*)SB<V>::in_lo(me) + par * inbox_half(me.sg, false);
      const V* hi = (const V*)SB<V>::in_hi(me) + par * inbox_half(me.sg, true);
      for (int k = 0; k < 4; ++k) {
        if (q > 0) from_inbox(X[q], me.sg, false, lo, k, sx);
        if (q + 1 < P_()) from_inbox(X[q], me.sg, true, hi, k, sx);
      }
    }
    if (!on_sx) {
      CK(cudaEventRecord(ev_x, sx));
      CK(cudaStreamWaitEvent(s, ev_x, 0));
    }
  }
  static int64_t inbox_half(const SlabGeo& sg, bool above) { return std::max<int64_t>(1, sg.inbox_size(above)); }

  // Output planes of slab q (window-local, [a, b)) whose rows read no ghost
  // plane: rows at plane z read planes z-1..z+1 of every component.
  void interior_rows(int q, const SlabGeo& sg, int& a, int& b) const {
    const int nz = sg.g.n[2];
    a = q > 0 ? (sg.Z0 - sg.W0()) + 1 : 0;
    b = q + 1 < P_() ? (sg.Z1 - sg.W0()) - 1 : nz + 1;
    if (b < a) b = a;
  }
  // r = b - H x on every local slab. When x's ghosts are stale (an update
  // since the last exchange) the exchange runs on sx while s computes the
  // interior rows; the rows next to the ghost planes follow the exchange.
  template <class V>
  void residual_all(int l, const std::vector<V*>& B, const std::vector<V*>& X, bool for_restrict) {
    auto out = [&](int q) {
      SlabLevel& sl = *L[l][q];
      return for_restrict ? SB<V>::r(sl) : sl.sm.resbuf((const V*)nullptr);
    };
    if (!pend[l]) {
      for (int q = q_lo; q < q_hi; ++q) {
        SlabLevel& sl = *L[l][q];
        launch_residual(sl.sg.g, P, sl.media.ref(), X[q], B[q], out(q), s);
      }
      return;
    }
    CK(cudaEventRecord(ev_upd, s));  // the update the pushes must see
    CK(cudaStreamWaitEvent(sx, ev_upd, 0));
    for (int q = q_lo; q < q_hi; ++q) {
      SlabLevel& sl = *L[l][q];
      int a, b;
      interior_rows(q, sl.sg, a, b);
      if (b > a) launch_residual(sl.sg.g, P, sl.media.ref(), X[q], B[q], out(q), s, a, b);
    }
    exchange(l, X, true);
    CK(cudaEventRecord(ev_x, sx));
    CK(cudaStreamWaitEvent(s, ev_x, 0));
    for (int q = q_lo; q < q_hi; ++q) {
      SlabLevel& sl = *L[l][q];
      int a, b;
      interior_rows(q, sl.sg, a, b);
      if (a > 0) launch_residual(sl.sg.g, P, sl.media.ref(), X[q], B[q], out(q), s, 0, a);
      if (b < sl.sg.g.n[2] + 1) launch_residual(sl.sg.g, P, sl.media.ref(), X[q], B[q], out(q), s, b, -1);
    }
    pend[l] = 0;
  }
  // refresh stale ghosts (before transfers read them)
  template <class V>
  void settle(int l, const std::vector<V*>& X) {
    if (!pend[l]) return;
    exchange(l, X);
    pend[l] = 0;
  }

  template <class V>
  void sweep_all(int l, const std::vector<V*>& B, const std::vector<V*>& X, bool xzero = false) {
    for (int color = 0; color < 2; ++color) {
      const bool first_zero = xzero && color == 0;  // residual is b itself
      if (!first_zero) residual_all(l, B, X, false);
      for (int q = q_lo; q < q_hi; ++q) {
        SlabLevel& sl = *L[l][q];
        const V* rr = first_zero ? (const V*)B[q] : (const V*)sl.sm.resbuf((const V*)nullptr);
        sl.sm.update(sl.sg.g, rr, X[q], opt.damping, color, s);
      }
      pend[l] = 1;
    }
  }

  // multigrid.hpp:217 cycle_at on the distributed levels (B ghosts valid)
  template <class V>
  void cycle(int l, const std::vector<V*>& B, const std::vector<V*>& X, bool xzero = false) {
    const int La = plan.La, nl = plan.nl;
    for (int q = 0; q < opt.nu1; ++q) sweep_all(l, B, X, xzero && q == 0);
    residual_all(l, B, X, true);
    const bool next_coarsest = (l + 2 == nl);
    const int repeat = (opt.cycle == 2 && !next_coarsest) ? 2 : 1;
    if (l + 1 < La) {
      std::vector<V*> BC(P_(), nullptr), EC(P_(), nullptr);
      for (int q = q_lo; q < q_hi; ++q) {
        SlabLevel& f = *L[l][q];
        SlabLevel& c = *L[l + 1][q];
        launch_transfer(f.sg.g, c.sg.g, true, (const V*)SB<V>::r(f), SB<V>::bc(c), false, s);
        CK(cudaMemsetAsync(SB<V>::ec(c), 0, sizeof(V) * c.sg.g.ndofs, s));
        BC[q] = SB<V>::bc(c);
        EC[q] = SB<V>::ec(c);
      }
      exchange(l + 1, BC);
      if constexpr (sizeof(V) == sizeof(cplx)) {
        if (opt.cycle == 3) kcycle(l + 1, BC, EC);
        else
          for (int r = 0; r < repeat; ++r) cycle(l + 1, BC, EC, r == 0);
      } else {
        for (int r = 0; r < repeat; ++r) cycle(l + 1, BC, EC, r == 0);
      }
      for (int q = q_lo; q < q_hi; ++q)
        launch_transfer(L[l][q]->sg.g, L[l + 1][q]->sg.g, false, (const V*)SB<V>::ec(*L[l + 1][q]), X[q], true, s);
    } else {
      // agglomerate: push each slab's restricted owned planes into every rank's full array
      const Geo& gc = G[La];
      sync_barrier();  // every rank finished reading its brep (previous cycle)
      for (int q = q_lo; q < q_hi; ++q) {
        SlabLevel& f = *L[l][q];
        const int c0 = f.sg.Z0 / 2, c1 = f.sg.Z1 / 2;
        const Geo cw = make_window(gc, c0, c1);
        launch_transfer(f.sg.g, cw, true, (const V*)SB<V>::r(f), SB<V>::ctmp(f), false, s);
        const bool last = (q + 1 == P_());
        for (V* dst : rep_of((V*)nullptr))
          for (int k = 0; k < 4; ++k) {
            const int b = (k == 2 && last) ? c1 + 1 : c1;
            const int64_t ps = slab_plane(gc, k);
            copy(dst + gc.off[k] + c0 * ps, (const V*)SB<V>::ctmp(f) + cw.off[k], ps * (b - c0));
          }
      }
      sync_barrier();  // the full coarse rhs is assembled on every rank
      V* bb = rep_b((V*)nullptr);
      V* ee = rep_e((V*)nullptr);
      CK(cudaMemsetAsync(ee, 0, sizeof(V) * gc.ndofs, s));
      CK(cudaStreamSynchronize(s));
      if constexpr (sizeof(V) == sizeof(cplx)) {
        if (opt.cycle == 3 && La + 1 < nl) rep->kcycle_top(bb, ee);
        else
          for (int r = 0; r < repeat; ++r) rep->cycle_t<V>(0, bb, ee, r == 0);
      } else {
        for (int r = 0; r < repeat; ++r) rep->cycle_t<V>(0, bb, ee, r == 0);
      }
      CK(cudaStreamSynchronize(rep->s));
      for (int q = q_lo; q < q_hi; ++q) launch_transfer(L[l][q]->sg.g, gc, false, (const V*)ee, X[q], true, s);
    }
    for (int q = 0; q < opt.nu2; ++q) sweep_all(l, B, X);
    settle(l, X);
  }

  // K-cycle coarse correction on distributed level l1 (multigrid.hpp:217, the
  // cycle_t K branch): inner FGMRES on this rank's window of level l1 with
  // the distributed operator (ghost exchange, then rows) and M = the
  // distributed cycle one level down; dot products over the owned planes,
  // summed in rank order. One local slab (one slab per process).
  void kcycle(int l1, const std::vector<cplx*>& BC, const std::vector<cplx*>& EC) {
    const int q = q_lo;
    SlabLevel& c = *L[l1][q];
    if (!kin[l1]) kin[l1].reset(new Fgmres());
    Fgmres& fg = *kin[l1];
    fg.init(c.sg.g.ndofs, opt.k_inner_iterations, s);
    fg.blas.comm = comm;
    fg.blas.owned = owned_ranges(l1, q);
    // inner K-cycle solves keep the reference's MGS order (orthogonalization = 1)
    ehmg_krylov_options ko{opt.k_inner_iterations, opt.k_inner_iterations, opt.k_inner_rtol, 0.99, 2, 1};
    std::vector<cplx*> VV(P_(), nullptr), WW(P_(), nullptr);
    Fgmres::Fn A = [&](const cplx* in, cplx* out) {
      VV[q] = const_cast<cplx*>(in);  // ghost planes are scratch
      exchange(l1, VV);
      launch_residual(c.sg.g, P, c.media.ref(), in, nullptr, out, s);
    };
    Fgmres::Fn M = [&](const cplx* in, cplx* out) {
      VV[q] = const_cast<cplx*>(in);
      WW[q] = out;
      exchange(l1, VV);
      CK(cudaMemsetAsync(out, 0, sizeof(cplx) * c.sg.g.ndofs, s));
      cycle(l1, VV, WW, true);
    };
    CK(cudaMemsetAsync(EC[q], 0, sizeof(cplx) * c.sg.g.ndofs, s));
    std::vector<double> hist;
    fg.run(A, M, BC[q], EC[q], ko, hist);
  }
  // element ranges of slab q's owned planes in its level-l window
  std::vector<std::pair<int64_t, int64_t>> owned_ranges(int l, int q) const {
    const SlabGeo& sg = L[l][q]->sg;
    const bool last = q + 1 == P_();
    std::vector<std::pair<int64_t, int64_t>> o;
    for (int k = 0; k < 4; ++k) {
      const int64_t ps = slab_plane(sg.g, k);
      const int b = (k == 2 && last) ? sg.Z1 + 1 : sg.Z1;
      o.push_back({sg.g.off[k] + (sg.Z0 - sg.g.zoff) * ps, sg.g.off[k] + (b - sg.g.zoff) * ps});
    }
    return o;
  }

  // z = M r on the level-0 windows of the local slabs (ghosts of B refreshed
  // here); precision 1 converts the windows to complex64 and back
  // (multigrid.hpp:310 convert_field) around the complex64 cycle.
  void precondition_windows(const std::vector<cplx*>& B, const std::vector<cplx*>& X) {
    if (prec == 0) {
      exchange(0, B);
      for (int q = q_lo; q < q_hi; ++q)
        CK(cudaMemsetAsync(X[q], 0, sizeof(cplx) * L[0][q]->sg.g.ndofs, s));
      cycle(0, B, X, true);
      return;
    }
    std::vector<cplxf*> Bf(P_(), nullptr), Xf(P_(), nullptr);
    for (int q = q_lo; q < q_hi; ++q) {
      const int64_t n = L[0][q]->sg.g.ndofs;
      Bf[q] = bwf[q - q_lo]->p;
      Xf[q] = xwf[q - q_lo]->p;
      k_convert<cplxf, cplx><<<grid_for(n, 148 * 64), kThreads, 0, s>>>(n, B[q], Bf[q]);
      CK(cudaGetLastError());
      CK(cudaMemsetAsync(Xf[q], 0, sizeof(cplxf) * n, s));
    }
    exchange(0, Bf);  // complex64 ghost planes
    cycle(0, Bf, Xf, true);
    for (int q = q_lo; q < q_hi; ++q) {
      const int64_t n = L[0][q]->sg.g.ndofs;
      k_convert<cplx, cplxf><<<grid_for(n, 148 * 64), kThreads, 0, s>>>(n, Xf[q], X[q]);
      CK(cudaGetLastError());
    }
  }

  // global array <-> level-0 windows of the local slabs
  void scatter(const cplx* full, std::vector<cplx*>& W) {
    for (int q = q_lo; q < q_hi; ++q) {
      const Geo& w = L[0][q]->sg.g;
      for (int k = 0; k < 4; ++k) {
        const int64_t ps = slab_plane(w, k);
        CK(cudaMemcpyAsync(W[q] + w.off[k], full + G[0].off[k] + (int64_t)w.zoff * ps,
                           sizeof(cplx) * ps * (w.n[2] + (k == 2)), cudaMemcpyDeviceToDevice, s));
      }
    }
  }
  void gather(const std::vector<cplx*>& W, cplx* full) {
    for (int q = q_lo; q < q_hi; ++q) {
      const SlabGeo& sg = L[0][q]->sg;
      const bool last = (q + 1 == P_());
      for (int k = 0; k < 4; ++k) {
        const int64_t ps = slab_plane(sg.g, k);
        const int b = (k == 2 && last) ? sg.Z1 + 1 : sg.Z1;
        CK(cudaMemcpyAsync(full + G[0].off[k] + (int64_t)sg.Z0 * ps, W[q] + sg.g.off[k] + (sg.Z0 - sg.g.zoff) * ps,
                           sizeof(cplx) * ps * (b - sg.Z0), cudaMemcpyDeviceToDevice, s));
      }
    }
  }
  std::vector<cplx*> windows(std::vector<std::unique_ptr<DBuf<cplx>>>& v) {
    std::vector<cplx*> out(P_(), nullptr);
    for (int q = q_lo; q < q_hi; ++q) out[q] = v[q - q_lo]->p;
    return out;
  }
  // full-array boundary: scatter r (ghosts included), cycle, gather owned planes
  void precondition(const cplx* r, cplx* z) {
    auto B = windows(bw), X = windows(xw);
    scatter(r, B);
    if (prec == 0) {
      for (int q = q_lo; q < q_hi; ++q)
        CK(cudaMemsetAsync(X[q], 0, sizeof(cplx) * L[0][q]->sg.g.ndofs, s));
      cycle(0, B, X, true);
    } else {
      precondition_windows(B, X);
    }
    gather(X, z);
    CK(cudaStreamSynchronize(s));
  }
};

static std::unique_ptr<ehmg_slab_mg_s> build_slab_mg(const Geo& g0, const double* const* host, const OpPar& P,
                                                     const ehmg_mg_options& opt, int nslabs, int agg_n2,
                                                     NodeComm* comm) {
  if (g0.nd != 3) throw Err(EHMG_EINVAL, "slab: z-slab decomposition is 3D only");
  if (opt.cycle == 3 && (comm ? comm->n != nslabs : nslabs != 1))
    throw Err(EHMG_EINVAL, "slab: K-cycles need one slab per process (the inner Krylov is distributed over ranks)");
  if (opt.cycle == 3 && opt.precision != 0) throw Err(EHMG_EINVAL, "mixed precision: K-cycles are not supported");
  if (opt.sweep != 1) throw Err(EHMG_EINVAL, "slab: only red-black sweeps decompose");
  if (opt.precision != 0 && opt.precision != 1) throw Err(EHMG_EINVAL, "slab: precision must be 0 or 1");
  if (!stencil3d_supported(g0)) throw Err(EHMG_EINVAL, "slab: needs an even x extent (TMA stencil)");
  auto sm = std::make_unique<ehmg_slab_mg_s>();
  sm->opt = opt;
  sm->prec = opt.precision;
  const bool mixed = opt.precision == 1;
  sm->P = P;
  sm->comm = comm;
  sm->plan = make_slab_plan(g0.n[2], opt.n_levels, nslabs, agg_n2);
  if (comm) {
    if (comm->n != nslabs) throw Err(EHMG_EINVAL, "slab: one slab per process");
    sm->q_lo = comm->rank;
    sm->q_hi = comm->rank + 1;
  } else {
    sm->q_lo = 0;
    sm->q_hi = nslabs;
  }
  const int La = sm->plan.La, nl = opt.n_levels;
  CK(cudaGetDevice(&sm->dev));
  CK(cudaStreamCreateWithFlags(&sm->s, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&sm->sx, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&sm->ev_upd, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&sm->ev_x, cudaEventDisableTiming));
  cudaStream_t s = sm->s;
  // global media per level [0, La] (every rank holds them; setup only)
  std::vector<std::unique_ptr<DevMedia>> gm;
  for (int l = 0; l <= La; ++l) {
    sm->G.push_back(l == 0 ? g0 : coarse_geo(sm->G[l - 1]));
    gm.emplace_back(new DevMedia());
    if (l == 0) gm[0]->upload(g0.ncells, host, s);
    else gm[l - 1]->coarsen_into(sm->G[l - 1], *gm[l], sm->G[l], s);
  }
  sm->L.resize(La);
  sm->pend.assign(La, 0);
  sm->xpar.assign(La, 0);
  sm->kin.resize(La);
  for (int l = 0; l < La; ++l) {
    for (int q = 0; q < nslabs; ++q) {
      auto sl = std::make_unique<SlabLevel>();
      sl->sg.Z0 = sm->plan.z0[q] >> l;
      sl->sg.Z1 = sm->plan.z0[q + 1] >> l;
      const int w0 = std::max(0, sl->sg.Z0 - kSlabGhostLo), w1 = std::min(sm->G[l].n[2], sl->sg.Z1 + kSlabGhostHi);
      sl->sg.g = make_window(sm->G[l], w0, w1);
      sl->local = sm->local(q);
      if (sl->local) {
        sl->media.window_of(*gm[l], sm->G[l], w0, w1, s);
        sl->sm.build(sm->G[l], P, gm[l]->packed.p, opt.vanka_mode == 0 ? 1 : 0, s, w0, w1, sl->media.soa.p);
        const int64_t nd = sl->sg.g.ndofs;
        // two halves per inbox (exchanges alternate between them)
        const int64_t ilo = 2 * ehmg_slab_mg_s::inbox_half(sl->sg, false);
        const int64_t ihi = 2 * ehmg_slab_mg_s::inbox_half(sl->sg, true);
        const int64_t nct = l == La - 1 ? make_window(sm->G[La], sl->sg.Z0 / 2, sl->sg.Z1 / 2).ndofs : 0;
        if (mixed) {
          // complex64 cache (factorised in double, rounded), float media, float vectors
          sl->sm.make_float(sl->sg.g, s);
          sl->media.make_float(sl->sg.g.ncells, s);
          sl->rf.alloc(nd);
          if (l > 0) {
            sl->bcf.alloc(nd);
            sl->ecf.alloc(nd);
          }
          sl->in_lof.alloc(ilo);
          sl->in_hif.alloc(ihi);
          sl->peer_lof = sl->in_lof.p;
          sl->peer_hif = sl->in_hif.p;
          if (nct) sl->ctmpf.alloc(nct);
          if (l == 0) {  // complex128 level-0 exchanges of the distributed FGMRES operator
            sl->in_lo.alloc(ilo);
            sl->in_hi.alloc(ihi);
            sl->peer_lo = sl->in_lo.p;
            sl->peer_hi = sl->in_hi.p;
          }
        } else {
          sl->r.alloc(nd);
          if (l > 0) {
            sl->bc.alloc(nd);
            sl->ec.alloc(nd);
          }
          sl->in_lo.alloc(ilo);
          sl->in_hi.alloc(ihi);
          sl->peer_lo = sl->in_lo.p;
          sl->peer_hi = sl->in_hi.p;
          if (nct) sl->ctmp.alloc(nct);
        }
      }
      sm->L[l].push_back(std::move(sl));
    }
  }
  for (int q = sm->q_lo; q < sm->q_hi; ++q) {
    sm->bw.emplace_back(new DBuf<cplx>(sm->L[0][q]->sg.g.ndofs));
    sm->xw.emplace_back(new DBuf<cplx>(sm->L[0][q]->sg.g.ndofs));
    if (mixed) {
      sm->bwf.emplace_back(new DBuf<cplxf>(sm->L[0][q]->sg.g.ndofs));
      sm->xwf.emplace_back(new DBuf<cplxf>(sm->L[0][q]->sg.g.ndofs));
    }
  }
  CK(cudaStreamSynchronize(s));
  sm->rep = build_mg(sm->G[La], nullptr, gm[La].get(), P, opt, nl - La);
  if (mixed) {
    sm->brepf.alloc(sm->G[La].ndofs);
    sm->erepf.alloc(sm->G[La].ndofs);
    sm->brepf_of.push_back(sm->brepf.p);
  } else {
    sm->brep.alloc(sm->G[La].ndofs);
    sm->erep.alloc(sm->G[La].ndofs);
    sm->brep_of.push_back(sm->brep.p);
  }
  if (comm && comm->n > 1) {
    // share inbox and coarse-rhs buffers through CUDA IPC (peer pointers)
    struct Blob {
      // inboxes per level, coarse rhs, complex128 level-0 inboxes (mixed), coarsest solution
      cudaIpcMemHandle_t h[2 * 8 + 1 + 2 + 1];
    } mine{}, all[kCommMaxRanks];
    // the coarsest level's solution buffer of the replicated hierarchy
    void* cx = nullptr;
    {
      ehmg_mg_s& R = *sm->rep;
      if (R.L.size() == 1) cx = mixed ? (void*)sm->erepf.p : (void*)sm->erep.p;
      else cx = mixed ? (void*)R.L.back()->ecf.p : (void*)R.L.back()->ec.p;
    }
    CK(cudaIpcGetMemHandle(&mine.h[19], cx));
    const int q = comm->rank;
    for (int l = 0; l < La; ++l) {
      SlabLevel& me = *sm->L[l][q];
      CK(cudaIpcGetMemHandle(&mine.h[2 * l], mixed ? (void*)me.in_lof.p : (void*)me.in_lo.p));
      CK(cudaIpcGetMemHandle(&mine.h[2 * l + 1], mixed ? (void*)me.in_hif.p : (void*)me.in_hi.p));
    }
    CK(cudaIpcGetMemHandle(&mine.h[16], mixed ? (void*)sm->brepf.p : (void*)sm->brep.p));
    if (mixed) {
      CK(cudaIpcGetMemHandle(&mine.h[17], sm->L[0][q]->in_lo.p));
      CK(cudaIpcGetMemHandle(&mine.h[18], sm->L[0][q]->in_hi.p));
    }
    comm->exchange_blob(&mine, sizeof(Blob), all);
    {
      // Event-ordered exchanges when the neighbours run on other GPUs; ranks
      // sharing one GPU keep the drain + host barrier (a stream waiting on
      // another process's event on the same GPU forces context switches:
      // 61 vs 13 ms per 128^3 cycle with 2 ranks on one B200,
      // profiles/round2/dist_overhead_128.json). EHMG_EXCHANGE=event|host
      // overrides (the tests run both on one GPU).
      struct EvBlob {
        cudaIpcEventHandle_t e[ehmg_slab_mg_s::kXEv];
        cudaUUID_t dev;
      } emine{}, eall[kCommMaxRanks];
      {
        cudaDeviceProp prop;
        CK(cudaGetDeviceProperties(&prop, sm->dev));
        emine.dev = prop.uuid;
      }
      for (int i = 0; i < ehmg_slab_mg_s::kXEv; ++i) {
        CK(cudaEventCreateWithFlags(&sm->xev[i], cudaEventDisableTiming | cudaEventInterprocess));
        CK(cudaIpcGetEventHandle(&emine.e[i], sm->xev[i]));
      }
      comm->exchange_blob(&emine, sizeof(EvBlob), eall);
      bool shared = false;
      for (int r = q - 1; r <= q + 1; r += 2)
        if (r >= 0 && r < comm->n && std::memcmp(&eall[r].dev, &emine.dev, sizeof(cudaUUID_t)) == 0) shared = true;
      const char* ex = std::getenv("EHMG_EXCHANGE");
      sm->ev_exchange = ex && std::strcmp(ex, "event") == 0 ? true : ex && std::strcmp(ex, "host") == 0 ? false : !shared;
      for (int i = 0; i < ehmg_slab_mg_s::kXEv; ++i) {
        if (q > 0) CK(cudaIpcOpenEventHandle(&sm->xev_lo[i], eall[q - 1].e[i]));
        if (q + 1 < comm->n) CK(cudaIpcOpenEventHandle(&sm->xev_hi[i], eall[q + 1].e[i]));
      }
    }
    sm->brep_of.clear();
    sm->brepf_of.clear();
    sm->cx_of.assign(comm->n, nullptr);
    for (int r = 0; r < comm->n; ++r) {
      if (r == q) {
        sm->cx_of[r] = cx;
        if (mixed) sm->brepf_of.push_back(sm->brepf.p);
        else sm->brep_of.push_back(sm->brep.p);
        continue;
      }
      auto open = [&](cudaIpcMemHandle_t h) {
        void* p = nullptr;
        CK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
        sm->mapped.push_back(p);
        return p;
      };
      for (int l = 0; l < La; ++l) {
        SlabLevel& peer = *sm->L[l][r];
        if (mixed) {
          peer.peer_lof = static_cast<cplxf*>(open(all[r].h[2 * l]));
          peer.peer_hif = static_cast<cplxf*>(open(all[r].h[2 * l + 1]));
        } else {
          peer.peer_lo = static_cast<cplx*>(open(all[r].h[2 * l]));
          peer.peer_hi = static_cast<cplx*>(open(all[r].h[2 * l + 1]));
        }
      }
      if (mixed) {
        sm->brepf_of.push_back(static_cast<cplxf*>(open(all[r].h[16])));
        sm->L[0][r]->peer_lo = static_cast<cplx*>(open(all[r].h[17]));
        sm->L[0][r]->peer_hi = static_cast<cplx*>(open(all[r].h[18]));
      } else {
        sm->brep_of.push_back(static_cast<cplx*>(open(all[r].h[16])));
      }
      sm->cx_of[r] = open(all[r].h[19]);
    }
    // Row-partitioned coarsest solve: rank q keeps rows [r0, r1) of S^-1
    // (the displacement Schur complement; 1/n of the dense inverse and of the
    // per-cycle GEMV), pushes its rows of u into every rank's buffer, and
    // every rank then recovers the pressure locally.
    {
      ehmg_mg_s& R = *sm->rep;
      const int64_t ncu = R.ncu, r0 = ncu * q / comm->n, r1 = ncu * (q + 1) / comm->n;
      R.split_coarse(r0, r1, R.s);
      ehmg_slab_mg_s* smp = sm.get();
      R.coarse_gather = [smp, r0, r1](void* x, size_t es) {
        ehmg_mg_s& RR = *smp->rep;
        NodeComm& cm = *smp->comm;
        CK(cudaStreamSynchronize(RR.s));
        cm.barrier();  // every rank has its rows and no longer reads its previous solution
        for (int r = 0; r < cm.n; ++r)
          if (r != cm.rank && r1 > r0)
            CK(cudaMemcpyAsync(static_cast<char*>(smp->cx_of[r]) + r0 * es, static_cast<char*>(x) + r0 * es,
                               (r1 - r0) * es, cudaMemcpyDeviceToDevice, RR.s));
        CK(cudaStreamSynchronize(RR.s));
        cm.barrier();  // all row blocks landed
      };
    }
  }
  CK(cudaStreamSynchronize(s));
  return sm;
}
