// pcg2d_pair.cuh — kernel (d), 2-D IC(0), TWO same-label samples per CTA.
//
// The IC(0) sweeps of pcg2d.cuh are latency-bound: 2 (2m - 1) dependent levels
// per application, each a short fp64 chain, a ring wait and a block barrier
// (≈ 585 cycles per level for one CTA; profiles/r02f_pcg2d_ncu.md). Here one CTA
// carries a pair of samples that share a label (cut from the label-major,
// cost-ordered queue): both samples' sweeps walk the levels together, so every
// level's barrier, loop control, address cursors and the centroid factor's
// operands (D, a_W, a_S, RN(1/D), prefetched once into the shared ring) serve
// two independent chains, which also overlap each other's latency. The flat
// passes (P1, P2) are pcg2d's, run once per sample. Arithmetic per sample is
// exactly pcg2d's (hence the oracle's): records are bit-identical to the
// one-sample kernel in both the throughput and the reference-order mode.
// A pair whose samples finish at different iterations continues with the
// remaining one (its sweeps then carry one chain).
#pragma once
#include "pcg2d.cuh"

namespace vqpc {

constexpr int P2P_NOPS = 8;  // ring operands per level: fwd r_A, r_B, W, S, D, R; bwd W_E, S_N, D, R, y_A, y_B, r_A, r_B
constexpr size_t P2P_RING_SM = sizeof(double) * P2_DEPTH * P2P_NOPS * P2_T;
constexpr size_t P2P_DSMEM = P2P_RING_SM > P2_FLAT_SM ? P2P_RING_SM : P2_FLAT_SM;

template <int MC>
__global__ void __launch_bounds__(P2_T, 2) pcg2d_pair_kernel(const Pcg2dParams prm) {
  constexpr int NW = P2_T / 32;
  extern __shared__ __align__(16) double dsm[];
  __shared__ double sbuf[2][2][P2_T + 2];  // [sample][level parity][iy + 1]
  __shared__ int2 lvl_dd[P2_MAXL];
  __shared__ double red[6][NW];
  __shared__ int s_grp;
  __shared__ double s_bval;
  Grid2D g = prm.g;
  if constexpr (MC > 0) {
    g.m = MC;
    g.n = MC * MC;
    g.L = 2 * MC - 1;
  }
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  for (int l = t; l < g.L; l += P2_T) lvl_dd[l] = make_int2(l > 0 ? wf_dw(l, g.m) : 0, l + 1 < g.L ? wf_de(l, g.m) : 0);
  __syncthreads();
  const int n = g.n, m = g.m;
  double* base = prm.work + static_cast<size_t>(blockIdx.x) * 2 * P2_WORK * n;
  double *Ad[2], *Aw[2], *As[2], *Xb[2][2], *Rv[2], *Pb[2][2], *Y[2], *Z[2], *Prod[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    double* b = base + static_cast<size_t>(q) * P2_WORK * n;
    Ad[q] = b;
    Aw[q] = b + n;
    As[q] = b + 2 * n;
    Xb[q][0] = b + 3 * n;
    Xb[q][1] = b + 4 * n;
    Rv[q] = b + 5 * n;
    Pb[q][0] = b + 6 * n;
    Pb[q][1] = b + 7 * n;
    Y[q] = b + 8 * n;
    Z[q] = b + 9 * n;
    Prod[q] = b + 10 * n;
  }
  const bool exact = prm.exact != 0;
  auto reduce = [&](int q, double part, double* red_slot) {
    return exact ? serial_sum2d(Prod[q], n, red_slot) : block_sum2d<NW>(part, red_slot, warp, lane);
  };
  auto nat = [&](int l) { return t * m + (l - t); };
  const bool trow = t < m;
  auto lin = [&](int l) {
    if (l < m) return ((l * (l + 1)) >> 1) + t;
    const int r = 2 * m - 1 - l;
    return m * m - ((r * (r + 1)) >> 1) + t - (l - m + 1);
  };
  auto up = [&](int l) { return l < m - 1 ? l + 1 : 2 * m - 2 - l; };
  auto on = [&](int l) { return trow && static_cast<unsigned>(l - t) < static_cast<unsigned>(m); };
  const unsigned ring_sa = static_cast<unsigned>(__cvta_generic_to_shared(dsm)) + t * 8u;
  const unsigned long long pol_fac = l2_policy_last();
  constexpr unsigned OPB = P2_T * 8u, SLOTB = P2P_NOPS * P2_T * 8u;
  auto next_slot = [](int sl) { return sl + 1 == P2_DEPTH ? 0 : sl + 1; };
  double (*ring)[P2P_NOPS][P2_T] = reinterpret_cast<double (*)[P2P_NOPS][P2_T]>(dsm);

  for (;;) {
    if (t == 0) s_grp = atomicAdd(prm.counter, 1);
    __syncthreads();
    const int grp = s_grp;
    __syncthreads();
    if (grp >= *prm.ngroups) break;
    const int2 gr = prm.groups[grp];
    int sid[2], J[2], mit[2], xc[2] = {0, 0}, pc[2] = {0, 0};
    int64_t gsv[2];
    bool act[2];
    double rel_rec[2], norm_b[2], rz[2], beta[2] = {0.0, 0.0}, alpha[2] = {0.0, 0.0};
    uint8_t st[2];
    int label = 0;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      act[q] = false;
      J[q] = 0;
      rel_rec[q] = 0.0;
      st[q] = VQPC_S_MAX_ITER;
      sid[q] = -1;
      gsv[q] = 0;
      mit[q] = 0;
      if (q < gr.y) {
        const int sm = prm.perm[gr.x + q];
        sid[q] = sm;
        gsv[q] = prm.out_base + sm;
        const int lb = prm.labels[sm];
        if (lb < 0 || prm.kflag[sm] || gsv[q] >= prm.solve_limit) {
          st[q] = gsv[q] >= prm.solve_limit ? VQPC_S_NOT_SOLVED
                  : lb < 0                  ? VQPC_S_INVALID_LATENT
                                            : (prm.kflag[sm] & 1) ? VQPC_S_COEFF_OVERFLOW : VQPC_S_INVALID_COEFF;
        } else {
          act[q] = true;
          label = lb;
        }
        mit[q] = prm.max_iter_arr ? prm.max_iter_arr[gsv[q]] : (prm.max_iter < 0 ? 10 * n : prm.max_iter);
      }
    }
    const double* FD = prm.fac + static_cast<size_t>(label) * P2_FAC * n;
    const double* FW = FD + n;
    const double* FS = FW + n;
    const double* FR = FS + n;

    // ---- setup: the samples' rows, x = 0, r = b ----------------------------------
    double bb[2] = {0.0, 0.0};
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      if (!act[q]) continue;
      const double* kap = prm.kappa + static_cast<size_t>(sid[q]) * prm.ldk;
      for (int l = 0; l < g.L; ++l) {
        const int a = wf_addr(g, l, t);
        if (a >= 0) {
          const RowCoef rc = assemble_row(kap, g, l - t, t);
          Ad[q][a] = rc.d;
          Aw[q][a] = rc.w;
          As[q][a] = rc.s;
          Xb[q][0][a] = 0.0;
          Rv[q][a] = rc.b;
          if (t == 0 && l == 0) s_bval = rc.b;
          bb[q] = fma(rc.b, rc.b, bb[q]);
          if (exact) Prod[q][nat(l)] = __dmul_rn(rc.b, rc.b);
        }
      }
    }
    __syncthreads();
    const double bval = s_bval;

    // ---- both samples' IC(0) sweeps, level by level (pcg2d's, two chains) --------
    auto fwd_issue = [&](int l, int a, int sl, bool aA, bool aB) {
      if (on(l)) {
        const unsigned r0 = ring_sa + sl * SLOTB;
        if (aA) cp_async8s(r0, Rv[0] + a);
        if (aB) cp_async8s(r0 + OPB, Rv[1] + a);
        cp_async8h(r0 + 2 * OPB, FW + a, pol_fac);
        cp_async8h(r0 + 3 * OPB, FS + a, pol_fac);
        cp_async8h(r0 + 4 * OPB, FD + a, pol_fac);
        cp_async8h(r0 + 5 * OPB, FR + a, pol_fac);
      }
      cp_commit();
    };
    auto bwd_issue = [&](int l, int a, int sl, bool aA, bool aB) {
      if (l >= 0 && on(l)) {
        const unsigned r0 = ring_sa + sl * SLOTB;
        const int ae = a + up(l);
        if (l - t < m - 1) cp_async8h(r0, FW + ae, pol_fac);
        if (t < m - 1) cp_async8h(r0 + OPB, FS + ae + 1, pol_fac);
        cp_async8h(r0 + 2 * OPB, FD + a, pol_fac);
        cp_async8h(r0 + 3 * OPB, FR + a, pol_fac);
        if (aA) {
          cp_async8s(r0 + 4 * OPB, Y[0] + a);
          cp_async8s(r0 + 6 * OPB, Rv[0] + a);
        }
        if (aB) {
          cp_async8s(r0 + 5 * OPB, Y[1] + a);
          cp_async8s(r0 + 7 * OPB, Rv[1] + a);
        }
      }
      cp_commit();
    };
    // returns the r.z partials of both samples in rzp
    auto sweeps = [&](double (&rzp)[2], bool aA, bool aB) {
      __syncthreads();
      int ai = lin(0), ac = ai;
      int si = 0, sc = 0;
      for (int l = 0; l < P2_DEPTH - 1; ++l) {
        fwd_issue(l, ai, si, aA, aB);
        ai += up(l);
        si = next_slot(si);
      }
      for (int l = 0; l < g.L; ++l) {
        fwd_issue(l + P2_DEPTH - 1, ai, si, aA, aB);
        ai += up(l + P2_DEPTH - 1);
        si = next_slot(si);
        cp_wait<P2_DEPTH - 1>();
        const int cur = l & 1, prv = cur ^ 1;
        if (on(l)) {
          const double* op = &ring[sc][0][t];
          const double fw = op[2 * P2_T], fs = op[3 * P2_T], fd = op[4 * P2_T], fr = op[5 * P2_T];
          VQPC_DCHECK(ac >= 0 && ac < n);
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            if (!(q == 0 ? aA : aB)) continue;
            double v = op[q * P2_T];
            if (l - t > 0) v = __dsub_rn(v, __dmul_rn(fw, sbuf[q][prv][t + 1]));
            if (t > 0) v = __dsub_rn(v, __dmul_rn(fs, sbuf[q][prv][t]));
            v = div_by_pivot(v, fd, fr);
            Y[q][ac] = v;
            sbuf[q][cur][t + 1] = v;
          }
        }
        ac += up(l);
        sc = next_slot(sc);
        __syncthreads();
      }
      cp_wait<0>();
      __syncthreads();
      rzp[0] = rzp[1] = 0.0;
      ai = lin(g.L - 1);
      ac = ai;
      si = sc = 0;
      for (int l = g.L - 1; l > g.L - P2_DEPTH; --l) {
        bwd_issue(l, ai, si, aA, aB);
        ai -= up(l - 1);
        si = next_slot(si);
      }
      for (int l = g.L - 1; l >= 0; --l) {
        bwd_issue(l - (P2_DEPTH - 1), ai, si, aA, aB);
        ai -= up(l - P2_DEPTH);
        si = next_slot(si);
        cp_wait<P2_DEPTH - 1>();
        const int cur = l & 1, prv = cur ^ 1;
        if (on(l)) {
          const double* op = &ring[sc][0][t];
          const double few = op[0], fsn = op[P2_T], fd = op[2 * P2_T], fr = op[3 * P2_T];
          VQPC_DCHECK(ac >= 0 && ac < n);
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            if (!(q == 0 ? aA : aB)) continue;
            double acc = 0.0;
            if (l - t < m - 1) acc = __dadd_rn(acc, __dmul_rn(few, sbuf[q][prv][t + 1]));
            if (t < m - 1) acc = __dadd_rn(acc, __dmul_rn(fsn, sbuf[q][prv][t + 2]));
            const double z = __dsub_rn(op[(4 + q) * P2_T], div_by_pivot(acc, fd, fr));
            Z[q][ac] = z;
            sbuf[q][cur][t + 1] = z;
            const double rv = op[(6 + q) * P2_T];
            rzp[q] = fma(rv, z, rzp[q]);
            if (exact) Prod[q][t * m + (l - t)] = __dmul_rn(rv, z);
          }
        }
        ac -= up(l - 1);
        sc = next_slot(sc);
        __syncthreads();
      }
      cp_wait<0>();
    };

    // ---- the flat passes of pcg2d.cuh for sample q ------------------------------------
    const int NC = (n + P2_T - 1) / P2_T;
    double* raw = dsm;
    double* xch = dsm + P2_RSLOT * P2_RAW * P2_T;
    int* rawi = reinterpret_cast<int*>(xch + 4 * P2_XCH * P2_T);
    auto RAW = [&](int k, int v) -> double* { return raw + ((static_cast<unsigned>(k) % P2_RSLOT) * P2_RAW + v) * P2_T + t; };
    auto XCH = [&](int x, int qq) -> double& { return xch[x * 4 * P2_T + (qq & (4 * P2_T - 1))]; };
    const unsigned long long pol_str = l2_policy_first();
    struct Nb { int s, w, e, nn, ix, iy; };
    auto nbrs = [&](int a, int lv) {
      const int l = lv & 0xffff, iy = lv >> 16, ix = l - iy;
      Nb b;
      const int2 dd = lvl_dd[l];
      b.w = ix > 0 ? a - dd.x : -1;
      b.s = iy > 0 ? a - dd.x - 1 : -1;
      b.e = ix < m - 1 ? a + dd.y : -1;
      b.nn = iy < m - 1 ? a + dd.y + 1 : -1;
      b.ix = ix;
      b.iy = iy;
      return b;
    };
    auto xv = [&](int x, int qq) { return qq < 0 ? 0.0 : XCH(x, qq); };
    // P1: p_new = z + beta p_old into the other half; returns this thread's pAp partial
    auto p1 = [&](int q, bool first) -> double {
      const double* Po = Pb[q][pc[q]];
      double* Pn = Pb[q][pc[q] ^ 1];
      const double* Zq = Z[q];
      const double bt = beta[q];
      double* Asq = As[q];
      double* Awq = Aw[q];
      double* Adq = Ad[q];
      auto flat_issue = [&](int k, const double* v0, const double* v1) {
        const int a = k * P2_T + t;
        if (k < NC && a < n) {
          if (v0) cp_async8p(RAW(k, 0), v0 + a, pol_str);
          if (v1) cp_async8p(RAW(k, 1), v1 + a, pol_str);
          cp_async8p(RAW(k, 3), Asq + a, pol_str);
          cp_async8p(RAW(k, 4), Awq + a, pol_str);
          cp_async8p(RAW(k, 5), Adq + a, pol_str);
          cp_async4(rawi + (static_cast<unsigned>(k) % P2_RSLOT) * P2_T + t, prm.gmap + a);
        }
        cp_commit();
      };
      double pap = 0.0;
      __syncthreads();
      for (int k = 0; k < P2_SD; ++k) flat_issue(k, Zq, first ? nullptr : Po);
      double cs = 0.0, cw = 0.0, cd = 0.0;
      int clv = 0;
      for (int k = 0; k <= NC; ++k) {
        const double ps = cs, pw = cw, pd = cd;
        const int plv = clv;
        if (k < NC) {
          cp_wait<P2_SD - 1>();
          const int a = k * P2_T + t;
          if (a < n) {
            const double z = *RAW(k, 0);
            const double pcv = first ? z : __dadd_rn(z, __dmul_rn(bt, *RAW(k, 1)));
            cs = *RAW(k, 3);
            cw = *RAW(k, 4);
            cd = *RAW(k, 5);
            clv = rawi[(static_cast<unsigned>(k) % P2_RSLOT) * P2_T + t];
            XCH(0, a) = pcv;
            XCH(2, a) = cw;
            XCH(3, a) = cs;
            Pn[a] = pcv;
          }
        }
        flat_issue(k + P2_SD, Zq, first ? nullptr : Po);
        __syncthreads();
        const int a = (k - 1) * P2_T + t;
        if (k >= 1 && a < n) {
          const Nb b = nbrs(a, plv);
          const double pcv = XCH(0, a);
          const double ap = row_apply(ps, pw, pd, xv(2, b.e), xv(3, b.nn), xv(0, b.s), xv(0, b.w), pcv, xv(0, b.e),
                                      xv(0, b.nn));
          pap = fma(pcv, ap, pap);
          if (exact) Prod[q][b.iy * m + b.ix] = __dmul_rn(pcv, ap);
        }
      }
      pc[q] ^= 1;
      return pap;
    };
    // P2: x_new = x + alpha p, r -= alpha A p, |b - A x_new|^2; returns the rr partial
    auto p2 = [&](int q) -> double {
      const double* Pv = Pb[q][pc[q]];
      const double* Xo = Xb[q][xc[q]];
      double* Xn = Xb[q][xc[q] ^ 1];
      double* Rq = Rv[q];
      const double al = alpha[q];
      double* Asq = As[q];
      double* Awq = Aw[q];
      double* Adq = Ad[q];
      auto flat_issue = [&](int k) {
        const int a = k * P2_T + t;
        if (k < NC && a < n) {
          cp_async8p(RAW(k, 0), Pv + a, pol_str);
          cp_async8p(RAW(k, 1), Xo + a, pol_str);
          cp_async8p(RAW(k, 2), Rq + a, pol_str);
          cp_async8p(RAW(k, 3), Asq + a, pol_str);
          cp_async8p(RAW(k, 4), Awq + a, pol_str);
          cp_async8p(RAW(k, 5), Adq + a, pol_str);
          cp_async4(rawi + (static_cast<unsigned>(k) % P2_RSLOT) * P2_T + t, prm.gmap + a);
        }
        cp_commit();
      };
      double rr = 0.0;
      __syncthreads();
      for (int k = 0; k < P2_SD; ++k) flat_issue(k);
      double cs = 0.0, cw = 0.0, cd = 0.0, cr = 0.0;
      int clv = 0;
      double cb = bval;
      for (int k = 0; k <= NC; ++k) {
        const double ps = cs, pw = cw, pd = cd, pr = cr, pb = cb;
        const int plv = clv;
        if (k < NC) {
          cp_wait<P2_SD - 1>();
          const int a = k * P2_T + t;
          if (a < n) {
            if (prm.bvec) cb = __ldg(prm.bvec + a);
            const double pvv = *RAW(k, 0);
            const double xn = __dadd_rn(*RAW(k, 1), __dmul_rn(al, pvv));
            cr = *RAW(k, 2);
            cs = *RAW(k, 3);
            cw = *RAW(k, 4);
            cd = *RAW(k, 5);
            clv = rawi[(static_cast<unsigned>(k) % P2_RSLOT) * P2_T + t];
            XCH(0, a) = pvv;
            XCH(1, a) = xn;
            XCH(2, a) = cw;
            XCH(3, a) = cs;
            Xn[a] = xn;
          }
        }
        flat_issue(k + P2_SD);
        __syncthreads();
        const int a = (k - 1) * P2_T + t;
        if (k >= 1 && a < n) {
          const Nb b = nbrs(a, plv);
          const double aE = xv(2, b.e), aN = xv(3, b.nn);
          const double ap = row_apply(ps, pw, pd, aE, aN, xv(0, b.s), xv(0, b.w), XCH(0, a), xv(0, b.e), xv(0, b.nn));
          const double ax = row_apply(ps, pw, pd, aE, aN, xv(1, b.s), xv(1, b.w), XCH(1, a), xv(1, b.e), xv(1, b.nn));
          const double rt = __dsub_rn(pb, ax);
          rr = fma(rt, rt, rr);
          if (exact) Prod[q][b.iy * m + b.ix] = __dmul_rn(rt, rt);
          Rq[a] = __dsub_rn(pr, __dmul_rn(al, ap));
        }
      }
      xc[q] ^= 1;
      return rr;
    };

    // ---- the PCG iterations of both samples (solver.cpp:186-245 per sample) -------------
#pragma unroll
    for (int q = 0; q < 2; ++q)
      if (act[q]) norm_b[q] = sqrt(reduce(q, bb[q], red[q]));
    {
      double rzp[2];
      sweeps(rzp, act[0], act[1]);
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        if (!act[q]) continue;
        rz[q] = reduce(q, rzp[q], red[2 + q]);
        if (norm_b[q] == 0.0) {
          st[q] = VQPC_S_CONVERGED;
          act[q] = false;
        } else if (!(rz[q] > 0.0)) {
          st[q] = VQPC_S_BREAKDOWN;
          act[q] = false;
        } else if (mit[q] < 1) {
          act[q] = false;
        }
      }
    }
    for (int j = 1; act[0] || act[1]; ++j) {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        if (!act[q]) continue;
        const double pAp = reduce(q, p1(q, j == 1), red[q]);
        if (!(pAp > 0.0)) {
          st[q] = VQPC_S_BREAKDOWN;
          act[q] = false;
          continue;
        }
        alpha[q] = rz[q] / pAp;
        const double rel = sqrt(reduce(q, p2(q), red[2 + q])) / norm_b[q];
        J[q] = j;
        rel_rec[q] = rel;
        if (rel < prm.eps) {
          st[q] = VQPC_S_CONVERGED;
          act[q] = false;
        }
      }
      if (!(act[0] || act[1])) break;
      double rzp[2];
      sweeps(rzp, act[0], act[1]);
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        if (!act[q]) continue;
        const double rz_next = reduce(q, rzp[q], red[4 + q]);
        if (!(rz_next > 0.0)) {
          st[q] = VQPC_S_BREAKDOWN;
          act[q] = false;
          continue;
        }
        beta[q] = rz_next / rz[q];
        rz[q] = rz_next;
        if (j >= mit[q]) act[q] = false;  // loop exhausted after its last preconditioner apply: MAX_ITER
      }
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      if (q >= gr.y) continue;
      if (t == 0) {
        prm.iters[gsv[q]] = J[q];
        prm.rel[gsv[q]] = rel_rec[q];
        prm.status[gsv[q]] = st[q];
      }
      const bool solved = st[q] == VQPC_S_CONVERGED || st[q] == VQPC_S_MAX_ITER || st[q] == VQPC_S_BREAKDOWN;
      if (prm.x_out && solved) {
        double* xo = prm.x_out + static_cast<size_t>(gsv[q]) * n;
        for (int l = 0; l < g.L; ++l) {
          const int a = wf_addr(g, l, t);
          if (a >= 0) xo[t * m + (l - t)] = Xb[q][xc[q]][a];
        }
      }
    }
    __syncthreads();
  }
}

}  // namespace vqpc
