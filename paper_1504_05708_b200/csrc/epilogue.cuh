// Row epilogues shared by every pass kernel (dense, CSR): identical arithmetic
// whatever produced the row value, so formats and shardings agree bit for bit
// on the vector part of the step.
#pragma once

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "duquad_internal.h"

namespace dq {

// Programmatic dependent launch (PDL).  A kernel launched with the programmatic-serialization
// attribute (launch_ex, LaunchCfg.pdl) may start while the previous kernel of the stream drains:
// before pdl_wait() it may only read data no kernel of the solve writes (the stored matrices);
// every read of an iterate / flag and every global write comes after it.  Without the attribute
// griddepcontrol.wait returns at once.  pdl_trigger() lets the next kernel's CTAs be scheduled as
// soon as resources free up.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// [v]_K per row tag: ZERO -> 0, NONPOS -> min(v, 0)
// (select forms: a NaN maps to 0 exactly as fmin/fmax(NaN, 0) would, in 3 SASS instead of ~14)
__device__ __forceinline__ double proj_K(double v, uint8_t c) {
    return c == DUQUAD_CONE_NONPOS && v < 0.0 ? v : 0.0;
}
// projection onto the polar cone K° (multiplier sign set): ZERO -> v, NONPOS -> max(v, 0)
__device__ __forceinline__ double proj_polar(double v, uint8_t c) {
    return c != DUQUAD_CONE_NONPOS || v > 0.0 ? v : 0.0;
}

__device__ __forceinline__ double warp_sum(double s) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return s;
}

template <int GS>
__device__ __forceinline__ double group_sum(double s) {
#pragma unroll
    for (int o = GS / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return s;
}

// ------------------------------------------------------------------ pass A
struct EpiA {
    double g, mu, lp, lh;
    uint8_t c;
};

struct OuterA {
    int dual;
    double beta_out;
    int mu_hat;      // DGM dual averaging: mu := the updated average
    double lhat_w;   // weight of this step's lambda in the running dual average (0: none)
};

__device__ __forceinline__ OuterA outer_a(const PassAArgs &a, int mode) {
    OuterA o{0, 0.0, 0, 0.0};
    if (mode == MODE_SOLVE && a.first_inner) {
        const OuterParam op = a.ops[*a.d_j];
        o.dual = op.dual_update;
        o.beta_out = op.beta_out;
        if (a.lam_hat) {
            o.mu_hat = op.mu_hat;
            o.lhat_w = op.lhat_w;
        }
    }
    return o;
}

// DGM dual averaging: lam_hat_j = lam_hat_{j-1} + (lambda^j - lam_hat_{j-1}) / (j+1), the
// running form of (1/(j+1)) sum_{i<=j} lambda^i; on the final averaging step mu := lam_hat.
__device__ __forceinline__ double dual_average(double lh, double lam, double m, const OuterA &o, double &lh_new) {
    lh_new = lh + o.lhat_w * (lam - lh);
    return o.mu_hat ? lh_new : m;
}

__device__ __forceinline__ EpiA epi_a_load(const PassAArgs &a, int mode, int64_t row, const OuterA &o) {
    EpiA e{0.0, 0.0, 0.0, 0.0, 0};
    if (mode == MODE_SOLVE && row >= a.nq) {
        const int64_t k = row - a.nq;
        e.g = a.g[k];
        e.mu = a.mu[k];
        e.c = a.cone[k];
        if (o.dual) e.lp = a.lam_prev[k];
        if (o.lhat_w != 0.0) e.lh = a.lam_hat[k];
    }
    return e;
}

// The DFOM step of one G row with the slack s(u, mu), given r = G y + g
// at y == u_bar^{j-1}: returns mu^{j+1} and sets lambda^j.
__device__ __forceinline__ double dfom_row(double r, double mu, double lp, uint8_t c, double rho, double step,
                                           int project_dual, double beta_out, double &lam) {
    const double sl = rho > 0.0 ? proj_K(r + mu / rho, c) : 0.0;
    lam = mu + step * (r - sl);
    if (project_dual && c == DUQUAD_CONE_NONPOS) lam = fmax(lam, 0.0);
    return lam + beta_out * (lam - lp);
}

// s = (row of [Q;G]) . y
__device__ __forceinline__ void epi_a_store(const PassAArgs &a, int mode, int64_t row, double s,
                                            const EpiA &e, const OuterA &o) {
    if (row < a.nq) {
        a.qy[row] = s;
        return;
    }
    const int64_t k = row - a.nq;
    if (mode == MODE_LIN) {
        a.w[k] = a.lin_coef * s;
        return;
    }
    const double r = s + e.g;                      // r = G y + g
    double m = e.mu;
    if (o.dual) {
        double lam;
        m = dfom_row(r, e.mu, e.lp, e.c, a.rho, a.step, a.project_dual, o.beta_out, lam);
        if (o.lhat_w != 0.0) {
            double lh;
            m = dual_average(e.lh, lam, m, o, lh);
            a.lam_hat[k] = lh;
        }
        a.lam_prev[k] = lam;
        a.mu[k] = m;
        if (a.h) a.h[k] = m + a.rho * e.g;   // batched: the constant part of the next w's
    }
    // multiplier term of grad L_rho: [mu + rho r]_{K°} (rho > 0), mu (rho = 0); on the
    // equality-QP H path the constant part mu + rho g (the rho G'G u part is inside H)
    a.w[k] = a.w_plus_g ? m + a.rho * e.g : a.rho > 0.0 ? proj_polar(m + a.rho * r, e.c) : m;
}

// ------------------------------------------------------------------ pass B
struct EpiB {
    double qy, q, lb, ub, x, y, xh;
};

__device__ __forceinline__ double avg_weight(const PassBArgs &b, int mode) {
    return (mode == MODE_SOLVE && b.last_inner) ? b.ops[*b.d_j].avg_w : 0.0;
}

__device__ __forceinline__ EpiB epi_b_load(const PassBArgs &b, int mode, int64_t j, double avg_w) {
    EpiB e{0, 0, 0, 0, 0, 0, 0};
    if (mode == MODE_SOLVE || b.use_qy) e.qy = b.qy[j];
    if (mode == MODE_SOLVE) {
        e.q = b.q[j];
        if (b.box_uniform) {   // U = [lb, ub]^n with scalar bounds (c4's [-1, 1]): no per-row loads
            e.lb = b.lb_u;
            e.ub = b.ub_u;
        } else {
            e.lb = b.lb[j];
            e.ub = b.ub[j];
        }
        e.x = b.x[j];
        e.y = b.y[j];
        if (avg_w != 0.0) e.xh = b.xhat[j];
    }
    return e;
}

// t = (row j of G') . w
__device__ __forceinline__ void epi_b_store(const PassBArgs &b, int mode, int64_t j, double t, const EpiB &e,
                                            double avg_w) {
    if (mode == MODE_LIN) {
        b.out[j] = e.qy + t;
        return;
    }
    const double grad = (e.qy + e.q) + t;
    const double xn = fmin(fmax(e.y - grad / b.L_in, e.lb), e.ub);
    const double yn = b.last_inner ? xn : xn + b.beta_in * (xn - e.x);
    if (avg_w != 0.0) b.xhat[j] = e.xh + avg_w * (xn - e.xh);      // P:700-706 (running form)
    if (b.gm_sq) {                                                 // eps_in mode: ||y - x+||^2 terms
        const double dd = e.y - xn;
        b.gm_sq[j] = dd * dd;
    }
    b.x[j] = xn;
    b.y[j] = yn;
    if (!isfinite(xn) || !isfinite(yn)) *b.flag = 1;
}

}  // namespace dq
