// face.cuh -- conforming-face Riemann fluxes, computed ONCE per face point.
//
// The surface integral of the DGSEM needs at every
// point of a face the numerical flux G = Roe(q_L, q_R; e_d) (reading A7,
// Lax-Friedrichs flag), shared by the two elements of the face.  Computing it
// inside the element kernel would evaluate it twice (once per side); this
// kernel evaluates it once, one thread per face point, into the flux buffer,
// where the element kernel (residual_t.cuh) picks the six face blocks of an
// element up with bulk copies.  Mortar faces (unequal tangential orders,
// reading A6) are handled by k_mortar2 into the same buffer; boundary faces
// (wall / far field, reading A10) here with a ghost state.
// Included by dgtau.cu only.
#pragma once

#include "residual_t.cuh"

namespace dgtau {

// Roe flux (no entropy fix, reading A7) for the axis normal e_d from
// the two conserved states; every reciprocal / square root comes from three
// rsqrt and one rcp (1/rho = (1/sqrt rho)^2, 1/c^2 = (1/c)^2).
__device__ __forceinline__ double sel3(int d, double a, double b, double c) { return d == 0 ? a : (d == 1 ? b : c); }

// Roe flux (no entropy fix, reading A7) for the axis normal e_d (d at
// run time, branch-free: points of one warp may lie on faces of different
// axes) from the two conserved states; every reciprocal / square root comes
// from three rsqrt and one rcp (1/rho = (1/sqrt rho)^2, 1/c^2 = (1/c)^2).
__device__ __forceinline__ void roe_axis_q(int d, const double* qL, const double* qR, double gm1, double* F)
{
    const double rL = rsqrt_nr(qL[0]), rR = rsqrt_nr(qR[0]);
    const double sL = qL[0] * rL, sR = qR[0] * rR;  // sqrt(rho)
    const double irL = rL * rL, irR = rR * rR;      // 1/rho
    double uL[3], uR[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) { uL[k] = qL[1 + k] * irL; uR[k] = qR[1 + k] * irR; }
    const double pL = gm1 * fma(-0.5, qL[1] * uL[0] + qL[2] * uL[1] + qL[3] * uL[2], qL[4]);
    const double pR = gm1 * fma(-0.5, qR[1] * uR[0] + qR[2] * uR[1] + qR[3] * uR[2], qR[4]);
    const double HL = (qL[4] + pL) * irL, HR = (qR[4] + pR) * irR;
    const double wl = sL * rcp_nr(sL + sR), wr = 1.0 - wl;
    double u[3], du[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) { u[k] = fma(wl, uL[k], wr * uR[k]); du[k] = uR[k] - uL[k]; }
    const double H = fma(wl, HL, wr * HR);
    const double uu = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
    const double c2 = gm1 * fma(-0.5, uu, H);
    const double rc = rsqrt_nr(c2);
    const double c = c2 * rc, ic2 = rc * rc;
    const double un = sel3(d, u[0], u[1], u[2]), dun = sel3(d, du[0], du[1], du[2]);
    const double uLd = sel3(d, uL[0], uL[1], uL[2]), uRd = sel3(d, uR[0], uR[1], uR[2]);
    const double mLd = qL[0] * uLd, mRd = qR[0] * uRd;
    const double rho = sL * sR;
    const double dp = pR - pL;
    const double rcd = rho * c * dun;
    const double a1 = 0.5 * (dp - rcd) * ic2, a5 = 0.5 * (dp + rcd) * ic2;
    const double a2 = (qR[0] - qL[0]) - dp * ic2;
    const double w1 = fabs(un - c) * a1, w5 = fabs(un + c) * a5, l2 = fabs(un);
    const double w15 = w1 + w5, l2r = l2 * rho;
    F[0] = 0.5 * ((mLd + mRd) - (w15 + l2 * a2));
    const double fn = pL + pR, dn = fma(c, w5 - w1, -l2r * dun);  // normal-momentum extras
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double fk = fma(qL[1 + k], uLd, qR[1 + k] * uRd) + (k == d ? fn : 0.0);
        const double dk = fma(w15 + l2 * a2, u[k], l2r * du[k]) + (k == d ? dn : 0.0);
        F[1 + k] = 0.5 * (fk - dk);
    }
    const double udu = u[0] * du[0] + u[1] * du[1] + u[2] * du[2];
    const double fe = fma(HL, mLd, HR * mRd);
    const double de = fma(w15, H, fma(un * c, w5 - w1, l2 * fma(a2 * 0.5, uu, rho * fma(-un, dun, udu))));
    F[4] = 0.5 * (fe - de);
}

// One thread per face point; its record (one 16-byte load) gives the trace
// positions of both sides in q, the flux position in G and the sizes.
__global__ void __launch_bounds__(FACE_BS, 8) k_face(FaceParams P)
{
    const int gp = blockIdx.x * FACE_BS + threadIdx.x;
    if (gp >= P.npts) return;
    const int4 r = __ldg(P.fcta + gp);
    const unsigned long long pol_last = l2_policy_last();
    const int nL = r.w & 1023, nR = (r.w >> 10) & 1023, d = (r.w >> 20) & 3, kind = (r.w >> 22) & 3;
    const int nf = ((r.w >> 24) & 127) + 1;
    double qL[NV], qR[NV];
    if (r.x >= 0) {
#pragma unroll
        for (int v = 0; v < NV; ++v) qL[v] = ld_hint(P.q + r.x + v * nL, pol_last);
    }
    if (r.y >= 0) {
#pragma unroll
        for (int v = 0; v < NV; ++v) qR[v] = ld_hint(P.q + r.y + v * nR, pol_last);
    }
    if (kind >= 2) {
        if (r.x < 0) ghost_state(qR, kind == 2 ? -1 : -2, P.ph, qL);
        else ghost_state(qL, kind == 2 ? -1 : -2, P.ph, qR);
    }
    double G[NV];
    if (P.ph.flux == 1) {
        const double nrm[3] = {d == 0 ? 1.0 : 0.0, d == 1 ? 1.0 : 0.0, d == 2 ? 1.0 : 0.0};
        llf_flux(qL, qR, nrm, P.ph.gamma, G);
    } else {
        roe_axis_q(d, qL, qR, P.ph.gm1, G);
    }
    double* o = P.G + r.z;
#pragma unroll
    for (int v = 0; v < NV; ++v) st_hint(o + v * nf, G[v], pol_last);
}

}  // namespace dgtau
