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

__global__ void __launch_bounds__(FACE_BS) k_face(FaceParams P)
{
    const int gp = blockIdx.x * FACE_BS + threadIdx.x;
    if (gp >= P.npts) return;
    // face of point gp: binary search in [fcta[b], fcta[b+1]]
    int lo = P.fcta[blockIdx.x], hi = P.fcta[blockIdx.x + 1];
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (__ldg(P.fpt + mid) <= gp) lo = mid;
        else hi = mid - 1;
    }
    const FaceItem& fi = P.faces[lo];
    const int pt = gp - __ldg(P.fpt + lo);
    const int nta = fi.nta;
    const int ta = pt % nta, tb = pt / nta;
    double qL[NV], qR[NV];
    if (fi.offL >= 0) {
        const double* s = P.q + fi.offL + (fi.baseL + ta * fi.saL + tb * fi.sbL);
        const int n = fi.nL;
#pragma unroll
        for (int v = 0; v < NV; ++v) qL[v] = __ldg(s + v * n);
    }
    if (fi.offR >= 0) {
        const double* s = P.q + fi.offR + (fi.baseR + ta * fi.saR + tb * fi.sbR);
        const int n = fi.nR;
#pragma unroll
        for (int v = 0; v < NV; ++v) qR[v] = __ldg(s + v * n);
    }
    if (fi.kind >= 2) {
        if (fi.offL < 0) ghost_state(qR, fi.kind == 2 ? -1 : -2, P.ph, qL);
        else ghost_state(qL, fi.kind == 2 ? -1 : -2, P.ph, qR);
    }
    const int d = fi.d;
    double G[NV];
    if (P.ph.flux == 1) {
        const double nrm[3] = {d == 0 ? 1.0 : 0.0, d == 1 ? 1.0 : 0.0, d == 2 ? 1.0 : 0.0};
        llf_flux(qL, qR, nrm, P.ph.gamma, G);
    } else {
        const double gm1 = P.ph.gm1;
        const double irL = rcp_nr(qL[0]), irR = rcp_nr(qR[0]);
        const double pL = gm1 * (qL[4] - 0.5 * irL * (qL[1] * qL[1] + qL[2] * qL[2] + qL[3] * qL[3]));
        const double pR = gm1 * (qR[4] - 0.5 * irR * (qR[1] * qR[1] + qR[2] * qR[2] + qR[3] * qR[3]));
        if (d == 0) roe_axis<0>(qL, irL, pL, qR, irR, pR, P.ph.gamma, G);
        else if (d == 1) roe_axis<1>(qL, irL, pL, qR, irR, pR, P.ph.gamma, G);
        else roe_axis<2>(qL, irL, pL, qR, irR, pR, P.ph.gamma, G);
    }
    double* o = P.G + fi.goff + pt;
    const int nf = fi.nf;
#pragma unroll
    for (int v = 0; v < NV; ++v) o[v * nf] = G[v];
}

}  // namespace dgtau
