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

#include <vector>

#include "kernels.cuh"
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
// Grid-stride and software-pipelined: a thread computes point gp while the
// traces of its next point (gp + stride) and the record of the one after are
// in flight, so the dependent record -> trace loads never sit on the critical
// path.
__device__ __forceinline__ void face_load(const FaceParams& P, const int4& r, double* qL, double* qR,
                                          unsigned long long pol)
{
    const int nL = r.w & 1023, nR = (r.w >> 10) & 1023;
    if (r.x >= 0) {
#pragma unroll
        for (int v = 0; v < NV; ++v) qL[v] = ld_hint(P.q + r.x + v * nL, pol);
    }
    if (r.y >= 0) {
#pragma unroll
        for (int v = 0; v < NV; ++v) qR[v] = ld_hint(P.q + r.y + v * nR, pol);
    }
}

__global__ void __launch_bounds__(FACE_BS, FACE_MINB) k_face(FaceParams P)
{
    const unsigned long long pol_last = l2_policy_last();
    const int stride = gridDim.x * FACE_BS;
    int gp = blockIdx.x * FACE_BS + threadIdx.x;
    const int4 none = make_int4(-1, -1, 0, 0);
    int4 r = gp < P.npts ? __ldg(P.fcta + gp) : none;
    int4 rn = gp + stride < P.npts ? __ldg(P.fcta + gp + stride) : none;
    double qL[NV], qR[NV];
    face_load(P, r, qL, qR, pol_last);
    for (; gp < P.npts; gp += stride) {
        const int4 rnn = gp + 2 * stride < P.npts ? __ldg(P.fcta + gp + 2 * stride) : none;
        double qLn[NV], qRn[NV];
        face_load(P, rn, qLn, qRn, pol_last);  // traces of the next point
        const int d = (r.w >> 20) & 3, kind = (r.w >> 22) & 3;
        const int nf = ((r.w >> 24) & 127) + 1;
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
        r = rn;
        rn = rnn;
#pragma unroll
        for (int v = 0; v < NV; ++v) { qL[v] = qLn[v]; qR[v] = qRn[v]; }
    }
}

// ---------------------------------------------------------------------------
// Mortar faces (unequal tangential orders, reading A6), v3: one CTA per face.
// Traces of both sides are interpolated to the mortar grid M_t = max(L_t, R_t)
// (two tensor passes), the Roe flux is evaluated at the mortar points, and the
// exact L2 projection (two passes) returns it to each side.  All 2-D arrays
// are zero-padded 9 x 9 per variable and the small 1-D operators zero-padded
// 9 x 9 in shared memory, so every contraction is a fixed 9-term unrolled sum
// of independent shared loads (no runtime-length dependent chains).
// ---------------------------------------------------------------------------
constexpr int MT_BS = 128;
constexpr int MT_A = NV * 81;  // one padded 5 x 9 x 9 array

// Mortar operators for side order ns < mortar order mm (1 <= ns < mm <= 8),
// zero padded 9 x 9: [pair][0] interpolation T^{ns->mm} ((mm+1) x (ns+1)),
// [pair][1] exact L2 projection P^{mm->ns} ((ns+1) x (mm+1)); pair =
// (mm-1)(mm-2)/2 + ns - 1.  36 KB of __constant__ memory, read warp-uniformly
// (constant-bank operands of the DFMAs).
constexpr int MT_PAIRS = 28;
static __constant__ double c_mop[MT_PAIRS][162];

__host__ __device__ constexpr int mt_pair(int ns, int mm) { return (mm - 1) * (mm - 2) / 2 + ns - 1; }

static inline void mortar_build_ops(const Tables* t, std::vector<double>& h)
{
    h.assign(MT_PAIRS * 2 * 81, 0.0);
    for (int mm = 2; mm <= NMAX; ++mm)
        for (int ns = 1; ns < mm; ++ns) {
            double* T = &h[(mt_pair(ns, mm) * 2 + 0) * 81];
            double* Pj = &h[(mt_pair(ns, mm) * 2 + 1) * 81];
            for (int row = 0; row <= mm; ++row)
                for (int col = 0; col <= ns; ++col) T[row * 9 + col] = t->T[ns][mm][row * (ns + 1) + col];
            for (int row = 0; row <= ns; ++row)
                for (int col = 0; col <= mm; ++col) Pj[row * 9 + col] = t->P[mm][ns][row * (mm + 1) + col];
        }
}

// One tensor pass over a padded [v][b*9 + a] array, thread l < 5 nl owns line (v, r):
//   along a: out[v][r*9 + i] = sum_{a<9} A[i*9 + a] in[v][r*9 + a]
//   along b: out[v][j*9 + r] = sum_{b<9} A[j*9 + b] in[v][b*9 + r]
// for outputs i (j) < ni.  A is zero padded beyond the input extent, so the
// fixed 9-term sums are exact whatever finite values the padding holds (all
// shared buffers are zeroed once at kernel start and only ever hold finite
// values).
__device__ __forceinline__ void mt_lines(const double* __restrict__ A, const double* __restrict__ in,
                                         double* __restrict__ out, int ni, int nl, bool along_a, int l)
{
    if (l >= NV * nl) return;
    const int v = (l >= nl) + (l >= 2 * nl) + (l >= 3 * nl) + (l >= 4 * nl), r = l - v * nl;
    const int xs = along_a ? 1 : 9;
    const double* x0 = in + v * 81 + (along_a ? r * 9 : r);
    double* o = out + v * 81 + (along_a ? r * 9 : r);
    double x[9];
#pragma unroll
    for (int a = 0; a < 9; ++a) x[a] = x0[a * xs];
    for (int i = 0; i < ni; ++i) {
        double s = 0.0;
#pragma unroll
        for (int a = 0; a < 9; ++a) s = fma(A[i * 9 + a], x[a], s);
        o[i * xs] = s;
    }
}

__device__ __forceinline__ void bar_side(int side)
{
    asm volatile("bar.sync %0, 64;\n" ::"r"(side + 1) : "memory");
}

// Mortar faces (unequal tangential orders, reading A6), v5: persistent CTAs
// walking mortar faces, traces of face k+1 prefetched by cp.async into the
// second trace stage while face k is computed.  Per face: traces of both
// sides are interpolated to the mortar grid M_t = max(L_t, R_t) (two tensor
// passes; a pass is skipped where the side already has the mortar order:
// T^{M->M} = I), the Roe flux is evaluated at the mortar points, and the
// exact L2 projection (two passes, identity skipped likewise) returns it to
// each side.  Threads 0-63 work on side L, 64-127 on side R.
constexpr int MT_MINB = 6;

__device__ __forceinline__ void mt_unpack(int o, int* N) { N[0] = o & 15; N[1] = (o >> 4) & 15; N[2] = (o >> 8) & 15; }

__global__ void __launch_bounds__(MT_BS, MT_MINB) k_mortar3(MortarParams P, const MortarFace* items, int nitems, int* queue)
{
    __shared__ double TR[3][2][MT_A];  // [stage][side] traces (zero padded), faces k, k+1, k+2 in flight
    __shared__ double TM[2][MT_A];     // pass-A results (interpolation, then projection)
    __shared__ double QM[2][MT_A];     // pass-B results (mortar states, then projected fluxes)
    __shared__ double GM[MT_A];        // Roe flux on the mortar
    const int t = threadIdx.x;
    const int me = t >= 64, l = t & 63;  // side and line slot of this thread in the tensor passes
    const int G = gridDim.x;
    const int f0 = blockIdx.x;
    if (f0 >= nitems) return;

    for (int w = t; w < 6 * MT_A; w += MT_BS) (&TR[0][0][0])[w] = 0.0;  // padding: finite once and for all
    for (int w = t; w < 2 * MT_A; w += MT_BS) { (&TM[0][0])[w] = 0.0; (&QM[0][0])[w] = 0.0; }
    for (int w = t; w < MT_A; w += MT_BS) GM[w] = 0.0;
    __syncthreads();
    // this thread's side of face `it` into trace stage st: one (v, b) row per thread
    auto issue = [&](const MortarFace& it, int st) {
        int NS[3];
        mt_unpack(me ? it.ordR : it.ordL, NS);
        const int d = it.d, ta = d == 0 ? 1 : 0, tb = d == 2 ? 1 : 2;
        const int s1 = NS[ta] + 1, s2 = NS[tb] + 1;
        if (l >= NV * s2) return;
        const int v = (l >= s2) + (l >= 2 * s2) + (l >= 3 * s2) + (l >= 4 * s2), b = l - v * s2;
        const int st1 = NS[0] + 1, st2 = (NS[0] + 1) * (NS[1] + 1);
        const int sta = ta == 0 ? 1 : st1, stb = tb == 1 ? st1 : st2, std_ = d == 0 ? 1 : (d == 1 ? st1 : st2);
        const int n = st2 * (NS[2] + 1);
        const double* src = P.q + (me ? it.offR : it.offL) + (me == 0 ? NS[d] * std_ : 0) + v * n + b * stb;
        double* dst = TR[st][me] + v * 81 + b * 9;
        for (int a = 0; a < s1; ++a) cp_async8(dst + a, src + a * sta);
    };
    // faces: f0, f0 + G, f0 + 2G, then dynamically from a work counter (mortar
    // sizes vary: a static round robin leaves a long tail).  Traces run two
    // faces ahead (3 stages); face records one more; thread 0 fetches the
    // counter one further, so no latency of the chain is exposed.
    __shared__ int s_nn[2];
    int fcur = f0, f1 = f0 + G, f2 = f0 + 2 * G, pend = 3 * G;
    if (t == 0) pend = 3 * G + atomicAdd(queue, 1);
    MortarFace cur = items[f0];
    MortarFace n1 = cur, n2 = cur;
    if (f1 < nitems) n1 = items[f1];
    if (f2 < nitems) n2 = items[f2];
    issue(cur, 0);
    asm volatile("cp.async.commit_group;\n" ::);
    if (f1 < nitems) issue(n1, 1);
    asm volatile("cp.async.commit_group;\n" ::);
    for (int k = 0;; ++k) {
        if (fcur >= nitems) break;
        if (t == 0) {
            s_nn[k & 1] = pend;  // face k+3
            pend = 3 * G + atomicAdd(queue, 1);
        }
        asm volatile("cp.async.wait_group 1;\n" ::: "memory");  // face k landed (k+1 may be in flight)
        __syncthreads();  // ... for every thread; face k-1 fully consumed
        const int f3 = s_nn[k & 1];
        MortarFace n3 = n2;
        if (f3 < nitems) n3 = items[f3];
        if (f2 < nitems) issue(n2, (k + 2) % 3);
        asm volatile("cp.async.commit_group;\n" ::);

        const int d = cur.d;
        const int ta = d == 0 ? 1 : 0, tb = d == 2 ? 1 : 2;
        int NL[3], NR[3];
        mt_unpack(cur.ordL, NL);
        mt_unpack(cur.ordR, NR);
        const int M1 = max(NL[ta], NR[ta]), M2 = max(NL[tb], NR[tb]);
        const int m1 = M1 + 1, m2 = M2 + 1;
        const int sa_me = (me ? NR[ta] : NL[ta]) + 1, sb_me = (me ? NR[tb] : NL[tb]) + 1;
        const bool ia = sa_me < m1, ib = sb_me < m2;
        const bool ia0 = NL[ta] < M1, ia1 = NR[ta] < M1, ib0 = NL[tb] < M2, ib1 = NR[tb] < M2;
        const double* opA = c_mop[mt_pair(sa_me - 1, M1)];
        const double* opB = c_mop[mt_pair(sb_me - 1, M2)];
        double* TRs = &TR[k % 3][0][0];
        // side traces -> mortar: along a where s_a < m1, then along b where s_b < m2
        if (ia) mt_lines(opA, TRs + me * MT_A, TM[me], m1, sb_me, true, l);
        bar_side(me);
        const double* Xme = ia ? TM[me] : TRs + me * MT_A;
        if (ib) mt_lines(opB, Xme, QM[me], m2, m1, false, l);
        __syncthreads();
        // Roe flux at the mortar points (0 outside the m1 x m2 grid)
        if (t < 81) {
            const double* Y0 = ib0 ? QM[0] : (ia0 ? TM[0] : TRs);
            const double* Y1 = ib1 ? QM[1] : (ia1 ? TM[1] : TRs + MT_A);
            const int j = t / 9, i = t - j * 9;
            double Gf[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) Gf[v] = 0.0;
            if (i < m1 && j < m2) {
                double qL[NV], qR[NV];
#pragma unroll
                for (int v = 0; v < NV; ++v) { qL[v] = Y0[v * 81 + t]; qR[v] = Y1[v * 81 + t]; }
                if (P.ph.flux == 1) {
                    const double nrm[3] = {d == 0 ? 1.0 : 0.0, d == 1 ? 1.0 : 0.0, d == 2 ? 1.0 : 0.0};
                    llf_flux(qL, qR, nrm, P.ph.gamma, Gf);
                } else {
                    roe_axis_q(d, qL, qR, P.ph.gm1, Gf);
                }
            }
#pragma unroll
            for (int v = 0; v < NV; ++v) GM[v * 81 + t] = Gf[v];
        }
        __syncthreads();
        // exact L2 projection back to each side (identity passes skipped)
        if (ia) mt_lines(opA + 81, GM, TM[me], sa_me, m2, true, l);
        bar_side(me);
        const double* Zme = ia ? TM[me] : GM;
        if (ib) mt_lines(opB + 81, Zme, QM[me], sb_me, sa_me, false, l);
        bar_side(me);
        if (l < NV * sb_me) {  // one (v, b) row per thread
            const double* W = ib ? QM[me] : Zme;
            const int v = (l >= sb_me) + (l >= 2 * sb_me) + (l >= 3 * sb_me) + (l >= 4 * sb_me), b = l - v * sb_me;
            double* dst = P.mortarG + (me ? cur.moR : cur.moL) + (v * sb_me + b) * sa_me;
            const double* src = W + v * 81 + b * 9;
            for (int a = 0; a < sa_me; ++a) dst[a] = src[a];
        }
        fcur = f1;
        f1 = f2;
        f2 = f3;
        cur = n1;
        n1 = n2;
        n2 = n3;
    }
}

}  // namespace dgtau
