// curved.cuh -- generic (runtime-order) sm_100a kernels for curved elements
// and the compressible Navier-Stokes equations with BR1 (cfg4 / cfg5).
//
// PAPER.md: P:106-126 (advection-diffusion split, first-order system with
// g = grad q), P:129-145 (eqs DGSEMsystem:1-2: weak form of the flux
// divergence and of the BR1 lifting of the gradient), P:144 (Jacobians of the
// geometry transformation), P:472 (Roe advective flux, BR1 diffusive flux).
// Readings A6 (mortars, metric from the L side's geometry), A8 (gradients of
// the conserved variables), A9 (nondimensionalisation), A10 (wall / far-field
// states), A11 (CFL / DFL), as in DESIGN.md.
//
// Metric terms (cross-product form, exact for the extruded meshes here):
//   Ja^1 = x_eta x x_zeta, Ja^2 = x_zeta x x_xi, Ja^3 = x_xi x x_eta,
//   J = x_xi . (x_eta x x_zeta),
// with x the interpolant at the solution nodes of the geometry polynomial and
// derivatives by D^N (as the oracle).  Per node 10 doubles: Ja^d_k at
// 3d+k, J at 9 (offset 2 x the state offset of the element).
// Gradient field: 15 doubles per node, [k][v] = d q_v / d x_k (offset 3 x).
//
// Strong form on the device (equal to the weak form for GL nodes):
//   J g_k = sum_d D^d (Ja^d_k q) + lifting of (qhat Ja^d_k|_face - q Ja^d_k|_own)/w
//   J Qdot = -sum_d D^d Ft^d - lifting of (G - Ft^d_own)/w,
//   Ft^d = Ja^d . (f^a - f^nu),
//   G = |Ja_f| Roe(q_L, q_R; n) - 1/2 (f^nu_L + f^nu_R) . Ja_f   (BR1 average).
#pragma once

#include "common.cuh"

namespace dgtau {

constexpr int CBS = 128;  // threads per CTA of the curved kernels (cfg5 elements: ~108 nodes)

struct CurvedMesh {
    const double* geo;   // [E][3][ng] geometry nodes
    int g1, g2, g3, ng;  // geometry orders and node count
};

// viscous flux along vector a (f^nu . a), A8-A9: stresses from conserved gradients
__device__ __forceinline__ void visc_dot(const double* q, const double* g /*[15] k*5+v*/, double ax, double ay,
                                         double az, const PhysDev& ph, double* fv)
{
    const double gam = ph.gamma, mu = ph.mu;
    const double ir = inv_pos(q[0]);
    const double u = q[1] * ir, v = q[2] * ir, w = q[3] * ir;
    const double p = (gam - 1.0) * (q[4] - 0.5 * q[0] * (u * u + v * v + w * w));
    const double T = p * ir;
    double du[3][3], dT[3];  // du[i][j] = d u_i / d x_j
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        const double* gj = g + 5 * j;
        du[0][j] = (gj[1] - u * gj[0]) * ir;
        du[1][j] = (gj[2] - v * gj[0]) * ir;
        du[2][j] = (gj[3] - w * gj[0]) * ir;
        const double dp = (gam - 1.0) * (gj[4] - (u * gj[1] + v * gj[2] + w * gj[3]) + 0.5 * (u * u + v * v + w * w) * gj[0]);
        dT[j] = (dp - T * gj[0]) * ir;
    }
    const double div = du[0][0] + du[1][1] + du[2][2];
    const double kappa = ph.kappa;
    const double a[3] = {ax, ay, az};
    double ta[3];  // tau . a
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < 3; ++j) s += mu * (du[i][j] + du[j][i] - (i == j ? 2.0 / 3.0 * div : 0.0)) * a[j];
        ta[i] = s;
    }
    fv[0] = 0.0;
    fv[1] = ta[0];
    fv[2] = ta[1];
    fv[3] = ta[2];
    fv[4] = u * ta[0] + v * ta[1] + w * ta[2] + kappa * (dT[0] * ax + dT[1] * ay + dT[2] * az);
}

// visc_dot split in two: the node's stress tensor and temperature gradient
// once (from q and its gradient), then the flux along any vector a with the
// same operations in the same order as visc_dot, except 1/rho: IEEE division
// here (rcp_nr measured slower in k_ns_res), inv_pos in the face kernels
struct ViscNode {
    double T[3][3];   // mu (du_i/dx_j + du_j/dx_i - 2/3 div delta_ij)
    double dT[3];     // grad T
    double u[3];
    double kappa;
};

__device__ __forceinline__ void visc_node(const double* q, const double* g, const PhysDev& ph, ViscNode& V)
{
    const double gam = ph.gamma, mu = ph.mu;
    const double ir = 1.0 / q[0];
    const double u = q[1] * ir, v = q[2] * ir, w = q[3] * ir;
    const double p = (gam - 1.0) * (q[4] - 0.5 * q[0] * (u * u + v * v + w * w));
    const double Tt = p * ir;
    double du[3][3];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        const double* gj = g + 5 * j;
        du[0][j] = (gj[1] - u * gj[0]) * ir;
        du[1][j] = (gj[2] - v * gj[0]) * ir;
        du[2][j] = (gj[3] - w * gj[0]) * ir;
        const double dp = (gam - 1.0) * (gj[4] - (u * gj[1] + v * gj[2] + w * gj[3]) + 0.5 * (u * u + v * v + w * w) * gj[0]);
        V.dT[j] = (dp - Tt * gj[0]) * ir;
    }
    const double div = du[0][0] + du[1][1] + du[2][2];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) V.T[i][j] = mu * (du[i][j] + du[j][i] - (i == j ? 2.0 / 3.0 * div : 0.0));
    V.u[0] = u;
    V.u[1] = v;
    V.u[2] = w;
    V.kappa = ph.kappa;
}

__device__ __forceinline__ void visc_along(const ViscNode& V, double ax, double ay, double az, double* fv)
{
    const double a[3] = {ax, ay, az};
    double ta[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < 3; ++j) s += V.T[i][j] * a[j];
        ta[i] = s;
    }
    fv[0] = 0.0;
    fv[1] = ta[0];
    fv[2] = ta[1];
    fv[3] = ta[2];
    fv[4] = V.u[0] * ta[0] + V.u[1] * ta[1] + V.u[2] * ta[2] + V.kappa * (V.dT[0] * ax + V.dT[1] * ay + V.dT[2] * az);
}

// advective flux along vector a
__device__ __forceinline__ void adv_dot(const double* q, double ax, double ay, double az, double gm1, double* f)
{
    const double ir = 1.0 / q[0];
    const double p = gm1 * (q[4] - 0.5 * ir * (q[1] * q[1] + q[2] * q[2] + q[3] * q[3]));
    const double ua = (q[1] * ax + q[2] * ay + q[3] * az) * ir;
    f[0] = q[0] * ua;
    f[1] = q[1] * ua + p * ax;
    f[2] = q[2] * ua + p * ay;
    f[3] = q[3] * ua + p * az;
    f[4] = (q[4] + p) * ua;
}

// Ft = a . (f^a - f^nu)
__device__ __forceinline__ void contra_flux(const double* q, const double* g, double ax, double ay, double az,
                                            const PhysDev& ph, double* F)
{
    adv_dot(q, ax, ay, az, ph.gm1, F);
    if (ph.physics == 1) {
        double fv[NV];
        visc_dot(q, g, ax, ay, az, ph, fv);
#pragma unroll
        for (int v = 0; v < NV; ++v) F[v] -= fv[v];
    }
}

// ---------------------------------------------------------------------------
// Double-double arithmetic (error-free transformations) for the metric terms:
// the coordinates are O(20) while elements are O(0.02..2) and D amplifies
// rounding by O(N^2), so a plain fp64 evaluation loses ~1e-13 relative in
// Ja; the cfg4 state (free stream + 1e-3 noise) makes the residual sensitive
// to that.  Evaluated in dd and rounded once, the metrics equal the
// correctly rounded values (as the long double oracle's).
// ---------------------------------------------------------------------------
struct dd {
    double hi, lo;
};
__device__ __forceinline__ dd two_sum(double a, double b)
{
    const double s = a + b;
    const double bb = s - a;
    return {s, (a - (s - bb)) + (b - bb)};
}
__device__ __forceinline__ dd dd_add(dd a, dd b)
{
    dd s = two_sum(a.hi, b.hi);
    const double lo = s.lo + a.lo + b.lo;
    return two_sum(s.hi, lo);
}
__device__ __forceinline__ dd dd_mul(dd a, dd b)
{
    const double p = a.hi * b.hi;
    const double e = fma(a.hi, b.hi, -p);
    const double lo = e + (a.hi * b.lo + a.lo * b.hi);
    return two_sum(p, lo);
}
__device__ __forceinline__ dd dd_neg(dd a) { return {-a.hi, -a.lo}; }
__device__ __forceinline__ dd mkdd(double a) { return {a, 0.0}; }

// Element geometry at orders (o1,o2,o3): X = T^{g->o} Xgeo (3 x no, dd in
// smem), then metrics via D^o (cross-product form) rounded to Mout[c*no+node].
__device__ void element_metrics(const CurvedMesh& cm, int e, int o1, int o2, int o3, const TablesDD* tdd, dd* Xs,
                                double* Mout)
{
    const int no = o1 * o2 * o3;
    const int ga = cm.g1 + 1, gb = cm.g2 + 1;
    const double* G = cm.geo + (long long)e * 3 * cm.ng;
    for (int t = threadIdx.x; t < no; t += blockDim.x) {
        int i, j, k;
        node_ijk(t, o1, o2, i, j, k);
        dd x[3] = {mkdd(0.0), mkdd(0.0), mkdd(0.0)};
        for (int c = 0; c <= cm.g3; ++c)
            for (int b = 0; b <= cm.g2; ++b)
                for (int a = 0; a <= cm.g1; ++a) {
                    const int i1 = i * ga + a, i2 = j * gb + b, i3 = k * (cm.g3 + 1) + c;
                    const dd w1 = {tdd->Thi[cm.g1][o1 - 1][i1], tdd->Tlo[cm.g1][o1 - 1][i1]};
                    const dd w2 = {tdd->Thi[cm.g2][o2 - 1][i2], tdd->Tlo[cm.g2][o2 - 1][i2]};
                    const dd w3 = {tdd->Thi[cm.g3][o3 - 1][i3], tdd->Tlo[cm.g3][o3 - 1][i3]};
                    const dd wgt = dd_mul(dd_mul(w1, w2), w3);
                    const int gi = a + ga * (b + gb * c);
                    for (int q = 0; q < 3; ++q) x[q] = dd_add(x[q], dd_mul(wgt, mkdd(__ldg(G + q * cm.ng + gi))));
                }
        Xs[t] = x[0];
        Xs[no + t] = x[1];
        Xs[2 * no + t] = x[2];
    }
    __syncthreads();
    for (int t = threadIdx.x; t < no; t += blockDim.x) {
        int i, j, k;
        node_ijk(t, o1, o2, i, j, k);
        dd dx[3][3];  // dx[dd][c] = d x_c / d xi_dd
        for (int c = 0; c < 3; ++c) {
            const dd* X = Xs + c * no;
            dd s0 = mkdd(0.0), s1 = mkdd(0.0), s2 = mkdd(0.0);
            for (int m = 0; m < o1; ++m) {
                const dd Dv = {tdd->Dhi[o1 - 1][i * o1 + m], tdd->Dlo[o1 - 1][i * o1 + m]};
                s0 = dd_add(s0, dd_mul(Dv, X[m + o1 * (j + o2 * k)]));
            }
            for (int m = 0; m < o2; ++m) {
                const dd Dv = {tdd->Dhi[o2 - 1][j * o2 + m], tdd->Dlo[o2 - 1][j * o2 + m]};
                s1 = dd_add(s1, dd_mul(Dv, X[i + o1 * (m + o2 * k)]));
            }
            for (int m = 0; m < o3; ++m) {
                const dd Dv = {tdd->Dhi[o3 - 1][k * o3 + m], tdd->Dlo[o3 - 1][k * o3 + m]};
                s2 = dd_add(s2, dd_mul(Dv, X[i + o1 * (j + o2 * m)]));
            }
            dx[0][c] = s0;
            dx[1][c] = s1;
            dx[2][c] = s2;
        }
        const dd* xa = dx[0];
        const dd* xb = dx[1];
        const dd* xc = dx[2];
        // c = a x b in dd
        auto cross = [](const dd* a, const dd* b, dd* r) {
            r[0] = dd_add(dd_mul(a[1], b[2]), dd_neg(dd_mul(a[2], b[1])));
            r[1] = dd_add(dd_mul(a[2], b[0]), dd_neg(dd_mul(a[0], b[2])));
            r[2] = dd_add(dd_mul(a[0], b[1]), dd_neg(dd_mul(a[1], b[0])));
        };
        dd c1[3], c2[3], c3[3];
        cross(xb, xc, c1);
        cross(xc, xa, c2);
        cross(xa, xb, c3);
        for (int q = 0; q < 3; ++q) {
            Mout[q * no + t] = c1[q].hi + c1[q].lo;
            Mout[(3 + q) * no + t] = c2[q].hi + c2[q].lo;
            Mout[(6 + q) * no + t] = c3[q].hi + c3[q].lo;
        }
        const dd J = dd_add(dd_add(dd_mul(xa[0], c1[0]), dd_mul(xa[1], c1[1])), dd_mul(xa[2], c1[2]));
        Mout[9 * no + t] = J.hi + J.lo;
    }
    __syncthreads();
}


// one launch per size class: CTA b handles element perm[pbase + b]
struct SizeClass {
    int base, count, maxn;
};

struct MetParams {
    const int* perm;
    int pbase;
    CurvedMesh cm;
    const int* orders;
    const long long* off;  // state offsets (metrics at 2x)
    double* met;
    const TablesDD* tdd;
};

__global__ void __launch_bounds__(CBS) k_metrics(MetParams P)
{
    extern __shared__ double sm[];
    const int e = P.perm[P.pbase + blockIdx.x];
    const int o1 = P.orders[3 * e] + 1, o2 = P.orders[3 * e + 1] + 1, o3 = P.orders[3 * e + 2] + 1;
    const int no = o1 * o2 * o3;
    dd* Xs = reinterpret_cast<dd*>(sm);
    double* Ms = sm + 6 * no;
    element_metrics(P.cm, e, o1, o2, o3, P.tdd, Xs, Ms);
    double* out = P.met + 2 * P.off[e];
    for (int t = threadIdx.x; t < 10 * no; t += blockDim.x) out[t] = Ms[t];
}

// ---------------------------------------------------------------------------
// generic sweep helpers: acc[c][node] (+)= sum_m D^{o_d}[a][m] F[c][..m..]
// ---------------------------------------------------------------------------

// sum_m D[a][m] Fl[c*cs + m*stride] for the NC components c of a line, with
// the line length OD a compile-time constant (no predicated-off FMAs); two
// partial sums (even / odd m) for a shorter FMA chain
template <int OD, int NC, typename Op>
__device__ __forceinline__ void dsum_comps_t(const double* Dr, const double* Fl, int cs, int stride, Op op)
{
    double r[OD];
#pragma unroll
    for (int m = 0; m < OD; ++m) r[m] = Dr[m];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int m = 0; m < OD; m += 2) {
            s0 = fma(r[m], Fl[c * cs + m * stride], s0);
            if (m + 1 < OD) s1 = fma(r[m + 1], Fl[c * cs + (m + 1) * stride], s1);
        }
        op(c, s0 + s1);
    }
}

template <int NC, typename Op>
__device__ __forceinline__ void dsum_comps(int od, const double* Dr, const double* Fl, int cs, int stride, Op op)
{
    switch (od) {
        case 2: dsum_comps_t<2, NC>(Dr, Fl, cs, stride, op); break;
        case 3: dsum_comps_t<3, NC>(Dr, Fl, cs, stride, op); break;
        case 4: dsum_comps_t<4, NC>(Dr, Fl, cs, stride, op); break;
        case 5: dsum_comps_t<5, NC>(Dr, Fl, cs, stride, op); break;
        case 6: dsum_comps_t<6, NC>(Dr, Fl, cs, stride, op); break;
        case 7: dsum_comps_t<7, NC>(Dr, Fl, cs, stride, op); break;
        case 8: dsum_comps_t<8, NC>(Dr, Fl, cs, stride, op); break;
        default: dsum_comps_t<9, NC>(Dr, Fl, cs, stride, op); break;
    }
}

// as dsum_comps with ONE accumulator (sequential fma over m, the order of the
// coarse metric terms' reference loop)
template <int OD, int NC, typename Op>
__device__ __forceinline__ void dchain_comps_t(const double* Dr, const double* Fl, int cs, int stride, Op op)
{
    double r[OD];
#pragma unroll
    for (int m = 0; m < OD; ++m) r[m] = Dr[m];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        double s = 0.0;
#pragma unroll
        for (int m = 0; m < OD; ++m) s = fma(r[m], Fl[c * cs + m * stride], s);
        op(c, s);
    }
}

template <int NC, typename Op>
__device__ __forceinline__ void dchain_comps(int od, const double* Dr, const double* Fl, int cs, int stride, Op op)
{
    switch (od) {
        case 2: dchain_comps_t<2, NC>(Dr, Fl, cs, stride, op); break;
        case 3: dchain_comps_t<3, NC>(Dr, Fl, cs, stride, op); break;
        case 4: dchain_comps_t<4, NC>(Dr, Fl, cs, stride, op); break;
        case 5: dchain_comps_t<5, NC>(Dr, Fl, cs, stride, op); break;
        case 6: dchain_comps_t<6, NC>(Dr, Fl, cs, stride, op); break;
        case 7: dchain_comps_t<7, NC>(Dr, Fl, cs, stride, op); break;
        case 8: dchain_comps_t<8, NC>(Dr, Fl, cs, stride, op); break;
        default: dchain_comps_t<9, NC>(Dr, Fl, cs, stride, op); break;
    }
}


// As element_metrics in plain fp64 (coarse tau levels, reading R6): X = T^{g->o}
// Xgeo, derivatives by D^o, cross-product form; Xs: 3 no doubles of scratch.
__device__ void element_metrics_fp64(const CurvedMesh& cm, int e, int o1, int o2, int o3, const Tables* tab,
                                     const double (*Ds)[NP * NP], const int* IJK, double* Xs, double* Mout)
{
    const int no = o1 * o2 * o3;
    const int ga = cm.g1 + 1, gb = cm.g2 + 1;
    const double* G = cm.geo + (long long)e * 3 * cm.ng;
    const double* T1 = tab->T[cm.g1][o1 - 1];
    const double* T2 = tab->T[cm.g2][o2 - 1];
    const double* T3 = tab->T[cm.g3][o3 - 1];
    // the element's geometry coefficients staged in Mout (written only below)
    const double* Gp = G;
    if (3 * cm.ng <= 10 * no) {
        for (int w = threadIdx.x; w < 3 * cm.ng; w += blockDim.x) Mout[w] = __ldg(G + w);
        __syncthreads();
        Gp = Mout;
    }
    // coordinates relative to the first geometry node (D annihilates the
    // shift; the sums run on O(h) values, not O(|x|): reading R6)
    const double x0[3] = {__ldg(G), __ldg(G + cm.ng), __ldg(G + 2 * cm.ng)};
    for (int t = threadIdx.x; t < no; t += blockDim.x) {
        const int pk = IJK[t];  // packed (i, j, k), see k_tau_curved
        const int i = pk & 255, j = (pk >> 8) & 255, k = pk >> 16;
        double x[3] = {0.0, 0.0, 0.0};
        for (int c = 0; c <= cm.g3; ++c) {
            const double w3 = T3[k * (cm.g3 + 1) + c];
            for (int b = 0; b <= cm.g2; ++b) {
                const double w23 = w3 * T2[j * gb + b];
                for (int a = 0; a <= cm.g1; ++a) {
                    const double wgt = w23 * T1[i * ga + a];
                    const int gi = a + ga * (b + gb * c);
#pragma unroll
                    for (int q = 0; q < 3; ++q) x[q] = fma(wgt, Gp[q * cm.ng + gi] - x0[q], x[q]);
                }
            }
        }
        Xs[t] = x[0];
        Xs[no + t] = x[1];
        Xs[2 * no + t] = x[2];
    }
    __syncthreads();
    for (int t = threadIdx.x; t < no; t += blockDim.x) {
        const int pk = IJK[t];
        const int ijk[3] = {pk & 255, (pk >> 8) & 255, pk >> 16};
        double dx[3][3];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            const int od = d == 0 ? o1 : (d == 1 ? o2 : o3);
            const int stride = d == 0 ? 1 : (d == 1 ? o1 : o1 * o2);
            const int a = ijk[d];
            dchain_comps<3>(od, Ds[d] + a * od, Xs + (t - a * stride), no, stride, [&](int cc, double s) { dx[d][cc] = s; });
        }
        const double* xa = dx[0];
        const double* xb = dx[1];
        const double* xc = dx[2];
        double c1[3], c2[3], c3[3];
        c1[0] = xb[1] * xc[2] - xb[2] * xc[1]; c1[1] = xb[2] * xc[0] - xb[0] * xc[2]; c1[2] = xb[0] * xc[1] - xb[1] * xc[0];
        c2[0] = xc[1] * xa[2] - xc[2] * xa[1]; c2[1] = xc[2] * xa[0] - xc[0] * xa[2]; c2[2] = xc[0] * xa[1] - xc[1] * xa[0];
        c3[0] = xa[1] * xb[2] - xa[2] * xb[1]; c3[1] = xa[2] * xb[0] - xa[0] * xb[2]; c3[2] = xa[0] * xb[1] - xa[1] * xb[0];
        for (int q = 0; q < 3; ++q) {
            Mout[q * no + t] = c1[q];
            Mout[(3 + q) * no + t] = c2[q];
            Mout[(6 + q) * no + t] = c3[q];
        }
        Mout[9 * no + t] = xa[0] * c1[0] + xa[1] * c1[1] + xa[2] * c1[2];
    }
    __syncthreads();
}

// D^{o_d - 1} of the three directions into shared memory (Ds[d][a*o_d + m])
__device__ __forceinline__ void stage_D(double (*Ds)[NP * NP], const Tables* tab, int o1, int o2, int o3)
{
    for (int t = threadIdx.x; t < 3 * NP * NP; t += blockDim.x) {
        const int d = t / (NP * NP), r = t - d * (NP * NP);
        const int od = d == 0 ? o1 : (d == 1 ? o2 : o3);
        if (r < od * od) Ds[d][r] = tab->D[od - 1][r];
    }
}

// ---------------------------------------------------------------------------
// Curved residual / RK stage (Euler or NS), per element.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void load_grad(const double* base, int stride, double* g)
{
#pragma unroll
    for (int c = 0; c < 15; ++c) g[c] = __ldg(base + (long long)c * stride);
}

// CFL (+DFL) rates of a state, curved metrics (reading A11)
struct CDtParams {
    const double* q;
    const int* orders;
    const long long* off;
    const double* met;
    PhysDev ph;
    unsigned long long* maxbits;  // [2]
};

__global__ void __launch_bounds__(CBS) k_dt_curved(CDtParams P)
{
    __shared__ double red[32];
    const int e = blockIdx.x;
    const int n1 = P.orders[3 * e] + 1, n2 = P.orders[3 * e + 1] + 1, n3 = P.orders[3 * e + 2] + 1;
    const int n = n1 * n2 * n3;
    const long long o = P.off[e];
    const double* M = P.met + 2 * o;
    double lmax = 0.0, vmax = 0.0;
    for (int t = threadIdx.x; t < n; t += CBS) {
        double q[NV];
        for (int v = 0; v < NV; ++v) q[v] = P.q[o + (long long)v * n + t];
        const double iJ = 1.0 / M[9 * n + t];
        const double ir = 1.0 / q[0];
        const double p = P.ph.gm1 * (q[4] - 0.5 * ir * (q[1] * q[1] + q[2] * q[2] + q[3] * q[3]));
        const double c = sqrt(P.ph.gamma * p * ir);
        const double numax = P.ph.mu * ir * fmax(4.0 / 3.0, P.ph.gamma / P.ph.Pr);
        double lam = 0.0, nu = 0.0;
        for (int d = 0; d < 3; ++d) {
            const double a0 = M[(3 * d) * n + t] * iJ, a1 = M[(3 * d + 1) * n + t] * iJ, a2 = M[(3 * d + 2) * n + t] * iJ;
            const double an2 = a0 * a0 + a1 * a1 + a2 * a2;
            const double ua = (q[1] * a0 + q[2] * a1 + q[3] * a2) * ir;
            const double np1 = d == 0 ? n1 : (d == 1 ? n2 : n3);
            lam += (fabs(ua) + c * sqrt(an2)) * np1 * np1 * 0.5;
            nu += numax * an2 * np1 * np1 * np1 * np1 * 0.25;
        }
        lmax = fmax(lmax, lam);
        vmax = fmax(vmax, nu);
    }
    lmax = block_max(lmax, red);
    vmax = block_max(vmax, red);
    if (threadIdx.x == 0) {
        atomicMax(P.maxbits, (unsigned long long)__double_as_longlong(lmax));
        if (P.ph.physics == 1) atomicMax(P.maxbits + 1, (unsigned long long)__double_as_longlong(vmax));
    }
}

// dt = min(CFL / lam_max, DFL / nu_max); resets the accumulators
__global__ void k_dt_final2(unsigned long long* maxbits, double cfl, double dfl, double* dt)
{
    const double lam = __longlong_as_double((long long)maxbits[0]);
    const double nu = __longlong_as_double((long long)maxbits[1]);
    double v = cfl / lam;
    if (nu > 0.0) v = fmin(v, dfl / nu);
    dt[0] = v;
    maxbits[0] = 0ull;
    maxbits[1] = 0ull;
}

// ---------------------------------------------------------------------------
// tau-estimation on curved elements (Euler or NS), one CTA per level (e,d,p):
// coarse geometry = geometry polynomial at the coarse nodes, metrics by D^O;
// isolated BR1 gradient (strong form) and isolated residual at O.
// ---------------------------------------------------------------------------
struct CTauParams {
    const TablesDD* tdd;
    const double* q;
    const double* qref;
    double* tau;
    const int* orders;
    const long long* off;
    const TauLevel* levels;
    CurvedMesh cm;
    const Tables* tab;
    int formulation;
    int restr;  // 0 interpolation (A3), 1 L2 projection (A3 flag)
    int lbase;  // size class: CTA b handles level lbase + b
    PhysDev ph;
};

// q_c = T_d q and T_d R at one coarse node (line length ND at compile time:
// the loads of a variable's line are issued together)
template <int ND>
__device__ __forceinline__ void tau_interp_node(const double* __restrict__ T, int ic, const double* __restrict__ qe,
                                                const double* __restrict__ re, int n, int base, int stride,
                                                double* Qc, double* Rc, int nO, int t)
{
    double w[ND];
#pragma unroll
    for (int a = 0; a < ND; ++a) w[a] = T[ic * ND + a];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        double xq[ND], xr[ND];
#pragma unroll
        for (int a = 0; a < ND; ++a) {
            xq[a] = __ldg(qe + (long long)v * n + base + a * stride);
            xr[a] = __ldg(re + (long long)v * n + base + a * stride);
        }
        double s = 0.0, r = 0.0;
#pragma unroll
        for (int a = 0; a < ND; ++a) {
            s += w[a] * xq[a];
            r += w[a] * xr[a];
        }
        Qc[v * nO + t] = s;
        Rc[v * nO + t] = r;
    }
}

template <int BS>
__global__ void __launch_bounds__(BS, BS == 256 ? 2 : (BS == 128 ? 5 : 10)) k_tau_curved(CTauParams P)
{
    extern __shared__ double sm[];
    __shared__ double red[32];
    const TauLevel lv = P.levels[P.lbase + blockIdx.x];
    const int e = lv.e, d = lv.d, p = lv.p;
    const int n1 = P.orders[3 * e] + 1, n2 = P.orders[3 * e + 1] + 1, n3 = P.orders[3 * e + 2] + 1;
    const int n = n1 * n2 * n3;
    const int nd = d == 0 ? n1 : (d == 1 ? n2 : n3);
    const int stride = d == 0 ? 1 : (d == 1 ? n1 : n1 * n2);
    const int o1 = d == 0 ? p + 1 : n1, o2 = d == 1 ? p + 1 : n2, o3 = d == 2 ? p + 1 : n3;
    const int nO = o1 * o2 * o3;
    const bool ns = P.ph.physics == 1;
    __shared__ double Ds[3][NP * NP];
    stage_D(Ds, P.tab, o1, o2, o3);
    double* Mc = sm;                         // 10 nO metrics
    double* Qc = Mc + 10 * nO;               // 5 nO
    double* Rc = Qc + NV * nO;               // 5 nO
    double* GA = Rc + NV * nO;               // 15 nO (NS)
    double* F = ns ? GA + 15 * nO : GA;      // 5 nO (NS: only the metric scratch, shared with A)
    double* A = ns ? F : F + NV * nO;        // 5 nO
    // (i, j, k) of every coarse node, packed i | j << 8 | k << 16, computed once
    int* IJK = reinterpret_cast<int*>(sm + (ns ? 40 : 30) * nO);
    for (int t = threadIdx.x; t < nO; t += BS) {
        int ii, jj, kk;
        node_ijk(t, o1, o2, ii, jj, kk);
        IJK[t] = ii | (jj << 8) | (kk << 16);
    }
    __syncthreads();
    element_metrics_fp64(P.cm, e, o1, o2, o3, P.tab, Ds, IJK, F, Mc);  // F: >= 5 nO >= 3 nO scratch (barriers inside)
    const long long o = P.off[e];
    const double* T = P.restr ? P.tab->P[nd - 1][p] : P.tab->T[nd - 1][p];
    for (int t = threadIdx.x; t < nO; t += BS) {
        const int pk = IJK[t];
        int i = pk & 255, j = (pk >> 8) & 255, k = pk >> 16;
        const int ic = d == 0 ? i : (d == 1 ? j : k);
        if (d == 0) i = 0; else if (d == 1) j = 0; else k = 0;
        const int base = i + n1 * (j + n2 * k);
        const double* qe = P.q + o;
        const double* re = P.qref + o;
        switch (nd) {
            case 2: tau_interp_node<2>(T, ic, qe, re, n, base, stride, Qc, Rc, nO, t); break;
            case 3: tau_interp_node<3>(T, ic, qe, re, n, base, stride, Qc, Rc, nO, t); break;
            case 4: tau_interp_node<4>(T, ic, qe, re, n, base, stride, Qc, Rc, nO, t); break;
            case 5: tau_interp_node<5>(T, ic, qe, re, n, base, stride, Qc, Rc, nO, t); break;
            case 6: tau_interp_node<6>(T, ic, qe, re, n, base, stride, Qc, Rc, nO, t); break;
            case 7: tau_interp_node<7>(T, ic, qe, re, n, base, stride, Qc, Rc, nO, t); break;
            case 8: tau_interp_node<8>(T, ic, qe, re, n, base, stride, Qc, Rc, nO, t); break;
            default: tau_interp_node<9>(T, ic, qe, re, n, base, stride, Qc, Rc, nO, t); break;
        }
        if (!ns)
            for (int v = 0; v < NV; ++v) A[v * nO + t] = 0.0;
    }
    __syncthreads();
    if (ns) {  // isolated gradient: J g_k = sum_d' D^{d'} (Ja^{d'}_k q), one thread per node in registers
        for (int t = threadIdx.x; t < nO; t += BS) {
            const int pk = IJK[t];
            const int ijk[3] = {pk & 255, (pk >> 8) & 255, pk >> 16};
            double g[15];
#pragma unroll
            for (int cc = 0; cc < 15; ++cc) g[cc] = 0.0;
            for (int dd = 0; dd < 3; ++dd) {
                const int od = dd == 0 ? o1 : (dd == 1 ? o2 : o3);
                const int str = dd == 0 ? 1 : (dd == 1 ? o1 : o1 * o2);
                const int a = ijk[dd];
                const int base = t - a * str;
                const double* Dr = Ds[dd] + a * od;
                for (int m = 0; m < od; ++m) {
                    const int nm = base + m * str;
                    const double dm = Dr[m];
                    double qv[NV];
#pragma unroll
                    for (int v = 0; v < NV; ++v) qv[v] = Qc[v * nO + nm];
#pragma unroll
                    for (int kk = 0; kk < 3; ++kk) {
                        const double jk = Mc[(3 * dd + kk) * nO + nm];
#pragma unroll
                        for (int v = 0; v < NV; ++v) g[kk * NV + v] = fma(dm, jk * qv[v], g[kk * NV + v]);
                    }
                }
            }
            const double iJ = 1.0 / Mc[9 * nO + t];
#pragma unroll
            for (int cc = 0; cc < 15; ++cc) GA[cc * nO + t] = g[cc] * iJ;
            for (int v = 0; v < NV; ++v) A[v * nO + t] = 0.0;
        }
        __syncthreads();
    }
    if (ns) {  // fluxes of the three directions from one viscous evaluation per node, in place of GA
        for (int t = threadIdx.x; t < nO; t += BS) {
            double qv[NV], gv[15];
            for (int v = 0; v < NV; ++v) qv[v] = Qc[v * nO + t];
            for (int cc = 0; cc < 15; ++cc) gv[cc] = GA[cc * nO + t];
            ViscNode V;
            visc_node(qv, gv, P.ph, V);
            for (int dd = 0; dd < 3; ++dd) {  // = contra_flux
                const double ax = Mc[(3 * dd) * nO + t], ay = Mc[(3 * dd + 1) * nO + t], az = Mc[(3 * dd + 2) * nO + t];
                double Fv[NV], fv[NV];
                adv_dot(qv, ax, ay, az, P.ph.gm1, Fv);
                visc_along(V, ax, ay, az, fv);
                for (int v = 0; v < NV; ++v) GA[(dd * NV + v) * nO + t] = Fv[v] - fv[v];
            }
        }
        __syncthreads();
        for (int t = threadIdx.x; t < nO; t += BS) {
            const int pk = IJK[t];
            const int ijk[3] = {pk & 255, (pk >> 8) & 255, pk >> 16};
            for (int dd = 0; dd < 3; ++dd) {
                const int od = dd == 0 ? o1 : (dd == 1 ? o2 : o3);
                const int str = dd == 0 ? 1 : (dd == 1 ? o1 : o1 * o2);
                const int a = ijk[dd];
                dsum_comps<NV>(od, Ds[dd] + a * od, GA + dd * NV * nO + (t - a * str), nO, str,
                               [&](int v, double sv) { A[v * nO + t] += sv; });
            }
        }
        __syncthreads();
    } else {
        for (int dd = 0; dd < 3; ++dd) {
            const int od = dd == 0 ? o1 : (dd == 1 ? o2 : o3);
            const int str = dd == 0 ? 1 : (dd == 1 ? o1 : o1 * o2);
            const double* Dd = Ds[dd];
            for (int t = threadIdx.x; t < nO; t += BS) {
                double qv[NV], gv[15], Fv[NV];
                for (int v = 0; v < NV; ++v) qv[v] = Qc[v * nO + t];
                if (ns)
                    for (int c = 0; c < 15; ++c) gv[c] = GA[c * nO + t];
                contra_flux(qv, gv, Mc[(3 * dd) * nO + t], Mc[(3 * dd + 1) * nO + t], Mc[(3 * dd + 2) * nO + t], P.ph, Fv);
                for (int v = 0; v < NV; ++v) F[v * nO + t] = Fv[v];
            }
            __syncthreads();
            for (int t = threadIdx.x; t < nO; t += BS) {
                int ijk[3];
                const int pk = IJK[t];
                ijk[0] = pk & 255; ijk[1] = (pk >> 8) & 255; ijk[2] = pk >> 16;
                const int a = dd == 0 ? ijk[0] : (dd == 1 ? ijk[1] : ijk[2]);
                const int base = t - a * str;
                dsum_comps<NV>(od, Dd + a * od, F + base, nO, str, [&](int v, double sv) { A[v * nO + t] += sv; });
            }
            __syncthreads();
        }
    }
    double tmax = 0.0;
    for (int t = threadIdx.x; t < nO; t += BS) {
        const int pk = IJK[t];
        int i = pk & 255, j = (pk >> 8) & 255, k = pk >> 16;
        const double J = Mc[9 * nO + t];
        double scale = 1.0;
        if (P.formulation == 1) scale = J * P.tab->w[o1 - 1][i] * P.tab->w[o2 - 1][j] * P.tab->w[o3 - 1][k];
        for (int v = 0; v < NV; ++v) tmax = fmax(tmax, fabs(scale * (Rc[v * nO + t] + A[v * nO + t] / J)));
    }
    tmax = block_max(tmax, red);
    if (threadIdx.x == 0) P.tau[(3 * (long long)e + d) * DG_TAU_STRIDE_DEV + p] = tmax;
}

}  // namespace dgtau
