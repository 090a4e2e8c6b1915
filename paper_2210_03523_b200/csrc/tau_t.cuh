// tau_t.cuh -- batched tau-estimation: tau[e][d][p] for every
// element e, direction d and coarse order p < N_d.
//
// tau-estimation with the variational DG reference term I F(q) ~ I (M^P)^-1
// F^P(q^P), eqs TEtildedef / TEdef, isolated
// coarse operators, decoupled directional coarse levels
// (reading A12): for every direction d and coarse order p < N_d of the
// element, O = N with O_d = p,
//   q_c = T_d^{N_d->p} q,  Qdot_c = -sum_d' (2/h_d') D^{O_d'} f_d'(q_c)
//   (strong form == weak form + own-trace lifting for GL),
//   tau~ = T_d R - Qdot_c,  tau = J w w w tau~ (traditional),
//   tau[e][d][p] = max |tau| over coarse nodes and variables.
// k_tau5 (below) evaluates groups of coarse orders of one (element,
// direction) per CTA; k_tau_norm fills the noise-scale slot (reading R1).
#pragma once

#include "residual_t.cuh"

namespace dgtau {

// (element, direction, coarse order) of the curved tau kernel (k_tau_curved)
struct TauLevel {
    int e, d, p, pad;
};

// Exact integer quotient a / b for 0 <= a < 4096, 1 <= b < 1024 from the
// correctly rounded float reciprocal: the float product's absolute error
// (< 4096 * 2^-23 < 5e-4) is below the distance 0.5/b >= 4.9e-4 of
// (a + 0.5)/b to the nearest integer.  Avoids ~20-instruction integer division.
__device__ __forceinline__ int fdiv(int a, float inv_b) { return __float2int_rz(((float)a + 0.5f) * inv_b); }

// variable index of a (v, l) task, 0 <= task < 5 * nl, by comparisons
__device__ __forceinline__ int var_of(int task, int nl)
{
    return (task >= nl) + (task >= 2 * nl) + (task >= 3 * nl) + (task >= 4 * nl);
}

// tau[e][d][0] = ||Qdot_ref,e||_inf and NaN for p >= N_d (one CTA per element)
// Non-isolated tau-estimation, one coarse level (d, p) (reading
// R7): tau[e][d][p] = max over the coarse nodes and variables of
// |scale (T_d R - Qdot_c)| for every element with p < N_d(e); rc, dc in the
// coarse layout (orders oc, offsets offc); scale = J w w w (traditional form,
// P:186-188; J from hgeo (affine) or the coarse metrics met (curved)), else 1.
__global__ void __launch_bounds__(128) k_tau_level(const double* rc, const double* dc, const int* ofine, const int* oc,
                                                   const long long* offc, int d, int p, int formulation,
                                                   const double* hgeo, const double* met, const Tables* tab,
                                                   double* tau)
{
    __shared__ double red[32];
    const int e = blockIdx.x;
    if (p >= ofine[3 * e + d]) return;  // level not defined for e (whole CTA)
    const int o1 = oc[3 * e] + 1, o2 = oc[3 * e + 1] + 1, o3 = oc[3 * e + 2] + 1;
    const int n = o1 * o2 * o3;
    const long long o = offc[e];
    const double Jel = met ? 0.0 : hgeo[3 * e] * hgeo[3 * e + 1] * hgeo[3 * e + 2] / 8.0;
    double tmax = 0.0;
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
        double scale = 1.0;
        if (formulation == 1) {
            const int k = t / (o1 * o2), r = t - k * o1 * o2, j = r / o1, i = r - j * o1;
            const double J = met ? met[2 * o + 9LL * n + t] : Jel;
            scale = J * tab->w[o1 - 1][i] * tab->w[o2 - 1][j] * tab->w[o3 - 1][k];
        }
#pragma unroll
        for (int v = 0; v < NV; ++v) tmax = fmax(tmax, fabs(scale * (rc[o + (long long)v * n + t] - dc[o + (long long)v * n + t])));
    }
    tmax = block_max(tmax, red);
    if (threadIdx.x == 0) tau[(3 * (long long)e + d) * DG_TAU_STRIDE_DEV + p] = tmax;
}

__global__ void __launch_bounds__(128) k_tau_norm(const double* qref, double* tau, const int* orders,
                                                  const long long* off)
{
    __shared__ double red[32];
    const int e = blockIdx.x;
    const int N1 = orders[3 * e], N2 = orders[3 * e + 1], N3 = orders[3 * e + 2];
    const int n = (N1 + 1) * (N2 + 1) * (N3 + 1);
    const double* re = qref + off[e];
    double rn = 0.0;
    for (int t = threadIdx.x; t < NV * n; t += blockDim.x) rn = fmax(rn, fabs(re[t]));
    rn = block_max(rn, red);
    if (threadIdx.x < 3 * DG_TAU_STRIDE_DEV) {
        const int d = threadIdx.x / DG_TAU_STRIDE_DEV, p = threadIdx.x % DG_TAU_STRIDE_DEV;
        const int Nd = d == 0 ? N1 : (d == 1 ? N2 : N3);
        if (p == 0) tau[(3 * (long long)e + d) * DG_TAU_STRIDE_DEV] = rn;
        else if (p >= Nd) tau[(3 * (long long)e + d) * DG_TAU_STRIDE_DEV + p] = __longlong_as_double(0x7ff8000000000000LL);
    }
}

}  // namespace dgtau

namespace dgtau {

// ---------------------------------------------------------------------------
// tau-estimation v5: one CTA per (element e, direction d, group of coarse
// orders p0..p1) (reading A12).  All levels of the group are
// evaluated at once, their coarse blocks (O_d = p+1) laid out back to back in
// shared memory, so each of the four phases has a few hundred independent
// tasks and the CTA needs only four barriers:
//   (A) q_c = T_d^{N_d->p} q for every level: one (line across d, variable)
//       task reads the fine line once (L1) and writes all levels' coarse lines;
//   (B) f_0, f_1, f_2 of q_c at every coarse node (f_0 in place of q_c);
//   (C) D^{O_d'} along every line of every axis of every level (even-odd,
//       compile-time line lengths through a switch);
//   (D) tau~ = T_d R + sum_d' (2/h_d') D f_d' per node and variable (T_d R from
//       the fine R through L1), traditional * J w w w, max-reduced
//       per level (shared atomicMax on the bits of non-negative doubles).
// ---------------------------------------------------------------------------

struct TauGroup {
    int e, d, p0, p1;
};

constexpr int TAU5_BS = 256;
constexpr int TAU5_MAXN = 384;  // coarse nodes per group (unless one level alone is larger)

struct Tau5Params {
    const double* q;
    const double* qref;
    double* tau;
    const int* orders;
    const long long* off;
    const double* hgeo;
    const TauGroup* groups;
    const Tables* tab;
    int formulation;
    int restr;  // 0 interpolation (A3), 1 L2 projection (A3 flag)
    double gm1;
};

// (A) of k_tau5 for a compile-time fine line length ND along d: one (field,
// variable, line) task reads the fine line once and writes the coarse lines of
// every level of the group.
template <int ND>
__device__ __forceinline__ void tau5_interp(const Tau5Params& P, long long o, int n, int n1, int n2, int d, int nx,
                                            int nlev, int p0, int strf, const int* lbase, const int* tbase,
                                            const double* Ts, double* F0, double* RC)
{
    const float inv_n1 = 1.0f / (float)n1;
    for (int task2 = threadIdx.x; task2 < 2 * NV * nx; task2 += TAU5_BS) {
        const bool isR = task2 >= NV * nx;
        const int task = isR ? task2 - NV * nx : task2;
        const double* qe = (isR ? P.qref : P.q) + o;
        double* dstb = isR ? RC : F0;
        const int v = var_of(task, nx), l = task - v * nx;
        int bf, i = 0, k = 0;
        if (d == 0) bf = l * ND;
        else if (d == 1) { k = fdiv(l, inv_n1); i = l - k * n1; bf = i + n1 * ND * k; }
        else bf = l;
        double f[ND];
#pragma unroll
        for (int a = 0; a < ND; ++a) f[a] = __ldg(qe + v * n + bf + a * strf);
        for (int li = 0; li < nlev; ++li) {
            const int pc = p0 + li + 1, nO = pc * nx;
            const int o1 = d == 0 ? pc : n1;
            int bc, strc;
            if (d == 0) { bc = l * pc; strc = 1; }
            else if (d == 1) { bc = i + o1 * pc * k; strc = o1; }
            else { bc = l; strc = n1 * n2; }
            const double* T = Ts + tbase[li];
            double* out = dstb + NV * lbase[li] + v * nO + bc;
            for (int ic = 0; ic < pc; ++ic) {
                const double* Tr = T + ic * ND;
                double s0 = Tr[0] * f[0], s1 = 0.0;
#pragma unroll
                for (int a = 1; a < ND; ++a) {
                    if (a & 1) s1 = fma(Tr[a], f[a], s1);
                    else s0 = fma(Tr[a], f[a], s0);
                }
                out[ic * strc] = s0 + s1;
            }
        }
    }
}

__global__ void __launch_bounds__(TAU5_BS, 3) k_tau5(Tau5Params P)
{
    extern __shared__ __align__(16) double sm[];
    __shared__ double Ts[NP * NP * NP / 2];      // T^{N_d -> p} of the group's levels, back to back
    __shared__ int lbase[NP + 1], tbase[NP];      // node / table offsets per level of the group
    __shared__ int abase[3][NP + 1];              // line-task prefix per axis over the levels
    __shared__ unsigned long long lmaxb[NP];
    const TauGroup tg = P.groups[blockIdx.x];
    const int e = tg.e, d = tg.d, p0 = tg.p0, nlev = tg.p1 - tg.p0 + 1;
    const int tid = threadIdx.x;
    const int N1 = P.orders[3 * e], N2 = P.orders[3 * e + 1], N3 = P.orders[3 * e + 2];
    const int n1 = N1 + 1, n2 = N2 + 1, n3 = N3 + 1;
    const int n = n1 * n2 * n3;
    const int Nd = d == 0 ? N1 : (d == 1 ? N2 : N3);
    const int nd = Nd + 1;
    const int nx = n / nd;  // coarse nodes per unit of O_d (cross-section of d)
    const long long o = P.off[e];
    // element size (phase D), loaded now so its latency hides behind phases A-C
    const double h0 = __ldg(P.hgeo + 3 * e), h1 = __ldg(P.hgeo + 3 * e + 1), h2 = __ldg(P.hgeo + 3 * e + 2);
    if (tid <= nlev) {  // closed forms: S(li) = sum_{j<li} (p0 + j + 1)
        const int li = tid, Sl = li * (p0 + 1) + li * (li - 1) / 2;
        lbase[li] = nx * Sl;
        if (li < nlev) tbase[li] = nd * Sl;
        const int na[3] = {n1, n2, n3};
#pragma unroll
        for (int a = 0; a < 3; ++a) abase[a][li] = a == d ? NV * nx * li : NV * (nx / na[a]) * Sl;
    }
    if (tid < nlev) lmaxb[tid] = 0ull;
    __syncthreads();
    const int ntot = lbase[nlev];
    for (int t = tid; t < tbase[nlev - 1] + (p0 + nlev) * nd; t += TAU5_BS) {
        int li = 0;
        while (li + 1 < nlev && tbase[li + 1] <= t) ++li;
        Ts[t] = (P.restr ? P.tab->P[Nd][p0 + li] : P.tab->T[Nd][p0 + li])[t - tbase[li]];
    }
    double* F0 = sm;               // coarse state, then f_0 and D^{O_0} f_0
    double* F1 = F0 + NV * ntot;
    double* F2 = F1 + NV * ntot;
    double* RC = F2 + NV * ntot;   // T_d R of every level
    const int strf = d == 0 ? 1 : (d == 1 ? n1 : n1 * n2);
    __syncthreads();
    // (A) q_c = T_d q and T_d R along d for every level (reading A3); layout per
    //     level: [v][coarse node of the level's (o1,o2,o3) block] at 5*lbase + v*nO
    switch (nd) {
        case 3: tau5_interp<3>(P, o, n, n1, n2, d, nx, nlev, p0, strf, lbase, tbase, Ts, F0, RC); break;
        case 4: tau5_interp<4>(P, o, n, n1, n2, d, nx, nlev, p0, strf, lbase, tbase, Ts, F0, RC); break;
        case 5: tau5_interp<5>(P, o, n, n1, n2, d, nx, nlev, p0, strf, lbase, tbase, Ts, F0, RC); break;
        case 6: tau5_interp<6>(P, o, n, n1, n2, d, nx, nlev, p0, strf, lbase, tbase, Ts, F0, RC); break;
        case 7: tau5_interp<7>(P, o, n, n1, n2, d, nx, nlev, p0, strf, lbase, tbase, Ts, F0, RC); break;
        case 8: tau5_interp<8>(P, o, n, n1, n2, d, nx, nlev, p0, strf, lbase, tbase, Ts, F0, RC); break;
        default: tau5_interp<9>(P, o, n, n1, n2, d, nx, nlev, p0, strf, lbase, tbase, Ts, F0, RC); break;
    }
    __syncthreads();
    // (B) the three Cartesian fluxes of every coarse node (f_0 in place of q_c)
    for (int t = tid; t < ntot; t += TAU5_BS) {
        int li = 0;
        while (li + 1 < nlev && lbase[li + 1] <= t) ++li;
        const int nO = lbase[li + 1] - lbase[li], r = t - lbase[li];
        double* b0 = F0 + NV * lbase[li] + r;
        double* b1 = F1 + NV * lbase[li] + r;
        double* b2 = F2 + NV * lbase[li] + r;
        double qv[NV], f[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) qv[v] = b0[v * nO];
        const double ir = rcp_nr(qv[0]);
        const double pr = P.gm1 * (qv[4] - 0.5 * ir * (qv[1] * qv[1] + qv[2] * qv[2] + qv[3] * qv[3]));
        flux_axis<1>(qv, ir, pr, f);
#pragma unroll
        for (int v = 0; v < NV; ++v) b1[v * nO] = f[v];
        flux_axis<2>(qv, ir, pr, f);
#pragma unroll
        for (int v = 0; v < NV; ++v) b2[v * nO] = f[v];
        flux_axis<0>(qv, ir, pr, f);
#pragma unroll
        for (int v = 0; v < NV; ++v) b0[v * nO] = f[v];
    }
    __syncthreads();
    // (C) D^{O_a} along every line of every axis a of every level (one pass per
    //     axis; a thread's tasks increase, so its level index only moves forward)
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        double* Fa = a == 0 ? F0 : (a == 1 ? F1 : F2);
        int li = 0;
        for (int task = tid; task < abase[a][nlev]; task += TAU5_BS) {
            while (abase[a][li + 1] <= task) ++li;
            const int u = task - abase[a][li];
            const int pc = p0 + li + 1, nO = pc * nx;
            const int o1 = d == 0 ? pc : n1, o2 = d == 1 ? pc : n2, o3 = d == 2 ? pc : n3;
            const int L = a == 0 ? o1 : (a == 1 ? o2 : o3);
            const int nl = nO / L;
            const int v = var_of(u, nl), l = u - v * nl;
            int base, str;
            if (a == 0) { base = l * L; str = 1; }
            else if (a == 1) { const int kk = fdiv(l, 1.0f / (float)o1); base = (l - kk * o1) + o1 * L * kk; str = o1; }
            else { base = l; str = o1 * o2; }
            double* Fb = Fa + NV * lbase[li] + v * nO + base;
            switch (L) {
                case 2: dline_inplace<2>(Fb, str); break;
                case 3: dline_inplace<3>(Fb, str); break;
                case 4: dline_inplace<4>(Fb, str); break;
                case 5: dline_inplace<5>(Fb, str); break;
                case 6: dline_inplace<6>(Fb, str); break;
                case 7: dline_inplace<7>(Fb, str); break;
                case 8: dline_inplace<8>(Fb, str); break;
                default: dline_inplace<9>(Fb, str); break;
            }
        }
    }
    __syncthreads();
    // (D) tau~ = T_d R + sum_a (2/h_a) D f_a; traditional * J w w w
    {
        const double sc0 = 2.0 / h0, sc1 = 2.0 / h1, sc2 = 2.0 / h2;
        const double Jel = h0 * h1 * h2 / 8.0;
        int lcur = -1;
        double tmax = 0.0;
        for (int t = tid; t < ntot; t += TAU5_BS) {
            int li = 0;
            while (li + 1 < nlev && lbase[li + 1] <= t) ++li;
            if (li != lcur) {
                if (lcur >= 0) atomicMax(&lmaxb[lcur], (unsigned long long)__double_as_longlong(tmax));
                lcur = li;
                tmax = 0.0;
            }
            const int pc = p0 + li + 1, nO = pc * nx, r = t - lbase[li];
            const int o1 = d == 0 ? pc : n1, o2 = d == 1 ? pc : n2, o3 = d == 2 ? pc : n3;
            const int kz = fdiv(r, 1.0f / (float)(o1 * o2)), rr = r - kz * o1 * o2, j = fdiv(rr, 1.0f / (float)o1),
                      i = rr - j * o1;
            double scale = 1.0;
            if (P.formulation == 1) scale = Jel * c_w[o1 - 1][i] * c_w[o2 - 1][j] * c_w[o3 - 1][kz];
            const double* rc = RC + NV * lbase[li] + r;
            const double* f0 = F0 + NV * lbase[li] + r;
            const double* f1 = F1 + NV * lbase[li] + r;
            const double* f2 = F2 + NV * lbase[li] + r;
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                const double acc = fma(sc2, f2[v * nO], fma(sc1, f1[v * nO], fma(sc0, f0[v * nO], rc[v * nO])));
                tmax = fmax(tmax, fabs(scale * acc));
            }
        }
        if (lcur >= 0) atomicMax(&lmaxb[lcur], (unsigned long long)__double_as_longlong(tmax));
    }
    __syncthreads();
    if (tid < nlev) P.tau[(3 * (long long)e + d) * DG_TAU_STRIDE_DEV + p0 + tid] = __longlong_as_double((long long)lmaxb[tid]);
}

}  // namespace dgtau
