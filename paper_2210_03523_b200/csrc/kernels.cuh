// kernels.cuh -- generic (runtime-order) sm_100a kernels of the DGSEM /
// tau-estimation hot path; included by dgtau.cu only.  Numerics: see
// common.cuh.
#pragma once

#include "common.cuh"

namespace dgtau {

// ---------------------------------------------------------------------------
// Residual / RK-stage kernel: one CTA per work item (1..32 elements of the
// same orders, from one (N1,N2,N3) bucket).
// ---------------------------------------------------------------------------

__global__ void __launch_bounds__(BLOCK) k_residual(ResParams P)
{
    extern __shared__ double sm[];
    __shared__ long long s_off[MAXSLOTS];
    __shared__ int s_e[MAXSLOTS];
    __shared__ double s_h[MAXSLOTS][3];

    const WorkItem w = P.work[blockIdx.x];
    int N[3];
    unpack_ord(w.ord, N[0], N[1], N[2]);
    const int n1 = N[0] + 1, n2 = N[1] + 1, n3 = N[2] + 1;
    const int n = n1 * n2 * n3;
    const int cnt = w.count;
    const int nf[3] = {n2 * n3, n1 * n3, n1 * n2};
    const int fsz = 2 * (nf[0] + nf[1] + nf[2]);  // face points per element (6 faces)
    int foff[6];
    {
        int acc = 0;
        for (int f = 0; f < 6; ++f) { foff[f] = acc; acc += NV * nf[f >> 1]; }
    }
    double* Dsm = sm;                  // 3 x 81
    double* qs = Dsm + 3 * NP * NP;    // cnt x 5 x n
    double* Fs = qs + cnt * NV * n;    // cnt x 5 x n
    double* Gs = Fs + cnt * NV * n;    // cnt x 5 x fsz

    const int tid = threadIdx.x;
    if (tid < cnt) {
        const int e = P.elist[w.start + tid];
        s_e[tid] = e;
        s_off[tid] = P.off[e];
        for (int d = 0; d < 3; ++d) s_h[tid][d] = P.hgeo[3 * e + d];
    }
    for (int t = tid; t < 3 * NP * NP; t += BLOCK) {
        const int d = t / (NP * NP), r = t % (NP * NP);
        const int nd = N[d] + 1;
        if (r < nd * nd) Dsm[d * NP * NP + r] = P.tab->D[N[d]][r];
    }
    __syncthreads();
    for (int t = tid; t < cnt * NV * n; t += BLOCK) {
        const int slot = t / (NV * n), r = t - slot * NV * n;
        qs[t] = P.q[s_off[slot] + r];
    }
    __syncthreads();

    const double gm1 = P.ph.gm1;
    double acc[NPT][NV];
#pragma unroll
    for (int it = 0; it < NPT; ++it)
#pragma unroll
        for (int v = 0; v < NV; ++v) acc[it][v] = 0.0;

    // ---- volume term: sum_d (2/h_d) D^{N_d} f_d -------------------------
    for (int d = 0; d < 3; ++d) {
        for (int t = tid; t < cnt * n; t += BLOCK) {
            const int slot = t / n, node = t - slot * n;
            double qv[NV], f[NV], p;
            for (int v = 0; v < NV; ++v) qv[v] = qs[(slot * NV + v) * n + node];
            flux_dir(qv, gm1, d, f, &p);
            if (d == 0 && !(qv[0] > 0.0 && p > 0.0)) {
                if (atomicAdd(P.flag, 1) == 0) P.flag[1] = s_e[slot];
            }
            for (int v = 0; v < NV; ++v) Fs[(slot * NV + v) * n + node] = f[v];
        }
        __syncthreads();
        const int nd = N[d] + 1;
        const int stride = d == 0 ? 1 : (d == 1 ? n1 : n1 * n2);
        const double* Dd = Dsm + d * NP * NP;
#pragma unroll
        for (int it = 0; it < NPT; ++it) {
            const int t = tid + it * BLOCK;
            if (t < cnt * n) {
                const int slot = t / n, node = t - slot * n;
                int ijk[3];
                node_ijk(node, n1, n2, ijk[0], ijk[1], ijk[2]);
                const int a = ijk[d];
                const int base = node - a * stride;
                const double sc = 2.0 / s_h[slot][d];
                for (int v = 0; v < NV; ++v) {
                    const double* Fl = Fs + (slot * NV + v) * n + base;
                    double s = 0.0;
                    for (int m = 0; m < nd; ++m) s += Dd[a * nd + m] * Fl[m * stride];
                    acc[it][v] += sc * s;
                }
            }
        }
        __syncthreads();
    }

    // ---- surface: Gs = G - f_own (strong form) on the 6 faces ----------
    if (P.variant == 0) {
        for (int t = tid; t < cnt * fsz; t += BLOCK) {
            const int slot = t / fsz;
            int r = t - slot * fsz;
            int f = 0;
            while (r >= nf[f >> 1]) { r -= nf[f >> 1]; ++f; }
            const int d = f >> 1, s = f & 1, pt = r;
            const int e = s_e[slot];
            // own boundary node
            int ijk[3];
            const int ta = d == 0 ? 1 : 0, tb = d == 2 ? 1 : 2;
            const int nta = N[ta] + 1;
            ijk[ta] = pt % nta;
            ijk[tb] = pt / nta;
            ijk[d] = s ? N[d] : 0;
            const int node = ijk[0] + n1 * (ijk[1] + n2 * ijk[2]);
            double qo[NV], fo[NV], p;
            for (int v = 0; v < NV; ++v) qo[v] = qs[(slot * NV + v) * n + node];
            flux_dir(qo, gm1, d, fo, &p);
            double Gv[NV];
            const int nb = P.nbr[6 * e + f];
            double nrm[3] = {0.0, 0.0, 0.0};
            nrm[d] = 1.0;
            if (nb < 0) {
                double qg[NV];
                ghost_state(qo, nb, P.ph, qg);
                if (s) riemann(qo, qg, nrm, P.ph, Gv); else riemann(qg, qo, nrm, P.ph, Gv);
            } else {
                const long long mo = P.moff[6 * e + f];
                if (mo >= 0) {
                    for (int v = 0; v < NV; ++v) Gv[v] = P.mortarG[mo + (long long)v * nf[d] + pt];
                } else {
                    const int B1 = P.orders[3 * nb] + 1, B2 = P.orders[3 * nb + 1] + 1, B3 = P.orders[3 * nb + 2] + 1;
                    int jb[3] = {ijk[0], ijk[1], ijk[2]};
                    const int Bd = d == 0 ? B1 : (d == 1 ? B2 : B3);
                    jb[d] = s ? 0 : Bd - 1;
                    const int nbn = B1 * B2 * B3;
                    const long long ob = P.off[nb] + jb[0] + B1 * (jb[1] + B2 * jb[2]);
                    double qn[NV];
                    for (int v = 0; v < NV; ++v) qn[v] = P.q[ob + (long long)v * nbn];
                    if (s) riemann(qo, qn, nrm, P.ph, Gv); else riemann(qn, qo, nrm, P.ph, Gv);
                }
            }
            double* Gd = Gs + slot * NV * fsz + foff[f];
            for (int v = 0; v < NV; ++v) Gd[v * nf[d] + pt] = Gv[v] - fo[v];
        }
        __syncthreads();
        // lifting onto the boundary nodes
#pragma unroll
        for (int it = 0; it < NPT; ++it) {
            const int t = tid + it * BLOCK;
            if (t < cnt * n) {
                const int slot = t / n, node = t - slot * n;
                int ijk[3];
                node_ijk(node, n1, n2, ijk[0], ijk[1], ijk[2]);
                for (int d = 0; d < 3; ++d) {
                    const int a = ijk[d];
                    if (a != 0 && a != N[d]) continue;
                    const int ta = d == 0 ? 1 : 0, tb = d == 2 ? 1 : 2;
                    const int pt = ijk[ta] + (N[ta] + 1) * ijk[tb];
                    const int f = 2 * d + (a == N[d] ? 1 : 0);
                    const double sgn = a == N[d] ? 1.0 : -1.0;
                    const double sc = sgn * 2.0 / (s_h[slot][d] * P.tab->w[N[d]][a]);
                    const double* Gd = Gs + slot * NV * fsz + foff[f];
                    for (int v = 0; v < NV; ++v) acc[it][v] += sc * Gd[v * nf[d] + pt];
                }
            }
        }
    }

    // ---- output: Qdot = -acc, or the fused low-storage RK update -------
    if (P.mode == 0) {
#pragma unroll
        for (int it = 0; it < NPT; ++it) {
            const int t = tid + it * BLOCK;
            if (t < cnt * n) {
                const int slot = t / n, node = t - slot * n;
                for (int v = 0; v < NV; ++v) P.out[s_off[slot] + (long long)v * n + node] = -acc[it][v];
            }
        }
    } else {
        const double dt = *P.dt;
#pragma unroll
        for (int it = 0; it < NPT; ++it) {
            const int t = tid + it * BLOCK;
            if (t < cnt * n) {
                const int slot = t / n, node = t - slot * n;
                for (int v = 0; v < NV; ++v) {
                    const long long ix = s_off[slot] + (long long)v * n + node;
                    const double gn = (P.rkA == 0.0 ? 0.0 : P.rkA * P.g[ix]) - dt * acc[it][v];
                    P.g[ix] = gn;
                    P.out[ix] = qs[(slot * NV + v) * n + node] + P.rkB * gn;
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Mortar kernel (reading A6): one CTA per face whose tangential orders differ.
// Traces interpolated to the mortar (orders max per tangential direction),
// Riemann flux there, exact L2 projection back to both sides.
// ---------------------------------------------------------------------------

struct MortarParams {
    const double* q;
    const int* orders;
    const long long* off;
    const MortarItem* items;
    const long long* moff;
    double* mortarG;
    const Tables* tab;
    PhysDev ph;
};

__global__ void __launch_bounds__(128) k_mortar(MortarParams P)
{
    __shared__ double GM[NV][NP * NP];
    const MortarItem it = P.items[blockIdx.x];
    const int d = it.d;
    const int ta = d == 0 ? 1 : 0, tb = d == 2 ? 1 : 2;
    int NL[3], NR[3];
    for (int k = 0; k < 3; ++k) { NL[k] = P.orders[3 * it.L + k]; NR[k] = P.orders[3 * it.R + k]; }
    const int M1 = max(NL[ta], NR[ta]), M2 = max(NL[tb], NR[tb]);
    const int nm = (M1 + 1) * (M2 + 1);
    const int nL = (NL[0] + 1) * (NL[1] + 1) * (NL[2] + 1), nR = (NR[0] + 1) * (NR[1] + 1) * (NR[2] + 1);
    const long long oL = P.off[it.L], oR = P.off[it.R];
    const double* TL1 = P.tab->T[NL[ta]][M1];
    const double* TL2 = P.tab->T[NL[tb]][M2];
    const double* TR1 = P.tab->T[NR[ta]][M1];
    const double* TR2 = P.tab->T[NR[tb]][M2];
    double nrm[3] = {0.0, 0.0, 0.0};
    nrm[d] = 1.0;
    for (int t = threadIdx.x; t < nm; t += blockDim.x) {
        const int m1 = t % (M1 + 1), m2 = t / (M1 + 1);
        double qL[NV] = {0, 0, 0, 0, 0}, qR[NV] = {0, 0, 0, 0, 0};
        // L's +1 face and R's -1 face, interpolated along both tangential directions
        for (int b = 0; b <= NL[tb]; ++b)
            for (int a = 0; a <= NL[ta]; ++a) {
                int ijk[3];
                ijk[d] = NL[d]; ijk[ta] = a; ijk[tb] = b;
                const long long ix = oL + ijk[0] + (NL[0] + 1) * (ijk[1] + (NL[1] + 1) * ijk[2]);
                const double wgt = TL1[m1 * (NL[ta] + 1) + a] * TL2[m2 * (NL[tb] + 1) + b];
                for (int v = 0; v < NV; ++v) qL[v] += wgt * P.q[ix + (long long)v * nL];
            }
        for (int b = 0; b <= NR[tb]; ++b)
            for (int a = 0; a <= NR[ta]; ++a) {
                int ijk[3];
                ijk[d] = 0; ijk[ta] = a; ijk[tb] = b;
                const long long ix = oR + ijk[0] + (NR[0] + 1) * (ijk[1] + (NR[1] + 1) * ijk[2]);
                const double wgt = TR1[m1 * (NR[ta] + 1) + a] * TR2[m2 * (NR[tb] + 1) + b];
                for (int v = 0; v < NV; ++v) qR[v] += wgt * P.q[ix + (long long)v * nR];
            }
        double F[NV];
        riemann(qL, qR, nrm, P.ph, F);
        for (int v = 0; v < NV; ++v) GM[v][t] = F[v];
    }
    __syncthreads();
    // project back: side X with tangential orders (S1, S2)
    for (int side = 0; side < 2; ++side) {
        const int* NS = side == 0 ? NL : NR;
        const int S1 = NS[ta], S2 = NS[tb];
        const int ns = (S1 + 1) * (S2 + 1);
        const long long mo = P.moff[6 * (side == 0 ? it.L : it.R) + 2 * d + (side == 0 ? 1 : 0)];
        const double* P1 = P.tab->P[M1][S1];
        const double* P2 = P.tab->P[M2][S2];
        for (int t = threadIdx.x; t < ns; t += blockDim.x) {
            const int a = t % (S1 + 1), b = t / (S1 + 1);
            double s[NV] = {0, 0, 0, 0, 0};
            for (int m2 = 0; m2 <= M2; ++m2)
                for (int m1 = 0; m1 <= M1; ++m1) {
                    const double wgt = P1[a * (M1 + 1) + m1] * P2[b * (M2 + 1) + m2];
                    for (int v = 0; v < NV; ++v) s[v] += wgt * GM[v][m1 + (M1 + 1) * m2];
                }
            for (int v = 0; v < NV; ++v) P.mortarG[mo + (long long)v * ns + t] = s[v];
        }
    }
}

// ---------------------------------------------------------------------------
// CFL time step (reading A11): affine
//   lambda = sum_d (|u_d| + c) (N_d+1)^2 / h_d,  dt = CFL / max lambda.
// ---------------------------------------------------------------------------

struct DtParams {
    const double* q;
    const WorkItem* work;
    const int* elist;
    const long long* off;
    const double* hgeo;
    double gamma;
    unsigned long long* maxbits;
};

__global__ void __launch_bounds__(BLOCK) k_dt(DtParams P)
{
    __shared__ double red[32];
    const WorkItem w = P.work[blockIdx.x];
    int N[3];
    unpack_ord(w.ord, N[0], N[1], N[2]);
    const int n = (N[0] + 1) * (N[1] + 1) * (N[2] + 1);
    double lmax = 0.0;
    for (int t = threadIdx.x; t < w.count * n; t += BLOCK) {
        const int slot = t / n, node = t - slot * n;
        const int e = P.elist[w.start + slot];
        const long long o = P.off[e] + node;
        double q[NV];
        for (int v = 0; v < NV; ++v) q[v] = P.q[o + (long long)v * n];
        const double ir = 1.0 / q[0];
        const double p = (P.gamma - 1.0) * (q[4] - 0.5 * ir * (q[1] * q[1] + q[2] * q[2] + q[3] * q[3]));
        const double c = sqrt(P.gamma * p * ir);
        double lam = 0.0;
        for (int d = 0; d < 3; ++d) {
            const double np1 = N[d] + 1.0;
            lam += (fabs(q[1 + d] * ir) + c) * np1 * np1 / P.hgeo[3 * e + d];
        }
        lmax = fmax(lmax, lam);
    }
    lmax = block_max(lmax, red);
    if (threadIdx.x == 0) atomicMax(P.maxbits, (unsigned long long)__double_as_longlong(lmax));
}

__global__ void k_dt_final(unsigned long long* maxbits, double cfl, double* dt)
{
    dt[0] = cfl / __longlong_as_double((long long)maxbits[0]);
    maxbits[0] = 0ull;  // ready for the next accumulation
}

// ---------------------------------------------------------------------------
// tau-estimation (eqs TEtildedef / TEdef; isolated coarse
// residuals P:469; decoupled directional levels, reading A12).  One CTA per
// element: for each direction d and coarse order p < N_d, the fine state is
// interpolated along d (I, reading A3), the isolated residual at the coarse
// orders is formed on chip, and
//   tau~ = I(Qdot_ref) - Qdot_c,   tau = J w w w tau~ (traditional),
//   tau[e][d][p] = max over coarse nodes and variables |tau|.
// ---------------------------------------------------------------------------

struct TauParams {
    const double* q;
    const double* qref;   // SOLVER reference or nullptr (SAME)
    double* tau;          // [E][3][9]
    const int* orders;
    const long long* off;
    const double* hgeo;
    const Tables* tab;
    int formulation;
    PhysDev ph;
};

// Isolated strong-form residual at orders O of a state held in registers for
// the CTA's owned nodes (t = tid + it*BLOCK < nO):  acc = sum_d (2/h_d) D f_d,
// i.e. Qdot = -acc.  Fs is scratch of 5*nO doubles.
__device__ __forceinline__ void iso_residual_regs(const int O[3], int nO, const double (&qc)[NPT][NV],
                                                  double (&acc)[NPT][NV], double* Fs, const double* h,
                                                  const Tables* tab, double gm1)
{
    const int tid = threadIdx.x;
    const int o1 = O[0] + 1, o2 = O[1] + 1;
#pragma unroll
    for (int it = 0; it < NPT; ++it)
#pragma unroll
        for (int v = 0; v < NV; ++v) acc[it][v] = 0.0;
    for (int d = 0; d < 3; ++d) {
#pragma unroll
        for (int it = 0; it < NPT; ++it) {
            const int t = tid + it * BLOCK;
            if (t < nO) {
                double f[NV], p;
                flux_dir(qc[it], gm1, d, f, &p);
                for (int v = 0; v < NV; ++v) Fs[v * nO + t] = f[v];
            }
        }
        __syncthreads();
        const int nd = O[d] + 1;
        const int stride = d == 0 ? 1 : (d == 1 ? o1 : o1 * o2);
        const double* Dd = tab->D[O[d]];
        const double sc = 2.0 / h[d];
#pragma unroll
        for (int it = 0; it < NPT; ++it) {
            const int t = tid + it * BLOCK;
            if (t < nO) {
                int ijk[3];
                node_ijk(t, o1, o2, ijk[0], ijk[1], ijk[2]);
                const int a = ijk[d];
                const int base = t - a * stride;
                for (int v = 0; v < NV; ++v) {
                    double s = 0.0;
                    for (int m = 0; m < nd; ++m) s += __ldg(&Dd[a * nd + m]) * Fs[v * nO + base + m * stride];
                    acc[it][v] += sc * s;
                }
            }
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(BLOCK) k_tau(TauParams P)
{
    extern __shared__ double sm[];
    __shared__ double red[32];
    const int e = blockIdx.x;
    const int tid = threadIdx.x;
    int N[3] = {P.orders[3 * e], P.orders[3 * e + 1], P.orders[3 * e + 2]};
    const int n1 = N[0] + 1, n2 = N[1] + 1, n3 = N[2] + 1;
    const int n = n1 * n2 * n3;
    double h[3] = {P.hgeo[3 * e], P.hgeo[3 * e + 1], P.hgeo[3 * e + 2]};
    const long long o = P.off[e];
    double* qs = sm;           // 5n
    double* Rs = qs + NV * n;  // 5n
    double* Fs = Rs + NV * n;  // 5n
    for (int t = tid; t < NV * n; t += BLOCK) qs[t] = P.q[o + t];
    const double gm1 = P.ph.gm1;
    double qc[NPT][NV], acc[NPT][NV];
    if (P.qref) {
        for (int t = tid; t < NV * n; t += BLOCK) Rs[t] = P.qref[o + t];
        __syncthreads();
    } else {  // SAME reference: isolated fine residual (reading A4)
        __syncthreads();
#pragma unroll
        for (int it = 0; it < NPT; ++it) {
            const int t = tid + it * BLOCK;
#pragma unroll
            for (int v = 0; v < NV; ++v) qc[it][v] = t < n ? qs[v * n + t] : 1.0;
        }
        iso_residual_regs(N, n, qc, acc, Fs, h, P.tab, gm1);
#pragma unroll
        for (int it = 0; it < NPT; ++it) {
            const int t = tid + it * BLOCK;
            if (t < n)
                for (int v = 0; v < NV; ++v) Rs[v * n + t] = -acc[it][v];
        }
        __syncthreads();
    }
    double rn = 0.0;
    for (int t = tid; t < NV * n; t += BLOCK) rn = fmax(rn, fabs(Rs[t]));
    rn = block_max(rn, red);
    if (tid == 0)
        for (int d = 0; d < 3; ++d) {
            P.tau[(3 * (long long)e + d) * DG_TAU_STRIDE_DEV + 0] = rn;
            for (int p = N[d]; p < DG_TAU_STRIDE_DEV; ++p)
                P.tau[(3 * (long long)e + d) * DG_TAU_STRIDE_DEV + p] = __longlong_as_double(0x7ff8000000000000LL);
        }
    const double Jel = h[0] * h[1] * h[2] / 8.0;
    for (int d = 0; d < 3; ++d) {
        const int nd = N[d] + 1;
        const int stride = d == 0 ? 1 : (d == 1 ? n1 : n1 * n2);
        for (int p = 1; p < N[d]; ++p) {
            int O[3] = {N[0], N[1], N[2]};
            O[d] = p;
            const int o1 = O[0] + 1, o2 = O[1] + 1;
            const int nO = o1 * o2 * (O[2] + 1);
            const double* T = P.tab->T[N[d]][p];
            // q_c = T^{N_d -> p} q along d
#pragma unroll
            for (int it = 0; it < NPT; ++it) {
                const int t = tid + it * BLOCK;
                if (t < nO) {
                    int ijk[3];
                    node_ijk(t, o1, o2, ijk[0], ijk[1], ijk[2]);
                    const int ic = ijk[d];
                    ijk[d] = 0;
                    const int base = ijk[0] + n1 * (ijk[1] + n2 * ijk[2]);
                    for (int v = 0; v < NV; ++v) {
                        double s = 0.0;
                        for (int a = 0; a < nd; ++a) s += __ldg(&T[ic * nd + a]) * qs[v * n + base + a * stride];
                        qc[it][v] = s;
                    }
                } else {
                    for (int v = 0; v < NV; ++v) qc[it][v] = 1.0;
                }
            }
            iso_residual_regs(O, nO, qc, acc, Fs, h, P.tab, gm1);
            double tmax = 0.0;
#pragma unroll
            for (int it = 0; it < NPT; ++it) {
                const int t = tid + it * BLOCK;
                if (t < nO) {
                    int ijk[3];
                    node_ijk(t, o1, o2, ijk[0], ijk[1], ijk[2]);
                    const int ic = ijk[d];
                    double scale = 1.0;
                    if (P.formulation == 1)
                        scale = Jel * P.tab->w[O[0]][ijk[0]] * P.tab->w[O[1]][ijk[1]] * P.tab->w[O[2]][ijk[2]];
                    ijk[d] = 0;
                    const int base = ijk[0] + n1 * (ijk[1] + n2 * ijk[2]);
                    for (int v = 0; v < NV; ++v) {
                        double s = 0.0;
                        for (int a = 0; a < nd; ++a) s += __ldg(&T[ic * nd + a]) * Rs[v * n + base + a * stride];
                        tmax = fmax(tmax, fabs(scale * (s + acc[it][v])));
                    }
                }
            }
            tmax = block_max(tmax, red);
            if (tid == 0) P.tau[(3 * (long long)e + d) * DG_TAU_STRIDE_DEV + p] = tmax;
        }
    }
}

// ---------------------------------------------------------------------------
// Map, extrapolation and selection (
// readings A12-A16).  One thread per element.
// ---------------------------------------------------------------------------

struct SelParams {
    const double* tau;
    const int* orders;
    double* total;     // [E][K^3] (static modes)
    int* sel;          // [E][3]
    double* margin;    // [E]
    int E;
    int mode;
    double tau_max;
    int Nmin, Nmax, dec_cap;
    int combine;   // 0 F_max, 1 F_av
    int nstages;   // n_e for the F_av finals
};

__device__ void directional_estimate(int Nd, const double* td, double* hat /* [NP+1] indexed by n */)
{
    const double SENT = 1e30;
    const double eps = 1e-13 * fmax(1.0, td[0]);
    double tmax = 0.0;
    for (int p = 1; p < Nd; ++p) tmax = fmax(tmax, td[p]);
    if (Nd <= 1) {  // not estimable: keep the order
        for (int m = 1; m <= NMAX; ++m) hat[m] = (m == Nd) ? 0.0 : SENT;
        return;
    }
    if (tmax <= eps) {  // resolved direction (A14)
        for (int m = 1; m <= NMAX; ++m) hat[m] = 0.0;
        return;
    }
    bool asym = false;
    double a = 0.0, b = 0.0;
    if (Nd >= 3) {  // ordinary least squares of log10 tau_d(p) on p (A13)
        const int K = Nd - 1;
        double sp = 0.0, sy = 0.0, spp = 0.0, spy = 0.0;
        for (int p = 1; p < Nd; ++p) {
            const double y = log10(fmax(td[p], 1e-300));
            sp += p;
            sy += y;
            spp += (double)p * p;
            spy += p * y;
        }
        b = (K * spy - sp * sy) / (K * spp - sp * sp);
        a = (sy - b * sp) / K;
        asym = b < 0.0;
    }
    for (int m = 1; m <= NMAX; ++m) {
        if (m < Nd) hat[m] = td[m];
        else hat[m] = asym ? pow(10.0, a + b * m) : SENT;
    }
}

__global__ void k_select(SelParams P)
{
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= P.E) return;
    double hat[3][NP + 1];
    int Ne[3];
    for (int d = 0; d < 3; ++d) {
        Ne[d] = P.orders[3 * e + d];
        directional_estimate(Ne[d], P.tau + (3 * (long long)e + d) * DG_TAU_STRIDE_DEV, hat[d]);
    }
    const int Nmin = P.Nmin, Nmax = P.Nmax, K = Nmax - Nmin + 1;
    double* tot = P.total ? P.total + (long long)e * K * K * K : nullptr;
    const bool a2 = P.mode == 1 || P.mode == 2, a1 = P.mode == 3 || P.mode == 4;
    if (a2) {  // approach 2: running F_max (eq totalTruncMap) or running sum (F_av) of the maps
        for (int n3 = Nmin; n3 <= Nmax; ++n3)
            for (int n2 = Nmin; n2 <= Nmax; ++n2)
                for (int n1 = Nmin; n1 <= Nmax; ++n1) {
                    const int ix = (n1 - Nmin) + K * ((n2 - Nmin) + K * (n3 - Nmin));
                    const double v = hat[0][n1] + hat[1][n2] + hat[2][n3];
                    tot[ix] = P.combine == 1 ? tot[ix] + v : fmax(tot[ix], v);
                }
        if (P.mode == 1) return;
    }
    const double nst = (P.mode == 2 && P.combine == 1) ? (double)P.nstages : 1.0;  // F_av: total / n_e
    int best[3] = {Nmax, Nmax, Nmax};
    long bestp = -1, bests = 0;
    double mg = INFINITY;
    for (int n1 = Nmin; n1 <= Nmax; ++n1)
        for (int n2 = Nmin; n2 <= Nmax; ++n2)
            for (int n3 = Nmin; n3 <= Nmax; ++n3) {
                const double v = !a2 ? hat[0][n1] + hat[1][n2] + hat[2][n3]
                                     : (P.combine == 1 ? tot[(n1 - Nmin) + K * ((n2 - Nmin) + K * (n3 - Nmin))] / nst
                                                       : tot[(n1 - Nmin) + K * ((n2 - Nmin) + K * (n3 - Nmin))]);
                mg = fmin(mg, fabs(v - P.tau_max) / P.tau_max);
                if (!(v < P.tau_max)) continue;
                const long pr = (long)(n1 + 1) * (n2 + 1) * (n3 + 1), sm = n1 + n2 + n3;
                if (bestp < 0 || pr < bestp || (pr == bestp && sm < bests)) {
                    bestp = pr;
                    bests = sm;
                    best[0] = n1; best[1] = n2; best[2] = n3;
                }
            }
    if (P.mode == 0)  // decrease cap
        for (int d = 0; d < 3; ++d) best[d] = max(best[d], Ne[d] - P.dec_cap);
    if (a1) {  // approach 1: combine this stage's degrees, N_i^e = F(N_i^{e,s})
        double* acc = P.total + 3LL * e;
        for (int d = 0; d < 3; ++d) acc[d] = P.combine == 1 ? acc[d] + best[d] : fmax(acc[d], (double)best[d]);
        if (P.mode == 3) return;
        for (int d = 0; d < 3; ++d) {  // F_av: mean rounded half up (reading R8)
            const int Nd = P.combine == 1 ? (int)floor(acc[d] / P.nstages + 0.5) : (int)acc[d];
            best[d] = min(max(Nd, Nmin), Nmax);
        }
    }
    for (int d = 0; d < 3; ++d) P.sel[3 * e + d] = best[d];
    if (P.margin) P.margin[e] = mg;
}

// Jump condition (eqs N23 / N_1): one Jacobi sweep of the monotone fixpoint.
__global__ void k_jump(const int* nbr, const int* in, int* out, int E, int rule, int Nmax, int* changed)
{
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= E) return;
    for (int d = 0; d < 3; ++d) {
        const int cur = in[3 * e + d];
        int v = cur;
        for (int f = 0; f < 6; ++f) {
            const int j = nbr[6 * e + f];
            if (j < 0) continue;
            const int x = in[3 * j + d];
            const int r = rule == 0 ? (2 * x) / 3 : x - 1;
            v = max(v, r);
        }
        v = max(cur, min(v, Nmax));
        out[3 * e + d] = v;
        if (v != cur) atomicOr(changed, 1);
    }
}

// Jump-condition least fixpoint in ONE launch: a single CTA runs
// the Jacobi sweeps of k_jump with a block barrier between sweeps until no
// order changes; the result ends in `a`.  For local meshes without halo rows.
constexpr int JUMP_FIX_BS = 1024;

__global__ void __launch_bounds__(JUMP_FIX_BS) k_jump_fix(const int* nbr, int* a, int* b, int E, int rule, int Nmax,
                                                          int maxsweeps)
{
    __shared__ int changed;
    int* in = a;
    int* out = b;
    for (int sweep = 0; sweep < maxsweeps; ++sweep) {
        if (threadIdx.x == 0) changed = 0;
        __syncthreads();
        for (int e = threadIdx.x; e < E; e += JUMP_FIX_BS)
            for (int d = 0; d < 3; ++d) {
                const int cur = in[3 * e + d];
                int v = cur;
                for (int f = 0; f < 6; ++f) {
                    const int j = nbr[6 * e + f];
                    if (j < 0) continue;
                    const int x = in[3 * j + d];
                    v = max(v, rule == 0 ? (2 * x) / 3 : x - 1);
                }
                v = max(cur, min(v, Nmax));
                out[3 * e + d] = v;
                if (v != cur) changed = 1;
            }
        __syncthreads();  // sweep complete and visible to the block
        int* t = in;
        in = out;
        out = t;
        if (!changed) break;
        __syncthreads();  // everyone has read `changed` before it is reset
    }
    if (in != a)
        for (int i = threadIdx.x; i < 3 * E; i += JUMP_FIX_BS) a[i] = in[i];
}

// ---------------------------------------------------------------------------
// Transfer: q_new = T_z T_y T_x q_old per element.
// ---------------------------------------------------------------------------

struct TransferParams {
    int smax0, smax1, smax2;  // max over elements of nA, n1, n2 (shared-memory layout)
    int restr;                // decreasing directions by the L2 projection P (A3 flag), else interpolation T
    const double* qold;
    double* qnew;
    const int* oold;
    const int* onew;
    const long long* offold;
    const long long* offnew;
    const Tables* tab;
};

// one tensor pass along a direction of a [v][c2][c1][c0] block in shared
// memory: nl lines per variable with input stride st, the m outputs of a line
// from its a inputs (T zero padded 9 x 9, row i = output i)
__device__ __forceinline__ void tr_pass(const double* __restrict__ T, const double* __restrict__ in,
                                        double* __restrict__ out, int nin, int nout, int nl, int lines_per_plane,
                                        int plane_in, int plane_out, int a, int m, int st)
{
    for (int task = threadIdx.x; task < NV * nl; task += blockDim.x) {
        const int v = task / nl, l = task - v * nl;
        const int pl = l / lines_per_plane, r = l - pl * lines_per_plane;  // (outer, inner) index of the line
        const double* x0 = in + v * nin + pl * plane_in + r;
        double* o = out + v * nout + pl * plane_out + r;
        double x[NP];
#pragma unroll
        for (int b = 0; b < NP; ++b) x[b] = b < a ? x0[b * st] : 0.0;
        for (int i = 0; i < m; ++i) {
            double s = 0.0;
#pragma unroll
            for (int b = 0; b < NP; ++b)
                if (b < a) s += T[i * NP + b] * x[b];
            o[i * st] = s;
        }
    }
}

__global__ void __launch_bounds__(BLOCK) k_transfer(TransferParams P)
{
    // per direction: T^{A_d -> B_d} along lines (identity passes skipped: the
    // table is exactly the identity then); [v][k][j][i] blocks in shared memory
    extern __shared__ double sm[];
    __shared__ double Ts[3][NP * NP];
    const int e = blockIdx.x;
    int A[3], B[3];
    for (int d = 0; d < 3; ++d) { A[d] = P.oold[3 * e + d] + 1; B[d] = P.onew[3 * e + d] + 1; }
    for (int t = threadIdx.x; t < 3 * NP * NP; t += blockDim.x) {
        const int d = t / (NP * NP), r = t - d * (NP * NP), i = r / NP, b = r - i * NP;
        Ts[d][r] = (i < B[d] && b < A[d]) ? ((P.restr && B[d] < A[d]) ? P.tab->P[A[d] - 1][B[d] - 1]
                                                                       : P.tab->T[A[d] - 1][B[d] - 1])[i * A[d] + b]
                                          : 0.0;
    }
    const int nA = A[0] * A[1] * A[2];
    double* buf[2] = {sm, sm + NV * P.smax0};
    double* s2 = sm + NV * (P.smax0 + P.smax1);
    const long long oa = P.offold[e], ob = P.offnew[e];
    for (int t = threadIdx.x; t < NV * nA; t += blockDim.x) buf[0][t] = P.qold[oa + t];
    __syncthreads();
    int c[3] = {A[0], A[1], A[2]};
    const double* cur = buf[0];
    int ncur = nA, nb = 0;
    for (int d = 0; d < 3; ++d) {
        if (A[d] == B[d]) continue;
        double* out = (nb == 0) ? buf[1] : (cur == buf[1] ? s2 : buf[1]);
        nb = 1;
        const int st = d == 0 ? 1 : (d == 1 ? c[0] : c[0] * c[1]);
        const int inner = st;                               // lines per plane (indices below d)
        const int outer = d == 0 ? c[1] * c[2] : (d == 1 ? c[2] : 1);
        const int nout = ncur / c[d] * B[d];
        tr_pass(Ts[d], cur, out, ncur, nout, inner * outer, inner, inner * c[d], inner * B[d], c[d], B[d], st);
        c[d] = B[d];
        ncur = nout;
        cur = out;
        __syncthreads();
    }
    for (int t = threadIdx.x; t < NV * ncur; t += blockDim.x) P.qnew[ob + t] = cur[t];
}

// ---------------------------------------------------------------------------
// Diagnostics: sum over nodes of (J w w w) v per variable; min rho, min p.
// ---------------------------------------------------------------------------

struct DiagParams {
    const double* q;
    const double* v;
    const int* orders;
    const long long* off;
    const double* hgeo;
    const double* met;             // curved: metric array (J at component 9), else nullptr
    const Tables* tab;
    double gamma;
    double* sums;                  // [5]
    unsigned long long* minbits;   // [2] (as ordered bits of positive doubles; negative -> 0)
    int* neg;                      // count of non-positive rho/p
};

__global__ void __launch_bounds__(BLOCK) k_diag(DiagParams P)
{
    const int e = blockIdx.x;
    int N[3] = {P.orders[3 * e], P.orders[3 * e + 1], P.orders[3 * e + 2]};
    const int n1 = N[0] + 1, n2 = N[1] + 1, n = n1 * n2 * (N[2] + 1);
    const long long o = P.off[e];
    const double Ja = P.met ? 0.0 : P.hgeo[3 * e] * P.hgeo[3 * e + 1] * P.hgeo[3 * e + 2] / 8.0;
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
        int i, j, k;
        node_ijk(t, n1, n2, i, j, k);
        const double J = P.met ? P.met[2 * o + 9 * n + t] : Ja;
        const double m = J * P.tab->w[N[0]][i] * P.tab->w[N[1]][j] * P.tab->w[N[2]][k];
        if (P.v)
            for (int v = 0; v < NV; ++v) atomicAdd(&P.sums[v], m * P.v[o + (long long)v * n + t]);
        double q[NV];
        for (int v = 0; v < NV; ++v) q[v] = P.q[o + (long long)v * n + t];
        const double p = (P.gamma - 1.0) * (q[4] - 0.5 * (q[1] * q[1] + q[2] * q[2] + q[3] * q[3]) / q[0]);
        if (!(q[0] > 0.0) || !(p > 0.0)) atomicAdd(P.neg, 1);
        else {
            atomicMin(&P.minbits[0], (unsigned long long)__double_as_longlong(q[0]));
            atomicMin(&P.minbits[1], (unsigned long long)__double_as_longlong(p));
        }
    }
}

}  // namespace dgtau
