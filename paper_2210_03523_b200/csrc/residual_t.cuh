// residual_t.cuh -- order-specialised fused DGSEM residual / RK-stage kernel.
//
// One template instance per (N1,N2,N3) bucket; a CTA processes CNT elements of
// that bucket (work items of the plan, spatially ordered).  Same numerics as
// the generic path (strong-form GL-DGSEM, see kernels.cuh header; PAPER.md
// P:129-155), arranged for the sm_100a fp64 pipes:
//   * element state read once from HBM into registers of node-owner threads
//     (ir = 1/rho and p computed once per node);
//   * per direction d the node owners write f_d to shared memory, then one
//     thread per (line, variable) holds the line in registers and applies
//     D^{N_d} with compile-time loops; D comes from __constant__ memory with
//     compile-time offsets (constant-bank operands of DFMA);
//   * surface: one thread per (face, face point), packed over the 6 faces of
//     all CTA elements; Roe flux with the neighbour trace read from L2;
//     (G - f_own) * lifting scale goes to shared memory;
//   * epilogue per node: Qdot = -(volume + lifting), or the Williamson
//     low-storage update g <- A g + dt Qdot, q' <- q + B g.
#pragma once

#include <cuda_runtime.h>

#include "common.cuh"

namespace dgtau {

// D^{N}[a][m] at c_D[N*NP*NP + a*(N+1) + m] and GL weights; one private copy
// per translation unit (internal linkage), filled by res_setup_* at startup.
static __constant__ double c_D[NP * NP * NP];
static __constant__ double c_w[NP][NP];
// even-odd (centro-antisymmetric, D_{N-a,N-m} = -D_{a,m}) split of D^N,
// H = floor((N+1)/2):  P[a][m] = (D_am - D_{a,N-m})/2, Q[a][m] = (D_am + D_{a,N-m})/2
// for a, m < H;  Qm[a] = D_{a,mid} (odd N+1);  M[m] = D_{mid,m} (odd N+1).
static __constant__ double c_EOP[NP][16];
static __constant__ double c_EOQ[NP][16];
static __constant__ double c_EOQm[NP][4];
static __constant__ double c_EOM[NP][4];

__host__ __device__ constexpr int cmin(int a, int b) { return a < b ? a : b; }
__host__ __device__ constexpr int cmax(int a, int b) { return a > b ? a : b; }

template <int N1, int N2, int N3>
struct Shape {
    static constexpr int n1 = N1 + 1, n2 = N2 + 1, n3 = N3 + 1;
    static constexpr int n = n1 * n2 * n3;
    // <= ~384 nodes per CTA so nodes, (line, variable) tasks and face tasks
    // each take one round of threads (no half-empty second rounds before the
    // barriers); two node passes only for n > 384.
    static constexpr int CNT = cmax(1, cmin(MAXSLOTS, 384 / n));
    static constexpr int T = CNT * n;
    static constexpr int NPT = T > 384 ? 2 : 1;
    static constexpr int BS = ((T + NPT - 1) / NPT + 31) / 32 * 32;
    static constexpr int nf0 = n2 * n3, nf1 = n1 * n3, nf2 = n1 * n2;
    static constexpr int FS = 2 * (nf0 + nf1 + nf2);
    // Q (5T) + F (5T) + RK register g (5T) + IR,P (2T) + outer traces / lifting terms (5 FS per element)
    static constexpr size_t smem_bytes = sizeof(double) * (size_t)(17 * T + NV * CNT * FS);
    static constexpr int MINB = BS <= 128 ? 4 : (BS <= 192 ? 3 : (BS <= 384 ? 2 : 1));
};

// f . e_d for the Euler flux, from q with precomputed 1/rho and p
template <int d>
__device__ __forceinline__ void flux_axis(const double* q, double ir, double p, double* f)
{
    const double ud = q[1 + d] * ir;
    f[0] = q[1 + d];
    f[1] = q[1] * ud;
    f[2] = q[2] * ud;
    f[3] = q[3] * ud;
    f[1 + d] += p;
    f[4] = (q[4] + p) * ud;
}

// Euler flux along a unit normal given as three scalars (no dynamic indexing)
__device__ __forceinline__ void flux_normal(const double* q, double nx, double ny, double nz, double gm1, double* f)
{
    const double ir = 1.0 / q[0];
    const double p = gm1 * (q[4] - 0.5 * ir * (q[1] * q[1] + q[2] * q[2] + q[3] * q[3]));
    const double un = (q[1] * nx + q[2] * ny + q[3] * nz) * ir;
    f[0] = q[0] * un;
    f[1] = q[1] * un + p * nx;
    f[2] = q[2] * un + p * ny;
    f[3] = q[3] * un + p * nz;
    f[4] = (q[4] + p) * un;
}

// In-place derivative of one line held in shared memory, F[m*stride] <-
// sum_m D_am F_m, by the even-odd decomposition of the GL differentiation
// matrix (about half the multiply-adds of the direct product):
//   o_m = v_m - v_{N-m}, e_m = v_m + v_{N-m}  (m < H),
//   out_a = sum_m P_am o_m + (sum_m Q_am e_m + Qm_a v_mid),
//   out_{N-a} = sum_m P_am o_m - (sum_m Q_am e_m + Qm_a v_mid),
//   out_mid = sum_m M_m o_m.
template <int L>
__device__ __forceinline__ void dline_inplace(double* Fl, int stride)
{
    constexpr int N = L - 1, H = L / 2;
    constexpr bool odd = (L & 1) != 0;
    double v[L];
#pragma unroll
    for (int m = 0; m < L; ++m) v[m] = Fl[m * stride];
    double o[H], ev[H];
#pragma unroll
    for (int m = 0; m < H; ++m) {
        o[m] = v[m] - v[N - m];
        ev[m] = v[m] + v[N - m];
    }
#pragma unroll
    for (int a = 0; a < H; ++a) {
        double p = c_EOP[N][a * H] * o[0];
        double q = c_EOQ[N][a * H] * ev[0];
#pragma unroll
        for (int m = 1; m < H; ++m) {
            p = fma(c_EOP[N][a * H + m], o[m], p);
            q = fma(c_EOQ[N][a * H + m], ev[m], q);
        }
        if (odd) q = fma(c_EOQm[N][a], v[H], q);
        Fl[a * stride] = p + q;
        Fl[(N - a) * stride] = p - q;
    }
    if (odd) {
        double s = c_EOM[N][0] * o[0];
#pragma unroll
        for (int m = 1; m < H; ++m) s = fma(c_EOM[N][m], o[m], s);
        Fl[H * stride] = s;
    }
}

__device__ __forceinline__ void cp_async8(double* dst, const double* src)
{
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src));
}

// decode face task r in [0, FS) -> face f and point pt
template <class S>
__device__ __forceinline__ void face_of(int r, int& f, int& pt)
{
    if (r < 2 * S::nf0) {
        f = r < S::nf0 ? 0 : 1;
        pt = r - f * S::nf0;
    } else if (r < 2 * (S::nf0 + S::nf1)) {
        const int r1 = r - 2 * S::nf0;
        f = r1 < S::nf1 ? 2 : 3;
        pt = r1 - (f - 2) * S::nf1;
    } else {
        const int r2 = r - 2 * (S::nf0 + S::nf1);
        f = r2 < S::nf2 ? 4 : 5;
        pt = r2 - (f - 4) * S::nf2;
    }
}

// Roe flux (no entropy fix, reading A7) for the axis normal e_d, with
// 1/rho and p of both states precomputed (same algebra as roe_flux with n = e_d).
template <int d>
__device__ __forceinline__ void roe_axis(const double* qL, double irL, double pL, const double* qR, double irR,
                                         double pR, double gamma, double* F)
{
    const double gm1 = gamma - 1.0;
    double uL[3], uR[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) { uL[k] = qL[1 + k] * irL; uR[k] = qR[1 + k] * irR; }
    const double HL = (qL[4] + pL) * irL, HR = (qR[4] + pR) * irR;
    const double sL = sqrt(qL[0]), sR = sqrt(qR[0]);
    const double is = 1.0 / (sL + sR);
    const double wl = sL * is, wr = sR * is;
    double u[3], du[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) { u[k] = wl * uL[k] + wr * uR[k]; du[k] = uR[k] - uL[k]; }
    const double H = wl * HL + wr * HR;
    const double uu = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
    const double c2 = gm1 * (H - 0.5 * uu);
    const double c = sqrt(c2);
    const double ic2 = 1.0 / c2;
    const double un = u[d], dun = du[d];
    const double rho = sL * sR;
    const double dp = pR - pL;
    const double rcd = rho * c * dun;
    const double a1 = 0.5 * (dp - rcd) * ic2, a5 = 0.5 * (dp + rcd) * ic2;
    const double a2 = (qR[0] - qL[0]) - dp * ic2;
    const double w1 = fabs(un - c) * a1, w5 = fabs(un + c) * a5, l2 = fabs(un);
    const double mL = qL[1 + d], mR = qR[1 + d];
    F[0] = 0.5 * (mL + mR) - 0.5 * (w1 + l2 * a2 + w5);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        double fk = qL[1 + k] * uL[d] + qR[1 + k] * uR[d];
        double dk = (w1 + w5) * u[k] + l2 * (a2 * u[k] + rho * du[k]);
        if (k == d) {
            fk += pL + pR;
            dk += c * (w5 - w1) - l2 * rho * dun;
        }
        F[1 + k] = 0.5 * fk - 0.5 * dk;
    }
    const double udu = u[0] * du[0] + u[1] * du[1] + u[2] * du[2];
    const double fe = (qL[4] + pL) * uL[d] + (qR[4] + pR) * uR[d];
    const double de = (w1 + w5) * H + un * c * (w5 - w1) + l2 * (a2 * 0.5 * uu + rho * (udu - un * dun));
    F[4] = 0.5 * fe - 0.5 * de;
}

// surface term of one face point for the compile-time axis d: G - f_own
template <int d>
__device__ __forceinline__ void face_point(const double* qo, double iro, double po, double* qx, int kind, int s,
                                           const PhysDev& ph, double* out)
{
    double fo[NV], G[NV];
    flux_axis<d>(qo, iro, po, fo);
    if (kind == 1) {
#pragma unroll
        for (int v = 0; v < NV; ++v) G[v] = qx[v];
    } else {
        if (kind >= 2) ghost_state(qo, kind == 2 ? -1 : -2, ph, qx);
        if (ph.flux == 1) {
            double nrm[3] = {d == 0 ? 1.0 : 0.0, d == 1 ? 1.0 : 0.0, d == 2 ? 1.0 : 0.0};
            if (s) llf_flux(qo, qx, nrm, ph.gamma, G); else llf_flux(qx, qo, nrm, ph.gamma, G);
        } else {
            const double irx = 1.0 / qx[0];
            const double px = ph.gm1 * (qx[4] - 0.5 * irx * (qx[1] * qx[1] + qx[2] * qx[2] + qx[3] * qx[3]));
            if (s) roe_axis<d>(qo, iro, po, qx, irx, px, ph.gamma, G);
            else roe_axis<d>(qx, irx, px, qo, iro, po, ph.gamma, G);
        }
    }
#pragma unroll
    for (int v = 0; v < NV; ++v) out[v] = G[v] - fo[v];
}

template <int N1, int N2, int N3>
__global__ void __launch_bounds__(Shape<N1, N2, N3>::BS, Shape<N1, N2, N3>::MINB) k_res_t(ResParams P, int item0)
{
    using S = Shape<N1, N2, N3>;
    constexpr int n = S::n, n1 = S::n1, n2 = S::n2, n3 = S::n3, BS = S::BS, NPTT = S::NPT, FS = S::FS;
    constexpr int T = S::T;
    extern __shared__ double sm[];
    double* Q = sm;               // [slot][v][node]  state
    double* F = Q + NV * T;       // [slot][v][node]  flux of one direction, then its derivative
    double* IR = F + NV * T;      // [slot*n + node]  1/rho
    double* PR = IR + T;          // [slot*n + node]  pressure
    double* GB = PR + T;          // [slot][v][node]  RK register g (prefetched)
    double* X = GB + NV * T;      // [slot][v][face point]  outer traces, then lifting terms
    __shared__ long long s_off[S::CNT];
    __shared__ int s_e[S::CNT];
    __shared__ double s_sc[S::CNT][3];

    const WorkItem w = P.work[item0 + blockIdx.x];
    const int cnt = w.count;
    const int tid = threadIdx.x;
    if (tid < cnt) {
        const SlotInfo si = P.slots[w.start + tid];
        s_e[tid] = si.e;
        s_off[tid] = si.off;
#pragma unroll
        for (int d = 0; d < 3; ++d) s_sc[tid][d] = si.sc[d];
    }
    __syncthreads();
    const double gm1 = P.ph.gm1;
    const int ntot = cnt * n;
    const bool surf = P.variant == 0;

    // ---- outer traces / mortar fluxes: asynchronous gather into X ---------
    if (surf) {
        for (int t = tid; t < cnt * FS; t += BS) {
            const int slot = t / FS;
            const int r = t - slot * FS;
            int f, pt;
            face_of<S>(r, f, pt);
            const FaceInfo fi = P.finfo[6 * s_e[slot] + f];
            const int nta = f < 2 ? n2 : n1;
            const int ta = pt % nta, tb = pt / nta;
            if (fi.kind == 0) {
                const double* src = P.q + fi.off + fi.base + ta * fi.sa + tb * fi.sb;
#pragma unroll
                for (int v = 0; v < NV; ++v) cp_async8(&X[(slot * NV + v) * FS + r], src + (long long)v * fi.n);
            } else if (fi.kind == 1) {
                const double* src = P.mortarG + fi.off + pt;
#pragma unroll
                for (int v = 0; v < NV; ++v) cp_async8(&X[(slot * NV + v) * FS + r], src + (long long)v * fi.n);
            }
        }
        asm volatile("cp.async.commit_group;\n" ::);
    }

    // ---- RK register g: asynchronous prefetch (needed only in the epilogue)
    const bool need_g = P.mode == 1 && P.rkA != 0.0;
    if (need_g) {
#pragma unroll
        for (int it = 0; it < NPTT; ++it) {
            const int t = tid + it * BS;
            if (t < ntot) {
                const int slot = t / n, node = t - slot * n;
                const double* ge = P.g + s_off[slot] + node;
#pragma unroll
                for (int v = 0; v < NV; ++v) cp_async8(&GB[(slot * NV + v) * n + node], ge + v * n);
            }
        }
    }
    asm volatile("cp.async.commit_group;\n" ::);

    // ---- state into shared memory (coalesced), 1/rho and p once per node -
#pragma unroll
    for (int it = 0; it < NPTT; ++it) {
        const int t = tid + it * BS;
        if (t < ntot) {
            const int slot = t / n, node = t - slot * n;
            const double* qe = P.q + s_off[slot] + node;
            double qv[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                qv[v] = qe[v * n];
                Q[(slot * NV + v) * n + node] = qv[v];
            }
            const double ir = 1.0 / qv[0];
            const double p = gm1 * (qv[4] - 0.5 * ir * (qv[1] * qv[1] + qv[2] * qv[2] + qv[3] * qv[3]));
            IR[t] = ir;
            PR[t] = p;
            if (!(qv[0] > 0.0 && p > 0.0)) {
                if (atomicAdd(P.flag, 1) == 0) P.flag[1] = s_e[slot];
            }
        }
    }

    // ---- volume term, direction by direction ------------------------------
    double acc[NPTT][NV];
#pragma unroll
    for (int it = 0; it < NPTT; ++it)
#pragma unroll
        for (int v = 0; v < NV; ++v) acc[it][v] = 0.0;

#pragma unroll
    for (int d = 0; d < 3; ++d) {
        if (d > 0) __syncthreads();  // previous direction's derivatives consumed
#pragma unroll
        for (int it = 0; it < NPTT; ++it) {
            const int t = tid + it * BS;
            if (t < ntot) {
                const int slot = t / n, node = t - slot * n;
                double qv[NV], f[NV];
#pragma unroll
                for (int v = 0; v < NV; ++v) qv[v] = Q[(slot * NV + v) * n + node];
                if (d == 0) flux_axis<0>(qv, IR[t], PR[t], f);
                else if (d == 1) flux_axis<1>(qv, IR[t], PR[t], f);
                else flux_axis<2>(qv, IR[t], PR[t], f);
#pragma unroll
                for (int v = 0; v < NV; ++v) F[(slot * NV + v) * n + node] = f[v];
            }
        }
        __syncthreads();
        constexpr int Ld[3] = {n1, n2, n3};
        const int nlines = n / Ld[d];
        for (int task = tid; task < cnt * NV * nlines; task += BS) {
            const int sv = task / nlines;  // slot * NV + v
            const int l = task - sv * nlines;
            if (d == 0) dline_inplace<n1>(F + sv * n + l * n1, 1);
            else if (d == 1) dline_inplace<n2>(F + sv * n + (l % n1) + n1 * n2 * (l / n1), n1);
            else dline_inplace<n3>(F + sv * n + l, n1 * n2);
        }
        __syncthreads();
#pragma unroll
        for (int it = 0; it < NPTT; ++it) {
            const int t = tid + it * BS;
            if (t < ntot) {
                const int slot = t / n, node = t - slot * n;
                const double sc = s_sc[slot][d];
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    acc[it][v] = fma(sc, F[(slot * NV + v) * n + node], acc[it][v]);
                    if (d == 2) F[(slot * NV + v) * n + node] = acc[it][v];  // park: frees registers
                }
            }
        }
    }

    // ---- surface: lifting terms +-(G - f_own) 2/(h_d w_end) into X ---------
    if (surf) {
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        __syncthreads();
        for (int t = tid; t < cnt * FS; t += BS) {
            const int slot = t / FS;
            const int r = t - slot * FS;
            int f, pt;
            face_of<S>(r, f, pt);
            const int d = f >> 1, s = f & 1;
            const int nta = d == 0 ? n2 : n1;
            const int ta = pt % nta, tb = pt / nta;
            int i, j, k, Nd;
            if (d == 0) { i = s ? N1 : 0; j = ta; k = tb; Nd = N1; }
            else if (d == 1) { i = ta; j = s ? N2 : 0; k = tb; Nd = N2; }
            else { i = ta; j = tb; k = s ? N3 : 0; Nd = N3; }
            const int node = i + n1 * (j + n2 * k);
            double qo[NV], qx[NV], out[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                qo[v] = Q[(slot * NV + v) * n + node];
                qx[v] = X[(slot * NV + v) * FS + r];
            }
            const double iro = IR[slot * n + node], po = PR[slot * n + node];
            const int kind = P.finfo[6 * s_e[slot] + f].kind;
            if (d == 0) face_point<0>(qo, iro, po, qx, kind, s, P.ph, out);
            else if (d == 1) face_point<1>(qo, iro, po, qx, kind, s, P.ph, out);
            else face_point<2>(qo, iro, po, qx, kind, s, P.ph, out);
            const double sc = (s ? 1.0 : -1.0) * s_sc[slot][d] / c_w[Nd][0];
#pragma unroll
            for (int v = 0; v < NV; ++v) X[(slot * NV + v) * FS + r] = sc * out[v];
        }
        __syncthreads();
    }

    // ---- epilogue per node --------------------------------------------------
    const double dt = P.mode ? *P.dt : 0.0;
    double lmax = 0.0;
    if (need_g) asm volatile("cp.async.wait_group 0;\n" ::: "memory");  // own g values only
#pragma unroll
    for (int it = 0; it < NPTT; ++it) {
        const int t = tid + it * BS;
        if (t >= ntot) continue;
        const int slot = t / n, node = t - slot * n;
        double accv[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) accv[v] = F[(slot * NV + v) * n + node];
        if (surf) {
            const int i = node % n1, j = (node / n1) % n2, k = node / (n1 * n2);
            const double* Xb = X + slot * NV * FS;
            if (i == 0 || i == N1) {
                const int r = (i == 0 ? 0 : S::nf0) + j + n2 * k;
#pragma unroll
                for (int v = 0; v < NV; ++v) accv[v] += Xb[v * FS + r];
            }
            if (j == 0 || j == N2) {
                const int r = 2 * S::nf0 + (j == 0 ? 0 : S::nf1) + i + n1 * k;
#pragma unroll
                for (int v = 0; v < NV; ++v) accv[v] += Xb[v * FS + r];
            }
            if (k == 0 || k == N3) {
                const int r = 2 * (S::nf0 + S::nf1) + (k == 0 ? 0 : S::nf2) + i + n1 * j;
#pragma unroll
                for (int v = 0; v < NV; ++v) accv[v] += Xb[v * FS + r];
            }
        }
        double* o = P.out + s_off[slot] + node;
        if (P.mode == 0) {
#pragma unroll
            for (int v = 0; v < NV; ++v) o[v * n] = -accv[v];
        } else {
            double* g = P.g + s_off[slot] + node;
            double qn[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                const double gn = (need_g ? P.rkA * GB[(slot * NV + v) * n + node] : 0.0) - dt * accv[v];
                g[v * n] = gn;
                qn[v] = Q[(slot * NV + v) * n + node] + P.rkB * gn;
                o[v * n] = qn[v];
            }
            if (P.lam_max) {  // CFL rate of q^{n+1} (reading A11), fused
                const double ir = 1.0 / qn[0];
                const double p = (P.gamma - 1.0) * (qn[4] - 0.5 * ir * (qn[1] * qn[1] + qn[2] * qn[2] + qn[3] * qn[3]));
                const double c = sqrt(P.gamma * p * ir);
                constexpr double L1 = (double)n1 * n1, L2 = (double)n2 * n2, L3 = (double)n3 * n3;
                const double lam = 0.5 * ((fabs(qn[1] * ir) + c) * L1 * s_sc[slot][0] +
                                          (fabs(qn[2] * ir) + c) * L2 * s_sc[slot][1] +
                                          (fabs(qn[3] * ir) + c) * L3 * s_sc[slot][2]);
                lmax = fmax(lmax, lam);
            }
        }
    }
    if (P.lam_max) {
        __shared__ double red[32];
        lmax = block_max(lmax, red);
        if (threadIdx.x == 0) atomicMax(P.lam_max, (unsigned long long)__double_as_longlong(lmax));
    }
}

// host-side: launcher table filled by the instantiation units
typedef void (*res_launcher)(const ResParams& P, int item0, int nitems, cudaStream_t st);

static inline cudaError_t res_copy_constants(const Tables* host)
{
    cudaError_t e = cudaMemcpyToSymbol(c_D, host->D, sizeof(c_D));
    if (e != cudaSuccess) return e;
    if ((e = cudaMemcpyToSymbol(c_w, host->w, sizeof(c_w))) != cudaSuccess) return e;
    double P[NP][16] = {}, Q[NP][16] = {}, Qm[NP][4] = {}, M[NP][4] = {};
    for (int N = 1; N <= NMAX; ++N) {
        const int L = N + 1, H = L / 2;
        const double* D = host->D[N];
        for (int a = 0; a < H; ++a)
            for (int m = 0; m < H; ++m) {
                P[N][a * H + m] = 0.5 * (D[a * L + m] - D[a * L + (N - m)]);
                Q[N][a * H + m] = 0.5 * (D[a * L + m] + D[a * L + (N - m)]);
            }
        if (L & 1)
            for (int a = 0; a < H; ++a) {
                Qm[N][a] = D[a * L + H];
                M[N][a] = D[H * L + a];
            }
    }
    if ((e = cudaMemcpyToSymbol(c_EOP, P, sizeof(P))) != cudaSuccess) return e;
    if ((e = cudaMemcpyToSymbol(c_EOQ, Q, sizeof(Q))) != cudaSuccess) return e;
    if ((e = cudaMemcpyToSymbol(c_EOQm, Qm, sizeof(Qm))) != cudaSuccess) return e;
    return cudaMemcpyToSymbol(c_EOM, M, sizeof(M));
}

template <int N1, int N2, int N3>
void launch_res_t(const ResParams& P, int item0, int nitems, cudaStream_t st)
{
    using S = Shape<N1, N2, N3>;
    k_res_t<N1, N2, N3><<<nitems, S::BS, S::smem_bytes, st>>>(P, item0);
}

template <int N1, int N2, int N3>
cudaError_t attr_res_t()
{
    using S = Shape<N1, N2, N3>;
    cudaError_t e = cudaFuncSetAttribute(k_res_t<N1, N2, N3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)S::smem_bytes);
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(k_res_t<N1, N2, N3>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                (int)cudaSharedmemCarveoutMaxShared);
}

}  // namespace dgtau
