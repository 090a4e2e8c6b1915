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
    // F (5T) + IR,P (2T) + 2 pipeline stages x {Q (5T), g (5T), outer traces (5 FS per element)}
    // + 3 meta buffers (slot info + face descriptors)
    static constexpr size_t smem_bytes =
        sizeof(double) * (size_t)(7 * T + 2 * (10 * T + NV * CNT * FS) + 3 * CNT * (5 + 24));
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

// Per-item metadata staged in shared memory: slot info (5 doubles) and the 6
// face descriptors (4 doubles each) of every element of the item.
constexpr int META_SLOT_W = 5, META_FACE_W = 4;

template <int N1, int N2, int N3>
__global__ void __launch_bounds__(Shape<N1, N2, N3>::BS, Shape<N1, N2, N3>::MINB)
    k_res_t(ResParams P, int start0, int nelem, int nitems)
{
    using S = Shape<N1, N2, N3>;
    constexpr int n = S::n, n1 = S::n1, n2 = S::n2, n3 = S::n3, BS = S::BS, NPTT = S::NPT, FS = S::FS;
    constexpr int T = S::T, CNT = S::CNT;
    constexpr int MW = CNT * (META_SLOT_W + 6 * META_FACE_W);  // meta words per item
    extern __shared__ double sm[];
    double* F = sm;                   // [slot][v][node]  flux of one direction, then its derivative
    double* IR = F + NV * T;          // 1/rho
    double* PR = IR + T;              // pressure
    double* STG = PR + T;             // 2 pipeline stages of {Q 5T, GB 5T, X 5 CNT FS}
    constexpr int STAGE = 10 * T + NV * CNT * FS;
    double* META = STG + 2 * STAGE;   // 3 meta buffers of MW words
    __shared__ double red[32];

    const int tid = threadIdx.x;
    const bool surf = P.variant == 0;
    const bool need_g = P.mode == 1 && P.rkA != 0.0;
    const double gm1 = P.ph.gm1;
    const int G = gridDim.x;

    auto item_cnt = [&](int item) { return min(CNT, nelem - item * CNT); };
    // meta (slot info + face descriptors) of `item` into meta buffer mb
    auto issue_meta = [&](int item, int mb) {
        double* M = META + mb * MW;
        const int cnt = item_cnt(item);
        const int start = start0 + item * CNT;
        const double* sl = reinterpret_cast<const double*>(P.slots + start);
        const double* fl = reinterpret_cast<const double*>(P.finfo_slot + 6LL * start);
        for (int w = tid; w < cnt * META_SLOT_W; w += BS) cp_async8(M + w, sl + w);
        for (int w = tid; w < cnt * 6 * META_FACE_W; w += BS) cp_async8(M + CNT * META_SLOT_W + w, fl + w);
    };
    auto slot_of = [&](const double* M, int s) { return reinterpret_cast<const SlotInfo*>(M + s * META_SLOT_W); };
    auto face_of_m = [&](const double* M, int s, int f) {
        return reinterpret_cast<const FaceInfo*>(M + CNT * META_SLOT_W + (s * 6 + f) * META_FACE_W);
    };
    // state, RK register and outer traces of `item` into pipeline stage st
    auto issue_data = [&](int item, const double* M, int st) {
        double* Q = STG + st * STAGE;
        double* GB = Q + NV * T;
        double* X = GB + NV * T;
        const int cnt = item_cnt(item);
#pragma unroll
        for (int it = 0; it < NPTT; ++it) {
            const int t = tid + it * BS;
            if (t < cnt * n) {
                const int slot = t / n, node = t - slot * n;
                const long long off = slot_of(M, slot)->off;
                const double* qe = P.q + off + node;
#pragma unroll
                for (int v = 0; v < NV; ++v) cp_async8(&Q[(slot * NV + v) * n + node], qe + v * n);
                if (need_g) {
                    const double* ge = P.g + off + node;
#pragma unroll
                    for (int v = 0; v < NV; ++v) cp_async8(&GB[(slot * NV + v) * n + node], ge + v * n);
                }
            }
        }
        if (surf) {
            for (int t = tid; t < cnt * FS; t += BS) {
                const int slot = t / FS;
                const int r = t - slot * FS;
                int f, pt;
                face_of<S>(r, f, pt);
                const FaceInfo* fi = face_of_m(M, slot, f);
                const int nta = f < 2 ? n2 : n1;
                const int ta = pt % nta, tb = pt / nta;
                if (fi->kind == 0) {
                    const double* src = P.q + fi->off + fi->base + ta * fi->sa + tb * fi->sb;
#pragma unroll
                    for (int v = 0; v < NV; ++v) cp_async8(&X[(slot * NV + v) * FS + r], src + (long long)v * fi->n);
                } else if (fi->kind == 1) {
                    const double* src = P.mortarG + fi->off + pt;
#pragma unroll
                    for (int v = 0; v < NV; ++v) cp_async8(&X[(slot * NV + v) * FS + r], src + (long long)v * fi->n);
                }
            }
        }
    };

    const int first = blockIdx.x;
    if (first >= nitems) return;
    // prologue: meta of items 0 and 1 of this CTA, then data of item 0
    issue_meta(first, 0);
    if (first + G < nitems) issue_meta(first + G, 1);
    asm volatile("cp.async.commit_group;\n" ::);
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
    issue_data(first, META, 0);
    asm volatile("cp.async.commit_group;\n" ::);

    const double dt = P.mode ? *P.dt : 0.0;
    double lmax = 0.0;
    for (int k = 0;; ++k) {
        const int item = first + k * G;
        if (item >= nitems) break;
        // data of item k (issued one iteration ago) and meta of item k+1 have landed
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        __syncthreads();
        if (item + 2 * G < nitems) issue_meta(item + 2 * G, (k + 2) % 3);
        if (item + G < nitems) issue_data(item + G, META + ((k + 1) % 3) * MW, (k + 1) & 1);
        asm volatile("cp.async.commit_group;\n" ::);

        const double* M = META + (k % 3) * MW;
        double* Q = STG + (k & 1) * STAGE;
        double* GB = Q + NV * T;
        double* X = GB + NV * T;
        const int cnt = item_cnt(item);
        const int ntot = cnt * n;

        // ---- 1/rho and p once per node; admissibility (reading A25) ----------
#pragma unroll
        for (int it = 0; it < NPTT; ++it) {
            const int t = tid + it * BS;
            if (t < ntot) {
                const int slot = t / n, node = t - slot * n;
                const double q0 = Q[(slot * NV) * n + node];
                const double ir = 1.0 / q0;
                const double m1 = Q[(slot * NV + 1) * n + node], m2 = Q[(slot * NV + 2) * n + node],
                             m3 = Q[(slot * NV + 3) * n + node];
                const double p = gm1 * (Q[(slot * NV + 4) * n + node] - 0.5 * ir * (m1 * m1 + m2 * m2 + m3 * m3));
                IR[t] = ir;
                PR[t] = p;
                if (!(q0 > 0.0 && p > 0.0)) {
                    if (atomicAdd(P.flag, 1) == 0) P.flag[1] = slot_of(M, slot)->e;
                }
            }
        }

        // ---- volume term, direction by direction --------------------------------
        double acc[NPTT][NV];
#pragma unroll
        for (int it = 0; it < NPTT; ++it)
#pragma unroll
            for (int v = 0; v < NV; ++v) acc[it][v] = 0.0;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            __syncthreads();  // IR/PR ready (d = 0); previous derivatives consumed (d > 0)
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
                    const double sc = slot_of(M, slot)->sc[d];
#pragma unroll
                    for (int v = 0; v < NV; ++v) acc[it][v] = fma(sc, F[(slot * NV + v) * n + node], acc[it][v]);
                }
            }
        }

        // ---- surface: lifting terms +-(G - f_own) 2/(h_d w_end) into X -------------
        if (surf) {
            for (int t = tid; t < cnt * FS; t += BS) {
                const int slot = t / FS;
                const int r = t - slot * FS;
                int f, pt;
                face_of<S>(r, f, pt);
                const int d = f >> 1, s = f & 1;
                const int nta = d == 0 ? n2 : n1;
                const int ta = pt % nta, tb = pt / nta;
                int i, j, kk, Nd;
                if (d == 0) { i = s ? N1 : 0; j = ta; kk = tb; Nd = N1; }
                else if (d == 1) { i = ta; j = s ? N2 : 0; kk = tb; Nd = N2; }
                else { i = ta; j = tb; kk = s ? N3 : 0; Nd = N3; }
                const int node = i + n1 * (j + n2 * kk);
                double qo[NV], qx[NV], out[NV];
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    qo[v] = Q[(slot * NV + v) * n + node];
                    qx[v] = X[(slot * NV + v) * FS + r];
                }
                const double iro = IR[slot * n + node], po = PR[slot * n + node];
                const int kind = face_of_m(M, slot, f)->kind;
                if (d == 0) face_point<0>(qo, iro, po, qx, kind, s, P.ph, out);
                else if (d == 1) face_point<1>(qo, iro, po, qx, kind, s, P.ph, out);
                else face_point<2>(qo, iro, po, qx, kind, s, P.ph, out);
                const double sc = (s ? 1.0 : -1.0) * slot_of(M, slot)->sc[d] / c_w[Nd][0];
#pragma unroll
                for (int v = 0; v < NV; ++v) X[(slot * NV + v) * FS + r] = sc * out[v];
            }
            __syncthreads();
        }

        // ---- epilogue per node: Qdot, or the low-storage RK update (+ CFL rate) ----
#pragma unroll
        for (int it = 0; it < NPTT; ++it) {
            const int t = tid + it * BS;
            if (t >= ntot) continue;
            const int slot = t / n, node = t - slot * n;
            const SlotInfo* si = slot_of(M, slot);
            if (surf) {
                const int i = node % n1, j = (node / n1) % n2, kk = node / (n1 * n2);
                const double* Xb = X + slot * NV * FS;
                if (i == 0 || i == N1) {
                    const int r = (i == 0 ? 0 : S::nf0) + j + n2 * kk;
#pragma unroll
                    for (int v = 0; v < NV; ++v) acc[it][v] += Xb[v * FS + r];
                }
                if (j == 0 || j == N2) {
                    const int r = 2 * S::nf0 + (j == 0 ? 0 : S::nf1) + i + n1 * kk;
#pragma unroll
                    for (int v = 0; v < NV; ++v) acc[it][v] += Xb[v * FS + r];
                }
                if (kk == 0 || kk == N3) {
                    const int r = 2 * (S::nf0 + S::nf1) + (kk == 0 ? 0 : S::nf2) + i + n1 * j;
#pragma unroll
                    for (int v = 0; v < NV; ++v) acc[it][v] += Xb[v * FS + r];
                }
            }
            double* o = P.out + si->off + node;
            if (P.mode == 0) {
#pragma unroll
                for (int v = 0; v < NV; ++v) o[v * n] = -acc[it][v];
            } else {
                double* g = P.g + si->off + node;
                double qn[NV];
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    const double gn = (need_g ? P.rkA * GB[(slot * NV + v) * n + node] : 0.0) - dt * acc[it][v];
                    g[v * n] = gn;
                    qn[v] = Q[(slot * NV + v) * n + node] + P.rkB * gn;
                    o[v * n] = qn[v];
                }
                if (P.lam_max) {  // CFL rate of q^{n+1} (reading A11), fused
                    const double ir = 1.0 / qn[0];
                    const double p = gm1 * (qn[4] - 0.5 * ir * (qn[1] * qn[1] + qn[2] * qn[2] + qn[3] * qn[3]));
                    const double c = sqrt(P.gamma * p * ir);
                    constexpr double L1 = (double)n1 * n1, L2 = (double)n2 * n2, L3 = (double)n3 * n3;
                    const double lam = 0.5 * ((fabs(qn[1] * ir) + c) * L1 * si->sc[0] + (fabs(qn[2] * ir) + c) * L2 * si->sc[1] +
                                              (fabs(qn[3] * ir) + c) * L3 * si->sc[2]);
                    lmax = fmax(lmax, lam);
                }
            }
        }
    }
    if (P.lam_max) {
        lmax = block_max(lmax, red);
        if (threadIdx.x == 0) atomicMax(P.lam_max, (unsigned long long)__double_as_longlong(lmax));
    }
}

// host-side: launcher table filled by the instantiation units
typedef void (*res_launcher)(const ResParams& P, int start0, int nelem, int nitems, int grid, cudaStream_t st);
typedef int (*res_occupancy)();

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

// persistent launch: `grid` CTAs (resident capacity), each walking the bucket's items
template <int N1, int N2, int N3>
void launch_res_t(const ResParams& P, int start0, int nelem, int nitems, int grid, cudaStream_t st)
{
    using S = Shape<N1, N2, N3>;
    k_res_t<N1, N2, N3><<<grid < nitems ? grid : nitems, S::BS, S::smem_bytes, st>>>(P, start0, nelem, nitems);
}

template <int N1, int N2, int N3>
int occ_res_t()
{
    using S = Shape<N1, N2, N3>;
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_res_t<N1, N2, N3>, S::BS, S::smem_bytes);
    return nb;
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
