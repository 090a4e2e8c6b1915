// kernels.cuh -- sm_100a kernels of the host-light steps of the hot path
// (CFL step size, order selection and the jump fixpoint, solution transfer,
// diagnostics) and the mortar parameter block of face.cuh; included by
// dgtau.cu only.  Numerics: see common.cuh.
#pragma once

#include "common.cuh"

namespace dgtau {

// Parameters of the affine mortar kernel k_mortar3 (face.cuh, reading A6).
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

// tall: the element's largest estimate over its three directions (reading R11)
__device__ void directional_estimate(int Nd, const double* td, double tall, double* hat /* [NP+1] indexed by n */)
{
    const double SENT = 1e30;
    const double eps = 1e-13 * fmax(1.0, td[0]);
    double tmax = 0.0;
    for (int p = 1; p < Nd; ++p) tmax = fmax(tmax, td[p]);
    if (Nd <= 1) {  // not estimable: keep the order
        for (int m = 1; m <= NMAX; ++m) hat[m] = (m == Nd) ? 0.0 : SENT;
        return;
    }
    if (tmax <= eps || tmax <= 1e-8 * tall) {  // resolved direction (A14), or rounding next to the others (R11)
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
        else if (Nd == 2) hat[m] = m == Nd ? 0.0 : SENT;  // no extrapolation possible: keep the order (R12)
        else hat[m] = asym ? pow(10.0, a + b * m) : SENT;
    }
}

__global__ void k_select(SelParams P)
{
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= P.E) return;
    double hat[3][NP + 1];
    int Ne[3];
    double tall = 0.0;
    for (int d = 0; d < 3; ++d) {
        Ne[d] = P.orders[3 * e + d];
        for (int p = 1; p < Ne[d]; ++p) tall = fmax(tall, P.tau[(3 * (long long)e + d) * DG_TAU_STRIDE_DEV + p]);
    }
    for (int d = 0; d < 3; ++d) {
        directional_estimate(Ne[d], P.tau + (3 * (long long)e + d) * DG_TAU_STRIDE_DEV, tall, hat[d]);
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

// ---------------------------------------------------------------------------
// Face-trace halo copies (partition.TracePlan): entry i =
// (buffer offset, 8 e + f); the trace of field component c (ncomp per node,
// element block at (ncomp / 5) x off[e]) on face f of element e at face point
// pt = ta + n_a tb is buf[offset + c nf + pt].  dir 0: field -> buf (pack),
// 1: buf -> field (unpack into the halo element's face nodes).  One warp per
// entry.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128) k_trace_copy(const long long* ent, int n, const int* orders, const long long* off,
                                                    double* field, int ncomp, double* buf, int dir)
{
    const int i = blockIdx.x * 4 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (i >= n) return;
    const long long boff = ent[2 * i];
    const int e = (int)(ent[2 * i + 1] >> 3), f = (int)(ent[2 * i + 1] & 7);
    const int d = f >> 1, s = f & 1;
    const int N[3] = {orders[3 * e] + 1, orders[3 * e + 1] + 1, orders[3 * e + 2] + 1};
    const int st[3] = {1, N[0], N[0] * N[1]};
    const int ta = d == 0 ? 1 : 0, tb = d == 2 ? 1 : 2;
    const int na = N[ta], nf = na * N[tb], nn = st[2] * N[2];
    const int base = s ? (N[d] - 1) * st[d] : 0;
    double* blk = field + (long long)(ncomp / NV) * off[e];
    for (int idx = lane; idx < ncomp * nf; idx += 32) {
        const int c = idx / nf, pt = idx - c * nf;
        const int b = pt / na, a = pt - b * na;
        double* x = blk + (long long)c * nn + base + a * st[ta] + b * st[tb];
        if (dir == 0) buf[boff + idx] = *x;
        else *x = buf[boff + idx];
    }
}

}  // namespace dgtau
