// residual_t.cuh -- order-specialised fused DGSEM residual / RK-stage kernel.
//
// One template instance per (N1,N2,N3) bucket; a persistent CTA walks work
// items of CNT same-order elements.  Same numerics as the generic path
// (strong-form GL-DGSEM, see kernels.cuh header; PAPER.md P:129-155,
// P:472-473), arranged for the sm_100a fp64 pipes (v7):
//   * the element states of item k+1 are fetched by ONE thread with 1-D TMA
//     bulk copies (cp.async.bulk, mbarrier complete_tx) into the second
//     shared stage while item k is computed; neighbour traces (or projected
//     mortar fluxes) by cp.async into a double-buffered trace stage; the RK
//     register g is loaded into registers at item start and consumed in the
//     epilogue (latency hidden behind the whole item);
//   * node phase: 1/rho, p and the three axis fluxes f_x, f_y, f_z of every
//     node go to shared memory at once (one barrier);
//   * task phase (one barrier): Roe face tasks (one thread per face point,
//     G - f_own times the lifting scale, in place in the trace buffer) run
//     beside the 5 x (lines) x 3 line-derivative tasks (even-odd split of D,
//     line in registers, in place);
//   * epilogue per node: Qdot = -(sum_d (2/h_d) D^d f_d + lifting), or the
//     Williamson low-storage update g <- A g + dt Qdot, q' <- q + B g, plus
//     the fused CFL rate of q' in the last stage.
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

// Elements per work item of the (n1, n2, n3)-node bucket: <= ~384 nodes per
// CTA (node tasks in one round of threads), capped so that the CTA's shared
// memory (2 state + 2 flux stages, 3 flux directions, meta) stays <= 76 KB
// and 3 CTAs fit an SM (small orders: the face-flux stage dominates).
// Shared by the host plans (dg_set_orders) and Shape<>.
__host__ __device__ constexpr int res_cnt(int n1, int n2, int n3)
{
    const int n = n1 * n2 * n3;
    const int sq = (NV * n + 2) / 2 * 2;
    const int gsl = 2 * ((NV * n2 * n3 + 1) / 2 * 2 + (NV * n1 * n3 + 1) / 2 * 2 + (NV * n1 * n2 + 1) / 2 * 2);
    const int per = 8 * (2 * sq + 2 * gsl + 3 * NV * n + 33);
    const int budget = (76 * 1024) / per;
    return cmax(1, cmin(cmin(MAXSLOTS, 384 / n), budget));
}

template <int N1, int N2, int N3>
struct Shape {
    static constexpr int n1 = N1 + 1, n2 = N2 + 1, n3 = N3 + 1;
    static constexpr int n = n1 * n2 * n3;
    static constexpr int CNT = res_cnt(n1, n2, n3);
    static constexpr int T = CNT * n;
    static constexpr int NPT = T > 384 ? 2 : 1;
    static constexpr int LT = NV * (n / n1 + n / n2 + n / n3);  // line tasks per element
    // threads: enough for one round of nodes; raised (up to 384) when that
    // saves a round of line tasks (N=6: 343 nodes, 735 line tasks -> 384)
    static constexpr int BS0 = ((T + NPT - 1) / NPT + 31) / 32 * 32;
    static constexpr int LR = (CNT * LT + BS0 - 1) / BS0;  // line rounds at BS0
    static constexpr int BS1 = LR > 1 ? ((CNT * LT + LR - 2) / (LR - 1) + 31) / 32 * 32 : BS0;
    static constexpr int BS = BS1 <= 384 && BS1 > BS0 ? BS1 : BS0;
    static constexpr int nf0 = n2 * n3, nf1 = n1 * n3, nf2 = n1 * n2;
    static constexpr int FS = 2 * (nf0 + nf1 + nf2);
    // state slot: 5n doubles + 1 (8-byte shift of odd-offset elements), even
    static constexpr int SQ = (NV * n + 2) / 2 * 2;
    static constexpr int QS = CNT * SQ;          // one state stage
    // face flux blocks of one element: [face][v][pt], each block padded to even
    __host__ __device__ static constexpr int gblk(int d) { return (NV * (d == 0 ? nf0 : d == 1 ? nf1 : nf2) + 1) / 2 * 2; }
    __host__ __device__ static constexpr int gbase(int f) {
        return (f >= 1 ? gblk(0) : 0) + (f >= 2 ? gblk(0) : 0) + (f >= 3 ? gblk(1) : 0) + (f >= 4 ? gblk(1) : 0) +
               (f >= 5 ? gblk(2) : 0);
    }
    static constexpr int GSL = 2 * (gblk(0) + gblk(1) + gblk(2));
    static constexpr int GS = CNT * GSL;         // one flux stage
    static constexpr int MW = CNT * (5 + 6);     // meta words per item (slot info + 6 face flux offsets)
    // 2 state stages + 2 flux stages + F (3 directions) + 3 meta buffers
    static constexpr size_t smem_bytes = sizeof(double) * (size_t)(2 * QS + 2 * GS + 3 * NV * T + 3 * MW);
    static constexpr int MINB_T = BS <= 128 ? 4 : (BS <= 192 ? 3 : (BS <= 384 ? 2 : 1));
    static constexpr int MINB_S = (int)((227 * 1024) / (smem_bytes + 1024 + 512));
    static constexpr int MINB = cmax(1, cmin(MINB_T, MINB_S));
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

// In-place derivative of one line held in shared memory, F[m*stride] <-
// sum_m D_am F_m, by the even-odd decomposition of the GL differentiation
// matrix (about half the multiply-adds of the direct product):
//   o_m = v_m - v_{N-m}, e_m = v_m + v_{N-m}  (m < H),
//   out_a = sum_m P_am o_m + (sum_m Q_am e_m + Qm_a v_mid),
//   out_{N-a} = sum_m P_am o_m - (sum_m Q_am e_m + Qm_a v_mid),
//   out_mid = sum_m M_m o_m.
template <int L>
__device__ __forceinline__ void dline_inplace(double* Fl, int stride);

// As dline_inplace, plus the strong-form lifting of the two end points of the
// line (GL end weight w_0 = 2/(N(N+1))): the face fluxes
// gm (at xi = -1) and gp (at xi = +1) enter as
//   out_0 -= (N(N+1)/2) (gm - f_0),   out_N += (N(N+1)/2) (gp - f_N),
// with f_0, f_N the line's own end values (the element's trace flux).
template <int L>
__device__ __forceinline__ void dline_lift(double* Fl, int stride, double gm, double gp)
{
    constexpr int N = L - 1, H = L / 2;
    constexpr bool odd = (L & 1) != 0;
    constexpr double CL = 0.5 * N * (N + 1);
    double v[L];
#pragma unroll
    for (int m = 0; m < L; ++m) v[m] = Fl[m * stride];
    const double l0 = -CL * (gm - v[0]), lN = CL * (gp - v[N]);
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
        Fl[a * stride] = a == 0 ? (p + q) + l0 : p + q;
        Fl[(N - a) * stride] = a == 0 ? (p - q) + lN : p - q;
    }
    if (odd) {
        double s = c_EOM[N][0] * o[0];
#pragma unroll
        for (int m = 1; m < H; ++m) s = fma(c_EOM[N][m], o[m], s);
        Fl[H * stride] = s;
    }
}

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

__device__ __forceinline__ void cp_async8s(unsigned d, const double* src)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src));
}

__device__ __forceinline__ void cp_async8(double* dst, const double* src)
{
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src));
}

// Per-item metadata staged in shared memory: slot info (5 doubles) and the 6
// face descriptors (4 doubles each) of every element of the item.
constexpr int META_SLOT_W = 5, META_FACE_W = 4;

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long* b, int count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity)
{
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void bulk_prefetch_l2(const void* src, unsigned bytes)
{
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
}

// 1-D TMA bulk copy global -> shared with an L2 cache policy
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, unsigned bytes, unsigned long long* b,
                                              unsigned long long pol)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(b)), "l"(pol)
        : "memory");
}

// 1-D TMA bulk copy global -> shared, completion counted on mbarrier b
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* b)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(b))
                 : "memory");
}

template <int N1, int N2, int N3>
__global__ void __launch_bounds__(Shape<N1, N2, N3>::BS, Shape<N1, N2, N3>::MINB)
    k_res_t(ResParams P, int start0, int nelem, int nitems)
{
    using S = Shape<N1, N2, N3>;
    constexpr int n = S::n, n1 = S::n1, n2 = S::n2, n3 = S::n3, BS = S::BS, NPTT = S::NPT;
    constexpr int T = S::T, CNT = S::CNT, SQ = S::SQ, QS = S::QS, GSL = S::GSL, GS = S::GS, MW = S::MW;
    constexpr int L0 = n / n1, L1 = n / n2, L2 = n / n3;  // lines per direction
    extern __shared__ __align__(16) double sm[];
    double* QST = sm;                 // 2 state stages [slot][SQ]: element data at +shift (0/1)
    double* GST = QST + 2 * QS;       // 2 flux stages [slot][face][v][pt] (face blocks 16-byte aligned)
    double* F = GST + 2 * GS;         // [slot][d][v][node]: f_d, then (in place) D^d f_d
    double* META = F + 3 * NV * T;    // 3 meta buffers of MW words
    __shared__ double red[32];
    __shared__ __align__(8) unsigned long long mbar[2];

    const int tid = threadIdx.x;
    const bool surf = P.variant == 0;
    const bool need_g = P.mode == 1 && P.rkA != 0.0;
    const double gm1 = P.ph.gm1;
    const int G = gridDim.x;
    const unsigned long long pol_first = l2_policy_first(), pol_last = l2_policy_last();

    auto item_cnt = [&](int item) { return min(CNT, nelem - item * CNT); };
    auto slot_of = [&](const double* M, int s) { return reinterpret_cast<const SlotInfo*>(M + s * META_SLOT_W); };
    auto fofs_of = [&](const double* M, int s, int f) {
        return reinterpret_cast<const long long*>(M + CNT * META_SLOT_W)[s * 6 + f];
    };
    // meta (slot info + face flux offsets) of `item` into meta buffer mb
    auto issue_meta = [&](int item, int mb) {
        double* M = META + mb * MW;
        const int cnt = item_cnt(item);
        const int start = start0 + item * CNT;
        const double* sl = reinterpret_cast<const double*>(P.slots + start);
        const double* fl = reinterpret_cast<const double*>(P.fofs_slot + 6LL * start);
        for (int w = tid; w < cnt * META_SLOT_W; w += BS) cp_async8(M + w, sl + w);
        for (int w = tid; w < cnt * 6; w += BS) cp_async8(M + CNT * META_SLOT_W + w, fl + w);
    };
    // element states and face flux blocks of `item` into stage st, by ONE
    // thread with 1-D bulk copies.  State: the 16-byte aligned envelope
    // [floor16(src), ceil16(src + 40n)) (data at shift off & 1), clipped at the
    // buffer end (last 8 bytes by hand).  Flux blocks are 16-byte aligned and
    // padded by construction.  The RK register g is prefetched into L2.
    auto issue_stage = [&](int item, const double* M, int st) {
        if (tid != 0) return;
        const int cnt = item_cnt(item);
        double* Q = QST + st * QS;
        double* Gs = GST + st * GS;
        unsigned total = 0;
        for (int s = 0; s < cnt; ++s) {
            const long long off = slot_of(M, s)->off;
            long long b = (off + NV * n + 1) & ~1LL;
            if (b > P.qlen) b -= 2;
            total += (unsigned)((b - (off & ~1LL)) * 8);
        }
        if (surf) total += (unsigned)(cnt * GSL * 8);
        mbar_expect_tx(&mbar[st], total);
        for (int s = 0; s < cnt; ++s) {
            const long long off = slot_of(M, s)->off;
            const long long a = off & ~1LL;
            long long b = (off + NV * n + 1) & ~1LL;
            const bool clip = b > P.qlen;
            if (clip) b -= 2;
            bulk_g2s_hint(Q + s * SQ, P.q + a, (unsigned)((b - a) * 8), &mbar[st], pol_first);
            if (clip) Q[s * SQ + (b - a)] = P.q[b];
            if (need_g) bulk_prefetch_l2(P.g + a, (unsigned)((b - a) * 8));
            if (surf) {
#pragma unroll
                for (int f = 0; f < 6; ++f)
                    bulk_g2s_hint(Gs + s * GSL + S::gbase(f), P.mortarG + fofs_of(M, s, f),
                                  (unsigned)(S::gblk(f >> 1) * 8), &mbar[st], pol_first);
            }
        }
    };

    const int first = blockIdx.x;
    if (first >= nitems) return;
    if (tid == 0) {
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    double dt = 0.0;
    if (P.mode) dt = P.lam_in ? P.cfl / __longlong_as_double((long long)*P.lam_in) : *P.dt;
    if (blockIdx.x == 0 && tid == 0) {
        if (P.dt_out) *P.dt_out = dt;
        if (P.lam_zero) *P.lam_zero = 0ull;
    }
    double lmax = 0.0;

    // node phase of local item k (state stage k&1, meta k%3): 1/rho, p,
    // admissibility (A25), f_d -> F.  Thread t owns nodes t + it*BS; their
    // states stay in registers (qreg) for the item's epilogue.
    double qreg[NPTT][NV];
    auto node_phase = [&](int k) {
        const double* M = META + (k % 3) * MW;
        const double* Q = QST + (k & 1) * QS;
        const int ntot = item_cnt(first + k * G) * n;
#pragma unroll
        for (int it = 0; it < NPTT; ++it) {
            const int t = tid + it * BS;
            if (t < ntot) {
                const int slot = t / n, node = t - slot * n;
                const SlotInfo* si = slot_of(M, slot);
                const double* qe = Q + slot * SQ + (si->off & 1) + node;
                double* qv = qreg[it];
#pragma unroll
                for (int v = 0; v < NV; ++v) qv[v] = qe[v * n];
                const double ir = rcp_nr(qv[0]);
                const double p = gm1 * (qv[4] - 0.5 * ir * (qv[1] * qv[1] + qv[2] * qv[2] + qv[3] * qv[3]));
                if (!(qv[0] > 0.0 && p > 0.0)) {
                    if (atomicAdd(P.flag, 1) == 0) P.flag[1] = si->e;
                }
                double* Fs = F + slot * 3 * NV * n + node;
                double f[NV];
                flux_axis<0>(qv, ir, p, f);
#pragma unroll
                for (int v = 0; v < NV; ++v) Fs[v * n] = f[v];
                flux_axis<1>(qv, ir, p, f);
#pragma unroll
                for (int v = 0; v < NV; ++v) Fs[(NV + v) * n] = f[v];
                flux_axis<2>(qv, ir, p, f);
#pragma unroll
                for (int v = 0; v < NV; ++v) Fs[(2 * NV + v) * n] = f[v];
            }
        }
    };
    // line phase of local item k: D^d along every line of every direction, in
    // place, with the lifting of the line's two face points (face point index
    // = line index)
    auto line_phase = [&](int k) {
        const int cnt = item_cnt(first + k * G);
        const double* Gs = GST + (k & 1) * GS;
        for (int u = tid; u < cnt * S::LT; u += BS) {
            const int slot = u / S::LT;
            int w = u - slot * S::LT;
            double* Fs = F + slot * 3 * NV * n;
            const double* Gsl = Gs + slot * GSL;
            if (w < NV * L0) {
                const int v = w / L0, l = w - v * L0;
                double* Fl = Fs + w * n1;  // lines of all 5 variables are back to back
                if (surf) dline_lift<n1>(Fl, 1, Gsl[S::gbase(0) + v * S::nf0 + l], Gsl[S::gbase(1) + v * S::nf0 + l]);
                else dline_inplace<n1>(Fl, 1);
            } else if (w < NV * (L0 + L1)) {
                w -= NV * L0;
                // for n1 >= 6 order (i, variable, k): consecutive threads then hit
                // distinct shared-memory banks (the (i, k) order collides on
                // i + k mod 16; bank simulation)
                int v, l;
                if (n1 >= 6) {
                    const int kk = w / (NV * n1), r = w - kk * NV * n1;
                    v = r / n1;
                    l = (r - v * n1) + n1 * kk;
                } else {
                    v = w / L1;
                    l = w - v * L1;
                }
                const int kk = l / n1, i = l - kk * n1;
                double* Fl = Fs + (NV + v) * n + i + n1 * n2 * kk;
                if (surf) dline_lift<n2>(Fl, n1, Gsl[S::gbase(2) + v * S::nf1 + l], Gsl[S::gbase(3) + v * S::nf1 + l]);
                else dline_inplace<n2>(Fl, n1);
            } else {
                w -= NV * (L0 + L1);
                const int v = w / L2, l = w - v * L2;
                double* Fl = Fs + (2 * NV + v) * n + l;
                if (surf) dline_lift<n3>(Fl, n1 * n2, Gsl[S::gbase(4) + v * S::nf2 + l], Gsl[S::gbase(5) + v * S::nf2 + l]);
                else dline_inplace<n3>(Fl, n1 * n2);
            }
        }
    };
    // RK register g of local item k (L2-prefetched with its stage) into registers
    double gr[NPTT][NV];
    auto load_g = [&](int k) {
        if (!need_g) return;
        const double* M = META + (k % 3) * MW;
        const int ntot = item_cnt(first + k * G) * n;
#pragma unroll
        for (int it = 0; it < NPTT; ++it) {
            const int t = tid + it * BS;
            if (t < ntot) {
                const int slot = t / n, node = t - slot * n;
                const double* ge = P.g + slot_of(M, slot)->off + node;
#pragma unroll
                for (int v = 0; v < NV; ++v) gr[it][v] = __ldcs(ge + v * n);
            }
        }
    };
    // epilogue of local item k for node slot it of this thread: Qdot, or the
    // low-storage RK update (+ fused CFL rate of the new state)
    auto epilogue = [&](int k, int it) {
        const double* M = META + (k % 3) * MW;
        const int ntot = item_cnt(first + k * G) * n;
        const int t = tid + it * BS;
        if (t >= ntot) return;
        const int slot = t / n, node = t - slot * n;
        const SlotInfo* si = slot_of(M, slot);
        const long long eoff = si->off;
        const double* Fs = F + slot * 3 * NV * n + node;
        double acc[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v)
            acc[v] = fma(si->sc[0], Fs[v * n], fma(si->sc[1], Fs[(NV + v) * n], si->sc[2] * Fs[(2 * NV + v) * n]));
        double* o = P.out + eoff + node;
        if (P.mode == 0) {
#pragma unroll
            for (int v = 0; v < NV; ++v) __stcs(o + v * n, -acc[v]);
        } else {
            double* g = P.g + eoff + node;
            double qn[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                const double gn = need_g ? fma(P.rkA, gr[it][v], -dt * acc[v]) : -dt * acc[v];
                __stcs(g + v * n, gn);
                qn[v] = fma(P.rkB, gn, qreg[it][v]);
                st_hint(o + v * n, qn[v], pol_last);
            }
            if (P.lam_max) {  // CFL rate of q^{n+1} (reading A11), fused
                const double ir = rcp_nr(qn[0]);
                const double p = gm1 * (qn[4] - 0.5 * ir * (qn[1] * qn[1] + qn[2] * qn[2] + qn[3] * qn[3]));
                const double c = sqrt(P.gamma * p * ir);
                constexpr double C1 = (double)n1 * n1, C2 = (double)n2 * n2, C3 = (double)n3 * n3;
                const double lam = 0.5 * ((fabs(qn[1] * ir) + c) * C1 * si->sc[0] + (fabs(qn[2] * ir) + c) * C2 * si->sc[1] +
                                          (fabs(qn[3] * ir) + c) * C3 * si->sc[2]);
                lmax = fmax(lmax, lam);
            }
        }
    };

    // Software pipeline over the CTA's items (local index k, item first + kG):
    //   [epilogue(k) + node(k+1)] | barrier | lines(k+1) | barrier
    // epilogue(k) and node(k+1) of the same thread touch the same F entries
    // (read, then overwrite), so one F buffer serves both.  State/flux stage
    // j&1 and meta buffer j%3 hold item j; the stage of item k+2 is issued as
    // soon as item k is consumed.
    issue_meta(first, 0);
    if (first + G < nitems) issue_meta(first + G, 1);
    asm volatile("cp.async.commit_group;\n" ::);
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
    issue_stage(first, META, 0);
    if (first + G < nitems) issue_stage(first + G, META + MW, 1);
    if (first + 2 * G < nitems) issue_meta(first + 2 * G, 2);
    asm volatile("cp.async.commit_group;\n" ::);
    mbar_wait(&mbar[0], 0);
    __syncthreads();  // thread 0's hand copy of a clipped state's last double (issue_stage) is visible
    node_phase(0);
    __syncthreads();
    load_g(0);
    line_phase(0);
    __syncthreads();
    for (int k = 0;; ++k) {
        const int item = first + k * G;
        const bool has_next = item + G < nitems;
        if (has_next) mbar_wait(&mbar[(k + 1) & 1], ((k + 1) >> 1) & 1);
#pragma unroll
        for (int it = 0; it < NPTT; ++it) epilogue(k, it);
        if (has_next) node_phase(k + 1);
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");  // meta of item k+2
        __syncthreads();
        // item k consumed: its stage k&1 takes item k+2, meta buffer k%3 item k+3
        if (item + 2 * G < nitems) issue_stage(item + 2 * G, META + ((k + 2) % 3) * MW, k & 1);
        if (item + 3 * G < nitems) issue_meta(item + 3 * G, k % 3);
        asm volatile("cp.async.commit_group;\n" ::);
        if (!has_next) break;
        load_g(k + 1);
        line_phase(k + 1);
        __syncthreads();
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
