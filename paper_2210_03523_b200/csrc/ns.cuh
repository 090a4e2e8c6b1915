// ns.cuh -- sm_100a kernels of the curved-mesh residual (Euler and
// compressible Navier-Stokes with BR1), round-2 layout:
//
//   k_ns_face<W, MODE>  one warp-group (W warps) per face -- conforming,
//                       mortar, wall or far field: the traces of both sides are
//                       gathered, interpolated to the mortar grid (identity
//                       passes skipped), the point quantity is formed ONCE per
//                       mortar point with the face metric, and projected back
//                       to each side's own face nodes (exact L2 projection,
//                       reading A6).  MODE_QHAT: BR1 face state qhat times the
//                       face metric (eq DGSEMsystem:2); MODE_FLUX_*: |Ja_f|
//                       Roe(q_L, q_R; n) minus the BR1 average of the viscous
//                       fluxes along Ja_f; wall / far-field states of
//                       reading A10.  No CTA-wide barrier: warp / named
//                       barriers of the group only.
//   k_ns_grad<EXT>      element kernel, items of same-order elements: the BR1
//                       gradient J g_k = sum_d D^d (Ja^d_k q) + lifting of
//                       (H - q Ja^d_k)/w at the line ends, line tasks (one
//                       line in registers, even-odd D) along every direction.
//   k_ns_res<EXT, NS>   element kernel: contravariant fluxes Ja^d.(f^a - f^nu)
//                       of the three directions per node (viscous stress once
//                       per node), in-place derivative + lifting of (G - Ft)/w
//                       along every line, then Qdot = -(sum_d)/J, or the
//                       Williamson RK update with the CFL / DFL rates.
//
// PAPER.md: P:106-126 (eqs SystemAdvDiff, first-order system g = grad q),
// P:129-145 (eqs DGSEMsystem:1-2), P:144 (metric terms), P:472 (Roe, BR1),
// P:473-475 (RK3, CFL).  Readings A6, A8-A11.
//
// EXT (extruded meshes: geometry linear in zeta, x and y independent of zeta,
// z independent of xi and eta -- the O-grids of cfg4 / cfg5) keeps the metric
// terms as 6 doubles per (i, j) column: Ja^1 = (a, b, 0), Ja^2 = (c, e, 0),
// Ja^3 = (0, 0, f), J.  These are the metric identities of such a mesh
// (x_zeta = (0, 0, z_zeta)); the zero components are exact zeros and the
// kernels skip them (80 B of metric per node -> 48 B per column).
#pragma once

#include "common.cuh"
#include "curved.cuh"
#include "face.cuh"
#include "residual_t.cuh"

namespace dgtau {

// ---------------------------------------------------------------------------
// plans (built by dg_set_orders)
// ---------------------------------------------------------------------------

// element work item: `count` elements of the same orders (elist[start ..])
struct NsItem {
    int start, count, ord, nodes;
};
constexpr int NS_BS = 256;        // threads of the element kernels
constexpr int NS_ITEM_NODES = 256;  // nodes per element item (one round of threads)
constexpr int NS_MAXSLOTS = 32;   // elements per item (n >= 8)

// One face of the face kernels.  L = the element on the -xi_d side (face +d
// of L), R = the element on the +xi_d side (face -d of R).  Boundary faces:
// the missing side has off = -1 and carries the own side's orders.  Output
// blocks [comp][pt] (pt = ta + s_a tb, ta fastest): numerical flux G at
// outL / outR, BR1 terms H at hL / hR (conforming and boundary faces: one
// shared block).  Face metric at the mortar points (L's geometry
// at +1, or the own face of a boundary element; reading A6):
// fg[mg + c m + p], c = 0..2, p = i + m_a j.
struct NsFace {
    long long offL, offR, outL, outR, hL, hR, mg;
    int eL, eR, ordL, ordR;
    int d, kind;  // kind: 0 conforming, 1 mortar, 2 wall, 3 far field
};

enum { MODE_QHAT = 0, MODE_FLUX_EULER = 1, MODE_FLUX_NS = 2 };

// nonzero face-metric / Ja^d components of an extruded mesh
__host__ __device__ __forceinline__ int ext_nk(int d) { return d == 2 ? 1 : 2; }
__host__ __device__ __forceinline__ int ext_k(int d, int kk) { return d == 2 ? 2 : kk; }

struct NsFaceParams {
    const NsFace* faces;
    int fbase, fend;        // faces [fbase, fend) of this launch (one W class)
    const double* q;
    const double* grad;     // 15 per node at 3 x offset (MODE_FLUX_NS)
    const double* fg;       // face metrics
    double* out;            // G (5 per point) or H (5 nk per point) blocks
    const Tables* tab;
    PhysDev ph;
    int ext;
};

struct NsElemParams {
    const NsItem* items;
    int ibase;              // CTA b handles item ibase + b
    const int* elist;
    const int* orders;
    const long long* off;
    const double* met;      // !EXT: 10 per node at 2 x offset
    const double* metc;     // EXT: 6 per column at coff[e]
    const long long* coff;
    const double* q;
    const double* grad;     // k_ns_res: gradient (15 per node at 3 x offset)
    double* gout;           // k_ns_grad: gradient output
    const double* blk;      // face blocks: H (k_ns_grad) or G (k_ns_res)
    const long long* fofs;  // [E][6] block offsets; nullptr: isolated (no lifting)
    double* out;            // mode 0: Qdot; mode 1: q' = q + B g
    double* g;
    const double* dt;
    double rkA, rkB;
    int mode;
    unsigned long long* lam_max;  // CFL / DFL rates of q' (2 slots), last RK stage
    PhysDev ph;
};

// ---------------------------------------------------------------------------
// geometry (once per layout, double-double as k_metrics)
// ---------------------------------------------------------------------------

// Face metric Ja^d at the mortar points of every face (reading A6: L's
// geometry at xi_d = +1 for interior faces; the own face for boundary ones).
struct FaceGeomParams {
    const NsFace* faces;
    int nfaces;
    CurvedMesh cm;
    const TablesDD* tdd;
    double* fg;
    int ext;
};

__global__ void __launch_bounds__(128) k_face_geom(FaceGeomParams P)
{
    __shared__ double Xs[4][2][3][NP * NP];  // [warp][hi/lo][c][point]
    const int wi = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int fid = blockIdx.x * 4 + wi;
    if (fid >= P.nfaces) return;
    double (*Xm)[NP * NP] = Xs[wi][0];
    double (*Xl)[NP * NP] = Xs[wi][1];
    const NsFace F = P.faces[fid];
    const int d = F.d;
    const int ta = d == 0 ? 1 : 0, tb = d == 2 ? 1 : 2;
    int NL[3], NR[3];
    mt_unpack(F.ordL, NL);
    mt_unpack(F.ordR, NR);
    const int M1 = max(NL[ta], NR[ta]), M2 = max(NL[tb], NR[tb]);
    const int nm = (M1 + 1) * (M2 + 1);
    const bool useL = F.offL >= 0;
    const int eg = useL ? F.eL : F.eR;
    const int layer = useL ? 1 : 0;
    const int gd[3] = {P.cm.g1, P.cm.g2, P.cm.g3};
    const double* G = P.cm.geo + (long long)eg * 3 * P.cm.ng;
    const int ga = gd[0] + 1, gb = gd[1] + 1;
    const TablesDD* tdd = P.tdd;
    for (int t = lane; t < nm; t += 32) {
        const int m1 = t % (M1 + 1), m2 = t / (M1 + 1);
        dd x[3] = {mkdd(0.0), mkdd(0.0), mkdd(0.0)};
        for (int b = 0; b <= gd[tb]; ++b)
            for (int a = 0; a <= gd[ta]; ++a) {
                int idx[3];
                idx[d] = layer ? gd[d] : 0;
                idx[ta] = a;
                idx[tb] = b;
                const int gi = idx[0] + ga * (idx[1] + gb * idx[2]);
                const int ia = m1 * (gd[ta] + 1) + a, ib = m2 * (gd[tb] + 1) + b;
                const dd wgt = dd_mul(dd{tdd->Thi[gd[ta]][M1][ia], tdd->Tlo[gd[ta]][M1][ia]},
                                      dd{tdd->Thi[gd[tb]][M2][ib], tdd->Tlo[gd[tb]][M2][ib]});
                for (int c = 0; c < 3; ++c) x[c] = dd_add(x[c], dd_mul(wgt, mkdd(G[c * P.cm.ng + gi])));
            }
        for (int c = 0; c < 3; ++c) {
            Xm[c][t] = x[c].hi;
            Xl[c][t] = x[c].lo;
        }
    }
    __syncwarp();
    double* out = P.fg + F.mg;
    for (int t = lane; t < nm; t += 32) {
        const int m1 = t % (M1 + 1), m2 = t / (M1 + 1);
        dd u[3], v[3];
        for (int c = 0; c < 3; ++c) {
            dd s1 = mkdd(0.0), s2 = mkdd(0.0);
            for (int m = 0; m <= M1; ++m) {
                const int ix = m + (M1 + 1) * m2;
                s1 = dd_add(s1, dd_mul(dd{tdd->Dhi[M1][m1 * (M1 + 1) + m], tdd->Dlo[M1][m1 * (M1 + 1) + m]},
                                       dd{Xm[c][ix], Xl[c][ix]}));
            }
            for (int m = 0; m <= M2; ++m) {
                const int ix = m1 + (M1 + 1) * m;
                s2 = dd_add(s2, dd_mul(dd{tdd->Dhi[M2][m2 * (M2 + 1) + m], tdd->Dlo[M2][m2 * (M2 + 1) + m]},
                                       dd{Xm[c][ix], Xl[c][ix]}));
            }
            u[c] = s1;
            v[c] = s2;
        }
        const dd* A = d == 1 ? v : u;  // Ja^2 = x_zeta x x_xi = x_tb x x_ta
        const dd* B = d == 1 ? u : v;
        dd w[3];
        w[0] = dd_add(dd_mul(A[1], B[2]), dd_neg(dd_mul(A[2], B[1])));
        w[1] = dd_add(dd_mul(A[2], B[0]), dd_neg(dd_mul(A[0], B[2])));
        w[2] = dd_add(dd_mul(A[0], B[1]), dd_neg(dd_mul(A[1], B[0])));
        for (int c = 0; c < 3; ++c) {
            double val = w[c].hi + w[c].lo;
            if (P.ext && (d == 2 ? c < 2 : c == 2)) val = 0.0;  // structural zeros of an extruded mesh
            out[c * nm + t] = val;
        }
    }
}

// Compact metrics of an extruded element at its (i, j) columns, double-double:
// x, y from the geometry polynomial of the zeta = -1 layer, zz = z_zeta
// = (z1 - z0)/2, then Ja^1 = zz (y_eta, -x_eta, 0), Ja^2 = zz (-y_xi, x_xi, 0),
// Ja^3 = (0, 0, x_xi y_eta - x_eta y_xi), J = zz (x_xi y_eta - x_eta y_xi)
// (the cross-product form of curved.cuh with x_zeta = (0, 0, zz)).
struct MetExtParams {
    CurvedMesh cm;
    const int* orders;
    const long long* coff;
    double* metc;
    const TablesDD* tdd;
    int E;
};

__global__ void __launch_bounds__(128) k_metrics_ext(MetExtParams P)
{
    __shared__ double Xs[2][2][NP * NP];  // [hi/lo][x/y][column]
    const int e = blockIdx.x;
    if (e >= P.E) return;
    const int n1 = P.orders[3 * e] + 1, n2 = P.orders[3 * e + 1] + 1;
    const int nc = n1 * n2;
    const int g1 = P.cm.g1, g2 = P.cm.g2;
    const int ga = g1 + 1, gb = g2 + 1;
    const double* G = P.cm.geo + (long long)e * 3 * P.cm.ng;
    const TablesDD* tdd = P.tdd;
    for (int t = threadIdx.x; t < nc; t += blockDim.x) {
        const int i = t % n1, j = t / n1;
        dd x[2] = {mkdd(0.0), mkdd(0.0)};
        for (int b = 0; b <= g2; ++b)
            for (int a = 0; a <= g1; ++a) {
                const int i1 = i * ga + a, i2 = j * gb + b;
                const dd wgt = dd_mul(dd{tdd->Thi[g1][n1 - 1][i1], tdd->Tlo[g1][n1 - 1][i1]},
                                      dd{tdd->Thi[g2][n2 - 1][i2], tdd->Tlo[g2][n2 - 1][i2]});
                const int gi = a + ga * b;  // layer zeta = -1
                for (int c = 0; c < 2; ++c) x[c] = dd_add(x[c], dd_mul(wgt, mkdd(G[c * P.cm.ng + gi])));
            }
        for (int c = 0; c < 2; ++c) {
            Xs[0][c][t] = x[c].hi;
            Xs[1][c][t] = x[c].lo;
        }
    }
    __syncthreads();
    const dd zz = dd_mul(mkdd(0.5), two_sum(G[2 * P.cm.ng + ga * gb], -G[2 * P.cm.ng]));
    double* out = P.metc + P.coff[e];
    for (int t = threadIdx.x; t < nc; t += blockDim.x) {
        const int i = t % n1, j = t / n1;
        dd dxi[2], deta[2];
        for (int c = 0; c < 2; ++c) {
            dd s1 = mkdd(0.0), s2 = mkdd(0.0);
            for (int m = 0; m < n1; ++m) {
                const int ix = m + n1 * j;
                s1 = dd_add(s1, dd_mul(dd{tdd->Dhi[n1 - 1][i * n1 + m], tdd->Dlo[n1 - 1][i * n1 + m]},
                                       dd{Xs[0][c][ix], Xs[1][c][ix]}));
            }
            for (int m = 0; m < n2; ++m) {
                const int ix = i + n1 * m;
                s2 = dd_add(s2, dd_mul(dd{tdd->Dhi[n2 - 1][j * n2 + m], tdd->Dlo[n2 - 1][j * n2 + m]},
                                       dd{Xs[0][c][ix], Xs[1][c][ix]}));
            }
            dxi[c] = s1;
            deta[c] = s2;
        }
        const dd j3 = dd_add(dd_mul(dxi[0], deta[1]), dd_neg(dd_mul(deta[0], dxi[1])));
        const dd v[6] = {dd_mul(zz, deta[1]), dd_neg(dd_mul(zz, deta[0])), dd_neg(dd_mul(zz, dxi[1])),
                         dd_mul(zz, dxi[0]), j3, dd_mul(zz, j3)};
        for (int c = 0; c < 6; ++c) out[c * nc + t] = v[c].hi + v[c].lo;
    }
}

// ---------------------------------------------------------------------------
// metric access in the element kernels
// ---------------------------------------------------------------------------
template <bool EXT>
struct Met {
    const double* p;  // EXT: the element's 6 x nc block; else its 10 x n block
    int n, nc, n12;
    __device__ __forceinline__ void init(const NsElemParams& P, int e, long long o, int n_, int n1, int n2)
    {
        n = n_;
        n12 = n1 * n2;
        if (EXT) p = P.metc + P.coff[e];
        else p = P.met + 2 * o;
    }
    // (Ja^d)_k at node t
    __device__ __forceinline__ double ja(int d, int k, int t) const
    {
        if (EXT) {
            const int c = t % n12;
            if (d < 2) return k == 2 ? 0.0 : __ldg(p + (2 * d + k) * n12 + c);
            return k == 2 ? __ldg(p + 4 * n12 + c) : 0.0;
        }
        return __ldg(p + (3 * d + k) * n + t);
    }
    __device__ __forceinline__ double J(int t) const
    {
        if (EXT) return __ldg(p + 5 * n12 + t % n12);
        return __ldg(p + 9 * n + t);
    }
};

// ---------------------------------------------------------------------------
// register line derivative: out_a = sum_m D_am v_m (even-odd split of the GL
// D, as dline_inplace), plus the strong-form lifting of the two end points
// out_0 -= (N(N+1)/2)(gm - v_0), out_N += (N(N+1)/2)(gp - v_N) when lift.
// ---------------------------------------------------------------------------
template <int L>
__device__ __forceinline__ void dline_reg(const double (&v)[L], double (&out)[L], bool lift, double gm, double gp)
{
    constexpr int N = L - 1, H = L / 2;
    constexpr bool odd = (L & 1) != 0;
    constexpr double CL = 0.5 * N * (N + 1);
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
        out[a] = p + q;
        out[N - a] = p - q;
    }
    if (odd) {
        double s = c_EOM[N][0] * o[0];
#pragma unroll
        for (int m = 1; m < H; ++m) s = fma(c_EOM[N][m], o[m], s);
        out[H] = s;
    }
    if (lift) {
        out[0] -= CL * (gm - v[0]);
        out[N] += CL * (gp - v[N]);
    }
}

__device__ __forceinline__ void line_geom(int d, int line, int n1, int n2, int& base, int& stride)
{
    if (d == 0) { base = n1 * line; stride = 1; }                                    // line = j + n2 k
    else if (d == 1) { base = line % n1 + n1 * n2 * (line / n1); stride = n1; }      // line = i + n1 k
    else { base = line; stride = n1 * n2; }                                           // line = i + n1 j
}

// ---------------------------------------------------------------------------
// k_ns_grad: BR1 gradient, one CTA per item
// ---------------------------------------------------------------------------
template <int L, bool EXT>
__device__ __forceinline__ void grad_line(const NsElemParams& P, const Met<EXT>& M, const double* Qs, double* GA, int n,
                                          int d, int k, int kk, int nk, int line, int base, int stride, bool first,
                                          long long fm, long long fp, int nf)
{
    double ja[L];
#pragma unroll
    for (int m = 0; m < L; ++m) ja[m] = M.ja(d, k, base + m * stride);
    const bool lift = fm >= 0;
#pragma unroll 1
    for (int v = 0; v < NV; ++v) {
        double pv[L], out[L];
#pragma unroll
        for (int m = 0; m < L; ++m) pv[m] = ja[m] * Qs[v * n + base + m * stride];
        double gm = 0.0, gp = 0.0;
        if (lift) {
            gm = __ldg(P.blk + fm + (long long)(kk * NV + v) * nf + line);
            gp = __ldg(P.blk + fp + (long long)(kk * NV + v) * nf + line);
        }
        dline_reg<L>(pv, out, lift, gm, gp);
        double* acc = GA + (k * NV + v) * n + base;
        if (first) {
#pragma unroll
            for (int m = 0; m < L; ++m) acc[m * stride] = out[m];
        } else {
#pragma unroll
            for (int m = 0; m < L; ++m) acc[m * stride] += out[m];
        }
    }
}

template <bool EXT>
__global__ void __launch_bounds__(NS_BS) k_ns_grad(NsElemParams P)
{
    extern __shared__ __align__(16) double sm[];
    __shared__ long long s_off[NS_MAXSLOTS];
    __shared__ int s_e[NS_MAXSLOTS];
    const NsItem it = P.items[P.ibase + blockIdx.x];
    int N1, N2, N3;
    unpack_ord(it.ord, N1, N2, N3);
    const int n1 = N1 + 1, n2 = N2 + 1, n3 = N3 + 1, n = n1 * n2 * n3;
    const int cnt = it.count, NN = cnt * n;
    if (threadIdx.x < cnt) {
        const int e = P.elist[it.start + threadIdx.x];
        s_e[threadIdx.x] = e;
        s_off[threadIdx.x] = P.off[e];
    }
    __syncthreads();
    double* Q = sm;               // [slot][v][node]
    double* GA = Q + NV * NN;     // [slot][k][v][node] = J g
    for (int idx = threadIdx.x; idx < NV * NN; idx += NS_BS) {
        const int slot = idx / (NV * n);
        Q[idx] = __ldg(P.q + s_off[slot] + (idx - slot * NV * n));
    }
    __syncthreads();
    const int nn[3] = {n1, n2, n3};
    for (int d = 0; d < 3; ++d) {
        const int nd = nn[d], nl = n / nd;
        const int nk = EXT ? ext_nk(d) : 3;
        const int ntask = cnt * nl * nk;
        for (int task = threadIdx.x; task < ntask; task += NS_BS) {
            const int kk = task % nk;
            const int rest = task / nk;
            const int line = rest % nl, slot = rest / nl;
            const int k = EXT ? ext_k(d, kk) : kk;
            const bool first = EXT ? (d == 0 || d == 2) : d == 0;
            int base, stride;
            line_geom(d, line, n1, n2, base, stride);
            const int e = s_e[slot];
            Met<EXT> M;
            M.init(P, e, s_off[slot], n, n1, n2);
            const long long fm = P.fofs ? P.fofs[6LL * e + 2 * d] : -1, fp = P.fofs ? P.fofs[6LL * e + 2 * d + 1] : -1;
            const double* Qs = Q + slot * NV * n;
            double* G = GA + slot * 15 * n;
            switch (nd) {
                case 2: grad_line<2, EXT>(P, M, Qs, G, n, d, k, kk, nk, line, base, stride, first, fm, fp, nl); break;
                case 3: grad_line<3, EXT>(P, M, Qs, G, n, d, k, kk, nk, line, base, stride, first, fm, fp, nl); break;
                case 4: grad_line<4, EXT>(P, M, Qs, G, n, d, k, kk, nk, line, base, stride, first, fm, fp, nl); break;
                case 5: grad_line<5, EXT>(P, M, Qs, G, n, d, k, kk, nk, line, base, stride, first, fm, fp, nl); break;
                case 6: grad_line<6, EXT>(P, M, Qs, G, n, d, k, kk, nk, line, base, stride, first, fm, fp, nl); break;
                case 7: grad_line<7, EXT>(P, M, Qs, G, n, d, k, kk, nk, line, base, stride, first, fm, fp, nl); break;
                case 8: grad_line<8, EXT>(P, M, Qs, G, n, d, k, kk, nk, line, base, stride, first, fm, fp, nl); break;
                default: grad_line<9, EXT>(P, M, Qs, G, n, d, k, kk, nk, line, base, stride, first, fm, fp, nl); break;
            }
        }
        __syncthreads();
    }
    // g = (J g) / J, written [k][v][node] at 3 x offset (coalesced per slot)
    for (int idx = threadIdx.x; idx < NN; idx += NS_BS) {
        const int slot = idx / n, t = idx - slot * n;
        Met<EXT> M;
        M.init(P, s_e[slot], s_off[slot], n, n1, n2);
        const double iJ = 1.0 / M.J(t);
        const double* G = GA + slot * 15 * n + t;
        double* o = P.gout + 3 * s_off[slot] + t;
#pragma unroll
        for (int c = 0; c < 15; ++c) o[(long long)c * n] = G[c * n] * iJ;
    }
}

// ---------------------------------------------------------------------------
// k_ns_res: residual / RK stage, one CTA per item
// ---------------------------------------------------------------------------
template <bool EXT, bool NSF>
__global__ void __launch_bounds__(NS_BS) k_ns_res(NsElemParams P)
{
    extern __shared__ __align__(16) double sm[];
    __shared__ long long s_off[NS_MAXSLOTS];
    __shared__ int s_e[NS_MAXSLOTS];
    __shared__ double red[32];
    const NsItem it = P.items[P.ibase + blockIdx.x];
    int N1, N2, N3;
    unpack_ord(it.ord, N1, N2, N3);
    const int n1 = N1 + 1, n2 = N2 + 1, n3 = N3 + 1, n = n1 * n2 * n3;
    const int cnt = it.count, NN = cnt * n;
    if (threadIdx.x < cnt) {
        const int e = P.elist[it.start + threadIdx.x];
        s_e[threadIdx.x] = e;
        s_off[threadIdx.x] = P.off[e];
    }
    __syncthreads();
    double* Q = sm;              // [slot][v][node]
    double* F = Q + NV * NN;     // [d][slot][v][node]
    // node phase: q, grad q, metrics -> contravariant fluxes of the three directions
    for (int idx = threadIdx.x; idx < NN; idx += NS_BS) {
        const int slot = idx / n, t = idx - slot * n;
        const long long o = s_off[slot];
        Met<EXT> M;
        M.init(P, s_e[slot], o, n, n1, n2);
        double qv[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            qv[v] = __ldg(P.q + o + (long long)v * n + t);
            Q[slot * NV * n + v * n + t] = qv[v];
        }
        ViscNode V;
        if (NSF) {
            double gv[15];
            load_grad(P.grad + 3 * o + t, n, gv);
            visc_node(qv, gv, P.ph, V);
        }
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            const double ax = M.ja(d, 0, t), ay = M.ja(d, 1, t), az = M.ja(d, 2, t);
            double Fv[NV];
            adv_dot(qv, ax, ay, az, P.ph.gm1, Fv);
            if (NSF) {
                double fv[NV];
                visc_along(V, ax, ay, az, fv);
#pragma unroll
                for (int v = 0; v < NV; ++v) Fv[v] -= fv[v];
            }
            double* Fd = F + d * NV * NN + slot * NV * n + t;
#pragma unroll
            for (int v = 0; v < NV; ++v) Fd[v * n] = Fv[v];
        }
    }
    __syncthreads();
    // line phase: every line of every direction, one variable per task, in place
    const int nl0 = n / n1, nl1 = n / n2, nl2 = n / n3;
    const int t0 = cnt * NV * nl0, t1 = t0 + cnt * NV * nl1, ntask = t1 + cnt * NV * nl2;
    for (int task = threadIdx.x; task < ntask; task += NS_BS) {
        int d, r, nl, nd;
        if (task < t0) { d = 0; r = task; nl = nl0; nd = n1; }
        else if (task < t1) { d = 1; r = task - t0; nl = nl1; nd = n2; }
        else { d = 2; r = task - t1; nl = nl2; nd = n3; }
        const int v = r % NV;
        const int rest = r / NV;
        const int line = rest % nl, slot = rest / nl;
        int base, stride;
        line_geom(d, line, n1, n2, base, stride);
        double* Fl = F + d * NV * NN + slot * NV * n + v * n + base;
        if (P.fofs) {
            const long long e6 = 6LL * s_e[slot] + 2 * d;
            const double gm = __ldg(P.blk + P.fofs[e6] + (long long)v * nl + line);
            const double gp = __ldg(P.blk + P.fofs[e6 + 1] + (long long)v * nl + line);
            switch (nd) {
                case 2: dline_lift<2>(Fl, stride, gm, gp); break;
                case 3: dline_lift<3>(Fl, stride, gm, gp); break;
                case 4: dline_lift<4>(Fl, stride, gm, gp); break;
                case 5: dline_lift<5>(Fl, stride, gm, gp); break;
                case 6: dline_lift<6>(Fl, stride, gm, gp); break;
                case 7: dline_lift<7>(Fl, stride, gm, gp); break;
                case 8: dline_lift<8>(Fl, stride, gm, gp); break;
                default: dline_lift<9>(Fl, stride, gm, gp); break;
            }
        } else {
            switch (nd) {
                case 2: dline_inplace<2>(Fl, stride); break;
                case 3: dline_inplace<3>(Fl, stride); break;
                case 4: dline_inplace<4>(Fl, stride); break;
                case 5: dline_inplace<5>(Fl, stride); break;
                case 6: dline_inplace<6>(Fl, stride); break;
                case 7: dline_inplace<7>(Fl, stride); break;
                case 8: dline_inplace<8>(Fl, stride); break;
                default: dline_inplace<9>(Fl, stride); break;
            }
        }
    }
    __syncthreads();
    // epilogue: Qdot = -(sum_d)/J, or the low-storage RK update (+ CFL / DFL rates)
    const double dt = P.mode ? *P.dt : 0.0;
    double lmax = 0.0, vmax = 0.0;
    for (int idx = threadIdx.x; idx < NN; idx += NS_BS) {
        const int slot = idx / n, t = idx - slot * n;
        const long long o = s_off[slot];
        Met<EXT> M;
        M.init(P, s_e[slot], o, n, n1, n2);
        const double iJ = 1.0 / M.J(t);
        const int si = slot * NV * n + t;
        double A[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) A[v] = (F[si + v * n] + F[NV * NN + si + v * n]) + F[2 * NV * NN + si + v * n];
        if (P.mode == 0) {
#pragma unroll
            for (int v = 0; v < NV; ++v) P.out[o + (long long)v * n + t] = -A[v] * iJ;
        } else {
            double qn[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                const long long ix = o + (long long)v * n + t;
                const double gn = (P.rkA == 0.0 ? 0.0 : P.rkA * P.g[ix]) - dt * A[v] * iJ;
                P.g[ix] = gn;
                qn[v] = Q[si + v * n] + P.rkB * gn;
                P.out[ix] = qn[v];
            }
            if (P.lam_max) {
                int ijk[3];
                node_ijk(t, n1, n2, ijk[0], ijk[1], ijk[2]);
                const double ir = 1.0 / qn[0];
                const double p = P.ph.gm1 * (qn[4] - 0.5 * ir * (qn[1] * qn[1] + qn[2] * qn[2] + qn[3] * qn[3]));
                const double c = sqrt(P.ph.gamma * p * ir);
                double lam = 0.0, nu = 0.0;
                const double numax = P.ph.mu * ir * fmax(4.0 / 3.0, P.ph.gamma / P.ph.Pr);
                const int np1[3] = {n1, n2, n3};
#pragma unroll
                for (int d = 0; d < 3; ++d) {
                    const double a0 = M.ja(d, 0, t) * iJ, a1 = M.ja(d, 1, t) * iJ, a2 = M.ja(d, 2, t) * iJ;
                    const double an2 = a0 * a0 + a1 * a1 + a2 * a2;
                    const double ua = (qn[1] * a0 + qn[2] * a1 + qn[3] * a2) * ir;
                    const double np = np1[d];
                    lam += (fabs(ua) + c * sqrt(an2)) * np * np * 0.5;
                    nu += numax * an2 * np * np * np * np * 0.25;
                }
                lmax = fmax(lmax, lam);
                vmax = fmax(vmax, nu);
            }
        }
    }
    if (P.lam_max) {
        lmax = block_max(lmax, red);
        vmax = block_max(vmax, red);
        if (threadIdx.x == 0) {
            atomicMax(P.lam_max, (unsigned long long)__double_as_longlong(lmax));
            if (NSF) atomicMax(P.lam_max + 1, (unsigned long long)__double_as_longlong(vmax));
        }
    }
}

// ---------------------------------------------------------------------------
// k_ns_face: one W-warp group per face
// ---------------------------------------------------------------------------
template <int W>
__device__ __forceinline__ void grp_sync(int gid)
{
    if (W == 1) {
        __syncwarp();
    } else {
        asm volatile("bar.sync %0, %1;\n" ::"r"(gid + 1), "r"(32 * W) : "memory");
    }
}

// groups per CTA and buffer sizes
template <int W>
struct FaceCfg {
    static constexpr int G = W == 1 ? 4 : 2;      // groups per CTA
    static constexpr int BS = G * 32 * W;
    static constexpr int CAP = 32 * W;            // points per component slot
    static constexpr int BUF = 15 * CAP;          // one buffer: 15 component slots
    static constexpr size_t smem = sizeof(double) * (size_t)G * 2 * BUF;
};

// side descriptor inside a face
struct FSide {
    long long off;  // state offset (-1: ghost)
    int n, sa, sb, base, sta, stb;
};

__device__ __forceinline__ FSide face_side(long long off, int ord, int d, bool isL)
{
    int N[3];
    mt_unpack(ord, N);
    const int ta = d == 0 ? 1 : 0, tb = d == 2 ? 1 : 2;
    const int st[3] = {1, N[0] + 1, (N[0] + 1) * (N[1] + 1)};
    FSide s;
    s.off = off;
    s.n = st[2] * (N[2] + 1);
    s.sa = N[ta] + 1;
    s.sb = N[tb] + 1;
    s.base = isL ? N[d] * st[d] : 0;
    s.sta = st[ta];
    s.stb = st[tb];
    return s;
}

// Interpolate `nc` components of a side trace to the mortar grid: gather
// (src + c * cstride + node) into X, pass A (along a) into Y where s_a < m_a;
// then each point owner (p < ma mb) reads its values through pass B (along b)
// into val[c].  Buffers hold CAP points per component.
template <int W, int NCM>
__device__ __forceinline__ void side_to_mortar(const double* __restrict__ src, long long cstride, const FSide& s, int nc,
                                               int ma, int mb, const Tables* tab, double* X, double* Y, int l, int gid,
                                               int p, double* val)
{
    constexpr int CAP = 32 * W;
    const int sa = s.sa, sb = s.sb, ns = sa * sb;
    for (int idx = l; idx < nc * ns; idx += 32 * W) {
        const int c = idx / ns, r = idx - c * ns;
        const int b = r / sa, a = r - b * sa;
        X[c * CAP + r] = __ldg(src + c * cstride + s.base + a * s.sta + b * s.stb);
    }
    grp_sync<W>(gid);
    const double* Z = X;
    if (sa < ma) {
        const double* Ta = tab->T[sa - 1][ma - 1];  // [i * sa + a]
        for (int idx = l; idx < nc * sb * ma; idx += 32 * W) {
            const int c = idx / (sb * ma), r = idx - c * (sb * ma);
            const int b = r / ma, i = r - b * ma;
            const double* x = X + c * CAP + b * sa;
            double acc = 0.0;
            for (int a = 0; a < sa; ++a) acc = fma(__ldg(Ta + i * sa + a), x[a], acc);
            Y[c * CAP + b * ma + i] = acc;
        }
        grp_sync<W>(gid);
        Z = Y;
    }
    if (p < ma * mb) {
        const int j = p / ma, i = p - j * ma;
        if (sb < mb) {
            const double* Tb = tab->T[sb - 1][mb - 1];
#pragma unroll
            for (int c = 0; c < NCM; ++c) {
                if (c >= nc) break;
                double acc = 0.0;
                for (int b = 0; b < sb; ++b) acc = fma(__ldg(Tb + j * sb + b), Z[c * CAP + b * ma + i], acc);
                val[c] = acc;
            }
        } else {
#pragma unroll
            for (int c = 0; c < NCM; ++c) {
                if (c >= nc) break;
                val[c] = Z[c * CAP + j * ma + i];
            }
        }
    }
    grp_sync<W>(gid);  // X / Y free for the next call
}

// Project nc components held at the mortar points (Fm[c * CAP + p]) onto a
// side's own face nodes and store them to out[c * (sa sb) + a + sa b].
template <int W>
__device__ __forceinline__ void mortar_to_side(const double* Fm, int nc, int ma, int mb, int sa, int sb, const Tables* tab,
                                               double* Y, double* __restrict__ out, int l, int gid)
{
    constexpr int CAP = 32 * W;
    const double* Z = Fm;
    int zrow = ma;  // row length of Z (points along a)
    if (sa < ma) {
        const double* Pa = tab->P[ma - 1][sa - 1];  // [i * ma + k]
        for (int idx = l; idx < nc * mb * sa; idx += 32 * W) {
            const int c = idx / (mb * sa), r = idx - c * (mb * sa);
            const int b = r / sa, i = r - b * sa;
            const double* f = Fm + c * CAP + b * ma;
            double acc = 0.0;
            for (int k = 0; k < ma; ++k) acc = fma(__ldg(Pa + i * ma + k), f[k], acc);
            Y[c * CAP + b * sa + i] = acc;
        }
        grp_sync<W>(gid);
        Z = Y;
        zrow = sa;
    }
    const int ns = sa * sb;
    if (sb < mb) {
        const double* Pb = tab->P[mb - 1][sb - 1];  // [j * mb + b]
        for (int idx = l; idx < nc * ns; idx += 32 * W) {
            const int c = idx / ns, r = idx - c * ns;
            const int j = r / sa, i = r - j * sa;
            double acc = 0.0;
            for (int b = 0; b < mb; ++b) acc = fma(__ldg(Pb + j * mb + b), Z[c * CAP + b * zrow + i], acc);
            out[(long long)c * ns + r] = acc;
        }
    } else {
        for (int idx = l; idx < nc * ns; idx += 32 * W) {
            const int c = idx / ns, r = idx - c * ns;
            out[(long long)c * ns + r] = Z[c * CAP + r];
        }
    }
    grp_sync<W>(gid);
}

template <int W, int MODE>
__global__ void __launch_bounds__(FaceCfg<W>::BS) k_ns_face(NsFaceParams P)
{
    using C = FaceCfg<W>;
    constexpr int CAP = C::CAP;
    extern __shared__ __align__(16) double fsm[];
    const int gid = threadIdx.x / (32 * W), l = threadIdx.x - gid * 32 * W;
    const int fi = P.fbase + blockIdx.x * C::G + gid;
    if (fi >= P.fend) return;  // the whole group leaves (named barriers are per group)
    double* X = fsm + gid * 2 * C::BUF;
    double* Y = X + C::BUF;
    const NsFace F = P.faces[fi];
    const int d = F.d;
    const bool hasL = F.offL >= 0, hasR = F.offR >= 0;
    const FSide SL = face_side(F.offL, F.ordL, d, true);
    const FSide SR = face_side(F.offR, F.ordR, d, false);
    const int ma = max(SL.sa, SR.sa), mb = max(SL.sb, SR.sb), nm = ma * mb;
    const int p = l;  // mortar point of this thread
    const bool pon = p < nm;
    double jf[3] = {0.0, 0.0, 1.0};
    if (pon) {
        const double* fg = P.fg + F.mg;
        jf[0] = __ldg(fg + p);
        jf[1] = __ldg(fg + nm + p);
        jf[2] = __ldg(fg + 2 * nm + p);
    }
    // ---- q of both sides at the mortar points ----
    double qL[NV] = {0, 0, 0, 0, 0}, qR[NV] = {0, 0, 0, 0, 0};
    if (hasL) side_to_mortar<W, NV>(P.q + SL.off, SL.n, SL, NV, ma, mb, P.tab, X, Y, l, gid, p, qL);
    if (hasR) side_to_mortar<W, NV>(P.q + SR.off, SR.n, SR, NV, ma, mb, P.tab, X, Y, l, gid, p, qR);
    const int kind = F.kind;
    int nout;
    if (MODE == MODE_QHAT) {
        const int nk = P.ext ? ext_nk(d) : 3;
        nout = NV * nk;
        if (pon) {
            const double* qi = hasL ? qL : qR;
            double qh[NV];
            if (kind == 2) {  // wall: zero velocity, keep rho and the internal energy (A10)
                qh[0] = qi[0];
                qh[1] = 0.0;
                qh[2] = 0.0;
                qh[3] = 0.0;
                qh[4] = qi[4] - 0.5 * (qi[1] * qi[1] + qi[2] * qi[2] + qi[3] * qi[3]) / qi[0];
            } else if (kind == 3) {
#pragma unroll
                for (int v = 0; v < NV; ++v) qh[v] = 0.5 * (qi[v] + P.ph.qinf[v]);
            } else {
#pragma unroll
                for (int v = 0; v < NV; ++v) qh[v] = 0.5 * (qL[v] + qR[v]);
            }
            for (int kk = 0; kk < nk; ++kk) {
                const int k = P.ext ? ext_k(d, kk) : kk;
#pragma unroll
                for (int v = 0; v < NV; ++v) X[(kk * NV + v) * CAP + p] = qh[v] * jf[k];
            }
        }
    } else {
        nout = NV;
        double G[NV] = {0, 0, 0, 0, 0};
        if (pon) {
            const double S = sqrt(jf[0] * jf[0] + jf[1] * jf[1] + jf[2] * jf[2]);
            const double nrm[3] = {jf[0] / S, jf[1] / S, jf[2] / S};
            if (kind >= 2) {
                double qg[NV];
                ghost_state(hasL ? qL : qR, kind == 2 ? -1 : -2, P.ph, qg);
                if (hasL) riemann(qL, qg, nrm, P.ph, G);
                else riemann(qg, qR, nrm, P.ph, G);
            } else {
                riemann(qL, qR, nrm, P.ph, G);
            }
#pragma unroll
            for (int v = 0; v < NV; ++v) G[v] *= S;
        }
        if (MODE == MODE_FLUX_NS) {
            // viscous fluxes along Ja_f: one side's interpolated gradient live at a time
            double fs[NV];
            double fsum[NV] = {0, 0, 0, 0, 0};
            for (int side = 0; side < 2; ++side) {
                const bool has = side ? hasR : hasL;
                if (!has) continue;
                const FSide& S = side ? SR : SL;
                double gv[15];
                side_to_mortar<W, 15>(P.grad + 3 * S.off, S.n, S, 15, ma, mb, P.tab, X, Y, l, gid, p, gv);
                if (pon) {
                    visc_dot(side ? qR : qL, gv, jf[0], jf[1], jf[2], P.ph, fs);
#pragma unroll
                    for (int v = 0; v < NV; ++v) fsum[v] += fs[v];
                }
            }
            if (pon) {
                if (kind == 2) {  // wall: inner viscous flux, u = 0 and adiabatic (A10)
                    fsum[4] = 0.0;
#pragma unroll
                    for (int v = 0; v < NV; ++v) G[v] -= fsum[v];
                } else if (kind == 3) {  // far field: inner viscous flux
#pragma unroll
                    for (int v = 0; v < NV; ++v) G[v] -= fsum[v];
                } else {  // BR1 average
#pragma unroll
                    for (int v = 0; v < NV; ++v) G[v] -= 0.5 * fsum[v];
                }
            }
        }
        if (pon) {
#pragma unroll
            for (int v = 0; v < NV; ++v) X[v * CAP + p] = G[v];
        }
    }
    grp_sync<W>(gid);
    // ---- back to the sides' own face nodes ----
    const long long oL = MODE == MODE_QHAT ? F.hL : F.outL, oR = MODE == MODE_QHAT ? F.hR : F.outR;
    if (kind == 0) {  // conforming: the mortar is the face, one shared block
        double* out = P.out + oL;
        for (int idx = l; idx < nout * nm; idx += 32 * W) {
            const int c = idx / nm, r = idx - c * nm;
            out[idx] = X[c * CAP + r];
        }
        return;
    }
    if (hasL) mortar_to_side<W>(X, nout, ma, mb, SL.sa, SL.sb, P.tab, Y, P.out + oL, l, gid);
    if (hasR) mortar_to_side<W>(X, nout, ma, mb, SR.sa, SR.sb, P.tab, Y, P.out + oR, l, gid);
}

}  // namespace dgtau
