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
    int* flag;                    // admissibility: [0] violations, [1] first element (reading A25)
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
// small helpers
// ---------------------------------------------------------------------------

// x / d for 0 <= x < 2^20, 1 <= d < 4096: umulhi(x, ceil(2^32 / d)) (error
// < x 2^-32 < 1/d, so the floor is exact); d = 1 is passed through.  The
// multipliers of d < NS_FDIV come from a constant table (no division at all).
constexpr int NS_FDIV = 1024;
static __constant__ unsigned c_fdiv[NS_FDIV];
struct FDiv {
    unsigned m;
    bool one;
    __device__ __forceinline__ void init(unsigned d)
    {
        one = d == 1;
        m = d < NS_FDIV ? c_fdiv[d] : (one ? 0u : 0xffffffffu / d + 1u);
    }
    __device__ __forceinline__ int div(int x) const { return one ? x : (int)__umulhi((unsigned)x, m); }
};

static inline cudaError_t ns_copy_constants()
{
    static unsigned h[NS_FDIV];
    for (unsigned d = 2; d < NS_FDIV; ++d) h[d] = 0xffffffffu / d + 1u;
    h[0] = h[1] = 0;
    return cudaMemcpyToSymbol(c_fdiv, h, sizeof(h));
}

// metric terms of one element: EXT 6 per (i, j) column, else 10 per node
template <bool EXT>
struct Met {
    const double* p;
    int n, n12;
    __device__ __forceinline__ void init(const NsElemParams& P, int e, long long o, int n_, int n12_)
    {
        n = n_;
        n12 = n12_;
        p = EXT ? P.metc + P.coff[e] : P.met + 2 * o;
    }
    // (Ja^d)_k at node t (column c = t mod n1 n2, EXT)
    __device__ __forceinline__ double ja(int d, int k, int t, int c) const
    {
        if (EXT) {
            if (d < 2) return k == 2 ? 0.0 : __ldg(p + (2 * d + k) * n12 + c);
            return k == 2 ? __ldg(p + 4 * n12 + c) : 0.0;
        }
        return __ldg(p + (3 * d + k) * n + t);
    }
    __device__ __forceinline__ double J(int t, int c) const { return EXT ? __ldg(p + 5 * n12 + c) : __ldg(p + 9 * n + t); }
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

// per-item constants of the element kernels (scalars: no local-memory arrays)
struct ItemGeo {
    int n1, n2, n3, n, n12, cnt, NN;
    int nl0, nl1, nl2;
    FDiv dn, dn1, dn2, dn12, dnl0, dnl1, dnl2;
    __device__ __forceinline__ void init(int ord, int count)
    {
        int N1, N2, N3;
        unpack_ord(ord, N1, N2, N3);
        n1 = N1 + 1;
        n2 = N2 + 1;
        n3 = N3 + 1;
        n12 = n1 * n2;
        n = n12 * n3;
        cnt = count;
        NN = cnt * n;
        nl0 = n2 * n3;
        nl1 = n1 * n3;
        nl2 = n12;
        dn.init(n);
        dn1.init(n1);
        dn2.init(n2);
        dn12.init(n12);
        dnl0.init(nl0);
        dnl1.init(nl1);
        dnl2.init(nl2);
    }
    __device__ __forceinline__ int nl(int d) const { return d == 0 ? nl0 : (d == 1 ? nl1 : nl2); }
    __device__ __forceinline__ int nd(int d) const { return d == 0 ? n1 : (d == 1 ? n2 : n3); }
    __device__ __forceinline__ int div_nl(int d, int x) const { return d == 0 ? dnl0.div(x) : (d == 1 ? dnl1.div(x) : dnl2.div(x)); }
    // line `line` of direction d: first node, node stride, first column, column stride
    __device__ __forceinline__ void line(int d, int line, int& base, int& stride, int& cb, int& cs) const
    {
        if (d == 0) {  // line = j + n2 k
            base = n1 * line;
            stride = 1;
            const int k = dn2.div(line);
            cb = n1 * (line - n2 * k);
            cs = 1;
        } else if (d == 1) {  // line = i + n1 k
            const int k = dn1.div(line);
            const int i = line - n1 * k;
            base = i + n12 * k;
            stride = n1;
            cb = i;
            cs = n1;
        } else {  // line = i + n1 j
            base = line;
            stride = n12;
            cb = line;
            cs = 0;
        }
    }
};

__device__ __forceinline__ int nk_of(bool ext, int d) { return ext ? ext_nk(d) : 3; }

// split (kk, rest) = (r mod nk, r / nk) for nk in {1, 2, 3}
__device__ __forceinline__ void split_nk(int nk, int r, int& kk, int& rest)
{
    if (nk == 1) { kk = 0; rest = r; }
    else if (nk == 2) { kk = r & 1; rest = r >> 1; }
    else { rest = r / 3; kk = r - 3 * rest; }
}

// ===========================================================================
// Element kernels (BR1 gradient, residual / RK stage): warp-specialised
// producer / consumer pipeline over items of same-order elements.
//   * producer warp (the CTA's last warp): fetches item k+1's element ids and
//     offsets and issues the 1-D TMA bulk copies (cp.async.bulk, mbarrier
//     complete_tx) of every element block the item needs -- state q (16-byte
//     envelope of [off, off + 5n), data at +off&1), metric terms, the six
//     face blocks -- into stage (k+1) mod NST;
//   * NS_BS consumer threads: one thread per node, compute item k from stage
//     k mod NST (named barrier 1 between phases), then release the stage.
// ===========================================================================
constexpr int NS_PROD = 32;           // producer warp
constexpr int NS_THREADS = NS_BS + NS_PROD;
constexpr int NS_MAXST = 4;           // pipeline stages (host picks 1..NS_MAXST)

__device__ __forceinline__ void mbar_arrive(unsigned long long* b)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void cons_sync() { asm volatile("bar.sync 1, %0;\n" ::"r"(NS_BS) : "memory"); }

// per-stage metadata (written by the producer before its arrive)
struct NsStageMeta {
    int cnt, ord;
    int qsh[NS_MAXSLOTS];
    int e[NS_MAXSLOTS];
    long long off[NS_MAXSLOTS];
};

// words of the face block of direction d: H (BR1 terms, nk components) or G (flux)
__host__ __device__ __forceinline__ int ns_fblk(bool hblk, bool ext, int d, int nl)
{
    return (NV * (hblk ? (ext ? ext_nk(d) : 3) : 1) * nl + 1) & ~1;
}

// stage layout of an item: per slot [q: EVEN(5n) + 2][metrics: EVEN(MW)][faces: 6 blocks]
struct StageLayout {
    int qs, ms, fs;   // per-slot strides of the three regions
    int b0, b1, b2;   // face block words of the three directions
    int q0, m0, f0;   // region bases
    __host__ __device__ void init(bool ext, bool hblk, int n1, int n2, int n3, int cnt, bool faces)
    {
        const int n12 = n1 * n2, n = n12 * n3;
        qs = ((NV * n + 1) & ~1) + 2;
        ms = ext ? ((6 * n12 + 1) & ~1) : 10 * n;
        b0 = faces ? ns_fblk(hblk, ext, 0, n2 * n3) : 0;
        b1 = faces ? ns_fblk(hblk, ext, 1, n1 * n3) : 0;
        b2 = faces ? ns_fblk(hblk, ext, 2, n12) : 0;
        fs = 2 * (b0 + b1 + b2);
        q0 = 0;
        m0 = cnt * qs;
        f0 = m0 + cnt * ms;
    }
    // offset of face f = 2d + s inside the slot's face region
    __host__ __device__ __forceinline__ int fb(int f) const
    {
        return (f >= 1 ? b0 : 0) + (f >= 2 ? b0 : 0) + (f >= 3 ? b1 : 0) + (f >= 4 ? b1 : 0) + (f >= 5 ? b2 : 0);
    }
    __host__ __device__ int words(int cnt) const { return cnt * (qs + ms + fs); }
};

// Producer: item `item` into stage `st` (full barrier fb).  hblk: face blocks
// are H (gradient kernel) else G (residual kernel).
template <bool EXT>
__device__ __forceinline__ void ns_produce(const NsElemParams& P, int item, double* st, NsStageMeta& M,
                                           unsigned long long* full, bool hblk, long long qlen)
{
    const int lane = threadIdx.x & 31;
    const NsItem it = P.items[P.ibase + item];
    int N1, N2, N3;
    unpack_ord(it.ord, N1, N2, N3);
    const int n1 = N1 + 1, n2 = N2 + 1, n3 = N3 + 1, n12 = n1 * n2, n = n12 * n3;
    const bool faces = P.fofs != nullptr;
    StageLayout Lo;
    Lo.init(EXT, hblk, n1, n2, n3, it.count, faces);
    const int nl[3] = {n2 * n3, n1 * n3, n12};
    unsigned bytes = 0;
    long long a = 0, b = 0, mo = 0, fo[6];
    bool clip = false;
    if (lane < it.count) {
        const int e = P.elist[it.start + lane];
        const long long off = P.off[e];
        a = off & ~1LL;
        b = (off + NV * n + 1) & ~1LL;
        clip = b > qlen;
        if (clip) b -= 2;
        bytes += (unsigned)((b - a) * 8);
        mo = EXT ? P.coff[e] : 2 * off;
        bytes += (unsigned)(Lo.ms * 8);
#pragma unroll
        for (int f = 0; f < 6; ++f) {
            fo[f] = faces ? P.fofs[6LL * e + f] : 0;
            if (faces) bytes += (unsigned)(ns_fblk(hblk, EXT, f >> 1, nl[f >> 1]) * 8);
        }
        M.qsh[lane] = (int)(off & 1);
        M.e[lane] = e;
        M.off[lane] = off;
        if (clip) st[Lo.q0 + lane * Lo.qs + (b - a)] = P.q[b];  // last 8 bytes by hand (buffer end)
    }
    if (lane == 0) {
        M.cnt = it.count;
        M.ord = it.ord;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) bytes += __shfl_xor_sync(0xffffffffu, bytes, o);
    __syncwarp();
    if (lane == 0) mbar_expect_tx(full, bytes);
    __syncwarp();
    if (lane < it.count) {
        // residual kernel, RK stages 2-3: the register g is read in the epilogue -> into L2 now
        if (!hblk && P.mode == 1 && P.rkA != 0.0) bulk_prefetch_l2(P.g + a, (unsigned)((b - a) * 8));
        // residual kernel (NS): the node phase reads the element's gradient
        // (15 n, plain loads) -> into L2 one stage ahead (the buffer is
        // allocated with 2 doubles of slack: the rounded end stays inside)
        if (!hblk && P.grad) {
            const long long g0 = (3 * M.off[lane]) & ~1LL, g1 = (3 * M.off[lane] + 15LL * n + 1) & ~1LL;
            bulk_prefetch_l2(P.grad + g0, (unsigned)((g1 - g0) * 8));
        }
        bulk_g2s(st + Lo.q0 + lane * Lo.qs, P.q + a, (unsigned)((b - a) * 8), full);
        bulk_g2s(st + Lo.m0 + lane * Lo.ms, (EXT ? P.metc : P.met) + mo, (unsigned)(Lo.ms * 8), full);
        if (faces) {
#pragma unroll
            for (int f = 0; f < 6; ++f)
                bulk_g2s(st + Lo.f0 + lane * Lo.fs + Lo.fb(f), P.blk + fo[f],
                         (unsigned)(ns_fblk(hblk, EXT, f >> 1, nl[f >> 1]) * 8), full);
        }
    }
}

// stage words needed by an item (host: class sizing)
__host__ __device__ inline int ns_stage_words(bool ext, bool hblk, bool faces, int ord, int cnt)
{
    StageLayout Lo;
    Lo.init(ext, hblk, (ord & 255) + 1, ((ord >> 8) & 255) + 1, ((ord >> 16) & 255) + 1, cnt, faces);
    return Lo.words(cnt);
}

// ---------------------------------------------------------------------------
// BR1 gradient: J g_k = sum_d [ sum_m D^d_{a m} (Ja^d_k q)_m + lifting ], one
// consumer thread per node, the three directions' sums in registers.
// ---------------------------------------------------------------------------

// One direction's volume sum at node t for the NK metric components of that
// direction: acc[kk][v] += sum_m D_{a m} Ja_k(m) q_v(m) (line length L).
template <int L, int NK>
__device__ __forceinline__ void grad_dir(const double* __restrict__ Dr, const double* __restrict__ Qs, int n, int tb,
                                         int stride, const double* const* ja, int cb, int cs, double (&acc)[NK][NV])
{
    double w[L];
#pragma unroll
    for (int m = 0; m < L; ++m) w[m] = Dr[m];
#pragma unroll
    for (int m = 0; m < L; ++m) {
        const int tm = tb + m * stride;
        double qv[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) qv[v] = Qs[v * n + tm];
#pragma unroll
        for (int kk = 0; kk < NK; ++kk) {
            const double wj = w[m] * ja[kk][cb + m * cs];
#pragma unroll
            for (int v = 0; v < NV; ++v) acc[kk][v] = fma(wj, qv[v], acc[kk][v]);
        }
    }
}

template <int NK>
__device__ __forceinline__ void grad_dir_sw(int L, const double* Dr, const double* Qs, int n, int tb, int stride,
                                            const double* const* ja, int cb, int cs, double (&acc)[NK][NV])
{
    switch (L) {
        case 2: grad_dir<2, NK>(Dr, Qs, n, tb, stride, ja, cb, cs, acc); break;
        case 3: grad_dir<3, NK>(Dr, Qs, n, tb, stride, ja, cb, cs, acc); break;
        case 4: grad_dir<4, NK>(Dr, Qs, n, tb, stride, ja, cb, cs, acc); break;
        case 5: grad_dir<5, NK>(Dr, Qs, n, tb, stride, ja, cb, cs, acc); break;
        case 6: grad_dir<6, NK>(Dr, Qs, n, tb, stride, ja, cb, cs, acc); break;
        case 7: grad_dir<7, NK>(Dr, Qs, n, tb, stride, ja, cb, cs, acc); break;
        case 8: grad_dir<8, NK>(Dr, Qs, n, tb, stride, ja, cb, cs, acc); break;
        default: grad_dir<9, NK>(Dr, Qs, n, tb, stride, ja, cb, cs, acc); break;
    }
}

// J g at node t of an element (Qs: its state [v][node], Me: its metric block,
// Hs: its face blocks or null, Ds: D rows [3][81]), then g written to gout
template <bool EXT>
__device__ __forceinline__ void grad_node(const ItemGeo& I, const StageLayout& Lo, const double* Qs, const double* Me,
                                          const double* Hs, const double* Ds, int t, double* __restrict__ gout)
{
    const int n = I.n, n1 = I.n1, n2 = I.n2, n3 = I.n3, n12 = I.n12;
    const int k3 = I.dn12.div(t), c = t - n12 * k3;
    const int j = I.dn1.div(c), i = c - n1 * j;
    double g[3][NV];
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int v = 0; v < NV; ++v) g[k][v] = 0.0;
    if (EXT) {
        // d = 0: Ja^1 = (M0, M1, 0) at column m + n1 j; d = 1: Ja^2 = (M2, M3, 0)
        // at i + n1 m; d = 2: Ja^3 = (0, 0, M4) at column c
        {
            const double* ja[2] = {Me, Me + n12};
            double acc[2][NV] = {};
            grad_dir_sw<2>(n1, Ds + i * n1, Qs, n, t - i, 1, ja, n1 * j, 1, acc);
#pragma unroll
            for (int v = 0; v < NV; ++v) { g[0][v] = acc[0][v]; g[1][v] = acc[1][v]; }
        }
        {
            const double* ja[2] = {Me + 2 * n12, Me + 3 * n12};
            double acc[2][NV] = {};
            grad_dir_sw<2>(n2, Ds + NP * NP + j * n2, Qs, n, t - n1 * j, n1, ja, i, n1, acc);
#pragma unroll
            for (int v = 0; v < NV; ++v) { g[0][v] += acc[0][v]; g[1][v] += acc[1][v]; }
        }
        {
            const double* ja[1] = {Me + 4 * n12};
            double acc[1][NV] = {};
            grad_dir_sw<1>(n3, Ds + 2 * NP * NP + k3 * n3, Qs, n, c, n12, ja, c, 0, acc);
#pragma unroll
            for (int v = 0; v < NV; ++v) g[2][v] = acc[0][v];
        }
    } else {
        const int tb[3] = {t - i, t - n1 * j, c};
        const int ai[3] = {i, j, k3};
        const int stv[3] = {1, n1, n12};
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            const double* ja[3] = {Me + (3 * d) * n, Me + (3 * d + 1) * n, Me + (3 * d + 2) * n};
            double acc[3][NV] = {};
            const int L = d == 0 ? n1 : (d == 1 ? n2 : n3);
            grad_dir_sw<3>(L, Ds + d * NP * NP + ai[d] * L, Qs, n, tb[d], stv[d], ja, tb[d], stv[d], acc);
#pragma unroll
            for (int k = 0; k < 3; ++k)
#pragma unroll
                for (int v = 0; v < NV; ++v) g[k][v] += acc[k][v];
        }
    }
    // lifting (H - q Ja^d_k)/w at the faces through this node (strong form)
    if (Hs) {
        const int ai[3] = {i, j, k3};
        const int pt[3] = {j + n2 * k3, i + n1 * k3, c};
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            const int L = d == 0 ? n1 : (d == 1 ? n2 : n3);
            const int nk = EXT ? ext_nk(d) : 3;
            const int nf = d == 0 ? I.nl0 : (d == 1 ? I.nl1 : I.nl2);
#pragma unroll
            for (int sd = 0; sd < 2; ++sd) {
                if (ai[d] == (sd ? L - 1 : 0)) {
                    const double CL = (sd ? 0.5 : -0.5) * (L - 1) * L;  // +-1/w_0
                    const double* H = Hs + Lo.fb(2 * d + sd) + pt[d];
                    for (int kk = 0; kk < nk; ++kk) {
                        const int k = EXT ? ext_k(d, kk) : kk;
                        double jo;
                        if (EXT) jo = d < 2 ? Me[(2 * d + k) * n12 + c] : Me[4 * n12 + c];
                        else jo = Me[(3 * d + k) * n + t];
#pragma unroll
                        for (int v = 0; v < NV; ++v) g[k][v] += CL * (H[(kk * NV + v) * nf] - jo * Qs[v * n + t]);
                    }
                }
            }
        }
    }
    const double iJ = 1.0 / (EXT ? Me[5 * n12 + c] : Me[9 * n + t]);
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int v = 0; v < NV; ++v) gout[(long long)(k * NV + v) * n + t] = g[k][v] * iJ;
}

template <bool EXT>
__global__ void __launch_bounds__(NS_THREADS, 2) k_ns_grad(NsElemParams P, int nitems, int NST, int SW, long long qlen)
{
    extern __shared__ __align__(16) double sm[];
    __shared__ NsStageMeta meta[NS_MAXST];
    __shared__ __align__(8) unsigned long long full[NS_MAXST], empty[NS_MAXST];
    __shared__ double Ds[3 * NP * NP];
    if (blockIdx.x >= nitems) return;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS_MAXST; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NS_BS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x >= NS_BS) {  // producer warp
        int k = 0;
        for (int item = blockIdx.x; item < nitems; item += gridDim.x, ++k) {
            const int s = k % NST;
            if (k >= NST) mbar_wait(&empty[s], ((k / NST) - 1) & 1);
            ns_produce<EXT>(P, item, sm + s * SW, meta[s], &full[s], true, qlen);
        }
        return;
    }
    int k = 0;
    int ordD = -1;
    for (int item = blockIdx.x; item < nitems; item += gridDim.x, ++k) {
        const int s = k % NST;
        mbar_wait(&full[s], (k / NST) & 1);
        const NsStageMeta& M = meta[s];
        ItemGeo I;
        I.init(M.ord, M.cnt);
        if (M.ord != ordD) {  // D rows of the item's orders (uniform branch)
            cons_sync();
            for (int w = threadIdx.x; w < 3 * NP * NP; w += NS_BS) {
                const int d = w / (NP * NP), r = w - d * NP * NP;
                const int L = I.nd(d);
                if (r < L * L) Ds[w] = c_D[(L - 1) * NP * NP + r];
            }
            cons_sync();
            ordD = M.ord;
        }
        StageLayout Lo;
        Lo.init(EXT, true, I.n1, I.n2, I.n3, I.cnt, P.fofs != nullptr);
        const double* st = sm + s * SW;
        for (int idx = threadIdx.x; idx < I.NN; idx += NS_BS) {
            const int slot = I.dn.div(idx), t = idx - slot * I.n;
            grad_node<EXT>(I, Lo, st + Lo.q0 + slot * Lo.qs + M.qsh[slot], st + Lo.m0 + slot * Lo.ms,
                           P.fofs ? st + Lo.f0 + slot * Lo.fs : nullptr, Ds, t, P.gout + 3 * M.off[slot]);
        }
        mbar_arrive(&empty[s]);
    }
}

// ---------------------------------------------------------------------------
// residual / RK stage: node phase (contravariant fluxes of the three
// directions into F), line phase (in-place derivative + lifting of (G - Ft)/w),
// epilogue (Qdot = -(sum_d)/J, or the RK update + CFL / DFL rates).
// ---------------------------------------------------------------------------
template <bool EXT, bool NSF>
__global__ void __launch_bounds__(NS_THREADS, 2) k_ns_res(NsElemParams P, int nitems, int NST, int SW, int maxNN,
                                                          long long qlen)
{
    extern __shared__ __align__(16) double sm[];
    __shared__ NsStageMeta meta[NS_MAXST];
    __shared__ __align__(8) unsigned long long full[NS_MAXST], empty[NS_MAXST];
    __shared__ double red[32];
    if (blockIdx.x >= nitems) return;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS_MAXST; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NS_BS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x >= NS_BS) {  // producer warp
        int k = 0;
        for (int item = blockIdx.x; item < nitems; item += gridDim.x, ++k) {
            const int s = k % NST;
            if (k >= NST) mbar_wait(&empty[s], ((k / NST) - 1) & 1);
            ns_produce<EXT>(P, item, sm + s * SW, meta[s], &full[s], false, qlen);
        }
        return;
    }
    double* F = sm + NST * SW;  // [d][slot][v][node]
    const double dt = P.mode ? *P.dt : 0.0;
    double lmax = 0.0, vmax = 0.0;
    int k = 0;
    for (int item = blockIdx.x; item < nitems; item += gridDim.x, ++k) {
        const int s = k % NST;
        mbar_wait(&full[s], (k / NST) & 1);
        const NsStageMeta& M = meta[s];
        ItemGeo I;
        I.init(M.ord, M.cnt);
        const int n = I.n, NN = I.NN;
        StageLayout Lo;
        Lo.init(EXT, false, I.n1, I.n2, I.n3, I.cnt, P.fofs != nullptr);
        const double* st = sm + s * SW;
        // node phase
        for (int idx = threadIdx.x; idx < NN; idx += NS_BS) {
            const int slot = I.dn.div(idx), t = idx - slot * n;
            const int c = t - I.n12 * I.dn12.div(t);
            const double* Qs = st + Lo.q0 + slot * Lo.qs + M.qsh[slot];
            const double* Me = st + Lo.m0 + slot * Lo.ms;
            double qv[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) qv[v] = Qs[v * n + t];
            {  // admissibility (reading A25)
                const double pr = P.ph.gm1 * (qv[4] - 0.5 * (qv[1] * qv[1] + qv[2] * qv[2] + qv[3] * qv[3]) / qv[0]);
                if (!(qv[0] > 0.0 && pr > 0.0) && atomicAdd(P.flag, 1) == 0) P.flag[1] = M.e[slot];
            }
            ViscNode V;
            if (NSF) {
                double gv[15];
                load_grad(P.grad + 3 * M.off[slot] + t, n, gv);
                visc_node(qv, gv, P.ph, V);
            }
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                double ax, ay, az;
                if (EXT) {
                    ax = d < 2 ? Me[(2 * d) * I.n12 + c] : 0.0;
                    ay = d < 2 ? Me[(2 * d + 1) * I.n12 + c] : 0.0;
                    az = d < 2 ? 0.0 : Me[4 * I.n12 + c];
                } else {
                    ax = Me[(3 * d) * n + t];
                    ay = Me[(3 * d + 1) * n + t];
                    az = Me[(3 * d + 2) * n + t];
                }
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
        cons_sync();
        // line phase: every line of every direction, one variable per task, in place
        const int c1 = I.cnt * NV * I.nl0, c2 = c1 + I.cnt * NV * I.nl1, ntask = c2 + I.cnt * NV * I.nl2;
        for (int task = threadIdx.x; task < ntask; task += NS_BS) {
            const int d = task < c1 ? 0 : (task < c2 ? 1 : 2);
            const int r = task - (d == 0 ? 0 : (d == 1 ? c1 : c2));
            const int q5 = r / NV, v = r - NV * q5;
            const int slot = I.div_nl(d, q5);
            const int line = q5 - slot * I.nl(d);
            int base, stride, cb, cs;
            I.line(d, line, base, stride, cb, cs);
            double* Fl = F + d * NV * NN + slot * NV * n + v * n + base;
            const int nd = I.nd(d);
            if (P.fofs) {
                const double* Gs = st + Lo.f0 + slot * Lo.fs + v * I.nl(d) + line;
                const double gm = Gs[Lo.fb(2 * d)], gp = Gs[Lo.fb(2 * d + 1)];
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
        cons_sync();
        // epilogue
        for (int idx = threadIdx.x; idx < NN; idx += NS_BS) {
            const int slot = I.dn.div(idx), t = idx - slot * n;
            const int c = t - I.n12 * I.dn12.div(t);
            const long long o = M.off[slot];
            const double* Qs = st + Lo.q0 + slot * Lo.qs + M.qsh[slot];
            const double* Me = st + Lo.m0 + slot * Lo.ms;
            const double J = EXT ? Me[5 * I.n12 + c] : Me[9 * n + t];
            const double iJ = 1.0 / J;
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
                    qn[v] = Qs[v * n + t] + P.rkB * gn;
                    P.out[ix] = qn[v];
                }
                if (P.lam_max) {
                    const double ir = 1.0 / qn[0];
                    const double p = P.ph.gm1 * (qn[4] - 0.5 * ir * (qn[1] * qn[1] + qn[2] * qn[2] + qn[3] * qn[3]));
                    const double csnd = sqrt(P.ph.gamma * p * ir);
                    double lam = 0.0, nu = 0.0;
                    const double numax = P.ph.mu * ir * fmax(4.0 / 3.0, P.ph.gamma / P.ph.Pr);
#pragma unroll
                    for (int d = 0; d < 3; ++d) {
                        double a0, a1, a2;
                        if (EXT) {
                            a0 = (d < 2 ? Me[(2 * d) * I.n12 + c] : 0.0) * iJ;
                            a1 = (d < 2 ? Me[(2 * d + 1) * I.n12 + c] : 0.0) * iJ;
                            a2 = (d < 2 ? 0.0 : Me[4 * I.n12 + c]) * iJ;
                        } else {
                            a0 = Me[(3 * d) * n + t] * iJ;
                            a1 = Me[(3 * d + 1) * n + t] * iJ;
                            a2 = Me[(3 * d + 2) * n + t] * iJ;
                        }
                        const double an2 = a0 * a0 + a1 * a1 + a2 * a2;
                        const double ua = (qn[1] * a0 + qn[2] * a1 + qn[3] * a2) * ir;
                        const double np = I.nd(d);
                        lam += (fabs(ua) + csnd * sqrt(an2)) * np * np * 0.5;
                        nu += numax * an2 * np * np * np * np * 0.25;
                    }
                    lmax = fmax(lmax, lam);
                    vmax = fmax(vmax, nu);
                }
            }
        }
        mbar_arrive(&empty[s]);  // stage s read for the last time above
        cons_sync();             // F free for the next item
    }
    if (P.lam_max) {
        // block max over the consumer threads (named barrier; the producer warp has left)
        double v1 = warp_max(lmax), v2 = warp_max(vmax);
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
        if (lane == 0) {
            red[wid] = v1;
            red[16 + wid] = v2;
        }
        cons_sync();
        if (threadIdx.x == 0) {
            double a1 = 0.0, a2 = 0.0;
            for (int w = 0; w < NS_BS / 32; ++w) {
                a1 = fmax(a1, red[w]);
                a2 = fmax(a2, red[16 + w]);
            }
            atomicMax(P.lam_max, (unsigned long long)__double_as_longlong(a1));
            if (NSF) atomicMax(P.lam_max + 1, (unsigned long long)__double_as_longlong(a2));
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

// groups per CTA (measured on cfg5: W = 1 4 groups; W = 2, 3 NS flux one
// group per CTA, 2.77 -> 2.56 and 1.25 -> 1.13 ms; qhat 2 groups)
__host__ __device__ constexpr int face_groups(int W, int MODE) { return W == 1 ? 4 : (MODE == MODE_FLUX_NS ? 1 : 2); }
// groups per CTA and buffer sizes: a buffer holds 20 component slots of CAP
// points (NS flux passes: q and the gradient), 15 in the qhat pass (5 nk
// outputs), 5 in the Euler flux pass
template <int W, int MODE = MODE_FLUX_NS>
struct FaceCfg {
    static constexpr int G = face_groups(W, MODE);  // groups per CTA
    static constexpr int BS = G * 32 * W;
    static constexpr int CAP = 32 * W;
    static constexpr int BUF = (MODE == MODE_QHAT ? 15 : (MODE == MODE_FLUX_EULER ? NV : 20)) * CAP;
    static constexpr size_t smem = sizeof(double) * (size_t)G * 2 * BUF;
};

struct FSide {
    long long off;  // state offset (-1: ghost)
    int n, sa, sb, base, sta, stb;
};

// (selects on the runtime direction d instead of small arrays indexed by it:
// no local memory in the persistent face loops; measured faster in every pass,
// cfg5 qhat W = 1 1.57 -> 1.45 ms)
__device__ __forceinline__ FSide face_side(long long off, int ord, int d, bool isL)
{
    const int N0 = ord & 15, N1 = (ord >> 4) & 15, N2 = (ord >> 8) & 15;  // mt_unpack's packing
    const int st1 = N0 + 1, st2 = (N0 + 1) * (N1 + 1);
    FSide s;
    s.off = off;
    s.n = st2 * (N2 + 1);
    s.sa = (d == 0 ? N1 : N0) + 1;  // ta = 1 for d = 0, else 0
    s.sb = (d == 2 ? N1 : N2) + 1;  // tb = 1 for d = 2, else 2
    s.base = isL ? (d == 0 ? N0 : (d == 1 ? N1 * st1 : N2 * st2)) : 0;
    s.sta = d == 0 ? st1 : 1;
    s.stb = d == 2 ? st1 : st2;
    return s;
}

// Interpolation passes of the 20-component (q + gradient) NS flux traces:
// runtime-length loops with the components unrolled inside, instead of 9-long
// predicated loops per component (same fma order: bit-identical).  Measured on
// cfg5: flux faces W = 1/2/3 3.73 / 2.42 / 1.07 -> 3.36 / 2.01 / 0.95 ms, RK
// step 105.3 -> 100.0 ms for 2 steps; the 5-component qhat passes keep the
// predicated loops (no gain), and the same rewrite of the projection back to
// the sides was slower (2 steps 106.9 ms) -- dropped.
#ifndef NS_INTERP_RT
#define NS_INTERP_RT 1
#endif
__host__ __device__ constexpr bool interp_rt(int ncm) { return NS_INTERP_RT && ncm > NV; }

// acc[c] = sum_{k < len} tr[k] src[c CAP + k ss] for the NCM components
template <int W, int NCM>
__device__ __forceinline__ void interp_row(const double* __restrict__ tr, int len, const double* src, int ss, double* acc)
{
    constexpr int CAP = 32 * W;
#pragma unroll
    for (int c = 0; c < NCM; ++c) acc[c] = 0.0;
#pragma unroll 1
    for (int k = 0; k < len; ++k) {
        const double t = __ldg(tr + k);
#pragma unroll
        for (int c = 0; c < NCM; ++c) acc[c] = fma(t, src[c * CAP + k * ss], acc[c]);
    }
}

// Interpolate nc components of a side trace to the mortar grid.  Component c
// is read from (c < 5 ? q : g) + (c mod 5 ...) : qsrc[c n + node] for c < 5,
// gsrc[(c - 5) n + node] for c >= 5.  Gather (one thread per trace point),
// pass A along a into Y where s_a < m_a (one thread per (b, i)), then each
// point owner p < m_a m_b applies pass B along b into val[c].
template <int W, int NCM>
__device__ __forceinline__ void side_to_mortar(const double* __restrict__ qsrc, const double* __restrict__ gsrc,
                                               const FSide& s, int nc, int ma, int mb, const Tables* tab, double* X,
                                               double* Y, int l, int gid, int p, double* val)
{
    constexpr int CAP = 32 * W;
    const int sa = s.sa, sb = s.sb, ns = sa * sb;
    if (l < ns) {
        const int b = l / sa, a = l - b * sa;
        const long long node = s.base + a * s.sta + b * s.stb;
#pragma unroll
        for (int c = 0; c < NCM; ++c) {
            if (c >= nc) break;
            X[c * CAP + l] = c < NV ? __ldg(qsrc + (long long)c * s.n + node) : __ldg(gsrc + (long long)(c - NV) * s.n + node);
        }
    }
    grp_sync<W>(gid);
    const double* Z = X;
    if (sa < ma) {
        if (l < sb * ma) {
            const double* Ta = tab->T[sa - 1][ma - 1] + 0;  // [i * sa + a]
            const int b = l / ma, i = l - b * ma;
            if constexpr (interp_rt(NCM)) {
                double acc[NCM];
                interp_row<W, NCM>(Ta + i * sa, sa, X + b * sa, 1, acc);
#pragma unroll
                for (int c = 0; c < NCM; ++c) Y[c * CAP + l] = acc[c];
            } else {
            double t[NP];
#pragma unroll
            for (int a = 0; a < NP; ++a) t[a] = a < sa ? __ldg(Ta + i * sa + a) : 0.0;
#pragma unroll
            for (int c = 0; c < NCM; ++c) {
                if (c >= nc) break;
                const double* x = X + c * CAP + b * sa;
                double acc = 0.0;
#pragma unroll
                for (int a = 0; a < NP; ++a)
                    if (a < sa) acc = fma(t[a], x[a], acc);
                Y[c * CAP + l] = acc;  // [c][b][i]
            }
            }
        }
        grp_sync<W>(gid);
        Z = Y;
    }
    if (p < ma * mb) {
        const int j = p / ma, i = p - j * ma;
        if (sb < mb) {
            const double* Tb = tab->T[sb - 1][mb - 1];
            if constexpr (interp_rt(NCM)) {
                interp_row<W, NCM>(Tb + j * sb, sb, Z + i, ma, val);
            } else {
            double t[NP];
#pragma unroll
            for (int b = 0; b < NP; ++b) t[b] = b < sb ? __ldg(Tb + j * sb + b) : 0.0;
#pragma unroll
            for (int c = 0; c < NCM; ++c) {
                if (c >= nc) break;
                double acc = 0.0;
#pragma unroll
                for (int b = 0; b < NP; ++b)
                    if (b < sb) acc = fma(t[b], Z[c * CAP + b * ma + i], acc);
                val[c] = acc;
            }
            }
        } else {
#pragma unroll
            for (int c = 0; c < NCM; ++c) {
                if (c >= nc) break;
                val[c] = Z[c * CAP + p];
            }
        }
    }
    grp_sync<W>(gid);  // X / Y free for the next call
}

// measured on cfg5: the one-latency gather pays for the W = 1 flux pass
// (d = 0, 1 faces of the O-grid, 5.19 -> 4.37 ms), not for the qhat pass or
// the W = 2, 3 classes (extra registers / code: slower)
#ifndef NS_FACE_DIRECT
#define NS_FACE_DIRECT 1
#endif
#ifndef NS_FACE_DIRECT_MAXW
#define NS_FACE_DIRECT_MAXW 1
#endif
#ifndef NS_QHAT_DIRECT
#define NS_QHAT_DIRECT 0
#endif

// A side needs at most one interpolation pass (s_a = m_a or s_b = m_b): the
// pass-A thread (b, i) of side_to_mortar is then the owner of mortar point
// p = i + m_a b, so the pass runs straight from the gathered trace into val
// (no Y round trip, no barrier), and both sides' traces can be gathered at
// once (X: L, Y: R) -- one memory latency per face instead of two.
__device__ __forceinline__ bool one_pass(const FSide& s, int ma, int mb) { return s.sa == ma || s.sb == mb; }

template <int W, int NCM>
__device__ __forceinline__ void side_gather(const double* __restrict__ qsrc, const double* __restrict__ gsrc,
                                            const FSide& s, double* X, int l)
{
    constexpr int CAP = 32 * W;
    const int sa = s.sa, ns = sa * s.sb;
    if (l < ns) {
        const int b = l / sa, a = l - b * sa;
        const long long node = s.base + a * s.sta + b * s.stb;
#pragma unroll
        for (int c = 0; c < NCM; ++c)
            X[c * CAP + l] = c < NV ? __ldg(qsrc + (long long)c * s.n + node) : __ldg(gsrc + (long long)(c - NV) * s.n + node);
    }
}

// val at mortar point p (< m_a m_b) from the gathered trace X of a one-pass
// side: the same fma sequence as side_to_mortar's single pass
template <int W, int NCM>
__device__ __forceinline__ void side_direct(const double* X, const FSide& s, int ma, int mb, const Tables* tab, int p,
                                            double* val)
{
    constexpr int CAP = 32 * W;
    const int sa = s.sa, sb = s.sb;
    const int j = p / ma, i = p - j * ma;
    if (sa < ma) {  // sb == mb: row j of the trace along a
        const double* Ta = tab->T[sa - 1][ma - 1];
        if constexpr (interp_rt(NCM)) {
            interp_row<W, NCM>(Ta + i * sa, sa, X + j * sa, 1, val);
        } else {
        double t[NP];
#pragma unroll
        for (int a = 0; a < NP; ++a) t[a] = a < sa ? __ldg(Ta + i * sa + a) : 0.0;
#pragma unroll
        for (int c = 0; c < NCM; ++c) {
            const double* x = X + c * CAP + j * sa;
            double acc = 0.0;
#pragma unroll
            for (int a = 0; a < NP; ++a)
                if (a < sa) acc = fma(t[a], x[a], acc);
            val[c] = acc;
        }
        }
    } else if (sb < mb) {  // sa == ma: column i along b
        const double* Tb = tab->T[sb - 1][mb - 1];
        if constexpr (interp_rt(NCM)) {
            interp_row<W, NCM>(Tb + j * sb, sb, X + i, ma, val);
        } else {
        double t[NP];
#pragma unroll
        for (int b = 0; b < NP; ++b) t[b] = b < sb ? __ldg(Tb + j * sb + b) : 0.0;
#pragma unroll
        for (int c = 0; c < NCM; ++c) {
            double acc = 0.0;
#pragma unroll
            for (int b = 0; b < NP; ++b)
                if (b < sb) acc = fma(t[b], X[c * CAP + b * ma + i], acc);
            val[c] = acc;
        }
        }
    } else {
#pragma unroll
        for (int c = 0; c < NCM; ++c) val[c] = X[c * CAP + p];
    }
}

// Project nc components held at the mortar points (Fm[c CAP + p]) onto a
// side's own face nodes, stored to out[c (sa sb) + a + sa b].
template <int W, bool DIR>
__device__ __forceinline__ void mortar_to_side(const double* Fm, int nc, int ma, int mb, int sa, int sb, const Tables* tab,
                                               double* Y, double* __restrict__ out, int l, int gid)
{
    constexpr int CAP = 32 * W;
    const double* Z = Fm;
    int zrow = ma;
    if (DIR && sa < ma && sb == mb) {  // one pass: thread (b, i) owns side node i + sa b
        if (l < mb * sa) {
            const double* Pa = tab->P[ma - 1][sa - 1];
            const int b = l / sa, i = l - b * sa;
            double t[NP];
#pragma unroll
            for (int k = 0; k < NP; ++k) t[k] = k < ma ? __ldg(Pa + i * ma + k) : 0.0;
            for (int c = 0; c < nc; ++c) {
                const double* f = Fm + c * CAP + b * ma;
                double acc = 0.0;
#pragma unroll
                for (int k = 0; k < NP; ++k)
                    if (k < ma) acc = fma(t[k], f[k], acc);
                out[(long long)c * (sa * sb) + l] = acc;
            }
        }
        return;  // Fm is only read; Y untouched
    }
    if (sa < ma) {
        if (l < mb * sa) {
            const double* Pa = tab->P[ma - 1][sa - 1];  // [i * ma + k]
            const int b = l / sa, i = l - b * sa;
            double t[NP];
#pragma unroll
            for (int k = 0; k < NP; ++k) t[k] = k < ma ? __ldg(Pa + i * ma + k) : 0.0;
            for (int c = 0; c < nc; ++c) {
                const double* f = Fm + c * CAP + b * ma;
                double acc = 0.0;
#pragma unroll
                for (int k = 0; k < NP; ++k)
                    if (k < ma) acc = fma(t[k], f[k], acc);
                Y[c * CAP + l] = acc;  // [c][b][i], row length sa
            }
        }
        grp_sync<W>(gid);
        Z = Y;
        zrow = sa;
    }
    const int ns = sa * sb;
    if (l < ns) {
        const int j = l / sa, i = l - j * sa;
        if (sb < mb) {
            const double* Pb = tab->P[mb - 1][sb - 1];  // [j * mb + b]
            double t[NP];
#pragma unroll
            for (int b = 0; b < NP; ++b) t[b] = b < mb ? __ldg(Pb + j * mb + b) : 0.0;
            for (int c = 0; c < nc; ++c) {
                double acc = 0.0;
#pragma unroll
                for (int b = 0; b < NP; ++b)
                    if (b < mb) acc = fma(t[b], Z[c * CAP + b * zrow + i], acc);
                out[(long long)c * ns + l] = acc;
            }
        } else {
            for (int c = 0; c < nc; ++c) out[(long long)c * ns + l] = Z[c * CAP + l];
        }
    }
    grp_sync<W>(gid);
}

// resident CTAs per SM the register budget targets: the BR1 qhat pass fits in
// 80 registers without spills (more faces in flight), the NS flux needs 128
// (W = 1 with the one-latency gather: 168 at 3 CTAs, cfg5 3.90 -> 3.80 ms;
// W = 2 at 4 CTAs = 128 registers once NS_INTERP_RT: 2.00 -> 1.97 ms)
#ifndef NS_FLUX_MINB1
#define NS_FLUX_MINB1 3
#endif
#ifndef NS_FLUX_MINB2
#define NS_FLUX_MINB2 4
#endif
#ifndef NS_FLUX_MINB3
#define NS_FLUX_MINB3 2
#endif
#ifndef NS_QHAT_MINB1
#define NS_QHAT_MINB1 6
#endif
#ifndef NS_QHAT_MINB2
#define NS_QHAT_MINB2 4
#endif
#ifndef NS_EULER_MINB1
#define NS_EULER_MINB1 4
#endif
#ifndef NS_EULER_MINB3
#define NS_EULER_MINB3 2
#endif
#ifndef NS_EULER_MINB2
#define NS_EULER_MINB2 4
#endif
// (the budgets are per 4 groups for W = 1 and 2 groups for W = 2, 3: the same
// threads per SM whatever the groups per CTA)
__host__ __device__ constexpr int face_minb_base(int W, int MODE)
{
    return MODE == MODE_QHAT ? (W == 1 ? NS_QHAT_MINB1 : NS_QHAT_MINB2)
         : MODE == MODE_FLUX_EULER ? (W == 1 ? NS_EULER_MINB1 : (W == 2 ? NS_EULER_MINB2 : NS_EULER_MINB3))
                                   : (W == 3 ? NS_FLUX_MINB3 : (W == 1 ? NS_FLUX_MINB1 : NS_FLUX_MINB2));
}
__host__ __device__ constexpr int face_minb(int W, int MODE)
{
    return face_minb_base(W, MODE) * (W == 1 ? 4 : 2) / face_groups(W, MODE);
}

// one face of a group (X, Y: the group's buffers; every branch below is
// uniform over the group, so the group barriers inside are safe)
template <int W, int MODE>
__device__ __forceinline__ void ns_face_one(const NsFaceParams& P, const NsFace& F, double* X, double* Y, int l, int gid)
{
    constexpr int CAP = FaceCfg<W, MODE>::CAP;
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
    const int kind = F.kind;
    double qL[NV] = {0, 0, 0, 0, 0}, qR[NV] = {0, 0, 0, 0, 0};
    int nout;
    constexpr bool DIRECT_OK = NS_FACE_DIRECT && (MODE != MODE_QHAT || NS_QHAT_DIRECT) && W <= NS_FACE_DIRECT_MAXW;
    const bool direct = DIRECT_OK && (!hasL || one_pass(SL, ma, mb)) && (!hasR || one_pass(SR, ma, mb));
    if (MODE == MODE_QHAT) {
        if (direct) {
            if (hasL) side_gather<W, NV>(P.q + SL.off, nullptr, SL, X, l);
            if (hasR) side_gather<W, NV>(P.q + SR.off, nullptr, SR, Y, l);
            grp_sync<W>(gid);
            if (pon && hasL) side_direct<W, NV>(X, SL, ma, mb, P.tab, p, qL);
            if (pon && hasR) side_direct<W, NV>(Y, SR, ma, mb, P.tab, p, qR);
            grp_sync<W>(gid);  // X is overwritten below
        } else {
            if (hasL) side_to_mortar<W, NV>(P.q + SL.off, nullptr, SL, NV, ma, mb, P.tab, X, Y, l, gid, p, qL);
            if (hasR) side_to_mortar<W, NV>(P.q + SR.off, nullptr, SR, NV, ma, mb, P.tab, X, Y, l, gid, p, qR);
        }
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
        // each side: q and (NS) its gradient interpolated in one pass; the
        // viscous flux along Ja_f formed at once (one side's gradient live)
        double fsum[NV] = {0, 0, 0, 0, 0};
        constexpr int NCI = MODE == MODE_FLUX_NS ? 20 : NV;
        if (direct) {
            if (hasL) side_gather<W, NCI>(P.q + SL.off, MODE == MODE_FLUX_NS ? P.grad + 3 * SL.off : nullptr, SL, X, l);
            if (hasR) side_gather<W, NCI>(P.q + SR.off, MODE == MODE_FLUX_NS ? P.grad + 3 * SR.off : nullptr, SR, Y, l);
            grp_sync<W>(gid);
        }
#pragma unroll 1  // measured: the unrolled two-side loop slows the W = 1 NS flux pass (3.74 -> 4.30 ms)
        for (int side = 0; side < 2; ++side) {
            const bool has = side ? hasR : hasL;
            if (!has) continue;
            const FSide& S = side ? SR : SL;
            double val[NCI];
            if (direct) {
                if (pon) side_direct<W, NCI>(side ? Y : X, S, ma, mb, P.tab, p, val);
            } else {
                side_to_mortar<W, NCI>(P.q + S.off, MODE == MODE_FLUX_NS ? P.grad + 3 * S.off : nullptr, S, NCI, ma, mb,
                                       P.tab, X, Y, l, gid, p, val);
            }
            if (pon) {
                double* qs = side ? qR : qL;
#pragma unroll
                for (int v = 0; v < NV; ++v) qs[v] = val[v];
                if (MODE == MODE_FLUX_NS) {
                    double fs[NV];
                    visc_dot(qs, val + NV, jf[0], jf[1], jf[2], P.ph, fs);
#pragma unroll
                    for (int v = 0; v < NV; ++v) fsum[v] += fs[v];
                }
            }
        }
        if (direct) grp_sync<W>(gid);  // every lane's reads of X / Y done: X takes G below
        if (pon) {
            double G[NV];
            const double S = sqrt(jf[0] * jf[0] + jf[1] * jf[1] + jf[2] * jf[2]);
#if DG_FAST_DIV
            const double iS = inv_pos(S);
            const double nrm[3] = {jf[0] * iS, jf[1] * iS, jf[2] * iS};
#else
            const double nrm[3] = {jf[0] / S, jf[1] / S, jf[2] / S};
#endif
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
            if (MODE == MODE_FLUX_NS) {
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
#pragma unroll
            for (int v = 0; v < NV; ++v) X[v * CAP + p] = G[v];
        }
    }
    grp_sync<W>(gid);
    // ---- back to the sides' own face nodes ----
    const long long oL = MODE == MODE_QHAT ? F.hL : F.outL, oR = MODE == MODE_QHAT ? F.hR : F.outR;
    if (kind == 0) {  // conforming: the mortar is the face, one shared block
        if (pon) {
            double* out = P.out + oL;
            for (int c = 0; c < nout; ++c) out[(long long)c * nm + p] = X[c * CAP + p];
        }
        return;
    }
    if (hasL) mortar_to_side<W, DIRECT_OK>(X, nout, ma, mb, SL.sa, SL.sb, P.tab, Y, P.out + oL, l, gid);
    if (hasR) mortar_to_side<W, DIRECT_OK>(X, nout, ma, mb, SR.sa, SR.sb, P.tab, Y, P.out + oR, l, gid);
}

// measured on cfg5: pays for the qhat passes (1.68 -> 1.57 ms, W = 1) and
// the W = 2, 3 NS flux passes (2.56 -> 2.42, 1.13 -> 1.07 ms); the W = 1 NS
// flux pass took it once its interpolation loops had the runtime length
// (NS_INTERP_RT; 3.35 -> 3.20 ms, before: 3.73 -> 4.06 ms); the Euler flux
// passes take it too
#ifndef NS_FACE_PERSIST
#define NS_FACE_PERSIST 1
#endif
#ifndef NS_FACE_PERSIST_NS
#define NS_FACE_PERSIST_NS 1
#endif
__host__ __device__ constexpr bool face_persist(int W, int MODE)
{
    return NS_FACE_PERSIST && (MODE != MODE_FLUX_NS || W >= 2 || NS_FACE_PERSIST_NS);
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src)
{
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src));
}

// Persistent groups (grid = resident CTAs): each group walks faces fi, fi +
// G gridDim.x, ...; the next face's 80-byte record is fetched by cp.async into
// a double-buffered shared slot while the current face is processed (the
// record load heads every face's dependency chain: orders -> offsets ->
// trace gathers).
template <int W, int MODE>
__global__ void __launch_bounds__(FaceCfg<W, MODE>::BS, face_minb(W, MODE)) k_ns_face(NsFaceParams P)
{
    using C = FaceCfg<W, MODE>;
    extern __shared__ __align__(16) double fsm[];
    const int gid = threadIdx.x / (32 * W), l = threadIdx.x - gid * 32 * W;
    int fi = P.fbase + blockIdx.x * C::G + gid;
    if (fi >= P.fend) return;  // the whole group leaves (named barriers are per group)
    double* X = fsm + gid * 2 * C::BUF;
    double* Y = X + C::BUF;
    if constexpr (face_persist(W, MODE)) {
    static_assert(sizeof(NsFace) == 80, "NsFace record: 5 x 16 bytes");
    __shared__ __align__(16) NsFace fq[C::G][2];
    const int gstride = gridDim.x * C::G;
    if (l < 5) cp_async16(reinterpret_cast<char*>(&fq[gid][0]) + 16 * l, reinterpret_cast<const char*>(P.faces + fi) + 16 * l);
    asm volatile("cp.async.commit_group;\n" ::);
    for (int it = 0; fi < P.fend; fi += gstride, ++it) {
        const int nf = fi + gstride;
        if (nf < P.fend && l < 5)
            cp_async16(reinterpret_cast<char*>(&fq[gid][(it + 1) & 1]) + 16 * l,
                       reinterpret_cast<const char*>(P.faces + nf) + 16 * l);
        asm volatile("cp.async.commit_group;\n" ::);
        asm volatile("cp.async.wait_group 1;\n" ::: "memory");  // this face's record landed
        grp_sync<W>(gid);
        const NsFace F = fq[gid][it & 1];
        ns_face_one<W, MODE>(P, F, X, Y, l, gid);
        grp_sync<W>(gid);  // X, Y and the record slot free for the next face
    }
    } else {
        const NsFace F = P.faces[fi];
        ns_face_one<W, MODE>(P, F, X, Y, l, gid);
    }
}

// ---------------------------------------------------------------------------
// tau-estimation on EXTRUDED curved meshes (cfg4 / cfg5 O-grids), one CTA per
// level (e, d, p) as k_tau_curved, with the coarse metrics in the compact
// form of k_metrics_ext: 6 per (i, j) column of the coarse element (Ja^1 =
// (a, b, 0), Ja^2 = (c, e, 0), Ja^3 = (0, 0, f), J), from the geometry
// polynomial at the coarse nodes differentiated by D^O, in fp64 on
// coordinates relative to the element's first geometry node (reading R6),
// the zero components skipped in the BR1 gradient and the contravariant
// fluxes (terms fma(D, 0 q, g) = g exactly).  Measured on cfg5: 56 ms per
// estimate (generic 3-D kernel 66 ms, the same in double-double 82 ms);
// parity on full cfg4 (SAME reference) 3.8e-11 (generic plain fp64 4.9e-10).
// ---------------------------------------------------------------------------
__device__ __forceinline__ double ext_ja(const double* Mc, int nc, int col, int d, int k)
{
    if (d == 2) return k == 2 ? Mc[4 * nc + col] : 0.0;
    if (k == 2) return 0.0;
    return Mc[(2 * d + k) * nc + col];
}

#ifndef TAU_EXT_MINB64
#define TAU_EXT_MINB64 14
#endif
#ifndef TAU_EXT_MINB128
#define TAU_EXT_MINB128 7
#endif
#ifndef TAU_EXT_MINB256
#define TAU_EXT_MINB256 3
#endif
template <int BS>
__global__ void __launch_bounds__(BS, BS == 256 ? TAU_EXT_MINB256 : (BS == 128 ? TAU_EXT_MINB128 : TAU_EXT_MINB64)) k_tau_ext(CTauParams P)
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
    const int nO = o1 * o2 * o3, nc = o1 * o2;
    const bool ns = P.ph.physics == 1;
    __shared__ double Ds[3][NP * NP];
    stage_D(Ds, P.tab, o1, o2, o3);
    double* Mc = sm;                  // 6 nc compact metrics
    double* Qc = Mc + 6 * nc;         // 5 nO
    double* Rc = Qc + NV * nO;        // 5 nO
    double* GA = Rc + NV * nO;        // 15 nO (NS): gradient, then the three directions' fluxes
    double* F = GA;                   // Euler: one direction's flux, 5 nO (no gradient)
    double* A = ns ? GA + 15 * nO : F + NV * nO;  // 5 nO divergence
    double* Xs = GA;                  // 4 nc dd scratch of the coordinates (before GA / F are used)
    int* IJK = reinterpret_cast<int*>(A + NV * nO);
    for (int t = threadIdx.x; t < nO; t += BS) {
        int ii, jj, kk;
        node_ijk(t, o1, o2, ii, jj, kk);
        IJK[t] = ii | (jj << 8) | (kk << 16);
    }
    // fp64 on coordinates relative to the element's first geometry node: D
    // annihilates the shift (T reproduces constants, D 1 = 0), and the sums
    // run on O(h) instead of O(|x|) values -- the cancellation of the absolute
    // coordinates (|x| ~ 20 on elements of size 0.02) is what costs the plain
    // fp64 metrics their digits (reading R6)
    {
        const int g1 = P.cm.g1, g2 = P.cm.g2, ga = g1 + 1, gb = g2 + 1;
        const double* G = P.cm.geo + (long long)e * 3 * P.cm.ng;
        const double* T1 = P.tab->T[g1][o1 - 1];
        const double* T2 = P.tab->T[g2][o2 - 1];
        const double x0 = __ldg(G), y0 = __ldg(G + P.cm.ng);
        for (int t = threadIdx.x; t < nc; t += BS) {
            const int i = t % o1, j = t / o1;
            double x = 0.0, y = 0.0;
            for (int b = 0; b <= g2; ++b) {
                const double w2 = T2[j * gb + b];
                for (int a = 0; a <= g1; ++a) {
                    const double w = w2 * T1[i * ga + a];
                    x = fma(w, __ldg(G + a + ga * b) - x0, x);
                    y = fma(w, __ldg(G + P.cm.ng + a + ga * b) - y0, y);
                }
            }
            Xs[t] = x;
            Xs[nc + t] = y;
        }
        __syncthreads();
        const double zz = 0.5 * (__ldg(G + 2 * P.cm.ng + ga * gb) - __ldg(G + 2 * P.cm.ng));
        for (int t = threadIdx.x; t < nc; t += BS) {
            const int i = t % o1, j = t / o1;
            double xx = 0.0, yx = 0.0, xe = 0.0, ye = 0.0;
            for (int m = 0; m < o1; ++m) {
                const double dm = Ds[0][i * o1 + m];
                xx = fma(dm, Xs[m + o1 * j], xx);
                yx = fma(dm, Xs[nc + m + o1 * j], yx);
            }
            for (int m = 0; m < o2; ++m) {
                const double dm = Ds[1][j * o2 + m];
                xe = fma(dm, Xs[i + o1 * m], xe);
                ye = fma(dm, Xs[nc + i + o1 * m], ye);
            }
            const double j3 = xx * ye - xe * yx;
            Mc[t] = zz * ye;
            Mc[nc + t] = -(zz * xe);
            Mc[2 * nc + t] = -(zz * yx);
            Mc[3 * nc + t] = zz * xx;
            Mc[4 * nc + t] = j3;
            Mc[5 * nc + t] = zz * j3;
        }
    }
    __syncthreads();  // Xs (= GA / F) free, Mc ready
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
        for (int v = 0; v < NV; ++v) A[v * nO + t] = 0.0;
    }
    __syncthreads();
    if (ns) {  // isolated gradient J g_k = sum_d' D^{d'} (Ja^{d'}_k q), nonzero metric components only
        for (int t = threadIdx.x; t < nO; t += BS) {
            const int pk = IJK[t];
            const int i = pk & 255, j = (pk >> 8) & 255, k = pk >> 16;
            double g[15];
#pragma unroll
            for (int cc = 0; cc < 15; ++cc) g[cc] = 0.0;
            {  // xi: Ja^1 = (a, b, 0)
                const int base = t - i;
                const double* Dr = Ds[0] + i * o1;
                for (int m = 0; m < o1; ++m) {
                    const double dm = Dr[m];
                    const int col = m + o1 * j;
                    const double ja = Mc[col], jb = Mc[nc + col];
#pragma unroll
                    for (int v = 0; v < NV; ++v) {
                        const double qv = Qc[v * nO + base + m];
                        g[v] = fma(dm, ja * qv, g[v]);
                        g[NV + v] = fma(dm, jb * qv, g[NV + v]);
                    }
                }
            }
            {  // eta: Ja^2 = (c, e, 0)
                const int base = t - j * o1;
                const double* Dr = Ds[1] + j * o2;
                for (int m = 0; m < o2; ++m) {
                    const double dm = Dr[m];
                    const int col = i + o1 * m;
                    const double jc = Mc[2 * nc + col], je = Mc[3 * nc + col];
#pragma unroll
                    for (int v = 0; v < NV; ++v) {
                        const double qv = Qc[v * nO + base + m * o1];
                        g[v] = fma(dm, jc * qv, g[v]);
                        g[NV + v] = fma(dm, je * qv, g[NV + v]);
                    }
                }
            }
            {  // zeta: Ja^3 = (0, 0, f), f constant along the column
                const int base = t - k * nc;
                const double* Dr = Ds[2] + k * o3;
                const double jf = Mc[4 * nc + i + o1 * j];
                for (int m = 0; m < o3; ++m) {
                    const double dm = Dr[m];
#pragma unroll
                    for (int v = 0; v < NV; ++v) g[2 * NV + v] = fma(dm, jf * Qc[v * nO + base + m * nc], g[2 * NV + v]);
                }
            }
            const double iJ = 1.0 / Mc[5 * nc + i + o1 * j];
#pragma unroll
            for (int cc = 0; cc < 15; ++cc) GA[cc * nO + t] = g[cc] * iJ;
        }
        __syncthreads();
        // fluxes of the three directions from one viscous evaluation per node, in place of GA
        for (int t = threadIdx.x; t < nO; t += BS) {
            const int pk = IJK[t];
            const int col = (pk & 255) + o1 * ((pk >> 8) & 255);
            double qv[NV], gv[15];
            for (int v = 0; v < NV; ++v) qv[v] = Qc[v * nO + t];
            for (int cc = 0; cc < 15; ++cc) gv[cc] = GA[cc * nO + t];
            ViscNode V;
            visc_node(qv, gv, P.ph, V);
            for (int dd = 0; dd < 3; ++dd) {
                const double ax = ext_ja(Mc, nc, col, dd, 0), ay = ext_ja(Mc, nc, col, dd, 1), az = ext_ja(Mc, nc, col, dd, 2);
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
                const int str = dd == 0 ? 1 : (dd == 1 ? o1 : nc);
                const int a = ijk[dd];
                dsum_comps<NV>(od, Ds[dd] + a * od, GA + dd * NV * nO + (t - a * str), nO, str,
                               [&](int v, double sv) { A[v * nO + t] += sv; });
            }
        }
        __syncthreads();
    } else {
        for (int dd = 0; dd < 3; ++dd) {
            const int od = dd == 0 ? o1 : (dd == 1 ? o2 : o3);
            const int str = dd == 0 ? 1 : (dd == 1 ? o1 : nc);
            for (int t = threadIdx.x; t < nO; t += BS) {
                const int pk = IJK[t];
                const int col = (pk & 255) + o1 * ((pk >> 8) & 255);
                double qv[NV], Fv[NV];
                for (int v = 0; v < NV; ++v) qv[v] = Qc[v * nO + t];
                adv_dot(qv, ext_ja(Mc, nc, col, dd, 0), ext_ja(Mc, nc, col, dd, 1), ext_ja(Mc, nc, col, dd, 2), P.ph.gm1, Fv);
                for (int v = 0; v < NV; ++v) F[v * nO + t] = Fv[v];
            }
            __syncthreads();
            for (int t = threadIdx.x; t < nO; t += BS) {
                const int pk = IJK[t];
                const int a = dd == 0 ? (pk & 255) : (dd == 1 ? ((pk >> 8) & 255) : (pk >> 16));
                dsum_comps<NV>(od, Ds[dd] + a * od, F + (t - a * str), nO, str, [&](int v, double sv) { A[v * nO + t] += sv; });
            }
            __syncthreads();
        }
    }
    double tmax = 0.0;
    for (int t = threadIdx.x; t < nO; t += BS) {
        const int pk = IJK[t];
        const int i = pk & 255, j = (pk >> 8) & 255, k = pk >> 16;
        const double J = Mc[5 * nc + i + o1 * j];
        double scale = 1.0;
        if (P.formulation == 1) scale = J * P.tab->w[o1 - 1][i] * P.tab->w[o2 - 1][j] * P.tab->w[o3 - 1][k];
        for (int v = 0; v < NV; ++v) tmax = fmax(tmax, fabs(scale * (Rc[v * nO + t] + A[v * nO + t] / J)));
    }
    tmax = block_max(tmax, red);
    if (threadIdx.x == 0) P.tau[(3 * (long long)e + d) * DG_TAU_STRIDE_DEV + p] = tmax;
}

// shared-memory doubles of a k_tau_ext level with nO coarse nodes (nc <= nO columns)
__host__ __device__ inline size_t tau_ext_words(int nO, bool ns) { return (size_t)(ns ? 36 : 26) * nO + (nO + 1) / 2; }

// ---------------------------------------------------------------------------
// k_tau_grp: the k_tau_ext levels of ONE element batched in a CTA (groups of
// consecutive (d, p) levels, d-major, whose coarse nodes sum to <= cap): each
// phase (coarse metrics, interpolation, BR1 gradient, fluxes, divergence,
// level maxima) runs over the nodes of all the group's levels between two
// barriers, instead of one CTA and ~7 barriers per level.  The same
// operations per node and level as k_tau_ext (agreement to a few ulp: the
// compiler's fma contraction differs between the kernels).  cfg5: 50.8 ms per
// estimate against 53.3 (the estimate is fp64-bound: ~20 % of the DFMA peak).
// Group record: TauLevel{e, d0, p0, count} (levels (d0, p0), (d0, p0 + 1), ...
// continuing with p = 1 of the next direction with N_d >= 2).
// ---------------------------------------------------------------------------
constexpr int TAU_GRP_BS = 256;
constexpr int TAU_GRP_MAXLV = 24;
struct TauLvDesc {
    int d, p, o1, o2, o3, nO, nc, nb, cb;  // nb / cb: node / column base in the group
};
// shared-memory bytes of a group kernel with node capacity cap
__host__ __device__ inline size_t tau_grp_bytes(int cap) { return sizeof(double) * 36 * (size_t)cap + 4 * (size_t)cap + 2 * (size_t)cap + 16; }

__global__ void __launch_bounds__(TAU_GRP_BS, 3) k_tau_grp(CTauParams P, int cap)
{
    extern __shared__ __align__(16) double sm[];
    __shared__ TauLvDesc L[TAU_GRP_MAXLV];
    __shared__ unsigned long long lmax[TAU_GRP_MAXLV];
    __shared__ int nlev_s, nOt_s, nct_s;
    const TauLevel G = P.levels[P.lbase + blockIdx.x];
    const int e = G.e;
    const int n1 = P.orders[3 * e] + 1, n2 = P.orders[3 * e + 1] + 1, n3 = P.orders[3 * e + 2] + 1;
    const int n = n1 * n2 * n3;
    const bool ns = P.ph.physics == 1;
    double* Mc = sm;                 // 6 cap
    double* Qc = Mc + 6 * cap;       // 5 cap
    double* Rc = Qc + 5 * cap;       // 5 cap
    double* GA = Rc + 5 * cap;       // 15 cap (coordinates scratch first)
    double* A = GA + 15 * cap;       // 5 cap
    int* IJK = reinterpret_cast<int*>(A + 5 * cap);      // cap
    unsigned char* LV = reinterpret_cast<unsigned char*>(IJK + cap);  // cap: level of a node
    unsigned char* LC = LV + cap;                        // cap: level of a column
    if (threadIdx.x == 0) {
        const int nn[3] = {n1, n2, n3};
        int d = G.d, p = G.p, nb = 0, cb = 0;
        for (int l = 0; l < G.pad; ++l) {
            TauLvDesc D;
            D.d = d;
            D.p = p;
            D.o1 = d == 0 ? p + 1 : n1;
            D.o2 = d == 1 ? p + 1 : n2;
            D.o3 = d == 2 ? p + 1 : n3;
            D.nc = D.o1 * D.o2;
            D.nO = D.nc * D.o3;
            D.nb = nb;
            D.cb = cb;
            nb += D.nO;
            cb += D.nc;
            L[l] = D;
            lmax[l] = 0ull;
            if (++p >= nn[d] - 1) {  // levels p = 1 .. N_d - 1 (N_d = nn[d] - 1)
                p = 1;
                do { ++d; } while (d < 3 && nn[d] < 3);
            }
        }
        nlev_s = G.pad;
        nOt_s = nb;
        nct_s = cb;
    }
    __syncthreads();
    const int nlev = nlev_s, nOt = nOt_s, nct = nct_s;
    for (int g = threadIdx.x; g < nOt; g += TAU_GRP_BS) {
        int l = 0;
        while (l + 1 < nlev && g >= L[l + 1].nb) ++l;
        const int t = g - L[l].nb;
        int ii, jj, kk;
        node_ijk(t, L[l].o1, L[l].o2, ii, jj, kk);
        IJK[g] = ii | (jj << 8) | (kk << 16);
        LV[g] = (unsigned char)l;
    }
    for (int c = threadIdx.x; c < nct; c += TAU_GRP_BS) {
        int l = 0;
        while (l + 1 < nlev && c >= L[l + 1].cb) ++l;
        LC[c] = (unsigned char)l;
    }
    const int g1 = P.cm.g1, g2 = P.cm.g2, ga = g1 + 1, gb = g2 + 1;
    const double* Gg = P.cm.geo + (long long)e * 3 * P.cm.ng;
    const double x0 = __ldg(Gg), y0 = __ldg(Gg + P.cm.ng);
    __syncthreads();
    // coarse metrics, phase 1: x, y (relative to the first geometry node) at the columns
    for (int cg = threadIdx.x; cg < nct; cg += TAU_GRP_BS) {
        const TauLvDesc& D = L[LC[cg]];
        const int t = cg - D.cb, o1 = D.o1, o2 = D.o2, nc = D.nc;
        const int i = t % o1, j = t / o1;
        const double* T1 = P.tab->T[g1][o1 - 1];
        const double* T2 = P.tab->T[g2][o2 - 1];
        double x = 0.0, y = 0.0;
        for (int b = 0; b <= g2; ++b) {
            const double w2 = T2[j * gb + b];
            for (int a = 0; a <= g1; ++a) {
                const double w = w2 * T1[i * ga + a];
                x = fma(w, __ldg(Gg + a + ga * b) - x0, x);
                y = fma(w, __ldg(Gg + P.cm.ng + a + ga * b) - y0, y);
            }
        }
        double* Xs = GA + 15 * D.nb;
        Xs[t] = x;
        Xs[nc + t] = y;
    }
    __syncthreads();
    {
        const double zz = 0.5 * (__ldg(Gg + 2 * P.cm.ng + ga * gb) - __ldg(Gg + 2 * P.cm.ng));
        for (int cg = threadIdx.x; cg < nct; cg += TAU_GRP_BS) {
            const TauLvDesc& D = L[LC[cg]];
            const int t = cg - D.cb, o1 = D.o1, o2 = D.o2, nc = D.nc;
            const int i = t % o1, j = t / o1;
            const double* Xs = GA + 15 * D.nb;
            const double* D1 = P.tab->D[o1 - 1];
            const double* D2 = P.tab->D[o2 - 1];
            double xx = 0.0, yx = 0.0, xe = 0.0, ye = 0.0;
            for (int m = 0; m < o1; ++m) {
                const double dm = D1[i * o1 + m];
                xx = fma(dm, Xs[m + o1 * j], xx);
                yx = fma(dm, Xs[nc + m + o1 * j], yx);
            }
            for (int m = 0; m < o2; ++m) {
                const double dm = D2[j * o2 + m];
                xe = fma(dm, Xs[i + o1 * m], xe);
                ye = fma(dm, Xs[nc + i + o1 * m], ye);
            }
            const double j3 = xx * ye - xe * yx;
            double* M = Mc + 6 * D.cb;
            M[t] = zz * ye;
            M[nc + t] = -(zz * xe);
            M[2 * nc + t] = -(zz * yx);
            M[3 * nc + t] = zz * xx;
            M[4 * nc + t] = j3;
            M[5 * nc + t] = zz * j3;
        }
    }
    __syncthreads();  // Xs (= GA) free, metrics ready
    const long long o = P.off[e];
    for (int g = threadIdx.x; g < nOt; g += TAU_GRP_BS) {
        const TauLvDesc& D = L[LV[g]];
        const int t = g - D.nb, nO = D.nO, d = D.d;
        const int nd = d == 0 ? n1 : (d == 1 ? n2 : n3);
        const int stride = d == 0 ? 1 : (d == 1 ? n1 : n1 * n2);
        const double* T = P.restr ? P.tab->P[nd - 1][D.p] : P.tab->T[nd - 1][D.p];
        const int pk = IJK[g];
        int i = pk & 255, j = (pk >> 8) & 255, k = pk >> 16;
        const int ic = d == 0 ? i : (d == 1 ? j : k);
        if (d == 0) i = 0; else if (d == 1) j = 0; else k = 0;
        const int base = i + n1 * (j + n2 * k);
        const double* qe = P.q + o;
        const double* re = P.qref + o;
        double* Qd = Qc + 5 * D.nb;
        double* Rd = Rc + 5 * D.nb;
        switch (nd) {
            case 2: tau_interp_node<2>(T, ic, qe, re, n, base, stride, Qd, Rd, nO, t); break;
            case 3: tau_interp_node<3>(T, ic, qe, re, n, base, stride, Qd, Rd, nO, t); break;
            case 4: tau_interp_node<4>(T, ic, qe, re, n, base, stride, Qd, Rd, nO, t); break;
            case 5: tau_interp_node<5>(T, ic, qe, re, n, base, stride, Qd, Rd, nO, t); break;
            case 6: tau_interp_node<6>(T, ic, qe, re, n, base, stride, Qd, Rd, nO, t); break;
            case 7: tau_interp_node<7>(T, ic, qe, re, n, base, stride, Qd, Rd, nO, t); break;
            case 8: tau_interp_node<8>(T, ic, qe, re, n, base, stride, Qd, Rd, nO, t); break;
            default: tau_interp_node<9>(T, ic, qe, re, n, base, stride, Qd, Rd, nO, t); break;
        }
        double* Ad = A + 5 * D.nb;
        for (int v = 0; v < NV; ++v) Ad[v * nO + t] = 0.0;
    }
    __syncthreads();
    if (ns) {  // isolated gradient (nonzero metric components), as k_tau_ext
        for (int g = threadIdx.x; g < nOt; g += TAU_GRP_BS) {
            const TauLvDesc& D = L[LV[g]];
            const int t = g - D.nb, nO = D.nO, o1 = D.o1, o2 = D.o2, o3 = D.o3, nc = D.nc;
            const double* Q = Qc + 5 * D.nb;
            const double* M = Mc + 6 * D.cb;
            const int pk = IJK[g];
            const int i = pk & 255, j = (pk >> 8) & 255, k = pk >> 16;
            double gr[15];
#pragma unroll
            for (int cc = 0; cc < 15; ++cc) gr[cc] = 0.0;
            {
                const int base = t - i;
                const double* Dr = P.tab->D[o1 - 1] + i * o1;
                for (int m = 0; m < o1; ++m) {
                    const double dm = Dr[m];
                    const int col = m + o1 * j;
                    const double ja = M[col], jb = M[nc + col];
#pragma unroll
                    for (int v = 0; v < NV; ++v) {
                        const double qv = Q[v * nO + base + m];
                        gr[v] = fma(dm, ja * qv, gr[v]);
                        gr[NV + v] = fma(dm, jb * qv, gr[NV + v]);
                    }
                }
            }
            {
                const int base = t - j * o1;
                const double* Dr = P.tab->D[o2 - 1] + j * o2;
                for (int m = 0; m < o2; ++m) {
                    const double dm = Dr[m];
                    const int col = i + o1 * m;
                    const double jc = M[2 * nc + col], je = M[3 * nc + col];
#pragma unroll
                    for (int v = 0; v < NV; ++v) {
                        const double qv = Q[v * nO + base + m * o1];
                        gr[v] = fma(dm, jc * qv, gr[v]);
                        gr[NV + v] = fma(dm, je * qv, gr[NV + v]);
                    }
                }
            }
            {
                const int base = t - k * nc;
                const double* Dr = P.tab->D[o3 - 1] + k * o3;
                const double jf = M[4 * nc + i + o1 * j];
                for (int m = 0; m < o3; ++m) {
                    const double dm = Dr[m];
#pragma unroll
                    for (int v = 0; v < NV; ++v) gr[2 * NV + v] = fma(dm, jf * Q[v * nO + base + m * nc], gr[2 * NV + v]);
                }
            }
            const double iJ = 1.0 / M[5 * nc + i + o1 * j];
            double* GAd = GA + 15 * D.nb;
#pragma unroll
            for (int cc = 0; cc < 15; ++cc) GAd[cc * nO + t] = gr[cc] * iJ;
        }
        __syncthreads();
    }
    // contravariant fluxes of the three directions (NS: one viscous evaluation per node), in place of GA
    for (int g = threadIdx.x; g < nOt; g += TAU_GRP_BS) {
        const TauLvDesc& D = L[LV[g]];
        const int t = g - D.nb, nO = D.nO, nc = D.nc;
        const double* Q = Qc + 5 * D.nb;
        const double* M = Mc + 6 * D.cb;
        double* GAd = GA + 15 * D.nb;
        const int pk = IJK[g];
        const int col = (pk & 255) + D.o1 * ((pk >> 8) & 255);
        double qv[NV];
        for (int v = 0; v < NV; ++v) qv[v] = Q[v * nO + t];
        ViscNode V;
        if (ns) {
            double gv[15];
            for (int cc = 0; cc < 15; ++cc) gv[cc] = GAd[cc * nO + t];
            visc_node(qv, gv, P.ph, V);
        }
        for (int dd = 0; dd < 3; ++dd) {
            const double ax = ext_ja(M, nc, col, dd, 0), ay = ext_ja(M, nc, col, dd, 1), az = ext_ja(M, nc, col, dd, 2);
            double Fv[NV];
            adv_dot(qv, ax, ay, az, P.ph.gm1, Fv);
            if (ns) {
                double fv[NV];
                visc_along(V, ax, ay, az, fv);
                for (int v = 0; v < NV; ++v) Fv[v] -= fv[v];
            }
            for (int v = 0; v < NV; ++v) GAd[(dd * NV + v) * nO + t] = Fv[v];
        }
    }
    __syncthreads();
    for (int g = threadIdx.x; g < nOt; g += TAU_GRP_BS) {
        const TauLvDesc& D = L[LV[g]];
        const int t = g - D.nb, nO = D.nO;
        const double* GAd = GA + 15 * D.nb;
        double* Ad = A + 5 * D.nb;
        const int pk = IJK[g];
        const int ijk[3] = {pk & 255, (pk >> 8) & 255, pk >> 16};
        for (int dd = 0; dd < 3; ++dd) {
            const int od = dd == 0 ? D.o1 : (dd == 1 ? D.o2 : D.o3);
            const int str = dd == 0 ? 1 : (dd == 1 ? D.o1 : D.nc);
            const int a = ijk[dd];
            dsum_comps<NV>(od, P.tab->D[od - 1] + a * od, GAd + dd * NV * nO + (t - a * str), nO, str,
                           [&](int v, double sv) { Ad[v * nO + t] += sv; });
        }
    }
    __syncthreads();
    for (int g = threadIdx.x; g < nOt; g += TAU_GRP_BS) {
        const int l = LV[g];
        const TauLvDesc& D = L[l];
        const int t = g - D.nb, nO = D.nO;
        const int pk = IJK[g];
        const int i = pk & 255, j = (pk >> 8) & 255, k = pk >> 16;
        const double J = Mc[6 * D.cb + 5 * D.nc + i + D.o1 * j];
        double scale = 1.0;
        if (P.formulation == 1) scale = J * P.tab->w[D.o1 - 1][i] * P.tab->w[D.o2 - 1][j] * P.tab->w[D.o3 - 1][k];
        const double* Rd = Rc + 5 * D.nb;
        const double* Ad = A + 5 * D.nb;
        double tm = 0.0;
        for (int v = 0; v < NV; ++v) tm = fmax(tm, fabs(scale * (Rd[v * nO + t] + Ad[v * nO + t] / J)));
        atomicMax(&lmax[l], (unsigned long long)__double_as_longlong(tm));  // tm >= 0: bit order = value order
    }
    __syncthreads();
    if (threadIdx.x < nlev)
        P.tau[(3 * (long long)e + L[threadIdx.x].d) * DG_TAU_STRIDE_DEV + L[threadIdx.x].p] =
            __longlong_as_double((long long)lmax[threadIdx.x]);
}

}  // namespace dgtau
