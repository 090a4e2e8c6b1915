/*
 * dgsem_oracle.c -- CPU ORACLE for the tau-estimation / DGSEM hot path of
 * arXiv 2210.03523 (Rueda-Ramirez, Ntoukas, Rubio, Valero, Ferrer).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_2210_03523_b200/) never imports, links or calls it,
 * and this file shares no code, header, table or constant generator with it.
 *
 * Plain, slow, obviously-correct fp64 loops (basis construction in long
 * double).  Every function cites the PAPER.md passage ("P:<line>") or the
 * DESIGN.md reading ("A<k>", numbered as in SURVEY.md section 8(c).2) it
 * follows.  Parallelism: OpenMP "guided" over elements, mirroring the paper's
 * own parallel model; no blocking, fusion or reordering beyond the
 * definitions.
 *
 * Conventions: N = (N1,N2,N3) is an element's current
 * (fine) order, p < N_d a coarse order.  Node index i + (N1+1)(j + (N2+1)k),
 * xi fastest.  State of element e: 5 conserved variables [v][node], elements
 * packed back to back in element order (canonical layout [e][v][k][j][i]).
 * Faces: f = 2d + s, d in {0,1,2} = {xi,eta,zeta}, s = 0 for the -1 side,
 * 1 for the +1 side.  neighbour[e][f] >= 0: element across f (whose face
 * 2d+(1-s) touches it); -1: no-slip adiabatic wall; -2: far field.
 *
 * Parity unpinned: the extrapolation law (A13) and the advective CFL
 * constants (A11) are pinned only by consistency pins and hand values.
 * Pinned since round 2: the Roe flux on general subsonic states (Q25, |A~|
 * as a matrix square root), BR1 / the viscous terms / wall and far-field
 * states (Q19-Q22 exact NS solutions and closed forms), the assembly (Q24
 * dense Galerkin form); see DESIGN.md section 2.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "dgsem_oracle.h"

#define NV 5
#define NMAXB ORC_NMAX /* largest order with basis tables */

/* ------------------------------------------------------------------------- */
/* 1. Basis: Gauss-Lobatto nodes/weights, Lagrange polynomials, D, D-hat,
 *    interpolation T and mortar L2 projection P.
 *    P:67 ("stores the data at the Gauss or Gauss-Lobatto nodes")
 *    ("quadrature rule of N+1 points"), reading A2 (Gauss-Lobatto), A6.      */
/* ------------------------------------------------------------------------- */

static double gl_x[NMAXB + 1][NMAXB + 1];
static double gl_w[NMAXB + 1][NMAXB + 1];
static double Dm[NMAXB + 1][NMAXB + 1][NMAXB + 1];   /* D[N][a][b] = l_b'(x_a)   */
static double Dh[NMAXB + 1][NMAXB + 1][NMAXB + 1];   /* Dhat = -w_b D_ba / w_a    */
static double lpm[NMAXB + 1][2][NMAXB + 1];          /* l_a(-1), l_a(+1)          */
static double Tm[NMAXB + 1][NMAXB + 1][(NMAXB + 1) * (NMAXB + 1)]; /* [from][to] */
static double Pm[NMAXB + 1][NMAXB + 1][(NMAXB + 1) * (NMAXB + 1)]; /* [M][s]     */
/* long double copies used for the geometry (metric) computation, so that
 * the metric terms are exact to the last double bit for affine elements */
static long double Dl[NMAXB + 1][NMAXB + 1][NMAXB + 1];
static long double lpml[NMAXB + 1][2][NMAXB + 1];
static long double Tl[NMAXB + 1][NMAXB + 1][(NMAXB + 1) * (NMAXB + 1)];
static int basis_ready = 0;

/* Legendre polynomial P_n(x) by the three-term recurrence. */
static long double legendre(int n, long double x)
{
    long double p0 = 1.0L, p1 = x;
    if (n == 0) return p0;
    for (int k = 2; k <= n; ++k) {
        long double p2 = ((2 * k - 1) * x * p1 - (k - 1) * p0) / k;
        p0 = p1;
        p1 = p2;
    }
    return p1;
}

/* Gauss-Lobatto nodes: roots of (1-x^2) P_N'(x), i.e. of
 * q(x) = P_{N+1}(x) - P_{N-1}(x) (q' = (2N+1) P_N).  Newton from the
 * Chebyshev-Lobatto points; weights w = 2 / (N(N+1) P_N(x)^2). */
static void gl_nodes_ld(int N, long double* x, long double* w)
{
    const long double pi = 3.141592653589793238462643383279502884L;
    for (int j = 0; j <= N; ++j) {
        long double t = -cosl(pi * j / N);
        if (j > 0 && j < N) {
            for (int it = 0; it < 200; ++it) {
                long double q = legendre(N + 1, t) - legendre(N - 1, t);
                long double dq = (2 * N + 1) * legendre(N, t);
                long double dt = q / dq;
                t -= dt;
                if (fabsl(dt) < 1e-21L) break;
            }
        }
        x[j] = t;
    }
    x[0] = -1.0L;
    x[N] = 1.0L;
    for (int j = 0; j <= N; ++j) {
        long double pn = legendre(N, x[j]);
        w[j] = 2.0L / ((long double)N * (N + 1) * pn * pn);
    }
}

/* Lagrange polynomial l_a(t) on nodes x[0..N], product formula. */
static long double lagrange_ld(int N, const long double* x, int a, long double t)
{
    long double r = 1.0L;
    for (int b = 0; b <= N; ++b)
        if (b != a) r *= (t - x[b]) / (x[a] - x[b]);
    return r;
}

/* Derivative l_a'(t) = sum_{c != a} 1/(x_a - x_c) prod_{b != a,c} (t-x_b)/(x_a-x_b). */
static long double dlagrange_ld(int N, const long double* x, int a, long double t)
{
    long double s = 0.0L;
    for (int c = 0; c <= N; ++c) {
        if (c == a) continue;
        long double pr = 1.0L / (x[a] - x[c]);
        for (int b = 0; b <= N; ++b)
            if (b != a && b != c) pr *= (t - x[b]) / (x[a] - x[b]);
        s += pr;
    }
    return s;
}

/* Solve A X = B (n x n, m right-hand sides) by Gaussian elimination with
 * partial pivoting, long double.  A and B overwritten; X returned in B. */
static void solve_ld(int n, int m, long double* A, long double* B)
{
    for (int c = 0; c < n; ++c) {
        int piv = c;
        for (int r = c + 1; r < n; ++r)
            if (fabsl(A[r * n + c]) > fabsl(A[piv * n + c])) piv = r;
        if (piv != c) {
            for (int k = 0; k < n; ++k) { long double t = A[c * n + k]; A[c * n + k] = A[piv * n + k]; A[piv * n + k] = t; }
            for (int k = 0; k < m; ++k) { long double t = B[c * m + k]; B[c * m + k] = B[piv * m + k]; B[piv * m + k] = t; }
        }
        for (int r = c + 1; r < n; ++r) {
            long double f = A[r * n + c] / A[c * n + c];
            for (int k = c; k < n; ++k) A[r * n + k] -= f * A[c * n + k];
            for (int k = 0; k < m; ++k) B[r * m + k] -= f * B[c * m + k];
        }
    }
    for (int c = n - 1; c >= 0; --c) {
        for (int k = 0; k < m; ++k) {
            long double s = B[c * m + k];
            for (int j = c + 1; j < n; ++j) s -= A[c * n + j] * B[j * m + k];
            B[c * m + k] = s / A[c * n + c];
        }
    }
}

void orc_init_basis(void)
{
    if (basis_ready) return;
    static long double X[NMAXB + 1][NMAXB + 1], W[NMAXB + 1][NMAXB + 1];
    for (int N = 1; N <= NMAXB; ++N) {
        gl_nodes_ld(N, X[N], W[N]);
        for (int a = 0; a <= N; ++a) { gl_x[N][a] = (double)X[N][a]; gl_w[N][a] = (double)W[N][a]; }
        for (int a = 0; a <= N; ++a)
            for (int b = 0; b <= N; ++b) {
                Dl[N][a][b] = dlagrange_ld(N, X[N], b, X[N][a]);
                Dm[N][a][b] = (double)Dl[N][a][b];
            }
        for (int a = 0; a <= N; ++a)
            for (int b = 0; b <= N; ++b)
                Dh[N][a][b] = (double)(-W[N][b] * (long double)dlagrange_ld(N, X[N], a, X[N][b]) / W[N][a]);
        for (int a = 0; a <= N; ++a) {
            lpml[N][0][a] = lagrange_ld(N, X[N], a, -1.0L);
            lpml[N][1][a] = lagrange_ld(N, X[N], a, 1.0L);
            lpm[N][0][a] = (double)lpml[N][0][a];
            lpm[N][1][a] = (double)lpml[N][1][a];
        }
    }
    /* Interpolation T^{Nf->Nt}[i][a] = l^{Nf}_a(x^{Nt}_i)  (sampling, A3). */
    for (int Nf = 1; Nf <= NMAXB; ++Nf)
        for (int Nt = 1; Nt <= NMAXB; ++Nt)
            for (int i = 0; i <= Nt; ++i)
                for (int a = 0; a <= Nf; ++a) {
                    Tl[Nf][Nt][i * (Nf + 1) + a] = lagrange_ld(Nf, X[Nf], a, X[Nt][i]);
                    Tm[Nf][Nt][i * (Nf + 1) + a] = (double)Tl[Nf][Nt][i * (Nf + 1) + a];
                }
    /* Mortar projection (A6): P^{M->s} = (T^T W_M T)^{-1} T^T W_M, T = T^{s->M}.
     * Exact L2 projection of a degree-M polynomial onto degree s <= M. */
    for (int M = 1; M <= NMAXB; ++M)
        for (int s = 1; s <= M; ++s) {
            int ns = s + 1, nm = M + 1;
            long double A[(NMAXB + 1) * (NMAXB + 1)], B[(NMAXB + 1) * (NMAXB + 1)];
            for (int a = 0; a < ns; ++a)
                for (int b = 0; b < ns; ++b) {
                    long double acc = 0.0L;
                    for (int i = 0; i < nm; ++i)
                        acc += lagrange_ld(s, X[s], a, X[M][i]) * W[M][i] * lagrange_ld(s, X[s], b, X[M][i]);
                    A[a * ns + b] = acc;
                }
            for (int a = 0; a < ns; ++a)
                for (int i = 0; i < nm; ++i)
                    B[a * nm + i] = lagrange_ld(s, X[s], a, X[M][i]) * W[M][i];
            solve_ld(ns, nm, A, B);
            for (int a = 0; a < ns; ++a)
                for (int i = 0; i < nm; ++i)
                    Pm[M][s][a * nm + i] = (double)B[a * nm + i];
        }
    basis_ready = 1;
}

int orc_basis(int N, double* x, double* w, double* D, double* Dhat, double* lm1, double* lp1)
{
    orc_init_basis();
    if (N < 1 || N > NMAXB) return -1;
    for (int a = 0; a <= N; ++a) {
        if (x) x[a] = gl_x[N][a];
        if (w) w[a] = gl_w[N][a];
        if (lm1) lm1[a] = lpm[N][0][a];
        if (lp1) lp1[a] = lpm[N][1][a];
        for (int b = 0; b <= N; ++b) {
            if (D) D[a * (N + 1) + b] = Dm[N][a][b];
            if (Dhat) Dhat[a * (N + 1) + b] = Dh[N][a][b];
        }
    }
    return 0;
}

int orc_interp_matrix(int Nf, int Nt, double* T)
{
    orc_init_basis();
    if (Nf < 1 || Nt < 1 || Nf > NMAXB || Nt > NMAXB) return -1;
    memcpy(T, Tm[Nf][Nt], sizeof(double) * (Nf + 1) * (Nt + 1));
    return 0;
}

int orc_projection_matrix(int M, int s, double* P)
{
    orc_init_basis();
    if (s < 1 || M < s || M > NMAXB) return -1;
    memcpy(P, Pm[M][s], sizeof(double) * (M + 1) * (s + 1));
    return 0;
}

/* ------------------------------------------------------------------------- */
/* 2. Tensor-product helpers.                                                */
/* ------------------------------------------------------------------------- */

static inline int npts(const int N[3]) { return (N[0] + 1) * (N[1] + 1) * (N[2] + 1); }

/* out[c][.. m ..] = sum_a A[m][a] in[c][.. a ..] along direction d.
 * in has point counts nin[3]; out has nin with nin[d] replaced by mout. */
static void tapply(int ncomp, const double* in, const int nin[3], int d, const double* A, int mout, double* out)
{
    int nout[3] = {nin[0], nin[1], nin[2]};
    nout[d] = mout;
    int nI = nin[0] * nin[1] * nin[2], nO = nout[0] * nout[1] * nout[2];
    for (int c = 0; c < ncomp; ++c)
        for (int k = 0; k < nout[2]; ++k)
            for (int j = 0; j < nout[1]; ++j)
                for (int i = 0; i < nout[0]; ++i) {
                    int o[3] = {i, j, k};
                    double acc = 0.0;
                    for (int a = 0; a < nin[d]; ++a) {
                        int t[3] = {i, j, k};
                        t[d] = a;
                        acc += A[o[d] * nin[d] + a] * in[c * nI + t[0] + nin[0] * (t[1] + nin[1] * t[2])];
                    }
                    out[c * nO + i + nout[0] * (j + nout[1] * k)] = acc;
                }
}

/* the same, in long double (geometry only) */
static void tapply_ld(int ncomp, const long double* in, const int nin[3], int d, const long double* A, int mout,
                      long double* out)
{
    int nout[3] = {nin[0], nin[1], nin[2]};
    nout[d] = mout;
    int nI = nin[0] * nin[1] * nin[2], nO = nout[0] * nout[1] * nout[2];
    for (int c = 0; c < ncomp; ++c)
        for (int k = 0; k < nout[2]; ++k)
            for (int j = 0; j < nout[1]; ++j)
                for (int i = 0; i < nout[0]; ++i) {
                    int o[3] = {i, j, k};
                    long double acc = 0.0L;
                    for (int a = 0; a < nin[d]; ++a) {
                        int t[3] = {i, j, k};
                        t[d] = a;
                        acc += A[o[d] * nin[d] + a] * in[c * nI + t[0] + nin[0] * (t[1] + nin[1] * t[2])];
                    }
                    out[c * nO + i + nout[0] * (j + nout[1] * k)] = acc;
                }
}

/* ------------------------------------------------------------------------- */
/* 3. Geometry and metric terms.  P:144 ("the J_j are the Jacobians of the
 *    geometry transformation").  Cross-product form
 *    Ja^1 = x_eta x x_zeta, Ja^2 = x_zeta x x_xi, Ja^3 = x_xi x x_eta,
 *    J = x_xi . (x_eta x x_zeta); exact for affine and extruded meshes.      */
/* ------------------------------------------------------------------------- */

static void cross3(const double a[3], const double b[3], double c[3])
{
    c[0] = a[1] * b[2] - a[2] * b[1];
    c[1] = a[2] * b[0] - a[0] * b[2];
    c[2] = a[0] * b[1] - a[1] * b[0];
}

/* Coordinates at the solution nodes of order N from the element's geometry
 * nodes (GL nodes of order g, [3][ng]).  Kept in long double (see Tl). */
static void element_coords(const orc_mesh* m, int e, const int N[3], long double* X)
{
    const int* g = m->gorder;
    int ng[3] = {g[0] + 1, g[1] + 1, g[2] + 1};
    int ngt = ng[0] * ng[1] * ng[2];
    long double* G = malloc(sizeof(long double) * 3 * ngt);
    for (int i = 0; i < 3 * ngt; ++i) G[i] = m->geo[(size_t)e * 3 * ngt + i];
    int n1[3] = {N[0] + 1, ng[1], ng[2]};
    int n2[3] = {N[0] + 1, N[1] + 1, ng[2]};
    long double* t1 = malloc(sizeof(long double) * 3 * n1[0] * n1[1] * n1[2]);
    long double* t2 = malloc(sizeof(long double) * 3 * n2[0] * n2[1] * n2[2]);
    tapply_ld(3, G, ng, 0, Tl[g[0]][N[0]], N[0] + 1, t1);
    tapply_ld(3, t1, n1, 1, Tl[g[1]][N[1]], N[1] + 1, t2);
    tapply_ld(3, t2, n2, 2, Tl[g[2]][N[2]], N[2] + 1, X);
    free(G);
    free(t1);
    free(t2);
}

static void dmat_ld(int N, long double* out) { for (int a = 0; a <= N; ++a) for (int b = 0; b <= N; ++b) out[a * (N + 1) + b] = Dl[N][a][b]; }

static void cross3l(const long double a[3], const long double b[3], long double c[3])
{
    c[0] = a[1] * b[2] - a[2] * b[1];
    c[1] = a[2] * b[0] - a[0] * b[2];
    c[2] = a[0] * b[1] - a[1] * b[0];
}

/* Metrics Ja[d][k][node] (k-th Cartesian component of J a^d) and J[node]
 * from nodal coordinates X[3][n] at order N (derivatives with D^{N_d}),
 * evaluated in long double and rounded once to double. */
static void metrics_from_coords(const int N[3], const long double* X, double* Ja, double* J)
{
    int np[3] = {N[0] + 1, N[1] + 1, N[2] + 1};
    int n = npts(N);
    long double* dX = malloc(sizeof(long double) * 9 * n); /* dX[dd][c][node] = d x_c / d xi_dd */
    for (int dd = 0; dd < 3; ++dd) {
        long double Dc[(NMAXB + 1) * (NMAXB + 1)];
        dmat_ld(N[dd], Dc);
        tapply_ld(3, X, np, dd, Dc, np[dd], dX + 3 * n * dd);
    }
    for (int i = 0; i < n; ++i) {
        long double xa[3], xb[3], xc[3], c[3];
        for (int k = 0; k < 3; ++k) { xa[k] = dX[0 * 3 * n + k * n + i]; xb[k] = dX[1 * 3 * n + k * n + i]; xc[k] = dX[2 * 3 * n + k * n + i]; }
        cross3l(xb, xc, c);
        for (int k = 0; k < 3; ++k) Ja[(0 * 3 + k) * n + i] = (double)c[k];
        J[i] = (double)(xa[0] * c[0] + xa[1] * c[1] + xa[2] * c[2]);
        cross3l(xc, xa, c);
        for (int k = 0; k < 3; ++k) Ja[(1 * 3 + k) * n + i] = (double)c[k];
        cross3l(xa, xb, c);
        for (int k = 0; k < 3; ++k) Ja[(2 * 3 + k) * n + i] = (double)c[k];
    }
    free(dX);
}

/* contiguous copies of padded tables */
static void dhat(int N, double* out) { for (int a = 0; a <= N; ++a) for (int b = 0; b <= N; ++b) out[a * (N + 1) + b] = Dh[N][a][b]; }

static const int TAN[3][2] = {{1, 2}, {0, 2}, {0, 1}};

/* Face metric J a^d at the mortar nodes (orders M1, M2 in the tangential
 * directions of d) of face (d, s) of element e, from e's geometry polynomial
 * (reading A6: the mortar metric comes from one side's geometry; the face is
 * watertight so both sides agree when their orders resolve the geometry).
 * Ja^d only needs the tangential derivatives of the face coordinates. */
static void face_metric(const orc_mesh* m, int e, int d, int s, int M1, int M2, double* Jaf /*[3][nf]*/)
{
    const int* g = m->gorder;
    int ng[3] = {g[0] + 1, g[1] + 1, g[2] + 1};
    int ngt = ng[0] * ng[1] * ng[2];
    int t1 = TAN[d][0], t2 = TAN[d][1];
    /* evaluate geometry on the face: along d with l^{g_d}(+-1), along t with T */
    int na[3] = {ng[0], ng[1], ng[2]};
    size_t big = 3 * (NMAXB + 1) * (NMAXB + 1) * (NMAXB + 1);
    long double* G = malloc(sizeof(long double) * 3 * ngt);
    for (int i = 0; i < 3 * ngt; ++i) G[i] = m->geo[(size_t)e * 3 * ngt + i];
    long double* a = malloc(sizeof(long double) * big);
    long double* b = malloc(sizeof(long double) * big);
    long double* c = malloc(sizeof(long double) * big);
    tapply_ld(3, G, na, d, lpml[g[d]][s], 1, a);
    na[d] = 1;
    tapply_ld(3, a, na, t1, Tl[g[t1]][M1], M1 + 1, b);
    na[t1] = M1 + 1;
    tapply_ld(3, b, na, t2, Tl[g[t2]][M2], M2 + 1, c);
    na[t2] = M2 + 1; /* c = face coordinates X[3][nf] with dims na (na[d]=1) */
    int nf = na[0] * na[1] * na[2];
    long double* d1 = malloc(sizeof(long double) * 3 * nf);
    long double* d2 = malloc(sizeof(long double) * 3 * nf);
    long double D1[(NMAXB + 1) * (NMAXB + 1)], D2[(NMAXB + 1) * (NMAXB + 1)];
    dmat_ld(M1, D1);
    dmat_ld(M2, D2);
    tapply_ld(3, c, na, t1, D1, M1 + 1, d1);
    tapply_ld(3, c, na, t2, D2, M2 + 1, d2);
    for (int i = 0; i < nf; ++i) {
        long double u[3], v[3], w[3];
        for (int k = 0; k < 3; ++k) { u[k] = d1[k * nf + i]; v[k] = d2[k * nf + i]; }
        if (d == 1) cross3l(v, u, w); /* Ja^2 = x_zeta x x_xi = x_t2 x x_t1 */
        else cross3l(u, v, w);        /* Ja^1 = x_eta x x_zeta, Ja^3 = x_xi x x_eta */
        for (int k = 0; k < 3; ++k) Jaf[k * nf + i] = (double)w[k];
    }
    free(G); free(a); free(b); free(c); free(d1); free(d2);
}

/* ------------------------------------------------------------------------- */
/* 4. Physics: Euler advective flux, Roe flux (via explicit eigenvectors),
 *    local Lax-Friedrichs, viscous flux.  P:106-126 (eqs NScons,
 *    SystemAdvDiff), P:472 (Roe, BR1), readings A7-A10.                     */
/* ------------------------------------------------------------------------- */

static double pressure(const double* q, double gam)
{
    return (gam - 1.0) * (q[4] - 0.5 * (q[1] * q[1] + q[2] * q[2] + q[3] * q[3]) / q[0]);
}

/* advective flux in Cartesian direction k: (rho u_k, rho u u_k + p e_k, (E+p) u_k) */
void orc_euler_flux(const double* q, int k, double gam, double* f)
{
    double p = pressure(q, gam);
    double uk = q[1 + k] / q[0];
    f[0] = q[1 + k];
    f[1] = q[1] * uk;
    f[2] = q[2] * uk;
    f[3] = q[3] * uk;
    f[1 + k] += p;
    f[4] = (q[4] + p) * uk;
}

static void flux_dot(const double* q, const double n[3], double gam, double* f)
{
    double fk[5];
    for (int v = 0; v < 5; ++v) f[v] = 0.0;
    for (int k = 0; k < 3; ++k) {
        orc_euler_flux(q, k, gam, fk);
        for (int v = 0; v < 5; ++v) f[v] += n[k] * fk[v];
    }
}

/* Roe approximate Riemann solver, no entropy fix (A7), written as
 * F = 1/2 (f_L + f_R).n - 1/2 R |Lambda| R^{-1} (q_R - q_L) with the
 * eigenvector matrix R of the Roe-averaged flux Jacobian built explicitly
 * and R^{-1} dq obtained by a linear solve. */
void orc_roe_flux(const double* qL, const double* qR, const double* n, double gam, double* F)
{
    double rl = sqrt(qL[0]), rr = sqrt(qR[0]);
    double pL = pressure(qL, gam), pR = pressure(qR, gam);
    double u[3], H;
    for (int k = 0; k < 3; ++k) u[k] = (qL[1 + k] / rl + qR[1 + k] / rr) / (rl + rr);
    H = ((qL[4] + pL) / rl + (qR[4] + pR) / rr) / (rl + rr);
    double uu = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
    double c = sqrt((gam - 1.0) * (H - 0.5 * uu));
    double un = u[0] * n[0] + u[1] * n[1] + u[2] * n[2];
    /* orthonormal tangents */
    int ax = 0;
    if (fabs(n[1]) < fabs(n[ax])) ax = 1;
    if (fabs(n[2]) < fabs(n[ax])) ax = 2;
    double t1[3] = {0, 0, 0}, t2[3];
    t1[ax] = 1.0;
    double dn = t1[0] * n[0] + t1[1] * n[1] + t1[2] * n[2];
    for (int k = 0; k < 3; ++k) t1[k] -= dn * n[k];
    double nt = sqrt(t1[0] * t1[0] + t1[1] * t1[1] + t1[2] * t1[2]);
    for (int k = 0; k < 3; ++k) t1[k] /= nt;
    cross3(n, t1, t2);
    /* columns r_1..r_5 */
    double R[5][5]; /* R[row][col] */
    double lam[5] = {un - c, un, un, un, un + c};
    double ut1 = u[0] * t1[0] + u[1] * t1[1] + u[2] * t1[2];
    double ut2 = u[0] * t2[0] + u[1] * t2[1] + u[2] * t2[2];
    R[0][0] = 1; R[0][1] = 1; R[0][2] = 0; R[0][3] = 0; R[0][4] = 1;
    for (int k = 0; k < 3; ++k) {
        R[1 + k][0] = u[k] - c * n[k];
        R[1 + k][1] = u[k];
        R[1 + k][2] = t1[k];
        R[1 + k][3] = t2[k];
        R[1 + k][4] = u[k] + c * n[k];
    }
    R[4][0] = H - un * c; R[4][1] = 0.5 * uu; R[4][2] = ut1; R[4][3] = ut2; R[4][4] = H + un * c;
    long double A[25], B[5];
    for (int r = 0; r < 5; ++r) {
        for (int cc = 0; cc < 5; ++cc) A[r * 5 + cc] = R[r][cc];
        B[r] = qR[r] - qL[r];
    }
    solve_ld(5, 1, A, B); /* B = alpha */
    double fL[5], fR[5];
    flux_dot(qL, n, gam, fL);
    flux_dot(qR, n, gam, fR);
    for (int v = 0; v < 5; ++v) {
        double dis = 0.0;
        for (int k = 0; k < 5; ++k) dis += R[v][k] * fabs(lam[k]) * (double)B[k];
        F[v] = 0.5 * (fL[v] + fR[v]) - 0.5 * dis;
    }
}

/* Local Lax-Friedrichs (Rusanov), a flag (A7). */
void orc_llf_flux(const double* qL, const double* qR, const double* n, double gam, double* F)
{
    double fL[5], fR[5];
    flux_dot(qL, n, gam, fL);
    flux_dot(qR, n, gam, fR);
    double unL = (qL[1] * n[0] + qL[2] * n[1] + qL[3] * n[2]) / qL[0];
    double unR = (qR[1] * n[0] + qR[2] * n[1] + qR[3] * n[2]) / qR[0];
    double cL = sqrt(gam * pressure(qL, gam) / qL[0]);
    double cR = sqrt(gam * pressure(qR, gam) / qR[0]);
    double lam = fmax(fabs(unL) + cL, fabs(unR) + cR);
    for (int v = 0; v < 5; ++v) F[v] = 0.5 * (fL[v] + fR[v]) - 0.5 * lam * (qR[v] - qL[v]);
}

/* Viscous flux f^nu_k(q, grad q) in Cartesian direction k (A8, A9):
 * conserved-variable gradients g[j][v] = d q_v / d x_j; chain rule to u, T. */
void orc_viscous_flux(const double* q, const double* g /*[3][5]*/, int k, const orc_phys* ph, double* f)
{
    double gam = ph->gamma, mu = ph->mu;
    double rho = q[0];
    double u[3] = {q[1] / rho, q[2] / rho, q[3] / rho};
    double p = pressure(q, gam);
    double T = p / rho;
    double du[3][3]; /* du[i][j] = d u_i / d x_j */
    double dT[3];
    for (int j = 0; j < 3; ++j) {
        const double* gj = g + 5 * j;
        for (int i = 0; i < 3; ++i) du[i][j] = (gj[1 + i] - u[i] * gj[0]) / rho;
        double dp = (gam - 1.0) * (gj[4] - (u[0] * gj[1] + u[1] * gj[2] + u[2] * gj[3]) + 0.5 * (u[0] * u[0] + u[1] * u[1] + u[2] * u[2]) * gj[0]);
        dT[j] = (dp - T * gj[0]) / rho;
    }
    double div = du[0][0] + du[1][1] + du[2][2];
    double tau[3];
    for (int i = 0; i < 3; ++i) tau[i] = mu * (du[i][k] + du[k][i] - (i == k ? 2.0 / 3.0 * div : 0.0));
    double kappa = mu * gam / ((gam - 1.0) * ph->Pr);
    f[0] = 0.0;
    f[1] = tau[0];
    f[2] = tau[1];
    f[3] = tau[2];
    f[4] = u[0] * tau[0] + u[1] * tau[1] + u[2] * tau[2] + kappa * dT[k];
}

/* ------------------------------------------------------------------------- */
/* 5. Element-level DGSEM operator.  P:129-155 (eqs DGSEMsystem, DGMassMatrix):
 *    Qdot_abc = -(1/J) sum_d [ sum_m Dhat^d_{a_d m} Ft^d(..m..)
 *                              + (l_{a_d}(+1) G^d_+ - l_{a_d}(-1) G^d_-)/w_{a_d} ]
 *    with Ft^d = Ja^d . (f^a - f^nu) and G the surface (numerical) flux on the
 *    element's own face nodes.  BR1 gradient (eq DGSEMsystem:2):
 *    J g_k = sum_d [ sum_m Dhat^d (Ja^d_k q) + (l(+1) qhat_+ Ja^d_k|_+ - l(-1) qhat_- Ja^d_k|_-)/w ]. */
/* ------------------------------------------------------------------------- */

typedef struct {
    int N[3], np[3], n;
    long double* X;     /* [3][n] */
    double *Ja, *J;     /* [3][3][n], [n] */
} egeo;

static void egeo_build(const orc_mesh* m, int e, const int N[3], egeo* G)
{
    for (int d = 0; d < 3; ++d) { G->N[d] = N[d]; G->np[d] = N[d] + 1; }
    G->n = npts(N);
    G->X = malloc(sizeof(long double) * 3 * G->n);
    G->Ja = malloc(sizeof(double) * 9 * G->n);
    G->J = malloc(sizeof(double) * G->n);
    element_coords(m, e, N, G->X);
    metrics_from_coords(N, G->X, G->Ja, G->J);
}

static void egeo_from_coords(const int N[3], const long double* X, egeo* G)
{
    for (int d = 0; d < 3; ++d) { G->N[d] = N[d]; G->np[d] = N[d] + 1; }
    G->n = npts(N);
    G->X = malloc(sizeof(long double) * 3 * G->n);
    memcpy(G->X, X, sizeof(long double) * 3 * G->n);
    G->Ja = malloc(sizeof(double) * 9 * G->n);
    G->J = malloc(sizeof(double) * G->n);
    metrics_from_coords(N, G->X, G->Ja, G->J);
}

static void egeo_free(egeo* G) { free(G->X); free(G->Ja); free(G->J); }

static int face_npts(const int N[3], int d) { return (N[TAN[d][0]] + 1) * (N[TAN[d][1]] + 1); }

/* trace of ncomp nodal fields on face (d,s): l(+-1) along d (GL: node values). */
static void trace(int ncomp, const double* u, const int N[3], int d, int s, double* out)
{
    int np[3] = {N[0] + 1, N[1] + 1, N[2] + 1};
    tapply(ncomp, u, np, d, lpm[N[d]][s], 1, out);
}

/* Gradient pass for one element: g[3 (j)][5][n], given qhat*Ja^d face terms
 * Hf[f][3 (k)][5][nf] on the element's own face nodes. */
static void element_gradient(const egeo* G, const double* q, double* const Hf[6], double* grad)
{
    int n = G->n;
    const int* N = G->N;
    double* tmp = malloc(sizeof(double) * 5 * n);
    double* out = malloc(sizeof(double) * 5 * n);
    double Dc[(NMAXB + 1) * (NMAXB + 1)];
    for (int j = 0; j < 3; ++j) { /* Cartesian component of the gradient */
        double* gj = grad + (size_t)j * 5 * n;
        for (int i = 0; i < 5 * n; ++i) gj[i] = 0.0;
        for (int d = 0; d < 3; ++d) {
            for (int v = 0; v < 5; ++v)
                for (int i = 0; i < n; ++i) tmp[v * n + i] = G->Ja[(d * 3 + j) * n + i] * q[v * n + i];
            dhat(N[d], Dc);
            tapply(5, tmp, G->np, d, Dc, G->np[d], out);
            for (int i = 0; i < 5 * n; ++i) gj[i] += out[i];
            /* lifting of qhat * Ja^d_j on the two faces normal to d */
            int nf = face_npts(N, d);
            for (int k = 0; k < G->np[2]; ++k)
                for (int jj = 0; jj < G->np[1]; ++jj)
                    for (int i = 0; i < G->np[0]; ++i) {
                        int idx[3] = {i, jj, k};
                        int a = idx[d];
                        int t1 = idx[TAN[d][0]], t2 = idx[TAN[d][1]];
                        int fi = t1 + (N[TAN[d][0]] + 1) * t2;
                        int node = i + G->np[0] * (jj + G->np[1] * k);
                        for (int v = 0; v < 5; ++v) {
                            double Hp = Hf[2 * d + 1][(j * 5 + v) * nf + fi];
                            double Hm = Hf[2 * d + 0][(j * 5 + v) * nf + fi];
                            gj[v * n + node] += (lpm[N[d]][1][a] * Hp - lpm[N[d]][0][a] * Hm) / gl_w[N[d]][a];
                        }
                    }
        }
        for (int v = 0; v < 5; ++v)
            for (int i = 0; i < n; ++i) gj[v * n + i] /= G->J[i];
    }
    free(tmp);
    free(out);
}

/* Volume + lifting for one element given its surface fluxes Gf[f][5][nf]. */
static void element_residual(const egeo* G, const double* q, const double* grad, double* const Gf[6],
                             const orc_phys* ph, double* qdot)
{
    int n = G->n;
    const int* N = G->N;
    double* Ft = malloc(sizeof(double) * 5 * n);
    double* out = malloc(sizeof(double) * 5 * n);
    double* acc = calloc(5 * n, sizeof(double));
    double Dc[(NMAXB + 1) * (NMAXB + 1)];
    for (int d = 0; d < 3; ++d) {
        /* contravariant flux Ft^d = sum_k Ja^d_k (f^a_k - f^nu_k) */
        for (int i = 0; i < n; ++i) {
            double qi[5], fk[5], fv[5], gi[15];
            for (int v = 0; v < 5; ++v) qi[v] = q[v * n + i];
            double F[5] = {0, 0, 0, 0, 0};
            for (int k = 0; k < 3; ++k) {
                double jak = G->Ja[(d * 3 + k) * n + i];
                orc_euler_flux(qi, k, ph->gamma, fk);
                if (ph->physics == ORC_NS) {
                    for (int jj = 0; jj < 3; ++jj)
                        for (int v = 0; v < 5; ++v) gi[jj * 5 + v] = grad[(jj * 5 + v) * n + i];
                    orc_viscous_flux(qi, gi, k, ph, fv);
                    for (int v = 0; v < 5; ++v) fk[v] -= fv[v];
                }
                for (int v = 0; v < 5; ++v) F[v] += jak * fk[v];
            }
            for (int v = 0; v < 5; ++v) Ft[v * n + i] = F[v];
        }
        dhat(N[d], Dc);
        tapply(5, Ft, G->np, d, Dc, G->np[d], out);
        for (int i = 0; i < 5 * n; ++i) acc[i] += out[i];
        int nf = face_npts(N, d);
        for (int k = 0; k < G->np[2]; ++k)
            for (int jj = 0; jj < G->np[1]; ++jj)
                for (int i = 0; i < G->np[0]; ++i) {
                    int idx[3] = {i, jj, k};
                    int a = idx[d];
                    int fi = idx[TAN[d][0]] + (N[TAN[d][0]] + 1) * idx[TAN[d][1]];
                    int node = i + G->np[0] * (jj + G->np[1] * k);
                    for (int v = 0; v < 5; ++v)
                        acc[v * n + node] += (lpm[N[d]][1][a] * Gf[2 * d + 1][v * nf + fi] -
                                              lpm[N[d]][0][a] * Gf[2 * d + 0][v * nf + fi]) / gl_w[N[d]][a];
                }
    }
    for (int v = 0; v < 5; ++v)
        for (int i = 0; i < n; ++i) qdot[v * n + i] = -acc[v * n + i] / G->J[i];
    free(Ft);
    free(out);
    free(acc);
}

/* Isolated face quantities: "simple evaluations of the flux with
 * the inner solution of each element".  Own face metric = volume metric
 * traced to the face. */
static void isolated_faces(const egeo* G, const double* q, const double* grad, const orc_phys* ph,
                           double* Gf[6], double* Hf[6] /* may be NULL */)
{
    const int* N = G->N;
    for (int f = 0; f < 6; ++f) {
        int d = f / 2, s = f % 2;
        int nf = face_npts(N, d);
        double* qt = malloc(sizeof(double) * 5 * nf);
        double* jt = malloc(sizeof(double) * 3 * nf);
        trace(5, q, N, d, s, qt);
        trace(3, G->Ja + (size_t)d * 3 * G->n, N, d, s, jt);
        double* gt = NULL;
        if (grad) {
            gt = malloc(sizeof(double) * 15 * nf);
            trace(15, grad, N, d, s, gt);
        }
        for (int i = 0; i < nf; ++i) {
            double qi[5], fk[5], fv[5], gi[15];
            for (int v = 0; v < 5; ++v) qi[v] = qt[v * nf + i];
            if (Hf)
                for (int k = 0; k < 3; ++k)
                    for (int v = 0; v < 5; ++v) Hf[f][(k * 5 + v) * nf + i] = qi[v] * jt[k * nf + i];
            if (Gf) {
                double F[5] = {0, 0, 0, 0, 0};
                for (int k = 0; k < 3; ++k) {
                    orc_euler_flux(qi, k, ph->gamma, fk);
                    if (gt && ph->physics == ORC_NS) {
                        for (int jj = 0; jj < 15; ++jj) gi[jj] = gt[jj * nf + i];
                        orc_viscous_flux(qi, gi, k, ph, fv);
                        for (int v = 0; v < 5; ++v) fk[v] -= fv[v];
                    }
                    for (int v = 0; v < 5; ++v) F[v] += jt[k * nf + i] * fk[v];
                }
                for (int v = 0; v < 5; ++v) Gf[f][v * nf + i] = F[v];
            }
        }
        free(qt); free(jt); free(gt);
    }
}

/* ------------------------------------------------------------------------- */
/* 6. Non-isolated surface terms with mortars (reading A6) and the
 *    wall / far-field boundary states (A10).                                 */
/* ------------------------------------------------------------------------- */

typedef struct {
    const orc_mesh* m;
    const int32_t* orders;
    const size_t* off;   /* state offset (doubles) of each element */
    const double* q;
    const double* grad;  /* [3][5][n] per element at 15*off/5, or NULL */
    const size_t* goff;  /* grad offsets */
    const orc_phys* ph;
} gctx;

static void boundary_ghost(const double* qin, int bc, const orc_phys* ph, double* qg)
{
    if (bc == ORC_BC_WALL) { /* mirrored momentum (no slip) */
        qg[0] = qin[0]; qg[1] = -qin[1]; qg[2] = -qin[2]; qg[3] = -qin[3]; qg[4] = qin[4];
    } else {
        for (int v = 0; v < 5; ++v) qg[v] = ph->qinf[v];
    }
}

static void riemann(const double* qL, const double* qR, const double* nrm, const orc_phys* ph, double* F)
{
    if (ph->flux == ORC_FLUX_LLF) orc_llf_flux(qL, qR, nrm, ph->gamma, F);
    else orc_roe_flux(qL, qR, nrm, ph->gamma, F);
}

/* For face f of element e, compute on e's own face nodes:
 *   which == 0: G  [5][nf]    = Ja^d.(f^a* - f^nu*)  (projected from the mortar)
 *   which == 1: H  [3][5][nf] = qhat Ja^d_k          (projected from the mortar) */
static void nonisolated_face(const gctx* C, int e, int f, int which, double* out)
{
    const orc_mesh* m = C->m;
    int d = f / 2, s = f % 2;
    int t1 = TAN[d][0], t2 = TAN[d][1];
    const int32_t* No = C->orders + 3 * e;
    int Ne[3] = {No[0], No[1], No[2]};
    int nb = m->nbr[6 * e + f];
    int nfo = face_npts(Ne, d);
    int ncomp = which == 0 ? 5 : 15;
    const orc_phys* ph = C->ph;

    if (nb < 0) {
        /* physical boundary: mortar = own face, metric from own geometry */
        double* qt = malloc(sizeof(double) * 5 * nfo);
        double* gt = malloc(sizeof(double) * 15 * nfo);
        double* jt = malloc(sizeof(double) * 3 * nfo);
        int n = npts(Ne);
        trace(5, C->q + C->off[e], Ne, d, s, qt);
        if (C->grad) trace(15, C->grad + C->goff[e], Ne, d, s, gt);
        face_metric(m, e, d, s, Ne[t1], Ne[t2], jt);
        (void)n;
        for (int i = 0; i < nfo; ++i) {
            double qi[5], qg[5], Ja[3], S, nrm[3];
            for (int v = 0; v < 5; ++v) qi[v] = qt[v * nfo + i];
            for (int k = 0; k < 3; ++k) Ja[k] = jt[k * nfo + i];
            S = sqrt(Ja[0] * Ja[0] + Ja[1] * Ja[1] + Ja[2] * Ja[2]);
            for (int k = 0; k < 3; ++k) nrm[k] = Ja[k] / S;
            boundary_ghost(qi, nb, ph, qg);
            if (which == 1) {
                double qh[5];
                if (nb == ORC_BC_WALL) {
                    qh[0] = qi[0]; qh[1] = 0; qh[2] = 0; qh[3] = 0;
                    qh[4] = qi[4] - 0.5 * (qi[1] * qi[1] + qi[2] * qi[2] + qi[3] * qi[3]) / qi[0];
                } else {
                    for (int v = 0; v < 5; ++v) qh[v] = 0.5 * (qi[v] + ph->qinf[v]);
                }
                for (int k = 0; k < 3; ++k)
                    for (int v = 0; v < 5; ++v) out[(k * 5 + v) * nfo + i] = qh[v] * Ja[k];
            } else {
                double F[5];
                if (s == 1) riemann(qi, qg, nrm, ph, F); else riemann(qg, qi, nrm, ph, F);
                for (int v = 0; v < 5; ++v) F[v] *= S;
                if (ph->physics == ORC_NS && C->grad) {
                    double gi[15], fv[5], Fv[5] = {0, 0, 0, 0, 0};
                    for (int jj = 0; jj < 15; ++jj) gi[jj] = gt[jj * nfo + i];
                    for (int k = 0; k < 3; ++k) {
                        orc_viscous_flux(qi, gi, k, ph, fv);
                        for (int v = 0; v < 5; ++v) Fv[v] += Ja[k] * fv[v];
                    }
                    if (nb == ORC_BC_WALL) Fv[4] = 0.0; /* u = 0 and adiabatic */
                    for (int v = 0; v < 5; ++v) F[v] -= Fv[v];
                }
                for (int v = 0; v < 5; ++v) out[v * nfo + i] = F[v];
            }
        }
        free(qt); free(gt); free(jt);
        return;
    }

    int L = s == 1 ? e : nb, R = s == 1 ? nb : e;
    int NL[3] = {C->orders[3 * L], C->orders[3 * L + 1], C->orders[3 * L + 2]};
    int NR[3] = {C->orders[3 * R], C->orders[3 * R + 1], C->orders[3 * R + 2]};
    int M1 = NL[t1] > NR[t1] ? NL[t1] : NR[t1];
    int M2 = NL[t2] > NR[t2] ? NL[t2] : NR[t2];
    int nfm = (M1 + 1) * (M2 + 1);
    int nfL = face_npts(NL, d), nfR = face_npts(NR, d);
    double *qtL = malloc(sizeof(double) * 15 * nfL), *qtR = malloc(sizeof(double) * 15 * nfR);
    double *gtL = malloc(sizeof(double) * 15 * nfL), *gtR = malloc(sizeof(double) * 15 * nfR);
    double *tmp = malloc(sizeof(double) * 15 * nfm * 2);
    double *qmL = malloc(sizeof(double) * 15 * nfm), *qmR = malloc(sizeof(double) * 15 * nfm);
    double *gmL = malloc(sizeof(double) * 15 * nfm), *gmR = malloc(sizeof(double) * 15 * nfm);
    double *jm = malloc(sizeof(double) * 3 * nfm), *om = malloc(sizeof(double) * 15 * nfm);
    int use_grad = (which == 0 && ph->physics == ORC_NS && C->grad);

    trace(5, C->q + C->off[L], NL, d, 1, qtL);
    trace(5, C->q + C->off[R], NR, d, 0, qtR);
    /* interpolate both traces to the mortar (orders M1, M2) */
    {
        int na[3] = {NL[0] + 1, NL[1] + 1, NL[2] + 1};
        na[d] = 1;
        tapply(5, qtL, na, t1, Tm[NL[t1]][M1], M1 + 1, tmp); na[t1] = M1 + 1;
        tapply(5, tmp, na, t2, Tm[NL[t2]][M2], M2 + 1, qmL);
        int nb3[3] = {NR[0] + 1, NR[1] + 1, NR[2] + 1};
        nb3[d] = 1;
        tapply(5, qtR, nb3, t1, Tm[NR[t1]][M1], M1 + 1, tmp); nb3[t1] = M1 + 1;
        tapply(5, tmp, nb3, t2, Tm[NR[t2]][M2], M2 + 1, qmR);
    }
    if (use_grad) {
        trace(15, C->grad + C->goff[L], NL, d, 1, gtL);
        trace(15, C->grad + C->goff[R], NR, d, 0, gtR);
        int na[3] = {NL[0] + 1, NL[1] + 1, NL[2] + 1};
        na[d] = 1;
        tapply(15, gtL, na, t1, Tm[NL[t1]][M1], M1 + 1, tmp); na[t1] = M1 + 1;
        tapply(15, tmp, na, t2, Tm[NL[t2]][M2], M2 + 1, gmL);
        int nb3[3] = {NR[0] + 1, NR[1] + 1, NR[2] + 1};
        nb3[d] = 1;
        tapply(15, gtR, nb3, t1, Tm[NR[t1]][M1], M1 + 1, tmp); nb3[t1] = M1 + 1;
        tapply(15, tmp, nb3, t2, Tm[NR[t2]][M2], M2 + 1, gmR);
    }
    face_metric(m, L, d, 1, M1, M2, jm); /* mortar metric from L's geometry (A6) */
    for (int i = 0; i < nfm; ++i) {
        double qL[5], qR[5], Ja[3], S, nrm[3];
        for (int v = 0; v < 5; ++v) { qL[v] = qmL[v * nfm + i]; qR[v] = qmR[v * nfm + i]; }
        for (int k = 0; k < 3; ++k) Ja[k] = jm[k * nfm + i];
        S = sqrt(Ja[0] * Ja[0] + Ja[1] * Ja[1] + Ja[2] * Ja[2]);
        for (int k = 0; k < 3; ++k) nrm[k] = Ja[k] / S;
        if (which == 1) {
            for (int k = 0; k < 3; ++k)
                for (int v = 0; v < 5; ++v) om[(k * 5 + v) * nfm + i] = 0.5 * (qL[v] + qR[v]) * Ja[k];
        } else {
            double F[5];
            riemann(qL, qR, nrm, ph, F);
            for (int v = 0; v < 5; ++v) F[v] *= S;
            if (use_grad) {
                double gL[15], gR[15], fvL[5], fvR[5];
                for (int jj = 0; jj < 15; ++jj) { gL[jj] = gmL[jj * nfm + i]; gR[jj] = gmR[jj * nfm + i]; }
                for (int k = 0; k < 3; ++k) {
                    orc_viscous_flux(qL, gL, k, ph, fvL);
                    orc_viscous_flux(qR, gR, k, ph, fvR);
                    for (int v = 0; v < 5; ++v) F[v] -= 0.5 * (fvL[v] + fvR[v]) * Ja[k];
                }
            }
            for (int v = 0; v < 5; ++v) om[v * nfm + i] = F[v];
        }
    }
    /* project the mortar quantity back to e's own face nodes (A6) */
    {
        int na[3] = {1, 1, 1};
        na[t1] = M1 + 1; na[t2] = M2 + 1;
        double P1[(NMAXB + 1) * (NMAXB + 1)], P2[(NMAXB + 1) * (NMAXB + 1)];
        memcpy(P1, Pm[M1][Ne[t1]], sizeof(double) * (M1 + 1) * (Ne[t1] + 1));
        memcpy(P2, Pm[M2][Ne[t2]], sizeof(double) * (M2 + 1) * (Ne[t2] + 1));
        tapply(ncomp, om, na, t1, P1, Ne[t1] + 1, tmp); na[t1] = Ne[t1] + 1;
        tapply(ncomp, tmp, na, t2, P2, Ne[t2] + 1, out);
    }
    free(qtL); free(qtR); free(gtL); free(gtR); free(tmp);
    free(qmL); free(qmR); free(gmL); free(gmR); free(jm); free(om);
}

/* ------------------------------------------------------------------------- */
/* 7. Global residual Qdot = -(M^N)^{-1} F^N(Q)  (eq DGMassMatrixRight). */
/* ------------------------------------------------------------------------- */

static size_t* make_offsets(int E, const int32_t* orders, int ncomp)
{
    size_t* off = malloc(sizeof(size_t) * (E + 1));
    off[0] = 0;
    for (int e = 0; e < E; ++e) {
        int N[3] = {orders[3 * e], orders[3 * e + 1], orders[3 * e + 2]};
        off[e + 1] = off[e] + (size_t)ncomp * npts(N);
    }
    return off;
}

int orc_rhs(const orc_mesh* m, const int32_t* orders, const double* q, int variant, const orc_phys* ph, double* qdot)
{
    orc_init_basis();
    int E = m->E;
    for (int e = 0; e < E; ++e)
        for (int d = 0; d < 3; ++d)
            if (orders[3 * e + d] < 1 || orders[3 * e + d] > NMAXB) return -1;
    size_t* off = make_offsets(E, orders, 5);
    size_t* goff = make_offsets(E, orders, 15);
    double* grad = NULL;
    gctx C = {m, orders, off, q, NULL, goff, ph};

    if (ph->physics == ORC_NS) {
        grad = malloc(sizeof(double) * goff[E]);
        /* pass 1: BR1 gradients of every element */
#pragma omp parallel for schedule(guided)
        for (int e = 0; e < E; ++e) {
            int N[3] = {orders[3 * e], orders[3 * e + 1], orders[3 * e + 2]};
            egeo G;
            egeo_build(m, e, N, &G);
            double* Hf[6];
            for (int f = 0; f < 6; ++f) Hf[f] = malloc(sizeof(double) * 15 * face_npts(N, f / 2));
            if (variant == ORC_ISOLATED) isolated_faces(&G, q + off[e], NULL, ph, NULL, Hf);
            else for (int f = 0; f < 6; ++f) nonisolated_face(&C, e, f, 1, Hf[f]);
            element_gradient(&G, q + off[e], Hf, grad + goff[e]);
            for (int f = 0; f < 6; ++f) free(Hf[f]);
            egeo_free(&G);
        }
        C.grad = grad;
    }
    /* pass 2: surface fluxes, volume term, lifting, mass matrix inverse */
#pragma omp parallel for schedule(guided)
    for (int e = 0; e < E; ++e) {
        int N[3] = {orders[3 * e], orders[3 * e + 1], orders[3 * e + 2]};
        egeo G;
        egeo_build(m, e, N, &G);
        double* Gf[6];
        for (int f = 0; f < 6; ++f) Gf[f] = malloc(sizeof(double) * 5 * face_npts(N, f / 2));
        const double* ge = grad ? grad + goff[e] : NULL;
        if (variant == ORC_ISOLATED) isolated_faces(&G, q + off[e], ge, ph, Gf, NULL);
        else for (int f = 0; f < 6; ++f) nonisolated_face(&C, e, f, 0, Gf[f]);
        element_residual(&G, q + off[e], ge, Gf, ph, qdot + off[e]);
        for (int f = 0; f < 6; ++f) free(Gf[f]);
        egeo_free(&G);
    }
    free(grad);
    free(off);
    free(goff);
    return 0;
}

/* Gradient field only (for tests): grad[e] = [3][5][n]. */
int orc_gradient(const orc_mesh* m, const int32_t* orders, const double* q, int variant, const orc_phys* ph, double* grad)
{
    orc_init_basis();
    int E = m->E;
    size_t* off = make_offsets(E, orders, 5);
    size_t* goff = make_offsets(E, orders, 15);
    gctx C = {m, orders, off, q, NULL, goff, ph};
#pragma omp parallel for schedule(guided)
    for (int e = 0; e < E; ++e) {
        int N[3] = {orders[3 * e], orders[3 * e + 1], orders[3 * e + 2]};
        egeo G;
        egeo_build(m, e, N, &G);
        double* Hf[6];
        for (int f = 0; f < 6; ++f) Hf[f] = malloc(sizeof(double) * 15 * face_npts(N, f / 2));
        if (variant == ORC_ISOLATED) isolated_faces(&G, q + off[e], NULL, ph, NULL, Hf);
        else for (int f = 0; f < 6; ++f) nonisolated_face(&C, e, f, 1, Hf[f]);
        element_gradient(&G, q + off[e], Hf, grad + goff[e]);
        for (int f = 0; f < 6; ++f) free(Hf[f]);
        egeo_free(&G);
    }
    free(off);
    free(goff);
    return 0;
}

/* Node coordinates at the solution nodes (for building inputs in tests). */
int orc_node_coords(const orc_mesh* m, const int32_t* orders, double* X)
{
    orc_init_basis();
    size_t* off = make_offsets(m->E, orders, 3);
    for (int e = 0; e < m->E; ++e) {
        int N[3] = {orders[3 * e], orders[3 * e + 1], orders[3 * e + 2]};
        int n = npts(N);
        long double* Xl = malloc(sizeof(long double) * 3 * n);
        element_coords(m, e, N, Xl);
        for (int i = 0; i < 3 * n; ++i) X[off[e] + i] = (double)Xl[i];
        free(Xl);
    }
    free(off);
    return 0;
}

/* Mass matrix diagonal J_j w_j at every node. */
int orc_mass(const orc_mesh* m, const int32_t* orders, double* M)
{
    orc_init_basis();
    size_t* off = make_offsets(m->E, orders, 1);
    for (int e = 0; e < m->E; ++e) {
        int N[3] = {orders[3 * e], orders[3 * e + 1], orders[3 * e + 2]};
        egeo G;
        egeo_build(m, e, N, &G);
        for (int k = 0; k <= N[2]; ++k)
            for (int j = 0; j <= N[1]; ++j)
                for (int i = 0; i <= N[0]; ++i) {
                    int nd = i + (N[0] + 1) * (j + (N[1] + 1) * k);
                    M[off[e] + nd] = G.J[nd] * gl_w[N[0]][i] * gl_w[N[1]][j] * gl_w[N[2]][k];
                }
        egeo_free(&G);
    }
    free(off);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* 8. Time step (reading A11) and Williamson low-storage RK3
 *    (P:473): g <- A_k g + dt Qdot(q); q <- q + B_k g.                       */
/* ------------------------------------------------------------------------- */

double orc_compute_dt(const orc_mesh* m, const int32_t* orders, const double* q, const orc_phys* ph, double cfl, double dfl)
{
    orc_init_basis();
    size_t* off = make_offsets(m->E, orders, 5);
    double lam_max = 0.0, nu_max = 0.0;
    for (int e = 0; e < m->E; ++e) {
        int N[3] = {orders[3 * e], orders[3 * e + 1], orders[3 * e + 2]};
        egeo G;
        egeo_build(m, e, N, &G);
        int n = G.n;
        const double* qe = q + off[e];
        for (int i = 0; i < n; ++i) {
            double qi[5];
            for (int v = 0; v < 5; ++v) qi[v] = qe[v * n + i];
            double rho = qi[0], u[3] = {qi[1] / rho, qi[2] / rho, qi[3] / rho};
            double c = sqrt(ph->gamma * pressure(qi, ph->gamma) / rho);
            double lam = 0.0, nu = 0.0;
            for (int d = 0; d < 3; ++d) {
                double a[3], an2 = 0.0, ua = 0.0;
                for (int k = 0; k < 3; ++k) { a[k] = G.Ja[(d * 3 + k) * n + i] / G.J[i]; an2 += a[k] * a[k]; ua += u[k] * a[k]; }
                double Np1 = N[d] + 1.0;
                lam += (fabs(ua) + c * sqrt(an2)) * Np1 * Np1 / 2.0;
                if (ph->physics == ORC_NS) {
                    double numax = ph->mu / rho * fmax(4.0 / 3.0, ph->gamma / ph->Pr);
                    nu += numax * an2 * Np1 * Np1 * Np1 * Np1 / 4.0;
                }
            }
            if (lam > lam_max) lam_max = lam;
            if (nu > nu_max) nu_max = nu;
        }
        egeo_free(&G);
    }
    free(off);
    double dt = cfl / lam_max;
    if (ph->physics == ORC_NS && nu_max > 0.0) {
        double dtv = dfl / nu_max;
        if (dtv < dt) dt = dtv;
    }
    return dt;
}

int orc_rk3_step(const orc_mesh* m, const int32_t* orders, double* q, double dt, const orc_phys* ph)
{
    static const double A[3] = {0.0, -5.0 / 9.0, -153.0 / 128.0};
    static const double B[3] = {1.0 / 3.0, 15.0 / 16.0, 8.0 / 15.0};
    size_t* off = make_offsets(m->E, orders, 5);
    size_t len = off[m->E];
    free(off);
    double* g = calloc(len, sizeof(double));
    double* qd = malloc(sizeof(double) * len);
    for (int k = 0; k < 3; ++k) {
        int rc = orc_rhs(m, orders, q, ORC_NONISOLATED, ph, qd);
        if (rc) { free(g); free(qd); return rc; }
        for (size_t i = 0; i < len; ++i) {
            g[i] = A[k] * g[i] + dt * qd[i];
            q[i] = q[i] + B[k] * g[i];
        }
    }
    free(g);
    free(qd);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* 9. tau-estimation (eqs TEtildedef, TEdef P:187;
 *    readings A3, A4, A12).  For element e, direction d, coarse p < N_d:
 *      O = N with O_d = p, q_c = T^{N_d->p}_d q, X_c = T^{N_d->p}_d X,
 *      Qdot_c = isolated residual at O,
 *      tau~ = T(Qdot_ref) - Qdot_c  (new form; I F(q) ~ -Qdot_ref),
 *      tau  = J_c w w w tau~        (traditional form),
 *      tau[e][d][p] = max over coarse nodes and variables of |tau|.
 *    tau[e][d][0] holds ||Qdot_ref,e||_inf (noise scale of reading A14).     */
/* ------------------------------------------------------------------------- */

int orc_tau_estimate(const orc_mesh* m, const int32_t* orders, const double* q, const double* qdot_ref,
                     int formulation, const orc_phys* ph, double* tau)
{
    return orc_tau_estimate_r(m, orders, q, qdot_ref, formulation, 0, ph, tau);
}

/* As orc_tau_estimate with the restriction of q and Qdot_ref along d chosen by
 * `restriction`: 0 = interpolation at the coarse nodes (reading A3, P:165
 * "simply sampling"), 1 = the exact L2 projection P^{N_d->p} (the A3 flag,
 * SURVEY 8(f) rank 4; the mortar projection of section 4).  The coarse
 * geometry is interpolated in both cases. */
int orc_tau_estimate_r(const orc_mesh* m, const int32_t* orders, const double* q, const double* qdot_ref,
                       int formulation, int restriction, const orc_phys* ph, double* tau)
{
    orc_init_basis();
    int E = m->E;
    size_t* off = make_offsets(E, orders, 5);
    for (size_t i = 0; i < (size_t)E * 3 * ORC_TAU_STRIDE; ++i) tau[i] = NAN;
#pragma omp parallel for schedule(guided)
    for (int e = 0; e < E; ++e) {
        int N[3] = {orders[3 * e], orders[3 * e + 1], orders[3 * e + 2]};
        int np[3] = {N[0] + 1, N[1] + 1, N[2] + 1};
        int n = npts(N);
        const double* qe = q + off[e];
        const double* re = qdot_ref + off[e];
        double rnorm = 0.0;
        for (int i = 0; i < 5 * n; ++i) rnorm = fmax(rnorm, fabs(re[i]));
        long double* X = malloc(sizeof(long double) * 3 * n);
        element_coords(m, e, N, X);
        for (int d = 0; d < 3; ++d) {
            tau[((size_t)e * 3 + d) * ORC_TAU_STRIDE + 0] = rnorm;
            for (int p = 1; p < N[d]; ++p) {
                int O[3] = {N[0], N[1], N[2]};
                O[d] = p;
                int nc = npts(O);
                const double* T = restriction ? Pm[N[d]][p] : Tm[N[d]][p];
                double* qc = malloc(sizeof(double) * 5 * nc);
                double* rc = malloc(sizeof(double) * 5 * nc);
                long double* Xc = malloc(sizeof(long double) * 3 * nc);
                double* dc = malloc(sizeof(double) * 5 * nc);
                tapply(5, qe, np, d, T, p + 1, qc);
                tapply(5, re, np, d, T, p + 1, rc);
                tapply_ld(3, X, np, d, Tl[N[d]][p], p + 1, Xc);
                egeo G;
                egeo_from_coords(O, Xc, &G);
                double* Gf[6];
                for (int f = 0; f < 6; ++f) Gf[f] = malloc(sizeof(double) * 5 * face_npts(O, f / 2));
                double* grad = NULL;
                if (ph->physics == ORC_NS) {
                    double* Hf[6];
                    for (int f = 0; f < 6; ++f) Hf[f] = malloc(sizeof(double) * 15 * face_npts(O, f / 2));
                    grad = malloc(sizeof(double) * 15 * nc);
                    isolated_faces(&G, qc, NULL, ph, NULL, Hf);
                    element_gradient(&G, qc, Hf, grad);
                    for (int f = 0; f < 6; ++f) free(Hf[f]);
                }
                isolated_faces(&G, qc, grad, ph, Gf, NULL);
                element_residual(&G, qc, grad, Gf, ph, dc);
                double tmax = 0.0;
                for (int k = 0; k <= O[2]; ++k)
                    for (int j = 0; j <= O[1]; ++j)
                        for (int i = 0; i <= O[0]; ++i) {
                            int nd = i + (O[0] + 1) * (j + (O[1] + 1) * k);
                            double scale = 1.0;
                            if (formulation == ORC_TAU_TRADITIONAL)
                                scale = G.J[nd] * gl_w[O[0]][i] * gl_w[O[1]][j] * gl_w[O[2]][k];
                            for (int v = 0; v < 5; ++v) {
                                double t = scale * (rc[v * nc + nd] - dc[v * nc + nd]);
                                tmax = fmax(tmax, fabs(t));
                            }
                        }
                tau[((size_t)e * 3 + d) * ORC_TAU_STRIDE + p] = tmax;
                for (int f = 0; f < 6; ++f) free(Gf[f]);
                free(grad);
                egeo_free(&G);
                free(qc); free(rc); free(Xc); free(dc);
            }
        }
        free(X);
    }
    free(off);
    return 0;
}

/* Full nodal tau field for one (e, d, p) (test aid: tau = M tau~ pin). */
int orc_tau_field(const orc_mesh* m, const int32_t* orders, const double* q, const double* qdot_ref,
                  int e, int d, int p, int formulation, const orc_phys* ph, double* out)
{
    orc_init_basis();
    size_t* off = make_offsets(m->E, orders, 5);
    int N[3] = {orders[3 * e], orders[3 * e + 1], orders[3 * e + 2]};
    int np[3] = {N[0] + 1, N[1] + 1, N[2] + 1};
    int n = npts(N);
    int O[3] = {N[0], N[1], N[2]};
    O[d] = p;
    int nc = npts(O);
    const double* T = Tm[N[d]][p];
    long double* X = malloc(sizeof(long double) * 3 * n);
    element_coords(m, e, N, X);
    double* qc = malloc(sizeof(double) * 5 * nc);
    double* rc = malloc(sizeof(double) * 5 * nc);
    long double* Xc = malloc(sizeof(long double) * 3 * nc);
    double* dc = malloc(sizeof(double) * 5 * nc);
    tapply(5, q + off[e], np, d, T, p + 1, qc);
    tapply(5, qdot_ref + off[e], np, d, T, p + 1, rc);
    tapply_ld(3, X, np, d, Tl[N[d]][p], p + 1, Xc);
    egeo G;
    egeo_from_coords(O, Xc, &G);
    double* Gf[6];
    for (int f = 0; f < 6; ++f) Gf[f] = malloc(sizeof(double) * 5 * face_npts(O, f / 2));
    double* grad = NULL;
    if (ph->physics == ORC_NS) {
        double* Hf[6];
        for (int f = 0; f < 6; ++f) Hf[f] = malloc(sizeof(double) * 15 * face_npts(O, f / 2));
        grad = malloc(sizeof(double) * 15 * nc);
        isolated_faces(&G, qc, NULL, ph, NULL, Hf);
        element_gradient(&G, qc, Hf, grad);
        for (int f = 0; f < 6; ++f) free(Hf[f]);
    }
    isolated_faces(&G, qc, grad, ph, Gf, NULL);
    element_residual(&G, qc, grad, Gf, ph, dc);
    for (int k = 0; k <= O[2]; ++k)
        for (int j = 0; j <= O[1]; ++j)
            for (int i = 0; i <= O[0]; ++i) {
                int nd = i + (O[0] + 1) * (j + (O[1] + 1) * k);
                double scale = 1.0;
                if (formulation == ORC_TAU_TRADITIONAL) scale = G.J[nd] * gl_w[O[0]][i] * gl_w[O[1]][j] * gl_w[O[2]][k];
                for (int v = 0; v < 5; ++v) out[v * nc + nd] = scale * (rc[v * nc + nd] - dc[v * nc + nd]);
            }
    for (int f = 0; f < 6; ++f) free(Gf[f]);
    free(grad);
    egeo_free(&G);
    free(X); free(qc); free(rc); free(Xc); free(dc); free(off);
    return nc;
}

/* ------------------------------------------------------------------------- */
/* 10. Truncation-error map, extrapolation and selection.
 *     P:229 (map, tau-extrapolation), P:90 (exponential decay)
 *     (approach 2, F_max), P:429 (minimise NDOF), P:441 (strict "< tau_max"),
 *     P:461-463 (sentinel when not asymptotic), readings A12-A16.          */
/* ------------------------------------------------------------------------- */

/* Directional estimate tauhat_d(n), n = 1..ORC_NMAX, for one element. */
/* tall = the element's largest estimate over all directions (reading R11). */
static void directional_hat(int Nd, const double* td /* tau[e][d][0..] */, double tall, double* hat /* [ORC_NMAX+1] */,
                            double* slope_out)
{
    double eps = 1e-13 * fmax(1.0, td[0]);
    double tmax = 0.0;
    for (int p = 1; p < Nd; ++p) tmax = fmax(tmax, td[p]);
    *slope_out = NAN;
    if (Nd <= 1) { /* not estimable: keep the order */
        for (int n = 1; n <= ORC_NMAX; ++n) hat[n] = n == Nd ? 0.0 : ORC_SENTINEL;
        return;
    }
    /* resolved direction: at the rounding floor (A14), or rounding against the
     * element's other directions (R11: 1e-8 of its largest estimate, e.g. the
     * span direction of a two-dimensional flow) */
    if (tmax <= eps || tmax <= 1e-8 * tall) {
        for (int n = 1; n <= ORC_NMAX; ++n) hat[n] = 0.0;
        return;
    }
    int asym = 0;
    double a = 0.0, b = 0.0;
    if (Nd >= 3) { /* OLS of log10 tau_d(p) = a + b p over p = 1..Nd-1 (A13) */
        int K = Nd - 1;
        double sp = 0, sy = 0, spp = 0, spy = 0;
        for (int p = 1; p < Nd; ++p) {
            double y = log10(fmax(td[p], 1e-300));
            sp += p; sy += y; spp += (double)p * p; spy += p * y;
        }
        b = (K * spy - sp * sy) / (K * spp - sp * sp);
        a = (sy - b * sp) / K;
        asym = b < 0.0;
        *slope_out = b;
    }
    for (int n = 1; n <= ORC_NMAX; ++n) {
        if (n < Nd) hat[n] = td[n];
        /* N_d = 2: one coarse level, no extrapolation possible (the
         * pulse "arrives at an area where ... no extrapolation is possible
         * (P < 3)" and escapes refinement): keep the order, as for N_d = 1
         * (reading R12) */
        else if (Nd == 2) hat[n] = n == Nd ? 0.0 : ORC_SENTINEL;
        else hat[n] = asym ? pow(10.0, a + b * n) : ORC_SENTINEL;
    }
}

/* map(n) = sum_d tauhat_d(n_d) on [Nmin,Nmax]^3, flattened
 * (n1-Nmin) + K((n2-Nmin) + K(n3-Nmin)), K = Nmax-Nmin+1. */
int orc_build_map(int E, const int32_t* orders, const double* tau, int Nmin, int Nmax, double* map, double* slopes)
{
    int K = Nmax - Nmin + 1;
    if (Nmin < 1 || Nmax > ORC_NMAX || K < 1) return -1;
    for (int e = 0; e < E; ++e) {
        double hat[3][ORC_NMAX + 1];
        double tall = 0.0;
        for (int d = 0; d < 3; ++d)
            for (int p = 1; p < orders[3 * e + d]; ++p)
                tall = fmax(tall, tau[((size_t)e * 3 + d) * ORC_TAU_STRIDE + p]);
        for (int d = 0; d < 3; ++d) {
            double s;
            directional_hat(orders[3 * e + d], tau + ((size_t)e * 3 + d) * ORC_TAU_STRIDE, tall, hat[d], &s);
            if (slopes) slopes[3 * e + d] = s;
        }
        for (int n3 = Nmin; n3 <= Nmax; ++n3)
            for (int n2 = Nmin; n2 <= Nmax; ++n2)
                for (int n1 = Nmin; n1 <= Nmax; ++n1)
                    map[(size_t)e * K * K * K + (n1 - Nmin) + K * ((n2 - Nmin) + K * (n3 - Nmin))] =
                        hat[0][n1] + hat[1][n2] + hat[2][n3];
    }
    return 0;
}

/* Approach 2 with F_max (eq totalTruncMap): total = max(total, map). */
void orc_combine_max(size_t len, double* total, const double* map)
{
    for (size_t i = 0; i < len; ++i) total[i] = fmax(total[i], map[i]);
}

/* Minimum-NDOF feasible combination (A15): feasible = map < tau_max;
 * minimise prod(n+1), then sum n, then lexicographic (n1,n2,n3);
 * empty set -> (Nmax,Nmax,Nmax).  margin[e] = min |map-tau_max|/tau_max. */
int orc_select_from_map(int E, const double* map, int Nmin, int Nmax, double tau_max, int32_t* out, double* margin)
{
    int K = Nmax - Nmin + 1;
    for (int e = 0; e < E; ++e) {
        const double* me = map + (size_t)e * K * K * K;
        int best[3] = {Nmax, Nmax, Nmax};
        long bestp = -1, bests = 0;
        double mg = INFINITY;
        /* enumerate in lexicographic order (n1 slowest) so ties keep the first */
        for (int n1 = Nmin; n1 <= Nmax; ++n1)
            for (int n2 = Nmin; n2 <= Nmax; ++n2)
                for (int n3 = Nmin; n3 <= Nmax; ++n3) {
                    double v = me[(n1 - Nmin) + K * ((n2 - Nmin) + K * (n3 - Nmin))];
                    mg = fmin(mg, fabs(v - tau_max) / tau_max);
                    if (!(v < tau_max)) continue;
                    long pr = (long)(n1 + 1) * (n2 + 1) * (n3 + 1), sm = n1 + n2 + n3;
                    if (bestp < 0 || pr < bestp || (pr == bestp && sm < bests)) {
                        bestp = pr; bests = sm;
                        best[0] = n1; best[1] = n2; best[2] = n3;
                    }
                }
        for (int d = 0; d < 3; ++d) out[3 * e + d] = best[d];
        if (margin) margin[e] = mg;
    }
    return 0;
}

/* Dynamic decrease cap (A16): n_d >= N_d - cap. */
void orc_decrease_cap(int E, const int32_t* cur, int cap, int32_t* sel)
{
    for (int i = 0; i < 3 * E; ++i)
        if (sel[i] < cur[i] - cap) sel[i] = cur[i] - cap;
}

/* Jump condition fixpoint (eqs N23 / N_1): repeat
 * n_{e,d} <- min(Nmax, max(n_{e,d}, max_{j in N(e)} r(n_{j,d}))),
 * r(x) = floor(2x/3) (rule a) or x - 1 (rule b), neighbours = face
 * neighbours.  Jacobi sweeps until no change; returns the sweep count. */
int orc_jump_fixpoint(int E, const int32_t* nbr, int rule, int Nmax, int32_t* ord)
{
    int32_t* nxt = malloc(sizeof(int32_t) * 3 * E);
    int sweeps = 0;
    for (;;) {
        int changed = 0;
        for (int e = 0; e < E; ++e)
            for (int d = 0; d < 3; ++d) {
                int v = ord[3 * e + d];
                for (int f = 0; f < 6; ++f) {
                    int j = nbr[6 * e + f];
                    if (j < 0) continue;
                    int x = ord[3 * j + d];
                    int r = rule == ORC_JUMP_A ? (2 * x) / 3 : x - 1;
                    if (r > v) v = r;
                }
                if (v > Nmax) v = Nmax;
                if (v < ord[3 * e + d]) v = ord[3 * e + d];
                nxt[3 * e + d] = v;
                changed |= v != ord[3 * e + d];
            }
        memcpy(ord, nxt, sizeof(int32_t) * 3 * E);
        ++sweeps;
        if (!changed) break;
    }
    free(nxt);
    return sweeps;
}

/* ------------------------------------------------------------------------- */
/* 11. Solution transfer at adaptation: per-direction Lagrange
 *     interpolation from the old to the new nodes (reading A3).           */
/* ------------------------------------------------------------------------- */

int orc_transfer(int E, const int32_t* old_orders, const double* qold, const int32_t* new_orders, double* qnew, int ncomp)
{
    orc_init_basis();
    size_t* oo = make_offsets(E, old_orders, ncomp);
    size_t* on = make_offsets(E, new_orders, ncomp);
#pragma omp parallel for schedule(guided)
    for (int e = 0; e < E; ++e) {
        int A[3] = {old_orders[3 * e], old_orders[3 * e + 1], old_orders[3 * e + 2]};
        int B[3] = {new_orders[3 * e], new_orders[3 * e + 1], new_orders[3 * e + 2]};
        int n1[3] = {A[0] + 1, A[1] + 1, A[2] + 1};
        int n2[3] = {B[0] + 1, A[1] + 1, A[2] + 1};
        int n3[3] = {B[0] + 1, B[1] + 1, A[2] + 1};
        double* t1 = malloc(sizeof(double) * ncomp * n2[0] * n2[1] * n2[2]);
        double* t2 = malloc(sizeof(double) * ncomp * n3[0] * n3[1] * n3[2]);
        tapply(ncomp, qold + oo[e], n1, 0, Tm[A[0]][B[0]], B[0] + 1, t1);
        tapply(ncomp, t1, n2, 1, Tm[A[1]][B[1]], B[1] + 1, t2);
        tapply(ncomp, t2, n3, 2, Tm[A[2]][B[2]], B[2] + 1, qnew + on[e]);
        free(t1);
        free(t2);
    }
    free(oo);
    free(on);
    return 0;
}
