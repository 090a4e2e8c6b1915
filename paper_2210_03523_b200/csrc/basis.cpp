// basis.cpp -- host construction of the Gauss-Lobatto collocation tables that
// the sm_100a kernels read (L0 of the build).  PAPER.md P:67 (nodal DGSEM at
// Gauss(-Lobatto) nodes), P:130 (N+1-point quadrature), reading A2 (Gauss-
// Lobatto), A3 (interpolation as the restriction I), A6 (mortar L2
// projection).
//
// Independent of the CPU oracle: nodes by Newton on P_N'(x) with P_N'' from
// the Legendre ODE, differentiation and interpolation in barycentric form
// (negative-sum diagonal, so D 1 = 0 exactly), mortar projection via a
// Cholesky solve of the side mass matrix.
#include "basis.h"

#include <cmath>
#include <cstring>

namespace dgtau {

namespace {

// P_N(x) and P_N'(x) by the three-term recurrence, long double.
void legendre_and_derivative(int N, long double x, long double* P, long double* dP)
{
    long double p0 = 1.0L, p1 = x;
    long double d0 = 0.0L, d1 = 1.0L;
    if (N == 0) { *P = 1.0L; *dP = 0.0L; return; }
    for (int k = 2; k <= N; ++k) {
        long double p2 = ((2 * k - 1) * x * p1 - (k - 1) * p0) / k;
        long double d2 = d0 + (2 * k - 1) * p1;  // P_k' = P_{k-2}' + (2k-1) P_{k-1}
        p0 = p1; p1 = p2;
        d0 = d1; d1 = d2;
    }
    *P = p1;
    *dP = d1;
}

void lobatto(int N, long double* x, long double* w)
{
    const long double pi = 3.14159265358979323846264338327950288L;
    x[0] = -1.0L;
    x[N] = 1.0L;
    for (int j = 1; j < N; ++j) {
        long double t = -cosl(pi * j / N);
        for (int it = 0; it < 100; ++it) {
            long double P, dP;
            legendre_and_derivative(N, t, &P, &dP);
            // Legendre ODE: (1 - t^2) P'' = 2 t P' - N(N+1) P
            long double d2P = (2.0L * t * dP - N * (N + 1.0L) * P) / (1.0L - t * t);
            long double step = dP / d2P;
            t -= step;
            if (fabsl(step) < 1e-22L) break;
        }
        x[j] = t;
    }
    // enforce exact symmetry
    for (int j = 0; j <= N / 2; ++j) {
        long double s = 0.5L * (x[N - j] - x[j]);
        x[j] = -s;
        x[N - j] = s;
    }
    if (N % 2 == 0) x[N / 2] = 0.0L;
    for (int j = 0; j <= N; ++j) {
        long double P, dP;
        legendre_and_derivative(N, x[j], &P, &dP);
        w[j] = 2.0L / (N * (N + 1.0L) * P * P);
    }
}

void bary_weights(int N, const long double* x, long double* lam)
{
    for (int j = 0; j <= N; ++j) {
        long double p = 1.0L;
        for (int k = 0; k <= N; ++k)
            if (k != j) p *= (x[j] - x[k]);
        lam[j] = 1.0L / p;
    }
}

// value of the j-th Lagrange polynomial at y (barycentric, second form)
void bary_row(int N, const long double* x, const long double* lam, long double y, long double* row)
{
    for (int j = 0; j <= N; ++j)
        if (y == x[j]) {
            for (int k = 0; k <= N; ++k) row[k] = (k == j) ? 1.0L : 0.0L;
            return;
        }
    long double den = 0.0L;
    for (int j = 0; j <= N; ++j) den += lam[j] / (y - x[j]);
    for (int j = 0; j <= N; ++j) row[j] = (lam[j] / (y - x[j])) / den;
}

}  // namespace

void build_tables(Tables* t)
{
    std::memset(t, 0, sizeof(Tables));
    long double X[NMAX + 1][NMAX + 1], Wt[NMAX + 1][NMAX + 1], L[NMAX + 1][NMAX + 1];
    for (int N = 1; N <= NMAX; ++N) {
        lobatto(N, X[N], Wt[N]);
        bary_weights(N, X[N], L[N]);
        for (int a = 0; a <= N; ++a) {
            t->x[N][a] = (double)X[N][a];
            t->w[N][a] = (double)Wt[N][a];
        }
        // strong-form differentiation matrix D_ab = l_b'(x_a)
        for (int a = 0; a <= N; ++a) {
            long double diag = 0.0L;
            for (int b = 0; b <= N; ++b) {
                if (a == b) continue;
                long double v = (L[N][b] / L[N][a]) / (X[N][a] - X[N][b]);
                t->D[N][a * (N + 1) + b] = (double)v;
                diag -= v;
            }
            t->D[N][a * (N + 1) + a] = (double)diag;
        }
    }
    // interpolation T^{Nf->Nt}[i][a] = l^{Nf}_a(x^{Nt}_i)
    for (int Nf = 1; Nf <= NMAX; ++Nf)
        for (int Nt = 1; Nt <= NMAX; ++Nt)
            for (int i = 0; i <= Nt; ++i) {
                long double row[NMAX + 1];
                bary_row(Nf, X[Nf], L[Nf], X[Nt][i], row);
                for (int a = 0; a <= Nf; ++a) t->T[Nf][Nt][i * (Nf + 1) + a] = (double)row[a];
            }
    // mortar projection P^{M->s} = Ms^{-1} B, Ms = T^T W_M T (the exact side
    // mass matrix since s + s <= 2M - 1), B = T^T W_M, T = T^{s->M}.
    for (int M = 1; M <= NMAX; ++M)
        for (int s = 1; s <= M; ++s) {
            int ns = s + 1, nm = M + 1;
            long double Tsm[NMAX + 1][NMAX + 1];  // [i over M][a over s]
            for (int i = 0; i < nm; ++i) {
                long double row[NMAX + 1];
                bary_row(s, X[s], L[s], X[M][i], row);
                for (int a = 0; a < ns; ++a) Tsm[i][a] = row[a];
            }
            long double A[NMAX + 1][NMAX + 1], B[NMAX + 1][NMAX + 1];
            for (int a = 0; a < ns; ++a)
                for (int b = 0; b < ns; ++b) {
                    long double acc = 0.0L;
                    for (int i = 0; i < nm; ++i) acc += Tsm[i][a] * Wt[M][i] * Tsm[i][b];
                    A[a][b] = acc;
                }
            for (int a = 0; a < ns; ++a)
                for (int i = 0; i < nm; ++i) B[a][i] = Tsm[i][a] * Wt[M][i];
            // Cholesky A = C C^T
            long double C[NMAX + 1][NMAX + 1] = {};
            for (int r = 0; r < ns; ++r)
                for (int c = 0; c <= r; ++c) {
                    long double sum = A[r][c];
                    for (int k = 0; k < c; ++k) sum -= C[r][k] * C[c][k];
                    C[r][c] = (r == c) ? sqrtl(sum) : sum / C[c][c];
                }
            for (int i = 0; i < nm; ++i) {
                long double y[NMAX + 1], z[NMAX + 1];
                for (int r = 0; r < ns; ++r) {
                    long double sum = B[r][i];
                    for (int k = 0; k < r; ++k) sum -= C[r][k] * y[k];
                    y[r] = sum / C[r][r];
                }
                for (int r = ns - 1; r >= 0; --r) {
                    long double sum = y[r];
                    for (int k = r + 1; k < ns; ++k) sum -= C[k][r] * z[k];
                    z[r] = sum / C[r][r];
                }
                for (int a = 0; a < ns; ++a) t->P[M][s][a * nm + i] = (double)z[a];
            }
        }
}

void build_tables_dd(TablesDD* t)
{
    std::memset(t, 0, sizeof(TablesDD));
    long double X[NMAX + 1][NMAX + 1], Wt[NMAX + 1][NMAX + 1], L[NMAX + 1][NMAX + 1];
    for (int N = 1; N <= NMAX; ++N) {
        lobatto(N, X[N], Wt[N]);
        bary_weights(N, X[N], L[N]);
        for (int a = 0; a <= N; ++a) {
            long double diag = 0.0L;
            long double row[NMAX + 1];
            for (int b = 0; b <= N; ++b) {
                if (a == b) continue;
                row[b] = (L[N][b] / L[N][a]) / (X[N][a] - X[N][b]);
                diag -= row[b];
            }
            row[a] = diag;
            for (int b = 0; b <= N; ++b) {
                const double hi = (double)row[b];
                t->Dhi[N][a * (N + 1) + b] = hi;
                t->Dlo[N][a * (N + 1) + b] = (double)(row[b] - (long double)hi);
            }
        }
    }
    for (int Nf = 1; Nf <= NMAX; ++Nf)
        for (int Nt = 1; Nt <= NMAX; ++Nt)
            for (int i = 0; i <= Nt; ++i) {
                long double row[NMAX + 1];
                bary_row(Nf, X[Nf], L[Nf], X[Nt][i], row);
                for (int a = 0; a <= Nf; ++a) {
                    const double hi = (double)row[a];
                    t->Thi[Nf][Nt][i * (Nf + 1) + a] = hi;
                    t->Tlo[Nf][Nt][i * (Nf + 1) + a] = (double)(row[a] - (long double)hi);
                }
            }
}

}  // namespace dgtau
