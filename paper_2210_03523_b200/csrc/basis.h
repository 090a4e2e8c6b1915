// basis.h -- collocation tables for orders 1..8 (see basis.cpp).
#pragma once

namespace dgtau {

constexpr int NMAX = 8;
constexpr int NP = NMAX + 1;

// Flat, trivially copyable: uploaded once to device global memory.
struct Tables {
    double x[NP][NP];         // x[N][a]   Gauss-Lobatto nodes
    double w[NP][NP];         // w[N][a]   weights
    double D[NP][NP * NP];    // D[N][a*(N+1)+b] = l_b'(x_a)
    double T[NP][NP][NP * NP];  // T[Nf][Nt][i*(Nf+1)+a] = l^{Nf}_a(x^{Nt}_i)
    double P[NP][NP][NP * NP];  // P[M][s][a*(M+1)+m], exact L2 projection M -> s <= M
};

// hi + lo (double-double) copies of T and D, exact to the long double value:
// used only where geometry is differentiated (metric terms), whose rounding
// errors are amplified by D (reading: DESIGN.md "Metric accuracy").
struct TablesDD {
    double Thi[NP][NP][NP * NP], Tlo[NP][NP][NP * NP];
    double Dhi[NP][NP * NP], Dlo[NP][NP * NP];
};

void build_tables(Tables* t);
void build_tables_dd(TablesDD* t);

}  // namespace dgtau
