/*
 * dgsem_oracle.h -- CPU oracle interface (TEST INFRASTRUCTURE ONLY; see
 * dgsem_oracle.c).  Not included by, and not linked into, the product.
 */
#ifndef DGSEM_ORACLE_H
#define DGSEM_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#define ORC_NMAX 16        /* basis tables for orders 1..16                 */
#define ORC_TAU_STRIDE 9   /* tau[e][d][0..8]; [0] = ||Qdot_ref,e||_inf     */
#define ORC_SENTINEL 1e30  /* "high value" for non-asymptotic data   */

enum { ORC_EULER = 0, ORC_NS = 1 };
enum { ORC_FLUX_ROE = 0, ORC_FLUX_LLF = 1 };
enum { ORC_NONISOLATED = 0, ORC_ISOLATED = 1 };
enum { ORC_TAU_NEW = 0, ORC_TAU_TRADITIONAL = 1 };
enum { ORC_JUMP_A = 0, ORC_JUMP_B = 1 };
enum { ORC_BC_WALL = -1, ORC_BC_FARFIELD = -2 };

typedef struct {
    double gamma;
    int physics; /* ORC_EULER | ORC_NS */
    int flux;    /* ORC_FLUX_ROE | ORC_FLUX_LLF */
    double mu, Pr;
    double qinf[5];
} orc_phys;

typedef struct {
    int E;
    const int32_t* nbr;    /* [E][6] */
    const int32_t* gorder; /* [3] geometry order per direction */
    const double* geo;     /* [E][3][(g3+1)(g2+1)(g1+1)] coordinates at GL nodes */
} orc_mesh;

void orc_init_basis(void);
int orc_basis(int N, double* x, double* w, double* D, double* Dhat, double* lm1, double* lp1);
int orc_interp_matrix(int Nf, int Nt, double* T);
int orc_projection_matrix(int M, int s, double* P);
void orc_euler_flux(const double* q, int k, double gam, double* f);
void orc_roe_flux(const double* qL, const double* qR, const double* n, double gam, double* F);
void orc_llf_flux(const double* qL, const double* qR, const double* n, double gam, double* F);
void orc_viscous_flux(const double* q, const double* g, int k, const orc_phys* ph, double* f);
int orc_rhs(const orc_mesh* m, const int32_t* orders, const double* q, int variant, const orc_phys* ph, double* qdot);
int orc_gradient(const orc_mesh* m, const int32_t* orders, const double* q, int variant, const orc_phys* ph, double* grad);
int orc_node_coords(const orc_mesh* m, const int32_t* orders, double* X);
int orc_mass(const orc_mesh* m, const int32_t* orders, double* M);
double orc_compute_dt(const orc_mesh* m, const int32_t* orders, const double* q, const orc_phys* ph, double cfl, double dfl);
int orc_rk3_step(const orc_mesh* m, const int32_t* orders, double* q, double dt, const orc_phys* ph);
int orc_tau_estimate(const orc_mesh* m, const int32_t* orders, const double* q, const double* qdot_ref,
                     int formulation, const orc_phys* ph, double* tau);
int orc_tau_estimate_r(const orc_mesh* m, const int32_t* orders, const double* q, const double* qdot_ref,
                       int formulation, int restriction, const orc_phys* ph, double* tau);
int orc_tau_field(const orc_mesh* m, const int32_t* orders, const double* q, const double* qdot_ref,
                  int e, int d, int p, int formulation, const orc_phys* ph, double* out);
int orc_build_map(int E, const int32_t* orders, const double* tau, int Nmin, int Nmax, double* map, double* slopes);
void orc_combine_max(size_t len, double* total, const double* map);
int orc_select_from_map(int E, const double* map, int Nmin, int Nmax, double tau_max, int32_t* out, double* margin);
void orc_decrease_cap(int E, const int32_t* cur, int cap, int32_t* sel);
int orc_jump_fixpoint(int E, const int32_t* nbr, int rule, int Nmax, int32_t* ord);
int orc_transfer(int E, const int32_t* old_orders, const double* qold, const int32_t* new_orders, double* qnew, int ncomp);

#endif
