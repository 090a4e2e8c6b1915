/*
 * dgtau.h -- C ABI of the B200 (sm_100a) hot path of tau-estimation-driven
 * anisotropic p-adaptation for the DGSEM (arXiv 2210.03523,
 * /root/reference/PAPER.md; "P:<n>" below = PAPER.md line n).
 *
 * Plain C types only.  Pointers named *_dev are CUDA device pointers owned by
 * the caller (e.g. torch tensors); pointers named *_host are host memory,
 * read (or written) during the call only.  `stream` is a cudaStream_t passed
 * as void*; every device call is stream-ordered on it and does not
 * synchronise it unless stated.  Every entry point returns a dg_status; on
 * error the context keeps a message readable with dg_last_error().  Nothing
 * aborts or throws across the ABI.
 *
 * Layouts (canonical, shared with the host):
 *   orders      int32 [E][3]        (N1,N2,N3) per element, 1 <= N_d <= 8
 *   state q     fp64  [e][v][k][j][i], elements back to back, v = (rho,
 *               rho u, rho v, rho w, E), node i fastest; element e starts at
 *               5 * sum_{e'<e} prod_d (N_d(e')+1)
 *   tau         fp64  [E][3][9]: tau[e][d][p] for 1 <= p <= N_d-1 (P:229:
 *               "estimated in all coarser meshes"), tau[e][d][0] =
 *               ||Qdot_ref,e||_inf (noise scale), other entries NaN
 *   neighbours  int32 [E][6], face f = 2d+s (d = xi,eta,zeta; s = 0 for the
 *               -1 side, 1 for the +1 side); >= 0 element id, -1 no-slip
 *               adiabatic wall, -2 far field
 *   geometry    fp64  [E][3][(g3+1)(g2+1)(g1+1)] coordinates of the
 *               geometry nodes (Gauss-Lobatto nodes of orders g)
 */
#ifndef DGTAU_H
#define DGTAU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    DG_OK = 0,
    DG_EINVAL = -1,       /* bad argument / size / order out of range           */
    DG_ENOMEM = -2,       /* device or host allocation failed                  */
    DG_ECUDA = -3,        /* CUDA runtime error (message has the CUDA text)    */
    DG_EADMISSIBLE = -5,  /* rho <= 0 or p <= 0 met (reading A25): the residual
                             kernels flag such nodes on the device; every call
                             that synchronises the stream (dg_compute_dt with a
                             host dt, dg_select_orders, dg_diagnostics) returns
                             this code with the first flagged element in
                             dg_last_error and clears the flag                */
    DG_ESTATE = -7,       /* call made before mesh / orders were set           */
    DG_EUNSUPPORTED = -8  /* geometry or physics not available in this build   */
} dg_status;

enum { DG_EULER = 0, DG_NS = 1 };
enum { DG_FLUX_ROE = 0, DG_FLUX_LLF = 1 };
enum { DG_NONISOLATED = 0, DG_ISOLATED = 1 };
enum { DG_TAU_NEW = 0, DG_TAU_TRADITIONAL = 1 };
enum { DG_REF_SOLVER = 0, DG_REF_SAME = 1 };
enum { DG_JUMP_A = 0, DG_JUMP_B = 1 };
enum { DG_SELECT_DYNAMIC = 0, DG_SELECT_STATIC_ACCUM = 1, DG_SELECT_STATIC_FINAL = 2,
       DG_SELECT_A1_ACCUM = 3, DG_SELECT_A1_FINAL = 4 };
enum { DG_COMBINE_MAX = 0, DG_COMBINE_AV = 1 };
enum { DG_PATH_AUTO = 0, DG_PATH_RUNTIME = 1, DG_PATH_BUCKETED = 2 };

#define DG_NMAX 8
#define DG_TAU_STRIDE 9

typedef struct dg_ctx dg_ctx;

/* Physics (readings A7-A10).  gamma ratio of specific heats; for
 * DG_NS mu = 1/Re, Pr, and qinf the far-field conserved state. */
typedef struct {
    int physics;   /* DG_EULER | DG_NS */
    int flux;      /* DG_FLUX_ROE | DG_FLUX_LLF (flag, A7) */
    double gamma;
    double mu, Pr;
    double qinf[5];
} dg_params;

/* tau-estimation options. */
typedef struct {
    int formulation; /* DG_TAU_NEW (eq TEtildedef) | DG_TAU_TRADITIONAL (eq TEdef) */
    int reference;   /* DG_REF_SOLVER: qdot_ref_dev is the non-isolated residual
                        -M^-1 F^N(q); DG_REF_SAME: the isolated
                        fine residual, computed in-kernel (reading A4) */
    int coarse_faces; /* 0 (default): ISOLATED coarse residuals, element-local
                        (the paper's choice P:469).  1: NON-ISOLATED
                        (reading R7): for direction d
                        and level p the whole mesh is taken at O(e) = N(e) with
                        O_d = min(p, N_d(e)); q and qdot_ref are interpolated per
                        direction (A3), the coarse residual couples the elements
                        through Roe faces / mortars (and BR1 for NS), and
                        tau[e][d][p] (p < N_d(e)) is the max of |T_d R - Qdot_c|.
                        Single rank only (DG_EUNSUPPORTED after dg_set_owned). */
    int restriction;  /* restriction of q and qdot_ref to the coarse orders along d:
                        0 (default) interpolation at the coarse nodes (reading A3,
                        P:165); 1 the exact L2 projection P^{N_d->p} (the A3 flag,
                        SURVEY 8(f) rank 4).  The coarse geometry is interpolated. */
} dg_tau_opts;

/* Order-selection policy (readings A13-A16). */
typedef struct {
    int mode;        /* DG_SELECT_DYNAMIC | _STATIC_ACCUM | _STATIC_FINAL */
    double tau_max;  /* threshold, strict "<" (Table 1 header)       */
    int Nmin, Nmax;  /* 1 <= Nmin <= Nmax <= 8                              */
    int jump_rule;   /* DG_JUMP_A (eq N23) | DG_JUMP_B (eq N_1)             */
    int dec_cap;     /* dynamic decrease cap per direction, >= 0    */
    int combine;     /* static stage combination F: DG_COMBINE_MAX (F_max,
                        the paper's choice) | DG_COMBINE_AV (F_av) */
    int nstages;     /* n_e, the number of estimation stages (F_av finals only) */
} dg_adapt_policy;

/* Create a context on the current CUDA device.  Returns DG_EINVAL for bad
 * parameters.  The context owns mesh tables, plans and basis tables. */
dg_status dg_create(const dg_params* params, dg_ctx** out);
void dg_destroy(dg_ctx* ctx);
const char* dg_last_error(const dg_ctx* ctx);

/* Kernel path of the residual (same discretisation, equal up to
 * rounding).  Two kernel families: the order-specialised kernels (affine Euler
 * only; one launch per (N1,N2,N3) bucket, replayed as a CUDA graph -- fastest
 * for uniform or few-bucket layouts) and the runtime-order kernels of the
 * curved path (element items of any orders in three size-class launches,
 * faces in three warp-width classes -- for many-bucket layouts, which dynamic
 * adaptation changes every few steps).  DG_PATH_AUTO (default):
 * curved meshes and NS take the runtime-order kernels; affine Euler layouts
 * are decided at every dg_set_orders by their bucket count (more than 24:
 * runtime-order).  DG_PATH_RUNTIME / DG_PATH_BUCKETED force one family
 * (BUCKETED: affine Euler only; curved meshes and NS still run the
 * runtime-order kernels).  Call before dg_mesh_upload (DG_ESTATE after it);
 * DG_EINVAL for an unknown path. */
dg_status dg_set_path(dg_ctx* ctx, int path);

/* Upload the mesh (copied).  gorder[3] geometry orders (1..4).  Elements
 * whose 8 geometry corners form an axis-aligned box are "affine"; others are
 * curved (metric terms from the geometry polynomial).  The local
 * axes of neighbours must be aligned (reading: SURVEY 8(c).1 step 2). */
dg_status dg_mesh_upload(dg_ctx* ctx, int E, const int32_t* nbr_host, const int32_t* gorder_host,
                         const double* geo_host);

/* Set the per-element orders (int32 [E][3], 1..8).  Builds offsets, the
 * (N1,N2,N3) bucket work list and the mortar face plan.  Synchronous. */
dg_status dg_set_orders(dg_ctx* ctx, const int32_t* orders_host);

/* Multi-rank local meshes: elements [0, n_owned) are owned (computed),
 * elements [n_owned, E) are halo copies of other ranks' elements whose state
 * the caller refreshes (one face-trace exchange per residual).
 * Neighbour code -3 marks "outside the local set" (allowed for halo elements
 * only).  Call after dg_mesh_upload and before dg_set_orders; default E. */
dg_status dg_set_owned(dg_ctx* ctx, int n_owned);

/* Number of doubles in a state vector for the current orders (5 * NDOF). */
int64_t dg_state_len(const dg_ctx* ctx);
/* NDOF = sum_e prod_d (N_d+1) over all local elements. */
int64_t dg_ndof(const dg_ctx* ctx);
/* Length (doubles) of the owned part of a state vector (owned elements first). */
int64_t dg_owned_state_len(const dg_ctx* ctx);

/* Node coordinates at the solution nodes, host [e][3][n] (for building
 * initial conditions).  Synchronous. */
dg_status dg_node_coords(dg_ctx* ctx, double* X_host);

/* Qdot = -(M^N)^-1 F^N(q)  (eq DGMassMatrixRight).  variant
 * DG_NONISOLATED uses the numerical fluxes at faces (mortars between unequal
 * orders, reading A6); DG_ISOLATED uses the inner trace flux.
 * The state pointer of the residual / RK calls must be 16-byte aligned (it is
 * read with 1-D bulk copies; cudaMalloc and torch allocations are), else
 * DG_EINVAL.  Non-isolated evaluations run k_mortar3 (mortar faces) and
 * k_face (conforming and boundary faces: each face point's Riemann flux once)
 * before the element kernels, all on `stream`. */
dg_status dg_rhs_eval(dg_ctx* ctx, int variant, const double* q_dev, double* qdot_dev, void* stream);

/* CFL time step (reading A11) from q, written to dt_dev[0]
 * (device, 1 double); if dt_host != NULL the stream is synchronised and the
 * value returned there too. */
dg_status dg_compute_dt(dg_ctx* ctx, const double* q_dev, double cfl, double* dt_dev, double* dt_host,
                        void* stream);

/* One Williamson low-storage RK3 step: for k = 1..3
 *   g <- A_k g + dt Qdot(q);  q <- q + B_k g.
 * q_in holds q^n on entry and is used as scratch; q_out receives q^{n+1};
 * g_dev is a register of the same length (no initialisation needed).
 * dt_dev: device pointer to dt (e.g. from dg_compute_dt); the step reads it
 * on the device, so no host synchronisation is needed. */
dg_status dg_rk_step(dg_ctx* ctx, double* q_in_dev, double* q_out_dev, double* g_dev, const double* dt_dev,
                     void* stream);

/* As dg_rk_step, and the CFL time step of the NEW state q^{n+1} (P:474-475,
 * reading A11) is reduced inside the last stage's kernel (no extra pass over
 * the state) and written to dt_next_dev[0] (device, != dt_dev). */
dg_status dg_rk_step_dt(dg_ctx* ctx, double* q_in_dev, double* q_out_dev, double* g_dev, const double* dt_dev,
                        double cfl, double* dt_next_dev, void* stream);

/* nsteps Williamson RK3 steps with the CFL step of each new state
 * fused into its last stage (reading A11): step s reads the state
 * from (s even ? qa : qb) and dt from (s even ? dt_a : dt_b), writes the new
 * state and the next dt into the other buffer of each pair, so after the call
 * the state is in (nsteps even ? qa : qb) and the next dt in (nsteps even ?
 * dt_a : dt_b).  Same kernels as nsteps dg_rk_step_dt calls, one host call.
 * Stream-ordered, no host sync. */
dg_status dg_rk_steps(dg_ctx* ctx, int nsteps, double* qa_dev, double* qb_dev, double* g_dev, double* dt_a_dev,
                      double* dt_b_dev, double cfl, void* stream);

/* One stage k in {0,1,2} of the Williamson RK3 step, for callers
 * that refresh halo states between stages: q_out = q_in + B_k g' with
 * g' = A_k g + dt Qdot(q_in) on owned elements.  If lam_accum_dev != NULL
 * (2 x uint64, zeroed, device) the CFL (and DFL) rates of q_out are
 * max-reduced into it (as bits of non-negative doubles, so an integer MAX
 * all-reduce across ranks is exact). */
dg_status dg_rk_stage(dg_ctx* ctx, int stage, const double* q_in_dev, double* q_out_dev, double* g_dev,
                      const double* dt_dev, unsigned long long* lam_accum_dev, int flags, void* stream);
/* flags for dg_rk_stage / dg_rhs_eval_flags: */
#define DG_FLAG_GRADIENT_READY 1 /* NS: skip the BR1 gradient pass; the caller ran dg_gradient
                                    and refreshed the halo rows of dg_gradient_buffer() */
/* Split face pass (the halo exchange overlapped with the faces
 * that do not touch it; runtime-order path only, non-isolated variant, NS with
 * DG_FLAG_GRADIENT_READY).  DG_FLAG_FACES_INTERIOR launches only the numerical
 * fluxes of the faces with no halo side and returns (nothing else runs); the
 * caller then completes the halo trace exchange on the same stream and calls
 * again with DG_FLAG_FACES_HALO and the same arguments: the faces with a halo
 * side, then the element kernel.  The pair is bit-identical to one call. */
#define DG_FLAG_FACES_INTERIOR 2
#define DG_FLAG_FACES_HALO 4
/* NS: BR1 gradient of q (eq DGSEMsystem:2) of the owned elements
 * into the context's gradient buffer (15 doubles per node, [k][v] = d q_v /
 * d x_k, element e at 3 x its state offset); the buffer's device pointer is
 * returned by dg_gradient_buffer() for halo exchange (owned by the context).
 * Every non-isolated residual, RK stage and tau-estimate (non-isolated coarse
 * levels included: their contexts borrow this buffer) overwrites it. */
dg_status dg_gradient(dg_ctx* ctx, int variant, const double* q_dev, void* stream);
/* dg_gradient with the split BR1 face pass (DG_FLAG_FACES_INTERIOR: only the
 * face states q^ of the faces without a halo side, nothing else; then
 * DG_FLAG_FACES_HALO after the state-trace exchange: the remaining faces and
 * the gradient kernel).  Non-isolated variant only. */
dg_status dg_gradient_flags(dg_ctx* ctx, int variant, const double* q_dev, int flags, void* stream);
double* dg_gradient_buffer(dg_ctx* ctx);
/* Non-isolated tau-estimation of ONE coarse level (d, p) on a rank-local mesh
 * (reading R7), in two phases.  phase 0:
 * builds the level's context (the local mesh at orders O = N with O_d =
 * min(p, N_d), owned count kept; once per layout, owned by ctx, returned in
 * *level_out), interpolates q_dev and qref_dev (the SOLVER reference) to it
 * and (NS) forms its BR1 gradient of the owned elements.  The caller then
 * refreshes the halo face traces of that gradient (dg_trace_copy on
 * *level_out, field = dg_gradient_buffer(*level_out), ncomp 15) -- the halo's
 * coarse STATE traces need no exchange (GL interpolation maps a face trace to
 * the coarse face trace alone).  phase 1: the level's face-coupled residual,
 * then tau[e][d][p] of the owned elements (tau_dev [E][3][9], o->formulation
 * and o->restriction as dg_tau_estimate).  Stream-ordered. */
dg_status dg_tau_level(dg_ctx* ctx, int d, int p, int phase, const dg_tau_opts* o, const double* q_dev,
                       const double* qref_dev, double* tau_dev, dg_ctx** level_out, void* stream);
/* Face-trace halo copies (north_star "face-trace halos"): the
 * face kernels read only the nodes of a neighbour's face toward an owned
 * element, so a rank exchanges partition-boundary face TRACES, not element
 * states.  entries_dev: int64 [n][2] device array, entry i = (offset into
 * buf_dev, 8 * local element id + face f), f = 2 d + s (s = 1: the +xi_d
 * face); field_dev: the state (ncomp = 5, element e at its state offset) or
 * the gradient buffer (ncomp = 15, at 3 x the offset); the trace of component
 * c at face point pt = ta + n_a tb is buf[offset + c * nf + pt] (nf = face
 * points).  direction 0 packs field -> buf, 1 unpacks buf -> the face nodes of
 * field.  Stream-ordered, no synchronisation; the caller owns every buffer
 * (partition.TracePlan builds the entries; dist.py posts the NCCL send/recv). */
dg_status dg_trace_copy(dg_ctx* ctx, const int64_t* entries_dev, int n, double* field_dev, int ncomp, double* buf_dev,
                        int direction, void* stream);
/* dg_rhs_eval with flags (DG_FLAG_GRADIENT_READY). */
dg_status dg_rhs_eval_flags(dg_ctx* ctx, int variant, const double* q_dev, double* qdot_dev, int flags, void* stream);
/* Max-reduce the CFL/DFL rates of q (owned elements) into lam_accum_dev. */
dg_status dg_dt_accumulate(dg_ctx* ctx, const double* q_dev, unsigned long long* lam_accum_dev, void* stream);
/* dt_dev[0] = min(cfl / lam, cfl / nu) from lam_accum_dev; resets it to 0. */
dg_status dg_dt_finalize(dg_ctx* ctx, unsigned long long* lam_accum_dev, double cfl, double* dt_dev, void* stream);

/* Batched tau-estimation over all coarse orders p < N_d of every element and
 * direction, isolated coarse residuals, in one launch.  qdot_ref_dev
 * is required for DG_REF_SOLVER and ignored for DG_REF_SAME.  tau_dev is
 * [E][3][9] (see layout). */
dg_status dg_tau_estimate(dg_ctx* ctx, const dg_tau_opts* opts, const double* q_dev, const double* qdot_ref_dev,
                          double* tau_dev, void* stream);

/* Order selection from tau.
 *   DYNAMIC:       map -> min-NDOF feasible -> decrease cap -> jump fixpoint
 *   STATIC_ACCUM:  total_map_dev <- max(total_map_dev, map)  (approach 2,
 *                  F_max, eq totalTruncMap); orders_out unchanged
 *   STATIC_FINAL:  as STATIC_ACCUM, then select on the total map -> jump
 *   (combine = F_av: the total map accumulates the sum of the stage maps and
 *   FINAL selects on sum / nstages)
 *   A1_ACCUM:      approach 1: select the min-NDOF feasible orders
 *                  of this stage's map (no decrease cap) and combine them into
 *                  total_map_dev[e][3]: F_max running max, F_av running sum
 *   A1_FINAL:      as A1_ACCUM, then orders = F(...) (F_av: the mean rounded
 *                  half up, reading R8; clamped to [Nmin, Nmax]) -> jump
 * total_map_dev: fp64 [E][K][K][K], K = Nmax-Nmin+1 (approach 1: [E][3]),
 * caller-owned, must be zero-filled before the first ACCUM (unused for
 * DYNAMIC, may be NULL).
 * orders_out_host: int32 [E][3] (written for DYNAMIC / STATIC_FINAL).
 * margin_host: optional fp64 [E], min |map - tau_max| / tau_max (parity aid).
 * Synchronises the stream. */
dg_status dg_select_orders(dg_ctx* ctx, const dg_adapt_policy* pol, const double* tau_dev, double* total_map_dev,
                           int32_t* orders_out_host, double* margin_host, void* stream);

/* Multi-rank selection pieces: map / min-NDOF / decrease cap for the owned
 * elements into orders_out_dev (int32 [E][3] device; halo rows = current
 * orders), and one Jacobi sweep of the jump fixpoint (eqs N23 / N_1) over
 * owned elements (halo rows copied through; *changed_dev |= 1 if any owned
 * order rose).  The caller exchanges halo rows and all-reduces `changed`. */
dg_status dg_select_local(dg_ctx* ctx, const dg_adapt_policy* pol, const double* tau_dev, double* total_map_dev,
                          int32_t* orders_out_dev, double* margin_dev, void* stream);
dg_status dg_jump_sweep(dg_ctx* ctx, const int32_t* orders_in_dev, int32_t* orders_out_dev, int rule, int Nmax,
                        int32_t* changed_dev, void* stream);

/* Project a state from the current orders to new_orders (P:299-301:
 * "the solution projected in the new polynomial spaces"; per-direction
 * Lagrange interpolation, reading A3).  q_new_dev must hold 5*NDOF(new)
 * doubles.  Does not change the context's orders: call dg_set_orders next. */
dg_status dg_transfer(dg_ctx* ctx, const int32_t* new_orders_host, const double* q_old_dev, double* q_new_dev,
                      void* stream);

/* Diagnostics: per-variable sum of M * v over all nodes (conservation check,
 * fp64 [5]) and min rho / min p of q; synchronises the stream. */
dg_status dg_diagnostics(dg_ctx* ctx, const double* q_dev, const double* v_dev, double* sums_host,
                         double* min_rho_p_host, void* stream);

/* Count of kernel launches issued by this context since creation (the bench
 * reports launches inside its timed region). */
int64_t dg_launch_count(const dg_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* DGTAU_H */
