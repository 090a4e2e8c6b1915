// common.cuh -- shared device helpers and launch parameter structs of the
// sm_100a fp64 DGSEM / tau-estimation kernels.
//
// PAPER.md references: P:129-155 (DGSEM weak form, diagonal mass matrix),
// P:217-218 (isolated truncation error), P:225-241 (tau-estimation with the
// variational reference term), P:404-423 + P:461-463 (maps, approach 2,
// sentinel), P:472-475 (Roe flux, Williamson RK3, CFL step), P:511-520 (jump
// conditions), P:672 (decrease cap).  Readings A1-A25 are those of
// DESIGN.md / SURVEY.md 8(c).2.
//
// Formulation on the device: the strong form of the GL-DGSEM, which equals the
// weak form (eq DGSEMsystem:1) exactly for Gauss-Lobatto nodes (summation by
// parts, W D + D^T W = B):
//   Qdot_abc = -(1/J) sum_d [ sum_m D^{N_d}_{a_d m} Ft^d(..m..)
//               + (delta_{a_d N_d} (G^d_+ - Ft^d_+) - delta_{a_d 0} (G^d_- - Ft^d_-)) / w_{a_d} ].
// For the isolated variant G == Ft (own trace) so the surface term vanishes.
// Affine axis-aligned elements: Ja^d = (prod_{d'!=d} h_d'/2) e_d, J =
// prod h_d / 8, so Ft^d / J = (2/h_d) f_d.
#pragma once

#include <cstdint>

#include "basis.h"

namespace dgtau {

constexpr int NV = 5;
constexpr int BLOCK = 256;     // threads per CTA for the element kernels
constexpr int NPT = 3;         // nodes per thread (256 * 3 >= 729 = 9^3)
constexpr int MAXSLOTS = 32;   // elements per work item (n >= 8)
constexpr int DG_TAU_STRIDE_DEV = 9;  // tau[e][d][0..8]

struct PhysDev {
    double gamma, gm1;
    int flux;
    int physics;
    double mu, Pr;
    double qinf[5];
    double kappa;  // mu gamma / ((gamma - 1) Pr), formed once on the host
};

struct WorkItem {
    int start;  // index into elist
    int count;  // elements in this item (all with the same orders)
    int ord;    // N1 | N2 << 8 | N3 << 16
    int pad;
};

struct MortarItem {
    int L, R, d, pad;
};

__device__ __forceinline__ void unpack_ord(int ord, int& N1, int& N2, int& N3)
{
    N1 = ord & 255;
    N2 = (ord >> 8) & 255;
    N3 = (ord >> 16) & 255;
}

// ---------------------------------------------------------------------------
// Branch-free fp64 reciprocal / square root for positive normal arguments:
// MUFU seed (rcp/rsqrt.approx.ftz.f64) + Newton steps, within ~1 ulp (the
// IEEE-rounded library versions carry slow-path branches).
// ---------------------------------------------------------------------------

__device__ __forceinline__ double rcp_nr(double x)
{
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double e = fma(-x, y, 1.0);
    y = fma(y, e, y);
    e = fma(-x, y, 1.0);
    return fma(y, e, y);
}

#ifndef DG_FAST_DIV
#define DG_FAST_DIV 1
#endif
// 1/x of the face and viscous point fluxes: rcp_nr (branch-free, ~1 ulp) or IEEE
__device__ __forceinline__ double inv_pos(double x)
{
#if DG_FAST_DIV
    return rcp_nr(x);
#else
    return 1.0 / x;
#endif
}

__device__ __forceinline__ double rsqrt_nr(double x)
{
    double r;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    const double hx = 0.5 * x;
    r = r * fma(-hx * r, r, 1.5);
    return r * fma(-hx * r, r, 1.5);
}

__device__ __forceinline__ double sqrt_nr(double x)
{
    const double r = rsqrt_nr(x);
    const double s = x * r;
    return fma(0.5 * r, fma(-s, s, x), s);
}

// ---------------------------------------------------------------------------
// L2 eviction-priority hints.  Within an RK stage the new state q' is read
// again by the next stage's face and element kernels (keep: evict_last); the
// state read by the element kernel and the face flux blocks are dead after it
// (evict_first).  Pure hints: results do not depend on them.
// ---------------------------------------------------------------------------

__device__ __forceinline__ unsigned long long l2_policy_first()
{
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
    return p;
}

__device__ __forceinline__ unsigned long long l2_policy_last()
{
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
    return p;
}

__device__ __forceinline__ void st_hint(double* a, double v, unsigned long long pol)
{
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;\n" ::"l"(a), "d"(v), "l"(pol) : "memory");
}

__device__ __forceinline__ double ld_hint(const double* a, unsigned long long pol)
{
    double v;
    asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;\n" : "=d"(v) : "l"(a), "l"(pol));
    return v;
}

// ---------------------------------------------------------------------------
// Pointwise physics
// ---------------------------------------------------------------------------

// Euler flux in Cartesian direction d.  Returns pressure in *pout.
__device__ __forceinline__ void flux_dir(const double* q, double gm1, int d, double* f, double* pout)
{
    const double ir = 1.0 / q[0];
    const double p = gm1 * (q[4] - 0.5 * ir * (q[1] * q[1] + q[2] * q[2] + q[3] * q[3]));
    const double ud = q[1 + d] * ir;
    f[0] = q[1 + d];
    f[1] = q[1] * ud;
    f[2] = q[2] * ud;
    f[3] = q[3] * ud;
    f[1 + d] += p;
    f[4] = (q[4] + p) * ud;
    *pout = p;
}

// Roe approximate Riemann solver, closed form of the wave
// decomposition (acoustic waves u_n -/+ c, entropy + shear waves u_n),
// no entropy fix (reading A7).  n unit normal.
__device__ __forceinline__ void roe_flux(const double* qL, const double* qR, const double* n, double gamma,
                                         double* F)
{
    const double gm1 = gamma - 1.0;
    const double irL = inv_pos(qL[0]), irR = inv_pos(qR[0]);
    double uL[3], uR[3];
    for (int k = 0; k < 3; ++k) { uL[k] = qL[1 + k] * irL; uR[k] = qR[1 + k] * irR; }
    const double pL = gm1 * (qL[4] - 0.5 * qL[0] * (uL[0] * uL[0] + uL[1] * uL[1] + uL[2] * uL[2]));
    const double pR = gm1 * (qR[4] - 0.5 * qR[0] * (uR[0] * uR[0] + uR[1] * uR[1] + uR[2] * uR[2]));
    const double HL = (qL[4] + pL) * irL, HR = (qR[4] + pR) * irR;
    const double sL = sqrt(qL[0]), sR = sqrt(qR[0]);
    const double is = inv_pos(sL + sR);
    double u[3];
    for (int k = 0; k < 3; ++k) u[k] = (sL * uL[k] + sR * uR[k]) * is;
    const double H = (sL * HL + sR * HR) * is;
    const double uu = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
    const double c2 = gm1 * (H - 0.5 * uu);
    const double c = sqrt(c2);
    const double un = u[0] * n[0] + u[1] * n[1] + u[2] * n[2];
    const double unL = uL[0] * n[0] + uL[1] * n[1] + uL[2] * n[2];
    const double unR = uR[0] * n[0] + uR[1] * n[1] + uR[2] * n[2];
    const double rho = sL * sR;
    const double dr = qR[0] - qL[0], dp = pR - pL, dun = unR - unL;
    double du[3];
    for (int k = 0; k < 3; ++k) du[k] = uR[k] - uL[k];
    const double ic2 = inv_pos(c2);
    const double a1 = 0.5 * (dp - rho * c * dun) * ic2;
    const double a5 = 0.5 * (dp + rho * c * dun) * ic2;
    const double a2 = dr - dp * ic2;
    const double l1 = fabs(un - c), l2 = fabs(un), l5 = fabs(un + c);
    const double w1 = l1 * a1, w5 = l5 * a5;
    const double udu = u[0] * du[0] + u[1] * du[1] + u[2] * du[2];
    F[0] = 0.5 * (qL[0] * unL + qR[0] * unR) - 0.5 * (w1 + l2 * a2 + w5);
    for (int k = 0; k < 3; ++k) {
        const double fk = 0.5 * (qL[1 + k] * unL + pL * n[k] + qR[1 + k] * unR + pR * n[k]);
        const double dk = w1 * (u[k] - c * n[k]) + l2 * (a2 * u[k] + rho * (du[k] - dun * n[k])) +
                          w5 * (u[k] + c * n[k]);
        F[1 + k] = fk - 0.5 * dk;
    }
    const double fe = 0.5 * ((qL[4] + pL) * unL + (qR[4] + pR) * unR);
    const double de = w1 * (H - un * c) + l2 * (a2 * 0.5 * uu + rho * (udu - un * dun)) + w5 * (H + un * c);
    F[4] = fe - 0.5 * de;
}

// Local Lax-Friedrichs (flag, reading A7).
__device__ __forceinline__ void llf_flux(const double* qL, const double* qR, const double* n, double gamma,
                                         double* F)
{
    const double gm1 = gamma - 1.0;
    double fL[5], fR[5];
    const double irL = 1.0 / qL[0], irR = 1.0 / qR[0];
    const double pL = gm1 * (qL[4] - 0.5 * irL * (qL[1] * qL[1] + qL[2] * qL[2] + qL[3] * qL[3]));
    const double pR = gm1 * (qR[4] - 0.5 * irR * (qR[1] * qR[1] + qR[2] * qR[2] + qR[3] * qR[3]));
    const double unL = (qL[1] * n[0] + qL[2] * n[1] + qL[3] * n[2]) * irL;
    const double unR = (qR[1] * n[0] + qR[2] * n[1] + qR[3] * n[2]) * irR;
    fL[0] = qL[0] * unL; fR[0] = qR[0] * unR;
    for (int k = 0; k < 3; ++k) { fL[1 + k] = qL[1 + k] * unL + pL * n[k]; fR[1 + k] = qR[1 + k] * unR + pR * n[k]; }
    fL[4] = (qL[4] + pL) * unL; fR[4] = (qR[4] + pR) * unR;
    const double lam = fmax(fabs(unL) + sqrt(gamma * pL * irL), fabs(unR) + sqrt(gamma * pR * irR));
    for (int v = 0; v < 5; ++v) F[v] = 0.5 * (fL[v] + fR[v]) - 0.5 * lam * (qR[v] - qL[v]);
}

__device__ __forceinline__ void riemann(const double* qL, const double* qR, const double* n, const PhysDev& ph,
                                        double* F)
{
    if (ph.flux == 1) llf_flux(qL, qR, n, ph.gamma, F);
    else roe_flux(qL, qR, n, ph.gamma, F);
}

// Boundary ghost states (reading A10): wall = mirrored momentum, far field = q_inf.
__device__ __forceinline__ void ghost_state(const double* qin, int bc, const PhysDev& ph, double* qg)
{
    if (bc == -1) {
        qg[0] = qin[0]; qg[1] = -qin[1]; qg[2] = -qin[2]; qg[3] = -qin[3]; qg[4] = qin[4];
    } else {
        for (int v = 0; v < 5; ++v) qg[v] = ph.qinf[v];
    }
}

// ---------------------------------------------------------------------------
// Block reductions
// ---------------------------------------------------------------------------

__device__ __forceinline__ double warp_max(double v)
{
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// all threads receive the block max; uses red[32]
__device__ __forceinline__ double block_max(double v, double* red)
{
    v = warp_max(v);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    const int nw = (blockDim.x + 31) >> 5;
    double r = lane < nw ? red[lane] : 0.0;
    r = warp_max(r);
    return r;
}

// ---------------------------------------------------------------------------
// Residual launch parameters (generic and order-specialised kernels)
// ---------------------------------------------------------------------------

// Per element-face source of the outer state / flux (built by the host plan):
//   kind 0 conforming neighbour: trace value of variable v at own face point
//          (ta, tb) is q[off + v*n + base + ta*sa + tb*sb];
//   kind 1 mortar: projected Riemann flux at mortarG[off + v*n + pt];
//   kind 2 wall, kind 3 far field (ghost state from the own trace).
struct FaceInfo {
    long long off;
    int kind, n, base, sa, sb, pad;
};

// Per work-item slot: element id, state offset and the affine metric scales
// 2/h_d (so the kernels need one dependent load instead of three).
struct SlotInfo {
    long long off;
    int e, pad;
    double sc[3];
};

struct ResParams {
    const double* q;        // state read (neighbour traces come from here too)
    double* out;            // mode 0: qdot; mode 1: q_out = q + B g
    double* g;              // RK register (mode 1)
    const double* dt;       // device dt (mode 1)
    double rkA, rkB;
    int mode;
    int variant;            // 0 non-isolated, 1 isolated
    const int* orders;      // [E][3]
    const long long* off;   // [E+1]
    const int* nbr;         // [E][6]
    const double* hgeo;     // [E][3]
    const WorkItem* work;
    const int* elist;
    const double* mortarG;  // projected Riemann fluxes for mortar faces
    const long long* moff;  // [E][6] offset into mortarG or -1
    const FaceInfo* finfo;  // [E][6]
    const SlotInfo* slots;  // [elist length], parallel to elist
    const FaceInfo* finfo_slot;  // [elist length][6]: finfo of elist[i] (one dependent load less)
    const long long* fofs_slot;  // [elist length][6]: offset of each face's Riemann flux block in mortarG
    const Tables* tab;
    PhysDev ph;
    int* flag;              // [0] admissibility violations, [1] element id
    unsigned long long* lam_max;  // if set (last RK stage): max CFL rate of the NEW state (bits of a double >= 0)
    double gamma;
    long long qlen;         // doubles in the state buffer q (bulk copies never read past it)
    // fused step size (first stage of RK steps 2..n in dg_rk_steps): dt = cfl / *lam_in
    // (the CFL rate accumulated by the previous step's last stage, as k_dt_final);
    // CTA 0 of the launch stores dt to dt_out and zeroes *lam_zero (each if set)
    const unsigned long long* lam_in;
    double cfl;
    double* dt_out;
    unsigned long long* lam_zero;
};

// One conforming (or boundary) face, Riemann flux computed once per face
// point by k_face: L = the element on the -xi_d side (its +1 face), R = the
// element on the +xi_d side (its -1 face).  Trace of variable v at face point
// (ta, tb) of side X: q[offX + v*nX + baseX + ta*saX + tb*sbX].  Boundary
// faces (kind 2 wall, 3 far field) have off = -1 on the ghost side.  The flux
// (normal +e_d) of point pt = ta + nta*tb goes to G[goff + v*nf + pt].
struct FaceItem {
    long long offL, offR, goff;
    int nL, nR, baseL, baseR;
    int saL, sbL, saR, sbR;
    int nta, nf, d, kind;
};

// One mortar face for k_mortar3: state offsets of L (-xi_d side) and R, the
// offsets of the two projected flux blocks, packed orders N1 | N2 << 4 | N3 << 8.
struct MortarFace {
    long long offL, offR, moL, moR;
    int ordL, ordR, d, pad;
};

constexpr int FACE_BS = 128;   // k_face threads per CTA
constexpr int FACE_MINB = 5;   // k_face CTAs per SM (persistent grid)

struct FaceParams {
    const double* q;
    double* G;
    const FaceItem* faces;
    const int* fpt;    // [nfaces+1] point prefix
    const int4* fcta;  // [npts] {L trace index, R trace index (-1: ghost), flux index, nL | nR<<10 | d<<20 | kind<<22 | (nf-1)<<24}
    int npts;
    PhysDev ph;
};

__device__ __forceinline__ void node_ijk(int node, int n1, int n2, int& i, int& j, int& k)
{
    i = node % n1;
    const int r = node / n1;
    j = r % n2;
    k = r / n2;
}

}  // namespace dgtau
