// dgtau.cu -- C ABI (include/dgtau.h) and host-side plans of the B200 hot path.
//
// Host work is O(E) plan building only (offsets, (N1,N2,N3) bucket work list,
// mortar face list); every step of the numerical path runs in the kernels of
// kernels.cuh.  There is no CPU fallback: without a CUDA device every call
// returns DG_ECUDA.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <unordered_map>
#include <string>
#include <vector>

#include "../../include/dgtau.h"
#include "basis.h"
#include "kernels.cuh"
#include "residual_t.cuh"
#include "face.cuh"
#include "tau_t.cuh"
#include "curved.cuh"
#include "ns.cuh"

using namespace dgtau;

namespace dgtau {
cudaError_t res_setup_1(const Tables*, res_launcher (*)[NP][NP], res_occupancy (*)[NP][NP]);
cudaError_t res_setup_2(const Tables*, res_launcher (*)[NP][NP], res_occupancy (*)[NP][NP]);
cudaError_t res_setup_3(const Tables*, res_launcher (*)[NP][NP], res_occupancy (*)[NP][NP]);
cudaError_t res_setup_4(const Tables*, res_launcher (*)[NP][NP], res_occupancy (*)[NP][NP]);
cudaError_t res_setup_5(const Tables*, res_launcher (*)[NP][NP], res_occupancy (*)[NP][NP]);
cudaError_t res_setup_6(const Tables*, res_launcher (*)[NP][NP], res_occupancy (*)[NP][NP]);
cudaError_t res_setup_7(const Tables*, res_launcher (*)[NP][NP], res_occupancy (*)[NP][NP]);
cudaError_t res_setup_8(const Tables*, res_launcher (*)[NP][NP], res_occupancy (*)[NP][NP]);
}  // namespace dgtau

struct Bucket {
    int ord, item0, nitems;
    int start0, nelem, grid;  // elist start, element count, persistent grid size
};

struct GraphKey {
    int variant, mode;
    const void *q, *out, *g, *dt, *lam;
    double A, B;
    const void *lam_in, *dt_out, *lam_zero;
    double cfl;
    bool operator<(const GraphKey& o) const
    {
        if (lam_in != o.lam_in) return lam_in < o.lam_in;
        if (dt_out != o.dt_out) return dt_out < o.dt_out;
        if (lam_zero != o.lam_zero) return lam_zero < o.lam_zero;
        if (cfl != o.cfl) return cfl < o.cfl;
        if (variant != o.variant) return variant < o.variant;
        if (mode != o.mode) return mode < o.mode;
        if (q != o.q) return q < o.q;
        if (out != o.out) return out < o.out;
        if (g != o.g) return g < o.g;
        if (dt != o.dt) return dt < o.dt;
        if (lam != o.lam) return lam < o.lam;
        if (A != o.A) return A < o.A;
        return B < o.B;
    }
};

inline bool same_key(const GraphKey& a, const GraphKey& b) { return !(a < b) && !(b < a); }

// Launch shape of a residual graph: what the captured topology depends on.
// Buffer pointers, RK coefficients and the CFL number are re-pointed in the
// instantiated graph (cudaGraphExecKernelNodeSetParams, ~0.1 ms for 300
// kernels) instead of capturing + instantiating a graph per buffer pair.
struct ShapeKey {
    int variant, mode;
    bool lam, lam_in, dt_out, lam_zero;
    bool operator<(const ShapeKey& o) const
    {
        if (variant != o.variant) return variant < o.variant;
        if (mode != o.mode) return mode < o.mode;
        if (lam != o.lam) return lam < o.lam;
        if (lam_in != o.lam_in) return lam_in < o.lam_in;
        if (dt_out != o.dt_out) return dt_out < o.dt_out;
        return lam_zero < o.lam_zero;
    }
};

struct GraphEntry {
    cudaGraphExec_t exec = nullptr;
    cudaGraph_t graph = nullptr;           // kept: its kernel nodes hold the template arguments
    long long kernels = 0;                 // kernel launches recorded in the graph
    std::vector<cudaGraphNode_t> knodes;   // kernel nodes of `graph`
    GraphKey cur{};                        // arguments the exec currently carries
};

struct dg_ctx {
    std::string err;
    dg_params prm{};
    int device = 0;
    // mesh
    int E = 0;       // local elements: owned [0, n_own) then halo copies
    int n_own = 0;   // elements whose residual this context computes
    int gorder[3] = {1, 1, 1};
    std::vector<int> nbr;
    std::vector<double> geo;
    std::vector<double> h;  // affine box sizes [E][3]
    // orders / plans
    bool have_orders = false;
    std::vector<int> orders;
    std::vector<long long> off;
    long long ndof = 0;
    int nwork = 0;
    size_t res_smem = 0;
    int nmortar = 0;
    long long mortar_len = 0;
    int maxn = 0;
    // device
    Tables* d_tab = nullptr;
    TablesDD* d_tdd = nullptr;
    int* d_nbr = nullptr;
    double* d_h = nullptr;
    int* d_orders = nullptr;
    long long* d_off = nullptr;
    WorkItem* d_work = nullptr;
    int* d_elist = nullptr;
    MortarItem* d_mortar = nullptr;
    long long* d_moff = nullptr;
    FaceInfo* d_finfo = nullptr;
    SlotInfo* d_slots = nullptr;
    TauLevel* d_levels = nullptr;
    TauLevel* d_tgrp = nullptr;  // extruded meshes: level groups of one element (k_tau_grp)
    int ntgrp = 0, tgrp_cap = 0;
    // curved kernels run one CTA per element (level): elements sorted by node
    // count into size classes, each launched with its own dynamic shared memory
    int* d_eperm = nullptr;
    std::vector<SizeClass> ecls_own, ecls_all, lcls;
    TauGroup* d_tgroups = nullptr;  // k_tau5 (element, direction, level group) work list
    int ntgroups = 0;
    size_t tau5_smem = 0;
    int nlevels = 0;
    int max_level = 0;
    double* d_ref_scratch = nullptr;  // isolated fine residual for DG_REF_SAME
    // non-isolated tau-estimation (dg_tau_opts.coarse_faces): one sub-context
    // per coarse level (d, p) holding the whole mesh at that level's orders
    struct CoarseLevel {
        dg_ctx* sub = nullptr;
        int d = 0, p = 0, smax = 1;
        int* d_orders = nullptr;
        long long* d_off = nullptr;
    };
    std::vector<CoarseLevel> coarse;
    bool coarse_streaming = false;  // levels built / run / freed one at a time (device memory)
    bool coarse_stream_force = false;  // DGTAU_NONISO_STREAM=1 (tests)
    double* d_cq = nullptr;  // coarse q, T_d R, Qdot_c (fine length each)
    long long c_len = 0;
    int* d_tr_orders = nullptr;       // transfer scratch
    long long* d_tr_off = nullptr;
    std::vector<int> tr_orders_host;
    // curved geometry / Navier-Stokes
    bool curved = false;
    int smem_limit = 0;
    double* d_geo = nullptr;
    double* d_met = nullptr;       // 10 per node
    double* d_grad = nullptr;      // 15 per node (NS)
    long long met_len = 0, grad_len = 0;
    std::vector<long long> tr_off_host;
    long long ref_len = 0;
    double* d_mortarG = nullptr;
    unsigned long long* d_scratch = nullptr;  // [8]
    int* d_flag = nullptr;                    // [8]: [0..1] admissibility, [2] jump, [3] diag, [4] mortar queue
    int* d_sel = nullptr;                     // [2][E][3]
    double* d_margin = nullptr;               // [E]
    double* d_sums = nullptr;                 // [5]
    long long launches = 0;
    std::vector<Bucket> buckets;
    res_launcher rtab[NP][NP][NP] = {};
    res_occupancy rocc[NP][NP][NP] = {};
    signed char occ_cache[NP][NP][NP];  // resident k_res_t CTAs per SM, -1 = not queried yet
    int nsm = 148;
    FaceInfo* d_finfo_slot = nullptr;
    MortarFace* d_mfaces = nullptr;    // mortar faces (k_mortar3)
    long long* d_fofs_slot = nullptr;  // [elist][6] flux offset (into d_mortarG) of each face of each slot
    FaceItem* d_faces = nullptr;       // conforming + boundary faces (one Riemann flux per face point)
    int* d_fpt = nullptr;              // [nfaces+1] point prefix
    int4* d_fcta = nullptr;            // [nface_pts] per face point: trace indices, flux index, packed sizes
    int nfaces = 0, nfblk = 0;
    long long nface_pts = 0;
    static constexpr int NSTREAMS = 8;  // concurrent bucket launches for mixed-order layouts
    cudaStream_t side[NSTREAMS] = {};
    cudaEvent_t ev_fork = nullptr, ev_join[NSTREAMS] = {};
    bool no_graphs = false;  // DGTAU_NO_GRAPHS=1: launch mixed-order residuals directly
    cudaStream_t cap_stream = nullptr;  // graph capture stream
    std::map<ShapeKey, GraphEntry> graphs;  // mixed-order residual graphs of the current layout
    std::map<ShapeKey, int> direct_uses;    // direct launches per shape since the layout was set
    // curved residual path (ns.cuh): element items, face list, face blocks
    bool extruded = false;     // extruded mesh (compact metrics, structural zeros), see ns.cuh
    bool borrowed = false;     // coarse-level sub-context: scratch lent by the parent, never reallocated
    int path = DG_PATH_AUTO;   // dg_set_path
    bool affine_geo = false;   // axis-aligned box elements (h per element is exact)
    bool tau_curved = false;   // tau levels by k_tau_curved (else k_tau5, affine Euler)
    double* d_metc = nullptr;  // EXT: 6 per (i, j) column
    long long* d_coff = nullptr;
    NsItem* d_nsitems = nullptr;
    int* d_nselist = nullptr;
    std::vector<SizeClass> nscls;  // item classes by node count: [base, base + count), max nodes
    std::vector<int> nscls_swH, nscls_swG;  // per class: max stage words of an item (gradient / residual kernel)
    NsFace* d_nsfaces = nullptr;
    int nsf_cls[4] = {0, 0, 0, 0};  // faces of W = 1..3 warps: [nsf_cls[W-1], nsf_cls[W])
    int nsf_mid[4] = {0, 0, 0, 0};  // inside class W: faces with a halo side from nsf_mid[W] on
    double* d_fg = nullptr;         // face metrics at the mortar points
    double* d_nsG = nullptr;        // numerical-flux blocks (scratch per residual)
    double* d_nsH = nullptr;        // BR1 face-term blocks (scratch per residual)
    long long nsG_cap = 0, nsH_cap = 0;
    long long* d_fofsG = nullptr;   // [E][6] flux block of each element face
    long long* d_fofsH = nullptr;   // [E][6] BR1 block of each element face
};

namespace {

dg_status fail(dg_ctx* c, dg_status s, const std::string& msg)
{
    if (c) c->err = msg;
    return s;
}

dg_status cuda_check(dg_ctx* c, cudaError_t e, const char* what)
{
    if (e == cudaSuccess) return DG_OK;
    return fail(c, DG_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CK(expr)                                                       \
    do {                                                               \
        dg_status _s = cuda_check(ctx, (expr), #expr);                 \
        if (_s != DG_OK) return _s;                                    \
    } while (0)

inline std::mutex& dcap_mu();
inline std::unordered_map<const void*, size_t>& dcap();

template <class T>
void dfree(T*& p)
{
    if (p) {
        {
            std::lock_guard<std::mutex> lk(dcap_mu());
            dcap().erase(p);
        }
        cudaFree(p);
    }
    p = nullptr;
}

// Grow-only device buffers for the per-layout tables: a layout change
// (dg_set_orders, every adaptation) reuses the allocations instead of
// cudaFree (device-synchronising) + cudaMalloc for each of ~25 tables.
inline std::mutex& dcap_mu()
{
    static std::mutex* m = new std::mutex;  // never destroyed: contexts may be freed during process exit
    return *m;
}
inline std::unordered_map<const void*, size_t>& dcap()
{
    static auto* m = new std::unordered_map<const void*, size_t>;
    return *m;
}

template <class T>
cudaError_t dalloc(T*& p, size_t count)
{
    const size_t bytes = sizeof(T) * count;
    {
        std::lock_guard<std::mutex> lk(dcap_mu());
        auto it = p ? dcap().find(p) : dcap().end();
        if (it != dcap().end() && it->second >= bytes) return cudaSuccess;
        if (p) dcap().erase(p);
    }
    if (p) cudaFree(p);
    p = nullptr;
    // 25 % slack: the tables of successive adapted layouts differ a little in size
    const size_t cap = bytes + bytes / 4;
    cudaError_t e = cudaMalloc(&p, cap ? cap : 1);
    if (e != cudaSuccess) {
        p = nullptr;
        return e;
    }
    std::lock_guard<std::mutex> lk(dcap_mu());
    dcap()[p] = cap;
    return cudaSuccess;
}

template <class T>
cudaError_t upload(T*& d, const std::vector<T>& h)
{
    if (h.empty()) {
        dfree(d);
        return cudaSuccess;
    }
    cudaError_t e = dalloc(d, h.size());
    if (e != cudaSuccess) return e;
    return cudaMemcpy(d, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice);
}

PhysDev phys_dev(const dg_params& p)
{
    PhysDev ph;
    ph.gamma = p.gamma;
    ph.gm1 = p.gamma - 1.0;
    ph.flux = p.flux;
    ph.physics = p.physics;
    ph.mu = p.mu;
    ph.Pr = p.Pr;
    ph.kappa = p.mu * p.gamma / ((p.gamma - 1.0) * p.Pr);
    for (int v = 0; v < 5; ++v) ph.qinf[v] = p.qinf[v];
    return ph;
}

inline int npts(const int* N) { return (N[0] + 1) * (N[1] + 1) * (N[2] + 1); }

inline bool getenv_flag(const char* name)
{
    const char* g = getenv(name);
    return g && g[0] == '1';
}

// pipeline depth of the NS element kernels (DGTAU_NS_NST=1..4 for A/B; default 2)
inline int ns_stages()
{
    const char* g = getenv("DGTAU_NS_NST");
    const int v = g ? atoi(g) : 2;
    return v < 1 ? 1 : (v > NS_MAXST ? NS_MAXST : v);
}

// DG_PATH_AUTO on affine Euler meshes: layouts with more (N1,N2,N3) buckets
// than this take the runtime-order kernels (profiles/r02_prof_adapt_n32.txt:
// 343 buckets, 1.54 -> 1.15 ms per residual; uniform orders stay 2.2x faster
// on the order-specialised kernels)
constexpr int RT_BUCKETS = 24;

// DGTAU_TIMING=1: host-side section times of dg_set_orders on stderr (device
// work synchronised at each mark)
struct PlanTimer {
    bool on;
    std::chrono::steady_clock::time_point t;
    PlanTimer() : on(getenv_flag("DGTAU_TIMING")), t(std::chrono::steady_clock::now()) {}
    void mark(const char* what)
    {
        if (!on) return;
        cudaDeviceSynchronize();
        const auto n = std::chrono::steady_clock::now();
        fprintf(stderr, "[set_orders] %-28s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(n - t).count());
        t = n;
    }
};

dg_status check_stream_error(dg_ctx* ctx, const char* what)
{
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(ctx, DG_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
    return DG_OK;
}

// Admissibility (reading A25): the residual kernels count nodes with rho <= 0
// or p <= 0 in d_flag[0] (first flagged element in d_flag[1]).  Every call
// that synchronises the stream reads it and fails with DG_EADMISSIBLE (the
// flag is reset so the caller can recover).
dg_status admissibility(dg_ctx* ctx, cudaStream_t st)
{
    int flag[2] = {0, 0};
    cudaError_t e = cudaMemcpyAsync(flag, ctx->d_flag, sizeof(flag), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return fail(ctx, DG_ECUDA, std::string("admissibility flag: ") + cudaGetErrorString(e));
    if (flag[0] > 0) {
        cudaMemsetAsync(ctx->d_flag, 0, 2 * sizeof(int), st);
        return fail(ctx, DG_EADMISSIBLE, "inadmissible state (rho <= 0 or p <= 0) at " + std::to_string(flag[0]) +
                                             " node evaluations since the last check; first flagged element " +
                                             std::to_string(flag[1]));
    }
    return DG_OK;
}

// Gauss-Lobatto nodes of the geometry orders, for evaluating node coordinates.
const Tables& host_tables()
{
    static Tables* t = nullptr;
    if (!t) {
        t = new Tables;
        build_tables(t);
    }
    return *t;
}

CurvedMesh curved_mesh(const dg_ctx* ctx)
{
    CurvedMesh cm;
    cm.geo = ctx->d_geo;
    cm.g1 = ctx->gorder[0];
    cm.g2 = ctx->gorder[1];
    cm.g3 = ctx->gorder[2];
    cm.ng = (cm.g1 + 1) * (cm.g2 + 1) * (cm.g3 + 1);
    return cm;
}

const TablesDD& host_tables_dd()
{
    static TablesDD* t = nullptr;
    if (!t) {
        t = new TablesDD;
        build_tables_dd(t);
    }
    return *t;
}

}  // namespace

extern "C" {

dg_status dg_create(const dg_params* params, dg_ctx** out)
{
    if (!params || !out) return DG_EINVAL;
    *out = nullptr;
    if (!(params->gamma > 1.0)) return DG_EINVAL;
    if (params->physics != DG_EULER && params->physics != DG_NS) return DG_EINVAL;
    if (params->flux != DG_FLUX_ROE && params->flux != DG_FLUX_LLF) return DG_EINVAL;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return DG_ECUDA;
    dg_ctx* ctx = new dg_ctx;
    std::memset(ctx->occ_cache, -1, sizeof(ctx->occ_cache));
    ctx->prm = *params;
    cudaGetDevice(&ctx->device);
    cudaDeviceGetAttribute(&ctx->nsm, cudaDevAttrMultiProcessorCount, ctx->device);
    const Tables& t = host_tables();
    dg_status s;
    if ((s = cuda_check(ctx, cudaMalloc(&ctx->d_tab, sizeof(Tables)), "cudaMalloc tables")) != DG_OK ||
        (s = cuda_check(ctx, cudaMemcpy(ctx->d_tab, &t, sizeof(Tables), cudaMemcpyHostToDevice), "tables")) != DG_OK ||
        (s = cuda_check(ctx, cudaMalloc(&ctx->d_scratch, 8 * sizeof(unsigned long long)), "scratch")) != DG_OK ||
        (s = cuda_check(ctx, cudaMemset(ctx->d_scratch, 0, 8 * sizeof(unsigned long long)), "scratch")) != DG_OK ||
        (s = cuda_check(ctx, cudaMalloc(&ctx->d_flag, 8 * sizeof(int)), "flag")) != DG_OK ||
        (s = cuda_check(ctx, cudaMemset(ctx->d_flag, 0, 8 * sizeof(int)), "flag")) != DG_OK ||
        (s = cuda_check(ctx, cudaMalloc(&ctx->d_sums, 8 * sizeof(double)), "sums")) != DG_OK ||
        (s = cuda_check(ctx, cudaMalloc(&ctx->d_tdd, sizeof(TablesDD)), "dd tables")) != DG_OK ||
        (s = cuda_check(ctx, cudaMemcpy(ctx->d_tdd, &host_tables_dd(), sizeof(TablesDD), cudaMemcpyHostToDevice),
                        "dd tables")) != DG_OK) {
        dg_destroy(ctx);
        return s;
    }
    {
        typedef cudaError_t (*setup_fn)(const Tables*, res_launcher (*)[NP][NP], res_occupancy (*)[NP][NP]);
        const setup_fn fns[8] = {res_setup_1, res_setup_2, res_setup_3, res_setup_4,
                                 res_setup_5, res_setup_6, res_setup_7, res_setup_8};
        for (int i = 0; i < 8; ++i)
            if ((s = cuda_check(ctx, fns[i](&t, ctx->rtab, ctx->rocc), "residual setup")) != DG_OK) {
                dg_destroy(ctx);
                return s;
            }
        {
            std::vector<double> mop;
            mortar_build_ops(&t, mop);
            if ((s = cuda_check(ctx, cudaMemcpyToSymbol(c_mop, mop.data(), sizeof(double) * mop.size()), "mortar operators")) != DG_OK) {
                dg_destroy(ctx);
                return s;
            }
        }
        if ((s = cuda_check(ctx, res_copy_constants(&t), "constants")) != DG_OK ||
            (s = cuda_check(ctx, ns_copy_constants(), "constants")) != DG_OK) {
            dg_destroy(ctx);
            return s;
        }
        for (int i = 0; i < dg_ctx::NSTREAMS && s == DG_OK; ++i) {
            s = cuda_check(ctx, cudaStreamCreateWithFlags(&ctx->side[i], cudaStreamNonBlocking), "side stream");
            if (s == DG_OK) s = cuda_check(ctx, cudaEventCreateWithFlags(&ctx->ev_join[i], cudaEventDisableTiming), "event");
        }
        if (s == DG_OK) s = cuda_check(ctx, cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming), "event");
        if (s != DG_OK) {
            dg_destroy(ctx);
            return s;
        }
        ctx->no_graphs = getenv_flag("DGTAU_NO_GRAPHS");
        ctx->coarse_stream_force = getenv_flag("DGTAU_NONISO_STREAM");
        if ((s = cuda_check(ctx, cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking), "capture stream")) !=
            DG_OK) {
            dg_destroy(ctx);
            return s;
        }
    }
    // large dynamic shared memory for the element kernels (opt-in limit minus static smem)
    {
        int optin = 0;
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device);
        const int lim = optin - 1024;  // headroom for static shared arrays
        cudaFuncSetAttribute(k_tau5, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - 4096);  // 3.1 KB static
        cudaFuncSetAttribute(k_tau5, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared);
        cudaFuncSetAttribute(k_transfer, cudaFuncAttributeMaxDynamicSharedMemorySize, std::min(200 * 1024, lim));
        const int limc = optin - 8192;  // curved kernels: up to ~6 KB static (staged D, reductions)
        cudaFuncSetAttribute(k_metrics, cudaFuncAttributeMaxDynamicSharedMemorySize, limc);
        cudaFuncSetAttribute(k_tau_curved<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, limc);
        cudaFuncSetAttribute(k_tau_curved<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, limc);
        cudaFuncSetAttribute(k_tau_curved<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, limc);
        cudaFuncSetAttribute(k_tau_ext<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, limc);
        cudaFuncSetAttribute(k_tau_grp, cudaFuncAttributeMaxDynamicSharedMemorySize, limc);
        cudaFuncSetAttribute(k_tau_ext<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, limc);
        cudaFuncSetAttribute(k_tau_ext<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, limc);
        ctx->smem_limit = limc;
        // curved residual path (ns.cuh): element kernels up to 20 x 729 doubles, face kernels per W
        const int lns = limc;
        cudaFuncSetAttribute(k_ns_grad<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, lns);
        cudaFuncSetAttribute(k_ns_grad<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, lns);
        cudaFuncSetAttribute(k_ns_res<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, lns);
        cudaFuncSetAttribute(k_ns_res<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, lns);
        cudaFuncSetAttribute(k_ns_res<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, lns);
        cudaFuncSetAttribute(k_ns_res<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, lns);
#define NSF_ATTR(W)                                                                                                   \
    cudaFuncSetAttribute(k_ns_face<W, MODE_QHAT>, cudaFuncAttributeMaxDynamicSharedMemorySize,                          \
                         (int)FaceCfg<W, MODE_QHAT>::smem);                                                             \
    cudaFuncSetAttribute(k_ns_face<W, MODE_FLUX_EULER>, cudaFuncAttributeMaxDynamicSharedMemorySize,                    \
                         (int)FaceCfg<W, MODE_FLUX_EULER>::smem);                                                       \
    cudaFuncSetAttribute(k_ns_face<W, MODE_FLUX_NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FaceCfg<W>::smem);
        NSF_ATTR(1)
        NSF_ATTR(2)
        NSF_ATTR(3)
#undef NSF_ATTR
        cudaError_t e = cudaGetLastError();  // attribute errors are fatal here, not stale later
        if (e != cudaSuccess) {
            s = cuda_check(ctx, e, "cudaFuncSetAttribute");
            dg_destroy(ctx);
            return s;
        }
    }
    *out = ctx;
    return DG_OK;
}

static void drop_graphs(dg_ctx* ctx)
{
    for (auto& kv : ctx->graphs) {
        cudaGraphExecDestroy(kv.second.exec);
        cudaGraphDestroy(kv.second.graph);
    }
    ctx->graphs.clear();
    ctx->direct_uses.clear();
}

// Coarse-level contexts borrow the fine context's residual scratch (BR1
// gradient, mortar / face flux buffers): the levels run one after another on
// the caller's stream and every coarse layout needs no more than the fine one
// (fewer nodes; mortars only where the fine layout has them, with smaller
// blocks).  Detach before destroying a level so the scratch stays the parent's.
// Coarse-level sub-contexts (non-isolated tau) borrow the parent's per-residual
// scratch: the gradient and the face blocks.  A borrowing context never
// reallocates them (dg_set_orders fails loudly if a coarse layout needed more
// than the fine one lent -- it cannot: every coarse order is <= the fine one).
static void lend_scratch(dg_ctx* parent, dg_ctx* sub)
{
    sub->borrowed = true;
    sub->d_grad = parent->d_grad;
    sub->grad_len = parent->grad_len;
    sub->d_nsG = parent->d_nsG;
    sub->nsG_cap = parent->nsG_cap;
    sub->d_nsH = parent->d_nsH;
    sub->nsH_cap = parent->nsH_cap;
}

static void unlend_scratch(dg_ctx* parent, dg_ctx* sub)
{
    if (!sub) return;
    if (sub->d_grad == parent->d_grad) sub->d_grad = nullptr;
    if (sub->d_nsG == parent->d_nsG) sub->d_nsG = nullptr;
    if (sub->d_nsH == parent->d_nsH) sub->d_nsH = nullptr;
}

static void drop_coarse(dg_ctx* ctx)
{
    for (auto& L : ctx->coarse) {
        unlend_scratch(ctx, L.sub);
        dg_destroy(L.sub);
        L.sub = nullptr;
        dfree(L.d_orders);
        dfree(L.d_off);
    }
    ctx->coarse.clear();
}

void dg_destroy(dg_ctx* ctx)
{
    if (!ctx) return;
    drop_coarse(ctx);
    dfree(ctx->d_cq);
    drop_graphs(ctx);
    if (ctx->cap_stream) cudaStreamDestroy(ctx->cap_stream);
    for (int i = 0; i < dg_ctx::NSTREAMS; ++i) {
        if (ctx->side[i]) cudaStreamDestroy(ctx->side[i]);
        if (ctx->ev_join[i]) cudaEventDestroy(ctx->ev_join[i]);
    }
    if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
    dfree(ctx->d_tab);
    dfree(ctx->d_tdd);
    dfree(ctx->d_nbr);
    dfree(ctx->d_h);
    dfree(ctx->d_orders);
    dfree(ctx->d_off);
    dfree(ctx->d_work);
    dfree(ctx->d_elist);
    dfree(ctx->d_mortar);
    dfree(ctx->d_moff);
    dfree(ctx->d_finfo);
    dfree(ctx->d_finfo_slot);
    dfree(ctx->d_fofs_slot);
    dfree(ctx->d_mfaces);
    dfree(ctx->d_faces);
    dfree(ctx->d_fpt);
    dfree(ctx->d_fcta);
    dfree(ctx->d_slots);
    dfree(ctx->d_levels);
    dfree(ctx->d_tgrp);
    dfree(ctx->d_eperm);
    dfree(ctx->d_tgroups);
    dfree(ctx->d_ref_scratch);
    dfree(ctx->d_tr_orders);
    dfree(ctx->d_geo);
    dfree(ctx->d_met);
    dfree(ctx->d_grad);
    dfree(ctx->d_tr_off);
    dfree(ctx->d_mortarG);
    dfree(ctx->d_metc);
    dfree(ctx->d_coff);
    dfree(ctx->d_nsitems);
    dfree(ctx->d_nselist);
    dfree(ctx->d_nsfaces);
    dfree(ctx->d_fg);
    dfree(ctx->d_nsG);
    dfree(ctx->d_nsH);
    dfree(ctx->d_fofsG);
    dfree(ctx->d_fofsH);
    dfree(ctx->d_scratch);
    dfree(ctx->d_flag);
    dfree(ctx->d_sel);
    dfree(ctx->d_margin);
    dfree(ctx->d_sums);
    delete ctx;
}

const char* dg_last_error(const dg_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int64_t dg_launch_count(const dg_ctx* ctx) { return ctx ? ctx->launches : 0; }

dg_status dg_set_path(dg_ctx* ctx, int path)
{
    if (!ctx) return DG_EINVAL;
    if (path != DG_PATH_AUTO && path != DG_PATH_RUNTIME && path != DG_PATH_BUCKETED)
        return fail(ctx, DG_EINVAL, "set_path: unknown path");
    if (ctx->E != 0) return fail(ctx, DG_ESTATE, "set_path: call before dg_mesh_upload");
    ctx->path = path;
    return DG_OK;
}

dg_status dg_mesh_upload(dg_ctx* ctx, int E, const int32_t* nbr_host, const int32_t* gorder_host, const double* geo_host)
{
    if (!ctx) return DG_EINVAL;
    if (E <= 0 || !nbr_host || !gorder_host || !geo_host) return fail(ctx, DG_EINVAL, "mesh: bad arguments");
    for (int d = 0; d < 3; ++d)
        if (gorder_host[d] < 1 || gorder_host[d] > NMAX) return fail(ctx, DG_EINVAL, "mesh: geometry order out of range");
    for (long long i = 0; i < 6LL * E; ++i)
        if (nbr_host[i] >= E || nbr_host[i] < -3) return fail(ctx, DG_EINVAL, "mesh: neighbour id out of range");
    // aligned-axes check: e's face f neighbour must see e across the opposite face
    for (int e = 0; e < E; ++e)
        for (int f = 0; f < 6; ++f) {
            int nb = nbr_host[6 * e + f];
            if (nb >= 0 && nbr_host[6 * nb + (f ^ 1)] != e && nbr_host[6 * nb + (f ^ 1)] != -3)
                return fail(ctx, DG_EINVAL, "mesh: neighbour local axes not aligned (face " + std::to_string(f) +
                                                " of element " + std::to_string(e) + ")");
        }
    ctx->E = E;
    ctx->n_own = E;
    for (int d = 0; d < 3; ++d) ctx->gorder[d] = gorder_host[d];
    const int ng = (gorder_host[0] + 1) * (gorder_host[1] + 1) * (gorder_host[2] + 1);
    ctx->nbr.assign(nbr_host, nbr_host + 6LL * E);
    ctx->geo.assign(geo_host, geo_host + 3LL * ng * E);
    // affine detection: geometry order (1,1,1), corners of an axis-aligned box
    ctx->h.assign(3LL * E, 0.0);
    bool affine = gorder_host[0] == 1 && gorder_host[1] == 1 && gorder_host[2] == 1;
    for (int e = 0; e < E && affine; ++e) {
        const double* G = geo_host + 3LL * ng * e;
        for (int c = 0; c < 3; ++c) {
            const double lo = G[c * 8 + 0];
            const double hi = G[c * 8 + (c == 0 ? 1 : (c == 1 ? 2 : 4))];
            for (int k = 0; k < 8; ++k) {
                const int bit = (k >> c) & 1;
                const double want = bit ? hi : lo;
                if (G[c * 8 + k] != want) affine = false;
            }
            ctx->h[3LL * e + c] = hi - lo;
            if (!(hi > lo)) affine = false;
        }
    }
    // kernel path (dg_set_path): curved meshes and NS take the runtime-order
    // kernels; affine Euler meshes are decided per layout in dg_set_orders
    // (AUTO: runtime-order kernels when the layout has many (N1,N2,N3) buckets)
    ctx->affine_geo = affine;
    ctx->curved = !affine || ctx->path == DG_PATH_RUNTIME || ctx->prm.physics == DG_NS;
    ctx->tau_curved = ctx->curved && !(affine && ctx->prm.physics == DG_EULER);
    // extruded mesh (ns.cuh): linear in zeta, x and y independent of zeta, z
    // independent of xi and eta and increasing with zeta
    bool ext = gorder_host[2] == 1 && !getenv_flag("DGTAU_NO_EXT");
    {
        const int L2 = (gorder_host[0] + 1) * (gorder_host[1] + 1);
        for (int e = 0; e < E && ext; ++e) {
            const double* G = geo_host + 3LL * ng * e;
            for (int ab = 0; ab < L2 && ext; ++ab) {
                if (G[ab] != G[ab + L2] || G[ng + ab] != G[ng + ab + L2]) ext = false;
                if (G[2 * ng + ab] != G[2 * ng] || G[2 * ng + L2 + ab] != G[2 * ng + L2]) ext = false;
            }
            if (!(G[2 * ng + L2] > G[2 * ng])) ext = false;
        }
    }
    ctx->extruded = ext;
    if (!affine)
        for (long long i = 0; i < 3LL * E; ++i) ctx->h[i] = 1.0;  // unused by the curved kernels
    CK(upload(ctx->d_geo, ctx->geo));  // (affine layouts may take the runtime-order kernels too)
    CK(upload(ctx->d_nbr, ctx->nbr));
    CK(upload(ctx->d_h, ctx->h));
    ctx->have_orders = false;
    return DG_OK;
}

// Sort idx[begin,end) by size (largest first) and cut it into classes whose
// largest member sets the class's shared-memory size (class edges ~ x1.25-1.5).
static void size_classes(std::vector<int>& idx, const std::vector<int>& sz, int begin, int end,
                         std::vector<SizeClass>& out)
{
    static const int edge[] = {16, 32, 48, 64, 80, 96, 128, 160, 192, 256, 320, 384, 512, 640, 1 << 30};
    auto cls = [](int n) { int c = 0; while (n > edge[c]) ++c; return c; };
    {  // stable sort by decreasing size: counting sort, O(n + max size)
        int smax = 0;
        for (int i = begin; i < end; ++i) smax = std::max(smax, sz[idx[i]]);
        std::vector<int> cnt(smax + 2, 0);
        for (int i = begin; i < end; ++i) ++cnt[smax - sz[idx[i]] + 1];
        for (int k = 0; k <= smax; ++k) cnt[k + 1] += cnt[k];
        std::vector<int> tmp(end - begin);
        for (int i = begin; i < end; ++i) tmp[cnt[smax - sz[idx[i]]]++] = idx[i];
        std::copy(tmp.begin(), tmp.end(), idx.begin() + begin);
    }
    for (int i = begin; i < end;) {
        const int c = cls(sz[idx[i]]);
        int j = i;
        while (j < end && cls(sz[idx[j]]) == c) ++j;
        out.push_back(SizeClass{i, j - i, sz[idx[i]]});
        i = j;
    }
}

// Elements [begin, end) grouped by their order triple, groups in increasing
// (N3, N2, N1) and element ids increasing inside (counting sort, O(E)).
static void order_buckets(const std::vector<int>& orders, int begin, int end, std::vector<int>& keys,
                          std::vector<int>& start, std::vector<int>& elems)
{
    constexpr int NK = NMAX * NMAX * NMAX;
    std::vector<int> cnt(NK + 1, 0);
    auto key = [&](int e) {
        const int* N = &orders[3 * e];
        return (N[0] - 1) + NMAX * ((N[1] - 1) + NMAX * (N[2] - 1));
    };
    for (int e = begin; e < end; ++e) ++cnt[key(e) + 1];
    for (int k = 0; k < NK; ++k) cnt[k + 1] += cnt[k];
    elems.resize(end - begin);
    std::vector<int> pos(cnt.begin(), cnt.end() - 1);
    for (int e = begin; e < end; ++e) elems[pos[key(e)]++] = e;
    keys.clear();
    start.clear();
    for (int k = 0; k < NK; ++k)
        if (cnt[k + 1] > cnt[k]) {
            keys.push_back(((k % NMAX) + 1) | (((k / NMAX) % NMAX + 1) << 8) | ((k / (NMAX * NMAX) + 1) << 16));
            start.push_back(cnt[k]);
        }
    start.push_back(end - begin);
}

// Scratch that a borrowing (coarse-level) context must not reallocate.
static dg_status scratch_need(dg_ctx* ctx, double*& p, long long& cap, long long need, const char* what)
{
    if (need <= cap && p) return DG_OK;
    if (need == 0) return DG_OK;
    if (ctx->borrowed)
        return fail(ctx, DG_EINVAL, std::string("set_orders: borrowed ") + what + " scratch too small (coarse layout larger than the fine one)");
    dfree(p);
    const long long c = need + need / 4;  // slack: successive adapted layouts differ a little
    CK(cudaMalloc(&p, sizeof(double) * c));
    cap = c;
    return DG_OK;
}

// 16-byte (even double) padding of the face / metric blocks: element kernels
// stage them with 1-D TMA bulk copies
static inline long long EVEN(long long x) { return (x + 1) & ~1LL; }

// Plans of the curved residual path (ns.cuh): element items, the face list
// (every interior face once, boundary faces of owned elements), face-block
// offsets, face metrics and (extruded meshes) compact volume metrics.
static dg_status build_ns_plans(dg_ctx* ctx, PlanTimer& tm)
{
    static const int TA[3] = {1, 0, 0}, TB[3] = {2, 2, 1};
    const int E = ctx->E;
    const bool ns = ctx->prm.physics == DG_NS;
    const bool ext = ctx->extruded;
    const long long L = ctx->off[E];
    // ---- element items: same-order owned elements, <= NS_ITEM_NODES nodes ----
    {
        std::vector<int> bkey, bstart, belem;
        order_buckets(ctx->orders, 0, ctx->n_own, bkey, bstart, belem);
        std::vector<NsItem> items;
        std::vector<int> el;
        el.reserve(ctx->n_own);
        for (size_t b = 0; b < bkey.size(); ++b) {
            const int ord = bkey[b];
            const int* be = belem.data() + bstart[b];
            const size_t bn = (size_t)(bstart[b + 1] - bstart[b]);
            const int N[3] = {ord & 255, (ord >> 8) & 255, (ord >> 16) & 255};
            const int n = npts(N);
            const int k = std::max(1, std::min(NS_MAXSLOTS, NS_ITEM_NODES / n));
            for (size_t i = 0; i < bn; i += k) {
                NsItem it;
                it.start = (int)el.size();
                it.count = (int)std::min<size_t>(k, bn - i);
                it.ord = ord;
                it.nodes = it.count * n;
                for (int j = 0; j < it.count; ++j) el.push_back(be[i + j]);
                items.push_back(it);
            }
        }
        // classes by node count (shared memory of the launch): <= 256, <= 512, larger
        static const int edge[3] = {256, 512, 1 << 30};
        std::vector<NsItem> sorted;
        sorted.reserve(items.size());
        ctx->nscls.clear();
        ctx->nscls_swH.clear();
        ctx->nscls_swG.clear();
        for (int c = 0; c < 3; ++c) {
            const int lo = c ? edge[c - 1] : 0;
            SizeClass cl{(int)sorted.size(), 0, 0};
            int swh = 0, swg = 0;
            for (const NsItem& it : items)
                if (it.nodes > lo && it.nodes <= edge[c]) {
                    sorted.push_back(it);
                    cl.count++;
                    cl.maxn = std::max(cl.maxn, it.nodes);
                    swh = std::max(swh, ns_stage_words(ext, true, true, it.ord, it.count));
                    swg = std::max(swg, ns_stage_words(ext, false, true, it.ord, it.count));
                }
            if (cl.count) {
                ctx->nscls.push_back(cl);
                ctx->nscls_swH.push_back(swh);
                ctx->nscls_swG.push_back(swg);
            }
        }
        CK(upload(ctx->d_nsitems, sorted));
        CK(upload(ctx->d_nselist, el));
    }
    tm.mark("ns items");
    // ---- faces ----
    std::vector<NsFace> fl;
    std::vector<int> fw;  // warps per face
    fl.reserve(3LL * E + 16);
    fw.reserve(3LL * E + 16);
    std::vector<long long> fofsG(6LL * E, -1), fofsH(6LL * E, -1);
    long long gl = 0, hl = 0, mgl = 0;
    auto pack = [&](int e) { const int* a = &ctx->orders[3 * e]; return a[0] | (a[1] << 4) | (a[2] << 8); };
    auto nkH = [&](int d) { return ext ? ext_nk(d) : 3; };
    for (int e = 0; e < E; ++e)
        for (int d = 0; d < 3; ++d) {
            const int* No = &ctx->orders[3 * e];
            const int so = (No[TA[d]] + 1) * (No[TB[d]] + 1);
            // interior face: e is L (its +d face)
            const int nb = ctx->nbr[6 * e + 2 * d + 1];
            if (nb >= 0 && !(e >= ctx->n_own && nb >= ctx->n_own)) {
                const int* Nn = &ctx->orders[3 * nb];
                const int sr = (Nn[TA[d]] + 1) * (Nn[TB[d]] + 1);
                const bool conf = No[TA[d]] == Nn[TA[d]] && No[TB[d]] == Nn[TB[d]];
                const int nm = (std::max(No[TA[d]], Nn[TA[d]]) + 1) * (std::max(No[TB[d]], Nn[TB[d]]) + 1);
                NsFace F{};
                F.offL = ctx->off[e];
                F.offR = ctx->off[nb];
                F.eL = e;
                F.eR = nb;
                F.ordL = pack(e);
                F.ordR = pack(nb);
                F.d = d;
                F.kind = conf ? 0 : 1;
                F.mg = mgl;
                mgl += 3LL * nm;
                F.outL = gl;
                fofsG[6LL * e + 2 * d + 1] = gl;
                gl += EVEN((long long)NV * so);
                F.outR = conf ? F.outL : gl;
                fofsG[6LL * nb + 2 * d] = F.outR;
                if (!conf) gl += EVEN((long long)NV * sr);
                if (ns) {
                    F.hL = hl;
                    fofsH[6LL * e + 2 * d + 1] = hl;
                    hl += EVEN((long long)NV * nkH(d) * so);
                    F.hR = conf ? F.hL : hl;
                    fofsH[6LL * nb + 2 * d] = F.hR;
                    if (!conf) hl += EVEN((long long)NV * nkH(d) * sr);
                }
                fl.push_back(F);
                fw.push_back((nm + 31) / 32);
            }
            // boundary faces of owned elements
            if (e >= ctx->n_own) continue;
            for (int s = 0; s < 2; ++s) {
                const int b = ctx->nbr[6 * e + 2 * d + s];
                if (b != -1 && b != -2) continue;
                NsFace F{};
                F.offL = s ? ctx->off[e] : -1;
                F.offR = s ? -1 : ctx->off[e];
                F.eL = s ? e : -1;
                F.eR = s ? -1 : e;
                F.ordL = F.ordR = pack(e);
                F.d = d;
                F.kind = b == -1 ? 2 : 3;
                F.mg = mgl;
                mgl += 3LL * so;
                F.outL = F.outR = gl;
                fofsG[6LL * e + 2 * d + s] = gl;
                gl += EVEN((long long)NV * so);
                if (ns) {
                    F.hL = F.hR = hl;
                    fofsH[6LL * e + 2 * d + s] = hl;
                    hl += EVEN((long long)NV * nkH(d) * so);
                }
                fl.push_back(F);
                fw.push_back((so + 31) / 32);
            }
        }
    tm.mark("ns face loop");
    {
        std::vector<NsFace> sorted;
        sorted.reserve(fl.size());
        ctx->nsf_cls[0] = 0;
        auto halo = [&](const NsFace& F) { return F.eL >= ctx->n_own || F.eR >= ctx->n_own; };
        for (int w = 1; w <= 3; ++w) {  // per class: interior faces, then those with a halo side
            for (size_t i = 0; i < fl.size(); ++i)
                if (fw[i] == w && !halo(fl[i])) sorted.push_back(fl[i]);
            ctx->nsf_mid[w] = (int)sorted.size();
            for (size_t i = 0; i < fl.size(); ++i)
                if (fw[i] == w && halo(fl[i])) sorted.push_back(fl[i]);
            ctx->nsf_cls[w] = (int)sorted.size();
        }
        if (sorted.size() != fl.size()) return fail(ctx, DG_EINVAL, "set_orders: face with more than 96 mortar points");
        fl.swap(sorted);
    }
    tm.mark("ns face list");
    CK(upload(ctx->d_nsfaces, fl));
    CK(upload(ctx->d_fofsG, fofsG));
    CK(upload(ctx->d_fofsH, fofsH));
    dg_status s;
    tm.mark("ns face uploads");
    if ((s = scratch_need(ctx, ctx->d_nsG, ctx->nsG_cap, gl, "flux-block")) != DG_OK) return s;
    if (ns && (s = scratch_need(ctx, ctx->d_nsH, ctx->nsH_cap, hl, "BR1-block")) != DG_OK) return s;
    if (ns && (s = scratch_need(ctx, ctx->d_grad, ctx->grad_len, 3 * L + 2, "gradient")) != DG_OK) return s;
    if (mgl > 0) {
        CK(dalloc(ctx->d_fg, (size_t)mgl));
        FaceGeomParams G;
        G.faces = ctx->d_nsfaces;
        G.nfaces = (int)fl.size();
        G.cm = curved_mesh(ctx);
        G.tdd = ctx->d_tdd;
        G.fg = ctx->d_fg;
        G.ext = ext ? 1 : 0;
        k_face_geom<<<(G.nfaces + 3) / 4, 128>>>(G);
        ctx->launches++;
        CK(cudaGetLastError());
    }
    // ---- volume metrics: full (10 per node, the dt / tau kernels) and compact (EXT) ----
    if (ctx->met_len < 2 * L) {
        dfree(ctx->d_met);
        CK(cudaMalloc(&ctx->d_met, sizeof(double) * (2 * L + L / 2)));
        ctx->met_len = 2 * L + L / 2;
    }
    tm.mark("ns uploads, face geometry");
    MetParams M;
    M.cm = curved_mesh(ctx);
    M.orders = ctx->d_orders;
    M.off = ctx->d_off;
    M.met = ctx->d_met;
    M.tdd = ctx->d_tdd;
    M.perm = ctx->d_eperm;
    for (const SizeClass& c : ctx->ecls_all) {
        M.pbase = c.base;
        k_metrics<<<c.count, CBS, sizeof(double) * 16 * (size_t)c.maxn>>>(M);
        ctx->launches++;
    }
    CK(cudaGetLastError());
    if (ext) {
        std::vector<long long> coff(E + 1, 0);
        for (int e = 0; e < E; ++e) {
            const int* N = &ctx->orders[3 * e];
            coff[e + 1] = coff[e] + EVEN(6LL * (N[0] + 1) * (N[1] + 1));
        }
        CK(upload(ctx->d_coff, coff));
        CK(dalloc(ctx->d_metc, (size_t)coff[E]));
        MetExtParams X;
        X.cm = curved_mesh(ctx);
        X.orders = ctx->d_orders;
        X.coff = ctx->d_coff;
        X.metc = ctx->d_metc;
        X.tdd = ctx->d_tdd;
        X.E = E;
        k_metrics_ext<<<E, 128>>>(X);
        ctx->launches++;
        CK(cudaGetLastError());
    }
    tm.mark("metrics");
    CK(cudaDeviceSynchronize());
    return DG_OK;
}

dg_status dg_set_orders(dg_ctx* ctx, const int32_t* orders_host)
{
    if (!ctx) return DG_EINVAL;
    if (ctx->E == 0) return fail(ctx, DG_ESTATE, "set_orders: no mesh");
    PlanTimer tm;
    drop_graphs(ctx);  // captured launches refer to the old plans
    drop_coarse(ctx);  // non-isolated tau levels of the old layout
    tm.mark("drop graphs / levels");
    ctx->coarse_streaming = false;
    const int E = ctx->E;
    for (long long i = 0; i < 3LL * E; ++i)
        if (orders_host[i] < 1 || orders_host[i] > NMAX) return fail(ctx, DG_EINVAL, "set_orders: order out of 1..8");
    ctx->orders.assign(orders_host, orders_host + 3LL * E);
    if (ctx->affine_geo && ctx->prm.physics == DG_EULER && ctx->path != DG_PATH_RUNTIME) {
        // AUTO: many (N1,N2,N3) buckets -> the class-batched runtime-order
        // kernels (a handful of launches; section 7.3 of DESIGN.md); few ->
        // the order-specialised ones (one launch per bucket, CUDA graph)
        bool seen[NMAX * NMAX * NMAX] = {};
        int nb = 0;
        for (int e = 0; e < ctx->n_own; ++e) {
            const int* N = &ctx->orders[3 * e];
            const int k = (N[0] - 1) + NMAX * ((N[1] - 1) + NMAX * (N[2] - 1));
            if (!seen[k]) { seen[k] = true; ++nb; }
        }
        ctx->curved = ctx->path == DG_PATH_AUTO && nb > RT_BUCKETS;
        ctx->tau_curved = false;  // affine Euler: k_tau5 on either path
    }
    ctx->off.assign(E + 1, 0);
    ctx->ndof = 0;
    ctx->maxn = 0;
    for (int e = 0; e < E; ++e) {
        const int n = npts(&ctx->orders[3 * e]);
        ctx->off[e + 1] = ctx->off[e] + (long long)NV * n;
        ctx->ndof += n;
        ctx->maxn = std::max(ctx->maxn, n);
    }
    // (N1,N2,N3) buckets -> work items of up to floor(256/n) elements, ordered
    // by their first element id (spatially coherent sweep, neighbour traces hit L2)
    std::vector<int> bkey, bstart, belem;
    order_buckets(ctx->orders, 0, ctx->curved ? 0 : ctx->n_own, bkey, bstart, belem);  // affine kernels only
    std::vector<int> elist;
    elist.reserve(E);
    std::vector<WorkItem> work;
    size_t smem = 0;
    for (size_t b = 0; b < bkey.size(); ++b) {
        const int ord = bkey[b];
        const int* be = belem.data() + bstart[b];
        const size_t bn = (size_t)(bstart[b + 1] - bstart[b]);
        const int N[3] = {ord & 255, (ord >> 8) & 255, (ord >> 16) & 255};
        const int n = npts(N);
        const int k = res_cnt(N[0] + 1, N[1] + 1, N[2] + 1);  // = Shape<N>::CNT
        const int nfs = 2 * ((N[1] + 1) * (N[2] + 1) + (N[0] + 1) * (N[2] + 1) + (N[0] + 1) * (N[1] + 1));
        for (size_t i = 0; i < bn; i += k) {
            WorkItem w;
            w.start = (int)elist.size();
            w.count = (int)std::min<size_t>(k, bn - i);
            w.ord = ord;
            w.pad = be[i];
            for (int j = 0; j < w.count; ++j) elist.push_back(be[i + j]);
            work.push_back(w);
            const size_t bytes = sizeof(double) * (3 * NP * NP + (size_t)w.count * NV * (2 * n + nfs));
            smem = std::max(smem, bytes);
        }
    }
    // items are grouped per bucket (one specialised launch each), element order inside
    ctx->buckets.clear();
    for (size_t i = 0; i < work.size(); ++i) {
        if (ctx->buckets.empty() || ctx->buckets.back().ord != work[i].ord)
            ctx->buckets.push_back(Bucket{work[i].ord, (int)i, 0, work[i].start, 0, 0});
        ctx->buckets.back().nitems++;
        ctx->buckets.back().nelem += work[i].count;
    }
    ctx->nwork = (int)work.size();
    ctx->res_smem = smem;
    std::vector<MortarItem> mort;
    std::vector<long long> moff;
    long long flen = 0;
    if (!ctx->curved) {  // ---- plans of the order-specialised (affine) kernels ----
    // mortar faces: + side of L against - side of R, tangential orders differ
    moff.assign(6LL * E, -1);
    long long mlen = 0;
    static const int TA[3] = {1, 0, 0}, TB[3] = {2, 2, 1};
    for (int e = 0; e < E; ++e)
        for (int d = 0; d < 3; ++d) {
            const int nb = ctx->nbr[6 * e + 2 * d + 1];
            if (nb < 0) continue;
            if (e >= ctx->n_own && nb >= ctx->n_own) continue;  // halo-halo face: not needed
            const int* NL = &ctx->orders[3 * e];
            const int* NR = &ctx->orders[3 * nb];
            if (NL[TA[d]] == NR[TA[d]] && NL[TB[d]] == NR[TB[d]]) continue;
            mort.push_back(MortarItem{e, nb, d, 0});
            moff[6LL * e + 2 * d + 1] = mlen;
            mlen += ((long long)NV * (NL[TA[d]] + 1) * (NL[TB[d]] + 1) + 1) & ~1LL;  // 16-byte aligned blocks
            moff[6LL * nb + 2 * d] = mlen;
            mlen += ((long long)NV * (NR[TA[d]] + 1) * (NR[TB[d]] + 1) + 1) & ~1LL;
        }
    ctx->nmortar = (int)mort.size();
    ctx->mortar_len = mlen;
    tm.mark("buckets, mortar list");
    {
        std::vector<MortarFace> mf(mort.size());
        for (size_t i = 0; i < mort.size(); ++i) {
            const MortarItem& m = mort[i];
            const int* a = &ctx->orders[3 * m.L];
            const int* b = &ctx->orders[3 * m.R];
            mf[i].offL = ctx->off[m.L];
            mf[i].offR = ctx->off[m.R];
            mf[i].moL = moff[6LL * m.L + 2 * m.d + 1];
            mf[i].moR = moff[6LL * m.R + 2 * m.d];
            mf[i].ordL = a[0] | (a[1] << 4) | (a[2] << 8);
            mf[i].ordR = b[0] | (b[1] << 4) | (b[2] << 8);
            mf[i].d = m.d;
            mf[i].pad = 0;
        }
        CK(upload(ctx->d_mfaces, mf));
    }
    // conforming faces and boundary faces of owned elements: the Riemann flux
    // of each face point is computed once (k_face) into the flux buffer after
    // the mortar blocks; fofs = flux offset of every element face.
    std::vector<long long> fofs(moff);
    std::vector<FaceItem> faces;
    std::vector<int> fpt(1, 0);
    flen = mlen;
    {
        auto strides = [&](int el, int* st) {
            const int* N = &ctx->orders[3 * el];
            st[0] = 1; st[1] = N[0] + 1; st[2] = (N[0] + 1) * (N[1] + 1);
        };
        // element-descending order: the faces of the elements the preceding
        // element kernel wrote last (still in L2) come first
        for (int e = E - 1; e >= 0; --e)
            for (int d = 0; d < 3; ++d) {
                const int* No = &ctx->orders[3 * e];
                const int nf = (No[TA[d]] + 1) * (No[TB[d]] + 1);
                for (int side = 0; side < 2; ++side) {  // side 1: + face of e (e = L); side 0: - face (BC only)
                    const int nb = ctx->nbr[6 * e + 2 * d + side];
                    FaceItem fi{};
                    fi.d = d;
                    fi.nf = nf;
                    fi.nta = No[TA[d]] + 1;
                    int st[3];
                    strides(e, st);
                    if (side == 1 && nb >= 0) {
                        if (moff[6LL * e + 2 * d + 1] >= 0) continue;       // mortar
                        if (e >= ctx->n_own && nb >= ctx->n_own) continue;  // halo-halo
                        int sr[3];
                        strides(nb, sr);
                        fi.kind = 0;
                        fi.offL = ctx->off[e];
                        fi.nL = npts(No);
                        fi.baseL = No[d] * st[d];
                        fi.saL = st[TA[d]];
                        fi.sbL = st[TB[d]];
                        fi.offR = ctx->off[nb];
                        fi.nR = npts(&ctx->orders[3 * nb]);
                        fi.baseR = 0;
                        fi.saR = sr[TA[d]];
                        fi.sbR = sr[TB[d]];
                        fi.goff = flen;
                        fofs[6LL * e + 2 * d + 1] = flen;
                        fofs[6LL * nb + 2 * d] = flen;
                    } else if ((nb == -1 || nb == -2) && e < ctx->n_own) {
                        fi.kind = nb == -1 ? 2 : 3;
                        const long long o = ctx->off[e];
                        if (side == 1) { fi.offL = o; fi.nL = npts(No); fi.baseL = No[d] * st[d]; fi.saL = st[TA[d]]; fi.sbL = st[TB[d]]; fi.offR = -1; }
                        else { fi.offR = o; fi.nR = npts(No); fi.baseR = 0; fi.saR = st[TA[d]]; fi.sbR = st[TB[d]]; fi.offL = -1; }
                        fi.goff = flen;
                        fofs[6LL * e + 2 * d + side] = flen;
                    } else {
                        continue;
                    }
                    faces.push_back(fi);
                    fpt.push_back(fpt.back() + nf);
                    flen += ((long long)NV * nf + 1) & ~1LL;
                }
            }
    }
    ctx->nfaces = (int)faces.size();
    ctx->nface_pts = fpt.back();
    {
        // k_face: one thread per face point with a precomputed record
        // {L trace index, R trace index, flux index, packed nL | nR | d | kind | nf-1}
        const long long np = ctx->nface_pts;
        ctx->nfblk = (int)((np + FACE_BS - 1) / FACE_BS);
        if (ctx->off[E] >= (1LL << 31) || flen >= (1LL << 31))
            return fail(ctx, DG_EINVAL, "set_orders: state or flux buffer beyond 2^31 doubles");
        std::vector<int4> fcode((size_t)np);
        for (size_t f = 0; f < faces.size(); ++f) {
            const FaceItem& fi = faces[f];
            for (int p = fpt[f]; p < fpt[f + 1]; ++p) {
                const int pt = p - fpt[f], ta = pt % fi.nta, tb = pt / fi.nta;
                int4 r;
                r.x = fi.offL >= 0 ? (int)(fi.offL + fi.baseL + ta * fi.saL + tb * fi.sbL) : -1;
                r.y = fi.offR >= 0 ? (int)(fi.offR + fi.baseR + ta * fi.saR + tb * fi.sbR) : -1;
                r.z = (int)(fi.goff + pt);
                r.w = (fi.offL >= 0 ? fi.nL : 0) | ((fi.offR >= 0 ? fi.nR : 0) << 10) | (fi.d << 20) | (fi.kind << 22) |
                      ((fi.nf - 1) << 24);
                fcode[p] = r;
            }
        }
        CK(upload(ctx->d_faces, faces));
        CK(upload(ctx->d_fpt, fpt));
        CK(upload(ctx->d_fcta, fcode));
    }
    tm.mark("face lists + upload");
    // per element-face source descriptors of the outer state (see FaceInfo)
    std::vector<FaceInfo> finfo(6LL * E);
    for (int e = 0; e < E; ++e)
        for (int f = 0; f < 6; ++f) {
            const int d = f >> 1, s = f & 1;
            FaceInfo fi{};
            const int nb = ctx->nbr[6 * e + f];
            const int* No = &ctx->orders[3 * e];
            if (nb == -1) fi.kind = 2;
            else if (nb == -2) fi.kind = 3;
            else if (nb == -3) fi.kind = 4;  // outside the local set (halo elements only; never read)
            else if (moff[6LL * e + f] >= 0) {
                fi.kind = 1;
                fi.off = moff[6LL * e + f];
                fi.n = (No[TA[d]] + 1) * (No[TB[d]] + 1);
            } else {
                const int* B = &ctx->orders[3 * nb];
                const int st[3] = {1, B[0] + 1, (B[0] + 1) * (B[1] + 1)};
                fi.kind = 0;
                fi.off = ctx->off[nb];
                fi.n = npts(B);
                fi.base = (s ? 0 : B[d]) * st[d];
                fi.sa = st[TA[d]];
                fi.sb = st[TB[d]];
            }
            finfo[6LL * e + f] = fi;
        }
    CK(upload(ctx->d_finfo, finfo));
    std::vector<SlotInfo> slots(elist.size());
    for (size_t i = 0; i < elist.size(); ++i) {
        const int e = elist[i];
        slots[i].off = ctx->off[e];
        slots[i].e = e;
        slots[i].pad = 0;
        for (int dd = 0; dd < 3; ++dd) slots[i].sc[dd] = 2.0 / ctx->h[3LL * e + dd];
    }
    CK(upload(ctx->d_slots, slots));
    std::vector<FaceInfo> fslot(6 * elist.size());
    for (size_t i = 0; i < elist.size(); ++i)
        for (int f = 0; f < 6; ++f) fslot[6 * i + f] = finfo[6LL * elist[i] + f];
    CK(upload(ctx->d_finfo_slot, fslot));
    std::vector<long long> fos(6 * elist.size());
    for (size_t i = 0; i < elist.size(); ++i)
        for (int f = 0; f < 6; ++f) fos[6 * i + f] = fofs[6LL * elist[i] + f];
    CK(upload(ctx->d_fofs_slot, fos));
    tm.mark("face info, slots");
    for (Bucket& b : ctx->buckets) {
        const int o1 = b.ord & 255, o2 = (b.ord >> 8) & 255, o3 = (b.ord >> 16) & 255;
        if (ctx->occ_cache[o1][o2][o3] < 0) ctx->occ_cache[o1][o2][o3] = (signed char)ctx->rocc[o1][o2][o3]();
        const int occ = ctx->occ_cache[o1][o2][o3];
        b.grid = std::max(1, occ) * ctx->nsm;
    }
    }  // affine plans
    // tau-estimation levels (e, d, p < N_d), largest first for load balance
    // (curved kernels only: the affine path batches levels in k_tau5 groups)
    std::vector<TauLevel> lv;
    ctx->max_level = 0;
    for (int e = 0; e < (ctx->tau_curved ? ctx->n_own : 0); ++e)
        for (int d = 0; d < 3; ++d)
            for (int p = 1; p < ctx->orders[3 * e + d]; ++p) {
                lv.push_back(TauLevel{e, d, p, 0});
                const int* No = &ctx->orders[3 * e];
                const int nO = npts(No) / (No[d] + 1) * (p + 1);
                ctx->max_level = std::max(ctx->max_level, nO);
            }
    ctx->nlevels = (int)lv.size();
    {
        std::vector<int> lsz(lv.size()), li(lv.size());
        for (size_t i = 0; i < lv.size(); ++i) {
            const int* No = &ctx->orders[3 * lv[i].e];
            lsz[i] = npts(No) / (No[lv[i].d] + 1) * (lv[i].p + 1);
            li[i] = (int)i;
        }
        ctx->lcls.clear();
        size_classes(li, lsz, 0, (int)lv.size(), ctx->lcls);
        std::vector<TauLevel> ls(lv.size());
        for (size_t i = 0; i < lv.size(); ++i) ls[i] = lv[li[i]];
        lv.swap(ls);
    }
    CK(upload(ctx->d_levels, lv));
    // extruded meshes: consecutive (d, p) levels of an element, d-major, in
    // groups of <= cap coarse nodes (k_tau_grp: one CTA per group)
    {
        std::vector<TauLevel> gr;
        ctx->tgrp_cap = std::max(256, ctx->max_level);
        if (ctx->tau_curved && ctx->extruded) {
            for (int e = 0; e < ctx->n_own; ++e) {
                const int* No = &ctx->orders[3 * e];
                TauLevel cur{e, -1, 0, 0};
                int sum = 0;
                for (int d = 0; d < 3; ++d)
                    for (int p = 1; p < No[d]; ++p) {
                        const int nO = npts(No) / (No[d] + 1) * (p + 1);
                        if (cur.pad > 0 && (sum + nO > ctx->tgrp_cap || cur.pad == TAU_GRP_MAXLV)) {
                            gr.push_back(cur);
                            cur.pad = 0;
                            sum = 0;
                        }
                        if (cur.pad == 0) {
                            cur.d = d;
                            cur.p = p;
                        }
                        cur.pad++;
                        sum += nO;
                    }
                if (cur.pad > 0) gr.push_back(cur);
            }
        }
        ctx->ntgrp = (int)gr.size();
        CK(upload(ctx->d_tgrp, gr));
    }
    tm.mark("tau levels");
    ctx->ecls_own.clear();
    ctx->ecls_all.clear();
    if (ctx->curved) {  // size classes of the curved element kernels
        std::vector<int> esz(E), ei(E);
        for (int e = 0; e < E; ++e) { esz[e] = npts(&ctx->orders[3 * e]); ei[e] = e; }
        size_classes(ei, esz, 0, ctx->n_own, ctx->ecls_own);
        ctx->ecls_all = ctx->ecls_own;
        size_classes(ei, esz, ctx->n_own, E, ctx->ecls_all);
        CK(upload(ctx->d_eperm, ei));
    }
    {   // k_tau5 work: (element, direction, coarse orders p0..p1) groups of <= TAU5_MAXN
        // coarse nodes (a single larger level forms its own group), largest first
        std::vector<TauGroup> tg;
        std::vector<int> gsz;
        int gmax = 0;
        for (int e = 0; e < (ctx->tau_curved ? 0 : ctx->n_own); ++e)
            for (int d = 0; d < 3; ++d) {
                const int* No = &ctx->orders[3 * e];
                const int nx = npts(No) / (No[d] + 1);
                int p = 1;
                while (p < No[d]) {
                    int q = p, sz = (p + 1) * nx;
                    while (q + 1 < No[d] && sz + (q + 2) * nx <= TAU5_MAXN) sz += (++q + 1) * nx;
                    tg.push_back(TauGroup{e, d, p, q});
                    gsz.push_back(sz);
                    gmax = std::max(gmax, sz);
                    p = q + 1;
                }
            }
        // largest first, stable: counting sort on the group size (O(groups))
        std::vector<int> cnt(gmax + 2, 0);
        for (int s : gsz) ++cnt[s];
        std::vector<int> start(gmax + 2, 0);
        for (int s = gmax - 1; s >= 0; --s) start[s] = start[s + 1] + cnt[s + 1];
        std::vector<TauGroup> sorted(tg.size());
        for (size_t i = 0; i < tg.size(); ++i) sorted[start[gsz[i]]++] = tg[i];
        ctx->ntgroups = (int)sorted.size();
        ctx->tau5_smem = sizeof(double) * 4 * NV * (size_t)gmax;
        CK(upload(ctx->d_tgroups, sorted));
    }
    tm.mark("tau5 groups");
    std::vector<int> ord_i(ctx->orders.begin(), ctx->orders.end());
    CK(upload(ctx->d_orders, ord_i));
    CK(upload(ctx->d_off, ctx->off));
    CK(upload(ctx->d_work, work));
    CK(upload(ctx->d_elist, elist));
    CK(upload(ctx->d_mortar, mort));
    CK(upload(ctx->d_moff, moff));
    if (flen > 0 && !ctx->curved) CK(dalloc(ctx->d_mortarG, (size_t)flen));
    CK(dalloc(ctx->d_sel, 6 * (size_t)E));
    CK(dalloc(ctx->d_margin, (size_t)E));
    tm.mark("tau5 groups, uploads");
    if (ctx->curved) {
        dg_status s = build_ns_plans(ctx, tm);
        if (s != DG_OK) return s;
    }
    ctx->have_orders = true;
    return DG_OK;
}

int64_t dg_state_len(const dg_ctx* ctx) { return ctx && ctx->have_orders ? ctx->off[ctx->E] : 0; }
int64_t dg_ndof(const dg_ctx* ctx) { return ctx && ctx->have_orders ? ctx->ndof : 0; }
int64_t dg_owned_state_len(const dg_ctx* ctx) { return ctx && ctx->have_orders ? ctx->off[ctx->n_own] : 0; }

dg_status dg_node_coords(dg_ctx* ctx, double* X)
{
    if (!ctx || !X) return DG_EINVAL;
    if (!ctx->have_orders) return fail(ctx, DG_ESTATE, "node_coords: orders not set");
    const Tables& t = host_tables();
    const int* g = ctx->gorder;
    const int ng = (g[0] + 1) * (g[1] + 1) * (g[2] + 1);
    long long o = 0;
    for (int e = 0; e < ctx->E; ++e) {
        const int* N = &ctx->orders[3 * e];
        const int n = npts(N);
        const double* G = &ctx->geo[3LL * ng * e];
        // x(i,j,k) = sum_abc T^{g1->N1}[i][a] T^{g2->N2}[j][b] T^{g3->N3}[k][c] X_geo[a,b,c]
        for (int k = 0; k <= N[2]; ++k)
            for (int j = 0; j <= N[1]; ++j)
                for (int i = 0; i <= N[0]; ++i) {
                    double x[3] = {0.0, 0.0, 0.0};
                    for (int c = 0; c <= g[2]; ++c)
                        for (int b = 0; b <= g[1]; ++b)
                            for (int a = 0; a <= g[0]; ++a) {
                                const double wgt = t.T[g[0]][N[0]][i * (g[0] + 1) + a] * t.T[g[1]][N[1]][j * (g[1] + 1) + b] *
                                                   t.T[g[2]][N[2]][k * (g[2] + 1) + c];
                                const int gi = a + (g[0] + 1) * (b + (g[1] + 1) * c);
                                for (int cc = 0; cc < 3; ++cc) x[cc] += wgt * G[cc * ng + gi];
                            }
                    const int node = i + (N[0] + 1) * (j + (N[1] + 1) * k);
                    for (int cc = 0; cc < 3; ++cc) X[o + (long long)cc * n + node] = x[cc];
                }
        o += 3LL * n;
    }
    return DG_OK;
}

}  // extern "C"
// part: FACES_ALL, FACES_INTERIOR (no halo side: may run while the halo
// traces are in flight), FACES_HALO (the rest)
enum { FACES_ALL = 0, FACES_INTERIOR = 1, FACES_HALO = 2 };
// CTAs of a face launch: one group per face, or (NS_FACE_PERSIST) the
// resident CTAs, each group walking faces with a stride
template <int W, int MODE>
static int face_grid(dg_ctx* ctx, int nf)
{
    using C = FaceCfg<W, MODE>;
    const int need = (nf + C::G - 1) / C::G;
    if (!face_persist(W, MODE)) return need;
    static int occ = 0;  // per instantiation, one device per process
    if (occ == 0) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_ns_face<W, MODE>, C::BS, C::smem);
        if (occ < 1) occ = 1;
    }
    return std::min(need, occ * ctx->nsm);
}

template <int MODE>
static void launch_ns_faces(dg_ctx* ctx, const NsFaceParams& base, cudaStream_t st, int part = FACES_ALL)
{
    for (int w = 1; w <= 3; ++w) {
        NsFaceParams P = base;
        P.fbase = part == FACES_HALO ? ctx->nsf_mid[w] : ctx->nsf_cls[w - 1];
        P.fend = part == FACES_INTERIOR ? ctx->nsf_mid[w] : ctx->nsf_cls[w];
        const int nf = P.fend - P.fbase;
        if (nf <= 0) continue;
        using C1 = FaceCfg<1, MODE>;
        using C2 = FaceCfg<2, MODE>;
        using C3 = FaceCfg<3, MODE>;
        if (w == 1) k_ns_face<1, MODE><<<face_grid<1, MODE>(ctx, nf), C1::BS, C1::smem, st>>>(P);
        else if (w == 2) k_ns_face<2, MODE><<<face_grid<2, MODE>(ctx, nf), C2::BS, C2::smem, st>>>(P);
        else k_ns_face<3, MODE><<<face_grid<3, MODE>(ctx, nf), C3::BS, C3::smem, st>>>(P);
        ctx->launches++;
    }
}

extern "C" {
static NsElemParams ns_elem_params(dg_ctx* ctx, const double* q)
{
    NsElemParams P{};
    P.items = ctx->d_nsitems;
    P.elist = ctx->d_nselist;
    P.orders = ctx->d_orders;
    P.off = ctx->d_off;
    P.met = ctx->d_met;
    P.metc = ctx->d_metc;
    P.coff = ctx->d_coff;
    P.q = q;
    P.ph = phys_dev(ctx->prm);
    P.flag = ctx->d_flag;
    return P;
}

static NsFaceParams ns_face_params(dg_ctx* ctx, const double* q)
{
    NsFaceParams F{};
    F.faces = ctx->d_nsfaces;
    F.q = q;
    F.grad = ctx->d_grad;
    F.fg = ctx->d_fg;
    F.tab = ctx->d_tab;
    F.ph = phys_dev(ctx->prm);
    F.ext = ctx->extruded ? 1 : 0;
    return F;
}

// BR1 gradient of the owned elements into d_grad (eq DGSEMsystem:2):
// face terms H (non-isolated), then the element kernel.
static dg_status launch_ns_gradient(dg_ctx* ctx, int variant, const double* q, cudaStream_t st, int part = FACES_ALL)
{
    const bool noniso = variant == DG_NONISOLATED;
    if (noniso) {
        NsFaceParams F = ns_face_params(ctx, q);
        F.out = ctx->d_nsH;
        launch_ns_faces<MODE_QHAT>(ctx, F, st, part);
        if (part == FACES_INTERIOR) return check_stream_error(ctx, "k_ns_face launch");
    }
    NsElemParams P = ns_elem_params(ctx, q);
    P.gout = ctx->d_grad;
    P.blk = ctx->d_nsH;
    P.fofs = noniso ? ctx->d_fofsH : nullptr;
    for (const SizeClass& c : ctx->nscls) {
        P.ibase = c.base;
        const int sw = ctx->nscls_swH[&c - &ctx->nscls[0]];
        int nst = ns_stages();
        while (nst > 1 && sizeof(double) * nst * (size_t)sw > (size_t)ctx->smem_limit) --nst;
        const size_t sm = sizeof(double) * nst * (size_t)sw;
        if (sm > (size_t)ctx->smem_limit) return fail(ctx, DG_EINVAL, "k_ns_grad: element item exceeds shared memory");
        auto kern = ctx->extruded ? k_ns_grad<true> : k_ns_grad<false>;
        int occ = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NS_THREADS, sm);
        const int grid = std::min(c.count, std::max(1, occ) * ctx->nsm);
        kern<<<grid, NS_THREADS, sm, st>>>(P, c.count, nst, sw, ctx->off[ctx->E]);
        ctx->launches++;
    }
    return check_stream_error(ctx, "k_ns_grad launch");
}

static dg_status launch_residual_curved(dg_ctx* ctx, int variant, const double* q, double* out, double* g,
                                        const double* dt, double A, double B, int mode, cudaStream_t st,
                                        unsigned long long* lam_max, int flags = 0)
{
    const bool ns = ctx->prm.physics == DG_NS;
    const bool noniso = variant == DG_NONISOLATED;
    const int part = (flags & DG_FLAG_FACES_INTERIOR) ? FACES_INTERIOR : ((flags & DG_FLAG_FACES_HALO) ? FACES_HALO : FACES_ALL);
    if (part != FACES_ALL && (!noniso || (ns && !(flags & DG_FLAG_GRADIENT_READY))))
        return fail(ctx, DG_EINVAL, "residual: split face passes need the non-isolated variant (NS: and the gradient formed)");
    if (ns && !(flags & 1)) {  // flag 1: the caller already formed the gradient (multi-rank halo)
        dg_status s = launch_ns_gradient(ctx, variant, q, st);
        if (s != DG_OK) return s;
    }
    if (noniso) {
        NsFaceParams F = ns_face_params(ctx, q);
        F.out = ctx->d_nsG;
        if (ns) launch_ns_faces<MODE_FLUX_NS>(ctx, F, st, part);
        else launch_ns_faces<MODE_FLUX_EULER>(ctx, F, st, part);
        if (part == FACES_INTERIOR) return check_stream_error(ctx, "k_ns_face launch");
    }
    NsElemParams P = ns_elem_params(ctx, q);
    P.grad = ctx->d_grad;
    P.blk = ctx->d_nsG;
    P.fofs = noniso ? ctx->d_fofsG : nullptr;
    P.out = out;
    P.g = g;
    P.dt = dt;
    P.rkA = A;
    P.rkB = B;
    P.mode = mode;
    P.lam_max = lam_max;
    for (const SizeClass& c : ctx->nscls) {
        P.ibase = c.base;
        const int sw = ctx->nscls_swG[&c - &ctx->nscls[0]];
        const size_t fw = (size_t)15 * c.maxn;  // F work area
        int nst = ns_stages();
        while (nst > 1 && sizeof(double) * (nst * (size_t)sw + fw) > (size_t)ctx->smem_limit) --nst;
        const size_t sm = sizeof(double) * (nst * (size_t)sw + fw);
        if (sm > (size_t)ctx->smem_limit) return fail(ctx, DG_EINVAL, "k_ns_res: element item exceeds shared memory");
        auto kern = ctx->extruded ? (ns ? k_ns_res<true, true> : k_ns_res<true, false>)
                                  : (ns ? k_ns_res<false, true> : k_ns_res<false, false>);
        int occ = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NS_THREADS, sm);
        const int grid = std::min(c.count, std::max(1, occ) * ctx->nsm);
        kern<<<grid, NS_THREADS, sm, st>>>(P, c.count, nst, sw, c.maxn, ctx->off[ctx->E]);
        ctx->launches++;
    }
    return check_stream_error(ctx, "curved residual launch");
}

// fused step size for the first RK stage (ResParams::lam_in ...), see dg_rk_steps
struct DtFuse {
    const unsigned long long* lam_in = nullptr;
    double cfl = 0.0;
    double* dt_out = nullptr;
    unsigned long long* lam_zero = nullptr;
};

static dg_status launch_residual_direct(dg_ctx* ctx, int variant, const double* q, double* out, double* g,
                                        const double* dt, double A, double B, int mode, cudaStream_t st,
                                        unsigned long long* lam_max, const DtFuse& fz = DtFuse())
{
    if (variant == DG_NONISOLATED && ctx->nmortar > 0) {
        MortarParams M;
        M.q = q;
        M.orders = ctx->d_orders;
        M.off = ctx->d_off;
        M.items = ctx->d_mortar;
        M.moff = ctx->d_moff;
        M.mortarG = ctx->d_mortarG;
        M.tab = ctx->d_tab;
        M.ph = phys_dev(ctx->prm);
        CK(cudaMemsetAsync(ctx->d_flag + 4, 0, sizeof(int), st));  // k_mortar3 work counter
        k_mortar3<<<std::min(ctx->nmortar, MT_MINB * ctx->nsm), MT_BS, 0, st>>>(M, ctx->d_mfaces, ctx->nmortar,
                                                                            ctx->d_flag + 4);
        ctx->launches++;
    }
    if (variant == DG_NONISOLATED && ctx->nface_pts > 0) {
        FaceParams FP;
        FP.q = q;
        FP.G = ctx->d_mortarG;
        FP.faces = ctx->d_faces;
        FP.fpt = ctx->d_fpt;
        FP.fcta = ctx->d_fcta;
        FP.npts = (int)ctx->nface_pts;
        FP.ph = phys_dev(ctx->prm);
        k_face<<<std::min(ctx->nfblk, FACE_MINB * ctx->nsm), FACE_BS, 0, st>>>(FP);
        ctx->launches++;
    }
    ResParams P;
    P.q = q;
    P.out = out;
    P.g = g;
    P.dt = dt;
    P.rkA = A;
    P.rkB = B;
    P.mode = mode;
    P.variant = variant;
    P.orders = ctx->d_orders;
    P.off = ctx->d_off;
    P.nbr = ctx->d_nbr;
    P.hgeo = ctx->d_h;
    P.work = ctx->d_work;
    P.elist = ctx->d_elist;
    P.mortarG = ctx->d_mortarG;
    P.moff = ctx->d_moff;
    P.finfo = ctx->d_finfo;
    P.slots = ctx->d_slots;
    P.finfo_slot = ctx->d_finfo_slot;
    P.fofs_slot = ctx->d_fofs_slot;
    P.tab = ctx->d_tab;
    P.ph = phys_dev(ctx->prm);
    P.flag = ctx->d_flag;
    P.lam_max = lam_max;
    P.gamma = ctx->prm.gamma;
    P.qlen = ctx->off[ctx->E];
    P.lam_in = fz.lam_in;
    P.cfl = fz.cfl;
    P.dt_out = fz.dt_out;
    P.lam_zero = fz.lam_zero;
    if ((reinterpret_cast<uintptr_t>(q) & 15) != 0)
        return fail(ctx, DG_EINVAL, "residual: state pointer must be 16-byte aligned");
    {
        if (ctx->buckets.size() == 1) {
            const Bucket& b = ctx->buckets[0];
            ctx->rtab[b.ord & 255][(b.ord >> 8) & 255][(b.ord >> 16) & 255](P, b.start0, b.nelem, b.nitems, b.grid, st);
            ctx->launches++;
        } else {  // mixed orders: the buckets are independent -> run them concurrently
            const int ns = std::min<int>(dg_ctx::NSTREAMS, (int)ctx->buckets.size());
            CK(cudaEventRecord(ctx->ev_fork, st));
            for (int i = 0; i < ns; ++i) CK(cudaStreamWaitEvent(ctx->side[i], ctx->ev_fork, 0));
            for (size_t i = 0; i < ctx->buckets.size(); ++i) {
                const Bucket& b = ctx->buckets[i];
                ResParams Pb = P;
                if (i > 0) {  // one writer of the fused dt
                    Pb.dt_out = nullptr;
                    Pb.lam_zero = nullptr;
                }
                ctx->rtab[b.ord & 255][(b.ord >> 8) & 255][(b.ord >> 16) & 255](Pb, b.start0, b.nelem, b.nitems, b.grid,
                                                                                    ctx->side[i % ns]);
                ctx->launches++;
            }
            for (int i = 0; i < ns; ++i) {
                CK(cudaEventRecord(ctx->ev_join[i], ctx->side[i]));
                CK(cudaStreamWaitEvent(st, ctx->ev_join[i], 0));
            }
        }
    }
    return check_stream_error(ctx, "k_residual launch");
}

// Mixed-order layouts launch one order-specialised kernel per (N1,N2,N3)
// bucket (cfg3: 216) plus the mortar and face passes: that sequence is
// captured once per argument set into a CUDA graph (fork/join over the side
// streams included) and replayed with a single launch.  Cache per layout.
constexpr int GRAPH_AFTER = 8;  // direct launches of a shape before its graph is captured

static dg_status launch_residual(dg_ctx* ctx, int variant, const double* q, double* out, double* g, const double* dt,
                                 double A, double B, int mode, cudaStream_t st, unsigned long long* lam_max = nullptr,
                                 int flags = 0, const DtFuse& fz = DtFuse())
{
    if (ctx->curved) return launch_residual_curved(ctx, variant, q, out, g, dt, A, B, mode, st, lam_max, flags);
    if (ctx->buckets.size() <= 1 || ctx->no_graphs)
        return launch_residual_direct(ctx, variant, q, out, g, dt, A, B, mode, st, lam_max, fz);
    const GraphKey key{variant, mode, q, out, g, dt, lam_max, A, B, fz.lam_in, fz.dt_out, fz.lam_zero, fz.cfl};
    const ShapeKey shape{variant, mode, lam_max != nullptr, fz.lam_in != nullptr, fz.dt_out != nullptr,
                         fz.lam_zero != nullptr};
    if ((reinterpret_cast<uintptr_t>(q) & 15) != 0)
        return fail(ctx, DG_EINVAL, "residual: state pointer must be 16-byte aligned");
    auto itg = ctx->graphs.find(shape);
    // a fresh layout (dynamic adaptation every few steps) launches directly at
    // first: capture + instantiate costs ~ a few residuals of launches, so a
    // graph is only built for a shape that keeps recurring
    if (itg == ctx->graphs.end() && ++ctx->direct_uses[shape] <= GRAPH_AFTER)
        return launch_residual_direct(ctx, variant, q, out, g, dt, A, B, mode, st, lam_max, fz);
    if (itg == ctx->graphs.end()) {
        const long long l0 = ctx->launches;
        CK(cudaStreamBeginCapture(ctx->cap_stream, cudaStreamCaptureModeRelaxed));
        dg_status s = launch_residual_direct(ctx, variant, q, out, g, dt, A, B, mode, ctx->cap_stream, lam_max, fz);
        cudaGraph_t graph = nullptr;
        const cudaError_t ec = cudaStreamEndCapture(ctx->cap_stream, &graph);
        if (s != DG_OK) {
            if (graph) cudaGraphDestroy(graph);
            return s;
        }
        CK(ec);
        GraphEntry G;
        G.graph = graph;
        G.kernels = ctx->launches - l0;
        G.cur = key;
        ctx->launches = l0;
        const cudaError_t ei = cudaGraphInstantiate(&G.exec, graph, 0);
        if (ei != cudaSuccess) {
            cudaGraphDestroy(graph);
            CK(ei);
        }
        size_t n = 0;
        CK(cudaGraphGetNodes(graph, nullptr, &n));
        std::vector<cudaGraphNode_t> nodes(n);
        CK(cudaGraphGetNodes(graph, nodes.data(), &n));
        for (cudaGraphNode_t nd : nodes) {
            cudaGraphNodeType ty;
            CK(cudaGraphNodeGetType(nd, &ty));
            if (ty == cudaGraphNodeTypeKernel) G.knodes.push_back(nd);
        }
        itg = ctx->graphs.emplace(shape, std::move(G)).first;
    } else if (!same_key(itg->second.cur, key)) {  // re-point the instantiated graph to these arguments
        GraphEntry& G = itg->second;
        for (cudaGraphNode_t nd : G.knodes) {
            cudaKernelNodeParams kp;
            CK(cudaGraphKernelNodeGetParams(nd, &kp));
            if (kp.func == reinterpret_cast<void*>(k_mortar3)) {
                MortarParams M = *static_cast<const MortarParams*>(kp.kernelParams[0]);
                M.q = q;
                void* args[4] = {&M, kp.kernelParams[1], kp.kernelParams[2], kp.kernelParams[3]};
                kp.kernelParams = args;
                CK(cudaGraphExecKernelNodeSetParams(G.exec, nd, &kp));
            } else if (kp.func == reinterpret_cast<void*>(k_face)) {
                FaceParams F = *static_cast<const FaceParams*>(kp.kernelParams[0]);
                F.q = q;
                void* args[1] = {&F};
                kp.kernelParams = args;
                CK(cudaGraphExecKernelNodeSetParams(G.exec, nd, &kp));
            } else {  // k_res_t<N1,N2,N3>(ResParams, int, int, int)
                ResParams R = *static_cast<const ResParams*>(kp.kernelParams[0]);
                R.q = q;
                R.out = out;
                R.g = g;
                R.dt = dt;
                R.rkA = A;
                R.rkB = B;
                R.cfl = fz.cfl;
                if (R.lam_max) R.lam_max = lam_max;  // (null in the buckets that do not write them)
                if (R.lam_in) R.lam_in = fz.lam_in;
                if (R.dt_out) R.dt_out = fz.dt_out;
                if (R.lam_zero) R.lam_zero = fz.lam_zero;
                void* args[4] = {&R, kp.kernelParams[1], kp.kernelParams[2], kp.kernelParams[3]};
                kp.kernelParams = args;
                CK(cudaGraphExecKernelNodeSetParams(G.exec, nd, &kp));
            }
        }
        G.cur = key;
    }
    CK(cudaGraphLaunch(itg->second.exec, st));
    ctx->launches += itg->second.kernels;
    return check_stream_error(ctx, "residual graph launch");
}

dg_status dg_rhs_eval(dg_ctx* ctx, int variant, const double* q_dev, double* qdot_dev, void* stream)
{
    if (!ctx || !q_dev || !qdot_dev) return DG_EINVAL;
    if (!ctx->have_orders) return fail(ctx, DG_ESTATE, "rhs_eval: orders not set");
    if (variant != DG_NONISOLATED && variant != DG_ISOLATED) return fail(ctx, DG_EINVAL, "rhs_eval: variant");
    if (ctx->prm.physics == DG_NS && !ctx->curved) return fail(ctx, DG_EUNSUPPORTED, "rhs_eval: NS needs the curved path");
    return launch_residual(ctx, variant, q_dev, qdot_dev, nullptr, nullptr, 0.0, 0.0, 0, (cudaStream_t)stream);
}

dg_status dg_compute_dt(dg_ctx* ctx, const double* q_dev, double cfl, double* dt_dev, double* dt_host, void* stream)
{
    if (!ctx || !q_dev || !dt_dev || !(cfl > 0)) return DG_EINVAL;
    if (!ctx->have_orders) return fail(ctx, DG_ESTATE, "compute_dt: orders not set");
    cudaStream_t st = (cudaStream_t)stream;
    CK(cudaMemsetAsync(ctx->d_scratch, 0, sizeof(unsigned long long), st));
    CK(cudaMemsetAsync(ctx->d_scratch + 4, 0, 2 * sizeof(unsigned long long), st));  // fused-dt accumulators
    if (ctx->curved) {
        CK(cudaMemsetAsync(ctx->d_scratch + 1, 0, sizeof(unsigned long long), st));
        CDtParams C;
        C.q = q_dev;
        C.orders = ctx->d_orders;
        C.off = ctx->d_off;
        C.met = ctx->d_met;
        C.ph = phys_dev(ctx->prm);
        C.maxbits = ctx->d_scratch;
        k_dt_curved<<<ctx->n_own, CBS, 0, st>>>(C);
        k_dt_final2<<<1, 1, 0, st>>>(ctx->d_scratch, cfl, cfl, dt_dev);
        ctx->launches += 2;
        dg_status s = check_stream_error(ctx, "k_dt_curved launch");
        if (s != DG_OK) return s;
        if (dt_host) {
            CK(cudaMemcpyAsync(dt_host, dt_dev, sizeof(double), cudaMemcpyDeviceToHost, st));
            return admissibility(ctx, st);
        }
        return DG_OK;
    }
    DtParams P;
    P.q = q_dev;
    P.work = ctx->d_work;
    P.elist = ctx->d_elist;
    P.off = ctx->d_off;
    P.hgeo = ctx->d_h;
    P.gamma = ctx->prm.gamma;
    P.maxbits = ctx->d_scratch;
    k_dt<<<ctx->nwork, BLOCK, 0, st>>>(P);
    k_dt_final<<<1, 1, 0, st>>>(ctx->d_scratch, cfl, dt_dev);
    ctx->launches += 2;
    dg_status s = check_stream_error(ctx, "k_dt launch");
    if (s != DG_OK) return s;
    if (dt_host) {
        CK(cudaMemcpyAsync(dt_host, dt_dev, sizeof(double), cudaMemcpyDeviceToHost, st));
        return admissibility(ctx, st);
    }
    return DG_OK;
}

dg_status dg_rk_step(dg_ctx* ctx, double* q_in, double* q_out, double* g, const double* dt_dev, void* stream)
{
    if (!ctx || !q_in || !q_out || !g || !dt_dev || q_in == q_out) return DG_EINVAL;
    if (!ctx->have_orders) return fail(ctx, DG_ESTATE, "rk_step: orders not set");
    if (ctx->prm.physics == DG_NS && !ctx->curved) return fail(ctx, DG_EUNSUPPORTED, "rk_step: NS needs the curved path");
    // Williamson (1980) low-storage RK3 coefficients
    static const double A[3] = {0.0, -5.0 / 9.0, -153.0 / 128.0};
    static const double B[3] = {1.0 / 3.0, 15.0 / 16.0, 8.0 / 15.0};
    cudaStream_t st = (cudaStream_t)stream;
    // stage 1: q_in -> q_out, stage 2: q_out -> q_in, stage 3: q_in -> q_out
    double* src[3] = {q_in, q_out, q_in};
    double* dst[3] = {q_out, q_in, q_out};
    for (int k = 0; k < 3; ++k) {
        dg_status s = launch_residual(ctx, DG_NONISOLATED, src[k], dst[k], g, dt_dev, A[k], B[k], 1, st);
        if (s != DG_OK) return s;
    }
    return DG_OK;
}

dg_status dg_rk_step_dt(dg_ctx* ctx, double* q_in, double* q_out, double* g, const double* dt_dev, double cfl,
                        double* dt_next_dev, void* stream)
{
    if (!ctx || !q_in || !q_out || !g || !dt_dev || !dt_next_dev || q_in == q_out || dt_next_dev == dt_dev || !(cfl > 0))
        return DG_EINVAL;
    if (!ctx->have_orders) return fail(ctx, DG_ESTATE, "rk_step_dt: orders not set");
    if (ctx->prm.physics == DG_NS && !ctx->curved) return fail(ctx, DG_EUNSUPPORTED, "rk_step_dt: NS needs the curved path");
    static const double A[3] = {0.0, -5.0 / 9.0, -153.0 / 128.0};
    static const double B[3] = {1.0 / 3.0, 15.0 / 16.0, 8.0 / 15.0};
    cudaStream_t st = (cudaStream_t)stream;
    double* src[3] = {q_in, q_out, q_in};
    double* dst[3] = {q_out, q_in, q_out};
    for (int k = 0; k < 3; ++k) {
        dg_status s = launch_residual(ctx, DG_NONISOLATED, src[k], dst[k], g, dt_dev, A[k], B[k], 1, st,
                                      k == 2 ? ctx->d_scratch + 4 : nullptr);
        if (s != DG_OK) return s;
    }
    if (ctx->curved) k_dt_final2<<<1, 1, 0, st>>>(ctx->d_scratch + 4, cfl, cfl, dt_next_dev);
    else k_dt_final<<<1, 1, 0, st>>>(ctx->d_scratch + 4, cfl, dt_next_dev);
    ctx->launches++;
    return check_stream_error(ctx, "k_dt_final launch");
}

dg_status dg_rk_steps(dg_ctx* ctx, int nsteps, double* qa, double* qb, double* g, double* dt_a, double* dt_b,
                      double cfl, void* stream)
{
    if (!ctx || nsteps < 1 || !qa || !qb || !g || !dt_a || !dt_b || qa == qb || dt_a == dt_b || !(cfl > 0))
        return DG_EINVAL;
    if (!ctx->have_orders) return fail(ctx, DG_ESTATE, "rk_steps: orders not set");
    if (ctx->prm.physics == DG_NS && !ctx->curved) return fail(ctx, DG_EUNSUPPORTED, "rk_steps: NS needs the curved path");
    static const double A[3] = {0.0, -5.0 / 9.0, -153.0 / 128.0};
    static const double B[3] = {1.0 / 3.0, 15.0 / 16.0, 8.0 / 15.0};
    cudaStream_t st = (cudaStream_t)stream;
    if (ctx->curved) {
        for (int s = 0; s < nsteps; ++s) {
            double* q_in = (s & 1) ? qb : qa;
            double* q_out = (s & 1) ? qa : qb;
            const double* dt = (s & 1) ? dt_b : dt_a;
            double* dt_next = (s & 1) ? dt_a : dt_b;
            double* src[3] = {q_in, q_out, q_in};
            double* dst[3] = {q_out, q_in, q_out};
            for (int k = 0; k < 3; ++k) {
                dg_status r = launch_residual(ctx, DG_NONISOLATED, src[k], dst[k], g, dt, A[k], B[k], 1, st,
                                              k == 2 ? ctx->d_scratch + 4 : nullptr);
                if (r != DG_OK) return r;
            }
            k_dt_final2<<<1, 1, 0, st>>>(ctx->d_scratch + 4, cfl, cfl, dt_next);
            ctx->launches++;
        }
        return check_stream_error(ctx, "k_dt_final launch");
    }
    // Euler: the step size of step s >= 1 is formed by its first stage from
    // the CFL rate the previous step's last stage accumulated (accumulators
    // alternate: acc[s & 1] collects step s); one k_dt_final at the end
    // Both accumulators are zero on entry and on exit: step s >= 1 reads
    // acc[(s-1)&1] in its first stage and zeroes it in its second; the final
    // k_dt_final resets the last one (rk_step_dt / compute_dt use acc[0] too).
    unsigned long long* acc[2] = {ctx->d_scratch + 4, ctx->d_scratch + 5};
    CK(cudaMemsetAsync(acc[0], 0, 2 * sizeof(unsigned long long), st));
    for (int s = 0; s < nsteps; ++s) {
        double* q_in = (s & 1) ? qb : qa;
        double* q_out = (s & 1) ? qa : qb;
        double* dt = (s & 1) ? dt_b : dt_a;
        double* src[3] = {q_in, q_out, q_in};
        double* dst[3] = {q_out, q_in, q_out};
        for (int k = 0; k < 3; ++k) {
            DtFuse fz;
            if (k == 0 && s > 0) {
                fz.lam_in = acc[(s - 1) & 1];
                fz.cfl = cfl;
                fz.dt_out = dt;
            } else if (k == 1 && s > 0) {
                fz.lam_zero = acc[(s - 1) & 1];
            }
            dg_status r = launch_residual(ctx, DG_NONISOLATED, src[k], dst[k], g, dt, A[k], B[k], 1, st,
                                          k == 2 ? acc[s & 1] : nullptr, 0, fz);
            if (r != DG_OK) return r;
        }
    }
    k_dt_final<<<1, 1, 0, st>>>(acc[(nsteps - 1) & 1], cfl, ((nsteps - 1) & 1) ? dt_a : dt_b);
    ctx->launches++;
    return check_stream_error(ctx, "k_dt_final launch");
}

dg_status dg_set_owned(dg_ctx* ctx, int n_owned)
{
    if (ctx) drop_graphs(ctx);
    if (!ctx) return DG_EINVAL;
    if (ctx->E == 0) return fail(ctx, DG_ESTATE, "set_owned: no mesh");
    if (n_owned < 1 || n_owned > ctx->E) return fail(ctx, DG_EINVAL, "set_owned: 1 <= n_owned <= E");
    for (long long i = 0; i < 6LL * n_owned; ++i)
        if (ctx->nbr[i] == -3) return fail(ctx, DG_EINVAL, "set_owned: an owned element has an outside neighbour");
    ctx->n_own = n_owned;
    ctx->have_orders = false;
    return DG_OK;
}

dg_status dg_rk_stage(dg_ctx* ctx, int stage, const double* q_in, double* q_out, double* g, const double* dt_dev,
                      unsigned long long* lam_accum_dev, int flags, void* stream)
{
    if (!ctx || !q_in || !q_out || !g || !dt_dev || q_in == q_out || stage < 0 || stage > 2) return DG_EINVAL;
    if (!ctx->have_orders) return fail(ctx, DG_ESTATE, "rk_stage: orders not set");
    if (ctx->prm.physics == DG_NS && !ctx->curved) return fail(ctx, DG_EUNSUPPORTED, "rk_stage: NS needs the curved path");
    static const double A[3] = {0.0, -5.0 / 9.0, -153.0 / 128.0};
    static const double B[3] = {1.0 / 3.0, 15.0 / 16.0, 8.0 / 15.0};
    if ((flags & (DG_FLAG_FACES_INTERIOR | DG_FLAG_FACES_HALO)) && !ctx->curved)
        return fail(ctx, DG_EUNSUPPORTED, "rk_stage: split face passes need the runtime-order path (dg_set_path)");
    return launch_residual(ctx, DG_NONISOLATED, q_in, q_out, g, dt_dev, A[stage], B[stage], 1, (cudaStream_t)stream,
                           lam_accum_dev, flags & (DG_FLAG_GRADIENT_READY | DG_FLAG_FACES_INTERIOR | DG_FLAG_FACES_HALO));
}

dg_status dg_gradient(dg_ctx* ctx, int variant, const double* q_dev, void* stream)
{
    if (!ctx || !q_dev) return DG_EINVAL;
    if (!ctx->have_orders) return fail(ctx, DG_ESTATE, "gradient: orders not set");
    if (ctx->prm.physics != DG_NS || !ctx->curved) return fail(ctx, DG_EUNSUPPORTED, "gradient: NS on the curved path only");
    return launch_ns_gradient(ctx, variant, q_dev, (cudaStream_t)stream);
}

dg_status dg_gradient_flags(dg_ctx* ctx, int variant, const double* q_dev, int flags, void* stream)
{
    if (!ctx || !q_dev) return DG_EINVAL;
    if (!ctx->have_orders) return fail(ctx, DG_ESTATE, "gradient: orders not set");
    if (ctx->prm.physics != DG_NS || !ctx->curved) return fail(ctx, DG_EUNSUPPORTED, "gradient: NS on the curved path only");
    const int part = (flags & DG_FLAG_FACES_INTERIOR) ? FACES_INTERIOR : ((flags & DG_FLAG_FACES_HALO) ? FACES_HALO : FACES_ALL);
    if (part != FACES_ALL && variant != DG_NONISOLATED) return fail(ctx, DG_EINVAL, "gradient: split face passes are non-isolated");
    return launch_ns_gradient(ctx, variant, q_dev, (cudaStream_t)stream, part);
}

double* dg_gradient_buffer(dg_ctx* ctx) { return ctx ? ctx->d_grad : nullptr; }

dg_status dg_trace_copy(dg_ctx* ctx, const int64_t* entries_dev, int n, double* field_dev, int ncomp, double* buf_dev,
                        int direction, void* stream)
{
    if (!ctx || n < 0 || (n > 0 && (!entries_dev || !field_dev || !buf_dev))) return DG_EINVAL;
    if (ncomp != NV && ncomp != 3 * NV) return fail(ctx, DG_EINVAL, "trace_copy: ncomp must be 5 (state) or 15 (gradient)");
    if (direction != 0 && direction != 1) return fail(ctx, DG_EINVAL, "trace_copy: direction 0 (pack) or 1 (unpack)");
    if (!ctx->have_orders) return fail(ctx, DG_ESTATE, "trace_copy: orders not set");
    if (n == 0) return DG_OK;
    k_trace_copy<<<(n + 3) / 4, 128, 0, (cudaStream_t)stream>>>(reinterpret_cast<const long long*>(entries_dev), n,
                                                                 ctx->d_orders, ctx->d_off, field_dev, ncomp, buf_dev,
                                                                 direction);
    ctx->launches++;
    return check_stream_error(ctx, "k_trace_copy launch");
}

dg_status dg_rhs_eval_flags(dg_ctx* ctx, int variant, const double* q_dev, double* qdot_dev, int flags, void* stream)
{
    if (!ctx || !q_dev || !qdot_dev) return DG_EINVAL;
    if (!ctx->have_orders) return fail(ctx, DG_ESTATE, "rhs_eval: orders not set");
    if ((flags & (DG_FLAG_FACES_INTERIOR | DG_FLAG_FACES_HALO)) && !ctx->curved)
        return fail(ctx, DG_EUNSUPPORTED, "rhs_eval: split face passes need the runtime-order path (dg_set_path)");
    return launch_residual(ctx, variant, q_dev, qdot_dev, nullptr, nullptr, 0.0, 0.0, 0, (cudaStream_t)stream, nullptr,
                           flags & (DG_FLAG_GRADIENT_READY | DG_FLAG_FACES_INTERIOR | DG_FLAG_FACES_HALO));
}

dg_status dg_dt_finalize(dg_ctx* ctx, unsigned long long* lam_accum_dev, double cfl, double* dt_dev, void* stream)
{
    if (!ctx || !lam_accum_dev || !dt_dev || !(cfl > 0)) return DG_EINVAL;
    k_dt_final2<<<1, 1, 0, (cudaStream_t)stream>>>(lam_accum_dev, cfl, cfl, dt_dev);
    ctx->launches++;
    return check_stream_error(ctx, "k_dt_final2 launch");
}

dg_status dg_dt_accumulate(dg_ctx* ctx, const double* q_dev, unsigned long long* lam_accum_dev, void* stream)
{
    if (!ctx || !q_dev || !lam_accum_dev) return DG_EINVAL;
    if (!ctx->have_orders) return fail(ctx, DG_ESTATE, "dt_accumulate: orders not set");
    cudaStream_t st = (cudaStream_t)stream;
    if (ctx->curved) {
        CDtParams C;
        C.q = q_dev;
        C.orders = ctx->d_orders;
        C.off = ctx->d_off;
        C.met = ctx->d_met;
        C.ph = phys_dev(ctx->prm);
        C.maxbits = lam_accum_dev;
        k_dt_curved<<<ctx->n_own, CBS, 0, st>>>(C);
    } else {
        DtParams P;
        P.q = q_dev;
        P.work = ctx->d_work;
        P.elist = ctx->d_elist;
        P.off = ctx->d_off;
        P.hgeo = ctx->d_h;
        P.gamma = ctx->prm.gamma;
        P.maxbits = lam_accum_dev;
        k_dt<<<ctx->nwork, BLOCK, 0, st>>>(P);
    }
    ctx->launches++;
    return check_stream_error(ctx, "dt accumulate launch");
}

dg_status dg_select_local(dg_ctx* ctx, const dg_adapt_policy* pol, const double* tau_dev, double* total_dev,
                          int32_t* orders_out_dev, double* margin_dev, void* stream)
{
    if (!ctx || !pol || !tau_dev || !orders_out_dev) return DG_EINVAL;
    if (!ctx->have_orders) return fail(ctx, DG_ESTATE, "select_local: orders not set");
    if (pol->Nmin < 1 || pol->Nmax > NMAX || pol->Nmin > pol->Nmax || !(pol->tau_max > 0) || pol->dec_cap < 0)
        return fail(ctx, DG_EINVAL, "select_local: bad policy");
    if (pol->mode != DG_SELECT_DYNAMIC && !total_dev) return fail(ctx, DG_EINVAL, "select_local: static needs total map");
    cudaStream_t st = (cudaStream_t)stream;
    CK(cudaMemcpyAsync(orders_out_dev, ctx->d_orders, sizeof(int) * 3LL * ctx->E, cudaMemcpyDeviceToDevice, st));
    SelParams P;
    P.tau = tau_dev;
    P.orders = ctx->d_orders;
    P.total = total_dev;
    P.sel = orders_out_dev;
    P.margin = margin_dev;
    P.E = ctx->n_own;
    P.mode = pol->mode;
    P.tau_max = pol->tau_max;
    P.Nmin = pol->Nmin;
    P.Nmax = pol->Nmax;
    P.dec_cap = pol->dec_cap;
    P.combine = pol->combine;
    P.nstages = pol->nstages;
    k_select<<<(ctx->n_own + 127) / 128, 128, 0, st>>>(P);
    ctx->launches++;
    return check_stream_error(ctx, "k_select launch");
}

dg_status dg_jump_sweep(dg_ctx* ctx, const int32_t* orders_in_dev, int32_t* orders_out_dev, int rule, int Nmax,
                        int32_t* changed_dev, void* stream)
{
    if (!ctx || !orders_in_dev || !orders_out_dev || !changed_dev || orders_in_dev == orders_out_dev) return DG_EINVAL;
    if (ctx->E == 0) return fail(ctx, DG_ESTATE, "jump_sweep: no mesh");
    cudaStream_t st = (cudaStream_t)stream;
    if (ctx->n_own < ctx->E)
        CK(cudaMemcpyAsync(orders_out_dev + 3LL * ctx->n_own, orders_in_dev + 3LL * ctx->n_own,
                           sizeof(int) * 3LL * (ctx->E - ctx->n_own), cudaMemcpyDeviceToDevice, st));
    k_jump<<<(ctx->n_own + 127) / 128, 128, 0, st>>>(ctx->d_nbr, orders_in_dev, orders_out_dev, ctx->n_own,
                                                      rule == DG_JUMP_A ? 0 : 1, Nmax, changed_dev);
    ctx->launches++;
    return check_stream_error(ctx, "k_jump launch");
}

// Non-isolated tau-estimation (dg_tau_opts.coarse_faces = 1, reading R7):
// per coarse level (d, p) the state and the reference residual are
// interpolated to the level's layout (k_transfer), the level's sub-context
// evaluates the full (face-coupled) residual there, and k_tau_level takes
// the per-element maxima.  Sub-contexts are built once per fine layout.
// one coarse level (d, p): the whole mesh at O(e) = N(e), O_d = min(p, N_d(e))
static dg_status build_level(dg_ctx* ctx, int d, int p, dg_ctx::CoarseLevel& L)
{
    const int E = ctx->E;
    L.d = d;
    L.p = p;
    std::vector<int32_t> oc(ctx->orders.begin(), ctx->orders.end());
    std::vector<long long> offc(E + 1, 0);
    for (int e = 0; e < E; ++e) {
        const int* a = &ctx->orders[3 * e];
        oc[3 * e + d] = std::min(p, a[d]);
        offc[e + 1] = offc[e] + (long long)NV * npts(&oc[3 * e]);
        L.smax = std::max(L.smax, npts(a));  // every transfer intermediate fits the fine element
    }
    dg_status s = dg_create(&ctx->prm, &L.sub);
    if (s != DG_OK) return fail(ctx, s, "tau_estimate: coarse level context");
    L.sub->path = ctx->path;
    if (ctx->curved) lend_scratch(ctx, L.sub);
    if ((s = dg_mesh_upload(L.sub, E, ctx->nbr.data(), ctx->gorder, ctx->geo.data())) != DG_OK ||
        (ctx->n_own < E && (s = dg_set_owned(L.sub, ctx->n_own)) != DG_OK) ||
        (s = dg_set_orders(L.sub, oc.data())) != DG_OK)
        return fail(ctx, s, std::string("tau_estimate: coarse level: ") + dg_last_error(L.sub));
    if (upload(L.d_orders, oc) != cudaSuccess || upload(L.d_off, offc) != cudaSuccess)
        return fail(ctx, DG_ECUDA, "tau_estimate: coarse level tables");
    return DG_OK;
}

static void free_level(dg_ctx* ctx, dg_ctx::CoarseLevel& L)
{
    unlend_scratch(ctx, L.sub);
    dg_destroy(L.sub);
    L.sub = nullptr;
    dfree(L.d_orders);
    dfree(L.d_off);
}

// phase 0: the state and the reference residual interpolated to the level's
// layout (k_transfer); NS: the level's BR1 gradient of the owned elements.
static dg_status level_phase0(dg_ctx* ctx, const dg_ctx::CoarseLevel& L, int restr, const double* q_dev, const double* ref,
                              cudaStream_t st)
{
    const int E = ctx->E;
    const long long len = ctx->off[E];
    double* qc = ctx->d_cq;
    double* rc = qc + len;
    TransferParams T;
    T.oold = ctx->d_orders;
    T.onew = L.d_orders;
    T.offold = ctx->d_off;
    T.offnew = L.d_off;
    T.tab = ctx->d_tab;
    T.smax0 = T.smax1 = T.smax2 = L.smax;
    T.restr = restr;
    const size_t sm = sizeof(double) * NV * 3 * (size_t)L.smax;
    T.qold = q_dev;
    T.qnew = qc;
    k_transfer<<<E, BLOCK, sm, st>>>(T);
    T.qold = ref;
    T.qnew = rc;
    k_transfer<<<E, BLOCK, sm, st>>>(T);
    ctx->launches += 2;
    if (ctx->prm.physics == DG_NS && L.sub->curved) {
        dg_status s = dg_gradient(L.sub, DG_NONISOLATED, qc, st);
        if (s != DG_OK) return fail(ctx, s, std::string("tau_estimate: coarse gradient: ") + dg_last_error(L.sub));
        ctx->launches += L.sub->launches;
        L.sub->launches = 0;
    }
    return check_stream_error(ctx, "non-isolated tau launch");
}

// phase 1: the level's face-coupled residual (its gradient ready) and the
// per-element maxima |T R - Qdot_c| of the owned elements (k_tau_level).
static dg_status level_phase1(dg_ctx* ctx, const dg_ctx::CoarseLevel& L, int formulation, double* tau_dev, cudaStream_t st)
{
    const long long len = ctx->off[ctx->E];
    double* qc = ctx->d_cq;
    double* rc = qc + len;
    double* dc = rc + len;
    const int flags = (ctx->prm.physics == DG_NS && L.sub->curved) ? DG_FLAG_GRADIENT_READY : 0;
    dg_status s = launch_residual(L.sub, DG_NONISOLATED, qc, dc, nullptr, nullptr, 0.0, 0.0, 0, st, nullptr, flags);
    if (s != DG_OK) return fail(ctx, s, std::string("tau_estimate: coarse residual: ") + dg_last_error(L.sub));
    ctx->launches += L.sub->launches;
    L.sub->launches = 0;
    k_tau_level<<<ctx->n_own, 128, 0, st>>>(rc, dc, ctx->d_orders, L.d_orders, L.d_off, L.d, L.p, formulation, ctx->d_h,
                                            ctx->curved ? L.sub->d_met : nullptr, ctx->d_tab, tau_dev);
    ctx->launches++;
    return check_stream_error(ctx, "non-isolated tau launch");
}

static dg_status run_level(dg_ctx* ctx, const dg_ctx::CoarseLevel& L, int formulation, int restr, const double* q_dev,
                           const double* ref, double* tau_dev, cudaStream_t st)
{
    dg_status s = level_phase0(ctx, L, restr, q_dev, ref, st);
    if (s != DG_OK) return s;
    return level_phase1(ctx, L, formulation, tau_dev, st);
}

static dg_status ensure_cq(dg_ctx* ctx)
{
    const long long len = ctx->off[ctx->E];
    if (ctx->c_len < 3 * len) {
        dfree(ctx->d_cq);
        CK(cudaMalloc(&ctx->d_cq, sizeof(double) * 3 * len));
        ctx->c_len = 3 * len;
    }
    return DG_OK;
}

// Non-isolated tau-estimation (dg_tau_opts.coarse_faces = 1, reading R7):
// per coarse level (d, p) the state and the reference residual are
// interpolated to the level's layout (k_transfer), the level's sub-context
// evaluates the full (face-coupled) residual there, and k_tau_level takes
// the per-element maxima.  The sub-contexts stay resident across calls (built
// once per fine layout); when they do not all fit in device memory (cfg5:
// 15 levels of a 42.5 M DOF mesh) the levels are built, run and freed one at
// a time instead.
static dg_status tau_noniso(dg_ctx* ctx, int formulation, int restr, const double* q_dev, const double* ref,
                            double* tau_dev, cudaStream_t st)
{
    if (ctx->n_own != ctx->E)
        return fail(ctx, DG_EUNSUPPORTED, "tau_estimate: non-isolated levels on a rank-local mesh: use dg_tau_level "
                                          "(the coarse gradient traces are exchanged between its two phases)");
    const int E = ctx->E;
    if (ensure_cq(ctx) != DG_OK) return DG_ECUDA;
    int nmax[3] = {0, 0, 0};
    for (int e = 0; e < E; ++e)
        for (int d = 0; d < 3; ++d) nmax[d] = std::max(nmax[d], ctx->orders[3 * e + d]);
    if (ctx->coarse_stream_force) ctx->coarse_streaming = true;
    if (ctx->coarse.empty() && !ctx->coarse_streaming) {
        for (int d = 0; d < 3 && !ctx->coarse_streaming; ++d)
            for (int p = 1; p < nmax[d]; ++p) {
                dg_ctx::CoarseLevel L;
                const dg_status s = build_level(ctx, d, p, L);
                ctx->coarse.push_back(L);  // owned from here (drop_coarse frees it)
                if (s == DG_ECUDA) {       // out of device memory: stream the levels instead
                    drop_coarse(ctx);
                    cudaGetLastError();
                    ctx->coarse_streaming = true;
                    break;
                }
                if (s != DG_OK) {
                    drop_coarse(ctx);
                    return s;
                }
            }
    }
    if (!ctx->coarse_streaming) {
        for (const dg_ctx::CoarseLevel& L : ctx->coarse) {
            const dg_status s = run_level(ctx, L, formulation, restr, q_dev, ref, tau_dev, st);
            if (s != DG_OK) return s;
        }
        return DG_OK;
    }
    for (int d = 0; d < 3; ++d)
        for (int p = 1; p < nmax[d]; ++p) {
            dg_ctx::CoarseLevel L;
            dg_status s = build_level(ctx, d, p, L);
            if (s == DG_OK) s = run_level(ctx, L, formulation, restr, q_dev, ref, tau_dev, st);
            CK(cudaStreamSynchronize(st));  // the level's buffers are in use until here
            free_level(ctx, L);
            if (s != DG_OK) return s;
        }
    return DG_OK;
}

dg_status dg_tau_estimate(dg_ctx* ctx, const dg_tau_opts* o, const double* q_dev, const double* qref_dev, double* tau_dev,
                          void* stream)
{
    if (!ctx || !o || !q_dev || !tau_dev) return DG_EINVAL;
    if (!ctx->have_orders) return fail(ctx, DG_ESTATE, "tau_estimate: orders not set");
    if (o->reference == DG_REF_SOLVER && !qref_dev) return fail(ctx, DG_EINVAL, "tau_estimate: SOLVER needs qdot_ref");
    if (ctx->prm.physics == DG_NS && !ctx->curved) return fail(ctx, DG_EUNSUPPORTED, "tau_estimate: NS needs the curved path");
    if (o->restriction != 0 && o->restriction != 1) return fail(ctx, DG_EINVAL, "tau_estimate: restriction");
    {
        cudaStream_t st = (cudaStream_t)stream;
        const double* ref = qref_dev;
        if (o->reference == DG_REF_SAME) {  // isolated fine residual first (reading A4)
            if (ctx->ref_len < ctx->off[ctx->E]) {
                dfree(ctx->d_ref_scratch);
                CK(cudaMalloc(&ctx->d_ref_scratch, sizeof(double) * ctx->off[ctx->E]));
                ctx->ref_len = ctx->off[ctx->E];
            }
            dg_status s = launch_residual(ctx, DG_ISOLATED, q_dev, ctx->d_ref_scratch, nullptr, nullptr, 0.0, 0.0, 0, st);
            if (s != DG_OK) return s;
            ref = ctx->d_ref_scratch;
        }
        k_tau_norm<<<ctx->n_own, 128, 0, st>>>(ref, tau_dev, ctx->d_orders, ctx->d_off);
        ctx->launches++;
        if (o->coarse_faces) return tau_noniso(ctx, o->formulation, o->restriction, q_dev, ref, tau_dev, st);
        if (ctx->tau_curved && ctx->nlevels > 0) {
            const size_t sm = sizeof(double) * ((ctx->prm.physics == DG_NS ? 40 : 30) * (size_t)ctx->max_level + (ctx->max_level + 1) / 2);
            if ((long long)sm > ctx->smem_limit) return fail(ctx, DG_EUNSUPPORTED, "tau_estimate: coarse level too large for shared memory");
            CTauParams C;
            C.tdd = ctx->d_tdd;
            C.q = q_dev;
            C.qref = ref;
            C.tau = tau_dev;
            C.orders = ctx->d_orders;
            C.off = ctx->d_off;
            C.levels = ctx->d_levels;
            C.cm = curved_mesh(ctx);
            C.tab = ctx->d_tab;
            C.formulation = o->formulation;
            C.restr = o->restriction;
            C.ph = phys_dev(ctx->prm);
            // extruded meshes: compact double-double coarse metrics (k_tau_ext);
            // DGTAU_TAU_GENERIC=1 keeps the generic 3-D kernel (tests run both)
            const bool ext = ctx->extruded && !getenv_flag("DGTAU_TAU_GENERIC");
            const size_t gsm = tau_grp_bytes(ctx->tgrp_cap);
            if (ext && ctx->ntgrp > 0 && !getenv_flag("DGTAU_TAU_PERLEVEL") && (long long)gsm <= ctx->smem_limit) {
                C.levels = ctx->d_tgrp;
                C.lbase = 0;
                k_tau_grp<<<ctx->ntgrp, TAU_GRP_BS, gsm, st>>>(C, ctx->tgrp_cap);
                ctx->launches++;
            } else
            for (const SizeClass& c : ctx->lcls) {
                C.lbase = c.base;
                if (ext) {
                    const size_t smc = sizeof(double) * tau_ext_words(c.maxn, ctx->prm.physics == DG_NS);
                    if (c.maxn <= 64) k_tau_ext<64><<<c.count, 64, smc, st>>>(C);
                    else if (c.maxn <= 160) k_tau_ext<128><<<c.count, 128, smc, st>>>(C);
                    else k_tau_ext<256><<<c.count, 256, smc, st>>>(C);
                } else {
                    const size_t smc = sizeof(double) * ((ctx->prm.physics == DG_NS ? 40 : 30) * (size_t)c.maxn + (c.maxn + 1) / 2);
                    if (c.maxn <= 64) k_tau_curved<64><<<c.count, 64, smc, st>>>(C);
                    else if (c.maxn <= 160) k_tau_curved<128><<<c.count, 128, smc, st>>>(C);
                    else k_tau_curved<256><<<c.count, 256, smc, st>>>(C);
                }
                ctx->launches++;
            }
        } else if (ctx->ntgroups > 0) {
            Tau5Params P;
            P.q = q_dev;
            P.qref = ref;
            P.tau = tau_dev;
            P.orders = ctx->d_orders;
            P.off = ctx->d_off;
            P.hgeo = ctx->d_h;
            P.groups = ctx->d_tgroups;
            P.tab = ctx->d_tab;
            P.formulation = o->formulation;
            P.restr = o->restriction;
            P.gm1 = ctx->prm.gamma - 1.0;
            k_tau5<<<ctx->ntgroups, TAU5_BS, ctx->tau5_smem, st>>>(P);
        }
    }
    ctx->launches++;
    return check_stream_error(ctx, "k_tau launch");
}

// Non-isolated tau level (d, p) in two phases for rank-local meshes (SURVEY
// 8(f) rank 1, include/dgtau.h): phase 0 builds the level's context once per
// layout (the rank's local mesh at the level's orders, owned count kept),
// moves q and R to the level's layout and (NS) forms the level's BR1
// gradient of the owned elements; the caller refreshes the halo face traces
// of that gradient; phase 1 evaluates the level's residual and writes
// tau[e][d][p] of the owned elements.
dg_status dg_tau_level(dg_ctx* ctx, int d, int p, int phase, const dg_tau_opts* o, const double* q_dev,
                       const double* qref_dev, double* tau_dev, dg_ctx** level_out, void* stream)
{
    if (!ctx || !o || d < 0 || d > 2 || p < 1 || (phase != 0 && phase != 1)) return DG_EINVAL;
    if (!ctx->have_orders) return fail(ctx, DG_ESTATE, "tau_level: orders not set");
    if (phase == 0 && (!q_dev || !qref_dev)) return fail(ctx, DG_EINVAL, "tau_level: q and the SOLVER reference needed");
    if (phase == 1 && !tau_dev) return fail(ctx, DG_EINVAL, "tau_level: tau needed");
    cudaStream_t st = (cudaStream_t)stream;
    if (ensure_cq(ctx) != DG_OK) return DG_ECUDA;
    dg_ctx::CoarseLevel* L = nullptr;
    for (auto& c : ctx->coarse)
        if (c.d == d && c.p == p) L = &c;
    if (!L) {
        if (phase == 1) return fail(ctx, DG_ESTATE, "tau_level: phase 1 before phase 0");
        dg_ctx::CoarseLevel nl;
        const dg_status s = build_level(ctx, d, p, nl);
        ctx->coarse.push_back(nl);  // owned from here (drop_coarse frees it)
        if (s != DG_OK) return s;
        L = &ctx->coarse.back();
    }
    if (level_out) *level_out = L->sub;
    if (phase == 0) return level_phase0(ctx, *L, o->restriction, q_dev, qref_dev, st);
    return level_phase1(ctx, *L, o->formulation, tau_dev, st);
}

dg_status dg_select_orders(dg_ctx* ctx, const dg_adapt_policy* pol, const double* tau_dev, double* total_dev,
                           int32_t* orders_out, double* margin_host, void* stream)
{
    if (!ctx || !pol || !tau_dev) return DG_EINVAL;
    if (!ctx->have_orders) return fail(ctx, DG_ESTATE, "select_orders: orders not set");
    if (pol->Nmin < 1 || pol->Nmax > NMAX || pol->Nmin > pol->Nmax || !(pol->tau_max > 0) || pol->dec_cap < 0)
        return fail(ctx, DG_EINVAL, "select_orders: bad policy");
    if (pol->mode < DG_SELECT_DYNAMIC || pol->mode > DG_SELECT_A1_FINAL || (pol->combine != DG_COMBINE_MAX &&
        pol->combine != DG_COMBINE_AV) || (pol->combine == DG_COMBINE_AV && pol->nstages < 1 &&
        (pol->mode == DG_SELECT_STATIC_FINAL || pol->mode == DG_SELECT_A1_FINAL)))
        return fail(ctx, DG_EINVAL, "select_orders: bad mode / combine / nstages");
    if (pol->mode != DG_SELECT_DYNAMIC && !total_dev) return fail(ctx, DG_EINVAL, "select_orders: static needs total map");
    const bool accum_only = pol->mode == DG_SELECT_STATIC_ACCUM || pol->mode == DG_SELECT_A1_ACCUM;
    if (!accum_only && !orders_out) return fail(ctx, DG_EINVAL, "select_orders: orders_out");
    cudaStream_t st = (cudaStream_t)stream;
    const int E = ctx->E;
    SelParams P;
    P.tau = tau_dev;
    P.orders = ctx->d_orders;
    P.total = total_dev;
    P.sel = ctx->d_sel;
    P.margin = ctx->d_margin;
    P.E = ctx->n_own;
    P.mode = pol->mode;
    P.tau_max = pol->tau_max;
    P.Nmin = pol->Nmin;
    P.Nmax = pol->Nmax;
    P.dec_cap = pol->dec_cap;
    P.combine = pol->combine;
    P.nstages = pol->nstages;
    // halo rows (multi-rank local meshes) keep their current orders
    if (ctx->n_own < E)
        CK(cudaMemcpyAsync(ctx->d_sel + 3LL * ctx->n_own, ctx->d_orders + 3LL * ctx->n_own,
                           sizeof(int) * 3LL * (E - ctx->n_own), cudaMemcpyDeviceToDevice, st));
    k_select<<<(ctx->n_own + 127) / 128, 128, 0, st>>>(P);
    ctx->launches++;
    dg_status s = check_stream_error(ctx, "k_select launch");
    if (s != DG_OK) return s;
    if (accum_only) return DG_OK;
    // jump-condition fixpoint: Jacobi sweeps until no element changes
    int* a = ctx->d_sel;
    int* b = ctx->d_sel + 3LL * E;
    if (ctx->n_own == E && E <= (1 << 18)) {  // one launch, no host round trips
        k_jump_fix<<<1, JUMP_FIX_BS, 0, st>>>(ctx->d_nbr, a, b, E, pol->jump_rule == DG_JUMP_A ? 0 : 1, pol->Nmax, 64);
        ctx->launches++;
    } else
    for (int sweep = 0; sweep < 64; ++sweep) {
        CK(cudaMemsetAsync(ctx->d_flag + 2, 0, sizeof(int), st));
        if (ctx->n_own < E)
            CK(cudaMemcpyAsync(b + 3LL * ctx->n_own, a + 3LL * ctx->n_own, sizeof(int) * 3LL * (E - ctx->n_own),
                               cudaMemcpyDeviceToDevice, st));
        k_jump<<<(ctx->n_own + 127) / 128, 128, 0, st>>>(ctx->d_nbr, a, b, ctx->n_own,
                                                          pol->jump_rule == DG_JUMP_A ? 0 : 1, pol->Nmax, ctx->d_flag + 2);
        ctx->launches++;
        int changed = 0;
        CK(cudaMemcpyAsync(&changed, ctx->d_flag + 2, sizeof(int), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        std::swap(a, b);
        if (!changed) break;
    }
    CK(cudaMemcpyAsync(orders_out, a, sizeof(int) * 3LL * E, cudaMemcpyDeviceToHost, st));
    if (margin_host) CK(cudaMemcpyAsync(margin_host, ctx->d_margin, sizeof(double) * E, cudaMemcpyDeviceToHost, st));
    return admissibility(ctx, st);
}

dg_status dg_transfer(dg_ctx* ctx, const int32_t* new_orders, const double* q_old, double* q_new, void* stream)
{
    if (!ctx || !new_orders || !q_old || !q_new) return DG_EINVAL;
    if (!ctx->have_orders) return fail(ctx, DG_ESTATE, "transfer: orders not set");
    const int E = ctx->E;
    std::vector<long long>& offn = ctx->tr_off_host;  // persistent: outlives the async copy
    offn.assign(E + 1, 0);
    int smax[3] = {1, 1, 1};  // shared memory sized to this transfer's largest element passes
    for (int e = 0; e < E; ++e) {
        for (int d = 0; d < 3; ++d)
            if (new_orders[3 * e + d] < 1 || new_orders[3 * e + d] > NMAX) return fail(ctx, DG_EINVAL, "transfer: order");
        offn[e + 1] = offn[e] + (long long)NV * npts(&new_orders[3 * e]);
        const int* a = &ctx->orders[3 * e];
        const int* b = &new_orders[3 * e];
        // every intermediate of the passes fits prod_d max(A_d, B_d) nodes
        const int m = (std::max(a[0], b[0]) + 1) * (std::max(a[1], b[1]) + 1) * (std::max(a[2], b[2]) + 1);
        smax[0] = smax[1] = smax[2] = std::max(smax[0], m);
    }
    cudaStream_t st = (cudaStream_t)stream;
    if (!ctx->d_tr_orders) {
        CK(cudaMalloc(&ctx->d_tr_orders, sizeof(int) * 3LL * E));
        CK(cudaMalloc(&ctx->d_tr_off, sizeof(long long) * (E + 1)));
    }
    int* d_on = ctx->d_tr_orders;
    long long* d_offn = ctx->d_tr_off;
    ctx->tr_orders_host.assign(new_orders, new_orders + 3LL * E);
    CK(cudaMemcpyAsync(d_on, ctx->tr_orders_host.data(), sizeof(int) * 3LL * E, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_offn, offn.data(), sizeof(long long) * (E + 1), cudaMemcpyHostToDevice, st));
    TransferParams P;
    P.qold = q_old;
    P.qnew = q_new;
    P.oold = ctx->d_orders;
    P.onew = d_on;
    P.offold = ctx->d_off;
    P.offnew = d_offn;
    P.tab = ctx->d_tab;
    P.smax0 = smax[0];
    P.smax1 = smax[1];
    P.smax2 = smax[2];
    P.restr = 0;
    k_transfer<<<E, BLOCK, sizeof(double) * NV * (size_t)(smax[0] + smax[1] + smax[2]), st>>>(P);
    ctx->launches++;
    return check_stream_error(ctx, "k_transfer launch");
}

dg_status dg_diagnostics(dg_ctx* ctx, const double* q_dev, const double* v_dev, double* sums_host, double* minrp_host,
                         void* stream)
{
    if (!ctx || !q_dev) return DG_EINVAL;
    if (!ctx->have_orders) return fail(ctx, DG_ESTATE, "diagnostics: orders not set");
    cudaStream_t st = (cudaStream_t)stream;
    CK(cudaMemsetAsync(ctx->d_sums, 0, 5 * sizeof(double), st));
    CK(cudaMemsetAsync(ctx->d_scratch + 1, 0xff, 2 * sizeof(unsigned long long), st));
    CK(cudaMemsetAsync(ctx->d_flag + 3, 0, sizeof(int), st));
    DiagParams P;
    P.q = q_dev;
    P.v = v_dev;
    P.orders = ctx->d_orders;
    P.off = ctx->d_off;
    P.hgeo = ctx->d_h;
    P.met = ctx->curved ? ctx->d_met : nullptr;
    P.tab = ctx->d_tab;
    P.gamma = ctx->prm.gamma;
    P.sums = ctx->d_sums;
    P.minbits = ctx->d_scratch + 1;
    P.neg = ctx->d_flag + 3;
    k_diag<<<ctx->n_own, 128, 0, st>>>(P);
    ctx->launches++;
    dg_status s = check_stream_error(ctx, "k_diag launch");
    if (s != DG_OK) return s;
    double sums[5];
    unsigned long long mb[2];
    int neg = 0, flag[2];
    CK(cudaMemcpyAsync(sums, ctx->d_sums, sizeof(sums), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(mb, ctx->d_scratch + 1, sizeof(mb), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&neg, ctx->d_flag + 3, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(flag, ctx->d_flag, sizeof(flag), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (sums_host) std::memcpy(sums_host, sums, sizeof(sums));
    if (minrp_host) {
        long long b0 = (long long)mb[0], b1 = (long long)mb[1];
        std::memcpy(&minrp_host[0], &b0, sizeof(double));
        std::memcpy(&minrp_host[1], &b1, sizeof(double));
    }
    if (neg > 0 || flag[0] > 0) {
        CK(cudaMemsetAsync(ctx->d_flag, 0, 2 * sizeof(int), st));
        return fail(ctx, DG_EADMISSIBLE,
                    "inadmissible state (rho<=0 or p<=0) at " + std::to_string(neg) + " nodes; first flagged element " +
                        std::to_string(flag[1]));
    }
    return DG_OK;
}

}  // extern "C"
