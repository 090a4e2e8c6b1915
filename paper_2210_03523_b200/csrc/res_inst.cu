// res_inst.cu -- instantiation unit of the order-specialised residual kernels
// k_res_t<RES_N1, N2, N3>, N2, N3 in 1..8 (residual_t.cuh).  The build
// compiles it once per RES_N1 = 1..8 (nvcc -DRES_N1=k), so the 512 instances
// build in parallel; res_setup_<RES_N1> fills the launch / occupancy tables.
#include "residual_t.cuh"

#ifndef RES_N1
#error "compile with -DRES_N1=1..8"
#endif

namespace dgtau {

namespace {  // internal linkage: every RES_N1 unit has its own ResInst<K>

template <int K>
struct ResInst {  // K = 8 (N2 - 1) + (N3 - 1)
    static cudaError_t run(res_launcher (*tab)[NP][NP], res_occupancy (*occ)[NP][NP])
    {
        constexpr int N2 = K / 8 + 1, N3 = K % 8 + 1;
        tab[RES_N1][N2][N3] = launch_res_t<RES_N1, N2, N3>;
        occ[RES_N1][N2][N3] = occ_res_t<RES_N1, N2, N3>;
        cudaError_t e = attr_res_t<RES_N1, N2, N3>();
        if (e != cudaSuccess) return e;
        return ResInst<K + 1>::run(tab, occ);
    }
};
template <>
struct ResInst<64> {
    static cudaError_t run(res_launcher (*)[NP][NP], res_occupancy (*)[NP][NP]) { return cudaSuccess; }
};

}  // namespace

#define RES_CAT2(a, b) a##b
#define RES_CAT(a, b) RES_CAT2(a, b)
cudaError_t RES_CAT(res_setup_, RES_N1)(const Tables* host, res_launcher (*tab)[NP][NP], res_occupancy (*occ)[NP][NP])
{
    cudaError_t e = res_copy_constants(host);
    if (e != cudaSuccess) return e;
    return ResInst<0>::run(tab, occ);
}

}  // namespace dgtau
