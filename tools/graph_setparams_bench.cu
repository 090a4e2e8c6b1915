// Micro-benchmark: cost of re-pointing an instantiated CUDA graph (one
// cudaGraphExecKernelNodeSetParams per kernel node) against capturing and
// instantiating it again -- the two ways to reuse a per-layout residual graph
// for a new (q, out) buffer pair.
#include <chrono>
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

struct Big { const double* q; double* out; double pad[24]; };

__global__ void k_dummy(Big p, int a, int b, int c) { if (threadIdx.x == 0 && blockIdx.x == 0 && a < 0) p.out[0] = p.q[0] + b + c; }

int main()
{
    const int NODES = 300;
    cudaStream_t s, cap;
    cudaStreamCreate(&s);
    cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking);
    double *q, *o;
    cudaMalloc(&q, 1024);
    cudaMalloc(&o, 1024);
    Big p{};
    p.q = q; p.out = o;
    auto capture = [&](cudaGraph_t& g, cudaGraphExec_t& e) {
        cudaStreamBeginCapture(cap, cudaStreamCaptureModeRelaxed);
        for (int i = 0; i < NODES; ++i) k_dummy<<<1, 32, 0, cap>>>(p, i, 1, 2);
        cudaStreamEndCapture(cap, &g);
        cudaGraphInstantiate(&e, g, 0);
    };
    cudaGraph_t g; cudaGraphExec_t e;
    capture(g, e);
    cudaGraphLaunch(e, s); cudaStreamSynchronize(s);
    // recapture + instantiate
    auto t0 = std::chrono::high_resolution_clock::now();
    for (int r = 0; r < 20; ++r) { cudaGraph_t g2; cudaGraphExec_t e2; capture(g2, e2); cudaGraphExecDestroy(e2); cudaGraphDestroy(g2); }
    auto t1 = std::chrono::high_resolution_clock::now();
    // repoint all nodes
    size_t n = 0;
    cudaGraphGetNodes(g, nullptr, &n);
    std::vector<cudaGraphNode_t> nodes(n);
    cudaGraphGetNodes(g, nodes.data(), &n);
    auto t2 = std::chrono::high_resolution_clock::now();
    for (int r = 0; r < 20; ++r) {
        for (auto nd : nodes) {
            cudaKernelNodeParams kp;
            cudaGraphKernelNodeGetParams(nd, &kp);
            Big b = *static_cast<Big*>(kp.kernelParams[0]);
            b.out = (r & 1) ? q : o;
            void* args[4] = {&b, kp.kernelParams[1], kp.kernelParams[2], kp.kernelParams[3]};
            kp.kernelParams = args;
            cudaGraphExecKernelNodeSetParams(e, nd, &kp);
        }
    }
    auto t3 = std::chrono::high_resolution_clock::now();
    cudaGraphLaunch(e, s);
    cudaError_t err = cudaStreamSynchronize(s);
    printf("nodes %zu: capture+instantiate %.3f ms, repoint %.3f ms (%s)\n", n,
           std::chrono::duration<double, std::milli>(t1 - t0).count() / 20,
           std::chrono::duration<double, std::milli>(t3 - t2).count() / 20, cudaGetErrorString(err));
    return 0;
}
