// pattern_probe_pairs.cu -- can two CTAs share the 128-byte runs of a strided
// column tile?  (For a 3-sweep N = 2^28 schedule: a 2^10-point sub-problem
// tile of 32 fp32 columns is 256 KiB per plane pair -- too big for one CTA --
// but two CTAs of a cluster could take 16 columns (64-byte half-runs) each.)
// No arithmetic: CTA b copies columns of a [SUB][n/SUB] view, both planes,
//   read in[j + e*RS], write out[j + e*RS]  (TJ*4-byte runs, RS apart).
// Variants:
//   solo  TJ=32: one CTA per 128-byte run (the reference point)
//   solo  TJ=16: 64-byte runs, neighbours unsynchronised (pattern_probe_runs.cu)
//   pair  TJ=16: 2-CTA clusters, the two halves of each 128-byte run, the
//                pair kept in step by a cluster barrier every chunk
//   load policy: .cs (evict-first) or default caching
// usage: pattern_probe_pairs
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

namespace cg = cooperative_groups;
constexpr int NT = 256, K = 16;

template <bool CS>
__device__ __forceinline__ float ld(const float *p)
{
    if constexpr (CS) return __ldcs(p);
    else return *p;
}

template <int TJ, int SUB, bool PAIR, bool CS>
__global__ void __launch_bounds__(NT) probe(const float *__restrict__ ir, const float *__restrict__ ii,
                                            float *__restrict__ orr, float *__restrict__ oi, int64_t rs)
{
    constexpr int ROWS = NT / TJ;
    constexpr int CHUNK_ROWS = ROWS * K;
    const int tid = threadIdx.x, jl = tid % TJ, t = tid / TJ;
    const int64_t j = (int64_t)blockIdx.x * TJ + jl;
#pragma unroll 1
    for (int c = 0; c < SUB; c += CHUNK_ROWS) {
        if constexpr (PAIR) cg::this_cluster().sync();
        float vr[K], vi[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int64_t a = j + (int64_t)(c + t + ROWS * k) * rs;
            vr[k] = ld<CS>(ir + a);
            vi[k] = ld<CS>(ii + a);
        }
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int64_t a = j + (int64_t)(c + t + ROWS * k) * rs;
            __stcs(orr + a, vr[k]);
            __stcs(oi + a, vi[k]);
        }
    }
}

template <int TJ, int SUB, bool PAIR, bool CS>
static void run(float *b[4], int64_t n, const char *name)
{
    const int64_t rs = n / SUB, blocks = rs / TJ;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)blocks);
    cfg.blockDim = dim3(NT);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = PAIR ? 2 : 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    auto k = probe<TJ, SUB, PAIR, CS>;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int w = 0; w < 3; ++w) cudaLaunchKernelEx(&cfg, k, (const float *)b[0], (const float *)b[1], b[2], b[3], rs);
    const int it = 10;
    cudaEventRecord(e0);
    for (int w = 0; w < it; ++w) cudaLaunchKernelEx(&cfg, k, (const float *)b[0], (const float *)b[1], b[2], b[3], rs);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= it;
    cudaError_t err = cudaGetLastError();
    printf("%-5s TJ=%2d (%3d B runs) SUB=%5d loads=%s  %8.3f ms  %7.1f GB/s %s\n", name, TJ, TJ * 4, SUB,
           CS ? "cs " : "def", ms, 16.0 * n / (ms * 1e6), err == cudaSuccess ? "" : cudaGetErrorString(err));
}

int main()
{
    const int64_t n = int64_t(1) << 28;
    float *b[4];
    for (int k = 0; k < 4; ++k) {
        if (cudaMalloc(&b[k], n * sizeof(float)) != cudaSuccess) return 1;
        cudaMemset(b[k], 0, n * sizeof(float));
    }
    for (int rep = 0; rep < 2; ++rep) {
        run<32, 1024, false, true>(b, n, "solo");
        run<32, 1024, false, false>(b, n, "solo");
        run<16, 1024, false, true>(b, n, "solo");
        run<16, 1024, false, false>(b, n, "solo");
        run<16, 1024, true, true>(b, n, "pair");
        run<16, 1024, true, false>(b, n, "pair");
        run<32, 512, false, true>(b, n, "solo");
        run<16, 512, true, false>(b, n, "pair");
        run<32, 128, false, true>(b, n, "solo");
    }
    return 0;
}
