// pattern_probe_runs.cu -- HBM efficiency of strided-run access patterns as a
// function of the run width, for choosing the column-tile width TJ of a
// 3-group (L = 10/9/9) schedule of the 2^28-point transform.  No arithmetic:
// CTA b owns columns j0 = b*TJ .. j0+TJ-1 of a [SUB][n/SUB] view (SUB = 2^L
// sub-problem points, stride n/SUB) and copies them, both fp32 planes, with
//   read  in [j + e*RS]    (TJ*4-byte runs, RS apart)
//   write out[j + e*WS]    (same)  or  out[j*SUB + e] (contiguous, "wc")
// usage: pattern_probe_runs   (prints GB/s per (TJ, SUB); 2 x 1 GiB planes in, 2 out)
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>

constexpr int NT = 256, K = 16;

template <int TJ, int SUB, bool WC>
__global__ void __launch_bounds__(NT) probe(const float *__restrict__ ir, const float *__restrict__ ii,
                                            float *__restrict__ orr, float *__restrict__ oi, int64_t rs)
{
    constexpr int ROWS = NT / TJ;                 // rows per k step
    constexpr int CHUNK_ROWS = ROWS * K;          // rows per chunk
    const int tid = threadIdx.x, jl = tid % TJ, t = tid / TJ;
    const int64_t j = (int64_t)blockIdx.x * TJ + jl;
#pragma unroll 1
    for (int c = 0; c < SUB; c += CHUNK_ROWS) {
        float vr[K], vi[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int64_t a = j + (int64_t)(c + t + ROWS * k) * rs;
            vr[k] = __ldcs(ir + a);
            vi[k] = __ldcs(ii + a);
        }
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int e = c + t + ROWS * k;
            const int64_t a = WC ? j * SUB + e : j + (int64_t)e * rs;
            __stcs(orr + a, vr[k]);
            __stcs(oi + a, vi[k]);
        }
    }
}

template <int TJ, int SUB, bool WC>
static void run(float *b[4], int64_t n)
{
    const int64_t rs = n / SUB, blocks = rs / TJ;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int w = 0; w < 3; ++w) probe<TJ, SUB, WC><<<blocks, NT>>>(b[0], b[1], b[2], b[3], rs);
    const int it = 10;
    cudaEventRecord(e0);
    for (int w = 0; w < it; ++w) probe<TJ, SUB, WC><<<blocks, NT>>>(b[0], b[1], b[2], b[3], rs);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= it;
    printf("TJ=%2d (%3d B runs) SUB=%5d write=%s  %8.3f ms  %7.1f GB/s\n", TJ, TJ * 4, SUB, WC ? "contig" : "runs  ",
           ms, 16.0 * n / (ms * 1e6));
    if (cudaGetLastError() != cudaSuccess) printf("error\n");
}

int main()
{
    const int64_t n = int64_t(1) << 28;
    float *b[4];
    for (int k = 0; k < 4; ++k) {
        if (cudaMalloc(&b[k], n * sizeof(float)) != cudaSuccess) return 1;
        cudaMemset(b[k], 0, n * sizeof(float));
    }
    run<32, 128, false>(b, n);
    run<32, 512, false>(b, n);
    run<32, 1024, false>(b, n);
    run<16, 512, false>(b, n);
    run<16, 1024, false>(b, n);
    run<8, 512, false>(b, n);
    run<8, 1024, false>(b, n);
    run<32, 1024, true>(b, n);
    run<16, 1024, true>(b, n);
    run<8, 1024, true>(b, n);
    run<16, 512, true>(b, n);
    return 0;
}
