// pattern_probe.cu -- HBM efficiency of the pass kernels' access patterns,
// without any arithmetic.  Each CTA moves one tile of 32 sub-problems x 128
// elements (two fp32 planes) from `in` to `out` with the address patterns of
// a 2^28-point pass group:
//   read  "s": in[j + e*RS]           (128-byte runs, RS apart)
//   read  "c": in[j0*128 + k]          (contiguous 16 KB)
//   write "s": out[j + o*WS]          (128-byte runs, WS apart)
//   write "c": out[j0*128 + k]         (contiguous, through a smem transpose)
// usage: pattern_probe   (prints GB/s per pattern; 2 x 2 GB planes in, 2 out)
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>

constexpr int TJ = 32, SUB = 128, NT = 256, RS_ = TJ + 1;

template <bool RC, bool WC, bool CS>
__global__ void __launch_bounds__(NT) probe(const float *__restrict__ ir, const float *__restrict__ ii,
                                            float *__restrict__ orr, float *__restrict__ oi, int64_t rs, int64_t ws)
{
    __shared__ float sr[SUB * RS_], si[SUB * RS_];
    const int tid = threadIdx.x, jl = tid % TJ, t = tid / TJ;
    const int64_t j0 = (int64_t)blockIdx.x * TJ, j = j0 + jl;
    float vr[16], vi[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        const int e = t + 8 * k;
        const int64_t a = RC ? j0 * SUB + (int64_t)(tid + NT * k) : j + (int64_t)e * rs;
        vr[k] = CS ? __ldcs(ir + a) : ir[a];
        vi[k] = CS ? __ldcs(ii + a) : ii[a];
    }
    // keep the compiler from forwarding loads to stores
    if (WC) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const int e = t + 8 * k;
            sr[e * RS_ + jl] = vr[k];
            si[e * RS_ + jl] = vi[k];
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const int idx = tid + NT * k, jj = idx / SUB, o = idx % SUB;
            if (CS) {
                __stcs(orr + j0 * SUB + idx, sr[o * RS_ + jj]);
                __stcs(oi + j0 * SUB + idx, si[o * RS_ + jj]);
            } else {
                orr[j0 * SUB + idx] = sr[o * RS_ + jj];
                oi[j0 * SUB + idx] = si[o * RS_ + jj];
            }
        }
    } else {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const int o = t + 8 * k;
            const int64_t a = j + (int64_t)o * ws;
            if (CS) {
                __stcs(orr + a, vr[k]);
                __stcs(oi + a, vi[k]);
            } else {
                orr[a] = vr[k];
                oi[a] = vi[k];
            }
        }
    }
}

template <bool RC, bool WC, bool CS>
static void run(const char *name, float *b[4], int64_t n, int64_t rs, int64_t ws)
{
    const int64_t tiles = (n / SUB) / TJ;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int w = 0; w < 3; ++w) probe<RC, WC, CS><<<tiles, NT>>>(b[0], b[1], b[2], b[3], rs, ws);
    const int it = 10;
    cudaEventRecord(e0);
    for (int w = 0; w < it; ++w) probe<RC, WC, CS><<<tiles, NT>>>(b[0], b[1], b[2], b[3], rs, ws);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= it;
    printf("%-34s %8.3f ms  %7.1f GB/s\n", name, ms, 16.0 * n / (ms * 1e6));
    if (cudaGetLastError() != cudaSuccess) printf("error\n");
}

int main()
{
    const int64_t n = int64_t(1) << 28, pad = 1 << 16;
    float *b[4];
    for (int k = 0; k < 4; ++k) {
        if (cudaMalloc(&b[k], (n + 2 * SUB * pad) * sizeof(float)) != cudaSuccess) return 1;
        cudaMemset(b[k], 0, (n + 2 * SUB * pad) * sizeof(float));
    }
    const int64_t S21 = int64_t(1) << 21;
    run<true, true, true>("copy contiguous (cs)", b, n, 0, 0);
    run<false, true, true>("read s 2^21, write c (cs)", b, n, S21, 0);
    run<false, true, false>("read s 2^21, write c (plain)", b, n, S21, 0);
    run<true, false, true>("read c, write s 2^21 (cs)", b, n, 0, S21);
    run<false, false, true>("read s 2^21, write s 2^21 (cs)", b, n, S21, S21);
    run<false, false, false>("read s 2^21, write s 2^21 (plain)", b, n, S21, S21);
    run<false, false, true>("read s +32, write s +32 (cs)", b, n, S21 + 32, S21 + 32);
    run<false, false, true>("read s +64, write s +64 (cs)", b, n, S21 + 64, S21 + 64);
    run<false, false, true>("read s +256, write s +256 (cs)", b, n, S21 + 256, S21 + 256);
    run<false, false, true>("read s 2^21, write s +32 (cs)", b, n, S21, S21 + 32);
    run<false, false, true>("read s +32, write s 2^21 (cs)", b, n, S21 + 32, S21);
    return 0;
}
