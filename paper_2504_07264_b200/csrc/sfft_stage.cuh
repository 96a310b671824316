// sfft_stage.cuh -- the literal per-stage operators on the interleaved
// layout: butterfly_stage W^(i) and twiddle_stage D^(i)
// (transform.py:88-120).  Not on the hot path -- the fused
// and pass kernels run the same arithmetic inside their register passes --
// but part of the reference's public operator API: the reference's own tests
// compose them with permute_pairwise_bitrev and compare the composition with
// fft_dit / fft_dif bit for bit (test_transform.py:145-167).
//
// One thread per butterfly pair (q, q + 2^(i-1)) of one row; rows are
// grid.y.  Arithmetic exactly as numpy does it on the complex128 view:
//   butterfly: a' = a + b, b' = a - b          (transform.py:96-101)
//   twiddle:   b' = b * w_i[q] for q >= 1       (transform.py:117-120; the
//              identity column q = 0 is left untouched, signed zeros included)
// with the complex product rounded as numpy's complex multiply (cmul,
// data operand first as in `v *= w`).
#pragma once
#include "sfft_common.cuh"

namespace sfft {

template <typename T, int KIND, typename TW>
__global__ void __launch_bounds__(256) sfft_stage_kernel(vec2_t<T> *data, int64_t stride, int log2n, int stage,
                                                         TW tw)
{
    const int64_t half = int64_t(1) << (log2n - 1);     // butterflies per row
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= half) return;
    vec2_t<T> *row = data + (int64_t)blockIdx.y * stride;
    const int64_t h = int64_t(1) << (stage - 1);
    const int64_t q = b & (h - 1);
    const int64_t p0 = ((b >> (stage - 1)) << stage) + q;   // pair q of its block
    vec2_t<T> *pa = row + p0, *pb = row + p0 + h;
    if constexpr (KIND == 0) {
        const vec2_t<T> a = *pa, v = *pb;
        *pa = adds(a, v);
        *pb = subs(a, v);
    } else {
        if (q == 0) return;
        const vec2_t<T> w = tw.get(stage, (typename TW::index_t)q);
        *pb = cmuls(*pb, w);
    }
}

}  // namespace sfft
