// sfft_pass_tma_host.h -- tensor maps + persistent launch of the TMA pass kernel.
#pragma once
#include "sfft_pass_tma.cuh"
#include "sfft_tma_host.h"

namespace sfft {

struct PassTmaLaunch {
    const void *x_re, *x_im;
    void *y_re, *y_im;
    int64_t batch, in_stride, out_stride;   // elements
    PassTmaArgs a;                          // m, S, scale, tables (tiles filled here)
};

// A plane as the 3-D box view (cols, rows, batch): `cols` contiguous
// elements per row, rows `row_stride` apart, batch rows `batch_stride` apart.
template <typename T>
inline cudaError_t encode_box_view(CUtensorMap *map, const void *ptr, uint64_t cols, uint64_t rows,
                                   uint64_t row_stride, int64_t batch, int64_t batch_stride, int box_rows)
{
    PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
    if (!enc) return cudaErrorNotSupported;
    constexpr int TJ = 128 / (int)sizeof(T);
    cuuint64_t dims[3] = {cols, rows, (cuuint64_t)batch};
    cuuint64_t strides[2] = {row_stride * sizeof(T), (cuuint64_t)batch_stride * sizeof(T)};
    cuuint32_t box[3] = {(cuuint32_t)TJ, (cuuint32_t)box_rows, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(map, sizeof(T) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3,
                     const_cast<void *>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <typename T, int L, int LR, bool DIF, int STAGES>
cudaError_t launch_pass_tma(const PassTmaLaunch &Lc, cudaStream_t st)
{
    using Sh = PassTmaShape<T, L, LR, STAGES>;
    auto k = sfft_pass_tma_kernel<T, L, LR, DIF, STAGES>;
    static int blocks_per_sm[32] = {0};
    static int num_sms[32] = {0};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    dev &= 31;
    if (!blocks_per_sm[dev]) {
        e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, Sh::SMEM);
        if (e != cudaSuccess) return e;
        int b = 0, sms = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k, Sh::NT, Sh::SMEM);
        if (e != cudaSuccess) return e;
        e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (e != cudaSuccess) return e;
        if (b < 1) return cudaErrorInvalidConfiguration;
        num_sms[dev] = sms;
        blocks_per_sm[dev] = b;
    }
    const int m = Lc.a.m, S = Lc.a.S;
    const uint64_t n = uint64_t(1) << m, nj = n >> L, ns = uint64_t(1) << S;
    CUtensorMap m_xr, m_xi, m_yr, m_yi;
    // e-side view: (NJ cols, 2^L rows at stride NJ); o-side: (2^S cols, N/2^S rows at stride 2^S)
    const bool e_in = !DIF;
    if (e_in) {
        if ((e = encode_box_view<T>(&m_xr, Lc.x_re, nj, uint64_t(1) << L, nj, Lc.batch, Lc.in_stride, 1 << L))) return e;
        if ((e = encode_box_view<T>(&m_xi, Lc.x_im, nj, uint64_t(1) << L, nj, Lc.batch, Lc.in_stride, 1 << L))) return e;
        if ((e = encode_box_view<T>(&m_yr, Lc.y_re, ns, n / ns, ns, Lc.batch, Lc.out_stride, 1 << L))) return e;
        if ((e = encode_box_view<T>(&m_yi, Lc.y_im, ns, n / ns, ns, Lc.batch, Lc.out_stride, 1 << L))) return e;
    } else {
        if ((e = encode_box_view<T>(&m_xr, Lc.x_re, ns, n / ns, ns, Lc.batch, Lc.in_stride, 1 << L))) return e;
        if ((e = encode_box_view<T>(&m_xi, Lc.x_im, ns, n / ns, ns, Lc.batch, Lc.in_stride, 1 << L))) return e;
        if ((e = encode_box_view<T>(&m_yr, Lc.y_re, nj, uint64_t(1) << L, nj, Lc.batch, Lc.out_stride, 1 << L))) return e;
        if ((e = encode_box_view<T>(&m_yi, Lc.y_im, nj, uint64_t(1) << L, nj, Lc.batch, Lc.out_stride, 1 << L))) return e;
    }
    PassTmaArgs a = Lc.a;
    a.tiles_per_row = (int64_t)(nj / Sh::TJ);
    a.ntiles = a.tiles_per_row * Lc.batch;
    int64_t grid = (int64_t)num_sms[dev] * blocks_per_sm[dev];
    if (grid > a.ntiles) grid = a.ntiles;
    if (grid < 1) grid = 1;
    k<<<(unsigned)grid, Sh::NT, Sh::SMEM, st>>>(m_xr, m_xi, m_yr, m_yi, a);
    count_launch();
    return cudaGetLastError();
}

}  // namespace sfft
