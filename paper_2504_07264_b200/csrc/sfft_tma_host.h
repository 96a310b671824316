// sfft_tma_host.h -- host side of the TMA kernel: tensor-map encoding and
// the persistent launch.  Included by the generated instantiation units.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <mutex>

#include "sfft_launch.h"
#include "sfft_tma.cuh"

namespace sfft {

struct TmaLaunch {
    const void *x_re, *x_im;
    void *y_re, *y_im;
    int64_t batch, in_stride, out_stride;   // elements
    int inverse;
    double scale;
    const void *tw;
};

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder();   // sfft_abi.cu

// One plane viewed as (W elements, N/W lines, rows) with 128-byte swizzle.
template <typename T>
inline cudaError_t encode_plane(CUtensorMap *map, const void *ptr, int n, int64_t rows, int64_t row_stride,
                                int box_rows)
{
    PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
    if (!enc) return cudaErrorNotSupported;
    constexpr int W = 128 / (int)sizeof(T);
    cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)(n / W), (cuuint64_t)rows};
    cuuint64_t strides[2] = {(cuuint64_t)W * sizeof(T), (cuuint64_t)row_stride * sizeof(T)};
    cuuint32_t box[3] = {(cuuint32_t)W, (cuuint32_t)(n / W), (cuuint32_t)box_rows};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(map, sizeof(T) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3,
                     const_cast<void *>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <typename T, int LOGN, int LR, bool DIF, int NT_REQ, int STAGES, int OB, bool PRE>
cudaError_t launch_tma(const TmaLaunch &L, cudaStream_t st)
{
    using Sh = TmaShape<T, LOGN, LR, NT_REQ, STAGES, OB>;
    auto k = sfft_tma_kernel<T, LOGN, LR, DIF, NT_REQ, STAGES, OB, PRE>;
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
    // the caller realises the inverse by swapping the re/im maps (channel swap)
    const void *xr = L.inverse ? L.x_im : L.x_re;
    const void *xi = L.inverse ? L.x_re : L.x_im;
    void *yr = L.inverse ? L.y_im : L.y_re;
    void *yi = L.inverse ? L.y_re : L.y_im;
    CUtensorMap m_xr, m_xi, m_yr, m_yi;
    constexpr int N = Sh::N;
    if ((e = encode_plane<T>(&m_xr, xr, N, L.batch, L.in_stride, Sh::S)) != cudaSuccess) return e;
    if ((e = encode_plane<T>(&m_xi, xi, N, L.batch, L.in_stride, Sh::S)) != cudaSuccess) return e;
    if ((e = encode_plane<T>(&m_yr, yr, N, L.batch, L.out_stride, Sh::S)) != cudaSuccess) return e;
    if ((e = encode_plane<T>(&m_yi, yi, N, L.batch, L.out_stride, Sh::S)) != cudaSuccess) return e;
    TmaArgs a;
    a.ntiles = (L.batch + Sh::S - 1) / Sh::S;
    a.scale = L.scale;
    a.scale_out = L.inverse;
    a.tw = L.tw;
    int64_t grid = (int64_t)num_sms[dev] * blocks_per_sm[dev];
    if (grid > a.ntiles) grid = a.ntiles;
    if (grid < 1) grid = 1;
#ifndef SFFT_TMA_NO_PDL
    // programmatic dependent launch: this grid may be scheduled while the
    // previous kernel of the stream drains; the kernel's griddepcontrol.wait
    // (before its first TMA load) orders every global access after it
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(Sh::NT);
    cfg.dynamicSmemBytes = Sh::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, k, m_xr, m_xi, m_yr, m_yi, a);
    count_launch();
    return e != cudaSuccess ? e : cudaGetLastError();
#else
    k<<<(unsigned)grid, Sh::NT, Sh::SMEM, st>>>(m_xr, m_xi, m_yr, m_yi, a);
    count_launch();
    return cudaGetLastError();
#endif
}

}  // namespace sfft
