// sfft_tma_host.h -- host side of the TMA kernel: tensor-map encoding and
// the persistent launch.  Included by the generated instantiation units.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <mutex>

#include "sfft_launch.h"
#include "sfft_tma.cuh"
#include "sfft_tma_warp.cuh"

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

// Resident CTAs of kernel `k` on device `dev` (shared-memory attribute set
// once per device and kernel).  Initialised under std::call_once per device,
// so concurrent first calls never see a half-written entry.
struct Residency {
    std::once_flag once[64];
    cudaError_t err[64] = {};
    int grid[64] = {};
    template <typename K>
    cudaError_t get(K k, int dev, int nt, int smem, int *out)
    {
        if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
        std::call_once(once[dev], [&] {
            cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            int b = 0, sms = 0;
            if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k, nt, smem);
            if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            if (e == cudaSuccess && b < 1) e = cudaErrorInvalidConfiguration;
            err[dev] = e;
            grid[dev] = e == cudaSuccess ? b * sms : 0;
        });
        *out = grid[dev];
        return err[dev];
    }
};

template <typename T, int LOGN, int LR, bool DIF, int NT_REQ, int STAGES, int OB, bool PRE, int MINB = 0>
cudaError_t launch_tma(const TmaLaunch &L, cudaStream_t st)
{
    using Sh = TmaShape<T, LOGN, LR, NT_REQ, STAGES, OB>;
    auto k = tma_kernel_for<T, LOGN, LR, DIF, NT_REQ, STAGES, OB, PRE, MINB>();
    static Residency res;
    int dev = 0, resident = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if ((e = res.get(k, dev, Sh::NT, Sh::SMEM, &resident)) != cudaSuccess) return e;
    // the caller realises the inverse by swapping the re/im maps (channel swap)
    const void *xr = L.inverse ? L.x_im : L.x_re;
    const void *xi = L.inverse ? L.x_re : L.x_im;
    void *yr = L.inverse ? L.y_im : L.y_re;
    void *yi = L.inverse ? L.y_re : L.y_im;
    CUtensorMap m_xr, m_xi, m_yr, m_yi;
    constexpr int N = Sh::N;
    if ((e = encode_plane<T>(&m_xr, xr, N, L.batch, L.in_stride, Sh::S)) != cudaSuccess) return e;
    if ((e = encode_plane<T>(&m_xi, xi, N, L.batch, L.in_stride, Sh::S)) != cudaSuccess) return e;
    if constexpr (OB > 0) {
        if ((e = encode_plane<T>(&m_yr, yr, N, L.batch, L.out_stride, Sh::S)) != cudaSuccess) return e;
        if ((e = encode_plane<T>(&m_yi, yi, N, L.batch, L.out_stride, Sh::S)) != cudaSuccess) return e;
    } else {
        m_yr = m_xr;   // unused: the last pass stores directly (a.y_re / a.y_im)
        m_yi = m_xi;
    }
    TmaArgs a;
    a.ntiles = (L.batch + Sh::S - 1) / Sh::S;
    a.scale = L.scale;
    a.scale_out = L.inverse;
    a.tw = L.tw;
    a.y_re = yr;
    a.y_im = yi;
    a.batch = L.batch;
    a.out_stride = L.out_stride;
    int64_t grid = resident;
    if (grid > a.ntiles) grid = a.ntiles;
    if (grid < 1) return cudaErrorInvalidConfiguration;   // batch > 0 here: never silently skip work
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

// Signal-group bulk-copy kernel (sfft_tma_warp.cuh): one CTA of WARPS warps
// per SM, WPS warps per signal, each group a persistent worker.
template <typename T, bool DIF, int WARPS, int HK, bool TM, bool RING = false, int XS = 1, int LOGN = 10,
          int WPS = 1, int PF = 0>
cudaError_t launch_tmaw(const TmaLaunch &L, cudaStream_t st)
{
    using Sh = TmaWShape<T, WARPS, RING, XS, LOGN, WPS>;
    auto k = &sfft_tmaw_kernel<T, DIF, WARPS, HK, TM, RING, XS, LOGN, WPS, PF>;
    static Residency res;
    int dev = 0, resident = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if ((e = res.get(k, dev, Sh::NT, Sh::SMEM, &resident)) != cudaSuccess) return e;
    TmaWArgs a;
    a.x_re = L.inverse ? L.x_im : L.x_re;
    a.x_im = L.inverse ? L.x_re : L.x_im;
    a.y_re = L.inverse ? L.y_im : L.y_re;
    a.y_im = L.inverse ? L.y_re : L.y_im;
    a.batch = L.batch;
    a.in_stride = L.in_stride;
    a.out_stride = L.out_stride;
    a.scale = L.scale;
    a.scale_out = L.inverse;
    a.tw = L.tw;
    int64_t grid = resident;
    const int64_t need = (L.batch + Sh::GROUPS - 1) / Sh::GROUPS;
    if (grid > need) grid = need;
    if (grid < 1) return cudaErrorInvalidConfiguration;   // batch > 0 here: never silently skip work
#ifndef SFFT_TMA_NO_PDL
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
    e = cudaLaunchKernelEx(&cfg, k, a);
    count_launch();
    return e != cudaSuccess ? e : cudaGetLastError();
#else
    k<<<(unsigned)grid, Sh::NT, Sh::SMEM, st>>>(a);
    count_launch();
    return cudaGetLastError();
#endif
}

}  // namespace sfft
