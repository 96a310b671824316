// sfft_pass_async.cuh -- persistent, cp.async-pipelined pass kernel for the
// groups with S > 0 of the multi-launch schedule (N > 4096).
//
// Same sub-problems, addressing (including the sharded owner-field maps) and
// arithmetic as sfft_pass.cuh.  What changes is latency hiding: the plain
// pass kernel loads its tile straight into registers and then computes, so
// an SM's loads stall while its CTAs compute (ncu: long_scoreboard on the
// first use of the loaded data).  Here each CTA is persistent over tiles and
// keeps STAGES tile buffers in shared memory: while tile k is transformed,
// per-thread asynchronous copies (cp.async, LDGSTS) of tile k+STAGES-1 are in
// flight into another buffer.  A buffer holds the tile as [e][jl] rows of TJ
// elements -- a warp is one row, so every shared access is conflict-free --
// and doubles as the exchange buffer of the internal register passes; the
// last pass writes global memory directly (128-byte runs for S > 0).
#pragma once
#include "sfft_pass.cuh"

namespace sfft {

__device__ __forceinline__ void cp_async4(void *smem_dst, const void *gmem_src)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(smem_dst)),
                 "l"(gmem_src)
                 : "memory");
}
__device__ __forceinline__ void cp_async8(void *smem_dst, const void *gmem_src)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(smem_dst)),
                 "l"(gmem_src)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <typename T>
__device__ __forceinline__ void cp_async_elem(T *dst, const T *src)
{
    if constexpr (sizeof(T) == 4) cp_async4(dst, src); else cp_async8(dst, src);
}

template <typename T, int L, int LR_REQ, int STAGES>
struct PassAsyncShape {
    static constexpr int SUB = 1 << L;
    static constexpr int LR = cmin(LR_REQ, L);
    static constexpr int R = 1 << LR;
    static constexpr int P = SUB / R;
    static constexpr int TJ = sizeof(T) == 4 ? 32 : 16;
    static constexpr int NT = TJ * P;
    static constexpr int NPI = (L + LR - 1) / LR;
    static constexpr int PLANE = SUB * TJ;            // elements per plane per tile
    static constexpr int SMEM = STAGES * 2 * PLANE * (int)sizeof(T);
};

template <typename T, int L, int LR_REQ, bool DIF, bool DIST, int STAGES>
__global__ void __launch_bounds__(PassAsyncShape<T, L, LR_REQ, STAGES>::NT)
sfft_pass_async_kernel(const PassArgs a)
{
    using Sh = PassAsyncShape<T, L, LR_REQ, STAGES>;
    constexpr int SUB = Sh::SUB, LR = Sh::LR, R = Sh::R, P = Sh::P, TJ = Sh::TJ, NPI = Sh::NPI,
                  PLANE = Sh::PLANE;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T *sbuf = reinterpret_cast<T *>(smem_raw);

    const int m = a.m, S = a.S;
    const uint32_t NJ = 1u << (m - L);
    const uint32_t tiles_row = (NJ >> (DIST ? a.jb : 0)) / TJ;
    const int64_t ntiles = (int64_t)tiles_row * a.batch;
    const int64_t nk = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const int tid = threadIdx.x;
    const int jl = tid % TJ, t = tid / TJ;
    const uint32_t ns = 1u << S;
    const AddrMap imap = a.in_map, omap = a.out_map;
    const PIO<T, false> src = make_pio<T, false>(a);
    const auto tw = make_pass_tw<T, false>(a);
    using I = typename PassTw<T, false>::type::index_t;
    const bool swap_in = a.swap_in != 0, swap_out = a.swap_out != 0;
    const T scale = (T)a.scale;
    const T *in_re = swap_in ? src.ai : src.ar;
    const T *in_im = swap_in ? src.ar : src.ai;
    T *out_re = swap_out ? (T *)a.y1 : (T *)a.y0;
    T *out_im = swap_out ? (T *)a.y0 : (T *)a.y1;

    // (row, first sub-problem) of the k-th tile of this CTA
    auto tile_of = [&](int64_t k, int64_t &row, uint32_t &j0) {
        const int64_t tile = blockIdx.x + k * gridDim.x;
        row = tile / tiles_row;
        j0 = (uint32_t)(tile % tiles_row) * TJ;
        if constexpr (DIST) {
            const uint32_t lo = j0 & ((1u << a.jpos) - 1u);
            j0 = ((j0 >> a.jpos) << (a.jpos + a.jb)) | ((uint32_t)a.jrank << a.jpos) | lo;
        }
    };
    // each thread copies the elements e = t + P*k of column jl of tile k into buffer st
    auto issue = [&](int64_t k, int st) {
        int64_t row;
        uint32_t j0;
        tile_of(k, row, j0);
        const int64_t ioff = row * a.in_stride;
        T *br = sbuf + st * 2 * PLANE;
        T *bi = br + PLANE;
        const uint32_t j = j0 + jl;
#pragma unroll
        for (int k2 = 0; k2 < R; ++k2) {
            const int e = t + P * k2;
            uint32_t x;
            if constexpr (!DIF) x = j + (uint32_t)e * NJ;
            else x = (j >> S) * ns * SUB + (j & (ns - 1u)) + ns * (uint32_t)e;
            const int64_t off = ioff + (DIST ? imap(x) : x);
            cp_async_elem(br + e * TJ + jl, in_re + off);
            cp_async_elem(bi + e * TJ + jl, in_im + off);
        }
    };

    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < nk) issue(s, s);
        cp_async_commit();
    }

    vec2_t<T> v[R];
    for (int64_t k = 0; k < nk; ++k) {
        const int st = (int)(k % STAGES);
        cp_async_wait<STAGES - 2>();
        __syncthreads();                       // tile k landed; tile k-1 fully consumed
        if (k + STAGES - 1 < nk) issue(k + STAGES - 1, (int)((k + STAGES - 1) % STAGES));
        cp_async_commit();

        int64_t row;
        uint32_t j0;
        tile_of(k, row, j0);
        const uint32_t j = j0 + jl;
        const uint32_t c = j & (ns - 1u);
        const uint32_t gbase = (j >> S) * ns * SUB + c;
        const int64_t ooff = row * a.out_stride;
        T *br = sbuf + st * 2 * PLANE;
        T *bi = br + PLANE;
        auto put = [&](uint32_t x, vec2_t<T> z) {
            if (swap_out) {
                z.x *= scale;
                z.y *= scale;
            }
            const int64_t off = ooff + (DIST ? omap(x) : x);
            if constexpr (DIST) {
                if (a.npeers > 0) {
                    const int h = (int)(off >> a.seg_log);
                    const int64_t r = ((int64_t)a.jrank << a.seg_log) + (off & ((int64_t(1) << a.seg_log) - 1));
                    st_stream((swap_out ? (T *)a.peer_im[h] : (T *)a.peer_re[h]) + r, z.x);
                    st_stream((swap_out ? (T *)a.peer_re[h] : (T *)a.peer_im[h]) + r, z.y);
                    return;
                }
            }
            st_stream(out_re + off, z.x);
            st_stream(out_im + off, z.y);
        };

        if constexpr (!DIF) {
#pragma unroll
            for (int pp = 0; pp < NPI; ++pp) {
                const int sp = pp * LR;
                const int kp = cmin(LR, L - sp);
#define SFFT_PA_DIT(KP)                                                                          \
    if constexpr (KP <= LR) if (kp == KP) {                                                      \
        constexpr int RP = 1 << KP, U = R / RP;                                                  \
        const int nsp = 1 << sp;                                                                 \
        _Pragma("unroll") for (int u = 0; u < U; ++u)                                            \
        {                                                                                        \
            const int jp = t + P * u;                                                            \
            _Pragma("unroll") for (int r = 0; r < RP; ++r)                                       \
            {                                                                                    \
                const int e = jp + r * (SUB / RP);                                               \
                v[u * RP + r].x = br[e * TJ + jl];                                               \
                v[u * RP + r].y = bi[e * TJ + jl];                                               \
            }                                                                                    \
        }                                                                                        \
        _Pragma("unroll") for (int u = 0; u < U; ++u)                                            \
        {                                                                                        \
            const int jp = t + P * u;                                                            \
            dit_stages<T, KP, false>(v + u * RP, S + sp, (I)(c + ((uint32_t)(jp & (nsp - 1)) << S)), tw); \
        }                                                                                        \
        if (pp < NPI - 1) {                                                                      \
            __syncthreads();                                                                     \
            _Pragma("unroll") for (int u = 0; u < U; ++u)                                        \
            {                                                                                    \
                const int jp = t + P * u;                                                        \
                const int base = (jp >> sp) * nsp * RP + (jp & (nsp - 1));                       \
                _Pragma("unroll") for (int f = 0; f < RP; ++f)                                   \
                {                                                                                \
                    const int e = base + nsp * f;                                                \
                    br[e * TJ + jl] = v[u * RP + brev(f, KP)].x;                                 \
                    bi[e * TJ + jl] = v[u * RP + brev(f, KP)].y;                                 \
                }                                                                                \
            }                                                                                    \
            __syncthreads();                                                                     \
        } else {                                                                                 \
            _Pragma("unroll") for (int u = 0; u < U; ++u)                                        \
            {                                                                                    \
                const int jp = t + P * u;                                                        \
                _Pragma("unroll") for (int f = 0; f < RP; ++f)                                   \
                    put(gbase + ns * (uint32_t)(jp + nsp * f), v[u * RP + brev(f, KP)]);         \
            }                                                                                    \
        }                                                                                        \
    }
                SFFT_PA_DIT(1)
                SFFT_PA_DIT(2)
                SFFT_PA_DIT(3)
                SFFT_PA_DIT(4)
                SFFT_PA_DIT(5)
#undef SFFT_PA_DIT
            }
        } else {
#pragma unroll
            for (int pp = NPI - 1; pp >= 0; --pp) {
                const int sp = pp * LR;
                const int kp = cmin(LR, L - sp);
#define SFFT_PA_DIF(KP)                                                                          \
    if constexpr (KP <= LR) if (kp == KP) {                                                      \
        constexpr int RP = 1 << KP, U = R / RP;                                                  \
        const int nsp = 1 << sp;                                                                 \
        _Pragma("unroll") for (int u = 0; u < U; ++u)                                            \
        {                                                                                        \
            const int jp = t + P * u;                                                            \
            const int base = (jp >> sp) * nsp * RP + (jp & (nsp - 1));                           \
            _Pragma("unroll") for (int f = 0; f < RP; ++f)                                       \
            {                                                                                    \
                const int e = base + nsp * f;                                                    \
                const int d = u * RP + brev(f, KP);                                              \
                v[d].x = br[e * TJ + jl];                                                        \
                v[d].y = bi[e * TJ + jl];                                                        \
            }                                                                                    \
        }                                                                                        \
        _Pragma("unroll") for (int u = 0; u < U; ++u)                                            \
        {                                                                                        \
            const int jp = t + P * u;                                                            \
            dif_stages<T, KP, false>(v + u * RP, S + sp, (I)(c + ((uint32_t)(jp & (nsp - 1)) << S)), tw); \
        }                                                                                        \
        if (pp != 0) {                                                                           \
            __syncthreads();                                                                     \
            _Pragma("unroll") for (int u = 0; u < U; ++u)                                        \
            {                                                                                    \
                const int jp = t + P * u;                                                        \
                _Pragma("unroll") for (int r = 0; r < RP; ++r)                                   \
                {                                                                                \
                    const int e = jp + r * (SUB / RP);                                           \
                    br[e * TJ + jl] = v[u * RP + r].x;                                           \
                    bi[e * TJ + jl] = v[u * RP + r].y;                                           \
                }                                                                                \
            }                                                                                    \
            __syncthreads();                                                                     \
        } else {                                                                                 \
            _Pragma("unroll") for (int u = 0; u < U; ++u)                                        \
            {                                                                                    \
                const int jp = t + P * u;                                                        \
                _Pragma("unroll") for (int r = 0; r < RP; ++r)                                   \
                    put(j + (uint32_t)(jp + r * (SUB / RP)) * NJ, v[u * RP + r]);                \
            }                                                                                    \
        }                                                                                        \
    }
                SFFT_PA_DIF(1)
                SFFT_PA_DIF(2)
                SFFT_PA_DIF(3)
                SFFT_PA_DIF(4)
                SFFT_PA_DIF(5)
#undef SFFT_PA_DIF
            }
        }
    }
    cp_async_wait<0>();
}

}  // namespace sfft
