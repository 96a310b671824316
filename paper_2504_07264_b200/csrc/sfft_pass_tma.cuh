// sfft_pass_tma.cuh -- persistent TMA-pipelined pass kernel for the groups
// with S > 0 of the multi-launch schedule (N > 4096, planar rows).
//
// Same sub-problems and arithmetic as sfft_pass.cuh (group (S, L): 2^L-point
// sub-problems j, in[j + e*NJ] -> out[(j>>S)*2^S*2^L + (j & (2^S-1)) + 2^S*o],
// DIF the transpose).  For S > 0 both global sides of a tile of TJ
// consecutive sub-problems are 2-D boxes of 128-byte rows:
//     rows e (stride NJ elements), TJ columns          -- in (DIT) / out (DIF)
//     rows o (stride 2^S elements), TJ columns         -- out (DIT) / in (DIF)
// so a tile moves with one cp.async.bulk.tensor per plane each way.  The
// CTA is persistent over (row, tile) pairs with STAGES tile buffers: a
// buffer receives the input tile (mbarrier complete_tx), is reused as the
// exchange buffer of the internal register passes, then holds the output
// tile that one thread stores with a bulk tensor store; it is refilled for
// tile k + STAGES - 1 once the store of tile k - 1 has finished reading it.
// With the 128-byte swizzle a warp (32 lanes = 32 consecutive sub-problems
// of one row e for fp32; 2 x 16 for fp64) always touches one 128-byte smem
// row, so every shared-memory access is conflict-free.
#pragma once
#include "sfft_pass.cuh"
#include "sfft_tma.cuh"

namespace sfft {

struct PassTmaArgs {
    int64_t tiles_per_row, ntiles;
    int m, S;
    int scale_out;         // multiply by `scale` at the store (inverse, last launch)
    double scale;
    const void *tw;
    int tw_cat_top;
    const void *tw_top_tab;
    const double2 *coarse;
    int coarse_log;
    const double2 *fine;
};

template <typename T, int L, int LR_REQ, int STAGES>
struct PassTmaShape {
    static constexpr int SUB = 1 << L;
    static constexpr int LR = cmin(LR_REQ, L);
    static constexpr int R = 1 << LR;
    static constexpr int P = SUB / R;
    static constexpr int TJ = 128 / (int)sizeof(T);      // one 128-byte row per e
    static constexpr int NT = TJ * P;
    static constexpr int NPI = (L + LR - 1) / LR;
    static constexpr int PLANE = SUB * 128;               // bytes per plane per tile
    static constexpr int BUF = 2 * PLANE;
    static constexpr int BAR_OFF = STAGES * BUF;
    static constexpr int SMEM = BAR_OFF + STAGES * 8 + 1024;
    // CTAs per SM the shared memory allows; handed to __launch_bounds__ so
    // ptxas keeps registers within 64K / (NT * MINB) instead of ~255
    static constexpr int MINB_SMEM = (227 * 1024) / SMEM;
    static constexpr int MINB = MINB_SMEM < 1 ? 1 : (MINB_SMEM * NT > 2048 ? 2048 / NT : MINB_SMEM);
    static_assert(SUB <= 256, "TMA box rows are limited to 256");
};

// byte offset of (row e, column jl) in a 128-byte-swizzled [e][TJ] tile
template <typename T>
__device__ __forceinline__ uint32_t swz_row(int e, int jl)
{
    const uint32_t L = (uint32_t)e * 128u + (uint32_t)jl * (uint32_t)sizeof(T);
    return L ^ ((L >> 3) & 0x70u);
}

template <typename T>
__device__ __forceinline__ typename PassTw<T, false>::type make_tma_pass_tw(const PassTmaArgs &a)
{
    typename PassTw<T, false>::type tw;
    tw.tab = (const vec2_t<T> *)a.tw;
    tw.cat_top = a.tw_cat_top;
    if constexpr (sizeof(T) == 8) {
        tw.top_tab = (const vec2_t<T> *)a.tw_top_tab;
        tw.top = a.m;
    } else {
        tw.set_tables(a.coarse, a.coarse_log, a.fine, a.m);
    }
    return tw;
}

template <typename T, int L, int LR_REQ, bool DIF, int STAGES>
__global__ void __launch_bounds__(PassTmaShape<T, L, LR_REQ, STAGES>::NT, PassTmaShape<T, L, LR_REQ, STAGES>::MINB)
sfft_pass_tma_kernel(const __grid_constant__ CUtensorMap in_re, const __grid_constant__ CUtensorMap in_im,
                     const __grid_constant__ CUtensorMap out_re, const __grid_constant__ CUtensorMap out_im,
                     const PassTmaArgs a)
{
    using Sh = PassTmaShape<T, L, LR_REQ, STAGES>;
    constexpr int SUB = Sh::SUB, LR = Sh::LR, R = Sh::R, P = Sh::P, TJ = Sh::TJ, NPI = Sh::NPI,
                  PLANE = Sh::PLANE, BUF = Sh::BUF;
    extern __shared__ unsigned char smem_raw[];
    unsigned char *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + Sh::BAR_OFF);

    const int tid = threadIdx.x;
    const int jl = tid % TJ, t = tid / TJ;
    const int S = a.S;
    const int64_t nk = a.ntiles > blockIdx.x ? (a.ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const auto tw = make_tma_pass_tw<T>(a);
    using I = typename PassTw<T, false>::type::index_t;
    const T scale = (T)a.scale;
    const bool do_scale = a.scale_out != 0;

    // tile -> (row b, first sub-problem j0); box coordinates of both sides
    auto tile_coords = [&](int64_t tile, int &b, uint32_t &j0) {
        b = (int)(tile / a.tiles_per_row);
        j0 = (uint32_t)(tile % a.tiles_per_row) * TJ;
    };
    // the "e-side" box: rows e at stride NJ, columns j0..j0+TJ  (DIT in / DIF out)
    // the "o-side" box: rows (j>>S)*SUB + o at stride 2^S, columns c0..c0+TJ
    auto load_tile = [&](int st, int64_t tile) {
        int b;
        uint32_t j0;
        tile_coords(tile, b, j0);
        uint64_t *bar = full + st;
        mbar_expect_tx(bar, BUF);
        unsigned char *dst = smem + st * BUF;
        if constexpr (!DIF) {
            tma_load_3d(dst, &in_re, bar, (int)j0, 0, b);
            tma_load_3d(dst + PLANE, &in_im, bar, (int)j0, 0, b);
        } else {
            const int c0 = (int)(j0 & ((1u << S) - 1u)), r0 = (int)((j0 >> S) * SUB);
            tma_load_3d(dst, &in_re, bar, c0, r0, b);
            tma_load_3d(dst + PLANE, &in_im, bar, c0, r0, b);
        }
    };
    auto store_tile = [&](int st, int64_t tile) {
        int b;
        uint32_t j0;
        tile_coords(tile, b, j0);
        const unsigned char *src = smem + st * BUF;
        if constexpr (!DIF) {
            const int c0 = (int)(j0 & ((1u << S) - 1u)), r0 = (int)((j0 >> S) * SUB);
            tma_store_3d(&out_re, src, c0, r0, b);
            tma_store_3d(&out_im, src + PLANE, c0, r0, b);
        } else {
            tma_store_3d(&out_re, src, (int)j0, 0, b);
            tma_store_3d(&out_im, src + PLANE, (int)j0, 0, b);
        }
        bulk_commit();
    };

    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(full + s, 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (tid == 0) {
        for (int s = 0; s < STAGES - 1 && s < nk; ++s) load_tile(s, blockIdx.x + (int64_t)s * gridDim.x);
    }

    vec2_t<T> v[R];
    for (int64_t k = 0; k < nk; ++k) {
        const int st = (int)(k % STAGES);
        const int64_t tile = blockIdx.x + k * gridDim.x;
        unsigned char *br = smem + st * BUF;
        unsigned char *bi = br + PLANE;
        int b;
        uint32_t j0;
        tile_coords(tile, b, j0);
        const uint32_t j = j0 + jl;
        const uint32_t c = j & ((1u << S) - 1u);
        mbar_wait(full + st, (uint32_t)((k / STAGES) & 1));

        if constexpr (!DIF) {
#pragma unroll
            for (int pp = 0; pp < NPI; ++pp) {
                const int sp = pp * LR;
                const int kp = cmin(LR, L - sp);
#define SFFT_PT_DIT(KP)                                                                         \
    if constexpr (KP <= LR) if (kp == KP) {                                                     \
        constexpr int RP = 1 << KP, U = R / RP;                                                 \
        const int nsp = 1 << sp;                                                                \
        _Pragma("unroll") for (int u = 0; u < U; ++u)                                           \
        {                                                                                       \
            const int jp = t + P * u;                                                           \
            _Pragma("unroll") for (int r = 0; r < RP; ++r)                                      \
            {                                                                                   \
                const int e = jp + r * (SUB / RP);                                              \
                v[u * RP + r].x = lds_at<T>(br, swz_row<T>(e, jl));                              \
                v[u * RP + r].y = lds_at<T>(bi, swz_row<T>(e, jl));                              \
            }                                                                                   \
        }                                                                                       \
        _Pragma("unroll") for (int u = 0; u < U; ++u)                                           \
        {                                                                                       \
            const int jp = t + P * u;                                                           \
            dit_stages<T, KP, false>(v + u * RP, S + sp,                          \
                                     (I)(c + ((uint32_t)(jp & (nsp - 1)) << S)), tw);           \
        }                                                                                       \
        __syncthreads();                                                                        \
        const bool last = pp == NPI - 1;                                                        \
        _Pragma("unroll") for (int u = 0; u < U; ++u)                                           \
        {                                                                                       \
            const int jp = t + P * u;                                                           \
            const int base = last ? jp : (jp >> sp) * nsp * RP + (jp & (nsp - 1));              \
            _Pragma("unroll") for (int f = 0; f < RP; ++f)                                      \
            {                                                                                   \
                const int e = base + nsp * f;                                                   \
                T re = v[u * RP + brev(f, KP)].x, im = v[u * RP + brev(f, KP)].y;                 \
                if (last && do_scale) { re *= scale; im *= scale; }                             \
                sts_at<T>(br, swz_row<T>(e, jl), re);                                           \
                sts_at<T>(bi, swz_row<T>(e, jl), im);                                           \
            }                                                                                   \
        }                                                                                       \
        if (!last) __syncthreads();                                                             \
    }
                SFFT_PT_DIT(1)
                SFFT_PT_DIT(2)
                SFFT_PT_DIT(3)
                SFFT_PT_DIT(4)
                SFFT_PT_DIT(5)
#undef SFFT_PT_DIT
            }
        } else {
#pragma unroll
            for (int pp = NPI - 1; pp >= 0; --pp) {
                const int sp = pp * LR;
                const int kp = cmin(LR, L - sp);
#define SFFT_PT_DIF(KP)                                                                         \
    if constexpr (KP <= LR) if (kp == KP) {                                                     \
        constexpr int RP = 1 << KP, U = R / RP;                                                 \
        const int nsp = 1 << sp;                                                                \
        _Pragma("unroll") for (int u = 0; u < U; ++u)                                           \
        {                                                                                       \
            const int jp = t + P * u;                                                           \
            const int base = (jp >> sp) * nsp * RP + (jp & (nsp - 1));                          \
            _Pragma("unroll") for (int f = 0; f < RP; ++f)                                      \
            {                                                                                   \
                const int e = base + nsp * f;                                                   \
                const int d = u * RP + brev(f, KP);                                             \
                v[d].x = lds_at<T>(br, swz_row<T>(e, jl));                                       \
                v[d].y = lds_at<T>(bi, swz_row<T>(e, jl));                                       \
            }                                                                                   \
        }                                                                                       \
        _Pragma("unroll") for (int u = 0; u < U; ++u)                                           \
        {                                                                                       \
            const int jp = t + P * u;                                                           \
            dif_stages<T, KP, false>(v + u * RP, S + sp,                          \
                                     (I)(c + ((uint32_t)(jp & (nsp - 1)) << S)), tw);           \
        }                                                                                       \
        __syncthreads();                                                                        \
        const bool last = pp == 0;                                                              \
        _Pragma("unroll") for (int u = 0; u < U; ++u)                                           \
        {                                                                                       \
            const int jp = t + P * u;                                                           \
            _Pragma("unroll") for (int r = 0; r < RP; ++r)                                      \
            {                                                                                   \
                const int e = jp + r * (SUB / RP);                                              \
                T re = v[u * RP + r].x, im = v[u * RP + r].y;                                     \
                if (last && do_scale) { re *= scale; im *= scale; }                             \
                sts_at<T>(br, swz_row<T>(e, jl), re);                                           \
                sts_at<T>(bi, swz_row<T>(e, jl), im);                                           \
            }                                                                                   \
        }                                                                                       \
        if (!last) __syncthreads();                                                             \
    }
                SFFT_PT_DIF(1)
                SFFT_PT_DIF(2)
                SFFT_PT_DIF(3)
                SFFT_PT_DIF(4)
                SFFT_PT_DIF(5)
#undef SFFT_PT_DIF
            }
        }
        // the output tile is in buffer st: store it, then refill the buffer
        // of tile k-1 (its store must have finished reading) with tile k+STAGES-1
        fence_async_smem();
        __syncthreads();
        if (tid == 0) {
            store_tile(st, tile);
            const int64_t next = k + STAGES - 1;
            if (next < nk) {
                bulk_wait_read<1>();
                load_tile((int)(next % STAGES), blockIdx.x + next * gridDim.x);
            }
        }
    }
    if (tid == 0) bulk_wait_all();
}

}  // namespace sfft
