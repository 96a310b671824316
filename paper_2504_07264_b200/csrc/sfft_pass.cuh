// sfft_pass.cuh -- multi-pass Stockham schedule for N = 2^m > 4096.
//
// Replaces the reference's cache-blocked wide-stage executor
// (transform.py:219-237 segments + _dit_stage_pair slabs, :153-200) for
// long signals.  The m stages are split into G groups of L_g <= 8
// consecutive stages; one launch per group.  Group (S, L) treats the array
// as N / 2^L independent 2^L-point sub-problems
//     sub-problem j:  elements  in[ j + e * N/2^L ],  e < 2^L
//     outputs          out[ (j>>S)*2^S*2^L + (j & (2^S-1)) + 2^S * o ]
// (DIT; DIF is the transpose, groups run last-to-first), i.e. the same
// Stockham map as the fused kernel one level up.  Inside a CTA a tile of TJ
// consecutive sub-problems (TJ = 32 fp32 / 16 fp64, so every global access is
// a 128-byte run) is staged in shared memory as [e][jl] rows of TJ+1 and
// processed with the register passes of sfft_common.cuh; the stage-(S+s'+t)
// factor index of internal virtual thread j' is
//     q = (j & (2^S-1)) + ((j' & (2^s'-1)) << S) + (f << (S+s')).
// The only non-unit-stride global pattern (DIT group S = 0 output, DIF group
// S = 0 input: rows of 2^L per sub-problem) goes through a shared-memory
// transpose so that the global side is one contiguous TJ*2^L block.
#pragma once
#include "sfft_common.cuh"

namespace sfft {

struct PassArgs {
    const void *x0, *x1;   // source planes (or pairs when the source is interleaved)
    void *y0, *y1;         // destination planes (or pairs)
    int64_t batch;
    int64_t in_stride, out_stride;
    int m;                 // log2 N
    int S;                 // stage offset of this group
    int swap_in, swap_out; // channel swap of the inverse (first / last launch)
    double scale;          // applied at the destination when swap_out
    const void *tw;        // stage-major table, stages 1..tw_cat_top (vec2_t<T>)
    int tw_cat_top;
    const void *tw_top_tab;// fp64, m > 20: stage-m table for the stages above tw_cat_top
    const double2 *coarse; // two-level fp32 twiddles (see TwTwoLevel)
    int coarse_log;
    const double2 *fine;
};

template <typename T, int L, int LR_REQ>
struct PassShape {
    static constexpr int SUB = 1 << L;
    static constexpr int LR = cmin(LR_REQ, L);
    static constexpr int R = 1 << LR;
    static constexpr int P = SUB / R;                 // threads per sub-problem
    static constexpr int TJ = sizeof(T) == 4 ? 32 : 16;
    static constexpr int NT = TJ * P;
    static constexpr int RS = TJ + 1;                 // smem row stride
    static constexpr int NPI = (L + LR - 1) / LR;     // internal register passes
    static constexpr int smem_bytes() { return 2 * SUB * RS * (int)sizeof(T); }
};

template <typename T, bool IL>
struct PIO;   // one side (source or destination) of a pass launch

template <typename T>
struct PIO<T, false> {
    const T *ar, *ai;
    T *br, *bi;
    __device__ __forceinline__ void load(int64_t off, T &re, T &im) const
    {
        re = ld_stream(ar + off);
        im = ld_stream(ai + off);
    }
    __device__ __forceinline__ void store(int64_t off, T re, T im) const
    {
        st_stream(br + off, re);
        st_stream(bi + off, im);
    }
};

template <typename T>
struct PIO<T, true> {
    const vec2_t<T> *a;
    vec2_t<T> *b;
    __device__ __forceinline__ void load(int64_t off, T &re, T &im) const
    {
        const vec2_t<T> v = ld_stream(a + off);
        re = v.x;
        im = v.y;
    }
    __device__ __forceinline__ void store(int64_t off, T re, T im) const
    {
        vec2_t<T> v;
        v.x = re;
        v.y = im;
        st_stream(b + off, v);
    }
};

template <typename T, bool IL>
__device__ __forceinline__ PIO<T, IL> make_pio(const PassArgs &a)
{
    PIO<T, IL> p;
    if constexpr (IL) {
        p.a = (const vec2_t<T> *)a.x0;
        p.b = (vec2_t<T> *)a.y0;
    } else {
        p.ar = (const T *)a.x0;
        p.ai = (const T *)a.x1;
        p.br = (T *)a.y0;
        p.bi = (T *)a.y1;
    }
    return p;
}

template <typename T, bool TWO>
struct TwSel { using type = TwCatTop<T>; };
template <typename T>
struct TwSel<T, true> { using type = TwTwoLevel<T>; };

template <typename T, bool TWO>
__device__ __forceinline__ typename TwSel<T, TWO>::type make_tw(const PassArgs &a)
{
    typename TwSel<T, TWO>::type tw;
    tw.tab = (const vec2_t<T> *)a.tw;
    tw.cat_top = a.tw_cat_top;
    if constexpr (!TWO) {
        tw.top_tab = (const vec2_t<T> *)a.tw_top_tab;
        tw.top = a.m;
    } else {
        tw.coarse = a.coarse;
        tw.coarse_log = a.coarse_log;
        tw.fine = a.fine;
        tw.m = a.m;
    }
    return tw;
}

template <typename T, int L, int LR_REQ, bool DIF, bool IL_IN, bool IL_OUT, bool TWO>
__global__ void __launch_bounds__(PassShape<T, L, LR_REQ>::NT)
sfft_pass_kernel(const PassArgs a)
{
    using Sh = PassShape<T, L, LR_REQ>;
    constexpr int SUB = Sh::SUB, LR = Sh::LR, R = Sh::R, P = Sh::P, TJ = Sh::TJ, NT = Sh::NT,
                  RS = Sh::RS, NPI = Sh::NPI;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T *sr = reinterpret_cast<T *>(smem_raw);
    T *si = sr + SUB * RS;

    const int m = a.m, S = a.S;
    const int64_t NJ = int64_t(1) << (m - L);         // sub-problems per row
    const int64_t tiles = NJ / TJ;
    const int64_t row = (int64_t)blockIdx.x / tiles;
    const int64_t j0 = ((int64_t)blockIdx.x % tiles) * TJ;
    const int tid = threadIdx.x;
    const int jl = tid % TJ, t = tid / TJ;
    const int64_t j = j0 + jl;
    const int64_t ns = int64_t(1) << S;
    const int64_t c = j & (ns - 1);
    const int64_t gbase = (j >> S) * ns * SUB + c;     // destination (DIT) / source (DIF) of o: gbase + ns*o
    const int64_t ioff = row * a.in_stride, ooff = row * a.out_stride;

    const PIO<T, IL_IN> src = make_pio<T, IL_IN>(a);
    const PIO<T, IL_OUT> dst = make_pio<T, IL_OUT>(a);
    const auto tw = make_tw<T, TWO>(a);
    const bool swap_in = a.swap_in != 0, swap_out = a.swap_out != 0;
    const T scale = (T)a.scale;

    T vr[R], vi[R];

    auto put_out = [&](int64_t off, T re, T im) {
        if (swap_out) dst.store(off, im * scale, re * scale);
        else dst.store(off, re, im);
    };
    auto get_in = [&](int64_t off, T &re, T &im) {
        T x, y;
        src.load(off, x, y);
        re = swap_in ? y : x;
        im = swap_in ? x : y;
    };

    if constexpr (!DIF) {
        // ------------------------------ DIT ------------------------------
#pragma unroll
        for (int pp = 0; pp < NPI; ++pp) {
            const int sp = pp * LR;
            const int kp = cmin(LR, L - sp);
            // kp is a compile-time constant after unrolling; dispatch on it
#define SFFT_DIT_INTERNAL(KP)                                                                   \
    if constexpr (KP <= LR) if (kp == KP) {                                                                             \
        constexpr int RP = 1 << KP, U = R / RP;                                                 \
        const int nsp = 1 << sp;                                                                \
        _Pragma("unroll") for (int u = 0; u < U; ++u)                                           \
        {                                                                                       \
            const int jp = t + P * u;                                                           \
            _Pragma("unroll") for (int r = 0; r < RP; ++r)                                      \
            {                                                                                   \
                const int e = jp + r * (SUB / RP);                                              \
                if (pp == 0) get_in(ioff + j + (int64_t)e * NJ, vr[u * RP + r], vi[u * RP + r]); \
                else {                                                                          \
                    vr[u * RP + r] = sr[e * RS + jl];                                           \
                    vi[u * RP + r] = si[e * RS + jl];                                           \
                }                                                                               \
            }                                                                                   \
        }                                                                                       \
        _Pragma("unroll") for (int u = 0; u < U; ++u)                                           \
        {                                                                                       \
            const int jp = t + P * u;                                                           \
            dit_stages<T, KP>(vr + u * RP, vi + u * RP, S + sp,                                 \
                              c + ((int64_t)(jp & (nsp - 1)) << S), tw);                        \
        }                                                                                       \
        const bool last = pp == NPI - 1;                                                        \
        if (!last || S == 0) {                                                                  \
            if (pp > 0) __syncthreads();                                                        \
            _Pragma("unroll") for (int u = 0; u < U; ++u)                                       \
            {                                                                                   \
                const int jp = t + P * u;                                                       \
                const int base = (jp >> sp) * nsp * RP + (jp & (nsp - 1));                      \
                _Pragma("unroll") for (int f = 0; f < RP; ++f)                                  \
                {                                                                               \
                    const int e = base + nsp * f;                                               \
                    sr[e * RS + jl] = vr[u * RP + brev(f, KP)];                                 \
                    si[e * RS + jl] = vi[u * RP + brev(f, KP)];                                 \
                }                                                                               \
            }                                                                                   \
            __syncthreads();                                                                    \
        } else {                                                                                \
            _Pragma("unroll") for (int u = 0; u < U; ++u)                                       \
            {                                                                                   \
                const int jp = t + P * u;                                                       \
                _Pragma("unroll") for (int f = 0; f < RP; ++f)                                  \
                {                                                                               \
                    const int o = jp + nsp * f;                                                 \
                    put_out(ooff + gbase + ns * o, vr[u * RP + brev(f, KP)],                    \
                            vi[u * RP + brev(f, KP)]);                                          \
                }                                                                               \
            }                                                                                   \
        }                                                                                       \
    }
            SFFT_DIT_INTERNAL(1)
            SFFT_DIT_INTERNAL(2)
            SFFT_DIT_INTERNAL(3)
            SFFT_DIT_INTERNAL(4)
            SFFT_DIT_INTERNAL(5)
#undef SFFT_DIT_INTERNAL
        }
        if (S == 0) {
            // outputs of this tile are the contiguous rows j0..j0+TJ of 2^L:
            // copy smem [o][jl] -> global in linear order
            const int64_t obase = ooff + j0 * SUB;
            for (int k = tid; k < TJ * SUB; k += NT) {
                const int jj = k >> L, o = k & (SUB - 1);
                put_out(obase + k, sr[o * RS + jj], si[o * RS + jj]);
            }
        }
    } else {
        // ------------------------------ DIF ------------------------------
        if (S == 0) {
            // inputs are the contiguous rows j0..j0+TJ of 2^L: stage them
            const int64_t ibase = ioff + j0 * SUB;
            for (int k = tid; k < TJ * SUB; k += NT) {
                const int jj = k >> L, o = k & (SUB - 1);
                T re, im;
                get_in(ibase + k, re, im);
                sr[o * RS + jj] = re;
                si[o * RS + jj] = im;
            }
            __syncthreads();
        }
#pragma unroll
        for (int pp = NPI - 1; pp >= 0; --pp) {
            const int sp = pp * LR;
            const int kp = cmin(LR, L - sp);
#define SFFT_DIF_INTERNAL(KP)                                                                   \
    if constexpr (KP <= LR) if (kp == KP) {                                                                             \
        constexpr int RP = 1 << KP, U = R / RP;                                                 \
        const int nsp = 1 << sp;                                                                \
        const bool first = pp == NPI - 1;                                                       \
        _Pragma("unroll") for (int u = 0; u < U; ++u)                                           \
        {                                                                                       \
            const int jp = t + P * u;                                                           \
            const int base = (jp >> sp) * nsp * RP + (jp & (nsp - 1));                          \
            _Pragma("unroll") for (int f = 0; f < RP; ++f)                                      \
            {                                                                                   \
                const int e = base + nsp * f;                                                   \
                const int d = u * RP + brev(f, KP);                                             \
                if (first && S != 0) get_in(ioff + gbase + ns * e, vr[d], vi[d]);               \
                else {                                                                          \
                    vr[d] = sr[e * RS + jl];                                                    \
                    vi[d] = si[e * RS + jl];                                                    \
                }                                                                               \
            }                                                                                   \
        }                                                                                       \
        _Pragma("unroll") for (int u = 0; u < U; ++u)                                           \
        {                                                                                       \
            const int jp = t + P * u;                                                           \
            dif_stages<T, KP>(vr + u * RP, vi + u * RP, S + sp,                                 \
                              c + ((int64_t)(jp & (nsp - 1)) << S), tw);                        \
        }                                                                                       \
        if (pp != 0) {                                                                          \
            if (!first || S == 0) __syncthreads();                                              \
            _Pragma("unroll") for (int u = 0; u < U; ++u)                                       \
            {                                                                                   \
                const int jp = t + P * u;                                                       \
                _Pragma("unroll") for (int r = 0; r < RP; ++r)                                  \
                {                                                                               \
                    const int e = jp + r * (SUB / RP);                                          \
                    sr[e * RS + jl] = vr[u * RP + r];                                           \
                    si[e * RS + jl] = vi[u * RP + r];                                           \
                }                                                                               \
            }                                                                                   \
            __syncthreads();                                                                    \
        } else {                                                                                \
            _Pragma("unroll") for (int u = 0; u < U; ++u)                                       \
            {                                                                                   \
                const int jp = t + P * u;                                                       \
                _Pragma("unroll") for (int r = 0; r < RP; ++r)                                  \
                {                                                                               \
                    const int e = jp + r * (SUB / RP);                                          \
                    put_out(ooff + j + (int64_t)e * NJ, vr[u * RP + r], vi[u * RP + r]);        \
                }                                                                               \
            }                                                                                   \
        }                                                                                       \
    }
            SFFT_DIF_INTERNAL(1)
            SFFT_DIF_INTERNAL(2)
            SFFT_DIF_INTERNAL(3)
            SFFT_DIF_INTERNAL(4)
            SFFT_DIF_INTERNAL(5)
#undef SFFT_DIF_INTERNAL
        }
    }
}

}  // namespace sfft
