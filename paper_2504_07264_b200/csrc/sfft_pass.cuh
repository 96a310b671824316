// sfft_pass.cuh -- multi-pass Stockham schedule for N = 2^m > 4096.
//
// Replaces the reference's cache-blocked wide-stage executor
// (transform.py:219-237 segments + _dit_stage_pair slabs, :153-200) for
// long signals.  The m stages are split into G groups of L_g <= 8
// consecutive stages; one launch per group.  Group (S, L) treats a row as
// N / 2^L independent 2^L-point sub-problems
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
//
// Specialisation: the group with S = 0 (template S0) is the only one whose
// stages can be stage 1 or carry trivial factors, so every other group runs
// with compile-time "generic factor" stages; in-row indices are 32-bit
// (m <= 30); the owner-field address maps of a sharded transform
// (sfft_dist_*) are compiled in only for DIST launches.
#pragma once
#include <type_traits>

#include "sfft_common.cuh"

namespace sfft {

// Global Stockham index -> local address, for a rank of a sharded transform
// (sfft_dist): remove the b-bit rank field at bit p1; optionally then move
// the b-bit destination field at bit p2 to the top (the all-to-all send
// layout: one contiguous segment per destination rank).
struct AddrMap {
    int b;      // field width (log2 ranks)
    int p1;     // position of the owner field that is removed
    int p2;     // position (after removal) of the destination field moved to the top, -1 = none
    int width;  // bits of the index after removal (m - b)
    __host__ __device__ __forceinline__ uint32_t operator()(uint32_t x) const
    {
        const uint32_t lo1 = x & ((1u << p1) - 1u);
        x = ((x >> (p1 + b)) << p1) | lo1;
        if (p2 < 0) return x;
        const uint32_t h = (x >> p2) & ((1u << b) - 1u);
        const uint32_t lo2 = x & ((1u << p2) - 1u);
        const uint32_t rest = ((x >> (p2 + b)) << p2) | lo2;
        return (h << (width - b)) | rest;
    }
};

struct PassArgs {
    const void *x0, *x1;   // source planes (or pairs when the source is interleaved)
    void *y0, *y1;         // destination planes (or pairs)
    int64_t batch;
    int64_t in_stride, out_stride;
    int m;                 // log2 N (<= 30)
    int S;                 // stage offset of this group
    int swap_in, swap_out; // channel swap of the inverse (first / last launch)
    double scale;          // applied at the destination when swap_out
    const void *tw;        // stage-major table, stages 1..tw_cat_top (vec2_t<T>)
    int tw_cat_top;
    const void *tw_top_tab;// fp64, m > 20: stage-m table for the stages above tw_cat_top
    const double2 *coarse; // two-level fp32 twiddles (see TwTwoLevel)
    int coarse_log;
    const double2 *fine;
    // sharded transforms: this launch runs the sub-problems whose index has
    // `jrank` in the jb-bit field at bit jpos; addresses go through the maps
    int jb, jpos, jrank;
    AddrMap in_map, out_map;
    // fused exchange (sfft_dist_exec_phase0_p2p): when npeers > 0 the output
    // address h*seg + r (send layout) is stored straight into peer h's
    // receive buffer at slot jrank: peer_{re,im}[h] + jrank*seg + r
    int npeers;
    int seg_log;
    void *peer_re[8], *peer_im[8];
    // L2-blocked schedule (sfft_abi.cu exec_blocked; DIST launches only):
    // keep_out -- the destination is a block scratch the next launch reads
    // back, store with the default (L2-resident) policy instead of
    // evict-first; discard_in -- the source is such a scratch, drop its lines
    // from L2 after reading them (discard.global.L2: no write-back of data
    // that is dead)
    int keep_out, discard_in;
};

// p + k * stride_bytes as one 32x32->64 multiply-add (IMAD.WIDE.U32): the
// strided plane addresses of a pass launch are a per-thread base plus a
// compile-time multiple of a launch-uniform stride.
template <typename P>
__device__ __forceinline__ P *at_stride(P *p, uint32_t stride_bytes, uint32_t k)
{
    using C = typename std::conditional<std::is_const<P>::value, const char, char>::type;
    return reinterpret_cast<P *>(reinterpret_cast<C *>(p) + (uint64_t)stride_bytes * k);
}

__device__ __forceinline__ void l2_discard(const void *p)
{
    asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}

template <typename T, int L, int LR_REQ>
struct PassShape {
    static constexpr int SUB = 1 << L;
    static constexpr int LR = cmin(LR_REQ, L);
    static constexpr int R = 1 << LR;
    static constexpr int P = SUB / R;                 // threads per sub-problem
    // sub-problems per CTA: 128-byte global runs (32 fp32 / 16 fp64), halved
    // for the 2^10-point groups so the [e][TJ+1] tile still fits one SM
#ifdef SFFT_PASS_TJ64
    static constexpr int TJ = (sizeof(T) == 4 ? (L <= 7 ? 64 : 32) : 16) >> (L >= 10 ? 1 : 0);
#else
    static constexpr int TJ = (sizeof(T) == 4 ? 32 : 16) >> (L >= 10 ? 1 : 0);
#endif
    static constexpr int NT = TJ * P;
    static constexpr int RS = TJ + 1;                 // smem row stride
    static constexpr int NPI = (L + LR - 1) / LR;     // internal register passes
    // + the per-tile stage factors w_{S+s}(c), s = 1..L, of the TJ columns
    static constexpr int smem_bytes() { return 2 * SUB * RS * (int)sizeof(T) + L * TJ * 2 * (int)sizeof(T); }
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

template <typename T>
__device__ __forceinline__ const T *src_plane(const PIO<T, false> &p, int k) { return k ? p.ai : p.ar; }
template <typename T>
__device__ __forceinline__ const T *src_plane(const PIO<T, true> &, int) { return nullptr; }
template <typename T>
__device__ __forceinline__ T *dst_plane(const PIO<T, false> &p, int k) { return k ? p.bi : p.br; }
template <typename T>
__device__ __forceinline__ T *dst_plane(const PIO<T, true> &, int) { return nullptr; }

// Twiddle source of a group: the S = 0 group only touches stages <= 8, all in
// the stage-major table; later groups may need the large-stage sources.
template <typename T, bool S0> struct PassTw { using type = TwCatTop<T>; };
template <> struct PassTw<float, false> { using type = TwTwoLevel<float>; };
template <> struct PassTw<float, true> { using type = TwCat<float>; };
template <> struct PassTw<double, true> { using type = TwCat<double>; };

template <typename T, bool S0>
__device__ __forceinline__ typename PassTw<T, S0>::type make_pass_tw(const PassArgs &a)
{
    typename PassTw<T, S0>::type tw;
    tw.tab = (const vec2_t<T> *)a.tw;
    if constexpr (!S0) {
        tw.cat_top = a.tw_cat_top;
        if constexpr (sizeof(T) == 8) {
            tw.top_tab = (const vec2_t<T> *)a.tw_top_tab;
            tw.top = a.m;
        } else {
            tw.set_tables(a.coarse, a.coarse_log, a.fine, a.m);
        }
    }
    return tw;
}

// (plain __launch_bounds__(NT): an explicit min-blocks of 1, 5 or 6 measured
// 20%, 4% and 50% slower on N = 2^28, tools/ab_variants.sh)
// fp32: at least 1024 threads' worth of CTAs per SM (<= 64 registers; the
// column-factor staging otherwise lands at 72-80 registers, 3 CTAs of 256
// per SM, measured 3-4% slower on N = 2^28 even though the cap spills 20
// bytes).  fp64: 0 = no minimum (the compiler's choice; 1 would let it take
// up to 233 registers).
// The address-map variants (sharded DIST launches, interleaved output) carry
// more live address state: at the 64-register cap they spilled 20-28 bytes
// per thread, so they take 3 CTAs of 256 (<= 85 registers) instead.
template <typename T, int L, int LR, bool WIDE = false>
struct PassMinBlocks {
    static constexpr int NT = PassShape<T, L, LR>::NT;
    static constexpr int TPS = WIDE ? 768 : 1024;    // threads per SM to fit
    static constexpr int value = sizeof(T) == 4 ? (TPS / NT < 1 ? 1 : (TPS / NT > 8 ? 8 : TPS / NT)) : 0;
};
#ifdef SFFT_PASS_MINB
#define SFFT_PASS_LB(T, L, LR, WIDE) __launch_bounds__(PassShape<T, L, LR>::NT, SFFT_PASS_MINB)
#else
#define SFFT_PASS_LB(T, L, LR, WIDE) __launch_bounds__(PassShape<T, L, LR>::NT, (PassMinBlocks<T, L, LR, WIDE>::value))
#endif
template <typename T, int L, int LR_REQ, bool DIF, bool IL_IN, bool IL_OUT, bool S0, bool DIST>
__global__ void SFFT_PASS_LB(T, L, LR_REQ, DIST || IL_OUT)
sfft_pass_kernel(const PassArgs a)
{
    using Sh = PassShape<T, L, LR_REQ>;
    constexpr int SUB = Sh::SUB, LR = Sh::LR, R = Sh::R, P = Sh::P, TJ = Sh::TJ, NT = Sh::NT,
                  RS = Sh::RS, NPI = Sh::NPI;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    // the [e][jl] tile: (re, im) pairs in one array (one 64/128-bit shared
    // access per complex value), or two planes with -DSFFT_PASS_PLANAR_X
    T *sr = reinterpret_cast<T *>(smem_raw);
    T *si = sr + SUB * RS;
    vec2_t<T> *sx = reinterpret_cast<vec2_t<T> *>(smem_raw);
    vec2_t<T> *cs = reinterpret_cast<vec2_t<T> *>(si + SUB * RS);   // [L][TJ] column factors
#ifdef SFFT_PASS_PLANAR_X
    constexpr bool PAIRX = false;
#else
    constexpr bool PAIRX = true;
#endif
    auto xld = [&](int i) -> vec2_t<T> {
        if constexpr (PAIRX) {
            return sx[i];
        } else {
            vec2_t<T> w;
            w.x = sr[i];
            w.y = si[i];
            return w;
        }
    };
    auto xst = [&](int i, vec2_t<T> w) {
        if constexpr (PAIRX) {
            sx[i] = w;
        } else {
            sr[i] = w.x;
            si[i] = w.y;
        }
    };

    const int m = a.m;
    const int S = S0 ? 0 : a.S;
    const uint32_t NJ = 1u << (m - L);                  // sub-problems per row (global)
    const uint32_t tiles = (NJ >> (DIST ? a.jb : 0)) / TJ;
    const int64_t row = (int64_t)(blockIdx.x / tiles);
    uint32_t j0 = (blockIdx.x % tiles) * TJ;
    if constexpr (DIST) {   // insert the rank field (jpos >= log2 TJ keeps a tile contiguous)
        const uint32_t lo = j0 & ((1u << a.jpos) - 1u);
        j0 = ((j0 >> a.jpos) << (a.jpos + a.jb)) | ((uint32_t)a.jrank << a.jpos) | lo;
    }
    const int tid = threadIdx.x;
    const int jl = tid % TJ, t = tid / TJ;
    const uint32_t j = j0 + jl;
    const uint32_t ns = 1u << S;
    const uint32_t c = j & (ns - 1u);
    const uint32_t gbase = (j >> S) * ns * SUB + c;     // DIT destination / DIF source of o: gbase + ns*o
    const int64_t ioff = row * a.in_stride, ooff = row * a.out_stride;
    const AddrMap imap = a.in_map, omap = a.out_map;
    auto iaddr = [&](uint32_t x) -> int64_t { return ioff + (DIST ? imap(x) : x); };
    auto oaddr = [&](uint32_t x) -> int64_t { return ooff + (DIST ? omap(x) : x); };

    PIO<T, IL_IN> src = make_pio<T, IL_IN>(a);
    PIO<T, IL_OUT> dst = make_pio<T, IL_OUT>(a);
    const auto tw = make_pass_tw<T, S0>(a);
    using I = typename PassTw<T, S0>::type::index_t;
    const bool swap_in = a.swap_in != 0, swap_out = a.swap_out != 0;
    const T scale = (T)a.scale;
    // the inverse's channel swap: planar sides exchange their plane pointers
    // once (no per-element selects); interleaved sides swap values
    if constexpr (!IL_IN) {
        if (swap_in) {
            const T *t0 = src.ar;
            src.ar = src.ai;
            src.ai = t0;
        }
    }
    if constexpr (!IL_OUT) {
        if (swap_out) {
            T *t0 = dst.br;
            dst.br = dst.bi;
            dst.bi = t0;
        }
    }

    auto put_out = [&](int64_t off, T re, T im) {
        if (swap_out) {
            if constexpr (IL_OUT) {
                const T t = re;
                re = im * scale;
                im = t * scale;
            } else {   // planes already exchanged
                re *= scale;
                im *= scale;
            }
        }
        if constexpr (DIST) {
            if (a.npeers > 0) {   // NVLink/NVSwitch peer store into the receiver's slot
                const int h = (int)(off >> a.seg_log);
                const int64_t r = ((int64_t)a.jrank << a.seg_log) + (off & ((int64_t(1) << a.seg_log) - 1));
                st_stream((T *)(swap_out ? a.peer_im[h] : a.peer_re[h]) + r, re);
                st_stream((T *)(swap_out ? a.peer_re[h] : a.peer_im[h]) + r, im);
                return;
            }
        }
        if constexpr (DIST && !IL_OUT) {
            if (a.keep_out) {   // block scratch: leave it in L2 for the next launch
                dst.br[off] = re;
                dst.bi[off] = im;
                return;
            }
        }
        dst.store(off, re, im);
    };
    auto get_in = [&](int64_t off, T &re, T &im) {
        T x, y;
        src.load(off, x, y);
        if constexpr (IL_IN) {
            re = swap_in ? y : x;
            im = swap_in ? x : y;
        } else {
            re = x;
            im = y;
        }
    };
    // Planar, unsharded launches: per-thread plane pointers + uniform byte
    // strides, so each strided access costs one IMAD.WIDE instead of the
    // 32-bit index -> 64-bit offset -> scaled address sequence (~6 integer
    // instructions per access on the S > 0 launches).
    constexpr bool FAST_IN = !DIST && !IL_IN, FAST_OUT = !DIST && !IL_OUT;
    const uint32_t nj_bytes = NJ * (uint32_t)sizeof(T), ns_bytes = ns * (uint32_t)sizeof(T);
    // DIT loads / DIF stores: element j + (t + k) * NJ of the row
    const T *in_r = nullptr, *in_i = nullptr;
    T *out_r = nullptr, *out_i = nullptr;
    if constexpr (FAST_IN && !DIF) {
        const int64_t b = ioff + j + (int64_t)t * NJ;
        in_r = (const T *)src_plane(src, 0) + b;
        in_i = (const T *)src_plane(src, 1) + b;
    }
    if constexpr (FAST_OUT && DIF) {
        const int64_t b = ooff + j + (int64_t)t * NJ;
        out_r = (T *)dst_plane(dst, 0) + b;
        out_i = (T *)dst_plane(dst, 1) + b;
    }
    // DIT stores (S > 0): element gbase + ns * (t + k)
    if constexpr (FAST_OUT && !DIF && !S0) {
        const int64_t b = ooff + gbase + (int64_t)ns * t;
        out_r = (T *)dst_plane(dst, 0) + b;
        out_i = (T *)dst_plane(dst, 1) + b;
    }
    auto put_fast = [&](T *pr, T *pi, T re, T im) {
        if (swap_out) {   // planes already exchanged
            re *= scale;
            im *= scale;
        }
        st_stream(pr, re);
        st_stream(pi, im);
    };

    // after the first internal pass consumed the tile (so every load of it
    // has landed): drop the scratch lines it came from.  A line is the TJ
    // sub-problems of one element row e (128 bytes); the first thread of each
    // row group issues the discards for its rows.
    auto discard_tile = [&]() {
        if constexpr (DIST && !DIF && !IL_IN) {
            if (a.discard_in && jl == 0) {
#pragma unroll
                for (int u = 0; u < R / (1 << LR); ++u)
#pragma unroll
                    for (int r = 0; r < (1 << LR); ++r) {
                        const int e = (t + P * u) + r * (SUB >> LR);
                        const int64_t off = iaddr(j0 + (uint32_t)e * NJ);
                        l2_discard(src.ar + off);
                        l2_discard(src.ai + off);
                    }
            }
        }
    };

    vec2_t<T> v[R];

    // fp32 groups after the first: every base factor of every internal pass,
    // fetched up front (independent of the data) -- pre[pass][u*K + t-1]
    // (measured: fetching them up front raises register use 63 -> 79 and
    // costs ~6% on N = 2^28, tools/ab_cfg5.sh; enable with -DSFFT_PASS_PRE)
#ifdef SFFT_PASS_PRE
    constexpr bool PRE = FactorTw<T>::value && !S0;
#else
    constexpr bool PRE = false;
#endif
    vec2_t<T> pre[NPI][R];
    // fp32 groups after the first: the factor of stage S+s at index
    // q = c + (x << S), x < 2^(s-1), is w_{S+s}(c) * w_s(x).  The CTA looks
    // the column parts w_{S+s}(c) up once per tile ([L][TJ] in shared memory,
    // L*TJ two-level lookups instead of L/LR*R per thread) while the tile's
    // loads are in flight; the x part is a small-stage table entry.
#ifdef SFFT_PASS_NO_CSTAGE
    constexpr bool CST = false;
#else
    constexpr bool CST = FactorTw<T>::value && !S0 && !PRE;
#endif
    auto stage_columns = [&]() {
        if constexpr (CST) {
            for (int k = tid; k < L * TJ; k += NT) {
                const int st = k / TJ, l = k - st * TJ;
                cs[k] = tw.get(S + 1 + st, (I)((j0 + (uint32_t)l) & (ns - 1u)));
            }
            __syncthreads();
        }
    };
    // base factors of stages S+sp+1 .. S+sp+KP for internal thread jp
    auto column_factors = [&](int sp, int KP, int jp, vec2_t<T> *cf) {
        const int x = jp & ((1 << sp) - 1);
        for (int tt = 1; tt <= KP; ++tt) {
            vec2_t<T> w = cs[(sp + tt - 1) * TJ + jl];
            if (sp > 0) {
                const vec2_t<T> sm = ldtw(tw.tab + ((1 << (sp + tt - 1)) - 1) + x);
                T r, i;
                cmul(w.x, w.y, sm.x, sm.y, r, i);
                w.x = r;
                w.y = i;
            }
            cf[tt - 1] = w;
        }
    };

    if constexpr (PRE) {
#pragma unroll
        for (int pp = 0; pp < NPI; ++pp) {
            const int sp = pp * LR;
            const int kp = cmin(LR, L - sp);
            const int nsp = 1 << sp;
#pragma unroll
            for (int u = 0; u < R / (1 << kp); ++u) {
                const int jp = t + P * u;
                const I cb = (I)(c + ((uint32_t)(jp & (nsp - 1)) << S));
#pragma unroll
                for (int tt = 1; tt <= kp; ++tt) pre[pp][u * kp + tt - 1] = tw.get(S + sp + tt, cb);
            }
        }
    }

    if constexpr (!DIF) {
        // ------------------------------ DIT ------------------------------
#pragma unroll
        for (int pp = 0; pp < NPI; ++pp) {
            const int sp = pp * LR;
            const int kp = cmin(LR, L - sp);
#define SFFT_DIT_INTERNAL(KP)                                                                   \
    if constexpr (KP <= LR) if (kp == KP) {                                                     \
        constexpr int RP = 1 << KP, U = R / RP;                                                 \
        const int nsp = 1 << sp;                                                                \
        _Pragma("unroll") for (int u = 0; u < U; ++u)                                           \
        {                                                                                       \
            const int jp = t + P * u;                                                           \
            _Pragma("unroll") for (int r = 0; r < RP; ++r)                                      \
            {                                                                                   \
                const int e = jp + r * (SUB / RP);                                              \
                if (pp == 0) {                                                                  \
                    if constexpr (FAST_IN) {                                                    \
                        const uint32_t k_ = (uint32_t)(P * u + r * (SUB / RP));                 \
                        v[u * RP + r].x = ld_stream(at_stride(in_r, nj_bytes, k_));             \
                        v[u * RP + r].y = ld_stream(at_stride(in_i, nj_bytes, k_));             \
                    } else {                                                                    \
                        get_in(iaddr(j + (uint32_t)e * NJ), v[u * RP + r].x, v[u * RP + r].y);  \
                    }                                                                           \
                }                                                                               \
                else {                                                                          \
                    v[u * RP + r] = xld(e * RS + jl);                                        \
                }                                                                               \
            }                                                                                   \
        }                                                                                       \
        if (pp == 0) stage_columns();                                                           \
        _Pragma("unroll") for (int u = 0; u < U; ++u)                                           \
        {                                                                                       \
            const int jp = t + P * u;                                                           \
            vec2_t<T> cf[KP];                                                                   \
            if constexpr (CST) column_factors(sp, KP, jp, cf);                                  \
            dit_stages<T, KP, S0>(v + u * RP, S + sp,                             \
                                  (I)(c + ((uint32_t)(jp & (nsp - 1)) << S)), tw,               \
                                  CST ? cf : PRE ? &pre[pp][u * KP] : nullptr);                 \
        }                                                                                       \
        if (DIST && pp == 0) discard_tile();                                                    \
        const bool last = pp == NPI - 1;                                                        \
        if (!last || S0) {                                                                      \
            if (pp > 0) __syncthreads();                                                        \
            _Pragma("unroll") for (int u = 0; u < U; ++u)                                       \
            {                                                                                   \
                const int jp = t + P * u;                                                       \
                const int base = (jp >> sp) * nsp * RP + (jp & (nsp - 1));                      \
                _Pragma("unroll") for (int f = 0; f < RP; ++f)                                  \
                {                                                                               \
                    const int e = base + nsp * f;                                               \
                    xst(e * RS + jl, v[u * RP + brev(f, KP)]);                                    \
                }                                                                               \
            }                                                                                   \
            __syncthreads();                                                                    \
        } else {                                                                                \
            _Pragma("unroll") for (int u = 0; u < U; ++u)                                       \
            {                                                                                   \
                const int jp = t + P * u;                                                       \
                _Pragma("unroll") for (int f = 0; f < RP; ++f)                                  \
                {                                                                               \
                    const uint32_t o = jp + nsp * f;                                            \
                    if constexpr (FAST_OUT) {                                                   \
                        const uint32_t k_ = (uint32_t)(P * u + nsp * f);                        \
                        put_fast(at_stride(out_r, ns_bytes, k_), at_stride(out_i, ns_bytes, k_), \
                                 v[u * RP + brev(f, KP)].x, v[u * RP + brev(f, KP)].y);         \
                    } else {                                                                    \
                        put_out(oaddr(gbase + ns * o), v[u * RP + brev(f, KP)].x,                \
                                v[u * RP + brev(f, KP)].y);                                      \
                    }                                                                           \
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
        if constexpr (S0) {
            // outputs of this tile are the contiguous rows j0..j0+TJ of 2^L:
            // copy smem [o][jl] -> global in linear order
            const uint32_t obase = j0 * SUB;
#pragma unroll
            for (int kk = 0; kk < R; ++kk) {
                const int k = tid + kk * NT, jj = k >> L, o = k & (SUB - 1);
                const vec2_t<T> w = xld(o * RS + jj);
                put_out(oaddr(obase + k), w.x, w.y);
            }
        }
    } else {
        // ------------------------------ DIF ------------------------------
        if constexpr (S0) {
            // inputs are the contiguous rows j0..j0+TJ of 2^L: stage them
            // (all R loads of a thread first, then the shared stores: the
            // loop written load->store serialised the load latencies, 2x
            // slower than the DIT S = 0 launch)
            const uint32_t ibase = j0 * SUB;
            static_assert(TJ * SUB == R * NT, "one tile = R elements per thread");
#pragma unroll
            for (int kk = 0; kk < R; ++kk) get_in(iaddr(ibase + tid + kk * NT), v[kk].x, v[kk].y);
#pragma unroll
            for (int kk = 0; kk < R; ++kk) {
                const int k = tid + kk * NT, jj = k >> L, o = k & (SUB - 1);
                xst(o * RS + jj, v[kk]);
            }
            __syncthreads();
        }
#pragma unroll
        for (int pp = NPI - 1; pp >= 0; --pp) {
            const int sp = pp * LR;
            const int kp = cmin(LR, L - sp);
#define SFFT_DIF_INTERNAL(KP)                                                                   \
    if constexpr (KP <= LR) if (kp == KP) {                                                     \
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
                if (first && !S0) {                                                             \
                    if constexpr (FAST_IN) {                                                    \
                        const int64_t b_ = ioff + gbase + (int64_t)ns * (uint32_t)base;         \
                        const uint32_t k_ = (uint32_t)(nsp * f);                                \
                        v[d].x = ld_stream(at_stride(src_plane(src, 0) + b_, ns_bytes, k_));    \
                        v[d].y = ld_stream(at_stride(src_plane(src, 1) + b_, ns_bytes, k_));    \
                    } else {                                                                    \
                        get_in(iaddr(gbase + ns * (uint32_t)e), v[d].x, v[d].y);                \
                    }                                                                           \
                }                                                                               \
                else {                                                                          \
                    v[d] = xld(e * RS + jl);                                                    \
                }                                                                               \
            }                                                                                   \
        }                                                                                       \
        if (first) stage_columns();                                                             \
        _Pragma("unroll") for (int u = 0; u < U; ++u)                                           \
        {                                                                                       \
            const int jp = t + P * u;                                                           \
            vec2_t<T> cf[KP];                                                                   \
            if constexpr (CST) column_factors(sp, KP, jp, cf);                                  \
            dif_stages<T, KP, S0>(v + u * RP, S + sp,                             \
                                  (I)(c + ((uint32_t)(jp & (nsp - 1)) << S)), tw,               \
                                  CST ? cf : PRE ? &pre[pp][u * KP] : nullptr);                 \
        }                                                                                       \
        if (pp != 0) {                                                                          \
            if (!first || S0) __syncthreads();                                                  \
            _Pragma("unroll") for (int u = 0; u < U; ++u)                                       \
            {                                                                                   \
                const int jp = t + P * u;                                                       \
                _Pragma("unroll") for (int r = 0; r < RP; ++r)                                  \
                {                                                                               \
                    const int e = jp + r * (SUB / RP);                                          \
                    xst(e * RS + jl, v[u * RP + r]);                                            \
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
                    if constexpr (FAST_OUT) {                                                   \
                        const uint32_t k_ = (uint32_t)(P * u + r * (SUB / RP));                 \
                        put_fast(at_stride(out_r, nj_bytes, k_), at_stride(out_i, nj_bytes, k_), \
                                 v[u * RP + r].x, v[u * RP + r].y);                             \
                    } else {                                                                    \
                        put_out(oaddr(j + (uint32_t)e * NJ), v[u * RP + r].x, v[u * RP + r].y);   \
                    }                                                                           \
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
