// sfft_fused_pair.cuh -- fp32 planar fused kernel that runs TWO signals per
// thread, packed across the pair: N = 2^LOGN <= 4096.
//
// Same stage sequence, Stockham register passes and shared-memory exchange
// order as sfft_fused.cuh (transform.py:208-270: DIT t = b*w; b = a - t;
// a = a + t, DIF t = a - b; a = a + b; b = t*w), but each virtual thread j
// holds element e of rows 2q and 2q+1 in one register pair:
//     vr[k] = (re[2q][e_k], re[2q+1][e_k]),  vi[k] = (im[2q][e_k], im[2q+1][e_k])
// so every butterfly and complex product is one packed f32x2 instruction for
// both signals with the factor broadcast, (wr, wr) / (wi, wi):
//     t.re = fma2(b.re, (wr,wr), (b.im * (-wi,-wi)))     = fma(br, wr, -(bi*wi))
//     t.im = fma2(b.re, (wi,wi), (b.im * ( wr, wr)))     = fma(br, wi, bi*wr)
// -- per lane exactly numpy's complex multiply rounding, the same values as
// the single-signal kernel.  Against that kernel it drops the operand
// duplication moves of the packed complex multiply, forms each factor once
// for two signals, and exchanges (s0, s1) pairs with 64-bit shared accesses
// (one address per pair; the 8-byte exchange layouts of sfft_layouts.h).
#pragma once
#include "sfft_fused.cuh"

namespace sfft {

__device__ __forceinline__ float2 bc2(float v) { return make_float2(v, v); }

// K consecutive DIT stages (global stages gs+1 .. gs+K) on 2^K pair-packed
// complex values; register map and factor indices as dit_stages.
template <int K, typename TW>
__device__ __forceinline__ void dit_stages_pair(float2 *vr, float2 *vi, int gs, int cbase, const TW &tw,
                                                const float2 *pre)
{
    const bool first = gs == 0;
#pragma unroll
    for (int t = 1; t <= K; ++t) {
        const int half = (1 << K) >> t;
        const int i = gs + t;
        float2 base = make_float2(1.f, 0.f);
        if (!first) base = pre ? pre[t - 1] : tw.get(i, cbase);
#pragma unroll
        for (int f = 0; f < (1 << (t - 1)); ++f) {
            const int rf = brev(f, t - 1) * 2 * half;
            const int kind = i == 1 ? 0 : (first && f == 0) ? 1 : (first && (f << 2) == (1 << t)) ? 2 : 3;
            float2 w = make_float2(1.f, 0.f);
            if (kind == 3) w = stage_factor<float>(t, f, i, first, cbase, gs, tw, base);
            const float2 WR = bc2(w.x), WI = bc2(w.y), NWI = bc2(-w.y);
#pragma unroll
            for (int r = 0; r < half; ++r) {
                const int p1 = r + rf, p2 = p1 + half;
                float2 tr, ti;
                if (kind == 3) {
                    tr = fma2(vr[p2], WR, mul2(vi[p2], NWI));
                    ti = fma2(vr[p2], WI, mul2(vi[p2], WR));
                } else if (kind == 2) {   // * (-j): (re, im) -> (im, -re)
                    tr = vi[p2];
                    ti = make_float2(-vr[p2].x, -vr[p2].y);
                } else {
                    tr = vr[p2];
                    ti = vi[p2];
                }
                vr[p2] = sub2(vr[p1], tr);
                vi[p2] = sub2(vi[p1], ti);
                vr[p1] = add2(vr[p1], tr);
                vi[p1] = add2(vi[p1], ti);
            }
        }
    }
}

// DIF stages gs+K .. gs+1 (transpose of dit_stages_pair).
template <int K, typename TW>
__device__ __forceinline__ void dif_stages_pair(float2 *vr, float2 *vi, int gs, int cbase, const TW &tw,
                                                const float2 *pre)
{
    const bool first = gs == 0;
#pragma unroll
    for (int t = K; t >= 1; --t) {
        const int half = (1 << K) >> t;
        const int i = gs + t;
        float2 base = make_float2(1.f, 0.f);
        if (!first) base = pre ? pre[t - 1] : tw.get(i, cbase);
#pragma unroll
        for (int f = 0; f < (1 << (t - 1)); ++f) {
            const int rf = brev(f, t - 1) * 2 * half;
            const int kind = i == 1 ? 0 : (first && f == 0) ? 1 : (first && (f << 2) == (1 << t)) ? 2 : 3;
            float2 w = make_float2(1.f, 0.f);
            if (kind == 3) w = stage_factor<float>(t, f, i, first, cbase, gs, tw, base);
            const float2 WR = bc2(w.x), WI = bc2(w.y), NWI = bc2(-w.y);
#pragma unroll
            for (int r = 0; r < half; ++r) {
                const int p1 = r + rf, p2 = p1 + half;
                const float2 dr = sub2(vr[p1], vr[p2]), di = sub2(vi[p1], vi[p2]);
                vr[p1] = add2(vr[p1], vr[p2]);
                vi[p1] = add2(vi[p1], vi[p2]);
                if (kind == 3) {
                    vr[p2] = fma2(dr, WR, mul2(di, NWI));
                    vi[p2] = fma2(dr, WI, mul2(di, WR));
                } else if (kind == 2) {
                    vr[p2] = di;
                    vi[p2] = make_float2(-dr.x, -dr.y);
                } else {
                    vr[p2] = dr;
                    vi[p2] = di;
                }
            }
        }
    }
}

// Global side: rows r0 = 2q and r1 = 2q + 1 of the planar caller arrays
// (r1 may be past the batch: loads give 0, stores are skipped).
struct PairIO {
    const float *xr, *xi;
    float *yr, *yi;
    int64_t is, os;
    bool inv, has1;
    float scale;
    __device__ __forceinline__ PairIO(const FusedArgs &a, int64_t q)
    {
        // the inverse's input channel swap is a plane-pointer exchange
        xr = (const float *)(a.inverse ? a.x1 : a.x0);
        xi = (const float *)(a.inverse ? a.x0 : a.x1);
        yr = (float *)a.y0;
        yi = (float *)a.y1;
        is = a.in_stride;
        os = a.out_stride;
        inv = a.inverse != 0;
        scale = (float)a.scale;
        has1 = 2 * q + 1 < a.batch;
        xr += 2 * q * is;
        xi += 2 * q * is;
        yr += 2 * q * os;
        yi += 2 * q * os;
    }
    __device__ __forceinline__ void load(int e, float2 &r, float2 &i) const
    {
        r.x = ld_stream(xr + e);
        i.x = ld_stream(xi + e);
        r.y = has1 ? ld_stream(xr + is + e) : 0.f;
        i.y = has1 ? ld_stream(xi + is + e) : 0.f;
    }
    __device__ __forceinline__ void store(int e, float2 r, float2 i) const
    {
        if (inv) {   // output channel swap + 1/N of the inverse
            const float2 s = bc2(scale);
            const float2 t = mul2(i, s);
            i = mul2(r, s);
            r = t;
        }
        st_stream(yr + e, r.x);
        st_stream(yi + e, i.x);
        if (has1) {
            st_stream(yr + os + e, r.y);
            st_stream(yi + os + e, i.y);
        }
    }
};

template <int LOGN, int LR_REQ>
using PairShape = FusedShape<LOGN, LR_REQ>;   // P threads per signal PAIR, S pairs per CTA

template <int LOGN, int LR_REQ, bool DIF>
__global__ void __launch_bounds__(PairShape<LOGN, LR_REQ>::NT)
sfft_fused_pair_kernel(const FusedArgs a)
{
    using Sh = PairShape<LOGN, LR_REQ>;
    constexpr int N = Sh::N, R = Sh::R, P = Sh::P, S = Sh::S, LR = Sh::LR, NPASS = Sh::NPASS, NT = Sh::NT;
    constexpr int SSTR = ex_sstr<double, LOGN, LR, NT>();   // 8-byte (s0, s1) elements
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float2 *sbase = reinterpret_cast<float2 *>(smem_raw);

    const int tid = threadIdx.x;
    const int sl = tid / P, t = tid % P;
    const int64_t q = (int64_t)blockIdx.x * S + sl;     // signal pair
    const bool valid = 2 * q < a.batch;
    const PairIO io(a, q);
    const TwCat<float> tw{reinterpret_cast<const float2 *>(a.tw)};
    float2 *sr = sbase + sl * SSTR;
    float2 *si = sbase + S * SSTR + sl * SSTR;
    float2 vr[R], vi[R];
    auto phys = [](int x, int e) { return ex_phys<double, LOGN, LR, NT>(x, e); };

    if constexpr (!DIF) {
#pragma unroll
        for (int p = 0; p < NPASS; ++p) {
            const int SP = p * LR;
            const int KP = cmin(LR, LOGN - SP);
#define SFFT_PAIR_DIT(KPC)                                                                         \
    if constexpr (KPC <= LR) if (KP == KPC) {                                                      \
        constexpr int RP = 1 << KPC, U = R / RP;                                                   \
        const int NS = 1 << SP;                                                                    \
        _Pragma("unroll") for (int u = 0; u < U; ++u)                                              \
        {                                                                                          \
            const int j = t + P * u;                                                               \
            _Pragma("unroll") for (int r = 0; r < RP; ++r)                                         \
            {                                                                                      \
                const int e = j + r * (N / RP);                                                    \
                if (p == 0) {                                                                      \
                    if (valid) io.load(e, vr[u * RP + r], vi[u * RP + r]);                         \
                    else { vr[u * RP + r] = bc2(0.f); vi[u * RP + r] = bc2(0.f); }                 \
                } else {                                                                           \
                    vr[u * RP + r] = sr[phys(p - 1, e)];                                           \
                    vi[u * RP + r] = si[phys(p - 1, e)];                                           \
                }                                                                                  \
            }                                                                                      \
        }                                                                                          \
        _Pragma("unroll") for (int u = 0; u < U; ++u)                                              \
        {                                                                                          \
            const int j = t + P * u;                                                               \
            dit_stages_pair<KPC>(vr + u * RP, vi + u * RP, SP, j & (NS - 1), tw, nullptr);         \
        }                                                                                          \
        if (p < NPASS - 1) {                                                                       \
            if (p > 0) sig_sync<P>();                                                              \
            _Pragma("unroll") for (int u = 0; u < U; ++u)                                          \
            {                                                                                      \
                const int j = t + P * u;                                                           \
                const int base = (j >> SP) * NS * RP + (j & (NS - 1));                             \
                _Pragma("unroll") for (int f = 0; f < RP; ++f)                                     \
                {                                                                                  \
                    const int e = base + NS * f;                                                   \
                    sr[phys(p, e)] = vr[u * RP + brev(f, KPC)];                                    \
                    si[phys(p, e)] = vi[u * RP + brev(f, KPC)];                                    \
                }                                                                                  \
            }                                                                                      \
            sig_sync<P>();                                                                         \
        } else if (valid) {                                                                        \
            _Pragma("unroll") for (int u = 0; u < U; ++u)                                          \
            {                                                                                      \
                const int j = t + P * u;                                                           \
                _Pragma("unroll") for (int f = 0; f < RP; ++f)                                     \
                    io.store(j + NS * f, vr[u * RP + brev(f, KPC)], vi[u * RP + brev(f, KPC)]);    \
            }                                                                                      \
        }                                                                                          \
    }
            SFFT_PAIR_DIT(1)
            SFFT_PAIR_DIT(2)
            SFFT_PAIR_DIT(3)
            SFFT_PAIR_DIT(4)
            SFFT_PAIR_DIT(5)
#undef SFFT_PAIR_DIT
        }
    } else {
#pragma unroll
        for (int qq = 0; qq < NPASS; ++qq) {
            const int p = NPASS - 1 - qq;
            const int SP = p * LR;
            const int KP = cmin(LR, LOGN - SP);
#define SFFT_PAIR_DIF(KPC)                                                                         \
    if constexpr (KPC <= LR) if (KP == KPC) {                                                      \
        constexpr int RP = 1 << KPC, U = R / RP;                                                   \
        const int NS = 1 << SP;                                                                    \
        _Pragma("unroll") for (int u = 0; u < U; ++u)                                              \
        {                                                                                          \
            const int j = t + P * u;                                                               \
            const int base = (j >> SP) * NS * RP + (j & (NS - 1));                                 \
            _Pragma("unroll") for (int f = 0; f < RP; ++f)                                         \
            {                                                                                      \
                const int e = base + NS * f;                                                       \
                const int d = u * RP + brev(f, KPC);                                               \
                if (qq == 0) {                                                                     \
                    if (valid) io.load(e, vr[d], vi[d]);                                           \
                    else { vr[d] = bc2(0.f); vi[d] = bc2(0.f); }                                   \
                } else {                                                                           \
                    vr[d] = sr[phys(p, e)];                                                        \
                    vi[d] = si[phys(p, e)];                                                        \
                }                                                                                  \
            }                                                                                      \
        }                                                                                          \
        _Pragma("unroll") for (int u = 0; u < U; ++u)                                              \
        {                                                                                          \
            const int j = t + P * u;                                                               \
            dif_stages_pair<KPC>(vr + u * RP, vi + u * RP, SP, j & (NS - 1), tw, nullptr);         \
        }                                                                                          \
        if (p > 0) {                                                                               \
            if (qq > 0) sig_sync<P>();                                                             \
            _Pragma("unroll") for (int u = 0; u < U; ++u)                                          \
            {                                                                                      \
                const int j = t + P * u;                                                           \
                _Pragma("unroll") for (int r = 0; r < RP; ++r)                                     \
                {                                                                                  \
                    const int e = j + r * (N / RP);                                                \
                    sr[phys(p - 1, e)] = vr[u * RP + r];                                           \
                    si[phys(p - 1, e)] = vi[u * RP + r];                                           \
                }                                                                                  \
            }                                                                                      \
            sig_sync<P>();                                                                         \
        } else if (valid) {                                                                        \
            _Pragma("unroll") for (int u = 0; u < U; ++u)                                          \
            {                                                                                      \
                const int j = t + P * u;                                                           \
                _Pragma("unroll") for (int r = 0; r < RP; ++r)                                     \
                    io.store(j + r * (N / RP), vr[u * RP + r], vi[u * RP + r]);                    \
            }                                                                                      \
        }                                                                                          \
    }
            SFFT_PAIR_DIF(1)
            SFFT_PAIR_DIF(2)
            SFFT_PAIR_DIF(3)
            SFFT_PAIR_DIF(4)
            SFFT_PAIR_DIF(5)
#undef SFFT_PAIR_DIF
        }
    }
}

template <int LOGN, int LR_REQ>
constexpr int pair_smem_bytes()
{
    using Sh = PairShape<LOGN, LR_REQ>;
    return Sh::NPASS >= 2 ? 2 * Sh::S * ex_sstr<double, LOGN, Sh::LR, Sh::NT>() * 8 : 0;
}

}  // namespace sfft
