// sfft_common.cuh -- shared device helpers for the split-format DFT kernels.
//
// Arithmetic contract: every kernel executes the
// reference's radix-2 stage factorization literally (PAPER.md:149-165,
// transform.py:131-150): DIT stage i does  t = b*w; b = a - t; a = a + t,
// DIF stage i does  t = a - b; a = a + b; b = t*w, with w the stage-i factor
// cos - j sin from the snapped table (twiddle.py:46-57).  Stage 1 never
// multiplies (transform.py:123-128).  The complex product is rounded the way
// numpy rounds complex128 multiply on x86-64 (re = fma(ar,br,-(ai*bi)),
// im = fma(ar,bi,ai*br)), with explicit _rn intrinsics so nvcc cannot
// re-contract it.  In fp64 this makes the GPU output bit-identical to the
// reference; in fp32 it is the same op sequence in single precision.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "sfft_layouts.h"
#include "sfft_small_tw.h"

namespace sfft {

template <typename T> struct Vec2;
template <> struct Vec2<float> { using type = float2; };
template <> struct Vec2<double> { using type = double2; };
template <typename T> using vec2_t = typename Vec2<T>::type;

__host__ __device__ constexpr int brev(int f, int bits)
{
    int r = 0;
    for (int b = 0; b < bits; ++b) { r = (r << 1) | (f & 1); f >>= 1; }
    return r;
}

__host__ __device__ constexpr int cmin(int a, int b) { return a < b ? a : b; }

template <int V> struct IntC { static constexpr int value = V; };

// f(IntC<g>) for a runtime g in [G, N_): compile-time register indices for
// code specialised per (warp-uniform) group position.
template <int G, int N_, typename F>
__device__ __forceinline__ void with_g(int g, F &&f)
{
    if constexpr (G < N_) {
        if (g == G) f(IntC<G>{});
        else with_g<G + 1, N_>(g, f);
    }
}

// f(IntC<0>), f(IntC<1>), ..., f(IntC<N_-1>) (compile-time loop)
template <int I, int N_, typename F>
__device__ __forceinline__ void static_for(F &&f)
{
    if constexpr (I < N_) {
        f(IntC<I>{});
        static_for<I + 1, N_>(f);
    }
}

__device__ __forceinline__ void cmul(float ar, float ai, float br, float bi, float &cr, float &ci)
{
    cr = __fmaf_rn(ar, br, -__fmul_rn(ai, bi));
    ci = __fmaf_rn(ar, bi, __fmul_rn(ai, br));
}

__device__ __forceinline__ void cmul(double ar, double ai, double br, double bi, double &cr, double &ci)
{
    cr = __fma_rn(ar, br, -__dmul_rn(ai, bi));
    ci = __fma_rn(ar, bi, __dmul_rn(ai, br));
}

__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }

// Read-only twiddle fetch (L1-resident table; never written by a kernel).
__device__ __forceinline__ float2 ldtw(const float2 *p) { return __ldg(p); }
__device__ __forceinline__ double2 ldtw(const double2 *p) { return __ldg(p); }

// Streaming (evict-first) global accesses for the signal planes: every
// element is read once and written once per launch.
__device__ __forceinline__ float ld_stream(const float *p) { return __ldcs(p); }
__device__ __forceinline__ double ld_stream(const double *p) { return __ldcs(p); }
__device__ __forceinline__ float2 ld_stream(const float2 *p) { return __ldcs(p); }
__device__ __forceinline__ double2 ld_stream(const double2 *p) { return __ldcs(p); }
__device__ __forceinline__ void st_stream(float *p, float v) { __stcs(p, v); }
__device__ __forceinline__ void st_stream(double *p, double v) { __stcs(p, v); }
__device__ __forceinline__ void st_stream(float2 *p, float2 v) { __stcs(p, v); }
__device__ __forceinline__ void st_stream(double2 *p, double2 v) { __stcs(p, v); }

// Twiddle sources.  All stage tables are bitwise strided views of the top one
// (SURVEY.md sec. 3B), but the kernels read them "stage-major": stage i's
// 2^(i-1) factors stored contiguously at offset 2^(i-1)-1, so that the lanes
// of a warp (consecutive q) read consecutive 8/16-byte entries instead of one
// cache line each.
//   TwCat:      stages 1..m from the stage-major table (m <= 20).
//   TwCatTop:   stage-major up to cat_top, then the stage-m table read with
//               stride 2^(m-i) (fp64 plans with m > 20 only).
//   TwTwoLevel: fp32 N > 4096: stage-major fp32 table up to cat_top (12);
//               above it w_i(q) = w_i(q & 31) * w_i(q & ~31), the first
//               from a per-stage 32-entry "lane" table (the lanes of a warp
//               hold consecutive q, so this read is contiguous), the second
//               lane-uniform as coarse[hi] * fine[lo]; all in fp64, rounded
//               to fp32 once.  (Reading w_m(q << (m-i)) directly made every
//               lane of a warp touch its own sector: l1tex at 89% on the
//               late N = 2^28 pass groups.)
template <typename T>
struct TwCat {
    using index_t = int;
    const vec2_t<T> *tab;
    __device__ __forceinline__ vec2_t<T> get(int i, int q) const
    {
        return ldtw(tab + ((1 << (i - 1)) - 1) + q);
    }
};

template <typename T>
struct TwCatTop {
    using index_t = int64_t;
    const vec2_t<T> *tab;      // stage-major, stages 1..cat_top
    int cat_top;
    const vec2_t<T> *top_tab;  // stage `top` table (2^(top-1) entries)
    int top;
    __device__ __forceinline__ vec2_t<T> get(int i, int64_t q) const
    {
        if (i <= cat_top) return ldtw(tab + ((int64_t(1) << (i - 1)) - 1) + q);
        return ldtw(top_tab + (q << (top - i)));
    }
};

template <typename T>
struct TwTwoLevel {
    using index_t = int64_t;   // (uint32_t indices measured slower: ptxas spills at 64 registers)
    const vec2_t<T> *tab;      // stage-major fp32, stages 1..cat_top
    int cat_top;
    const double2 *coarse;     // stage coarse_log factors, 2^(coarse_log-1) entries
    int coarse_log;
    const double2 *fine;       // exp(-j 2 pi lo / 2^m), lo < 2^(m - coarse_log),
                               // then the lane table: w_i(l) at (i-1)*32 + l, l < 32
    int m;
    __device__ __forceinline__ void set_tables(const double2 *c, int clog, const double2 *f, int m_)
    {
        coarse = c;
        coarse_log = clog;
        fine = f;
        m = m_;
    }
    __device__ __forceinline__ vec2_t<T> get(int i, int64_t q) const
    {
        if (i <= cat_top) return ldtw(tab + ((int64_t(1) << (i - 1)) - 1) + q);
        const int fb = m - coarse_log;
        const int64_t qq = (q >> 5) << (m - i + 5);          // w_m(qq) = w_i(q & ~31)
        const double2 a = __ldg(coarse + (qq >> fb));
        const double2 b = __ldg(fine + (qq & ((int64_t(1) << fb) - 1)));
        const double2 l = __ldg(fine + (int64_t(1) << fb) + (i - 1) * 32 + (int)(q & 31));
        double r, im, r2, im2;
        cmul(a.x, a.y, b.x, b.y, r, im);
        cmul(r, im, l.x, l.y, r2, im2);
        vec2_t<T> w;
        w.x = (T)r2;
        w.y = (T)im2;
        return w;
    }
};

// Physical slot of logical element e in shared-memory exchange x (the buffer
// between register pass x and x+1, DIT numbering), per a planned layout L
// (sfft_layouts.h, tools/plan_layouts.py): ExLayout (separate exchange
// buffer, padding allowed) or ExLayoutIP (in place in a tile slot: XOR or
// identity only, a bijection on [0, N)).
template <typename L, int ESZ>
__device__ __forceinline__ int ex_phys_l(int x, int e)
{
    constexpr int mask = ESZ == 4 ? 31 : 15;
    const int kind = L::kind(x), a = L::arg(x);
    return kind == 0 ? e
         : kind == 1 ? e + (e >> a)
         : kind == 3 ? e + ((e >> (a & 255)) << (a >> 8))   // shifted pad
                     : (e ^ ((e >> a) & mask));
}

// Exchange slots split as (per-thread part) + (compile-time part) when the
// planner proved the layout additive on that side (L::lin bit 0 = Stockham
// writes, bit 1 = next-pass reads): e = e(t,0,0), ec = e(0,u,k), so the
// kernel addresses the exchange as one base register plus immediates.
template <typename L, int ESZ>
__device__ __forceinline__ int ex_wr_l(int x, int e, int et, int ec)
{
    if (L::lin(x) & 1) return ex_phys_l<L, ESZ>(x, et) + ex_phys_l<L, ESZ>(x, ec);
    return ex_phys_l<L, ESZ>(x, e);
}

template <typename L, int ESZ>
__device__ __forceinline__ int ex_rd_l(int x, int e, int et, int ec)
{
    if (L::lin(x) & 2) return ex_phys_l<L, ESZ>(x, et) + ex_phys_l<L, ESZ>(x, ec);
    return ex_phys_l<L, ESZ>(x, e);
}

template <typename T, int LOGN, int LR, int NT>
__device__ __forceinline__ int ex_phys(int x, int e)
{
    return ex_phys_l<ExLayout<(int)sizeof(T), LOGN, LR, NT>, (int)sizeof(T)>(x, e);
}

template <typename T, int LOGN, int LR, int NT>
__device__ __forceinline__ int ex_wr(int x, int e, int et, int ec)
{
    return ex_wr_l<ExLayout<(int)sizeof(T), LOGN, LR, NT>, (int)sizeof(T)>(x, e, et, ec);
}

template <typename T, int LOGN, int LR, int NT>
__device__ __forceinline__ int ex_rd(int x, int e, int et, int ec)
{
    return ex_rd_l<ExLayout<(int)sizeof(T), LOGN, LR, NT>, (int)sizeof(T)>(x, e, et, ec);
}

template <typename T, int LOGN, int LR, int NT>
__host__ __device__ constexpr int ex_sstr()
{
    return ExLayout<(int)sizeof(T), LOGN, LR, NT>::sstr;
}

// fp32 skips the identity and quarter-turn factors of the first stages
// (count_flops' census: identity rotations cost nothing, a quarter turn is a
// swap/negate, transform.py:312-321).  fp64 multiplies by every factor
// exactly as the reference executor does (transform.py:131-150), which keeps
// it bit-identical including signed zeros.
template <typename T> struct SkipTrivial { static constexpr bool value = false; };
template <> struct SkipTrivial<float> { static constexpr bool value = true; };

// Stage-t factors, t <= 5, as immediates (index 2^(t-1)-1+f); bitwise the
// table values (generated from the same formula, sfft_small_tw.h).
template <typename T> struct SmallTw;
template <> struct SmallTw<float> {
    static __device__ __forceinline__ float2 get(int k) { return make_float2(small_tw_re32(k), small_tw_im32(k)); }
};
template <> struct SmallTw<double> {
    static __device__ __forceinline__ double2 get(int k) { return make_double2(small_tw_re64(k), small_tw_im64(k)); }
};

// fp32 forms the 2^(t-1) factors of a stage from ONE table/two-level lookup:
// w_i(c + f 2^gs) = w_i(c) * w_{2^t}^f (t = i - gs), the second factor an
// immediate.  fp64 reads every factor from the table (bit-exact contract).
template <typename T> struct FactorTw { static constexpr bool value = false; };
template <> struct FactorTw<float> { static constexpr bool value = true; };

// Per-stage base factors w_{gs+t}(cbase), t = 1..K, of one virtual thread
// (fp32 factored twiddles).  Kernels call this once, ahead of the data (and
// for persistent kernels once for all tiles), and pass the array to
// dit_stages/dif_stages as `pre`, so no table or two-level lookup sits on
// the critical path of a pass.
template <typename T, int K, typename TW>
__device__ __forceinline__ void load_bases(vec2_t<T> *pre, int gs, typename TW::index_t cbase, const TW &tw)
{
#pragma unroll
    for (int t = 1; t <= K; ++t) pre[t - 1] = tw.get(gs + t, cbase);
}

// Packed fp32 pair arithmetic (sm_100a FADD2/FMUL2/FFMA2): each lane is
// rounded exactly like the scalar instruction, so the packed path is
// bit-identical to the scalar one -- it only halves the instruction count.
__device__ __forceinline__ unsigned long long f2u(float2 a) { return *reinterpret_cast<unsigned long long *>(&a); }
__device__ __forceinline__ float2 u2f(unsigned long long a) { return *reinterpret_cast<float2 *>(&a); }
__device__ __forceinline__ float2 add2(float2 a, float2 b)
{
    unsigned long long d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)));
    return u2f(d);
}
__device__ __forceinline__ float2 sub2(float2 a, float2 b)
{
    unsigned long long d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)));
    return u2f(d);
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b)
{
    unsigned long long d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)));
    return u2f(d);
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c)
{
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)), "l"(f2u(c)));
    return u2f(d);
}

// c = b * w for a complex value held as (re, im), numpy's rounding:
// (fma(br, wr, -(bi*wi)), fma(br, wi, bi*wr)).  `wq` = (-wi, wr) precomputed.
__device__ __forceinline__ float2 cmulv(float2 b, float2 w, float2 wq)
{
    const float2 q = mul2(make_float2(b.y, b.y), wq);          // (-(bi*wi), bi*wr), exact negation
    return fma2(make_float2(b.x, b.x), w, q);
}
__device__ __forceinline__ double2 cmulv(double2 b, double2 w, double2)
{
    double2 c;
    cmul(b.x, b.y, w.x, w.y, c.x, c.y);
    return c;
}
__device__ __forceinline__ float2 addv(float2 a, float2 b) { return add2(a, b); }
__device__ __forceinline__ float2 subv(float2 a, float2 b) { return sub2(a, b); }
__device__ __forceinline__ double2 addv(double2 a, double2 b) { return make_double2(add_rn(a.x, b.x), add_rn(a.y, b.y)); }
__device__ __forceinline__ double2 subv(double2 a, double2 b) { return make_double2(sub_rn(a.x, b.x), sub_rn(a.y, b.y)); }

// Scalar fp32 forms (same rounding), for kernels where the packed
// instructions' longer dependency chains cost more than the issue slots they
// save (latency-bound shapes; chosen per kernel).
__device__ __forceinline__ float2 cmuls(float2 b, float2 w)
{
    float2 c;
    cmul(b.x, b.y, w.x, w.y, c.x, c.y);
    return c;
}
__device__ __forceinline__ double2 cmuls(double2 b, double2 w) { return cmulv(b, w, w); }
__device__ __forceinline__ float2 adds(float2 a, float2 b) { return make_float2(add_rn(a.x, b.x), add_rn(a.y, b.y)); }
__device__ __forceinline__ float2 subs(float2 a, float2 b) { return make_float2(sub_rn(a.x, b.x), sub_rn(a.y, b.y)); }
__device__ __forceinline__ double2 adds(double2 a, double2 b) { return addv(a, b); }
__device__ __forceinline__ double2 subs(double2 a, double2 b) { return subv(a, b); }

template <bool PACK, typename V>
__device__ __forceinline__ V vadd(V a, V b) { if constexpr (PACK) return addv(a, b); else return adds(a, b); }
template <bool PACK, typename V>
__device__ __forceinline__ V vsub(V a, V b) { if constexpr (PACK) return subv(a, b); else return subs(a, b); }
template <bool PACK, typename V>
__device__ __forceinline__ V vmul(V b, V w, V wq) { if constexpr (PACK) return cmulv(b, w, wq); else return cmuls(b, w); }

template <typename T>
__device__ __forceinline__ vec2_t<T> wquad(vec2_t<T> w)
{
    vec2_t<T> q;
    q.x = -w.y;
    q.y = w.x;
    return q;
}

// Factor of stage t (= i - gs), index f, of a virtual thread with base
// factor `base` = w_i(cbase) (see dit_stages).
template <typename T, typename TW>
__device__ __forceinline__ vec2_t<T> stage_factor(int t, int f, int i, bool first, typename TW::index_t cbase,
                                                  int gs, const TW &tw, vec2_t<T> base)
{
    using I = typename TW::index_t;
    if (first) return SmallTw<T>::get((1 << (t - 1)) - 1 + f);
    if (FactorTw<T>::value) {
        if (f == 0) return base;
        const vec2_t<T> s = SmallTw<T>::get((1 << (t - 1)) - 1 + f);
        vec2_t<T> w;
        cmul(base.x, base.y, s.x, s.y, w.x, w.y);
        return w;
    }
    return tw.get(i, cbase + ((I)f << gs));
}

// No factor provider (see dit_stages' `fp`).
struct NoFP {
    template <typename V>
    __device__ __forceinline__ void fetch(int, V *) const {}
};

// One stage of dit with the stage index a template constant (radix
// 64, K >= 6: the runtime-indexed loop form does not unroll early enough for
// v[] to stay in registers).
template <typename T, int K, int t, bool TRIV, bool PACK, int HK, typename TW, typename FP>
__device__ __forceinline__ void dit_stage_ct(vec2_t<T> *v, int gs, typename TW::index_t cbase, const TW &tw,
                                              const vec2_t<T> *pre, const vec2_t<T> *hw, const FP *fp)
{
    constexpr bool HAS_FP = !std::is_same<FP, NoFP>::value;
    const bool first = TRIV && gs == 0;

        const int half = (1 << K) >> t;
        const int i = gs + t;
        vec2_t<T> wf[HAS_FP ? (1 << (K - 1)) : 1];
        if constexpr (HAS_FP) {
            if (!first) fp->fetch(t, wf);
        }
        vec2_t<T> base;
        if (!first && FactorTw<T>::value && !HAS_FP) base = pre ? pre[t - 1] : tw.get(i, cbase);
#pragma unroll
        for (int f = 0; f < (1 << (t - 1)); ++f) {
            const int rf = brev(f, t - 1) * 2 * half;
            // 0: stage 1 (no factor), 1: identity, 2: quarter turn, 3: generic
            const int kind = !TRIV ? 3
                           : i == 1 ? 0
                           : (SkipTrivial<T>::value && first && f == 0) ? 1
                           : (SkipTrivial<T>::value && first && (f << 2) == (1 << t)) ? 2 : 3;
            vec2_t<T> w, wq;
            if (kind == 3) {
                if constexpr (HAS_FP) {
                    w = first ? stage_factor<T>(t, f, i, first, cbase, gs, tw, base) : wf[f];
                } else {
                    w = (hw && !first && t <= HK) ? hw[(1 << (t - 1)) - 1 + f]
                                                  : stage_factor<T>(t, f, i, first, cbase, gs, tw, base);
                }
                wq = wquad<T>(w);
            }
#pragma unroll
            for (int r = 0; r < half; ++r) {
                const int p1 = r + rf, p2 = p1 + half;
                vec2_t<T> tt;
                if (kind == 3) {
                    tt = vmul<PACK>(v[p2], w, wq);
                } else if (kind == 2) {
                    tt.x = v[p2].y;
                    tt.y = -v[p2].x;
                } else {
                    tt = v[p2];
                }
                v[p2] = vsub<PACK>(v[p1], tt);
                v[p1] = vadd<PACK>(v[p1], tt);
            }
        }
    }

// One stage of dif with the stage index a template constant (radix
// 64, K >= 6: the runtime-indexed loop form does not unroll early enough for
// v[] to stay in registers).
template <typename T, int K, int t, bool TRIV, bool PACK, int HK, typename TW, typename FP>
__device__ __forceinline__ void dif_stage_ct(vec2_t<T> *v, int gs, typename TW::index_t cbase, const TW &tw,
                                              const vec2_t<T> *pre, const vec2_t<T> *hw, const FP *fp)
{
    constexpr bool HAS_FP = !std::is_same<FP, NoFP>::value;
    const bool first = TRIV && gs == 0;

        const int half = (1 << K) >> t;
        const int i = gs + t;
        vec2_t<T> wf[HAS_FP ? (1 << (K - 1)) : 1];
        if constexpr (HAS_FP) {
            if (!first) fp->fetch(t, wf);
        }
        vec2_t<T> base;
        if (!first && FactorTw<T>::value && !HAS_FP) base = pre ? pre[t - 1] : tw.get(i, cbase);
#pragma unroll
        for (int f = 0; f < (1 << (t - 1)); ++f) {
            const int rf = brev(f, t - 1) * 2 * half;
            const int kind = !TRIV ? 3
                           : i == 1 ? 0
                           : (SkipTrivial<T>::value && first && f == 0) ? 1
                           : (SkipTrivial<T>::value && first && (f << 2) == (1 << t)) ? 2 : 3;
            vec2_t<T> w, wq;
            if (kind == 3) {
                if constexpr (HAS_FP) {
                    w = first ? stage_factor<T>(t, f, i, first, cbase, gs, tw, base) : wf[f];
                } else {
                    w = (hw && !first && t <= HK) ? hw[(1 << (t - 1)) - 1 + f]
                                                  : stage_factor<T>(t, f, i, first, cbase, gs, tw, base);
                }
                wq = wquad<T>(w);
            }
#pragma unroll
            for (int r = 0; r < half; ++r) {
                const int p1 = r + rf, p2 = p1 + half;
                const vec2_t<T> d = vsub<PACK>(v[p1], v[p2]);
                v[p1] = vadd<PACK>(v[p1], v[p2]);
                if (kind == 3) {
                    v[p2] = vmul<PACK>(d, w, wq);
                } else if (kind == 2) {
                    v[p2].x = d.y;
                    v[p2].y = -d.x;
                } else {
                    v[p2] = d;
                }
            }
        }
    }

// K consecutive DIT stages (global stages gs+1 .. gs+K) on the 2^K complex
// values v[0..2^K) (re, im) of one virtual thread.  Register position p
// holds, before stage t, the (size 2^(gs+t-1)) partial transform of
// sub-sequence (p mod 2^K/2^(t-1)) at frequency index
// rev_{t-1}(p / (2^K/2^(t-1))); the stage-(gs+t) factor index is
// q = cbase + (f << gs).  After the K stages register rev_K(f) holds output
// frequency f.  Validated bitwise against the reference by
// tests/test_schedule_model.py (a numpy restatement of this index map).
// TRIV = false promises gs >= 1 and no trivial factors to skip (every pass
// group after the first), which removes the per-stage kind tests.
// `hw` (optional): every factor of the K stages already in registers, stage
// t's 2^(t-1) factors at hw[2^(t-1) - 1 + f] (the persistent kernels load
// them once per thread for all tiles -- the factors depend on the thread's
// column only -- so no table read sits in the tile loop); only stages
// t <= HK come from `hw`, the rest from the table.
// `fp` (optional, replaces hw/table for passes after the first): a factor
// provider whose fetch(t, w) fills w[f], f < 2^(t-1), with stage t's factors
// once per stage before they are used (e.g. factors parked in tensor memory,
// sfft_tma_warp.cuh).
template <typename T, int K, bool TRIV = true, bool PACK = true, int HK = 99, typename TW, typename FP = NoFP>
__device__ __forceinline__ void dit_stages(vec2_t<T> *v, int gs, typename TW::index_t cbase, const TW &tw,
                                           const vec2_t<T> *pre = nullptr, const vec2_t<T> *hw = nullptr,
                                           const FP *fp = nullptr)
{
    constexpr bool HAS_FP = !std::is_same<FP, NoFP>::value;
    const bool first = TRIV && gs == 0;   // first pass: every factor is a compile-time constant
    if constexpr (K >= 6) {
        static_for<1, K + 1>([&](auto TC) {
            dit_stage_ct<T, K, decltype(TC)::value, TRIV, PACK, HK>(v, gs, cbase, tw, pre, hw, fp);
        });
        return;
    }
#pragma unroll
    for (int t = 1; t <= K; ++t) {
        const int half = (1 << K) >> t;
        const int i = gs + t;
        vec2_t<T> wf[HAS_FP ? (1 << (K - 1)) : 1];
        if constexpr (HAS_FP) {
            if (!first) fp->fetch(t, wf);
        }
        vec2_t<T> base;
        if (!first && FactorTw<T>::value && !HAS_FP) base = pre ? pre[t - 1] : tw.get(i, cbase);
#pragma unroll
        for (int f = 0; f < (1 << (t - 1)); ++f) {
            const int rf = brev(f, t - 1) * 2 * half;
            // 0: stage 1 (no factor), 1: identity, 2: quarter turn, 3: generic
            const int kind = !TRIV ? 3
                           : i == 1 ? 0
                           : (SkipTrivial<T>::value && first && f == 0) ? 1
                           : (SkipTrivial<T>::value && first && (f << 2) == (1 << t)) ? 2 : 3;
            vec2_t<T> w, wq;
            if (kind == 3) {
                if constexpr (HAS_FP) {
                    w = first ? stage_factor<T>(t, f, i, first, cbase, gs, tw, base) : wf[f];
                } else {
                    w = (hw && !first && t <= HK) ? hw[(1 << (t - 1)) - 1 + f]
                                                  : stage_factor<T>(t, f, i, first, cbase, gs, tw, base);
                }
                wq = wquad<T>(w);
            }
#pragma unroll
            for (int r = 0; r < half; ++r) {
                const int p1 = r + rf, p2 = p1 + half;
                vec2_t<T> tt;
                if (kind == 3) {
                    tt = vmul<PACK>(v[p2], w, wq);
                } else if (kind == 2) {
                    tt.x = v[p2].y;
                    tt.y = -v[p2].x;
                } else {
                    tt = v[p2];
                }
                v[p2] = vsub<PACK>(v[p1], tt);
                v[p1] = vadd<PACK>(v[p1], tt);
            }
        }
    }
}

// Transpose of dit_stages: DIF stages gs+K .. gs+1 (descending), same
// register map run backwards.
template <typename T, int K, bool TRIV = true, bool PACK = true, int HK = 99, typename TW, typename FP = NoFP>
__device__ __forceinline__ void dif_stages(vec2_t<T> *v, int gs, typename TW::index_t cbase, const TW &tw,
                                           const vec2_t<T> *pre = nullptr, const vec2_t<T> *hw = nullptr,
                                           const FP *fp = nullptr)
{
    constexpr bool HAS_FP = !std::is_same<FP, NoFP>::value;
    const bool first = TRIV && gs == 0;
    if constexpr (K >= 6) {
        static_for<0, K>([&](auto IC) {
            dif_stage_ct<T, K, K - decltype(IC)::value, TRIV, PACK, HK>(v, gs, cbase, tw, pre, hw, fp);
        });
        return;
    }
#pragma unroll
    for (int t = K; t >= 1; --t) {
        const int half = (1 << K) >> t;
        const int i = gs + t;
        vec2_t<T> wf[HAS_FP ? (1 << (K - 1)) : 1];
        if constexpr (HAS_FP) {
            if (!first) fp->fetch(t, wf);
        }
        vec2_t<T> base;
        if (!first && FactorTw<T>::value && !HAS_FP) base = pre ? pre[t - 1] : tw.get(i, cbase);
#pragma unroll
        for (int f = 0; f < (1 << (t - 1)); ++f) {
            const int rf = brev(f, t - 1) * 2 * half;
            const int kind = !TRIV ? 3
                           : i == 1 ? 0
                           : (SkipTrivial<T>::value && first && f == 0) ? 1
                           : (SkipTrivial<T>::value && first && (f << 2) == (1 << t)) ? 2 : 3;
            vec2_t<T> w, wq;
            if (kind == 3) {
                if constexpr (HAS_FP) {
                    w = first ? stage_factor<T>(t, f, i, first, cbase, gs, tw, base) : wf[f];
                } else {
                    w = (hw && !first && t <= HK) ? hw[(1 << (t - 1)) - 1 + f]
                                                  : stage_factor<T>(t, f, i, first, cbase, gs, tw, base);
                }
                wq = wquad<T>(w);
            }
#pragma unroll
            for (int r = 0; r < half; ++r) {
                const int p1 = r + rf, p2 = p1 + half;
                const vec2_t<T> d = vsub<PACK>(v[p1], v[p2]);
                v[p1] = vadd<PACK>(v[p1], v[p2]);
                if (kind == 3) {
                    v[p2] = vmul<PACK>(d, w, wq);
                } else if (kind == 2) {
                    v[p2].x = d.y;
                    v[p2].y = -d.x;
                } else {
                    v[p2] = d;
                }
            }
        }
    }
}

}  // namespace sfft
