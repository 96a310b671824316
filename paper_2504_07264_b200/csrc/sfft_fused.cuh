// sfft_fused.cuh -- one fused kernel per batch tile for N = 2^LOGN <= 4096.
//
// Replaces transform.py:208-270 (fft_dit / fft_dif) batched over rows.
// Each signal is split over P = N / R threads that each hold R = 2^LR complex
// values in registers.  The m radix-2 stages are executed LR at a time
// ("passes"); pass p runs stages p*LR+1 .. p*LR+K_p of the reference's
// factorization in registers (sfft_common.cuh dit_stages/dif_stages) and
// exchanges data between passes through shared memory in Stockham order, so
// the bit-reversal permutation S of the paper costs no pass of its own:
//   DIT pass p (ns = 2^(p*LR), R' = 2^K_p), virtual thread j:
//     reads  in [ j + r * N/R' ]                 r < R'
//     writes out[ (j>>s)*ns*R' + (j&(ns-1)) + ns*f ] = reg[rev(f)]
//   DIF runs the passes in reverse with reads and writes exchanged.
// The first pass reads global memory directly and the last pass writes it
// directly; both patterns are unit-stride across the threads of a signal, so
// every warp-wide access covers whole 32-byte sectors.  Shared-memory
// addresses are padded by one element per R (phys = e + e/R) which makes
// both exchange patterns bank-conflict free for the shipped radix choices.
#pragma once
#include <type_traits>

#include "sfft_common.cuh"

namespace sfft {

// fp32 exchanges as (re, im) pairs (see Exch): one 64-bit shared access per
// complex value.  cfg4 (N = 4096, issue-bound on LSU instructions) +4..8%,
// N = 1024 radix 32 neutral (profiles/r02i_ab_x2.txt); -DSFFT_FUSED_NO_X2
// restores the planar exchange for A/B builds.
#ifdef SFFT_FUSED_NO_X2
template <typename T> struct FusedX2 { static constexpr bool value = false; };
#else
template <typename T> struct FusedX2 { static constexpr bool value = sizeof(T) == 4; };
#endif

struct FusedArgs {
    const void *x0, *x1;   // planar: re, im planes; interleaved: x0 = pairs
    void *y0, *y1;
    const void *tw;        // stage-major factor table, stages 1..LOGN (N-1 entries)
    int64_t batch;
    int64_t in_stride, out_stride;   // elements (planar) or pairs (interleaved)
    int inverse;           // channel-swap inverse (transform.py:286-298)
    double scale;          // 1/N for the inverse, 1 otherwise
};

// Global-memory view of the caller's rows.
// RB: the row is folded into the pointers once (rebase) and per-element
// addresses are base + constant.  Used by DIF, whose first-pass index
// expression made the compiler recompute row * stride + e per element (~7
// instructions per access; N = 4096 DIF 0.78 -> 0.88 of peak); DIT measured
// 4% slower with it and keeps the row term.
template <typename T, bool IL, bool RB = false>
struct GIO;

template <typename T, bool RB>
struct GIO<T, false, RB> {
    const T *xr, *xi;
    T *yr, *yi;
    int64_t is, os;
    bool inv;
    T scale;
    // the inverse's input channel swap is a plane-pointer exchange (no
    // per-element selects); its output swap + 1/N stays a uniform branch
    __device__ __forceinline__ GIO(const FusedArgs &a)
        : xr((const T *)(a.inverse ? a.x1 : a.x0)), xi((const T *)(a.inverse ? a.x0 : a.x1)), yr((T *)a.y0),
          yi((T *)a.y1), is(a.in_stride), os(a.out_stride), inv(a.inverse != 0), scale((T)a.scale) {}
    __device__ __forceinline__ void rebase(int64_t row)
    {
        xr += row * is;
        xi += row * is;
        yr += row * os;
        yi += row * os;
    }
    __device__ __forceinline__ void load(int64_t row, int64_t e, T &re, T &im) const
    {
        const int64_t o = RB ? e : row * is + e;
        re = ld_stream(xr + o);
        im = ld_stream(xi + o);
    }
    __device__ __forceinline__ void store(int64_t row, int64_t e, T re, T im) const
    {
        const int64_t o = RB ? e : row * os + e;
        if (inv) {
            st_stream(yr + o, im * scale);
            st_stream(yi + o, re * scale);
        } else {
            st_stream(yr + o, re);
            st_stream(yi + o, im);
        }
    }
};

template <typename T, bool RB>
struct GIO<T, true, RB> {
    using V = vec2_t<T>;
    const V *x;
    V *y;
    int64_t is, os;
    bool inv;
    T scale;
    __device__ __forceinline__ GIO(const FusedArgs &a)
        : x((const V *)a.x0), y((V *)a.y0), is(a.in_stride), os(a.out_stride),
          inv(a.inverse != 0), scale((T)a.scale) {}
    __device__ __forceinline__ void rebase(int64_t row)
    {
        x += row * is;
        y += row * os;
    }
    __device__ __forceinline__ void load(int64_t row, int64_t e, T &re, T &im) const
    {
        const V v = ld_stream(x + (RB ? e : row * is + e));
        re = inv ? v.y : v.x;
        im = inv ? v.x : v.y;
    }
    __device__ __forceinline__ void store(int64_t row, int64_t e, T re, T im) const
    {
        V v;
        if (inv) {
            v.x = im * scale;
            v.y = re * scale;
        } else {
            v.x = re;
            v.y = im;
        }
        st_stream(y + (RB ? e : row * os + e), v);
    }
};

template <int LOGN, int LR_REQ>
struct FusedShape {
    static constexpr int N = 1 << LOGN;
    static constexpr int LR = LOGN == 0 ? 0 : cmin(LR_REQ, LOGN);
    static constexpr int R = 1 << LR;
    static constexpr int P = N / R;                       // threads per signal
    // threads per block: one signal's P threads, at least 256 (128 for radix
    // 32: 64 register values per thread; gen_inst.py fused_nt mirrors this)
    static constexpr int NTMIN = LR >= 5 ? 128 : 256;
    static constexpr int NT = P > NTMIN ? P : NTMIN;
    static constexpr int S = NT / P;                      // signals per block
#ifdef SFFT_FUSED_MINB
    static constexpr int MINB = SFFT_FUSED_MINB * NT > 2048 ? 2048 / NT : SFFT_FUSED_MINB;
#else
    // radix 32 only (sfft_fused_kernel_r32): <= 168 registers so three
    // 128-thread CTAs fit an SM (the compiler's own choice, 170, rounds to 176
    // and leaves two).  Other shapes carry no min-blocks hint: an explicit 1
    // is not the default (fp64 N = 1024 radix 8: 64 -> 116 registers).
    static constexpr int MINB = 3;
#endif
    static constexpr int NPASS = LOGN == 0 ? 0 : (LOGN + LR - 1) / LR;
    // per-signal stride of the exchange (elements of one plane, or (re, im)
    // pairs when FusedX2: then the 8-byte layouts of the same shape apply)
    template <typename T>
    static constexpr int sstr()
    {
        if constexpr (FusedX2<T>::value) return LOGN == 0 ? 1 : ex_sstr<double, LOGN, LR, NT>();
        else return LOGN == 0 ? 1 : ex_sstr<T, LOGN, LR, NT>();
    }
    template <typename T>
    static constexpr int smem_bytes() { return NPASS >= 2 ? 2 * S * sstr<T>() * (int)sizeof(T) : 0; }
};

// The shared-memory exchange of one signal.  Planar (two T planes, 4-byte
// slots for fp32) or, with FusedX2, (re, im) pairs in one array of 8-byte
// slots: one LDS.64/STS.64 per complex value instead of two 32-bit
// accesses (same bytes, half the LSU instructions), laid out by the planned
// 8-byte layout of the same shape.  ld_r/st_r address slot ex_rd(...),
// ld_w/st_w slot ex_wr(...).
template <typename T, int LOGN, int LR_REQ>
struct Exch {
    using Sh = FusedShape<LOGN, LR_REQ>;
    static constexpr int LR = Sh::LR, NT = Sh::NT;
    static constexpr bool X2 = FusedX2<T>::value;
    using LT = typename std::conditional<X2, double, T>::type;   // layout element size
    using V = vec2_t<T>;
    T *sr = nullptr, *si = nullptr;
    V *sx = nullptr;
    __device__ __forceinline__ V at(int i) const
    {
        if constexpr (X2) {
            return sx[i];
        } else {
            V v;
            v.x = sr[i];
            v.y = si[i];
            return v;
        }
    }
    __device__ __forceinline__ void put(int i, V v) const
    {
        if constexpr (X2) {
            sx[i] = v;
        } else {
            sr[i] = v.x;
            si[i] = v.y;
        }
    }
    __device__ __forceinline__ V ld_r(int x, int e, int et, int ec) const { return at(ex_rd<LT, LOGN, LR, NT>(x, e, et, ec)); }
    __device__ __forceinline__ V ld_w(int x, int e, int et, int ec) const { return at(ex_wr<LT, LOGN, LR, NT>(x, e, et, ec)); }
    __device__ __forceinline__ void st_r(int x, int e, int et, int ec, V v) const { put(ex_rd<LT, LOGN, LR, NT>(x, e, et, ec), v); }
    __device__ __forceinline__ void st_w(int x, int e, int et, int ec, V v) const { put(ex_wr<LT, LOGN, LR, NT>(x, e, et, ec), v); }
};


template <int P>
__device__ __forceinline__ void sig_sync()
{
    if constexpr (P <= 32) __syncwarp(); else __syncthreads();
}

// Partial last exchange.  When the last register pass runs KPL < LR stages
// (RPL = 2^KPL), the exchange before it only permutes values inside groups
// of RPL threads: thread t of group position g = t / (P/RPL) needs, for
// each u < R/RPL, the value of Stockham position f = g + RPL*u from each
// group member -- and the one from itself it already holds.  So each thread
// keeps 1/RPL of its values in registers and moves only the rest through
// shared memory (fp64 N = 1024, radix 8, passes 3+3+3+1: the last exchange
// shrinks by half).  g is warp-uniform when P/RPL >= 32; the code is
// specialised per g (compile-time register indices).
template <int LOGN, int LR_REQ>
struct LastX {
    using Sh = FusedShape<LOGN, LR_REQ>;
    static constexpr int KPL = Sh::NPASS >= 1 ? LOGN - (Sh::NPASS - 1) * Sh::LR : 0;
    static constexpr int RPL = 1 << KPL;
#ifdef SFFT_NO_PARTIAL_EXCHANGE
    static constexpr bool on = false;
#else
    static constexpr bool on = Sh::NPASS >= 2 && KPL < Sh::LR && Sh::P / RPL >= 32;
#endif
    static constexpr int GSTRIDE = Sh::P / RPL;      // threads per group position
};

// ---- DIT pass p -----------------------------------------------------------
template <typename T, int LOGN, int LR_REQ, bool IL, int p>
__device__ __forceinline__ void dit_pass(vec2_t<T> *v, int t, int64_t row, bool valid,
                                         const Exch<T, LOGN, LR_REQ> &xc, const GIO<T, IL, false> &io,
                                         const TwCat<T> &tw, const vec2_t<T> *pre)
{
    using Sh = FusedShape<LOGN, LR_REQ>;
    constexpr int N = Sh::N, R = Sh::R, P = Sh::P, LR = Sh::LR;
    constexpr int SP = p * LR;
    constexpr int KP = cmin(LR, LOGN - SP);
    constexpr int RP = 1 << KP, U = R / RP, NS = 1 << SP;
    const int et = (t >> SP) * NS * RP + (t & (NS - 1));   // this thread's write slot at u = 0, f = 0
    constexpr bool FIRST = p == 0, LAST = p == Sh::NPASS - 1;

    using LX = LastX<LOGN, LR_REQ>;
    // gather this pass's inputs
    if constexpr (LAST && !FIRST && LX::on) {
        // own values: Stockham position f = G + RP*u of the previous pass,
        // held in register brev(f, LR) (copied out before v is overwritten)
        with_g<0, RP>(t / LX::GSTRIDE, [&](auto GC) {
            constexpr int G = decltype(GC)::value;
            vec2_t<T> own[U];
#pragma unroll
            for (int u = 0; u < U; ++u) own[u] = v[brev(G + RP * u, LR)];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int j = t + P * u;
#pragma unroll
                for (int r = 0; r < RP; ++r) {
                    const int e = j + r * (N / RP);
                    if (r == G) {
                        v[u * RP + r] = own[u];
                    } else {
                        v[u * RP + r] = xc.ld_r(p - 1, e, t, P * u + r * (N / RP));
                    }
                }
            }
        });
    } else {
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int j = t + P * u;
#pragma unroll
        for (int r = 0; r < RP; ++r) {
            const int e = j + r * (N / RP);
            if constexpr (FIRST) {
                if (valid) io.load(row, e, v[u * RP + r].x, v[u * RP + r].y);
                else { v[u * RP + r].x = T(0); v[u * RP + r].y = T(0); }
            } else {
                v[u * RP + r] = xc.ld_r(p - 1, e, t, P * u + r * (N / RP));
            }
        }
    }
    }
    // stages SP+1 .. SP+KP
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int j = t + P * u;
        dit_stages<T, KP>(v + u * RP, SP, (j & (NS - 1)), tw,
                          (pre && p > 0) ? pre + p * R + u * KP : nullptr);
    }
    // scatter in Stockham order
    if constexpr (!LAST) {
        if constexpr (!FIRST) sig_sync<P>();
        if constexpr (p == Sh::NPASS - 2 && LX::on) {
            // partial last exchange: positions f = G (mod RPL) stay in registers
            static_assert(U == 1, "the pass before the last runs the full radix");
            with_g<0, LX::RPL>(t / LX::GSTRIDE, [&](auto GC) {
                constexpr int G = decltype(GC)::value;
                const int base = (t >> SP) * NS * RP + (t & (NS - 1));
#pragma unroll
                for (int f = 0; f < RP; ++f) {
                    if (f % LX::RPL == G) continue;
                    const int e = base + NS * f;
                    xc.st_w(p, e, et, NS * f, v[brev(f, KP)]);
                }
            });
        } else {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int j = t + P * u;
            const int base = (j >> SP) * NS * RP + (j & (NS - 1));
#pragma unroll
            for (int f = 0; f < RP; ++f) {
                const int e = base + NS * f;
                xc.st_w(p, e, et, ((P * u) >> SP) * NS * RP + ((P * u) & (NS - 1)) + NS * f, v[u * RP + brev(f, KP)]);
            }
        }
        }
        sig_sync<P>();
    } else {
        if (valid) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int j = t + P * u;     // NS*RP == N here, so (j >> SP) == 0
#pragma unroll
                for (int f = 0; f < RP; ++f)
                    io.store(row, j + NS * f, v[u * RP + brev(f, KP)].x, v[u * RP + brev(f, KP)].y);
            }
        }
    }
}

template <typename T, int LOGN, int LR_REQ, bool IL, int p>
__device__ __forceinline__ void dit_from(vec2_t<T> *v, int t, int64_t row, bool valid,
                                         const Exch<T, LOGN, LR_REQ> &xc, const GIO<T, IL, false> &io, const TwCat<T> &tw,
                                         const vec2_t<T> *pre)
{
    if constexpr (p < FusedShape<LOGN, LR_REQ>::NPASS) {
        dit_pass<T, LOGN, LR_REQ, IL, p>(v, t, row, valid, xc, io, tw, pre);
        dit_from<T, LOGN, LR_REQ, IL, p + 1>(v, t, row, valid, xc, io, tw, pre);
    }
}

// ---- DIF pass p (executed for p = NPASS-1 .. 0) --------------------------
template <typename T, int LOGN, int LR_REQ, bool IL, int p>
__device__ __forceinline__ void dif_pass(vec2_t<T> *v, int t, int64_t row, bool valid,
                                         const Exch<T, LOGN, LR_REQ> &xc, const GIO<T, IL, true> &io,
                                         const TwCat<T> &tw, const vec2_t<T> *pre)
{
    using Sh = FusedShape<LOGN, LR_REQ>;
    constexpr int N = Sh::N, R = Sh::R, P = Sh::P, LR = Sh::LR;
    constexpr int SP = p * LR;
    constexpr int KP = cmin(LR, LOGN - SP);
    constexpr int RP = 1 << KP, U = R / RP, NS = 1 << SP;
    const int et = (t >> SP) * NS * RP + (t & (NS - 1));   // this thread's write slot at u = 0, f = 0
    constexpr bool FIRST = p == Sh::NPASS - 1, LAST = p == 0;
    using LX = LastX<LOGN, LR_REQ>;

    if constexpr (p == Sh::NPASS - 2 && LX::on) {
        // partial exchange (transpose of the DIT one): position f = G + RPL*u'
        // is this thread's own register u'*RPL + G of the previous pass
        static_assert(U == 1, "the pass after the first runs the full radix");
        with_g<0, LX::RPL>(t / LX::GSTRIDE, [&](auto GC) {
            constexpr int G = decltype(GC)::value;
            constexpr int UL = R / LX::RPL;
            vec2_t<T> own[UL];
#pragma unroll
            for (int u = 0; u < UL; ++u) own[u] = v[u * LX::RPL + G];
            const int base = (t >> SP) * NS * RP + (t & (NS - 1));
#pragma unroll
            for (int f = 0; f < RP; ++f) {
                const int e = base + NS * f;
                const int d = brev(f, KP);
                if (f % LX::RPL == G) {
                    v[d] = own[f / LX::RPL];
                } else {
                    v[d] = xc.ld_w(p, e, et, NS * f);
                }
            }
        });
    } else {
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int j = t + P * u;
        const int base = (j >> SP) * NS * RP + (j & (NS - 1));
#pragma unroll
        for (int f = 0; f < RP; ++f) {
            const int e = base + NS * f;
            const int d = u * RP + brev(f, KP);
            if constexpr (FIRST) {
                if (valid) io.load(row, e, v[d].x, v[d].y);
                else { v[d].x = T(0); v[d].y = T(0); }
            } else {
                v[d] = xc.ld_w(p, e, et, ((P * u) >> SP) * NS * RP + ((P * u) & (NS - 1)) + NS * f);
            }
        }
    }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int j = t + P * u;
        dif_stages<T, KP>(v + u * RP, SP, (j & (NS - 1)), tw,
                          (pre && p > 0) ? pre + p * R + u * KP : nullptr);
    }
    if constexpr (!LAST) {
        if constexpr (!FIRST) sig_sync<P>();
        if constexpr (FIRST && LX::on) {
            // partial exchange: r == G stays in registers for the next pass
            with_g<0, RP>(t / LX::GSTRIDE, [&](auto GC) {
                constexpr int G = decltype(GC)::value;
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int j = t + P * u;
#pragma unroll
                    for (int r = 0; r < RP; ++r) {
                        if (r == G) continue;
                        const int e = j + r * (N / RP);
                        xc.st_r(p - 1, e, t, P * u + r * (N / RP), v[u * RP + r]);
                    }
                }
            });
        } else {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int j = t + P * u;
#pragma unroll
            for (int r = 0; r < RP; ++r) {
                const int e = j + r * (N / RP);
                xc.st_r(p - 1, e, t, P * u + r * (N / RP), v[u * RP + r]);
            }
        }
        }
        sig_sync<P>();
    } else {
        if (valid) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int j = t + P * u;
#pragma unroll
                for (int r = 0; r < RP; ++r)
                    io.store(row, j + r * (N / RP), v[u * RP + r].x, v[u * RP + r].y);
            }
        }
    }
}

template <typename T, int LOGN, int LR_REQ, bool IL, int p>
__device__ __forceinline__ void dif_from(vec2_t<T> *v, int t, int64_t row, bool valid,
                                         const Exch<T, LOGN, LR_REQ> &xc, const GIO<T, IL, true> &io, const TwCat<T> &tw,
                                         const vec2_t<T> *pre)
{
    if constexpr (p >= 0) {
        dif_pass<T, LOGN, LR_REQ, IL, p>(v, t, row, valid, xc, io, tw, pre);
        dif_from<T, LOGN, LR_REQ, IL, p - 1>(v, t, row, valid, xc, io, tw, pre);
    }
}

// PRE (fp32 only): fetch the base factors of passes >= 1 before the data.
// Whether that pays depends on the size (register pressure vs latency);
// tools/tune.py measures both and gen_inst.py's AUTO table records the pick.
template <typename T, int LOGN, int LR_REQ, bool DIF, bool IL, bool PRE>
__device__ __forceinline__ void fused_body(const FusedArgs &a)
{
    using Sh = FusedShape<LOGN, LR_REQ>;
    constexpr int R = Sh::R, P = Sh::P, S = Sh::S, SSTR = Sh::template sstr<T>();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T *sbase = reinterpret_cast<T *>(smem_raw);

    const int tid = threadIdx.x;
    const int sl = tid / P, t = tid % P;
    const int64_t row = (int64_t)blockIdx.x * S + sl;
    const bool valid = row < a.batch;
    GIO<T, IL, DIF> io(a);
    if constexpr (DIF) io.rebase(row);
    const TwCat<T> tw{reinterpret_cast<const vec2_t<T> *>(a.tw)};

    if constexpr (LOGN == 0) {
        if (valid) {
            T re, im;
            io.load(row, 0, re, im);
            io.store(row, 0, re, im);
        }
    } else {
        vec2_t<T> v[R];
        Exch<T, LOGN, LR_REQ> xc;
        if constexpr (FusedX2<T>::value) {
            xc.sx = reinterpret_cast<vec2_t<T> *>(smem_raw) + sl * SSTR;
        } else {
            xc.sr = sbase + sl * SSTR;
            xc.si = sbase + S * SSTR + sl * SSTR;
        }
        // fp32: the base factors of passes >= 1, fetched before any data
        vec2_t<T> pre[Sh::NPASS * R];
        if constexpr (PRE && FactorTw<T>::value) {
#pragma unroll
            for (int p = 1; p < Sh::NPASS; ++p) {
                const int sp = p * Sh::LR;
                const int kp = cmin(Sh::LR, LOGN - sp);
#pragma unroll
                for (int u = 0; u < R / (1 << kp); ++u) {
                    const int j = t + P * u;
#pragma unroll
                    for (int tt = 1; tt <= kp; ++tt)
                        pre[p * R + u * kp + tt - 1] = tw.get(sp + tt, j & ((1 << sp) - 1));
                }
            }
        }
        if constexpr (DIF)
            dif_from<T, LOGN, LR_REQ, IL, Sh::NPASS - 1>(v, t, row, valid, xc, io, tw,
                                                         (PRE && FactorTw<T>::value) ? pre : nullptr);
        else
            dit_from<T, LOGN, LR_REQ, IL, 0>(v, t, row, valid, xc, io, tw,
                                             (PRE && FactorTw<T>::value) ? pre : nullptr);
    }
}

#ifdef SFFT_FUSED_MINB
template <typename T, int LOGN, int LR_REQ, bool DIF, bool IL, bool PRE = false>
__global__ void __launch_bounds__(FusedShape<LOGN, LR_REQ>::NT, FusedShape<LOGN, LR_REQ>::MINB)
sfft_fused_kernel(const FusedArgs a)
{
    fused_body<T, LOGN, LR_REQ, DIF, IL, PRE>(a);
}
#else
template <typename T, int LOGN, int LR_REQ, bool DIF, bool IL, bool PRE = false>
__global__ void __launch_bounds__(FusedShape<LOGN, LR_REQ>::NT)
sfft_fused_kernel(const FusedArgs a)
{
    fused_body<T, LOGN, LR_REQ, DIF, IL, PRE>(a);
}
#endif

template <typename T, int LOGN, int LR_REQ, bool DIF, bool IL, bool PRE = false>
__global__ void __launch_bounds__(FusedShape<LOGN, LR_REQ>::NT, FusedShape<LOGN, LR_REQ>::MINB)
sfft_fused_kernel_r32(const FusedArgs a)
{
    fused_body<T, LOGN, LR_REQ, DIF, IL, PRE>(a);
}

// the kernel a shape launches: radix 32 takes the register-capped variant
template <typename T, int LOGN, int LR_REQ, bool DIF, bool IL, bool PRE>
constexpr auto fused_kernel_for()
{
    if constexpr (FusedShape<LOGN, LR_REQ>::LR >= 5) return &sfft_fused_kernel_r32<T, LOGN, LR_REQ, DIF, IL, PRE>;
    else return &sfft_fused_kernel<T, LOGN, LR_REQ, DIF, IL, PRE>;
}

}  // namespace sfft
