// sfft_tma.cuh -- persistent TMA-fed fused kernel for planar rows, N <= 4096.
//
// Same arithmetic and Stockham register passes as sfft_fused.cuh (the
// reference's radix-2 stages, transform.py:208-270), but the global side is
// moved by the Tensor Memory Accelerator instead of per-thread LDG/STG:
//   * a tile = S consecutive signals of one plane is a 3-D TMA box
//     (W elements per 128-byte line, N/W lines per signal, S signals) landing
//     in shared memory with the 128-byte swizzle (16-byte chunk index XOR
//     line index mod 8), STAGES tiles in flight per CTA (mbarrier
//     complete_tx), so HBM reads never occupy the LSU/L1 wavefront pipe;
//   * the first register pass reads the swizzled tile, intermediate passes
//     exchange through a padded buffer (phys = e + e/R), the last pass writes
//     a swizzled output tile that one thread stores with a TMA bulk tensor
//     store (bulk_group, double-buffered);
//   * CTAs are persistent (grid = resident CTAs, tiles round-robin).
// Rows beyond the batch are zero-filled by the TMA load and clipped by the
// TMA store, so the tail tile needs no predication.
#pragma once
#include <cuda.h>

#include "sfft_common.cuh"

namespace sfft {

// Measured back to back on cfg2 (tools/ab_launch2.sh): this kernel runs
// 172 us per 1 GiB step with scalar fp32 math and generic-pointer shared
// accesses, 190 us with packed FFMA2/FADD2 and 196 us with LDS/STS -- the
// persistent pipeline is latency- not issue-bound -- so both stay off here
// (the LDG fused and pass kernels, which are issue-bound, use packed math).
#ifdef SFFT_TMA_PACK
constexpr bool TMA_PACK = true;
#else
constexpr bool TMA_PACK = false;
#endif

struct TmaArgs {
    int64_t ntiles;
    double scale;        // 1/N when the caller swapped the maps for the inverse
    int scale_out;
    const void *tw;
    // OB == 0 (direct stores from the last register pass): output planes
    // (already channel-swapped for the inverse), rows, row stride (elements)
    void *y_re, *y_im;
    int64_t batch, out_stride;
};

__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_LOOP:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@P1 bra WAIT_DONE;\n"
        "bra WAIT_LOOP;\n"
        "WAIT_DONE:\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1, int c2)
{
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::
            "r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}

__device__ __forceinline__ void tma_store_3d(const CUtensorMap *map, const void *src, int c0, int c1, int c2)
{
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
                 : "memory");
}

__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }

template <int N>
__device__ __forceinline__ void bulk_wait_read()
{
    if constexpr (N >= 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

// Shape of the TMA kernel.  NT_REQ: requested threads per CTA (>= P).
// OB = 0: the last register pass stores straight to global memory (no output
// tile, no TMA store) -- frees OB*2*TILE bytes of shared memory per CTA.
template <typename T, int LOGN, int LR_REQ, int NT_REQ, int STAGES, int OB>
struct TmaShape {
    static constexpr int N = 1 << LOGN;
    static constexpr int LR = cmin(LR_REQ, LOGN);
    static constexpr int R = 1 << LR;
    static constexpr int P = N / R;
    static constexpr int NT = P > NT_REQ ? P : NT_REQ;
    static constexpr int S = NT / P;                          // signals per tile
    static constexpr int NPASS = (LOGN + LR - 1) / LR;
    static constexpr int W = 128 / (int)sizeof(T);            // elements per 128-byte line
    static constexpr int TILE = S * N * (int)sizeof(T);       // bytes per plane per tile
    static constexpr int SSTR = ex_sstr<T, LOGN, LR, NT>();   // planned exchange stride
    static constexpr int EXB = NPASS >= 2 ? 2 * S * SSTR * (int)sizeof(T) : 0;
    static constexpr int IN_OFF = 0;
    static constexpr int OUT_OFF = IN_OFF + STAGES * 2 * TILE;
    static constexpr int EX_OFF = OUT_OFF + OB * 2 * TILE;
    static constexpr int BAR_OFF = (EX_OFF + EXB + 15) / 16 * 16;
    static constexpr int SMEM = BAR_OFF + STAGES * 8 + 1024;   // + alignment slack
    static_assert(N >= W, "TMA path needs rows of at least one 128-byte line");
    static_assert(N / W <= 256 && S <= 256, "TMA box dims are limited to 256");
    static_assert(TILE % 1024 == 0, "swizzled tiles must stay 1024-byte aligned");
};

// byte offset of logical element e of local signal s inside a swizzled tile
template <typename T, int N>
__device__ __forceinline__ uint32_t swz(int s, int e)
{
    const uint32_t L = (uint32_t)(s * N + e) * (uint32_t)sizeof(T);
    return L ^ ((L >> 3) & 0x70u);
}

template <typename T>
__device__ __forceinline__ T lds_at(const unsigned char *base, uint32_t off)
{
    return *reinterpret_cast<const T *>(base + off);
}

template <typename T>
__device__ __forceinline__ void sts_at(unsigned char *base, uint32_t off, T v)
{
    *reinterpret_cast<T *>(base + off) = v;
}

template <typename T, int LOGN, int LR_REQ, bool DIF, int NT_REQ, int STAGES, int OB, bool PRE_T>
__device__ __forceinline__ void tma_body(const CUtensorMap &in_re, const CUtensorMap &in_im,
                                         const CUtensorMap &out_re, const CUtensorMap &out_im, const TmaArgs &a)
{
    using Sh = TmaShape<T, LOGN, LR_REQ, NT_REQ, STAGES, OB>;
    constexpr int N = Sh::N, R = Sh::R, P = Sh::P, S = Sh::S, LR = Sh::LR, NPASS = Sh::NPASS,
                  TILE = Sh::TILE, SSTR = Sh::SSTR, W = Sh::W;
    extern __shared__ unsigned char smem_raw[];
    // 1024-byte alignment for the 128B swizzle.  fp32 addresses shared
    // memory through generic pointers (measured faster on cfg2, see TMA_PACK);
    // fp64 keeps the shared window (LDS/STS: 0.864 -> 0.880 of the HBM peak on
    // cfg3 fp64, profiles/r02a_ab_f64_tma.txt)
#ifdef SFFT_TMA_LDS
    constexpr bool kShWindow = true;
#else
    constexpr bool kShWindow = sizeof(T) == 8;
#endif
    unsigned char *smem = kShWindow
        ? smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u)
        : reinterpret_cast<unsigned char *>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    unsigned char *in_buf = smem + Sh::IN_OFF;      // [STAGES][2 planes][TILE]
    unsigned char *out_buf = smem + Sh::OUT_OFF;    // [OB][2][TILE]
    T *ex = reinterpret_cast<T *>(smem + Sh::EX_OFF);
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + Sh::BAR_OFF);

    const int tid = threadIdx.x;
    const int sl = tid / P, t = tid % P;
    const int64_t nk = a.ntiles > blockIdx.x ? (a.ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const TwCat<T> tw{reinterpret_cast<const vec2_t<T> *>(a.tw)};
    const T scale = (T)a.scale;
    const bool do_scale = a.scale_out != 0;

    auto issue_load = [&](int st, int64_t tile) {
        uint64_t *bar = full + st;
        mbar_expect_tx(bar, 2 * TILE);
        const int row0 = (int)(tile * S);
        tma_load_3d(in_buf + (st * 2 + 0) * TILE, &in_re, bar, 0, 0, row0);
        tma_load_3d(in_buf + (st * 2 + 1) * TILE, &in_im, bar, 0, 0, row0);
    };

    if (tid == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&in_re)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&in_im)) : "memory");
        for (int s = 0; s < STAGES; ++s) mbar_init(full + s, 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (tid == 0) {
#ifndef SFFT_TMA_NO_PDL
        // dependent launch (sfft_tma_host.h): wait for the previous grid of
        // the stream (and its memory) before touching the signal planes --
        // every global data access of this kernel is a TMA issued by this
        // thread after this point; then let the next grid be scheduled
        asm volatile("griddepcontrol.wait;" ::: "memory");
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
        for (int s = 0; s < STAGES && s < nk; ++s) issue_load(s, blockIdx.x + (int64_t)s * gridDim.x);
    }

    vec2_t<T> v[R];
    // fp32: base factors of passes >= 1 depend only on the thread, not on
    // the tile -- fetch them once for the whole persistent loop
    constexpr bool PRE = PRE_T && FactorTw<T>::value;
    vec2_t<T> pre[NPASS][R];
    if constexpr (PRE) {
#pragma unroll
        for (int p = 1; p < NPASS; ++p) {
            const int sp = p * LR;
            const int kp = cmin(LR, LOGN - sp);
#pragma unroll
            for (int u = 0; u < R / (1 << kp); ++u) {
                const int j = t + P * u;
#pragma unroll
                for (int tt = 1; tt <= kp; ++tt) pre[p][u * kp + tt - 1] = tw.get(sp + tt, j & ((1 << sp) - 1));
            }
        }
    }
    // fp64 (table factors, bit-exact contract): every factor of passes >= 1
    // depends on the thread's column only, so the whole per-thread set is
    // loaded once here and lives in registers for all tiles (fp64 N = 1024
    // radix 8: 18 complex factors) -- the tile loop issues no table reads,
    // which took ~40% of the L1 wavefronts of the per-use loads.  Virtual
    // threads u > 0 whose column equals u = 0's share its slots.
    constexpr bool HOIST = !FactorTw<T>::value && NPASS >= 2;
    vec2_t<T> hw[NPASS][R];
    if constexpr (HOIST) {
#pragma unroll
        for (int p = 1; p < NPASS; ++p) {
            const int sp = p * LR;
            const int kp = cmin(LR, LOGN - sp);
            const int rp = 1 << kp, ns = 1 << sp;
#pragma unroll
            for (int u = 0; u < R / rp; ++u) {
                if (u > 0 && ((P * u) & (ns - 1)) == 0) continue;
                const int j = t + P * u;
#pragma unroll
                for (int tt = 1; tt <= kp; ++tt)
#pragma unroll
                    for (int f = 0; f < (1 << (tt - 1)); ++f)
                        hw[p][u * (rp - 1) + (1 << (tt - 1)) - 1 + f] = tw.get(sp + tt, (j & (ns - 1)) + (f << sp));
            }
        }
    }
    T *exr = ex + sl * SSTR;
    T *exi = ex + S * SSTR + sl * SSTR;
    T *ygr = reinterpret_cast<T *>(a.y_re);
    T *ygi = reinterpret_cast<T *>(a.y_im);

    // Partial last exchange (as sfft_fused.cuh LastX): when the last DIT
    // pass runs KPL < LR stages, the exchange before it only permutes values
    // inside groups of RPL threads, so 1/RPL of each thread's values stay in
    // registers (fp64 N = 1024 radix 8, passes 3+3+3+1: half of that
    // exchange).  g = t / GSTRIDE is warp-uniform (GSTRIDE >= 32).
    constexpr int KPL = LOGN - (NPASS - 1) * LR;
    constexpr int RPL = 1 << KPL;
#ifdef SFFT_NO_PARTIAL_EXCHANGE
    constexpr bool PX = false;
#else
    constexpr bool PX = NPASS >= 2 && KPL < LR && P / RPL >= 32;
#endif
    constexpr int GSTRIDE = P / RPL;
    const int g = t / GSTRIDE;

    for (int64_t k = 0; k < nk; ++k) {
        const int st = (int)(k % STAGES);
        const int ob = OB > 0 ? (int)(k % OB) : 0;
        const int64_t tile = blockIdx.x + k * gridDim.x;
        const unsigned char *inr = in_buf + (st * 2 + 0) * TILE;
        const unsigned char *ini = in_buf + (st * 2 + 1) * TILE;
        unsigned char *outr = out_buf + (ob * 2 + 0) * TILE;
        unsigned char *outi = out_buf + (ob * 2 + 1) * TILE;
        const int64_t orow = tile * S + sl;   // OB == 0: this thread's output row
        mbar_wait(full + st, (uint32_t)((k / STAGES) & 1));

        // input slot consumed (and, OB > 0, output buffer `ob` free): refill
        auto release_input = [&]() {
            if (tid == 0) bulk_wait_read<OB - 1>();
            __syncthreads();
            if (tid == 0 && k + STAGES < nk) issue_load(st, tile + (int64_t)STAGES * gridDim.x);
        };
        auto put = [&](int e, T re, T im) {
            if (do_scale) {
                re *= scale;
                im *= scale;
            }
            if constexpr (OB == 0) {
                if (orow < a.batch) {
                    st_stream(ygr + orow * a.out_stride + e, re);
                    st_stream(ygi + orow * a.out_stride + e, im);
                }
            } else {
                sts_at<T>(outr, swz<T, N>(sl, e), re);
                sts_at<T>(outi, swz<T, N>(sl, e), im);
            }
        };
        // hoisted-factor slot of virtual thread u in pass p (u > 0 with u = 0's column shares it)
        auto hwp = [&](int p, int u, int rp) -> const vec2_t<T> * {
            const int ns = 1 << (p * LR);
            return &hw[p][((u > 0 && ((P * u) & (ns - 1)) == 0) ? 0 : u) * (rp - 1)];
        };

        if constexpr (!DIF) {
            // ---------------- DIT: passes 0 .. NPASS-1 ----------------
            static_for<0, NPASS>([&](auto PC) {
                constexpr int p = decltype(PC)::value;
                constexpr int sp = p * LR, KP = cmin(LR, LOGN - sp), RP = 1 << KP, U = R / RP, ns = 1 << sp;
                constexpr bool FIRST = p == 0, LAST = p == NPASS - 1;
                const int et = (t >> sp) * ns * RP + (t & (ns - 1));
                // gather
                if constexpr (FIRST) {
#pragma unroll
                    for (int u = 0; u < U; ++u)
#pragma unroll
                        for (int r = 0; r < RP; ++r) {
                            const int e = t + P * u + r * (N / RP);
                            v[u * RP + r].x = lds_at<T>(inr, swz<T, N>(sl, e));
                            v[u * RP + r].y = lds_at<T>(ini, swz<T, N>(sl, e));
                        }
                } else if constexpr (LAST && PX) {
                    with_g<0, RP>(g, [&](auto GC) {
                        constexpr int G = decltype(GC)::value;
                        vec2_t<T> own[U];
#pragma unroll
                        for (int u = 0; u < U; ++u) own[u] = v[brev(G + RP * u, LR)];
#pragma unroll
                        for (int u = 0; u < U; ++u)
#pragma unroll
                            for (int r = 0; r < RP; ++r) {
                                const int e = t + P * u + r * (N / RP);
                                if (r == G) {
                                    v[u * RP + r] = own[u];
                                } else {
                                    const int x = ex_rd<T, LOGN, LR, Sh::NT>(p - 1, e, t, P * u + r * (N / RP));
                                    v[u * RP + r].x = exr[x];
                                    v[u * RP + r].y = exi[x];
                                }
                            }
                    });
                } else {
#pragma unroll
                    for (int u = 0; u < U; ++u)
#pragma unroll
                        for (int r = 0; r < RP; ++r) {
                            const int e = t + P * u + r * (N / RP);
                            const int x = ex_rd<T, LOGN, LR, Sh::NT>(p - 1, e, t, P * u + r * (N / RP));
                            v[u * RP + r].x = exr[x];
                            v[u * RP + r].y = exi[x];
                        }
                }
                // stages sp+1 .. sp+KP
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int j = t + P * u;
                    dit_stages<T, KP, true, TMA_PACK>(v + u * RP, sp, (j & (ns - 1)), tw,
                                                      (PRE && p > 0) ? &pre[p][u * KP] : nullptr,
                                                      (HOIST && p > 0) ? hwp(p, u, RP) : nullptr);
                }
                if constexpr (!LAST) {
                    // Stockham scatter
                    if constexpr (!FIRST) __syncthreads();
                    if constexpr (p == NPASS - 2 && PX) {
                        static_assert(U == 1, "the pass before the last runs the full radix");
                        with_g<0, RPL>(g, [&](auto GC) {
                            constexpr int G = decltype(GC)::value;
#pragma unroll
                            for (int f = 0; f < RP; ++f) {
                                if (f % RPL == G) continue;      // stays in registers
                                const int x = ex_wr<T, LOGN, LR, Sh::NT>(p, et + ns * f, et, ns * f);
                                exr[x] = v[brev(f, KP)].x;
                                exi[x] = v[brev(f, KP)].y;
                            }
                        });
                    } else {
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            const int j = t + P * u;
                            const int base = (j >> sp) * ns * RP + (j & (ns - 1));
#pragma unroll
                            for (int f = 0; f < RP; ++f) {
                                const int x = ex_wr<T, LOGN, LR, Sh::NT>(
                                    p, base + ns * f, et, ((P * u) >> sp) * ns * RP + ((P * u) & (ns - 1)) + ns * f);
                                exr[x] = v[u * RP + brev(f, KP)].x;
                                exi[x] = v[u * RP + brev(f, KP)].y;
                            }
                        }
                    }
                    if constexpr (FIRST) release_input();
                    else __syncthreads();
                } else {
                    if constexpr (NPASS == 1) release_input();
#pragma unroll
                    for (int u = 0; u < U; ++u)
#pragma unroll
                        for (int f = 0; f < RP; ++f)
                            put(t + P * u + ns * f, v[u * RP + brev(f, KP)].x, v[u * RP + brev(f, KP)].y);
                }
            });
        } else {
            // ---------------- DIF (transpose): passes NPASS-1 .. 0 ----------------
            static_for<0, NPASS>([&](auto QC) {
                constexpr int q = decltype(QC)::value;
                constexpr int p = NPASS - 1 - q;
                constexpr int sp = p * LR, KP = cmin(LR, LOGN - sp), RP = 1 << KP, U = R / RP, ns = 1 << sp;
                constexpr bool FIRST = q == 0, LAST = p == 0;
                const int et = (t >> sp) * ns * RP + (t & (ns - 1));
                // gather
                if constexpr (FIRST) {
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int j = t + P * u;
                        const int base = (j >> sp) * ns * RP + (j & (ns - 1));
#pragma unroll
                        for (int f = 0; f < RP; ++f) {
                            const int e = base + ns * f;
                            const int d = u * RP + brev(f, KP);
                            v[d].x = lds_at<T>(inr, swz<T, N>(sl, e));
                            v[d].y = lds_at<T>(ini, swz<T, N>(sl, e));
                        }
                    }
                } else if constexpr (p == NPASS - 2 && PX) {
                    static_assert(U == 1, "the pass after the first runs the full radix");
                    with_g<0, RPL>(g, [&](auto GC) {
                        constexpr int G = decltype(GC)::value;
                        constexpr int UL = R / RPL;
                        vec2_t<T> own[UL];
#pragma unroll
                        for (int u = 0; u < UL; ++u) own[u] = v[u * RPL + G];
#pragma unroll
                        for (int f = 0; f < RP; ++f) {
                            const int d = brev(f, KP);
                            if (f % RPL == G) {
                                v[d] = own[f / RPL];
                            } else {
                                const int x = ex_wr<T, LOGN, LR, Sh::NT>(p, et + ns * f, et, ns * f);
                                v[d].x = exr[x];
                                v[d].y = exi[x];
                            }
                        }
                    });
                } else {
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int j = t + P * u;
                        const int base = (j >> sp) * ns * RP + (j & (ns - 1));
#pragma unroll
                        for (int f = 0; f < RP; ++f) {
                            const int d = u * RP + brev(f, KP);
                            const int x = ex_wr<T, LOGN, LR, Sh::NT>(
                                p, base + ns * f, et, ((P * u) >> sp) * ns * RP + ((P * u) & (ns - 1)) + ns * f);
                            v[d].x = exr[x];
                            v[d].y = exi[x];
                        }
                    }
                }
                // stages sp+KP .. sp+1
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int j = t + P * u;
                    dif_stages<T, KP, true, TMA_PACK>(v + u * RP, sp, (j & (ns - 1)), tw,
                                                      (PRE && p > 0) ? &pre[p][u * KP] : nullptr,
                                                      (HOIST && p > 0) ? hwp(p, u, RP) : nullptr);
                }
                if constexpr (!LAST) {
                    if constexpr (!FIRST) __syncthreads();
                    if constexpr (FIRST && PX) {
                        with_g<0, RP>(g, [&](auto GC) {
                            constexpr int G = decltype(GC)::value;
#pragma unroll
                            for (int u = 0; u < U; ++u)
#pragma unroll
                                for (int r = 0; r < RP; ++r) {
                                    if (r == G) continue;        // stays in registers
                                    const int e = t + P * u + r * (N / RP);
                                    const int x = ex_rd<T, LOGN, LR, Sh::NT>(p - 1, e, t, P * u + r * (N / RP));
                                    exr[x] = v[u * RP + r].x;
                                    exi[x] = v[u * RP + r].y;
                                }
                        });
                    } else {
#pragma unroll
                        for (int u = 0; u < U; ++u)
#pragma unroll
                            for (int r = 0; r < RP; ++r) {
                                const int e = t + P * u + r * (N / RP);
                                const int x = ex_rd<T, LOGN, LR, Sh::NT>(p - 1, e, t, P * u + r * (N / RP));
                                exr[x] = v[u * RP + r].x;
                                exi[x] = v[u * RP + r].y;
                            }
                    }
                    if constexpr (FIRST) release_input();
                    else __syncthreads();
                } else {
                    if constexpr (NPASS == 1) release_input();
#pragma unroll
                    for (int u = 0; u < U; ++u)
#pragma unroll
                        for (int r = 0; r < RP; ++r)
                            put(t + P * u + r * (N / RP), v[u * RP + r].x, v[u * RP + r].y);
                }
            });
        }
        if constexpr (OB == 0) {
            // the next tile's first scatter reuses the exchange buffer
            if constexpr (NPASS >= 2) __syncthreads();
        } else {
            // output tile complete in shared memory -> one TMA store per plane
            fence_async_smem();
            __syncthreads();
            if (tid == 0) {
                const int row0 = (int)(tile * S);
                tma_store_3d(&out_re, outr, 0, 0, row0);
                tma_store_3d(&out_im, outi, 0, 0, row0);
                bulk_commit();
            }
        }
    }
    if (OB > 0 && tid == 0) bulk_wait_all();
    (void)W;
}

// MINB = 0: no min-blocks hint (an explicit 1 is not the default: the cfg2
// shape went from 48 to 71 registers with it); MINB > 0 caps the registers
// so MINB CTAs fit an SM (fp64 N = 1024: 4 x 128 threads at <= 128).
template <typename T, int LOGN, int LR_REQ, bool DIF, int NT_REQ, int STAGES, int OB, bool PRE_T = false,
          int MINB = 0>
__global__ void __launch_bounds__(TmaShape<T, LOGN, LR_REQ, NT_REQ, STAGES, OB>::NT)
sfft_tma_kernel(const __grid_constant__ CUtensorMap in_re, const __grid_constant__ CUtensorMap in_im,
                const __grid_constant__ CUtensorMap out_re, const __grid_constant__ CUtensorMap out_im,
                const TmaArgs a)
{
    tma_body<T, LOGN, LR_REQ, DIF, NT_REQ, STAGES, OB, PRE_T>(in_re, in_im, out_re, out_im, a);
}

template <typename T, int LOGN, int LR_REQ, bool DIF, int NT_REQ, int STAGES, int OB, bool PRE_T, int MINB>
__global__ void __launch_bounds__(TmaShape<T, LOGN, LR_REQ, NT_REQ, STAGES, OB>::NT, MINB)
sfft_tma_kernel_mb(const __grid_constant__ CUtensorMap in_re, const __grid_constant__ CUtensorMap in_im,
                   const __grid_constant__ CUtensorMap out_re, const __grid_constant__ CUtensorMap out_im,
                   const TmaArgs a)
{
    tma_body<T, LOGN, LR_REQ, DIF, NT_REQ, STAGES, OB, PRE_T>(in_re, in_im, out_re, out_im, a);
}

template <typename T, int LOGN, int LR_REQ, bool DIF, int NT_REQ, int STAGES, int OB, bool PRE_T, int MINB>
constexpr auto tma_kernel_for()
{
    if constexpr (MINB > 0) return &sfft_tma_kernel_mb<T, LOGN, LR_REQ, DIF, NT_REQ, STAGES, OB, PRE_T, MINB>;
    else return &sfft_tma_kernel<T, LOGN, LR_REQ, DIF, NT_REQ, STAGES, OB, PRE_T, 0>;
}

}  // namespace sfft
