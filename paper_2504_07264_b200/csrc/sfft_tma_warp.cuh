// sfft_tma_warp.cuh -- warp-per-signal bulk-copy kernel, N = 1024 (radix 32).
//
// The reference's radix-2 stages (transform.py:208-270) in two register
// passes of 5 stages: one warp owns one signal (32 threads x 32 complex
// values), so a signal needs ONE shared-memory exchange instead of the three
// of the radix-8 schedule -- the L1 data pipe (shared wavefronts of the
// exchanges + global stores), not HBM, bounded the radix-8 TMA kernel on fp64
// N = 1024 (ncu: l1tex 81%, 1025 shared wavefronts per signal).
//
//   * Each warp is an independent persistent worker; the CTA's warps share
//     one ring of WARPS + XS slots (both planes of one signal each), signal
//     i of the CTA in slot i % NSLOT, consumed by warp i % WARPS.  The warp
//     that releases a slot refills it (lane 0: two non-tensor bulk copies,
//     cp.async.bulk, one contiguous 8 KiB row per plane for fp64) with
//     signal i + NSLOT, so global reads never use LSU wavefronts, every
//     warp's next signal is in flight for about one signal period, and a
//     warp costs ~1 slot instead of 2: 9 warps per SM (11 slots, 176 KiB)
//     instead of 7 with two slots each (RING = false), +3-5%.
//   * The slot is linear: the first pass's reads (lane-contiguous) are
//     conflict-free without a swizzle.  The exchange is written IN PLACE
//     into the slot once the first pass has read it (XOR layout
//     phys = e ^ ((e >> 5) & MASK), conflict-free for the Stockham write
//     (e = 32 lane + f) and the second pass's read (e = lane + 32 r)), and
//     the slot is released (and refilled) right after that read.
//   * The last pass stores straight to global memory (coalesced 256-byte
//     warp stores, streaming).
//   * Factors of the second pass depend only on the lane (column c = lane):
//     TM = true (shipped): all 31 parked in tensor memory once, fetched per
//     stage with tcgen05.ld (TmemFactors below); TM = false: stages
//     6..5+HK held in registers, the rest read per signal from the
//     L1-resident stage-major table (DIT serialised on those loads: 0.77).
// Arithmetic is the same dit_stages/dif_stages as every other kernel, so
// fp64 stays bit-identical to the reference.
#pragma once
#include "sfft_tma.cuh"

namespace sfft {

struct TmaWArgs {
    const void *x_re, *x_im;   // input planes (channel-swapped by the host for the inverse)
    void *y_re, *y_im;         // output planes (likewise)
    int64_t batch, in_stride, out_stride;   // rows, row strides in elements
    double scale;              // 1/N for the inverse
    int scale_out;
    const void *tw;            // stage-major table
};

// L2 prefetch of a contiguous row (no shared memory, no completion to wait for)
__device__ __forceinline__ void bulk_prefetch_l2(const void *src, uint32_t bytes)
{
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes, uint64_t *bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// Second-pass factors parked in tensor memory (TMEM, 512 x 32-bit columns x
// 128 lanes per SM, otherwise unused by this CUDA-core kernel).  Warp w owns
// lanes 32*(w%4).. and a 128-column block (w/4); its lane L holds factor i
// (stage 5+t, index f: i = 2^(t-1) - 1 + f) of column c = L in columns
// 4i .. 4i+3 (fp64 re, im as 2 x 2 words).  A stage's factors come back with
// tcgen05.ld (~12 cycles, no LSU/L1 traffic) right before the stage -- the
// register file keeps only the current stage's factors, where L1 loads of
// the whole set either spilled (all 31 factors hoisted: 124 registers next
// to the 128 of the data) or serialised on their latency.
template <typename T>
struct TmemFactors {
    static constexpr int W = 2 * (int)sizeof(T) / 4;   // 32-bit columns per complex factor
    uint32_t taddr;            // lane quarter << 16 | column block
    __device__ __forceinline__ void fetch(int t, vec2_t<T> *w) const
    {
        const int n = 1 << (t - 1), i0 = n - 1;
        uint32_t r[32][4];
        // constant trip counts (guarded) so the loops unroll before t is known
#pragma unroll
        for (int f = 0; f < 32; ++f) {
            if (f < n) {
                if constexpr (W == 4)
                    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                                 : "=r"(r[f][0]), "=r"(r[f][1]), "=r"(r[f][2]), "=r"(r[f][3])
                                 : "r"(taddr + W * (i0 + f)));
                else
                    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];"
                                 : "=r"(r[f][0]), "=r"(r[f][1])
                                 : "r"(taddr + W * (i0 + f)));
            }
        }
#pragma unroll
        for (int f = 0; f < 32; ++f) {
            if (f >= n) break;
            // the wait names the registers it makes valid, so no use is
            // scheduled above it (only the first one actually waits)
            if constexpr (W == 4) {
                asm volatile("tcgen05.wait::ld.sync.aligned;"
                             : "+r"(r[f][0]), "+r"(r[f][1]), "+r"(r[f][2]), "+r"(r[f][3]));
                w[f] = make_double2(__hiloint2double((int)r[f][1], (int)r[f][0]),
                                    __hiloint2double((int)r[f][3], (int)r[f][2]));
            } else {
                asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(r[f][0]), "+r"(r[f][1]));
                vec2_t<T> x;
                x.x = __uint_as_float(r[f][0]);
                x.y = __uint_as_float(r[f][1]);
                w[f] = x;
            }
        }
    }
    __device__ __forceinline__ void put(int i, vec2_t<T> w) const
    {
        if constexpr (W == 4) {
            const uint32_t lo0 = (uint32_t)__double2loint(w.x), hi0 = (uint32_t)__double2hiint(w.x);
            const uint32_t lo1 = (uint32_t)__double2loint(w.y), hi1 = (uint32_t)__double2hiint(w.y);
            asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr + W * i),
                         "r"(lo0), "r"(hi0), "r"(lo1), "r"(hi1)
                         : "memory");
        } else {
            asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(taddr + W * i),
                         "r"(__float_as_uint(w.x)), "r"(__float_as_uint(w.y))
                         : "memory");
        }
    }
};

// RING = false: each warp owns two slots.  RING = true: the CTA's signal
// groups share one ring of GROUPS + XS slots -- CTA-local signal i lives in
// slot i % NSLOT and is consumed by group i % GROUPS, and the group that
// releases a slot refills it with signal i + NSLOT (consumed by the next
// group) -- so a group needs ~1 slot instead of 2 and more warps fit an SM
// (the limit becomes the register file).
// A signal of N = 2^LOGN points is owned by a group of WPS warps (P = 32 WPS
// threads x R = N / P values, two register passes of LR = log2 R stages):
// fp64 N = 1024: one warp, radix 32; fp32 N = 4096: two warps, radix 64.
template <typename T, int WARPS, bool RING = false, int XS = 1, int LOGN_ = 10, int WPS = 1>
struct TmaWShape {
    static constexpr int LOGN = LOGN_, N = 1 << LOGN, P = 32 * WPS, R = N / P;
    static constexpr int LR = LOGN / 2;
    static_assert((1 << LR) == R && 2 * LR == LOGN, "two register passes of log2(N/P) stages");
    static_assert(WARPS % WPS == 0, "whole signal groups per CTA");
    static constexpr int GROUPS = WARPS / WPS;
    static constexpr int PLANE = N * (int)sizeof(T);       // bytes of one plane of one signal
    static constexpr int SLOT = 2 * PLANE;                 // both planes
    static constexpr int STAGES = 2;
    static constexpr int NSLOT = RING ? GROUPS + XS : STAGES * WARPS;
    static constexpr int WARP_BYTES = STAGES * SLOT;
    static constexpr int NT = 32 * WARPS;
    static constexpr int BAR_OFF = NSLOT * SLOT;
    static constexpr int REL_OFF = BAR_OFF + NSLOT * 8;     // RING: last released use of each slot
    static constexpr int TADDR_OFF = REL_OFF + (NSLOT * 4 + 15) / 16 * 16;   // TMEM base (tcgen05.alloc)
    static constexpr int SMEM = TADDR_OFF + 16;
    static constexpr int TMEM_COLS = WARPS > 8 ? 512 : (WARPS > 4 ? 256 : 128);
};

// exchange slot of logical element e, 8-byte elements (fp64 planar values or
// fp32 (re, im) pairs): XOR of the 16 slots of each 128-byte line with the
// element's "row" e >> LR -- conflict-free for the Stockham write
// (e = P t + f) and the next pass's read (e = t + P r) when P = 2^LR.
template <int LR>
__device__ __forceinline__ int xw_phys(int e)
{
    return e ^ ((e >> LR) & 15);
}

// PF > 0 (ring mode): when a group refills its slot with signal i + NSLOT it
// also prefetches signal i + NSLOT + PF into L2, so the later bulk copy of
// that signal is an L2 hit.
template <typename T, bool DIF, int WARPS, int HK, bool TM, bool RING = false, int XS = 1, int LOGN_ = 10, int WPS = 1,
          int PF = 0>
__global__ void __launch_bounds__(32 * WARPS, 1) sfft_tmaw_kernel(const TmaWArgs a)
{
    static_assert(!TM || WARPS <= 12, "TMEM factors: <= 3 warps per lane quarter");
    static_assert(RING || WPS == 1, "groups of several warps use the slot ring");
    using Sh = TmaWShape<T, WARPS, RING, XS, LOGN_, WPS>;
    constexpr int N = Sh::N, R = Sh::R, LR = Sh::LR, P = Sh::P, NSLOT = Sh::NSLOT, GROUPS = Sh::GROUPS;
    // fp32: (re, im) pairs in the exchange, packed f32x2 math, stage factors
    // formed from per-thread base factors (FactorTw); fp64: planar exchange,
    // scalar math, table factors (bit-exact contract)
    constexpr bool F32 = sizeof(T) == 4;
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int grp = warp / WPS;                       // signal group of this warp
    const int t = threadIdx.x % P;                    // thread of the signal
    // per-warp mode: this warp's two slots / barriers; ring mode: all of them
    unsigned char *wbuf = RING ? smem : smem + warp * Sh::WARP_BYTES;
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + Sh::BAR_OFF) + (RING ? 0 : warp * Sh::STAGES);
    volatile int *rel = reinterpret_cast<volatile int *>(smem + Sh::REL_OFF);
    const int64_t gw = (int64_t)blockIdx.x * WARPS + warp;
    const int64_t G = (int64_t)gridDim.x * WARPS;
    // ring mode: CTA-local signals i = 0 .. nloc-1 (row blockIdx.x + i * gridDim.x)
    const int64_t nloc = blockIdx.x < a.batch ? (a.batch - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const int64_t nk = RING ? (nloc > grp ? (nloc - 1 - grp) / GROUPS + 1 : 0)
                            : (gw < a.batch ? (a.batch - 1 - gw) / G + 1 : 0);
    auto ring_row = [&](int64_t i) { return (int64_t)blockIdx.x + i * gridDim.x; };
    const T *xr = reinterpret_cast<const T *>(a.x_re);
    const T *xi = reinterpret_cast<const T *>(a.x_im);
    T *yr = reinterpret_cast<T *>(a.y_re);
    T *yi = reinterpret_cast<T *>(a.y_im);
    const TwCat<T> tw{reinterpret_cast<const vec2_t<T> *>(a.tw)};
    const T scale = (T)a.scale;
    const bool do_scale = a.scale_out != 0;
    // barrier among the P threads of this signal
    auto gsync = [&]() {
        if constexpr (WPS == 1) __syncwarp();
        else asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "n"(P) : "memory");
    };

    auto issue = [&](int st, int64_t row) {
        mbar_expect_tx(bar + st, Sh::SLOT);
        unsigned char *dst = wbuf + st * Sh::SLOT;
        bulk_load(dst, xr + row * a.in_stride, Sh::PLANE, bar + st);
        bulk_load(dst + Sh::PLANE, xi + row * a.in_stride, Sh::PLANE, bar + st);
    };
    if constexpr (RING) {
        if (threadIdx.x == 0) {
            for (int s = 0; s < NSLOT; ++s) {
                mbar_init(bar + s, 1);
                rel[s] = -1;
            }
            fence_mbar_init();
#ifndef SFFT_TMA_NO_PDL
            // dependent launch: every load is issued by this thread or by a
            // group after its data arrived; every store follows its data
            asm volatile("griddepcontrol.wait;" ::: "memory");
            asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
            for (int s = 0; s < NSLOT && s < nloc; ++s) issue(s, ring_row(s));
        }
        __syncthreads();
    } else {
        if (lane == 0) {
            for (int s = 0; s < Sh::STAGES; ++s) mbar_init(bar + s, 1);
            fence_mbar_init();
#ifndef SFFT_TMA_NO_PDL
            // dependent launch: every global access of this warp follows this
            // wait (its loads are issued here, its stores follow their data)
            asm volatile("griddepcontrol.wait;" ::: "memory");
            if (warp == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
            for (int s = 0; s < Sh::STAGES && s < nk; ++s) issue(s, gw + s * G);
        }
        __syncwarp();
    }

    // second-pass factors of stages LR+1 .. LR+HK (fp64, TM = false): the
    // thread's column only
    constexpr int NH = (TM || F32) ? 0 : (1 << HK) - 1;
    vec2_t<T> hw[NH > 0 ? NH : 1];
#pragma unroll
    for (int tt = 1; tt <= ((TM || F32) ? 0 : HK); ++tt)
#pragma unroll
        for (int f = 0; f < (1 << (tt - 1)); ++f) hw[(1 << (tt - 1)) - 1 + f] = tw.get(LR + tt, t + (f << LR));
    // fp32: base factors w_{LR+tt}(t) of the second pass, once for all signals
    vec2_t<T> pre[F32 ? LR : 1];
    if constexpr (F32 && !TM) {
#pragma unroll
        for (int tt = 1; tt <= LR; ++tt) pre[tt - 1] = tw.get(LR + tt, t);
    }
    // TM: all second-pass factors in tensor memory instead
    TmemFactors<T> tf;
    uint32_t *taddr_sm = reinterpret_cast<uint32_t *>(smem + Sh::TADDR_OFF);
    if constexpr (TM) {
        if (warp == 0) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(taddr_sm)),
                         "r"(Sh::TMEM_COLS)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        tf.taddr = *taddr_sm + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(128 * (warp >> 2));
        // every second-pass factor of column t, exactly as the stage helpers
        // form it (fp64: table values; fp32: base x immediate, FactorTw)
#pragma unroll
        for (int tt = 1; tt <= LR; ++tt) {
            vec2_t<T> base{};
            if constexpr (F32) base = tw.get(LR + tt, t);
#pragma unroll
            for (int f = 0; f < (1 << (tt - 1)); ++f)
                tf.put((1 << (tt - 1)) - 1 + f, stage_factor<T>(tt, f, LR + tt, false, t, LR, tw, base));
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }

    auto put = [&](int64_t row, int e, vec2_t<T> v) {
        if (do_scale) {
            v.x *= scale;
            v.y *= scale;
        }
        st_stream(yr + row * a.out_stride + e, v.x);
        st_stream(yi + row * a.out_stride + e, v.y);
    };
    // second-pass stages (DIT ascending / DIF descending), column t
    auto pass1 = [&](vec2_t<T> *v) {
        if constexpr (TM) {
            if constexpr (!DIF) dit_stages<T, LR, true, F32>(v, LR, t, tw, nullptr, nullptr, &tf);
            else dif_stages<T, LR, true, F32>(v, LR, t, tw, nullptr, nullptr, &tf);
        } else if constexpr (F32) {
            if constexpr (!DIF) dit_stages<T, LR, true, true>(v, LR, t, tw, pre);
            else dif_stages<T, LR, true, true>(v, LR, t, tw, pre);
        } else {
            if constexpr (!DIF) dit_stages<T, LR, true, false, HK>(v, LR, t, tw, nullptr, hw);
            else dif_stages<T, LR, true, false, HK>(v, LR, t, tw, nullptr, hw);
        }
    };

    for (int64_t k = 0; k < nk; ++k) {
        // ring: local signal i, slot i % NSLOT, its q-th use
        const int64_t i = grp + k * GROUPS;
        const int st = RING ? (int)(i % NSLOT) : (int)(k & 1);
        const int64_t q = RING ? i / NSLOT : k >> 1;
        const int64_t row = RING ? ring_row(i) : gw + k * G;
        T *pr = reinterpret_cast<T *>(wbuf + st * Sh::SLOT);
        T *pi = reinterpret_cast<T *>(wbuf + st * Sh::SLOT + Sh::PLANE);
        vec2_t<T> *px = reinterpret_cast<vec2_t<T> *>(wbuf + st * Sh::SLOT);
        // exchange access (8-byte elements): fp64 planar, fp32 pairs
        auto xget = [&](int e) -> vec2_t<T> {
            const int x = xw_phys<LR>(e);
            vec2_t<T> w;
            if constexpr (F32) {
                w = px[x];
            } else {
                w.x = pr[x];
                w.y = pi[x];
            }
            return w;
        };
        auto xput = [&](int e, vec2_t<T> w) {
            const int x = xw_phys<LR>(e);
            if constexpr (F32) {
                px[x] = w;
            } else {
                pr[x] = w.x;
                pi[x] = w.y;
            }
        };
        if constexpr (RING) {
            // the slot's previous use (another group's signal i - NSLOT) must
            // have completed its phase before this group waits on the next
            // one -- an mbarrier parity wait cannot tell phase q-1 from q+1
            if (q > 0)
                while (rel[st] < (int)(q - 1)) {
                }
        }
        mbar_wait(bar + st, (uint32_t)(q & 1));
        // release this slot (all reads of it are done) and refill it
        auto release = [&]() {
            fence_async_smem();
            gsync();
            if (t == 0) {
                if constexpr (RING) {
                    rel[st] = (int)q;
                    if (i + NSLOT < nloc) issue(st, ring_row(i + NSLOT));
                    if constexpr (PF > 0) {
                        if (i + NSLOT + PF < nloc) {
                            const int64_t pr_ = ring_row(i + NSLOT + PF);
                            bulk_prefetch_l2(xr + pr_ * a.in_stride, Sh::PLANE);
                            bulk_prefetch_l2(xi + pr_ * a.in_stride, Sh::PLANE);
                        }
                    }
                } else {
                    if (k + Sh::STAGES < nk) issue(st, row + Sh::STAGES * G);
                }
            }
        };
        vec2_t<T> v[R];
        if constexpr (!DIF) {
            // pass 0: stages 1..LR on e = t + P r (linear slot)
#pragma unroll
            for (int r = 0; r < R; ++r) {
                v[r].x = pr[t + P * r];
                v[r].y = pi[t + P * r];
            }
            dit_stages<T, LR, true, F32>(v, 0, 0, tw);
            gsync();
            // Stockham scatter in place: e = P t + f <- register rev(f)
#pragma unroll
            for (int f = 0; f < R; ++f) xput(P * t + f, v[brev(f, LR)]);
            gsync();
#pragma unroll
            for (int r = 0; r < R; ++r) v[r] = xget(t + P * r);
            release();
            if constexpr (WPS == 1) __syncwarp();
            // pass 1: stages LR+1 .. 2 LR, column t
            pass1(v);
#pragma unroll
            for (int f = 0; f < R; ++f) put(row, t + P * f, v[brev(f, LR)]);
        } else {
            // DIF pass 1 (stages 2 LR .. LR+1, column t) reads e = t + P f into register rev(f)
#pragma unroll
            for (int f = 0; f < R; ++f) {
                v[brev(f, LR)].x = pr[t + P * f];
                v[brev(f, LR)].y = pi[t + P * f];
            }
            pass1(v);
            gsync();
#pragma unroll
            for (int r = 0; r < R; ++r) xput(t + P * r, v[r]);
            gsync();
#pragma unroll
            for (int f = 0; f < R; ++f) v[brev(f, LR)] = xget(P * t + f);
            release();
            if constexpr (WPS == 1) __syncwarp();
            // pass 0: stages LR..1
            dif_stages<T, LR, true, F32>(v, 0, 0, tw);
#pragma unroll
            for (int r = 0; r < R; ++r) put(row, t + P * r, v[r]);
        }
    }
    if constexpr (TM) {
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        if (warp == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*taddr_sm), "r"(Sh::TMEM_COLS)
                         : "memory");
        }
    }
    (void)N;
}

}  // namespace sfft
