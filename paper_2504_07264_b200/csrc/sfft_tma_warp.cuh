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
//     stage with tcgen05.ld (TmemFactors64 below); TM = false: stages
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
struct TmemFactors64 {
    uint32_t taddr;            // lane quarter << 16 | column block
    __device__ __forceinline__ void fetch(int t, double2 *w) const
    {
        const int n = 1 << (t - 1), i0 = n - 1;
        uint32_t r[16][4];
        // constant trip counts (guarded) so the loops unroll before t is known
#pragma unroll
        for (int f = 0; f < 16; ++f)
            if (f < n)
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(r[f][0]), "=r"(r[f][1]), "=r"(r[f][2]), "=r"(r[f][3])
                         : "r"(taddr + 4 * (i0 + f)));
#pragma unroll
        for (int f = 0; f < 16; ++f) {
            if (f >= n) break;
            // the wait names the registers it makes valid, so no use is
            // scheduled above it (only the first one actually waits)
            asm volatile("tcgen05.wait::ld.sync.aligned;"
                         : "+r"(r[f][0]), "+r"(r[f][1]), "+r"(r[f][2]), "+r"(r[f][3]));
            w[f] = make_double2(__hiloint2double((int)r[f][1], (int)r[f][0]),
                                __hiloint2double((int)r[f][3], (int)r[f][2]));
        }
    }
    __device__ __forceinline__ void put(int i, double2 w) const
    {
        const uint32_t lo0 = (uint32_t)__double2loint(w.x), hi0 = (uint32_t)__double2hiint(w.x);
        const uint32_t lo1 = (uint32_t)__double2loint(w.y), hi1 = (uint32_t)__double2hiint(w.y);
        asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr + 4 * i), "r"(lo0),
                     "r"(hi0), "r"(lo1), "r"(hi1)
                     : "memory");
    }
};

// RING = false: each warp owns two slots.  RING = true: the CTA's warps
// share one ring of WARPS + XS slots -- CTA-local signal i lives in slot
// i % NSLOT and is consumed by warp i % WARPS, and the warp that releases a
// slot refills it with signal i + NSLOT (consumed by the next warp) -- so a
// warp needs ~1 slot instead of 2 and more warps fit an SM (the limit
// becomes the register file).
template <typename T, int WARPS, bool RING = false, int XS = 1>
struct TmaWShape {
    static constexpr int LOGN = 10, N = 1 << LOGN, LR = 5, R = 32, P = 32;
    static constexpr int PLANE = N * (int)sizeof(T);       // bytes of one plane of one signal
    static constexpr int SLOT = 2 * PLANE;                 // both planes
    static constexpr int STAGES = 2;
    static constexpr int NSLOT = RING ? WARPS + XS : STAGES * WARPS;
    static constexpr int WARP_BYTES = STAGES * SLOT;
    static constexpr int NT = 32 * WARPS;
    static constexpr int BAR_OFF = NSLOT * SLOT;
    static constexpr int REL_OFF = BAR_OFF + NSLOT * 8;     // RING: last released use of each slot
    static constexpr int TADDR_OFF = REL_OFF + (NSLOT * 4 + 15) / 16 * 16;   // TMEM base (tcgen05.alloc)
    static constexpr int SMEM = TADDR_OFF + 16;
    static constexpr int TMEM_COLS = WARPS > 8 ? 512 : (WARPS > 4 ? 256 : 128);
    static constexpr int MASK = sizeof(T) == 8 ? 15 : 31;  // slots per 128 bytes - 1
};

// exchange slot of logical element e (see the header comment)
template <typename T>
__device__ __forceinline__ int xw_phys(int e)
{
    return e ^ ((e >> 5) & (sizeof(T) == 8 ? 15 : 31));
}

template <typename T, bool DIF, int WARPS, int HK, bool TM, bool RING = false, int XS = 1>
__global__ void __launch_bounds__(32 * WARPS, 1) sfft_tmaw_kernel(const TmaWArgs a)
{
    static_assert(!TM || (sizeof(T) == 8 && WARPS <= 12), "TMEM factors: fp64, <= 12 warps");
    using Sh = TmaWShape<T, WARPS, RING, XS>;
    constexpr int N = Sh::N, R = Sh::R, LR = Sh::LR, NSLOT = Sh::NSLOT;
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // per-warp mode: this warp's two slots / barriers; ring mode: all of them
    unsigned char *wbuf = RING ? smem : smem + warp * Sh::WARP_BYTES;
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + Sh::BAR_OFF) + (RING ? 0 : warp * Sh::STAGES);
    volatile int *rel = reinterpret_cast<volatile int *>(smem + Sh::REL_OFF);
    const int64_t gw = (int64_t)blockIdx.x * WARPS + warp;
    const int64_t G = (int64_t)gridDim.x * WARPS;
    // ring mode: CTA-local signals i = 0 .. nloc-1 (row blockIdx.x + i * gridDim.x)
    const int64_t nloc = blockIdx.x < a.batch ? (a.batch - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const int64_t nk = RING ? (nloc > warp ? (nloc - 1 - warp) / WARPS + 1 : 0)
                            : (gw < a.batch ? (a.batch - 1 - gw) / G + 1 : 0);
    auto ring_row = [&](int64_t i) { return (int64_t)blockIdx.x + i * gridDim.x; };
    const T *xr = reinterpret_cast<const T *>(a.x_re);
    const T *xi = reinterpret_cast<const T *>(a.x_im);
    T *yr = reinterpret_cast<T *>(a.y_re);
    T *yi = reinterpret_cast<T *>(a.y_im);
    const TwCat<T> tw{reinterpret_cast<const vec2_t<T> *>(a.tw)};
    const T scale = (T)a.scale;
    const bool do_scale = a.scale_out != 0;

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
            // warp after its data arrived; every store follows its data
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

    // second-pass factors of stages LR+1 .. LR+HK: the lane's column only
    constexpr int NH = TM ? 0 : (1 << HK) - 1;
    vec2_t<T> hw[NH > 0 ? NH : 1];
#pragma unroll
    for (int t = 1; t <= (TM ? 0 : HK); ++t)
#pragma unroll
        for (int f = 0; f < (1 << (t - 1)); ++f) hw[(1 << (t - 1)) - 1 + f] = tw.get(LR + t, lane + (f << LR));
    // TM: all 31 second-pass factors in tensor memory instead
    TmemFactors64 tf;
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
#pragma unroll
        for (int t = 1; t <= LR; ++t)
#pragma unroll
            for (int f = 0; f < (1 << (t - 1)); ++f)
                tf.put((1 << (t - 1)) - 1 + f, tw.get(LR + t, lane + (f << LR)));
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

    for (int64_t k = 0; k < nk; ++k) {
        // ring: local signal i, slot i % NSLOT, its q-th use
        const int64_t i = warp + k * WARPS;
        const int st = RING ? (int)(i % NSLOT) : (int)(k & 1);
        const int64_t q = RING ? i / NSLOT : k >> 1;
        const int64_t row = RING ? ring_row(i) : gw + k * G;
        T *pr = reinterpret_cast<T *>(wbuf + st * Sh::SLOT);
        T *pi = reinterpret_cast<T *>(wbuf + st * Sh::SLOT + Sh::PLANE);
        if constexpr (RING) {
            // the slot's previous use (another warp's signal i - NSLOT) must
            // have completed its phase before this warp waits on the next
            // one -- an mbarrier parity wait cannot tell phase q-1 from q+1
            if (q > 0)
                while (rel[st] < (int)(q - 1)) {
                }
        }
        mbar_wait(bar + st, (uint32_t)(q & 1));
        // release this slot (all lanes' reads of it are done) and refill it
        auto release = [&]() {
            fence_async_smem();
            __syncwarp();
            if (lane == 0) {
                if constexpr (RING) {
                    rel[st] = (int)q;
                    if (i + NSLOT < nloc) issue(st, ring_row(i + NSLOT));
                } else {
                    if (k + Sh::STAGES < nk) issue(st, row + Sh::STAGES * G);
                }
            }
        };
        vec2_t<T> v[R];
        if constexpr (!DIF) {
            // pass 0: stages 1..5 on e = lane + 32 r (linear slot)
#pragma unroll
            for (int r = 0; r < R; ++r) {
                v[r].x = pr[lane + 32 * r];
                v[r].y = pi[lane + 32 * r];
            }
            dit_stages<T, LR, true, false>(v, 0, 0, tw);
            __syncwarp();
            // Stockham scatter in place: e = 32 lane + f <- register rev(f)
#pragma unroll
            for (int f = 0; f < R; ++f) {
                const int x = xw_phys<T>(32 * lane + f);
                pr[x] = v[brev(f, LR)].x;
                pi[x] = v[brev(f, LR)].y;
            }
            __syncwarp();
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int x = xw_phys<T>(lane + 32 * r);
                v[r].x = pr[x];
                v[r].y = pi[x];
            }
            release();
            __syncwarp();
            // pass 1: stages 6..10, column lane
            if constexpr (TM) dit_stages<T, LR, true, false>(v, LR, lane, tw, nullptr, nullptr, &tf);
            else dit_stages<T, LR, true, false, HK>(v, LR, lane, tw, nullptr, hw);
#pragma unroll
            for (int f = 0; f < R; ++f) put(row, lane + 32 * f, v[brev(f, LR)]);
        } else {
            // DIF pass 1 (stages 10..6, column lane) reads e = lane + 32 f into register rev(f)
#pragma unroll
            for (int f = 0; f < R; ++f) {
                v[brev(f, LR)].x = pr[lane + 32 * f];
                v[brev(f, LR)].y = pi[lane + 32 * f];
            }
            if constexpr (TM) dif_stages<T, LR, true, false>(v, LR, lane, tw, nullptr, nullptr, &tf);
            else dif_stages<T, LR, true, false, HK>(v, LR, lane, tw, nullptr, hw);
            __syncwarp();
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int x = xw_phys<T>(lane + 32 * r);
                pr[x] = v[r].x;
                pi[x] = v[r].y;
            }
            __syncwarp();
#pragma unroll
            for (int f = 0; f < R; ++f) {
                const int x = xw_phys<T>(32 * lane + f);
                v[brev(f, LR)].x = pr[x];
                v[brev(f, LR)].y = pi[x];
            }
            release();
            __syncwarp();
            // pass 0: stages 5..1
            dif_stages<T, LR, true, false>(v, 0, 0, tw);
#pragma unroll
            for (int r = 0; r < R; ++r) put(row, lane + 32 * r, v[r]);
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
