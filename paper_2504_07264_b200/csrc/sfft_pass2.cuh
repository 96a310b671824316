// sfft_pass2.cuh -- L2-fused pairs of pass groups: one HBM sweep for two
// stage groups of the multi-launch schedule (N = 2^m > 4096).
//
// The pass schedule (sfft_pass.cuh) runs group (S, L) as N/2^L independent
// 2^L-point sub-problems and moves the whole row through HBM once per group
// (4 sweeps for N = 2^28).  Two consecutive groups (S, L1), (S+L1, L2) are
// one group (S, L = L1+L2) whose 2^L-point sub-problems j are independent;
// TJ consecutive ones (a "block", TJ * 2^L elements = 4 MiB fp32 at L = 14)
// close under both groups:
//   group (S, L1) sub-problems   j' = j + E2 * NJ            (E2 < 2^L2, NJ = N/2^L)
//   write positions               j'' + E2 * 2^(m-L2),  j'' = (j>>S) 2^(S+L1) + (j mod 2^S) + 2^S o
//   group (S+L1, L2) sub-problems j''  (o < 2^L1)  read exactly those.
// So a persistent kernel runs, block after block, the first group's tiles
// of a block (HBM -> a block scratch slot) and, D blocks behind, the second
// group's tiles (scratch -> HBM).  The scratch ring (NSLOT slots of one
// block) stays in L2, so each pair of groups costs one HBM read and one
// HBM write of the row instead of two of each.
//
// Scratch layout of a block, (re, im) pairs (one 64/128-bit access per complex
// value; every scratch stride is a compile-time constant, so the scratch
// side of a tile is addressed as one per-thread base plus immediates)
// (columns jl < TJ = the block's sub-problems, E2 < 2^L2, o < 2^L1):
//   S > 0:  ((E2 << L1) + o) * TJ + jl   -- both sides 256-byte runs over jl
//   S = 0:  ((jl << L2) + E2 << L1) + o  -- the first group's outputs are rows
//           of 2^L1 per sub-problem (the S = 0 transpose); the second group
//           reads 256-byte runs over o
// The tiles are the pass kernel's tiles (TJ columns x 2^Lg points, register
// passes + shared exchanges, the same factor formation), so every output
// is bit-identical to the multi-launch schedule with the same groups.
//
// Ordering: work items (tiles) are dealt by an atomic ticket in the order
//   step s: [first-group tiles of block s] [second-group tiles of block s-D]
// and an item only waits for items with smaller tickets (block b's second
// group waits for its first group; the first group of block b waits for the
// second group of block b - NSLOT, whose slot it reuses, NSLOT > D), so the
// smallest unfinished ticket always makes progress (no co-residency needed).
// Per-slot completion counters are cumulative (epoch b / NSLOT).
//
// DIF runs the transposed schedule: super-groups last to first, inside one
// the second group first (reading the positions DIT writes) and the first
// group second.
#pragma once
#include "sfft_pass.cuh"

namespace sfft {

struct Pass2Args {
    const void *x0, *x1;   // super-group source planes (the host exchanges them for the inverse)
    void *y0, *y1;         // destination planes
    void *s0, *s1;         // s0: scratch ring of nslot blocks of TJ * 2^L (re, im) pairs (s1 unused)
    unsigned *ctr;         // [0] ticket, [1 + slot] first-group tiles done, [1 + nslot + slot] second
    int64_t batch, in_stride, out_stride;
    int m, S;              // log2 N, stage offset of the super-group
    int nslot_log, lag;    // ring of 2^nslot_log block slots, second phase `lag` blocks behind
    int scale_out;         // multiply the destination by `scale` (the inverse's last launch)
    int flags;             // P2_DEFER | P2_PREFETCH (see the kernel)
    double scale;
    const void *tw;        // as PassArgs
    int tw_cat_top;
    const void *tw_top_tab;
    const double2 *coarse;
    int coarse_log;
    const double2 *fine;
};

// flags: P2_NOPIPE turns the look-ahead load of the next tile off (every tile
// then loads through its landing buffer at its own start; A/B).
constexpr int P2_NOPIPE = 1;

template <typename T> struct P2TJ { static constexpr int value = sizeof(T) == 4 ? 32 : 16; };

// 8 threads per column (R = 2^(Lg-3) values each), TJ columns per tile
template <typename T, int L1, int L2>
struct P2Shape {
    static constexpr int TJ = P2TJ<T>::value;
    static constexpr int P = 8;
    static constexpr int NT = TJ * P;
    static constexpr int RS = TJ + 1;
    static constexpr int LMAX = 7;   // p2_tile places the column factors after a 2^7-point tile
    // landing buffer of one source tile (2^LMAX rows of TJ complex values:
    // two planes of 128-byte rows, or 256-byte rows of pairs), then the
    // exchange tile and the column factors
    static constexpr int LB_PLANE = (1 << LMAX) * TJ * (int)sizeof(T);
    static constexpr int LB_BYTES = 2 * LB_PLANE;
    static constexpr int smem_bytes()
    {
        return LB_BYTES + (1 << LMAX) * RS * 2 * (int)sizeof(T) + LMAX * TJ * 2 * (int)sizeof(T);
    }
};

template <typename T, int L1, int L2>
struct P2MinBlocks {
    static constexpr int NT = P2Shape<T, L1, L2>::NT;
    static constexpr int value = sizeof(T) == 4 ? 3 : 0;   // 66 KiB of shared memory per CTA: three per SM
};

// Asynchronous 16-byte copies global -> shared (L2 only: the block scratch is
// written by other SMs during the kernel), one commit group per tile.
__device__ __forceinline__ void p2_cp16(uint32_t dst, const void *src)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void p2_cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void p2_cp_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Issue the copies of one source tile into the landing buffer `lb` (shared
// address): 2^rows_log rows of TJ complex values at p0 (+ p1: the second
// plane) with `stride_b` bytes between rows.  pairs: rows of TJ (re, im)
// pairs (256 bytes) land at lb + 256 e; planes: two 128-byte rows per e land
// at lb + 128 e and lb + LB_PLANE + 128 e.  16 << rows_log chunks either way.
template <int NT, int LB_PLANE>
__device__ __forceinline__ void p2_issue_tile(uint32_t lb, bool pairs, const char *p0, const char *p1,
                                              uint32_t stride_b, int rows_log, int tid)
{
    const int chunks = 16 << rows_log;
    if (pairs) {
        const int c = tid & 15;
        const char *src = p0 + (size_t)(tid >> 4) * stride_b + c * 16;
        uint32_t dst = lb + (uint32_t)tid * 16u;
        const size_t step = (size_t)(NT / 16) * stride_b;
        for (int q = tid; q < chunks; q += NT) {
            p2_cp16(dst, src);
            src += step;
            dst += NT * 16u;
        }
    } else {
        const int per_plane = 8 << rows_log;
        for (int q = tid; q < chunks; q += NT) {
            const int pl = q >= per_plane, r = q - pl * per_plane;
            const char *src = (pl ? p1 : p0) + (size_t)(r >> 3) * stride_b + (r & 7) * 16;
            p2_cp16(lb + (uint32_t)pl * LB_PLANE + (uint32_t)r * 16u, src);
        }
    }
    p2_cp_commit();
}

template <typename T, bool S0G>
__device__ __forceinline__ typename PassTw<T, S0G>::type make_p2_tw(const Pass2Args &a)
{
    typename PassTw<T, S0G>::type tw;
    tw.tab = (const vec2_t<T> *)a.tw;
    if constexpr (!S0G) {
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

// One tile: TJ columns of 2^L-point sub-problems of group (S, L), column jl's
// factor column c0 + jl (S > 0).  Column side: element e of column jl at
// base + jl + e * stride; row side (the S = 0 group: DIT destination, DIF
// source): element o of column jl at base + jl * stride + o.
// Scheduler hooks, each run once per tile: `mid()` after the first register
// pass (the look-ahead for the next tile, off the tile's critical path),
// `px()` after the CTA barrier that follows `mid()` (every thread has read
// its part of the landing buffer by then: the next tile's copies start here).
// The scratch side (IN_SCR: source, OUT_SCR: destination) is `scr`, pairs
// with the compile-time element stride SSTR; the plane pointers and the
// runtime stride of that side are unused.
// USE_LB: the source tile (column side) is in the landing buffer at the
// start of smem_raw, its copies issued by the caller (p2_issue_tile); the
// tile waits for them.  Otherwise (the S = 0 DIF group's row-side source) it
// loads straight from global memory.
template <typename T, int L, bool DIF, bool S0G, bool IN_SCR, bool OUT_SCR, uint32_t SSTR, bool USE_LB, typename Mid,
          typename Px>
__device__ __forceinline__ void p2_tile(const T *ir, const T *ii, uint32_t istr, T *orr, T *oi, uint32_t ostr,
                                        vec2_t<T> *scr, int S, uint32_t c0, const Pass2Args &a,
                                        unsigned char *smem_raw, const Mid &mid, const Px &px)
{
    constexpr int TJ = P2TJ<T>::value, P = 8, SUB = 1 << L, LR = L - 3, R = 1 << LR, NT = TJ * P;
    constexpr int RS = TJ + 1, NPI = (L + LR - 1) / LR;
    static_assert(L >= 5 && L <= 7, "fused pair groups are 2^5..2^7 points");
    using V = vec2_t<T>;
    constexpr int LMAX = 7;
    constexpr int LB_PLANE = (1 << LMAX) * TJ * (int)sizeof(T);
    static_assert(USE_LB || (DIF && S0G), "only the row-side source bypasses the landing buffer");
    const T *lbp = reinterpret_cast<const T *>(smem_raw);    // planes: [2][row][TJ]
    const V *lbv = reinterpret_cast<const V *>(smem_raw);    // pairs: [row][TJ]
    V *sx = reinterpret_cast<V *>(smem_raw + 2 * LB_PLANE);
    V *cs = sx + (1 << LMAX) * RS;   // [L][TJ] column factors (after the largest tile)
    const int tid = threadIdx.x;
    const int jl = tid % TJ, t = tid / TJ;
    const uint32_t c = S0G ? 0u : c0 + (uint32_t)jl;
    const auto tw = make_p2_tw<T, S0G>(a);
    using I = typename PassTw<T, S0G>::type::index_t;
    const bool scale_out = !OUT_SCR && a.scale_out != 0;   // only the super-group's destination
    const T scale = (T)a.scale;
    constexpr bool CST = FactorTw<T>::value && !S0G;
    const uint32_t os_b = ostr * (uint32_t)sizeof(T);

    // source element of row `e` (landing buffer: rows of TJ values, this thread's column jl)
    auto get_row = [&](uint32_t e) {
        V w;
        if constexpr (IN_SCR) {
            w = lbv[e * TJ + jl];
        } else {
            w.x = lbp[e * TJ + jl];
            w.y = lbp[LB_PLANE / (int)sizeof(T) + e * TJ + jl];
        }
        return w;
    };
    auto put = [&](T *pr, T *pi, V *ps, V w) {
        if constexpr (OUT_SCR) {
            __stcg(ps, w);   // the block scratch: default L2 policy, read back soon
        } else {
            if (scale_out) {
                w.x *= scale;
                w.y *= scale;
            }
            st_stream(pr, w.x);
            st_stream(pi, w.y);
        }
    };
    auto put_k = [&](T *pr, T *pi, V *ps, uint32_t k, V w) {
        if constexpr (OUT_SCR) put(nullptr, nullptr, ps + k * SSTR, w);
        else put(at_stride(pr, os_b, k), at_stride(pi, os_b, k), nullptr, w);
    };
    auto stage_columns = [&]() {
        if constexpr (CST) {
            for (int k = tid; k < L * TJ; k += NT) {
                const int st = k / TJ, l = k - st * TJ;
                cs[k] = tw.get(S + 1 + st, (I)(c0 + (uint32_t)l));
            }
        }
        if constexpr (USE_LB) p2_cp_wait_all();          // this thread's copies of the source tile
        if constexpr (USE_LB || CST) __syncthreads();    // everyone's copies and the column factors
    };
    auto column_factors = [&](int sp, int KP, int jp, V *cf) {
        const int x = jp & ((1 << sp) - 1);
        for (int tt = 1; tt <= KP; ++tt) {
            V w = cs[(sp + tt - 1) * TJ + jl];
            if (sp > 0) {
                const V sm = ldtw(tw.tab + ((1 << (sp + tt - 1)) - 1) + x);
                T r, i;
                cmul(w.x, w.y, sm.x, sm.y, r, i);
                w.x = r;
                w.y = i;
            }
            cf[tt - 1] = w;
        }
    };

    V v[R];
    if constexpr (!DIF) {
        // column-side source: element (t + k) of column jl
        static_for<0, NPI>([&](auto PPC) {
            constexpr int pp = decltype(PPC)::value;
            constexpr int sp = pp * LR, KP = cmin(LR, L - sp), RP = 1 << KP, U = R / RP, nsp = 1 << sp;
            constexpr bool last = pp == NPI - 1;
            if constexpr (pp == 0) stage_columns();
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int jp = t + P * u;
#pragma unroll
                for (int r = 0; r < RP; ++r) {
                    if constexpr (pp == 0) {
                        const uint32_t k = (uint32_t)(P * u + r * (SUB / RP));
                        v[u * RP + r] = get_row((uint32_t)t + k);
                    } else {
                        v[u * RP + r] = sx[(jp + r * (SUB / RP)) * RS + jl];
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int jp = t + P * u;
                V cf[KP];
                if constexpr (CST) column_factors(sp, KP, jp, cf);
                dit_stages<T, KP, S0G>(v + u * RP, S + sp, (I)(c + ((uint32_t)(jp & (nsp - 1)) << S)), tw,
                                       CST ? cf : nullptr);
            }
            if constexpr (pp == 0) mid();
            if constexpr (!last || S0G) {
                if constexpr (pp > 0) __syncthreads();
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int jp = t + P * u;
                    const int base = (jp >> sp) * nsp * RP + (jp & (nsp - 1));
#pragma unroll
                    for (int f = 0; f < RP; ++f) sx[(base + nsp * f) * RS + jl] = v[u * RP + brev(f, KP)];
                }
                __syncthreads();
                if constexpr (pp == 0) px();
            } else {
                T *out_r = OUT_SCR ? nullptr : orr + jl + (size_t)t * ostr;
                T *out_i = OUT_SCR ? nullptr : oi + jl + (size_t)t * ostr;
                V *out_s = OUT_SCR ? scr + jl + t * SSTR : nullptr;
#pragma unroll
                for (int u = 0; u < U; ++u) {
#pragma unroll
                    for (int f = 0; f < RP; ++f) {
                        const uint32_t k = (uint32_t)(P * u + nsp * f);
                        put_k(out_r, out_i, out_s, k, v[u * RP + brev(f, KP)]);
                    }
                }
            }
        });
        if constexpr (S0G) {
            // row-side destination: smem [o][jj] -> rows of 2^L per column
#pragma unroll
            for (int kk = 0; kk < R; ++kk) {
                const int k = tid + kk * NT, jj = k >> L, o = k & (SUB - 1);
                if constexpr (OUT_SCR) {
                    put(nullptr, nullptr, scr + (uint32_t)jj * SSTR + o, sx[o * RS + jj]);
                } else {
                    const size_t off = (size_t)jj * ostr + o;
                    put(orr + off, oi + off, nullptr, sx[o * RS + jj]);
                }
            }
        }
    } else {
        if constexpr (S0G) {
            // row-side source (all R loads first, then the shared stores)
#pragma unroll
            for (int kk = 0; kk < R; ++kk) {
                const int k = tid + kk * NT, jj = k >> L, o = k & (SUB - 1);
                if constexpr (IN_SCR) {
                    v[kk] = __ldcg(scr + (uint32_t)jj * SSTR + o);
                } else {
                    const size_t off = (size_t)jj * istr + o;
                    v[kk].x = ld_stream(ir + off);
                    v[kk].y = ld_stream(ii + off);
                }
            }
#pragma unroll
            for (int kk = 0; kk < R; ++kk) {
                const int k = tid + kk * NT, jj = k >> L, o = k & (SUB - 1);
                sx[o * RS + jj] = v[kk];
            }
            __syncthreads();
        }
        static_for<0, NPI>([&](auto QC) {
            constexpr int pp = NPI - 1 - decltype(QC)::value;
            constexpr int sp = pp * LR, KP = cmin(LR, L - sp), RP = 1 << KP, U = R / RP, nsp = 1 << sp;
            constexpr bool first = pp == NPI - 1;
            if constexpr (first && !S0G) stage_columns();
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int jp = t + P * u;
                const int base = (jp >> sp) * nsp * RP + (jp & (nsp - 1));
#pragma unroll
                for (int f = 0; f < RP; ++f) {
                    const int d = u * RP + brev(f, KP);
                    if constexpr (first && !S0G) {
                        v[d] = get_row((uint32_t)(base + nsp * f));
                    } else {
                        v[d] = sx[(base + nsp * f) * RS + jl];
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int jp = t + P * u;
                V cf[KP];
                if constexpr (CST) column_factors(sp, KP, jp, cf);
                dif_stages<T, KP, S0G>(v + u * RP, S + sp, (I)(c + ((uint32_t)(jp & (nsp - 1)) << S)), tw,
                                       CST ? cf : nullptr);
            }
            if constexpr (first) mid();
            if constexpr (pp != 0) {
                if constexpr (!first || S0G) __syncthreads();
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int jp = t + P * u;
#pragma unroll
                    for (int r = 0; r < RP; ++r) sx[(jp + r * (SUB / RP)) * RS + jl] = v[u * RP + r];
                }
                __syncthreads();
                if constexpr (first) px();
            } else {
                T *out_r = OUT_SCR ? nullptr : orr + jl + (size_t)t * ostr;
                T *out_i = OUT_SCR ? nullptr : oi + jl + (size_t)t * ostr;
                V *out_s = OUT_SCR ? scr + jl + t * SSTR : nullptr;
#pragma unroll
                for (int u = 0; u < U; ++u) {
#pragma unroll
                    for (int r = 0; r < RP; ++r) {
                        const uint32_t k = (uint32_t)(P * u + r * (SUB / RP));
                        put_k(out_r, out_i, out_s, k, v[u * RP + r]);
                    }
                }
            }
        });
    }
}

// Completion counters: polled with relaxed loads (an acquire load costs an
// L1 invalidation, CCTL.IVALL, and every access to data another CTA wrote is
// an L2 access, ld.cg / st.cg, anyway); published with a release reduction
// after a CTA barrier.
__device__ __forceinline__ unsigned p2_ld_relaxed(const unsigned *p)
{
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void p2_signal(unsigned *p)
{
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p) : "memory");
}

// One scheduled tile: phase (0: the group run first), block, tile index, and
// the counter (+ target) it depends on (none: dep = nullptr).
struct P2Item {
    uint32_t b;
    int ph, tile, slot;
    const unsigned *dep;
    unsigned target;
};

// Geometry of the two groups' tiles of block (row, J0) (DIT numbering):
//   first group (S, L1), tile E2 < 2^L2: row side x + J0 + E2 NJ, stride NJ 2^L2;
//     scratch side (S > 0) (E2 << L1) TJ, stride TJ; (S = 0) E2 << L1, row stride 2^L
//   second group (S+L1, L2), tile u < 2^L1:
//     (S > 0) scratch u TJ, stride TJ 2^L1; row side (J0>>S) 2^(S+L) + (J0 mod 2^S) + 2^S u,
//             stride 2^(S+L1); factor column (J0 mod 2^S) + 2^S u
//     (S = 0) column jl = u / (2^L1/TJ), o0 = (u mod (2^L1/TJ)) TJ: scratch jl 2^L + o0,
//             stride 2^L1; row side (J0 + jl) 2^L + o0, stride 2^L1; factor column o0
template <typename T, int L1, int L2, bool DIF, bool SZ>
__global__ void __launch_bounds__(P2Shape<T, L1, L2>::NT, (P2MinBlocks<T, L1, L2>::value))
sfft_pass2_kernel(const Pass2Args a)
{
    using Sh = P2Shape<T, L1, L2>;
    constexpr int TJ = Sh::TJ, L = L1 + L2;
    constexpr int LTJ = TJ == 32 ? 5 : 4;
    static_assert(!SZ || L1 >= LTJ, "S = 0 second-group tiles take TJ consecutive outputs o");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ unsigned s_item[2];   // this tile's / the next tile's ticket
    const int m = a.m;
    const int S = SZ ? 0 : a.S;
    const uint32_t NJ = 1u << (m - L);            // 2^L-point sub-problems per row
    const uint32_t nbr = NJ / TJ;                  // blocks per row
    const int64_t NB = a.batch * (int64_t)nbr;
    // tiles per block of the phase run first / second (DIF: the second group first)
    constexpr int TA = DIF ? (1 << L1) : (1 << L2);
    constexpr int TB = DIF ? (1 << L2) : (1 << L1);
    const int64_t D = a.lag;
    const uint32_t total = (uint32_t)(NB * (TA + TB));
    const int nslot = 1 << a.nslot_log;
    unsigned *doneA = a.ctr + 1, *doneB = a.ctr + 1 + nslot;
    const size_t slot_elems = (size_t)TJ << L;
    const int tid = threadIdx.x;

    // ticket -> scheduled tile (see the header comment for the order); all
    // 32-bit (tickets < 2^32, checked by the host), slots a power of two
    const uint32_t Du = (uint32_t)D, NBu = (uint32_t)NB;
    const uint32_t D1 = Du < NBu ? Du : NBu, n2 = NBu > Du ? NBu - Du : 0u;
    const uint32_t b0 = (Du > NBu ? Du : NBu) - Du;
    const int slog = a.nslot_log;
    auto decode = [&](uint32_t r) {
        P2Item q;
        uint32_t b;
        if (r < D1 * TA) {
            q.ph = 0;
            b = r / TA;
            r -= b * TA;
        } else if ((r -= D1 * TA) < n2 * (TA + TB)) {
            const uint32_t s = r / (TA + TB);
            r -= s * (TA + TB);
            if (r < TA) {
                q.ph = 0;
                b = s + Du;
            } else {
                q.ph = 1;
                b = s;
                r -= TA;
            }
        } else {
            r -= n2 * (TA + TB);
            q.ph = 1;
            b = b0 + r / TB;
            r -= (b - b0) * TB;
        }
        q.b = b;
        q.tile = (int)r;
        q.slot = (int)(b & ((1u << slog) - 1u));
        const unsigned epoch = b >> slog;
        if (q.ph == 0) {   // the slot's previous block fully read
            q.dep = epoch > 0 ? doneB + q.slot : nullptr;
            q.target = (unsigned)TB * epoch;
        } else {           // this block's first phase fully written
            q.dep = doneA + q.slot;
            q.target = (unsigned)TA * (epoch + 1);
        }
        return q;
    };

    __shared__ int s_ok[2];
    // the next tile's source, written by thread 0 in mid(): kind 0 none
    // (not loaded ahead), 1 planes (the super-group's source), 2 scratch pairs
    __shared__ const char *s_src[2];
    __shared__ uint32_t s_src_stride;
    __shared__ int s_src_kind, s_src_rows_log;
    const uint32_t lb = (uint32_t)__cvta_generic_to_shared(smem_raw);
    constexpr int LBP = Sh::LB_PLANE;

    // the two groups' tile geometry (see the comment above the kernel)
    struct Geom {
        size_t so, xo;
        uint32_t xs, cc;
    };
    auto geom = [&](bool first_group, uint32_t tile, uint32_t J0) {
        Geom g;
        if (first_group) {
            const uint32_t E2 = tile;
            g.xo = J0 + (size_t)E2 * NJ;
            g.xs = NJ << L2;
            g.so = SZ ? ((size_t)E2 << L1) : (((size_t)E2 << L1) * TJ);
            g.cc = J0 & ((1u << S) - 1u);
        } else {
            const uint32_t u = tile;
            if constexpr (SZ) {
                constexpr int CPT = (1 << L1) / TJ;   // tiles per column
                const uint32_t jl = u / CPT, o0 = (u % CPT) * TJ;
                g.so = ((size_t)jl << L) + o0;
                g.xo = ((size_t)(J0 + jl) << L) + o0;
                g.xs = 1u << L1;
                g.cc = o0;
            } else {
                g.so = (size_t)u * TJ;
                const uint32_t jm = J0 & ((1u << S) - 1u);
                g.xo = (((size_t)(J0 >> S)) << (S + L)) + jm + ((size_t)u << S);
                g.xs = 1u << (S + L1);
                g.cc = jm + (u << S);
            }
        }
        return g;
    };
    // compile-time scratch strides of the two groups (pairs)
    constexpr uint32_t SS1 = SZ ? (1u << L) : (uint32_t)TJ;
    constexpr uint32_t SS2 = SZ ? (1u << L1) : ((uint32_t)TJ << L1);
    // the source tile of scheduled item q as the landing-buffer copies see it;
    // kind 0: the S = 0 DIF group's row-side source (loaded by the tile itself)
    struct Src {
        const char *p0, *p1;
        uint32_t stride;
        int kind, rows_log;
    };
    auto source = [&](const P2Item &q) {
        Src r;
        const int64_t row = q.b >> (m - L - LTJ);
        const uint32_t J0 = ((uint32_t)q.b & (nbr - 1u)) * TJ;
        const bool fg = (q.ph == 0) != DIF;
        const Geom g = geom(fg, (uint32_t)q.tile, J0);
        r.rows_log = fg ? L1 : L2;
        if (q.ph == 0) {   // the super-group's source planes
            r.kind = 1;
            r.p0 = (const char *)((const T *)a.x0 + row * a.in_stride + g.xo);
            r.p1 = (const char *)((const T *)a.x1 + row * a.in_stride + g.xo);
            r.stride = g.xs * (uint32_t)sizeof(T);
        } else {           // the block scratch
            r.kind = (DIF && SZ) ? 0 : 2;
            r.p0 = (const char *)((const vec2_t<T> *)a.s0 + q.slot * slot_elems + g.so);
            r.p1 = nullptr;
            r.stride = (fg ? SS1 : SS2) * 2u * (uint32_t)sizeof(T);
        }
        return r;
    };

    // tickets are taken two tiles ahead: s_item[it & 1] is this tile's,
    // s_item[(it + 1) & 1] the next one's (its dependency is polled at the top
    // of this tile and its source loaded ahead from px()), and the ticket
    // after that is requested at the top and stored at the end of this tile
    if (tid == 0) {
        s_item[0] = atomicAdd(a.ctr, 1u);
        s_item[1] = atomicAdd(a.ctr, 1u);
        s_ok[0] = 0;
        s_src_kind = 0;
    }
    __syncthreads();
    for (int it = 0;; ++it) {
        const uint32_t g = s_item[it & 1];
        if (g >= total) return;
        const bool ok = s_ok[it & 1] != 0;
        const bool loaded = s_src_kind != 0;   // this tile's source copies are in flight (or landed)
        const P2Item q = decode(g);
        unsigned nn = 0, polled = 0, want = 0;
        bool nodep = true;
        if (tid == 0) {
            nn = atomicAdd(a.ctr, 1u);
            const uint32_t gn = s_item[(it + 1) & 1];
            if (gn < total) {
                const P2Item n = decode(gn);
                nodep = n.dep == nullptr;
                if (!nodep) {
                    polled = p2_ld_relaxed(n.dep);   // consumed in mid()
                    want = n.target;
                }
            }
            if (!ok && q.dep)   // the look-ahead poll did not see this tile's dependency satisfied
                while (p2_ld_relaxed(q.dep) < q.target) __nanosleep(64);
        }
        if (!ok) __syncthreads();
        const Src cur = source(q);
        if (!loaded && cur.kind != 0)
            p2_issue_tile<Sh::NT, LBP>(lb, cur.kind == 2, cur.p0, cur.p1, cur.stride, cur.rows_log, tid);

        // look-ahead: is the next tile's dependency satisfied?  If so (or if it
        // reads the super-group's source, which nothing writes), describe its
        // source for px()
        auto mid = [&]() {
            if (tid == 0) {
                int kind = 0;
                const bool okn = nodep || polled >= want;
                const uint32_t gn = s_item[(it + 1) & 1];
                if (gn < total && !(a.flags & P2_NOPIPE)) {
                    const P2Item n = decode(gn);
                    if (n.ph == 0 || okn) {
                        const Src sn = source(n);
                        kind = sn.kind;
                        s_src[0] = sn.p0;
                        s_src[1] = sn.p1;
                        s_src_stride = sn.stride;
                        s_src_rows_log = sn.rows_log;
                    }
                }
                s_src_kind = kind;
                s_ok[(it + 1) & 1] = okn;
            }
        };
        auto px = [&]() {
            const int kind = s_src_kind;
            if (kind != 0)
                p2_issue_tile<Sh::NT, LBP>(lb, kind == 2, s_src[0], s_src[1], s_src_stride, s_src_rows_log, tid);
        };

        const int64_t row = q.b >> (m - L - LTJ);
        const uint32_t J0 = ((uint32_t)q.b & (nbr - 1u)) * TJ;
        vec2_t<T> *sc = (vec2_t<T> *)a.s0 + q.slot * slot_elems;
        const bool first_group = (q.ph == 0) != DIF;   // group (S, L1)?
        const Geom gm = geom(first_group, (uint32_t)q.tile, J0);
        if (first_group) {
            if constexpr (!DIF) {
                p2_tile<T, L1, false, SZ, false, true, SS1, true>(nullptr, nullptr, 0u, nullptr, nullptr, 0u, sc + gm.so,
                                                                  S, gm.cc, a, smem_raw, mid, px);
            } else {
                T *yr = (T *)a.y0 + row * a.out_stride + gm.xo, *yi = (T *)a.y1 + row * a.out_stride + gm.xo;
                p2_tile<T, L1, true, SZ, true, false, SS1, !SZ>(nullptr, nullptr, 0u, yr, yi, gm.xs, sc + gm.so, S,
                                                                gm.cc, a, smem_raw, mid, px);
            }
        } else {
            if constexpr (!DIF) {
                T *yr = (T *)a.y0 + row * a.out_stride + gm.xo, *yi = (T *)a.y1 + row * a.out_stride + gm.xo;
                p2_tile<T, L2, false, false, true, false, SS2, true>(nullptr, nullptr, 0u, yr, yi, gm.xs, sc + gm.so,
                                                                     S + L1, gm.cc, a, smem_raw, mid, px);
            } else {
                p2_tile<T, L2, true, false, false, true, SS2, true>(nullptr, nullptr, 0u, nullptr, nullptr, 0u,
                                                                    sc + gm.so, S + L1, gm.cc, a, smem_raw, mid, px);
            }
        }
        if (tid == 0) s_item[it & 1] = nn;   // the ticket of tile it + 2
        __syncthreads();   // every thread's stores of this tile issued; shared reads done
        if (tid == 0) p2_signal(a.ctr + 1 + (q.ph == 0 ? 0 : nslot) + q.slot);   // doneA / doneB
    }
}

}  // namespace sfft
