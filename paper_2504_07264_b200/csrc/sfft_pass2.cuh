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

// flags: publish a tile's completion after the NEXT tile's loads are issued
// (the release fence then waits next to loads every warp waits for, instead
// of holding warp 0 back at the tile boundary); prefetch the next tile's
// HBM-side source runs into L2 once its ticket is known (one 128-byte line
// per thread with prefetch.global.L2; P2_PREFETCH_BULK: cp.async.bulk.prefetch,
// which the uniform datapath serialises lane by lane -- measured, not used).
constexpr int P2_DEFER = 1, P2_PREFETCH = 2, P2_PREFETCH_BULK = 4;

template <typename T> struct P2TJ { static constexpr int value = sizeof(T) == 4 ? 32 : 16; };

// 8 threads per column (R = 2^(Lg-3) values each), TJ columns per tile
template <typename T, int L1, int L2>
struct P2Shape {
    static constexpr int TJ = P2TJ<T>::value;
    static constexpr int P = 8;
    static constexpr int NT = TJ * P;
    static constexpr int RS = TJ + 1;
    static constexpr int LMAX = 7;   // p2_tile places the column factors after a 2^7-point tile
    static constexpr int smem_bytes() { return (1 << LMAX) * RS * 2 * (int)sizeof(T) + LMAX * TJ * 2 * (int)sizeof(T); }
};

template <typename T, int L1, int L2>
struct P2MinBlocks {
    static constexpr int NT = P2Shape<T, L1, L2>::NT;
    static constexpr int value = sizeof(T) == 4 ? 1024 / NT : 0;
};

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
// Scheduler hooks, each run once per tile: `ldh()` after the tile's global
// loads (and column-factor lookups) are issued, `mid()` after the first
// register pass (the look-ahead for the next tile, off the tile's critical
// path), `px()` after the CTA barrier that follows `mid()`.
// The scratch side (IN_SCR: source, OUT_SCR: destination) is `scr`, pairs
// with the compile-time element stride SSTR; the plane pointers and the
// runtime stride of that side are unused.
template <typename T, int L, bool DIF, bool S0G, bool IN_SCR, bool OUT_SCR, uint32_t SSTR, typename Ldh,
          typename Mid, typename Px>
__device__ __forceinline__ void p2_tile(const T *ir, const T *ii, uint32_t istr, T *orr, T *oi, uint32_t ostr,
                                        vec2_t<T> *scr, int S, uint32_t c0, const Pass2Args &a,
                                        unsigned char *smem_raw, const Ldh &ldh, const Mid &mid, const Px &px)
{
    constexpr int TJ = P2TJ<T>::value, P = 8, SUB = 1 << L, LR = L - 3, R = 1 << LR, NT = TJ * P;
    constexpr int RS = TJ + 1, NPI = (L + LR - 1) / LR;
    static_assert(L >= 5 && L <= 7, "fused pair groups are 2^5..2^7 points");
    using V = vec2_t<T>;
    V *sx = reinterpret_cast<V *>(smem_raw);
    constexpr int LMAX = 7;
    V *cs = sx + (1 << LMAX) * RS;   // [L][TJ] column factors (after the largest tile)
    const int tid = threadIdx.x;
    const int jl = tid % TJ, t = tid / TJ;
    const uint32_t c = S0G ? 0u : c0 + (uint32_t)jl;
    const auto tw = make_p2_tw<T, S0G>(a);
    using I = typename PassTw<T, S0G>::type::index_t;
    const bool scale_out = !OUT_SCR && a.scale_out != 0;   // only the super-group's destination
    const T scale = (T)a.scale;
    constexpr bool CST = FactorTw<T>::value && !S0G;
    const uint32_t is_b = istr * (uint32_t)sizeof(T), os_b = ostr * (uint32_t)sizeof(T);

    // source element at `k` strides / `off` elements from the thread's base
    // (planes pr, pi or scratch pairs ps); destination likewise
    auto get_k = [&](const T *pr, const T *pi, const V *ps, uint32_t k) {
        V w;
        if constexpr (IN_SCR) {
            w = __ldcg(ps + k * SSTR);   // written by other SMs during this kernel: L2, never L1
        } else {
            w.x = ld_stream(at_stride(pr, is_b, k));
            w.y = ld_stream(at_stride(pi, is_b, k));
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
            ldh();
            __syncthreads();
        } else {
            ldh();
        }
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
        const T *in_r = IN_SCR ? nullptr : ir + jl + (size_t)t * istr;
        const T *in_i = IN_SCR ? nullptr : ii + jl + (size_t)t * istr;
        const V *in_s = IN_SCR ? scr + jl + t * SSTR : nullptr;
        static_for<0, NPI>([&](auto PPC) {
            constexpr int pp = decltype(PPC)::value;
            constexpr int sp = pp * LR, KP = cmin(LR, L - sp), RP = 1 << KP, U = R / RP, nsp = 1 << sp;
            constexpr bool last = pp == NPI - 1;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int jp = t + P * u;
#pragma unroll
                for (int r = 0; r < RP; ++r) {
                    if constexpr (pp == 0) {
                        const uint32_t k = (uint32_t)(P * u + r * (SUB / RP));
                        v[u * RP + r] = get_k(in_r, in_i, in_s, k);
                    } else {
                        v[u * RP + r] = sx[(jp + r * (SUB / RP)) * RS + jl];
                    }
                }
            }
            if constexpr (pp == 0) stage_columns();
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
            ldh();
#pragma unroll
            for (int kk = 0; kk < R; ++kk) {
                const int k = tid + kk * NT, jj = k >> L, o = k & (SUB - 1);
                sx[o * RS + jj] = v[kk];
            }
            __syncthreads();
        }
        const T *in_r = IN_SCR ? nullptr : ir + jl, *in_i = IN_SCR ? nullptr : ii + jl;
        const V *in_s = IN_SCR ? scr + jl : nullptr;
        static_for<0, NPI>([&](auto QC) {
            constexpr int pp = NPI - 1 - decltype(QC)::value;
            constexpr int sp = pp * LR, KP = cmin(LR, L - sp), RP = 1 << KP, U = R / RP, nsp = 1 << sp;
            constexpr bool first = pp == NPI - 1;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int jp = t + P * u;
                const int base = (jp >> sp) * nsp * RP + (jp & (nsp - 1));
#pragma unroll
                for (int f = 0; f < RP; ++f) {
                    const int d = u * RP + brev(f, KP);
                    if constexpr (first && !S0G) {
                        const uint32_t k = (uint32_t)(nsp * f);
                        if constexpr (IN_SCR) {
                            v[d] = get_k(nullptr, nullptr, in_s + (uint32_t)base * SSTR, k);
                        } else {
                            const T *pr = in_r + (size_t)base * istr, *pi = in_i + (size_t)base * istr;
                            v[d] = get_k(pr, pi, nullptr, k);
                        }
                    } else {
                        v[d] = sx[(base + nsp * f) * RS + jl];
                    }
                }
            }
            if constexpr (first && !S0G) stage_columns();
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

// L2 prefetch of one contiguous run (no destination, nothing to wait for)
__device__ __forceinline__ void p2_prefetch_run(const void *src, uint32_t bytes)
{
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
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
    __shared__ const char *s_pf[2];    // the next tile's HBM-side source runs (P2_PREFETCH)
    __shared__ uint32_t s_pf_stride;
    __shared__ int s_pf_rows;

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

    int pend = 0;   // thread 0: index in ctr[] of a finished tile's counter, not yet published (P2_DEFER)
    auto flush = [&]() {
        if (pend) {
            p2_signal(a.ctr + pend);
            pend = 0;
        }
    };
    if (tid == 0) {
        s_item[0] = atomicAdd(a.ctr, 1u);
        s_ok[0] = 0;
    }
    __syncthreads();
    for (int it = 0;; ++it) {
        const uint32_t g = s_item[it & 1];
        if (g >= total) {
            if (tid == 0) flush();
            return;
        }
        const bool ok = s_ok[it & 1] != 0;
        const P2Item q = decode(g);
        // the next ticket: issued now, consumed after the first register pass
        unsigned nxt = 0;
        if (tid == 0) nxt = atomicAdd(a.ctr, 1u);
        if (!ok) {   // the look-ahead poll did not see the dependency satisfied
            if (tid == 0) {
                flush();   // what this CTA still owes may be what it is about to wait for
                if (q.dep)
                    while (p2_ld_relaxed(q.dep) < q.target) __nanosleep(64);
            }
            __syncthreads();
        }
        auto ldh = [&]() {
            if (tid == 0) flush();
        };
        // look-ahead: decode the next ticket and poll its dependency once;
        // the poll's value is only needed at the end of this tile
        unsigned polled = 0, want = 0;
        bool nodep = true;
        auto mid = [&]() {
            if (tid == 0) {
                int pf_rows = 0;
                if (nxt < total) {
                    const P2Item n = decode(nxt);
                    nodep = n.dep == nullptr;
                    if (!nodep) {
                        polled = p2_ld_relaxed(n.dep);
                        want = n.target;
                    }
                    if ((a.flags & P2_PREFETCH) && n.ph == 0) {   // phase 0 reads the super-group's source planes
                        const int64_t nrow = n.b >> (m - L - LTJ);
                        const uint32_t nJ0 = ((uint32_t)n.b & (nbr - 1u)) * TJ;
                        const Geom ng = geom(!DIF, (uint32_t)n.tile, nJ0);
                        s_pf[0] = (const char *)((const T *)a.x0 + nrow * a.in_stride + ng.xo);
                        s_pf[1] = (const char *)((const T *)a.x1 + nrow * a.in_stride + ng.xo);
                        s_pf_stride = ng.xs * (uint32_t)sizeof(T);
                        pf_rows = 1 << (DIF ? L2 : L1);
                    }
                }
                if (a.flags & P2_PREFETCH) s_pf_rows = pf_rows;
            }
        };
        auto px = [&]() {
            if (a.flags & P2_PREFETCH) {
                const int rows = s_pf_rows;
                for (int k = tid; k < 2 * rows; k += Sh::NT) {
                    const int pl = k >= rows, e = k - pl * rows;
                    const char *run = s_pf[pl] + (size_t)e * s_pf_stride;   // one 128-byte line
                    if (a.flags & P2_PREFETCH_BULK)
                        p2_prefetch_run(run, TJ * (uint32_t)sizeof(T));
                    else
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(run) : "memory");
                }
            }
        };

        const int64_t row = q.b >> (m - L - LTJ);
        const uint32_t J0 = ((uint32_t)q.b & (nbr - 1u)) * TJ;
        vec2_t<T> *sc = (vec2_t<T> *)a.s0 + q.slot * slot_elems;
        const bool first_group = (q.ph == 0) != DIF;   // group (S, L1)?
        const Geom gm = geom(first_group, (uint32_t)q.tile, J0);
        // compile-time scratch strides of the two groups (see geom: g.ss)
        constexpr uint32_t SS1 = SZ ? (1u << L) : (uint32_t)TJ;
        constexpr uint32_t SS2 = SZ ? (1u << L1) : ((uint32_t)TJ << L1);
        if (first_group) {
            if constexpr (!DIF) {
                const T *xr = (const T *)a.x0 + row * a.in_stride + gm.xo, *xi = (const T *)a.x1 + row * a.in_stride + gm.xo;
                p2_tile<T, L1, false, SZ, false, true, SS1>(xr, xi, gm.xs, nullptr, nullptr, 0u, sc + gm.so, S, gm.cc,
                                                            a, smem_raw, ldh, mid, px);
            } else {
                T *yr = (T *)a.y0 + row * a.out_stride + gm.xo, *yi = (T *)a.y1 + row * a.out_stride + gm.xo;
                p2_tile<T, L1, true, SZ, true, false, SS1>(nullptr, nullptr, 0u, yr, yi, gm.xs, sc + gm.so, S, gm.cc,
                                                           a, smem_raw, ldh, mid, px);
            }
        } else {
            if constexpr (!DIF) {
                T *yr = (T *)a.y0 + row * a.out_stride + gm.xo, *yi = (T *)a.y1 + row * a.out_stride + gm.xo;
                p2_tile<T, L2, false, false, true, false, SS2>(nullptr, nullptr, 0u, yr, yi, gm.xs, sc + gm.so, S + L1,
                                                               gm.cc, a, smem_raw, ldh, mid, px);
            } else {
                const T *xr = (const T *)a.x0 + row * a.in_stride + gm.xo, *xi = (const T *)a.x1 + row * a.in_stride + gm.xo;
                p2_tile<T, L2, true, false, false, true, SS2>(xr, xi, gm.xs, nullptr, nullptr, 0u, sc + gm.so, S + L1,
                                                              gm.cc, a, smem_raw, ldh, mid, px);
            }
        }
        if (tid == 0) {
            s_item[(it + 1) & 1] = nxt;
            s_ok[(it + 1) & 1] = nodep || polled >= want;
        }
        __syncthreads();   // every thread's stores of this tile issued; shared reads done
        if (tid == 0) {
            const int c = 1 + (q.ph == 0 ? 0 : nslot) + q.slot;   // doneA / doneB
            if (a.flags & P2_DEFER)
                pend = c;   // published by flush(): after the next tile's loads, or before a wait / the exit
            else
                p2_signal(a.ctr + c);
        }
    }
}

}  // namespace sfft
