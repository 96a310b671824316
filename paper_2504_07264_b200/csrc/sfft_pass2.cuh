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
// Scratch layout of a block (columns jl < TJ = the block's sub-problems,
// E2 < 2^L2, o < 2^L1):
//   S > 0:  ((E2 << L1) + o) * TJ + jl   -- both sides 128-byte runs over jl
//   S = 0:  ((jl << L2) + E2 << L1) + o  -- the first group's outputs are rows
//           of 2^L1 per sub-problem (the S = 0 transpose); the second group
//           reads 128-byte runs over o
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
    void *s0, *s1;         // scratch ring planes: nslot blocks of TJ * 2^L elements
    unsigned *ctr;         // [0] ticket, [1 + slot] first-group tiles done, [1 + nslot + slot] second
    int64_t batch, in_stride, out_stride;
    int m, S;              // log2 N, stage offset of the super-group
    int nslot_log, lag;    // ring of 2^nslot_log block slots, second phase `lag` blocks behind
    int scale_out;         // multiply the destination by `scale` (the inverse's last launch)
    double scale;
    const void *tw;        // as PassArgs
    int tw_cat_top;
    const void *tw_top_tab;
    const double2 *coarse;
    int coarse_log;
    const double2 *fine;
};

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

template <bool SCR, typename T>
__device__ __forceinline__ T p2_ld(const T *p)
{
    if constexpr (SCR) return __ldcg(p);   // written by other SMs during this kernel: L2, never L1
    else return ld_stream(p);
}

template <bool SCR, typename T>
__device__ __forceinline__ void p2_st(T *p, T v)
{
    if constexpr (SCR) __stcg(p, v);      // the block scratch: default L2 policy, read back soon
    else st_stream(p, v);
}

// One tile: TJ columns of 2^L-point sub-problems of group (S, L), column jl's
// factor column c0 + jl (S > 0).  Column side: element e of column jl at
// base + jl + e * stride; row side (the S = 0 group: DIT destination, DIF
// source): element o of column jl at base + jl * stride + o.
// `mid()` runs once, after the first register pass (the scheduler's
// look-ahead for the next tile, off the tile's critical path).
template <typename T, int L, bool DIF, bool S0G, bool IN_SCR, bool OUT_SCR, typename Mid>
__device__ __forceinline__ void p2_tile(const T *ir, const T *ii, uint32_t istr, T *orr, T *oi, uint32_t ostr,
                                        int S, uint32_t c0, const Pass2Args &a, unsigned char *smem_raw,
                                        const Mid &mid)
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

    auto put = [&](T *pr, T *pi, V w) {
        if (scale_out) {
            w.x *= scale;
            w.y *= scale;
        }
        p2_st<OUT_SCR>(pr, w.x);
        p2_st<OUT_SCR>(pi, w.y);
    };
    auto stage_columns = [&]() {
        if constexpr (CST) {
            for (int k = tid; k < L * TJ; k += NT) {
                const int st = k / TJ, l = k - st * TJ;
                cs[k] = tw.get(S + 1 + st, (I)(c0 + (uint32_t)l));
            }
            __syncthreads();
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
        const T *in_r = ir + jl + (size_t)t * istr;
        const T *in_i = ii + jl + (size_t)t * istr;
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
                        v[u * RP + r].x = p2_ld<IN_SCR>(at_stride(in_r, is_b, k));
                        v[u * RP + r].y = p2_ld<IN_SCR>(at_stride(in_i, is_b, k));
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
            } else {
                T *out_r = orr + jl + (size_t)t * ostr;
                T *out_i = oi + jl + (size_t)t * ostr;
#pragma unroll
                for (int u = 0; u < U; ++u) {
#pragma unroll
                    for (int f = 0; f < RP; ++f) {
                        const uint32_t k = (uint32_t)(P * u + nsp * f);
                        put(at_stride(out_r, os_b, k), at_stride(out_i, os_b, k), v[u * RP + brev(f, KP)]);
                    }
                }
            }
        });
        if constexpr (S0G) {
            // row-side destination: smem [o][jj] -> rows of 2^L per column
#pragma unroll
            for (int kk = 0; kk < R; ++kk) {
                const int k = tid + kk * NT, jj = k >> L, o = k & (SUB - 1);
                const size_t off = (size_t)jj * ostr + o;
                put(orr + off, oi + off, sx[o * RS + jj]);
            }
        }
    } else {
        if constexpr (S0G) {
            // row-side source (all R loads first, then the shared stores)
#pragma unroll
            for (int kk = 0; kk < R; ++kk) {
                const int k = tid + kk * NT, jj = k >> L, o = k & (SUB - 1);
                const size_t off = (size_t)jj * istr + o;
                v[kk].x = p2_ld<IN_SCR>(ir + off);
                v[kk].y = p2_ld<IN_SCR>(ii + off);
            }
#pragma unroll
            for (int kk = 0; kk < R; ++kk) {
                const int k = tid + kk * NT, jj = k >> L, o = k & (SUB - 1);
                sx[o * RS + jj] = v[kk];
            }
            __syncthreads();
        }
        const T *in_r = ir + jl, *in_i = ii + jl;
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
                        const T *pr = in_r + (size_t)base * istr, *pi = in_i + (size_t)base * istr;
                        const uint32_t k = (uint32_t)(nsp * f);
                        v[d].x = p2_ld<IN_SCR>(at_stride(pr, is_b, k));
                        v[d].y = p2_ld<IN_SCR>(at_stride(pi, is_b, k));
                    } else {
                        v[d] = sx[(base + nsp * f) * RS + jl];
                    }
                }
            }
            if constexpr (first) stage_columns();
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
            } else {
                T *out_r = orr + jl + (size_t)t * ostr;
                T *out_i = oi + jl + (size_t)t * ostr;
#pragma unroll
                for (int u = 0; u < U; ++u) {
#pragma unroll
                    for (int r = 0; r < RP; ++r) {
                        const uint32_t k = (uint32_t)(P * u + r * (SUB / RP));
                        put(at_stride(out_r, os_b, k), at_stride(out_i, os_b, k), v[u * RP + r]);
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
    if (tid == 0) {
        s_item[0] = atomicAdd(a.ctr, 1u);
        s_ok[0] = 0;
    }
    __syncthreads();
    for (int it = 0;; ++it) {
        const uint32_t g = s_item[it & 1];
        if (g >= total) return;
        const bool ok = s_ok[it & 1] != 0;
        const P2Item q = decode(g);
        // the next ticket: issued now, consumed after the first register pass
        unsigned nxt = 0;
        if (tid == 0) nxt = atomicAdd(a.ctr, 1u);
        if (!ok) {   // the look-ahead poll did not see the dependency satisfied
            if (tid == 0 && q.dep)
                while (p2_ld_relaxed(q.dep) < q.target) __nanosleep(64);
            __syncthreads();
        }
        // look-ahead: decode the next ticket and poll its dependency once;
        // the poll's value is only needed at the end of this tile
        unsigned polled = 0, want = 0;
        bool nodep = true;
        auto mid = [&]() {
            if (tid == 0 && nxt < total) {
                const P2Item n = decode(nxt);
                nodep = n.dep == nullptr;
                if (!nodep) {
                    polled = p2_ld_relaxed(n.dep);
                    want = n.target;
                }
            }
        };

        const int64_t row = q.b >> (m - L - LTJ);
        const uint32_t J0 = ((uint32_t)q.b & (nbr - 1u)) * TJ;
        T *sr = (T *)a.s0 + q.slot * slot_elems, *si = (T *)a.s1 + q.slot * slot_elems;
        const bool first_group = (q.ph == 0) != DIF;   // group (S, L1)?
        if (first_group) {
            const uint32_t E2 = (uint32_t)q.tile;
            const size_t xo = J0 + (size_t)E2 * NJ;
            const uint32_t xs = NJ << L2;
            const size_t so = SZ ? ((size_t)E2 << L1) : (((size_t)E2 << L1) * TJ);
            const uint32_t ss = SZ ? (1u << L) : (uint32_t)TJ;
            const uint32_t cc = J0 & ((1u << S) - 1u);
            if constexpr (!DIF) {
                const T *xr = (const T *)a.x0 + row * a.in_stride + xo, *xi = (const T *)a.x1 + row * a.in_stride + xo;
                p2_tile<T, L1, false, SZ, false, true>(xr, xi, xs, sr + so, si + so, ss, S, cc, a, smem_raw, mid);
            } else {
                T *yr = (T *)a.y0 + row * a.out_stride + xo, *yi = (T *)a.y1 + row * a.out_stride + xo;
                p2_tile<T, L1, true, SZ, true, false>(sr + so, si + so, ss, yr, yi, xs, S, cc, a, smem_raw, mid);
            }
        } else {
            const uint32_t u = (uint32_t)q.tile;
            size_t so, xo;
            uint32_t ss, xs, cc;
            if constexpr (SZ) {
                constexpr int CPT = (1 << L1) / TJ;   // tiles per column
                const uint32_t jl = u / CPT, o0 = (u % CPT) * TJ;
                so = ((size_t)jl << L) + o0;
                ss = 1u << L1;
                xo = ((size_t)(J0 + jl) << L) + o0;
                xs = 1u << L1;
                cc = o0;
            } else {
                so = (size_t)u * TJ;
                ss = (uint32_t)TJ << L1;
                const uint32_t jm = J0 & ((1u << S) - 1u);
                xo = (((size_t)(J0 >> S)) << (S + L)) + jm + ((size_t)u << S);
                xs = 1u << (S + L1);
                cc = jm + (u << S);
            }
            if constexpr (!DIF) {
                T *yr = (T *)a.y0 + row * a.out_stride + xo, *yi = (T *)a.y1 + row * a.out_stride + xo;
                p2_tile<T, L2, false, false, true, false>(sr + so, si + so, ss, yr, yi, xs, S + L1, cc, a, smem_raw,
                                                          mid);
            } else {
                const T *xr = (const T *)a.x0 + row * a.in_stride + xo, *xi = (const T *)a.x1 + row * a.in_stride + xo;
                p2_tile<T, L2, true, false, false, true>(xr, xi, xs, sr + so, si + so, ss, S + L1, cc, a, smem_raw,
                                                         mid);
            }
        }
        if (tid == 0) {
            s_item[(it + 1) & 1] = nxt;
            s_ok[(it + 1) & 1] = nodep || polled >= want;
        }
        __syncthreads();   // every thread's stores of this tile issued; shared reads done
        if (tid == 0) p2_signal(q.ph == 0 ? doneA + q.slot : doneB + q.slot);
    }
}

}  // namespace sfft
