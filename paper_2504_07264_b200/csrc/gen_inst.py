"""Generate the kernel instantiation units sfft_inst_*.cu.

Every fused (log2 N, log2 radix) combination the tuner may pick is
instantiated for planar DIT/DIF; the interleaved variants only for the
default radix (sfft_launch.h).  Run by the Makefile; the outputs are build
artefacts.
"""

import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))

# default register radix (log2) per log2 N; see DESIGN.md sec. 4 for why
DEFAULT_LR = {
    "f32": {0: 0, 1: 1, 2: 2, 3: 3, 4: 2, 5: 2, 6: 3, 7: 3, 8: 4, 9: 4, 10: 4, 11: 4, 12: 4},
    "f64": {0: 0, 1: 1, 2: 2, 3: 3, 4: 1, 5: 2, 6: 2, 7: 3, 8: 3, 9: 3, 10: 3, 11: 3, 12: 4},
}
# kernel=auto choice per size, from tools/tune.py on a B200 (profiles/r01_tune6.txt,
# re-swept after the radix-32 CTA change: profiles/r01l_tune_{dit,dif}.txt):
# ("tma" | "ldg", log2 radix, fetch base factors up front (fp32 only)
#  [, (TMA log2 radix below, batch) -- a batch-size switch: fp64 N = 1024's
#  warp-per-signal kernel (radix 32) wins from 2^16 rows, the radix-8 TMA
#  kernel below (fixed per-launch costs; profiles/r02q_f64_n1024_batch_sweep_ring.txt);
#  radix 0 = the LDG kernel at its default radix])
AUTO = {
    "f32": {4: ("ldg", 2, False), 5: ("tma", 3, False), 6: ("tma", 3, False), 7: ("tma", 4, False),
            8: ("ldg", 3, False), 9: ("ldg", 3, False), 10: ("ldg", 5, False), 11: ("ldg", 4, False),
            12: ("tma", 6, False, (0, 1 << 13))},
    "f64": {4: ("tma", 2, False), 5: ("ldg", 2, False), 6: ("ldg", 2, False), 7: ("ldg", 3, False),
            8: ("ldg", 3, False), 9: ("ldg", 3, False), 10: ("tma", 5, False, (3, 1 << 16)), 11: ("ldg", 3, False),
            12: ("ldg", 3, False)},
}
RADIX_CHOICES = {"f32": [1, 2, 3, 4, 5], "f64": [1, 2, 3, 4, 5]}


def fused_nt(logn, lr):
    """Threads per CTA of the LDG fused kernel (sfft_fused.cuh FusedShape::NT):
    one signal's P = 2^(logn-lr) threads, at least 256 -- 128 for radix 32,
    whose 64-value register files would leave one 256-thread CTA per SM."""
    return max(1 << (logn - lr), 128 if lr >= 5 else 256)
CTYPE = {"f32": "float", "f64": "double"}
PASS_L = [4, 5, 6, 7, 8, 9, 10]

# TMA kernel configs: (log2 radix, threads requested, input stages, output buffers
# [, min resident CTAs for __launch_bounds__]); OB = 0 stores the last pass
# straight to global memory.  The first entry per size is the default.  Keys
# (dtype, log2N, log2 radix) are unique.
TMA_CONFIGS = {
    "f32": {
        5: [(3, 256, 3, 2)],
        6: [(3, 128, 2, 2), (2, 256, 3, 2)],   # settled power state: 128 threads x 2 stages 0.176 vs 0.190 ms for 256 x 3 (profiles/r02ay_*)
        7: [(3, 256, 3, 2), (4, 128, 3, 2)],
        8: [(3, 256, 3, 2), (4, 128, 3, 2)],
        9: [(3, 256, 3, 2), (4, 128, 3, 2)],
        10: [(4, 128, 3, 2), (3, 256, 3, 2), (5, 64, 3, 2)],
        11: [(4, 128, 3, 2), (3, 256, 3, 2)],
        12: [(4, 256, 2, 1), (3, 512, 2, 1)],
    },
    "f64": {
        4: [(2, 256, 3, 2)],
        5: [(3, 128, 3, 2)],
        6: [(3, 128, 3, 2)],
        7: [(3, 128, 3, 2), (4, 64, 3, 2)],
        8: [(3, 128, 3, 2), (4, 64, 3, 2)],
        9: [(3, 128, 3, 2)],
        10: [(3, 128, 2, 0, 4), (4, 128, 2, 1)],
        11: [(4, 128, 2, 1)],
    },
}
# warp-per-signal bulk-copy kernel (sfft_tma_warp.cuh, N = 1024, radix 32):
# (warps per CTA, second-pass factor stages held in registers, factors in
# tensor memory instead, shared slot ring, ring slots beyond one per warp);
# selected as the TMA family's radix 2^5 for these sizes.  10 warps sharing a
# ring of 12 slots (192 KiB).  Timed right after an idle gap (boosted 1.9 GHz
# SM clock) 9 warps + 11 slots measured best (profiles/r02p_ab_slot_ring.txt,
# r02q_ab_ring_depth.txt); in the settled power state (1.4-1.5 GHz under the
# 1000 W cap, the state bench.py times since r02al) the tenth warp is worth
# 3-4%: 1.370 vs 1.421 ms DIT, 1.379 vs 1.420 ms DIF, 11 / 12 warps, an
# L2 prefetch-ahead and a 13-slot ring all slower (profiles/r02ao_*, r02ap_*)
TMAW_CONFIGS = {"f64": {10: (10, 3, 1, 1, 2, 1)}, "f32": {12: (8, 0, 0, 1, 2, 2)}}
# fp32 N = 4096: two warps per signal, radix 64, 8 warps / 6 slots per SM,
# factors formed from per-thread base factors (TMEM factors measured no
# better for fp32: profiles/r02u_ab_cfg4_group_kernel_tmem.txt); +2% over the
# LDG radix-16 kernel (profiles/r02t_*, r02u_*)
_tw = os.environ.get("SFFT_TMAW")          # developer override "dt:logn:warps,hk,tm,ring,xs,wps[,pf]"
if _tw:
    _dt, _m, _cfg = _tw.split(":")
    TMAW_CONFIGS[_dt][int(_m)] = tuple(int(v) for v in _cfg.split(","))
PASS_LR = {"f32": 4, "f64": 4}
if os.environ.get("SFFT_PASS_LR"):          # developer override for A/B builds
    PASS_LR = {k: int(os.environ["SFFT_PASS_LR"]) for k in PASS_LR}

# developer override for A/B builds: SFFT_TMA_OVERRIDE="f32:6:3,128,4,2" replaces
# the default (first) TMA config of that size
_ov = os.environ.get("SFFT_TMA_OVERRIDE")
if _ov:
    _dt, _m, _cfg = _ov.split(":")
    TMA_CONFIGS[_dt][int(_m)][0] = tuple(int(v) for v in _cfg.split(","))
# developer override of the kernel=auto table: SFFT_AUTO_OVERRIDE="f64:10:tma,3"
_ao = os.environ.get("SFFT_AUTO_OVERRIDE")
if _ao:
    for _item in _ao.split(";"):
        _dt, _m, _cfg = _item.split(":")
        _fam, _lr = _cfg.split(",")
        AUTO[_dt][int(_m)] = (_fam, int(_lr), False)


def fused_unit(dt, algo):
    T = CTYPE[dt]
    dif = "true" if algo == "dif" else "false"
    out = [
        "// GENERATED by gen_inst.py -- do not edit",
        "#include <atomic>",
        '#include "sfft_fused.cuh"',
        '#include "sfft_launch.h"',
        "namespace sfft {",
        "template <int LOGN, int LR, bool IL, bool PRE>",
        f"static cudaError_t launch_{algo}_{dt}(const FusedArgs &a, cudaStream_t st)",
        "{",
        "    using Sh = FusedShape<LOGN, LR>;",
        f"    auto k = fused_kernel_for<{T}, LOGN, LR, {dif}, IL, PRE>();",
        f"    constexpr int smem = Sh::template smem_bytes<{T}>();",
        "    if (smem > 48 * 1024) {",
        "        // per-device 'attribute set' bits; concurrent first calls may both set",
        "        // it (idempotent), none launches before its own call returned",
        "        static std::atomic<unsigned> done_mask{0u};",
        "        int dev = 0;",
        "        cudaGetDevice(&dev);",
        "        if (!(done_mask.load(std::memory_order_acquire) & (1u << (dev & 31)))) {",
        "            cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);",
        "            if (e != cudaSuccess) return e;",
        "            done_mask.fetch_or(1u << (dev & 31), std::memory_order_release);",
        "        }",
        "    }",
        "    const int64_t grid = (a.batch + Sh::S - 1) / Sh::S;",
        "    if (grid > 0x7fffffffLL) return cudaErrorInvalidConfiguration;   // caller splits larger batches",
        "    k<<<(unsigned)grid, Sh::NT, smem, st>>>(a);",
        "    count_launch();",
        "    return cudaGetLastError();",
        "}",
    ]
    entries = []
    for logn in range(0, 13):
        lrs = sorted({min(lr, logn) for lr in RADIX_CHOICES[dt]}) if logn else [0]
        lrs = [lr for lr in lrs if (1 << (logn - lr)) <= 1024]   # <= 1024 threads per signal
        for lr in lrs:
            il_too = lr == min(DEFAULT_LR[dt][logn], logn)
            entries.append((logn, lr, il_too))
    out.append(f"FusedLaunchFn fused_{algo}_{dt}_table(int logn, int lr, bool il, bool pre)")
    out.append("{")
    for logn, lr, il_too in entries:
        out.append(f"    if (logn == {logn} && lr == {lr}) {{")
        if il_too:
            out.append(f"        if (il) return [](const FusedArgs &a, bool, bool, cudaStream_t st) {{ return launch_{algo}_{dt}<{logn}, {lr}, true, false>(a, st); }};")
        else:
            out.append("        if (il) return nullptr;")
        if dt == "f32" and lr >= 2 and logn >= 5:
            out.append(f"        if (pre) return [](const FusedArgs &a, bool, bool, cudaStream_t st) {{ return launch_{algo}_{dt}<{logn}, {lr}, false, true>(a, st); }};")
        out.append(f"        return [](const FusedArgs &a, bool, bool, cudaStream_t st) {{ return launch_{algo}_{dt}<{logn}, {lr}, false, false>(a, st); }};")
        out.append("    }")
    out.append("    return nullptr;")
    out.append("}")
    out.append("}  // namespace sfft")
    return "\n".join(out) + "\n"


def pass_unit(dt):
    T = CTYPE[dt]
    lr = PASS_LR[dt]
    # (dif, il_in, il_out, s0, dist) combinations a schedule can produce
    combos = [(False, True, False, True, False), (False, False, False, True, False),
              (False, False, True, False, False), (False, False, False, False, False),
              (True, True, False, False, False), (True, False, False, False, False),
              (True, False, True, True, False), (True, False, False, True, False),
              (False, False, False, True, True), (False, False, False, False, True)]
    out = [
        "// GENERATED by gen_inst.py -- do not edit",
        "#include <atomic>",
        '#include "sfft_pass.cuh"',
        '#include "sfft_launch.h"',
        "namespace sfft {",
        "template <int L, bool DIF, bool ILI, bool ILO, bool S0, bool DIST>",
        f"static cudaError_t launch_pass_{dt}(const PassArgs &a, int64_t grid, cudaStream_t st)",
        "{",
        f"    using Sh = PassShape<{T}, L, {lr}>;",
        f"    auto k = sfft_pass_kernel<{T}, L, {lr}, DIF, ILI, ILO, S0, DIST>;",
        "    constexpr int smem = Sh::smem_bytes();",
        "    if (smem > 48 * 1024) {",
        "        // per-device 'attribute set' bits; concurrent first calls may both set",
        "        // it (idempotent), none launches before its own call returned",
        "        static std::atomic<unsigned> done_mask{0u};",
        "        int dev = 0;",
        "        cudaGetDevice(&dev);",
        "        if (!(done_mask.load(std::memory_order_acquire) & (1u << (dev & 31)))) {",
        "            cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);",
        "            if (e != cudaSuccess) return e;",
        "            done_mask.fetch_or(1u << (dev & 31), std::memory_order_release);",
        "        }",
        "    }",
        "    k<<<(unsigned)grid, Sh::NT, smem, st>>>(a);",
        "    count_launch();",
        "    return cudaGetLastError();",
        "}",
        "template <int L>",
        f"static cudaError_t dispatch_pass_{dt}(const PassArgs &a, bool dif, bool ili, bool ilo, int64_t grid, cudaStream_t st)",
        "{",
        "    const bool s0 = a.S == 0, dist = a.jb > 0;",
    ]
    for (dif, ili, ilo, s0, dst) in combos:
        b = lambda v: "true" if v else "false"
        out.append(f"    if (dif == {b(dif)} && ili == {b(ili)} && ilo == {b(ilo)} && s0 == {b(s0)} && dist == {b(dst)}) "
                   f"return launch_pass_{dt}<L, {b(dif)}, {b(ili)}, {b(ilo)}, {b(s0)}, {b(dst)}>(a, grid, st);")
    out += ["    return cudaErrorInvalidValue;", "}",
            f"PassLaunchFn pass_launcher_{dt}(int L)", "{"]
    for L in PASS_L:
        out.append(f"    if (L == {L}) return dispatch_pass_{dt}<{L}>;")
    out += ["    return nullptr;", "}", "}  // namespace sfft"]
    return "\n".join(out) + "\n"


# L2-fused group pairs (sfft_pass2.cuh): (L1, L2) of the balanced 4-group
# splits of m = 20..28 (5,5,5,5 .. 7,7,7,7)
PASS2_PAIRS = [(5, 5), (6, 5), (6, 6), (7, 6), (7, 7)]


def pass2_unit(dt):
    T = CTYPE[dt]
    out = [
        "// GENERATED by gen_inst.py -- do not edit",
        "#include <atomic>",
        '#include "sfft_pass2.cuh"',
        '#include "sfft_launch.h"',
        "namespace sfft {",
        "template <int L1, int L2, bool DIF, bool SZ>",
        f"static cudaError_t launch_pass2_{dt}(const Pass2Args &a, int64_t items, cudaStream_t st)",
        "{",
        f"    using Sh = P2Shape<{T}, L1, L2>;",
        f"    auto k = sfft_pass2_kernel<{T}, L1, L2, DIF, SZ>;",
        "    constexpr int smem = Sh::smem_bytes();",
        "    // per-device: 'attribute set' bit + resident CTAs (published once, release/acquire)",
        "    static std::atomic<unsigned> done_mask{0u};",
        "    static std::atomic<int> grid_of[32];",
        "    int dev = 0;",
        "    cudaGetDevice(&dev);",
        "    const unsigned bit = 1u << (dev & 31);",
        "    if (!(done_mask.load(std::memory_order_acquire) & bit)) {",
        "        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);",
        "        if (e != cudaSuccess) return e;",
        "        int per_sm = 0, sms = 0;",
        "        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, Sh::NT, smem);",
        "        if (e != cudaSuccess) return e;",
        "        e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);",
        "        if (e != cudaSuccess) return e;",
        "        if (per_sm < 1 || sms < 1) return cudaErrorInvalidConfiguration;",
        "        grid_of[dev & 31].store(per_sm * sms, std::memory_order_relaxed);",
        "        done_mask.fetch_or(bit, std::memory_order_release);",
        "    }",
        "    int64_t grid = grid_of[dev & 31].load(std::memory_order_relaxed);",
        "    if (grid > items) grid = items;",
        "    if (grid < 1) return cudaErrorInvalidConfiguration;",
        "    k<<<(unsigned)grid, Sh::NT, smem, st>>>(a);",
        "    count_launch();",
        "    return cudaGetLastError();",
        "}",
        f"Pass2LaunchFn pass2_launcher_{dt}(int L1, int L2, bool dif, bool sz)",
        "{",
    ]
    b = lambda v: "true" if v else "false"   # noqa: E731
    for (l1, l2) in PASS2_PAIRS:
        for dif in (False, True):
            for sz in (False, True):
                out.append(f"    if (L1 == {l1} && L2 == {l2} && dif == {b(dif)} && sz == {b(sz)}) "
                           f"return launch_pass2_{dt}<{l1}, {l2}, {b(dif)}, {b(sz)}>;")
    out += ["    return nullptr;", "}", "}  // namespace sfft"]
    return "\n".join(out) + "\n"


def tma_unit(dt):
    T = CTYPE[dt]
    out = [
        "// GENERATED by gen_inst.py -- do not edit",
        '#include "sfft_tma_host.h"',
        "namespace sfft {",
        f"TmaLaunchFn tma_launcher_{dt}(int logn, int lr, bool dif, bool pre)",
        "{",
    ]
    for logn, c in sorted(TMAW_CONFIGS[dt].items()):
        warps, hk, tm, ring, xs, wps = c[:6]
        pf = c[6] if len(c) > 6 else 0
        tm = "true" if tm else "false"
        ring = "true" if ring else "false"
        a = f"{warps}, {hk}, {tm}, {ring}, {xs}, {logn}, {wps}, {pf}"
        out.append(f"    if (logn == {logn} && lr == {logn // 2}) return dif ? launch_tmaw<{T}, true, {a}> "
                   f": launch_tmaw<{T}, false, {a}>;")
    for logn, cfgs in sorted(TMA_CONFIGS[dt].items()):
        for c in cfgs:
            lr, nt, stages, ob = c[:4]
            minb = c[4] if len(c) > 4 else 0
            args = f"{T}, {logn}, {lr}, %s, {nt}, {stages}, {ob}"
            if dt == "f32":
                out.append(f"    if (logn == {logn} && lr == {lr} && pre) return dif ? launch_tma<{args % 'true'}, true, {minb}> : launch_tma<{args % 'false'}, true, {minb}>;")
            out.append(f"    if (logn == {logn} && lr == {lr}) return dif ? launch_tma<{args % 'true'}, false, {minb}> : launch_tma<{args % 'false'}, false, {minb}>;")
    out += ["    return nullptr;", "}", "}  // namespace sfft"]
    return "\n".join(out) + "\n"


def registry_unit():
    out = [
        "// GENERATED by gen_inst.py -- do not edit",
        '#include "sfft_launch.h"',
        "namespace sfft {",
    ]
    for dt in ("f32", "f64"):
        for algo in ("dit", "dif"):
            out.append(f"FusedLaunchFn fused_{algo}_{dt}_table(int logn, int lr, bool il, bool pre);")
    for dt in ("f32", "f64"):
        vals = [str(TMA_CONFIGS[dt][i][0][0]) if i in TMA_CONFIGS[dt] else "-1" for i in range(13)]
        out.append(f"static const int kTmaLr_{dt}[13] = {{{', '.join(vals)}}};")
        fam = [{"ldg": "0", "tma": "1"}[AUTO[dt][i][0]] if i in AUTO[dt] else "0" for i in range(13)]
        alr = [str(AUTO[dt][i][1]) if i in AUTO[dt] else str(DEFAULT_LR[dt][i]) for i in range(13)]
        apre = [("1" if AUTO[dt][i][2] else "0") if i in AUTO[dt] else "0" for i in range(13)]
        out.append(f"static const int kAutoTma_{dt}[13] = {{{', '.join(fam)}}};")
        out.append(f"static const int kAutoLr_{dt}[13] = {{{', '.join(alr)}}};")
        out.append(f"static const int kAutoPre_{dt}[13] = {{{', '.join(apre)}}};")
        slr = [str(AUTO[dt][i][3][0]) if i in AUTO[dt] and len(AUTO[dt][i]) > 3 else "-1" for i in range(13)]
        sbl = [f"{AUTO[dt][i][3][1]}LL" if i in AUTO[dt] and len(AUTO[dt][i]) > 3 else "0LL" for i in range(13)]
        out.append(f"static const int kAutoSmallLr_{dt}[13] = {{{', '.join(slr)}}};")
        out.append(f"static const long long kAutoSmallBelow_{dt}[13] = {{{', '.join(sbl)}}};")
    out += [
        "// kernel=auto: (use TMA?, log2 radix, up-front factors) per size, tuned on B200",
        "void auto_choice(int dtype, int logn, int *family, int *lr, bool *pre)",
        "{",
        "    *family = dtype == 0 ? kAutoTma_f32[logn] : kAutoTma_f64[logn];",
        "    *lr = dtype == 0 ? kAutoLr_f32[logn] : kAutoLr_f64[logn];",
        "    *pre = dtype == 0 ? kAutoPre_f32[logn] : kAutoPre_f64[logn];",
        "}",
        "// kernel=auto batch-size switch: TMA radix for batches below *below (-1: none)",
        "void auto_small_batch(int dtype, int logn, int *lr, long long *below)",
        "{",
        "    *lr = dtype == 0 ? kAutoSmallLr_f32[logn] : kAutoSmallLr_f64[logn];",
        "    *below = dtype == 0 ? kAutoSmallBelow_f32[logn] : kAutoSmallBelow_f64[logn];",
        "}",
    ]
    out += [
        "int tma_default_lr(int dtype, int logn)",
        "{",
        "    if (logn < 0 || logn > kFusedMaxLog) return -1;",
        "    return dtype == 0 ? kTmaLr_f32[logn] : kTmaLr_f64[logn];",
        "}",
        "TmaLaunchFn tma_launcher(int dtype, int logn, int lr, bool dif, bool pre)",
        "{",
        "    return dtype == 0 ? tma_launcher_f32(logn, lr, dif, pre) : tma_launcher_f64(logn, lr, dif, pre);",
        "}",
    ]
    for dt in ("f32", "f64"):
        out.append(f"static const int kDefaultLr_{dt}[13] = {{{', '.join(str(DEFAULT_LR[dt][i]) for i in range(13))}}};")
    out += [
        "int fused_default_lr(int dtype, int logn)",
        "{",
        "    if (logn < 0 || logn > kFusedMaxLog) return -1;",
        "    return dtype == 0 ? kDefaultLr_f32[logn] : kDefaultLr_f64[logn];",
        "}",
        "// dif selects the table; the registry returns a launcher bound to (algo, layout)",
        "FusedLaunchFn fused_launcher_algo(int dtype, int logn, int lr, bool dif, bool il, bool pre)",
        "{",
        "    if (dtype == 0) return dif ? fused_dif_f32_table(logn, lr, il, pre) : fused_dit_f32_table(logn, lr, il, pre);",
        "    return dif ? fused_dif_f64_table(logn, lr, il, pre) : fused_dit_f64_table(logn, lr, il, pre);",
        "}",
        f"int pass_default_lr(int dtype) {{ return dtype == 0 ? {PASS_LR['f32']} : {PASS_LR['f64']}; }}",
        "#ifdef SFFT_PASS_TJ64",
        "int pass_tile(int dtype, int L) { return (dtype == 0 ? (L <= 7 ? 64 : 32) : 16) >> (L >= 10 ? 1 : 0); }",
        "#else",
        "int pass_tile(int dtype, int L) { return (dtype == 0 ? 32 : 16) >> (L >= 10 ? 1 : 0); }",
        "#endif",
        "PassLaunchFn pass_launcher(int dtype, int L) { return dtype == 0 ? pass_launcher_f32(L) : pass_launcher_f64(L); }",
        "Pass2LaunchFn pass2_launcher(int dtype, int L1, int L2, bool dif, bool sz)",
        "{",
        "    return dtype == 0 ? pass2_launcher_f32(L1, L2, dif, sz) : pass2_launcher_f64(L1, L2, dif, sz);",
        "}",
        "}  // namespace sfft",
    ]
    return "\n".join(out) + "\n"


def small_tw_unit():
    """Stage-t factors (t <= 6) as literals: w_{2^t}^f = cos - j sin of
    2 pi f / 2^t, snapped exactly like twiddle.py:46-57 (Python's math.cos /
    math.sin are libm, bit-identical to the library's host tables).  The
    first register pass of every kernel uses them as immediates, and fp32
    later passes form w_i(c + f 2^gs) = w_i(c) * w_{2^t}^f from them."""
    import math
    import struct
    re64, im64 = [], []
    for t in range(1, 7):
        for f in range(1 << (t - 1)):
            ang = 2.0 * math.pi * f / float(1 << t)
            c, sn = math.cos(ang), math.sin(ang)
            if (4 * f) % (1 << t) == 0:
                c, sn = float(round(c)), float(round(sn))
            c += 0.0
            sn += 0.0
            re64.append(0.0 if c == 0.0 else c)
            im64.append(0.0 - sn)
    f32 = lambda v: struct.unpack("f", struct.pack("f", v))[0]   # noqa: E731
    def chain(vals, fmt):
        expr = fmt(vals[-1])
        for k in range(len(vals) - 2, -1, -1):
            expr = f"k == {k} ? {fmt(vals[k])} : ({expr})"
        return expr
    d = lambda v: repr(float(v))                                   # noqa: E731
    fl = lambda v: repr(f32(v)) + "f" if f32(v) != int(f32(v)) or abs(f32(v)) > 1 else f"{f32(v):.1f}f"  # noqa: E731
    out = [
        "// GENERATED by gen_inst.py -- small-stage factors as literals (t <= 6)",
        "#pragma once",
        "namespace sfft {",
        "// index k = 2^(t-1) - 1 + f for stage t, factor f < 2^(t-1)",
        f"__host__ __device__ constexpr double small_tw_re64(int k) {{ return {chain(re64, d)}; }}",
        f"__host__ __device__ constexpr double small_tw_im64(int k) {{ return {chain(im64, d)}; }}",
        f"__host__ __device__ constexpr float small_tw_re32(int k) {{ return {chain(re64, lambda v: repr(f32(v)) + 'f')}; }}",
        f"__host__ __device__ constexpr float small_tw_im32(int k) {{ return {chain(im64, lambda v: repr(f32(v)) + 'f')}; }}",
        "}  // namespace sfft",
    ]
    return "\n".join(out) + "\n"


def main(outdir):
    files = {}
    files["sfft_small_tw.h"] = small_tw_unit()
    for dt in ("f32", "f64"):
        for algo in ("dit", "dif"):
            files[f"sfft_inst_fused_{algo}_{dt}.cu"] = fused_unit(dt, algo)
        files[f"sfft_inst_pass_{dt}.cu"] = pass_unit(dt)
        files[f"sfft_inst_tma_{dt}.cu"] = tma_unit(dt)
        files[f"sfft_inst_pass2_{dt}.cu"] = pass2_unit(dt)
    files["sfft_inst_registry.cu"] = registry_unit()
    for name, text in files.items():
        path = os.path.join(outdir, name)
        old = open(path).read() if os.path.exists(path) else None
        if old != text:
            with open(path, "w") as f:
                f.write(text)
    print(" ".join(sorted(files)))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else HERE)
