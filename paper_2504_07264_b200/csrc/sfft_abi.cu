// sfft_abi.cu -- the C ABI declared in include/splitfft_b200.h.
//
// Plan construction mirrors make_plan (transform.py:65-85): same validation
// order and messages, same snapped stage-factor values (twiddle.py:46-57,
// transform.py:82) computed on the host with libm and uploaded once per
// plan.  Exec is a pure stream-ordered launch sequence: one fused kernel for
// log2n <= 12, otherwise one launch per stage group (sfft_pass.cuh).
#include <cuda_runtime.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <string>
#include <thread>
#include <utility>

#include <vector>

#include "../../include/splitfft_b200.h"
#include "sfft_fused.cuh"
#include "sfft_launch.h"
#include "sfft_pass.cuh"
#include "sfft_pass2.cuh"
#include "sfft_stage.cuh"
#include "sfft_tma_host.h"

#include <mutex>

namespace sfft {
static std::atomic<int64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder()
{
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}
}  // namespace sfft

using namespace sfft;

namespace {

thread_local std::string g_err;

int fail(int code, const char *fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

int cuda_fail(cudaError_t e, const char *what)
{
    return fail(SFFT_ECUDA, "%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
}

// twiddle.py:46-57 then transform.py:82 (w = cos - 1j*sin as numpy forms it:
// real part cos, imaginary part 0.0 - sin, so sin == 0 gives +0.0).
inline void stage_factor(int i, int64_t q, double *wr, double *wi)
{
    double angle = 2.0 * M_PI * (double)q / (double)(int64_t(1) << i);
    double c = cos(angle);
    double s = sin(angle);
    if (((4 * q) % (int64_t(1) << i)) == 0) {
        c = nearbyint(c);
        s = nearbyint(s);
    }
    c += 0.0;
    s += 0.0;
    *wr = c == 0.0 ? 0.0 : c;
    *wi = 0.0 - s;
}

void stage_table(int i, int64_t count, double *wr, double *wi)
{
    // count <= 2^(i-1); parallel for the 2^27-entry tables of very long plans
    const int64_t chunk = int64_t(1) << 20;
    if (count <= chunk) {
        for (int64_t q = 0; q < count; ++q) stage_factor(i, q, wr + q, wi + q);
        return;
    }
    unsigned nt = std::thread::hardware_concurrency();
    if (nt == 0) nt = 4;
    if (nt > 32) nt = 32;
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nt; ++t) {
        th.emplace_back([=] {
            for (int64_t q0 = (int64_t)t * chunk; q0 < count; q0 += (int64_t)nt * chunk) {
                int64_t q1 = q0 + chunk < count ? q0 + chunk : count;
                for (int64_t q = q0; q < q1; ++q) stage_factor(i, q, wr + q, wi + q);
            }
        });
    }
    for (auto &x : th) x.join();
}

struct DeviceGuard {
    int prev = -1;
    cudaError_t err = cudaSuccess;
    explicit DeviceGuard(int dev)
    {
        err = cudaGetDevice(&prev);
        if (err == cudaSuccess && prev != dev) err = cudaSetDevice(dev);
    }
    ~DeviceGuard()
    {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

struct Group {
    int S, L;
};

}  // namespace

struct sfft_plan {
    int log2n = 0, dtype = 0, algo = 0, device = 0, lr = 0;
    int kernel = SFFT_KERNEL_AUTO;  // fused-path kernel family
    int lr_tma = -1;                // radix of the TMA kernel (-1: none)
    int lr_tma_small = -1;          // kernel=auto: TMA radix for batches < small_below
    int64_t small_below = 0;
    int lr_ldg_il = 0;              // radix of the interleaved LDG kernel
    bool pre = false;               // fp32: fetch pass base factors up front
    // fused path
    void *d_tw = nullptr;          // stage-major vec2_t<T> table, stages 1..cat_top
    int cat_top = 0;
    void *d_top = nullptr;         // fp64 m > 20: stage-m table for stages > cat_top
    // large path
    double2 *d_coarse = nullptr;
    int coarse_log = 0;
    double2 *d_fine = nullptr;
    std::vector<Group> groups;
    // L2-fused schedule (sfft_pass2.cuh): groups = 4 balanced groups, run as
    // two launches (groups 0+1, 2+3), one HBM sweep each
    bool fuse2 = false;
};

namespace {

template <typename T>
int upload_table(sfft_plan *p, int cat_top, bool with_top)
{
    // stage-major: stage i (1..cat_top) at offset 2^(i-1)-1, bitwise the
    // strided view [::2^(cat_top-i)] of the stage-cat_top table
    const int64_t total = cat_top >= 1 ? (int64_t(1) << cat_top) - 1 : 1;
    std::vector<vec2_t<T>> host((size_t)total);
    if (cat_top >= 1) {
        const int64_t h = int64_t(1) << (cat_top - 1);
        std::vector<double> wr((size_t)h), wi((size_t)h);
        stage_table(cat_top, h, wr.data(), wi.data());
        for (int i = 1; i <= cat_top; ++i) {
            const int64_t off = (int64_t(1) << (i - 1)) - 1, sh = cat_top - i;
            for (int64_t q = 0; q < (int64_t(1) << (i - 1)); ++q) {
                host[off + q].x = (T)wr[q << sh];
                host[off + q].y = (T)wi[q << sh];
            }
        }
    } else {
        host[0].x = (T)1;
        host[0].y = (T)0;
    }
    cudaError_t e = cudaMalloc(&p->d_tw, sizeof(vec2_t<T>) * (size_t)total);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(twiddle table)");
    e = cudaMemcpy(p->d_tw, host.data(), sizeof(vec2_t<T>) * (size_t)total, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy(twiddle table)");
    p->cat_top = cat_top;
    if (with_top) {
        const int64_t h = int64_t(1) << (p->log2n - 1);
        std::vector<double> wr((size_t)h), wi((size_t)h);
        stage_table(p->log2n, h, wr.data(), wi.data());
        std::vector<vec2_t<T>> top((size_t)h);
        for (int64_t q = 0; q < h; ++q) {
            top[q].x = (T)wr[q];
            top[q].y = (T)wi[q];
        }
        e = cudaMalloc(&p->d_top, sizeof(vec2_t<T>) * (size_t)h);
        if (e == cudaSuccess) e = cudaMemcpy(p->d_top, top.data(), sizeof(vec2_t<T>) * (size_t)h, cudaMemcpyHostToDevice);
        if (e != cudaSuccess) return cuda_fail(e, "uploading the stage-m table");
    }
    return SFFT_OK;
}

int upload_two_level(sfft_plan *p)
{
    // coarse: stage CL factors; fine: stage m factors for lo < 2^(m-CL)
    const int m = p->log2n;
    const int CL = m < 16 ? m : 16;
    const int64_t hc = int64_t(1) << (CL - 1);
    const int64_t hf = int64_t(1) << (m - CL);
    std::vector<double> cr((size_t)hc), ci((size_t)hc), fr((size_t)hf), fi((size_t)hf);
    stage_table(CL, hc, cr.data(), ci.data());
    stage_table(m, hf, fr.data(), fi.data());
    // fine table, then the lane table: stage i's factors w_i(l), l < 32, at
    // hf + (i-1)*32 + l (entries past 2^(i-1) are never read)
    const int64_t nf = hf + 32 * (int64_t)m;
    std::vector<double2> c2((size_t)hc), f2((size_t)nf, make_double2(0.0, 0.0));
    for (int64_t q = 0; q < hc; ++q) c2[q] = make_double2(cr[q], ci[q]);
    for (int64_t q = 0; q < hf; ++q) f2[q] = make_double2(fr[q], fi[q]);
    for (int i = 1; i <= m; ++i) {
        const int64_t hl = std::min<int64_t>(32, int64_t(1) << (i - 1));
        std::vector<double> lr((size_t)hl), li((size_t)hl);
        stage_table(i, hl, lr.data(), li.data());
        for (int64_t l = 0; l < hl; ++l) f2[hf + 32 * (i - 1) + l] = make_double2(lr[l], li[l]);
    }
    cudaError_t e = cudaMalloc(&p->d_coarse, sizeof(double2) * (size_t)hc);
    if (e == cudaSuccess) e = cudaMalloc(&p->d_fine, sizeof(double2) * (size_t)nf);
    if (e == cudaSuccess)
        e = cudaMemcpy(p->d_coarse, c2.data(), sizeof(double2) * (size_t)hc, cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
        e = cudaMemcpy(p->d_fine, f2.data(), sizeof(double2) * (size_t)nf, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_fail(e, "uploading two-level twiddles");
    p->coarse_log = CL;
    return SFFT_OK;
}

void free_plan(sfft_plan *p)
{
    if (!p) return;
    if (p->d_tw) cudaFree(p->d_tw);
    if (p->d_top) cudaFree(p->d_top);
    if (p->d_coarse) cudaFree(p->d_coarse);
    if (p->d_fine) cudaFree(p->d_fine);
    delete p;
}

// Largest group (log2 sub-problem size) of the multi-launch schedule.
// 8 measured best for fp32 N = 2^28 (4 groups of 7 beat 3 groups of 9-10:
// the 2^9/2^10-point groups fit one CTA per SM); SFFT_PASS_MAX_L overrides
// (developer knob for tools/tune_large.py).
static int pass_max_l()
{
    const char *e = getenv("SFFT_PASS_MAX_L");
    int v = e ? atoi(e) : 8;
    return v < kPassMinL ? kPassMinL : (v > kPassMaxL ? kPassMaxL : v);
}

// Groups of at most pass_max_l() stages covering `stages` consecutive stages
// from S0 (balanced, each >= kPassMinL when stages allows).
static std::vector<Group> split_range(int S0, int stages)
{
    const int maxl = pass_max_l();
    const int G = (stages + maxl - 1) / maxl;
    std::vector<Group> g;
    int S = S0;
    for (int k = 0; k < G; ++k) {
        const int L = stages / G + (k < stages % G ? 1 : 0);
        g.push_back({S, L});
        S += L;
    }
    return g;
}

std::vector<Group> split_groups(int m)
{
    // developer knob for A/B runs: SFFT_PASS_SPLIT="8,7,7,6" (group sizes in
    // launch order, each in [kPassMinL, kPassMaxL], summing to m)
    if (const char *e = getenv("SFFT_PASS_SPLIT")) {
        std::vector<Group> g;
        int S = 0;
        bool ok = true;
        for (const char *c = e; *c && ok;) {
            const int L = atoi(c);
            ok = L >= kPassMinL && L <= kPassMaxL;
            g.push_back({S, L});
            S += L;
            while (*c && *c != ',') ++c;
            if (*c == ',') ++c;
        }
        if (ok && S == m) return g;
    }
    const int maxl = pass_max_l();
    const int G = (m + maxl - 1) / maxl;
    std::vector<Group> g;
    int S = 0;
    for (int k = 0; k < G; ++k) {
        int L = m / G + (k < m % G ? 1 : 0);
        g.push_back({S, L});
        S += L;
    }
    return g;
}

// L2-fused pairs: m = 20..28 as 4 balanced groups of 5..7 stages (the
// pairs 0+1 and 2+3 are one sweep each).  SFFT_PASS2=0 turns it off (A/B);
// the SFFT_PASS_SPLIT / SFFT_PASS_MAX_L developer knobs imply the unfused
// schedule.
constexpr int kPass2MinLog = 20, kPass2MaxLog = 28;
// kernel=auto takes it only for fp64 at m = 28 (6.2-6.9 vs 7.7 ms: the fp64
// pass launches are issue-bound with 2 of 4 sweeps' loads exposed).  Below
// that the per-group launches win by 1.5-4x (m = 26: 2.0 vs 3.0 ms, m = 20:
// 0.045 vs 0.17 ms -- smaller rows leave the persistent kernel few blocks
// and half-size tiles), and fp32 per-group launches run at 0.9 of the HBM
// peak while the persistent tile chain is latency-bound (m = 28: 2.71 vs
// 2.79 ms; profiles/r02z*, r02aa-ac).  SFFT_PASS2=1 / 0 forces it on / off
// for every size and type it supports.
bool pass2_enabled(int m, int dtype)
{
    if (m < kPass2MinLog || m > kPass2MaxLog) return false;
    if (getenv("SFFT_PASS_SPLIT") || getenv("SFFT_PASS_MAX_L")) return false;
    const char *e = getenv("SFFT_PASS2");
    if (e && e[0] == '0') return false;
    if (e && e[0] == '1') return true;
    return dtype == SFFT_F64 && m == 28;
}
std::vector<Group> balanced4(int m)
{
    std::vector<Group> g;
    int S = 0;
    for (int k = 0; k < 4; ++k) {
        const int L = m / 4 + (k < m % 4 ? 1 : 0);
        g.push_back({S, L});
        S += L;
    }
    return g;
}
int pass2_env(const char *name, int dflt, int lo, int hi)
{
    const char *e = getenv(name);
    int v = e ? atoi(e) : dflt;
    return v < lo ? lo : (v > hi ? hi : v);
}
constexpr int kPass2MaxSlots = 32;
constexpr size_t kPass2CtrBytes = 2 * (1 + 2 * kPass2MaxSlots) * sizeof(unsigned);

int validate_exec(const sfft_plan *p, int64_t batch, int64_t is, int64_t os, int direction)
{
    if (!p) return fail(SFFT_EINVAL, "plan is NULL");
    if (batch < 0) return fail(SFFT_EINVAL, "batch must be >= 0, got %lld", (long long)batch);
    const int64_t n = int64_t(1) << p->log2n;
    if (batch > 1 && (is < n || os < n))
        return fail(SFFT_EINVAL, "row strides (%lld, %lld) must be >= N = %lld", (long long)is,
                    (long long)os, (long long)n);
    if (direction != SFFT_FORWARD && direction != SFFT_INVERSE)
        return fail(SFFT_EINVAL, "direction must be -1 (forward) or +1 (inverse), got %d", direction);
    if (batch > (int64_t(1) << 40)) return fail(SFFT_ECAPACITY, "batch %lld exceeds the launch limit", (long long)batch);
    return SFFT_OK;
}

// The L2-fused schedule: two persistent launches (sfft_pass2.cuh), groups
// 0+1 then 2+3 (DIT) or 2+3 then 0+1 (DIF), through one intermediate plane
// pair; the block scratch ring and the tile counters live in the rest of
// the workspace.  Planar only.
int exec_fused2(const sfft_plan *p, const void *x0, const void *x1, void *y0, void *y1, int64_t batch,
                int64_t is, int64_t os, bool inv, double scale, void *workspace, cudaStream_t st)
{
    const int m = p->log2n;
    const int64_t n = int64_t(1) << m;
    const size_t esz = p->dtype == SFFT_F32 ? 4 : 8;
    const int TJ = p->dtype == SFFT_F32 ? 32 : 16;
    const size_t plane = (size_t)batch * (size_t)n * esz;
    char *ws = (char *)workspace;
    void *mid[2] = {ws, ws + plane};
    char *scr = ws + 2 * plane;
    unsigned *ctr = (unsigned *)(ws + 4 * plane);
    // ring geometry and scheduler variant (profiles/r02ab_*): fp32 6 blocks
    // behind in a 16-slot ring with the L2 prefetch of the next tile; fp64 4
    // behind in 8 slots, no prefetch
    const bool f32 = p->dtype == SFFT_F32;
    const int lag = pass2_env("SFFT_P2_LAG", f32 ? 6 : 4, 1, kPass2MaxSlots - 1);
    int nslot = pass2_env("SFFT_P2_SLOTS", f32 ? 16 : 8, 2, kPass2MaxSlots);
    if (nslot <= lag) nslot = lag + 1;
    const int flags = pass2_env("SFFT_P2_FLAGS", f32 ? P2_PREFETCH : 0, 0, 7);
    int nslot_log = 0;
    while ((1 << nslot_log) < nslot) ++nslot_log;   // a power of two
    const std::vector<Group> &g = p->groups;
    const int words = 1 + 2 * kPass2MaxSlots;
    cudaError_t e = cudaMemsetAsync(ctr, 0, 2 * words * sizeof(unsigned), st);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync");
    const bool dif = p->algo == SFFT_DIF;
    for (int k = 0; k < 2; ++k) {
        const int sg = dif ? 1 - k : k;   // super-group: groups 2sg, 2sg+1
        const Group g1 = g[2 * sg], g2 = g[2 * sg + 1];
        const int L = g1.L + g2.L;
        const int64_t nb = batch * ((n >> L) / TJ);    // blocks
        int ns_log = nslot_log;
        while (ns_log > 0 && (int64_t(1) << (ns_log - 1)) >= nb) --ns_log;   // no more slots than blocks
        const int ns = 1 << ns_log;
        Pass2LaunchFn fn = pass2_launcher(p->dtype, g1.L, g2.L, dif, g1.S == 0);
        if (!fn) return fail(SFFT_EINVAL, "no fused pass pair for L=%d+%d", g1.L, g2.L);
        if ((size_t)ns * ((size_t)TJ << L) * esz > plane)
            return fail(SFFT_EINVAL, "scratch ring exceeds the workspace (log2n=%d)", m);
        Pass2Args a;
        memset(&a, 0, sizeof a);
        const bool first = k == 0, last = k == 1;
        // the inverse: input planes exchanged on the first launch, output
        // planes exchanged (and scaled) on the last
        if (first) {
            a.x0 = inv ? x1 : x0;
            a.x1 = inv ? x0 : x1;
            a.in_stride = is;
        } else {
            a.x0 = mid[0];
            a.x1 = mid[1];
            a.in_stride = n;
        }
        if (last) {
            a.y0 = inv ? y1 : y0;
            a.y1 = inv ? y0 : y1;
            a.out_stride = os;
        } else {
            a.y0 = mid[0];
            a.y1 = mid[1];
            a.out_stride = n;
        }
        a.s0 = scr;   // (re, im) pairs: the ring takes up to two planes' worth
        a.s1 = nullptr;
        a.ctr = ctr + k * words;
        a.batch = batch;
        a.m = m;
        a.S = g1.S;
        a.nslot_log = ns_log;
        a.lag = lag;
        a.scale_out = last && inv;
        a.scale = last ? scale : 1.0;
        a.flags = flags;
        // the L2 prefetch issues 128-byte bulk requests: 16-byte aligned source runs only
        if ((((uintptr_t)a.x0 | (uintptr_t)a.x1) & 15) || (batch > 1 && ((size_t)a.in_stride * esz) % 16))
            a.flags &= ~P2_PREFETCH;
        a.tw = p->d_tw;
        a.tw_cat_top = p->cat_top;
        a.tw_top_tab = p->d_top;
        a.coarse = p->d_coarse;
        a.coarse_log = p->coarse_log;
        a.fine = p->d_fine;
        const int64_t items = nb * ((int64_t(1) << g1.L) + (int64_t(1) << g2.L));
        if (items + 1024 * 1024 > 0xffffffffLL) return fail(SFFT_ECAPACITY, "batch %lld too large for one fused launch", (long long)batch);
        e = fn(a, items, st);
        if (e != cudaSuccess) return cuda_fail(e, "fused pass pair launch");
    }
    return SFFT_OK;
}

int exec_common(const sfft_plan *p, const void *x0, const void *x1, void *y0, void *y1, bool il,
                int64_t batch, int64_t is, int64_t os, int direction, void *workspace, void *stream)
{
    int rc = validate_exec(p, batch, is, os, direction);
    if (rc) return rc;
    if (batch == 0) return SFFT_OK;
    if (!x0 || !y0 || (!il && (!x1 || !y1))) return fail(SFFT_EINVAL, "NULL signal pointer");
    DeviceGuard dg(p->device);
    if (dg.err != cudaSuccess) return cuda_fail(dg.err, "cudaSetDevice");
    cudaStream_t st = (cudaStream_t)stream;
    const bool inv = direction == SFFT_INVERSE;
    const int m = p->log2n;
    const double scale = inv ? 1.0 / (double)(int64_t(1) << m) : 1.0;

    if (m <= kFusedMaxLog) {
        if (batch > 0x7fffffffLL)
            return fail(SFFT_ECAPACITY, "batch %lld exceeds one launch (2^31 rows); split the batch", (long long)batch);
        const size_t esz = p->dtype == SFFT_F32 ? 4 : 8;
        const bool aligned = ((uintptr_t)x0 | (uintptr_t)x1 | (uintptr_t)y0 | (uintptr_t)y1) % 16 == 0 &&
                             ((size_t)is * esz) % 16 == 0 && ((size_t)os * esz) % 16 == 0 &&
                             batch < (int64_t(1) << 31);
        // kernel=auto batch-size switch (fp64: every kernel is the same
        // arithmetic, bitwise; fp32: within the same tolerance)
        const bool small = p->lr_tma_small >= 0 && batch < p->small_below;
        if (!il && p->lr_tma >= 0 && p->kernel != SFFT_KERNEL_LDG && aligned && !(small && p->lr_tma_small == 0)) {
            const int lr_t = small ? p->lr_tma_small : p->lr_tma;
            TmaLaunchFn tf = tma_launcher(p->dtype, m, lr_t, p->algo == SFFT_DIF, p->pre);
            if (tf) {
                TmaLaunch L;
                L.x_re = x0;
                L.x_im = x1;
                L.y_re = y0;
                L.y_im = y1;
                L.batch = batch;
                L.in_stride = batch > 1 ? is : (int64_t(1) << m);
                L.out_stride = batch > 1 ? os : (int64_t(1) << m);
                L.inverse = inv ? 1 : 0;
                L.scale = scale;
                L.tw = p->d_tw;
                cudaError_t e = tf(L, st);
                if (e != cudaSuccess) return cuda_fail(e, "TMA kernel launch");
                return SFFT_OK;
            }
        }
        if (p->kernel == SFFT_KERNEL_TMA)
            return fail(SFFT_EINVAL, "the TMA kernel needs planar, 16-byte aligned rows with 16-byte row strides "
                                     "and a size with a TMA configuration (log2n=%d)", m);
        const int lr = il ? p->lr_ldg_il : p->lr;
        FusedLaunchFn fn = fused_launcher_algo(p->dtype, m, lr, p->algo == SFFT_DIF, il, !il && p->pre);
        if (!fn) return fail(SFFT_EINVAL, "no fused kernel for log2n=%d radix=2^%d layout=%s", m, lr,
                             il ? "interleaved" : "planar");
        FusedArgs a;
        a.x0 = x0;
        a.x1 = x1;
        a.y0 = y0;
        a.y1 = y1;
        a.tw = p->d_tw;
        a.batch = batch;
        a.in_stride = is;
        a.out_stride = os;
        a.inverse = inv ? 1 : 0;
        a.scale = scale;
        cudaError_t e = fn(a, p->algo == SFFT_DIF, il, st);
        if (e != cudaSuccess) return cuda_fail(e, "fused kernel launch");
        return SFFT_OK;
    }

    // multi-launch schedule: groups in order (DIT) or reverse order (DIF)
    if (!workspace) return fail(SFFT_EINVAL, "log2n=%d needs a workspace (sfft_workspace_bytes)", m);
    const int64_t n = int64_t(1) << m;
    const size_t esz = p->dtype == SFFT_F32 ? 4 : 8;
    if (p->fuse2 && !il) return exec_fused2(p, x0, x1, y0, y1, batch, is, os, inv, scale, workspace, st);
    const int G = (int)p->groups.size();
    char *ws = (char *)workspace;
    const size_t plane = (size_t)batch * (size_t)n * esz;
    void *bufA[2] = {ws, ws + plane};
    void *bufB[2] = {ws + 2 * plane, ws + 3 * plane};
    for (int k = 0; k < G; ++k) {
        const Group gr = p->algo == SFFT_DIF ? p->groups[G - 1 - k] : p->groups[k];
        const int TJ = pass_tile(p->dtype, gr.L);
        PassLaunchFn fn = pass_launcher(p->dtype, gr.L);
        if (!fn) return fail(SFFT_EINVAL, "no pass kernel for L=%d", gr.L);
        PassArgs a;
        memset(&a, 0, sizeof a);
        const bool first = k == 0, last = k == G - 1;
        void **src = (k % 2 == 1) ? bufA : bufB;   // k-1 wrote A when k-1 even
        void **dst = last ? nullptr : ((k % 2 == 0) ? bufA : bufB);
        if (first) {
            a.x0 = x0;
            a.x1 = x1;
            a.in_stride = is;
        } else {
            a.x0 = src[0];
            a.x1 = src[1];
            a.in_stride = n;
        }
        if (last) {
            a.y0 = y0;
            a.y1 = y1;
            a.out_stride = os;
        } else {
            a.y0 = dst[0];
            a.y1 = dst[1];
            a.out_stride = n;
        }
        a.batch = batch;
        a.m = m;
        a.S = gr.S;
        a.swap_in = first && inv;
        a.swap_out = last && inv;
        a.scale = last ? scale : 1.0;
        a.tw = p->d_tw;
        a.tw_cat_top = p->cat_top;
        a.tw_top_tab = p->d_top;
        a.coarse = p->d_coarse;
        a.coarse_log = p->coarse_log;
        a.fine = p->d_fine;
        a.jb = 0;
        a.in_map.b = a.out_map.b = 0;
        const int64_t grid = batch * ((n >> gr.L) / TJ);
        if (grid > 0x7fffffffLL)
            return fail(SFFT_ECAPACITY, "batch %lld x N=2^%d exceeds one launch; split the batch", (long long)batch, m);
        cudaError_t e = fn(a, p->algo == SFFT_DIF, first && il, last && il, grid, st);
        if (e != cudaSuccess) return cuda_fail(e, "pass kernel launch");
    }
    return SFFT_OK;
}

}  // namespace

extern "C" {

int sfft_abi_version(void) { return SFFT_ABI_VERSION; }

const char *sfft_last_error(void) { return g_err.c_str(); }

int64_t sfft_launch_count(void) { return g_launches.load(); }

int sfft_twiddle_table(int log2n, double *wr, double *wi)
{
    if (log2n < 1 || log2n > SFFT_MAX_LOG2N) return fail(SFFT_EINVAL, "log2n must be in [1, %d], got %d", SFFT_MAX_LOG2N, log2n);
    if (!wr || !wi) return fail(SFFT_EINVAL, "NULL output pointer");
    stage_table(log2n, int64_t(1) << (log2n - 1), wr, wi);
    return SFFT_OK;
}

int sfft_count_flops(int log2n, int64_t *out5)
{
    // transform.py:312-335 with the closed forms pinned by
    // test_transform.py:323-332: identity = m, quarter = m-1, generic = N-2m
    if (log2n < 0) return fail(SFFT_EINVAL, "stage count m must be >= 0, got %d", log2n);
    if (log2n > SFFT_MAX_LOG2N) return fail(SFFT_ECAPACITY, "m=%d exceeds the plan limit max_m=%d", log2n, SFFT_MAX_LOG2N);
    if (!out5) return fail(SFFT_EINVAL, "NULL output pointer");
    const int64_t m = log2n, n = int64_t(1) << log2n;
    const int64_t ident = m, quarter = m > 0 ? m - 1 : 0, generic = m > 0 ? n - 2 * m : 0;
    out5[0] = 4 * generic;
    out5[1] = 4 * (n >> 1) * m;
    out5[2] = generic;
    out5[3] = quarter;
    out5[4] = ident;
    return SFFT_OK;
}

int sfft_plan_create_ex(int log2n, int dtype, int algorithm, int device, int max_log2n, int log2_radix,
                        int kernel, sfft_plan **out)
{
    if (!out) return fail(SFFT_EINVAL, "out is NULL");
    *out = nullptr;
    // validation order of make_plan (transform.py:72-76)
    if (log2n < 0) return fail(SFFT_EINVAL, "stage count m must be >= 0, got %d", log2n);
    if (log2n > max_log2n) return fail(SFFT_ECAPACITY, "m=%d exceeds the plan limit max_m=%d", log2n, max_log2n);
    if (log2n > SFFT_MAX_LOG2N)
        return fail(SFFT_ECAPACITY, "m=%d exceeds the plan limit max_m=%d", log2n, SFFT_MAX_LOG2N);
    if (algorithm != SFFT_DIT && algorithm != SFFT_DIF)
        return fail(SFFT_EINVAL, "%d is not a valid Algorithm (0 = dit, 1 = dif)", algorithm);
    if (dtype != SFFT_F32 && dtype != SFFT_F64) return fail(SFFT_EINVAL, "unknown dtype %d", dtype);
    const int pre_pref = (kernel >> 4) & 3;   // 0 auto, 1 off, 2 on
    kernel &= 0xf;
    if ((kernel != SFFT_KERNEL_AUTO && kernel != SFFT_KERNEL_LDG && kernel != SFFT_KERNEL_TMA &&
         kernel != SFFT_KERNEL_PASS && kernel != SFFT_KERNEL_PASS2) || pre_pref == 3)
        return fail(SFFT_EINVAL, "unknown kernel family %d", kernel);
    if (kernel == SFFT_KERNEL_PASS && log2n <= kFusedMaxLog)
        return fail(SFFT_EINVAL, "kernel 'pass' is the multi-launch schedule of log2n > %d, got log2n=%d",
                    kFusedMaxLog, log2n);
    if (kernel == SFFT_KERNEL_PASS2 && (log2n < kPass2MinLog || log2n > kPass2MaxLog))
        return fail(SFFT_EINVAL, "kernel 'pass2' (L2-fused group pairs) needs %d <= log2n <= %d, got log2n=%d",
                    kPass2MinLog, kPass2MaxLog, log2n);
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
    if (device < 0 || device >= ndev) return fail(SFFT_EINVAL, "device %d out of range (%d devices)", device, ndev);

    sfft_plan *p = new sfft_plan;
    p->log2n = log2n;
    p->dtype = dtype;
    p->algo = algorithm;
    p->device = device;
    DeviceGuard dg(device);
    if (dg.err != cudaSuccess) {
        delete p;
        return cuda_fail(dg.err, "cudaSetDevice");
    }
    int rc = SFFT_OK;
    p->kernel = kernel;
    if (log2n <= kFusedMaxLog) {
        bool auto_pre = false;
        int auto_lr = 0, auto_family = 0;
        auto_choice(dtype, log2n, &auto_family, &auto_lr, &auto_pre);
        const bool auto_tma = auto_family == 1;
        p->pre = pre_pref == 2 || (pre_pref == 0 && kernel == SFFT_KERNEL_AUTO && log2_radix <= 0 && auto_pre);
        int lr;
        if (log2_radix > 0) lr = log2_radix;
        else if (kernel == SFFT_KERNEL_AUTO) lr = auto_lr;
        else if (kernel == SFFT_KERNEL_TMA) lr = tma_default_lr(dtype, log2n);
        else lr = fused_default_lr(dtype, log2n);
        if (log2n == 0) lr = 0;
        if (lr > log2n) lr = log2n;
        const bool want_tma_ = kernel == SFFT_KERNEL_TMA ||
                               (kernel == SFFT_KERNEL_AUTO && (log2_radix > 0 || auto_tma));
        // a radix may exist for the TMA family only (the fp32 N = 4096
        // signal-group kernel's radix 64): the LDG kernel (unaligned rows,
        // interleaved layout) then runs its default radix
        const bool ldg_ok = lr >= 0 && fused_launcher_algo(dtype, log2n, lr, algorithm == SFFT_DIF, false);
        const bool tma_only = lr >= 0 && !ldg_ok && want_tma_ && tma_launcher(dtype, log2n, lr, false, false);
        if (!ldg_ok && !tma_only) {
            delete p;
            return fail(SFFT_EINVAL, "radix 2^%d is not available for log2n=%d", lr, log2n);
        }
        p->lr = ldg_ok ? lr : fused_default_lr(dtype, log2n);
        p->lr_ldg_il = fused_default_lr(dtype, log2n);
        const bool want_tma = want_tma_;
        if (want_tma && tma_launcher(dtype, log2n, lr, false, p->pre)) p->lr_tma = lr;
        if (kernel == SFFT_KERNEL_AUTO && log2_radix <= 0 && p->lr_tma >= 0) {
            int slr = -1;
            long long below = 0;
            auto_small_batch(dtype, log2n, &slr, &below);
            // slr == 0: the LDG kernel below `below` rows
            if (slr == 0 || (slr > 0 && tma_launcher(dtype, log2n, slr, false, p->pre))) {
                p->lr_tma_small = slr;
                p->small_below = below;
            }
        }
        if (kernel == SFFT_KERNEL_TMA && p->lr_tma < 0) {
            delete p;
            return fail(SFFT_EINVAL, "no TMA kernel for log2n=%d radix=2^%d", log2n, lr);
        }
        rc = dtype == SFFT_F32 ? upload_table<float>(p, log2n, false) : upload_table<double>(p, log2n, false);
    } else {
        p->lr = pass_default_lr(dtype);
        p->groups = split_groups(log2n);
        if (kernel == SFFT_KERNEL_PASS2 || (kernel != SFFT_KERNEL_PASS && pass2_enabled(log2n, dtype))) {
            p->groups = balanced4(log2n);
            p->fuse2 = true;
        }
        if (dtype == SFFT_F32) {
            rc = upload_table<float>(p, kFusedMaxLog, false);
            if (rc == SFFT_OK) rc = upload_two_level(p);
        } else {
            // fp64 keeps every stage in the stage-major table (bit-exact factors,
            // coalesced reads; 2^m - 1 entries = 4 GiB at m = 28)
            rc = upload_table<double>(p, log2n, false);
        }
    }
    if (rc != SFFT_OK) {
        free_plan(p);
        return rc;
    }
    *out = p;
    return SFFT_OK;
}

int sfft_plan_create(int log2n, int dtype, int algorithm, int device, int max_log2n, sfft_plan **out)
{
    return sfft_plan_create_ex(log2n, dtype, algorithm, device, max_log2n, 0, SFFT_KERNEL_AUTO, out);
}

int sfft_plan_destroy(sfft_plan *plan)
{
    if (!plan) return SFFT_OK;
    DeviceGuard dg(plan->device);
    free_plan(plan);
    return SFFT_OK;
}

int sfft_plan_info(const sfft_plan *p, int *log2n, int *dtype, int *algorithm, int *device, int *launches,
                   int *log2_radix, int *kernel)
{
    if (kernel && p)
        *kernel = p->lr_tma >= 0 ? SFFT_KERNEL_TMA
                                   : (p->log2n <= kFusedMaxLog ? SFFT_KERNEL_LDG
                                                               : (p->fuse2 ? SFFT_KERNEL_PASS2 : SFFT_KERNEL_PASS));
    if (!p) return fail(SFFT_EINVAL, "plan is NULL");
    if (log2n) *log2n = p->log2n;
    if (dtype) *dtype = p->dtype;
    if (algorithm) *algorithm = p->algo;
    if (device) *device = p->device;
    if (launches) *launches = p->log2n <= kFusedMaxLog ? 1 : (p->fuse2 ? 2 : (int)p->groups.size());
    if (log2_radix) *log2_radix = p->lr;
    return SFFT_OK;
}

int sfft_exec_kernel(const sfft_plan *p, int64_t batch, int interleaved, int *family, int *log2_radix, int *warp)
{
    if (!p) return fail(SFFT_EINVAL, "plan is NULL");
    if (batch < 0) return fail(SFFT_EINVAL, "batch must be >= 0, got %lld", (long long)batch);
    int fam, lr, w = 0;
    if (p->log2n > kFusedMaxLog) {
        fam = p->fuse2 && !interleaved ? SFFT_KERNEL_PASS2 : SFFT_KERNEL_PASS;
        lr = p->fuse2 && !interleaved ? 4 : p->lr;   // pass2: 8 threads per column, 2^(Lg-3) values each
    } else if (!interleaved && p->lr_tma >= 0 && p->kernel != SFFT_KERNEL_LDG &&
               !(p->lr_tma_small == 0 && batch < p->small_below)) {
        fam = SFFT_KERNEL_TMA;
        lr = (p->lr_tma_small >= 0 && batch < p->small_below) ? p->lr_tma_small : p->lr_tma;
        // the signal-group ring kernel (sfft_tma_warp.cuh): radix 2^(log2n/2)
        w = (p->dtype == SFFT_F64 && p->log2n == 10 && lr == 5) || (p->dtype == SFFT_F32 && p->log2n == 12 && lr == 6);
    } else {
        fam = SFFT_KERNEL_LDG;
        lr = interleaved ? p->lr_ldg_il : p->lr;
    }
    if (family) *family = fam;
    if (log2_radix) *log2_radix = lr;
    if (warp) *warp = w;
    return SFFT_OK;
}

int sfft_exec_schedule(const sfft_plan *p, int64_t batch, int interleaved, int *launches, int *sweeps)
{
    if (!p) return fail(SFFT_EINVAL, "plan is NULL");
    if (batch < 0) return fail(SFFT_EINVAL, "batch must be >= 0, got %lld", (long long)batch);
    int nl = 1, ns = 1;
    if (p->log2n > kFusedMaxLog) nl = ns = (int)p->groups.size();
    if (p->fuse2 && !interleaved) nl = ns = 2;
    if (launches) *launches = nl;
    if (sweeps) *sweeps = ns;
    return SFFT_OK;
}

int sfft_workspace_bytes(const sfft_plan *p, int64_t batch, size_t *bytes)
{
    if (!p) return fail(SFFT_EINVAL, "plan is NULL");
    if (!bytes) return fail(SFFT_EINVAL, "bytes is NULL");
    if (batch < 0) return fail(SFFT_EINVAL, "batch must be >= 0, got %lld", (long long)batch);
    if (p->log2n <= kFusedMaxLog) {
        *bytes = 0;
        return SFFT_OK;
    }
    const size_t esz = p->dtype == SFFT_F32 ? 4 : 8;
    const size_t planes = p->groups.size() >= 3 ? 4 : 2;   // ping-pong A (and B)
    *bytes = planes * (size_t)batch * ((size_t)1 << p->log2n) * esz;
    if (p->fuse2) *bytes += kPass2CtrBytes;   // tile tickets + per-slot counters after the planes
    return SFFT_OK;
}

int sfft_exec_split(const sfft_plan *plan, const void *x_re, const void *x_im, void *y_re, void *y_im,
                    int64_t batch, int64_t in_stride, int64_t out_stride, int direction, void *workspace,
                    void *stream)
{
    return exec_common(plan, x_re, x_im, y_re, y_im, false, batch, in_stride, out_stride, direction, workspace,
                       stream);
}

// transform.py:88-120 (butterfly_stage / twiddle_stage) on the interleaved
// layout, batched over rows; see sfft_stage.cuh.
static int exec_stage(int kind, int dtype, int log2n, int stage, const sfft_plan *p, void *data, int64_t batch,
                      int64_t stride, int device, void *stream)
{
    if (log2n < 0 || log2n > SFFT_MAX_LOG2N) return fail(SFFT_EINVAL, "stage count m must be >= 0, got %d", log2n);
    if (stage < 1 || stage > log2n) return fail(SFFT_EINVAL, "stage index %d out of range for m=%d", stage, log2n);
    if (dtype != SFFT_F32 && dtype != SFFT_F64) return fail(SFFT_EINVAL, "unknown dtype %d", dtype);
    if (batch < 0) return fail(SFFT_EINVAL, "batch must be >= 0, got %lld", (long long)batch);
    const int64_t n = int64_t(1) << log2n;
    if (batch > 1 && stride < n) return fail(SFFT_EINVAL, "row stride %lld must be >= N = %lld", (long long)stride, (long long)n);
    if (batch == 0 || (kind == 1 && stage == 1)) return SFFT_OK;   // the stage-1 rotation is the identity
    if (!data) return fail(SFFT_EINVAL, "NULL data pointer");
    if (batch > 65535) return fail(SFFT_ECAPACITY, "batch %lld exceeds one stage launch (65535 rows)", (long long)batch);
    DeviceGuard dg(device);
    if (dg.err != cudaSuccess) return cuda_fail(dg.err, "cudaSetDevice");
    const int64_t half = n >> 1;
    const dim3 grid((unsigned)((half + 255) / 256), (unsigned)batch);
    cudaStream_t st = (cudaStream_t)stream;
    if (dtype == SFFT_F64) {
        TwCat<double> tw{(const double2 *)(p ? p->d_tw : nullptr)};
        if (kind == 0) sfft_stage_kernel<double, 0><<<grid, 256, 0, st>>>((double2 *)data, stride, log2n, stage, tw);
        else sfft_stage_kernel<double, 1><<<grid, 256, 0, st>>>((double2 *)data, stride, log2n, stage, tw);
    } else if (kind == 0 || !p || stage <= p->cat_top) {
        TwCat<float> tw{(const float2 *)(p ? p->d_tw : nullptr)};
        if (kind == 0) sfft_stage_kernel<float, 0><<<grid, 256, 0, st>>>((float2 *)data, stride, log2n, stage, tw);
        else sfft_stage_kernel<float, 1><<<grid, 256, 0, st>>>((float2 *)data, stride, log2n, stage, tw);
    } else {
        // fp32 plans above the stage-major table: the two-level factors the
        // pass kernels use (sfft_common.cuh TwTwoLevel)
        TwTwoLevel<float> tw;
        tw.tab = (const float2 *)p->d_tw;
        tw.cat_top = p->cat_top;
        tw.coarse = p->d_coarse;
        tw.coarse_log = p->coarse_log;
        tw.fine = p->d_fine;
        tw.m = p->log2n;
        sfft_stage_kernel<float, 1><<<grid, 256, 0, st>>>((float2 *)data, stride, log2n, stage, tw);
    }
    count_launch();
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? SFFT_OK : cuda_fail(e, "stage kernel launch");
}

int sfft_exec_butterfly_stage(int dtype, int log2n, int stage, void *data, int64_t batch, int64_t stride,
                              int device, void *stream)
{
    return exec_stage(0, dtype, log2n, stage, nullptr, data, batch, stride, device, stream);
}

int sfft_exec_twiddle_stage(const sfft_plan *p, int stage, void *data, int64_t batch, int64_t stride, void *stream)
{
    if (!p) return fail(SFFT_EINVAL, "plan is NULL");
    return exec_stage(1, p->dtype, p->log2n, stage, p, data, batch, stride, p->device, stream);
}

int sfft_exec_interleaved(const sfft_plan *plan, const void *x, void *y, int64_t batch, int64_t in_stride,
                          int64_t out_stride, int direction, void *workspace, void *stream)
{
    return exec_common(plan, x, nullptr, y, nullptr, true, batch, in_stride, out_stride, direction, workspace,
                       stream);
}

/* ---------------- sharded four-step (one transform over nranks GPUs) ------------- */

struct sfft_dist_plan {
    sfft_plan *base = nullptr;   // tables of the full-size plan
    int nranks = 1, rank = 0, logg = 0, L1 = 0;
    std::vector<Group> ga, gb;   // phase 0: stages 1..L1, phase 1: L1+1..m (split_range)
};

int sfft_dist_plan_create(int log2n, int dtype, int nranks, int rank, int device, sfft_dist_plan **out)
{
    if (!out) return fail(SFFT_EINVAL, "out is NULL");
    *out = nullptr;
    if (nranks < 1 || (nranks & (nranks - 1)))
        return fail(SFFT_EINVAL, "nranks must be a power of two >= 1, got %d", nranks);
    if (rank < 0 || rank >= nranks) return fail(SFFT_EINVAL, "rank %d out of range for %d ranks", rank, nranks);
    int logg = 0;
    while ((1 << logg) < nranks) ++logg;
    if (log2n < 0) return fail(SFFT_EINVAL, "stage count m must be >= 0, got %d", log2n);
    if (log2n > SFFT_MAX_LOG2N)
        return fail(SFFT_ECAPACITY, "m=%d exceeds the plan limit max_m=%d", log2n, SFFT_MAX_LOG2N);
    if (dtype != SFFT_F32 && dtype != SFFT_F64) return fail(SFFT_EINVAL, "unknown dtype %d", dtype);
    const int tjlog = dtype == SFFT_F32 ? 5 : 4;
    const int L1 = log2n / 2, L2 = log2n - L1;
    if (L1 < kPassMinL || L1 - logg < tjlog || L2 - logg < tjlog)
        return fail(SFFT_ECAPACITY, "a sharded transform over %d ranks needs log2n >= %d, got %d", nranks,
                    2 * (tjlog + logg > kPassMinL ? tjlog + logg : kPassMinL), log2n);
    // the full-size plan provides the stage tables (stage-major up to its
    // cat_top, which covers every stage for log2n <= 12)
    sfft_plan *base = nullptr;
    int rc = sfft_plan_create_ex(log2n, dtype, SFFT_DIT, device, SFFT_MAX_LOG2N, 0, SFFT_KERNEL_AUTO, &base);
    if (rc) return rc;
    sfft_dist_plan *d = new sfft_dist_plan;
    d->base = base;
    d->nranks = nranks;
    d->rank = rank;
    d->logg = logg;
    d->L1 = L1;
    d->ga = split_range(0, L1);
    d->gb = split_range(L1, L2);
    *out = d;
    return SFFT_OK;
}

int sfft_dist_plan_destroy(sfft_dist_plan *d)
{
    if (!d) return SFFT_OK;
    sfft_plan_destroy(d->base);
    delete d;
    return SFFT_OK;
}

int sfft_dist_layout(const sfft_dist_plan *d, int64_t *local_elems, int *log2n1, int64_t *segment_elems)
{
    if (!d) return fail(SFFT_EINVAL, "plan is NULL");
    const int64_t n = int64_t(1) << d->base->log2n;
    if (local_elems) *local_elems = n >> d->logg;
    if (log2n1) *log2n1 = d->L1;
    if (segment_elems) *segment_elems = n >> (2 * d->logg);
    return SFFT_OK;
}

int sfft_dist_schedule(const sfft_dist_plan *d, int *launches_phase0, int *launches_phase1)
{
    if (!d) return fail(SFFT_EINVAL, "plan is NULL");
    if (launches_phase0) *launches_phase0 = (int)d->ga.size();
    if (launches_phase1) *launches_phase1 = (int)d->gb.size();
    return SFFT_OK;
}

int sfft_dist_workspace_bytes(const sfft_dist_plan *d, size_t *bytes)
{
    if (!d || !bytes) return fail(SFFT_EINVAL, "NULL argument");
    const size_t esz = d->base->dtype == SFFT_F32 ? 4 : 8;
    *bytes = 4 * ((size_t)1 << (d->base->log2n - d->logg)) * esz;
    return SFFT_OK;
}

static int dist_exec(const sfft_dist_plan *d, int phase, const void *x_re, const void *x_im, void *y_re,
                     void *y_im, int direction, void *workspace, void *stream, void *const *peer_re,
                     void *const *peer_im, int npeers);

int sfft_dist_exec_phase(const sfft_dist_plan *d, int phase, const void *x_re, const void *x_im, void *y_re,
                         void *y_im, int direction, void *workspace, void *stream)
{
    return dist_exec(d, phase, x_re, x_im, y_re, y_im, direction, workspace, stream, nullptr, nullptr, 0);
}

int sfft_dist_exec_phase0_p2p(const sfft_dist_plan *d, const void *x_re, const void *x_im, void *const *peer_re,
                              void *const *peer_im, int npeers, int direction, void *workspace, void *stream)
{
    if (!d) return fail(SFFT_EINVAL, "plan is NULL");
    if (npeers != d->nranks || npeers > 8 || !peer_re || !peer_im)
        return fail(SFFT_EINVAL, "need one receive buffer per rank (%d, at most 8), got %d", d->nranks, npeers);
    for (int h = 0; h < npeers; ++h)
        if (!peer_re[h] || !peer_im[h]) return fail(SFFT_EINVAL, "NULL receive buffer of rank %d", h);
    // y is unused by the last launch (it stores to the peers); earlier launches use the workspace
    return dist_exec(d, 0, x_re, x_im, peer_re[0], peer_im[0], direction, workspace, stream, peer_re, peer_im,
                     npeers);
}

static int dist_exec(const sfft_dist_plan *d, int phase, const void *x_re, const void *x_im, void *y_re,
                     void *y_im, int direction, void *workspace, void *stream, void *const *peer_re,
                     void *const *peer_im, int npeers)
{
    if (!d) return fail(SFFT_EINVAL, "plan is NULL");
    if (phase != 0 && phase != 1) return fail(SFFT_EINVAL, "phase must be 0 or 1, got %d", phase);
    if (direction != SFFT_FORWARD && direction != SFFT_INVERSE)
        return fail(SFFT_EINVAL, "direction must be -1 (forward) or +1 (inverse), got %d", direction);
    if (!x_re || !x_im || !y_re || !y_im) return fail(SFFT_EINVAL, "NULL signal pointer");
    const std::vector<Group> &gs = phase == 0 ? d->ga : d->gb;
    if (gs.size() > 1 && !workspace) return fail(SFFT_EINVAL, "this phase needs a workspace (sfft_dist_workspace_bytes)");
    const sfft_plan *p = d->base;
    DeviceGuard dg(p->device);
    if (dg.err != cudaSuccess) return cuda_fail(dg.err, "cudaSetDevice");
    const int m = p->log2n, b = d->logg, L1 = d->L1;
    const int64_t n = int64_t(1) << m, nl = n >> b;
    const size_t esz = p->dtype == SFFT_F32 ? 4 : 8;
    char *ws = (char *)workspace;
    void *bufA[2] = {ws, ws + nl * esz};
    void *bufB[2] = {ws + 2 * nl * esz, ws + 3 * nl * esz};
    const bool inv = direction == SFFT_INVERSE;
    const int G = (int)gs.size();
    for (int k = 0; k < G; ++k) {
        const Group gr = gs[k];
        const int TJ = pass_tile(p->dtype, gr.L);
        PassLaunchFn fn = pass_launcher(p->dtype, gr.L);
        if (!fn) return fail(SFFT_EINVAL, "no pass kernel for L=%d", gr.L);
        PassArgs a;
        memset(&a, 0, sizeof a);
        const bool first = k == 0, last = k == G - 1;
        void **src = (k % 2 == 1) ? bufA : bufB;
        void **dst = (k % 2 == 0) ? bufA : bufB;
        a.x0 = first ? x_re : src[0];
        a.x1 = first ? x_im : src[1];
        a.y0 = last ? y_re : dst[0];
        a.y1 = last ? y_im : dst[1];
        a.batch = 1;
        a.in_stride = a.out_stride = nl;
        a.m = m;
        a.S = gr.S;
        a.swap_in = phase == 0 && first && inv;
        a.swap_out = phase == 1 && last && inv;
        a.scale = (phase == 1 && last && inv) ? 1.0 / (double)n : 1.0;
        a.tw = p->d_tw;
        a.tw_cat_top = p->cat_top;
        a.tw_top_tab = p->d_top;
        a.coarse = p->d_coarse;
        a.coarse_log = p->coarse_log;
        a.fine = p->d_fine;
        a.jb = b;
        a.jrank = d->rank;
        if (phase == 0) {
            // owner field = top b bits of the column index n2 = (index >> s) mod 2^(m-L1)
            a.jpos = gr.S + (m - L1) - b;
            a.in_map = {b, gr.S + (m - L1) - b, -1, m - b};
            if (last) a.out_map = {b, m - b, L1 - b, m - b};   // send layout [dest][n2_local][k1_local]
            else a.out_map = {b, gr.S + gr.L + (m - L1) - b, -1, m - b};
            if (last && npeers > 0) {   // fused exchange: store into the peers' receive buffers
                a.npeers = npeers;
                a.seg_log = m - 2 * b;
                for (int h = 0; h < npeers; ++h) {
                    a.peer_re[h] = peer_re[h];
                    a.peer_im[h] = peer_im[h];
                }
            }
        } else {
            // owner field = top b bits of k1 = index mod 2^L1
            a.jpos = L1 - b;
            a.in_map = {b, L1 - b, -1, m - b};
            a.out_map = {b, L1 - b, -1, m - b};
        }
        const int64_t grid = ((n >> gr.L) >> b) / TJ;
        cudaError_t e = fn(a, false, false, false, grid, (cudaStream_t)stream);
        if (e != cudaSuccess) return cuda_fail(e, "pass kernel launch (sharded)");
    }
    return SFFT_OK;
}

}  // extern "C"
