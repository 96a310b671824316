// sfft_launch.h -- host-side launcher registry shared by the generated
// instantiation units (sfft_inst_*.cu) and the C ABI (sfft_abi.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace sfft {

struct FusedArgs;
struct PassArgs;
struct TmaLaunch;
struct Pass2Args;

// Launch one fused kernel (N = 2^logn <= 4096) over a.batch rows.
using FusedLaunchFn = cudaError_t (*)(const FusedArgs &a, bool dif, bool interleaved, cudaStream_t st);
// Launch one pass group (2^L-point sub-problems) over a.batch rows.
using PassLaunchFn = cudaError_t (*)(const PassArgs &a, bool dif, bool il_in, bool il_out,
                                     int64_t grid, cudaStream_t st);

// Launch one L2-fused group pair (sfft_pass2.cuh), persistent grid capped at
// `items` CTAs (the launcher zeroes nothing: a.ctr must be zero).
using Pass2LaunchFn = cudaError_t (*)(const Pass2Args &a, int64_t items, cudaStream_t st);

// Launch the persistent TMA-fed fused kernel (planar, 16-byte aligned rows).
using TmaLaunchFn = cudaError_t (*)(const TmaLaunch &L, cudaStream_t st);


constexpr int kFusedMaxLog = 12;
constexpr int kMaxRadixLog = 5;
constexpr int kPassMinL = 4, kPassMaxL = 10;

// Registry lookups (nullptr when the combination was not instantiated).
// dtype: 0 = f32, 1 = f64.  Interleaved variants exist only for the
// default radix of each size.  The returned fused launcher is bound to
// (dif, il) already and ignores those two arguments.
FusedLaunchFn fused_launcher_algo(int dtype, int logn, int lr, bool dif, bool il, bool pre = false);
int fused_default_lr(int dtype, int logn);
PassLaunchFn pass_launcher(int dtype, int L);
int pass_tile(int dtype, int L);    // TJ: sub-problems per CTA of a 2^L-point group
int pass_default_lr(int dtype);
PassLaunchFn pass_launcher_f32(int L);
PassLaunchFn pass_launcher_f64(int L);
Pass2LaunchFn pass2_launcher(int dtype, int L1, int L2, bool dif, bool sz);
Pass2LaunchFn pass2_launcher_f32(int L1, int L2, bool dif, bool sz);
Pass2LaunchFn pass2_launcher_f64(int L1, int L2, bool dif, bool sz);

TmaLaunchFn tma_launcher(int dtype, int logn, int lr, bool dif, bool pre = false);
TmaLaunchFn tma_launcher_f32(int logn, int lr, bool dif, bool pre);
TmaLaunchFn tma_launcher_f64(int logn, int lr, bool dif, bool pre);
int tma_default_lr(int dtype, int logn);   // -1: no TMA config for this size
// kernel=auto pick, 0 <= logn <= 12: family 0 = LDG fused, 1 = TMA
void auto_choice(int dtype, int logn, int *family, int *lr, bool *pre);
void auto_small_batch(int dtype, int logn, int *lr, long long *below);
void count_launch();

}  // namespace sfft
