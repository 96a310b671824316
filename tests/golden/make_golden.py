"""Generate the golden vectors in tests/golden/ from the REFERENCE itself.

Run in the build container only (it imports the read-only reference from
/root/reference/pkg/src; that tree does not exist on the GPU box, which only
reads the committed .npz files):

    python tests/golden/make_golden.py

Every output is produced by the reference's own public API (make_plan, fft,
fft_dif, ifft, interleave/deinterleave, build_twiddle_table, count_flops,
bit_reverse_indices), on seeded inputs.  The oracle (oracle/) and the GPU
path are pinned against these files.
"""

import importlib.util
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = "/root/reference/pkg/src/splitfft"
sys.path.insert(0, ROOT)


def load_reference():
    spec = importlib.util.spec_from_file_location(
        "splitfft_ref", os.path.join(REF, "__init__.py"), submodule_search_locations=[REF])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["splitfft_ref"] = mod
    spec.loader.exec_module(mod)
    return mod


def ref_split(sf, plan, re, im, inverse=False):
    buf = sf.interleave(sf.SplitSignal(re, im))
    (sf.ifft if inverse else sf.fft)(plan, buf)
    out = sf.deinterleave(buf)
    return out.re, out.im


def batch(sf, m, algo, re, im, inverse=False):
    plan = sf.make_plan(m, algo)
    yr = np.empty(re.shape)
    yi = np.empty(re.shape)
    for b in range(re.shape[0]):
        yr[b], yi[b] = ref_split(sf, plan, re[b], im[b], inverse)
    return yr, yi


def main():
    sf = load_reference()
    import workloads

    out = {}
    # 1. random signals for every fused size and two multi-pass sizes
    for m in list(range(0, 13)) + [13, 14]:
        rng = np.random.default_rng(900 + m)
        b = 3 if m <= 12 else 1
        re = rng.standard_normal((b, 1 << m))
        im = rng.standard_normal((b, 1 << m))
        out[f"m{m}_x_re"], out[f"m{m}_x_im"] = re, im
        for algo in ("dit", "dif"):
            for inv in (False, True):
                tag = f"m{m}_{algo}_{'inv' if inv else 'fwd'}"
                out[tag + "_re"], out[tag + "_im"] = batch(sf, m, algo, re, im, inv)

    # 2. BASELINE configs[0] in full: N=8 fp64 B=1024 U[-1,1) seed 0
    c1 = workloads.CONFIGS["cfg1_n8_f64"]
    re, im = workloads.generate(c1)
    out["cfg1_x_re"], out["cfg1_x_im"] = re, im
    out["cfg1_dit_re"], out["cfg1_dit_im"] = batch(sf, 3, "dit", re, im)
    out["cfg1_dif_re"], out["cfg1_dif_im"] = batch(sf, 3, "dif", re, im)

    # 3. prefixes of configs 2-4 (fp32 inputs, upcast exactly, layout.py:29-30)
    for name, rows in (("cfg2_n64_f32", 16), ("cfg3_n1024_f32", 4), ("cfg3_n1024_f64", 4),
                       ("cfg4_n4096_f32", 2)):
        c = workloads.CONFIGS[name]
        re, im = workloads.generate(c, rows=rows)
        out[f"{name}_x_re"], out[f"{name}_x_im"] = re, im
        out[f"{name}_dit_re"], out[f"{name}_dit_im"] = batch(
            sf, c.log2n, "dit", re.astype(np.float64), im.astype(np.float64))

    # 4. tables and census
    for m in (1, 2, 3, 6, 12, 16):
        plan = sf.make_plan(m)
        w = plan.stage_factors[m - 1]
        out[f"stage_factor_m{m}_re"] = np.ascontiguousarray(w.real)
        out[f"stage_factor_m{m}_im"] = np.ascontiguousarray(w.imag)
        st = plan.twiddles.stage(m)
        out[f"cos_m{m}"], out[f"sin_m{m}"] = st.cos.copy(), st.sin.copy()
    census = []
    for m in range(0, 21):
        r = sf.count_flops(sf.make_plan(m))
        census.append([m, r.real_mults, r.real_adds, r.generic_rotations, r.quarter_turns,
                       r.identity_rotations])
    out["census"] = np.array(census, dtype=np.int64)
    from splitfft_ref.layout import bit_reverse_indices
    for m in (0, 3, 5, 10):
        out[f"bitrev_m{m}"] = bit_reverse_indices(m).astype(np.int64)

    path = os.path.join(HERE, "reference_vectors.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(out)} arrays, {os.path.getsize(path) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
