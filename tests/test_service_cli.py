"""Service / CLI routing and signal files (row 4).

CPU part: the JSON contract, status-code mapping and file formats, all
decided before any device work.  GPU part (-m gpu): the reference's inline
known answers through the service and the CLI (test_service.py:25-33,
test_cli.py:25-63), and the pinned .bin fast path byte-for-byte against the
reference's output from the golden file.
"""

import os
import subprocess
import sys

import numpy as np
import pytest
import torch
from fastapi.testclient import TestClient

import paper_2504_07264_b200 as sf
from paper_2504_07264_b200 import signalio
from paper_2504_07264_b200.service import create_app

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_vectors.npz"))


@pytest.fixture(scope="module")
def client():
    return TestClient(create_app())


def run_cli(*args):
    return subprocess.run([sys.executable, "-m", "paper_2504_07264_b200", *map(str, args)],
                          capture_output=True, text=True, cwd=ROOT)


def write_csv(path, rows):
    path.write_text("".join(f"{r},{i}\n" for r, i in rows))


# ------------------------------------------------------------------ CPU ---

def test_health(client):
    body = client.get("/health").json()
    assert body["status"] == "ok" and body["version"] == sf.__version__


def test_schema_violations_are_422(client):
    assert client.post("/transform", json={"re": [1, 2]}).status_code == 422
    assert client.post("/transform", json={"re": [1], "im": [0], "algorithm": "fast"}).status_code == 422


def test_value_errors_are_400(client):
    r = client.post("/transform", json={"re": [1, 2, 3], "im": [0, 0, 0]})
    assert r.status_code == 400 and "power of two" in r.json()["detail"]
    r = client.post("/transform", json={"re": [1, 2], "im": [0, 0, 0, 0]})
    assert r.status_code == 400 and "channel lengths differ" in r.json()["detail"]


def test_cli_non_power_of_two_exits_2(tmp_path):
    src = tmp_path / "six.csv"
    write_csv(src, [(k, 0) for k in range(6)])
    proc = run_cli("transform", src, tmp_path / "out.csv")
    assert proc.returncode == 2
    assert "6" in proc.stderr and "power of two" in proc.stderr
    assert not (tmp_path / "out.csv").exists()


def test_cli_unreadable_input_exits_1(tmp_path):
    bad = tmp_path / "bad.csv"
    bad.write_text("re,im\n1,2\nnot,a,pair\n")
    proc = run_cli("transform", bad, tmp_path / "out.csv")
    assert proc.returncode == 1 and "line 3" in proc.stderr


def test_csv_round_trip_is_exact(tmp_path):
    rng = np.random.default_rng(5)
    re, im = rng.standard_normal(16), rng.standard_normal(16)
    re[2] = -0.0
    signalio.write_signal(tmp_path / "a.csv", sf.SplitSignal(re, im))
    back = signalio.read_signal(tmp_path / "a.csv")
    assert np.array_equal(np.asarray(back.re).view(np.int64), re.view(np.int64))
    assert np.array_equal(np.asarray(back.im), im)


def test_bin_layout_is_little_endian_interleaved(tmp_path):
    re, im = np.array([1.0, 2.0]), np.array([3.0, 4.0])
    signalio.write_signal(tmp_path / "a.bin", sf.SplitSignal(re, im))
    raw = np.fromfile(tmp_path / "a.bin", dtype="<f8")
    assert raw.tolist() == [1.0, 3.0, 2.0, 4.0]
    back = signalio.read_signal(tmp_path / "a.bin")
    assert back.re.tolist() == [1.0, 2.0] and back.im.tolist() == [3.0, 4.0]
    (tmp_path / "odd.bin").write_bytes(np.zeros(3).tobytes())
    with pytest.raises(signalio.SignalReadError, match="whole"):
        signalio.read_signal(tmp_path / "odd.bin")
    with pytest.raises(signalio.SignalReadError, match="infer"):
        signalio.detect_format("x.txt")


# ------------------------------------------------------------------ GPU ---

@pytest.mark.gpu
def test_service_known_answer(client):
    resp = client.post("/transform", json={"re": [1, 2, 3, 4], "im": [0, 0, 0, 0]})
    assert resp.status_code == 200
    body = resp.json()
    assert body["re"] == [10.0, -2.0, -2.0, -2.0] and body["im"] == [0.0, 2.0, 0.0, -2.0]
    assert body["m"] == 2 and body["algorithm"] == "dit" and body["inverse"] is False


@pytest.mark.gpu
def test_service_batch_and_inverse(client):
    rng = np.random.default_rng(4)
    re = rng.standard_normal((3, 32))
    im = rng.standard_normal((3, 32))
    f = client.post("/transform", json={"re": re.tolist(), "im": im.tolist(), "algorithm": "dif"}).json()
    b = client.post("/transform", json={"re": f["re"], "im": f["im"], "inverse": True}).json()
    assert np.max(np.abs(np.array(b["re"]) - re)) <= 1e-12


@pytest.mark.gpu
def test_cli_four_point_exact_output(tmp_path):
    src, dst = tmp_path / "ramp.csv", tmp_path / "out.csv"
    write_csv(src, [(1, 0), (2, 0), (3, 0), (4, 0)])
    proc = run_cli("transform", src, dst)
    assert proc.returncode == 0, proc.stderr
    assert dst.read_text() == "10,0\n-2,2\n-2,0\n-2,-2\n"
    src2 = tmp_path / "impulse.csv"
    write_csv(src2, [(1, 0)] + [(0, 0)] * 7)
    assert run_cli("transform", src2, dst).returncode == 0
    assert dst.read_text() == "1,0\n" * 8


@pytest.mark.gpu
@pytest.mark.parametrize("algo", ["dit", "dif"])
def test_direct_bin_path_matches_reference_bytes(tmp_path, algo):
    m = 12
    x = np.empty(2 << m)
    x[0::2] = GOLD[f"m{m}_x_re"][0]
    x[1::2] = GOLD[f"m{m}_x_im"][0]
    x.astype("<f8").tofile(tmp_path / "in.bin")
    proc = run_cli("transform", tmp_path / "in.bin", tmp_path / "out.bin", "--direct", "--algorithm", algo)
    assert proc.returncode == 0, proc.stderr
    want = np.empty(2 << m)
    want[0::2] = GOLD[f"m{m}_{algo}_fwd_re"][0]
    want[1::2] = GOLD[f"m{m}_{algo}_fwd_im"][0]
    assert (tmp_path / "out.bin").read_bytes() == want.astype("<f8").tobytes()
    # the JSON route writes the same file
    proc = run_cli("transform", tmp_path / "in.bin", tmp_path / "out2.bin", "--algorithm", algo)
    assert proc.returncode == 0 and (tmp_path / "out2.bin").read_bytes() == want.astype("<f8").tobytes()
