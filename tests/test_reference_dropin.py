"""The drop-in at the reference's own boundary, on the GPU.

The UNMODIFIED reference package (installed into baseline/_ref by
`pip install --target baseline/_ref`, git-ignored, travels to the GPU box) gets our
`cuda_kernels` module registered in its backend registry (backend.py:23-26) exactly as
INTEGRATION.md shows; then the reference's own callers run on the B200:
`linear.gemm` (bit-identical to its compiled backend, any thread sharding),
`pack_matrix` / `quantize_rows`, and `tritpack.cli verify` on a reference-written TPK1 file.
"""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def tritpack():
    if not os.path.isdir(os.path.join(REF, "tritpack")):
        pytest.skip("reference not installed in baseline/_ref")
    sys.path.insert(0, REF)
    import tritpack
    from tritpack import backend

    from paper_2506_23025_b200 import cuda_kernels   # the three-line binding of INTEGRATION.md
    backend._BY_NAME["cuda"] = cuda_kernels
    yield tritpack
    backend._BY_NAME.pop("cuda", None)


@pytest.mark.parametrize("fmt_name", ["TQ2", "TQ1"])
@pytest.mark.parametrize("rows,cols,batch,threads", [(37, 1500, 3, 1), (128, 4096, 2, 4), (300, 777, 5, 3)])
def test_reference_gemm_on_cuda_backend_is_bit_identical(tritpack, fmt_name, rows, cols, batch, threads):
    from tritpack.blocks import DType
    from tritpack.linear import gemm, pack_matrix

    rng = np.random.default_rng(rows + cols)
    W = rng.normal(size=(rows, cols)).astype(np.float32)
    fmt = getattr(DType, fmt_name)
    pm = pack_matrix(W, fmt, backend="compiled")
    pm_cuda = pack_matrix(W, fmt, backend="cuda")          # quantize + pack through our kernels
    np.testing.assert_array_equal(pm_cuda.payload, pm.payload)
    np.testing.assert_array_equal(pm_cuda.scales.view(np.uint16), pm.scales.view(np.uint16))
    X = rng.uniform(-1, 1, size=(batch, cols)).astype(np.float32)
    want = gemm(pm, X, threads=threads, backend="compiled")
    got = gemm(pm, X, threads=threads, backend="cuda")
    np.testing.assert_array_equal(got.view(np.uint32), want.view(np.uint32))


def test_reference_cli_verify_on_cuda_backend(tritpack, capsys, monkeypatch):
    from tritpack import backend, cli

    monkeypatch.setenv("TRITPACK_BACKEND", "cuda")   # the CLI's --backend choices predate "cuda"
    assert backend.default_name() == "cuda"
    rc = cli.main(["verify", "--in", os.path.join(GOLDEN, "model.tpk1")])
    out = capsys.readouterr().out
    assert rc == 0, out
    assert "verified 5 tensors: OK" in out


def test_reference_own_suite_on_cuda_backend():
    """The reference's OWN test suite (pkg/tests: 281 tests, 10 acceptance criteria) with this
    repo's kernels registered as backend "cuda" and selected by TRITPACK_BACKEND=cuda
    (scripts/run_reference_suite.sh, tests/ref_cuda_plugin.py), re-run on every GPU round."""
    import subprocess

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    if not os.path.isdir(os.path.join(REF, "tritpack_tests")):
        pytest.skip("reference tests not installed next to baseline/_ref (__graft_entry__.build)")
    r = subprocess.run(["bash", os.path.join(root, "scripts", "run_reference_suite.sh")], capture_output=True,
                       text=True, timeout=900)
    tail = r.stdout[-3000:] + r.stderr[-2000:]
    assert r.returncode == 0, tail
    assert " failed" not in r.stdout and " error" not in r.stdout.splitlines()[-1], tail
    assert " passed" in r.stdout.splitlines()[-1], tail


def test_reference_reader_records_to_device(tritpack):
    """record_to_device takes the reference's OWN TensorRecord (tritpack.container.read_container)
    and the device tiles invert to the reference's PackedMatrix arrays bit for bit."""
    from tritpack.container import read_container

    from paper_2506_23025_b200.container import record_to_device

    g = np.load(os.path.join(GOLDEN, "model_tpk1.npz"))
    recs = {r.name: r for r in read_container(os.path.join(GOLDEN, "model.tpk1"))}
    for key, name in [("qkv", "layers.0.attn.qkv"), ("down", "layers.0.mlp.down"), ("up", "layers.0.mlp.up")]:
        w = record_to_device(recs[name])
        p, s = w.unpack()
        np.testing.assert_array_equal(p.cpu().numpy(), g[f"{key}_payload"])
        np.testing.assert_array_equal(s.cpu().numpy().view(np.uint16), g[f"{key}_scales"])
    import torch

    assert torch.equal(record_to_device(recs["norm"]).cpu(), torch.from_numpy(g["norm"]))
