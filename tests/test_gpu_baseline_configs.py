"""Parity at the full BASELINE.json configs: the CUDA path vs the float64 oracle.

Every shape and batch the bench reports is checked here against
``oracle.gemv_reference_batch`` (linear.py:177-208 restated in C, float64, no dense
matrix) on the same fp16-rounded activations -- not against the repo's own dequantize.
Weights follow the BASELINE idiom: random trits, per-channel
gamma_r = fp16(0.02 (1 + U)), packed by tr_quantize_pack (bit-exact with the oracle's
pack_matrix, tests/test_gpu_parity.py) and read back for the oracle.

Tolerance (north star: max rel err <= 1e-2; cli.py:87-96 metric, per vector
max |y - ref| / max |ref|): asserted at 2e-3 for fp16 and 6e-3 for bf16 outputs.
"""

from __future__ import annotations

import numpy as np
import pytest

import oracle as orc

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def tp():
    import paper_2506_23025_b200 as tp

    return tp


def rel_err(y, ref):
    y = np.asarray(y, np.float64)
    ref = np.asarray(ref, np.float64)
    den = np.max(np.abs(ref), axis=-1)
    den = np.where(den == 0, 1.0, den)
    return float(np.max(np.max(np.abs(y - ref), axis=-1) / den))


_CACHE: dict = {}


def _weight(tp, rows, cols, fmt, seed):
    """(TernaryWeight, payload, scales) for a BASELINE-style random ternary matrix (cached per module)."""
    key = (rows, cols, int(fmt), seed)
    if key not in _CACHE:
        _CACHE.clear()   # keep one large matrix alive at a time
        g = torch.Generator(device="cuda").manual_seed(seed)
        T = torch.randint(0, 3, (rows, cols), generator=g, device="cuda", dtype=torch.int8).float() - 1
        gam = (0.02 * (1 + torch.rand((rows, 1), generator=g, device="cuda"))).half().float()
        w = tp.TernaryWeight.from_float(gam * T, fmt)
        del T
        p, s = w.unpack()
        _CACHE[key] = (w, p.cpu().numpy(), s.cpu().numpy())
    return _CACHE[key]


def _x(batch, cols, seed, dtype=torch.float16):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return (torch.rand(batch, cols, generator=g, device="cuda") * 2 - 1).to(dtype)


def _check(tp, rows, cols, fmt, batch, dtype="float16", path="auto", seed=0):
    w, payload, scales = _weight(tp, rows, cols, fmt, seed)
    x = _x(batch, cols, seed + batch, getattr(torch, dtype))
    y = tp.linear(x, w, path=path).float().cpu().numpy()
    ref = orc.gemv_reference_batch(payload, scales, cols, int(fmt), x.float().cpu().numpy())
    err = rel_err(y, ref)
    assert err <= (2e-3 if dtype == "float16" else 6e-3), f"{rows}x{cols} b={batch} {dtype}: rel err {err:.3e}"
    return err


# configs[0] / configs[1]: 4096x4096, batch 1, fp16, per-channel scale
def test_config1_4096sq_b1(tp):
    _check(tp, 4096, 4096, tp.DType.TQ2, 1)


# configs[1]: the Llama shapes over the whole batch sweep (GEMV and tcgen05 GEMM paths)
@pytest.mark.parametrize("rows,cols", [(11008, 4096), (4096, 11008), (4096, 4096)])
@pytest.mark.parametrize("batch", [1, 2, 4, 8, 16, 32, 64, 128])
def test_config2_llama_sweep(tp, rows, cols, batch):
    _check(tp, rows, cols, tp.DType.TQ2, batch)


@pytest.mark.parametrize("batch", [1, 4, 16, 128])
def test_config2_llama_sweep_bf16(tp, batch):
    _check(tp, 11008, 4096, tp.DType.TQ2, batch, dtype="bfloat16")


# configs[3]: TQ1 (1.6 bit) 8192x8192 decoded on the fly, batch 1..8
@pytest.mark.parametrize("batch", [1, 2, 4, 8, 16])
@pytest.mark.parametrize("dtype", ["float16", "bfloat16"])
def test_config4_tq1_8192(tp, batch, dtype):
    _check(tp, 8192, 8192, tp.DType.TQ1, batch, dtype=dtype)


# configs[4]: 70B layer shapes on one GPU
@pytest.mark.parametrize("rows,cols", [(28672, 8192), (8192, 28672)])
@pytest.mark.parametrize("batch", [1, 16])
def test_config5_70b_shapes(tp, rows, cols, batch):
    _check(tp, rows, cols, tp.DType.TQ2, batch)


# configs[4]: row-parallel recombination at the real 70B down-projection width: the 256-block
# K shards (parallel.shard_cols) of 8192x28672 at TP 2/4/8, each product on the GPU with an
# fp32 partial, summed in rank order (what the all-reduce computes), vs the float64 oracle
@pytest.mark.parametrize("tpn", [2, 4, 8])
@pytest.mark.parametrize("batch", [1, 16])
def test_config5_row_parallel_recombination(tp, tpn, batch):
    from paper_2506_23025_b200.parallel import shard_bounds

    rows, cols = 8192, 28672
    w, payload, scales = _weight(tp, rows, cols, tp.DType.TQ2, 0)
    x = _x(batch, cols, 99 + batch)
    nb = cols // 256
    total = torch.zeros(batch, rows, dtype=torch.float32, device="cuda")
    for i in range(tpn):
        b0, b1 = shard_bounds(nb, tpn, i)
        pm = tp.PackedMatrix(rows=rows, cols=(b1 - b0) * 256, fmt=tp.DType.TQ2,
                             payload=np.ascontiguousarray(payload[:, b0:b1]), scales=np.ascontiguousarray(scales[:, b0:b1]))
        ws = pm.to_device()
        part = tp.linear(x[:, b0 * 256:b1 * 256].contiguous(), ws, out_dtype=torch.float32)
        assert part.dtype == torch.float32
        total += part
        del ws
    ref = orc.gemv_reference_batch(payload, scales, cols, 2, x.float().cpu().numpy())
    err = rel_err(total.cpu().numpy(), ref)
    assert err <= 1e-3, f"TP{tpn} b={batch}: rel err {err:.3e}"


# configs[2]: the 3.9B decoder's layer shapes (d 3072, qkv 9216, SwiGLU 9216) at decode batch 1
@pytest.mark.parametrize("rows,cols", [(9216, 3072), (3072, 3072), (18432, 3072), (3072, 9216)])
def test_config3_decoder_layer_shapes(tp, rows, cols):
    _check(tp, rows, cols, tp.DType.TQ2, 1)


# the bench's timed stack itself (bench.make_stack_weights + graph.LinearStack): activations stay
# finite through the chained layers (its synthetic gamma keeps each layer's RMS; a fixed 0.02-0.04
# had overflowed fp16 to NaN from layer 16 on), and the last layer matches the oracle on the input
# the chain actually fed it
@pytest.mark.parametrize("batch,dtype", [(1, "float16"), (16, "float16"), (4, "bfloat16")])
def test_bench_stack_finite_and_last_layer_vs_oracle(tp, batch, dtype):
    import bench
    from paper_2506_23025_b200.graph import LinearStack

    dt = getattr(torch, dtype)
    ws = bench.make_stack_weights(8, seed=1234)   # 24 chained layers
    st = LinearStack(ws, batch=batch, dtype=dt)
    st.x.copy_(bench.uniform_x(batch, st.x.shape[1], 4242 + batch, dt))
    st.replay()
    torch.cuda.synchronize()
    for i, o in enumerate(st.bufs):
        assert bool(torch.isfinite(o).all()), f"layer {i}: non-finite output"
        m = float(o.float().abs().max())
        assert 0.1 < m < 100.0, f"layer {i}: |y|max {m:.3g} drifted"
    w = ws[-1]
    p, s = w.unpack()
    ref = orc.gemv_reference_batch(p.cpu().numpy(), s.cpu().numpy(), w.cols, int(w.fmt),
                                   st.bufs[-2].float().cpu().numpy())
    err = rel_err(st.bufs[-1].float().cpu().numpy(), ref)
    assert err <= (2e-3 if dtype == "float16" else 6e-3), f"last layer b={batch} {dtype}: rel err {err:.3e}"
