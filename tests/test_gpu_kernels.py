"""Parity of the standalone sm_100a kernels (fold, update, momentum, tree
reduction) with the CPU oracle (oracle/restated.py) and the reference's own
golden outputs (tests/golden/tree_sums.npz).  Integer/byte-level results are
compared bit for bit: the fixed-order path has no tolerance."""

import ctypes as C
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import restated as R  # noqa: E402
from paper_1908_04207_b200 import _lib, tree_order_sum  # noqa: E402
from paper_1908_04207_b200._lib import call  # noqa: E402

DEV = "cuda:0"
CODES = {np.float32: _lib.EC_F32, np.float64: _lib.EC_F64, np.int64: _lib.EC_I64}
SIZES = [1, 3, 4, 5, 7, 8, 63, 1027, (1 << 20) + 3]


def _t(a):
    return torch.as_tensor(a, device=DEV)


def _np(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def _stream():
    return torch.cuda.current_stream().cuda_stream


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("mode", [0, 1])
def test_fold_matches_oracle(dtype, n, mode):
    rng = np.random.default_rng(n * 7 + mode)
    g = rng.standard_normal(n).astype(dtype)
    s = rng.standard_normal(n).astype(dtype)
    g[0] = -0.0
    if mode == 0:
        want = R.snapshot_leaf(g, np.zeros(n, dtype))     # null stash: 0 + g
    else:
        gb = R.GradientBuffer(s.copy())
        gb.fold(g, 0)
        want = gb.data
    st, gt = _t(s), _t(g)
    flag = torch.zeros(1, dtype=torch.int32, device=DEV)
    call("ec_fold_raw", st.data_ptr(), gt.data_ptr(), n, CODES[dtype], mode,
         C.cast(flag.data_ptr(), C.POINTER(C.c_uint32)), _stream())
    assert _np(st).tobytes() == want.tobytes()
    assert int(_np(flag)[0]) == 0


def test_fold_misaligned_and_nonfinite():
    n = 1001
    base = torch.zeros(n + 3, dtype=torch.float32, device=DEV)
    st = base[1:n + 1]                   # 4-byte aligned only: scalar path
    g = np.arange(n, dtype=np.float32)
    g[500] = np.inf
    gt = _t(g)
    flag = torch.zeros(1, dtype=torch.int32, device=DEV)
    call("ec_fold_raw", st.data_ptr(), gt.data_ptr(), n, _lib.EC_F32, 1,
         C.cast(flag.data_ptr(), C.POINTER(C.c_uint32)), _stream())
    out = _np(st)
    assert out.tobytes() == (np.zeros(n, np.float32) + g).tobytes()
    assert int(_np(flag)[0]) == 1
    assert _np(base)[0] == 0 and _np(base)[n + 1] == 0


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("n", SIZES)
def test_sgd_update_two_roundings(dtype, n):
    rng = np.random.default_rng(n)
    w = rng.standard_normal(n).astype(dtype)
    u = rng.standard_normal(n).astype(dtype)
    lr = 0.05
    want = R.sgd_update(w, u, lr)
    wt = _t(w)
    call("ec_sgd_update", wt.data_ptr(), _t(u).data_ptr(), lr, n, CODES[dtype], _stream())
    assert _np(wt).tobytes() == want.tobytes()


def test_sgd_update_is_not_fused():
    n = 1 << 16
    rng = np.random.default_rng(5)
    w = rng.standard_normal(n).astype(np.float32)
    u = rng.standard_normal(n).astype(np.float32)
    fused = (w.astype(np.float64) - np.float64(np.float32(0.05)) * u.astype(np.float64)).astype(np.float32)
    two = R.sgd_update(w, u, 0.05)
    assert (fused != two).mean() > 0.01     # the difference is observable ...
    wt = _t(w)
    call("ec_sgd_update", wt.data_ptr(), _t(u).data_ptr(), 0.05, n, _lib.EC_F32, _stream())
    assert _np(wt).tobytes() == two.tobytes()  # ... and the kernel rounds twice


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_momentum_update(dtype):
    n = 4099
    rng = np.random.default_rng(9)
    w, b, u = (rng.standard_normal(n).astype(dtype) for _ in range(3))
    want_w, want_b = R.momentum_update(w, b, u, 0.1, 0.9)
    wt, bt = _t(w), _t(b)
    call("ec_momentum_update", wt.data_ptr(), bt.data_ptr(), _t(u).data_ptr(), 0.1, 0.9, n,
         CODES[dtype], _stream())
    assert _np(bt).tobytes() == want_b.tobytes()
    assert _np(wt).tobytes() == want_w.tobytes()


def _reduce(vectors, has=None, divide=True):
    ts = [_t(v) for v in vectors]
    p = len(ts)
    out = torch.empty_like(ts[0])
    srcs = (C.c_void_p * p)(*[t.data_ptr() for t in ts])
    has = (1 << p) - 1 if has is None else has
    code = CODES[vectors[0].dtype.type]
    call("ec_local_reduce", srcs, p, has, out.data_ptr(), ts[0].numel(), code, int(divide), _stream())
    return _np(out)


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 7, 8, 13])
def test_reduce_matches_reference_golden(golden_dir, p):
    g = np.load(os.path.join(golden_dir, "tree_sums.npz"))
    # f64: the reference engine's own allreduce output (run_allreduce, sync)
    assert _reduce(list(g[f"sync_in_p{p}"])).tobytes() == g[f"sync_u_p{p}"].tobytes()
    # f32: the reference's dtype-generic tree_order_sum
    x = g[f"f32_in_p{p}"]
    assert _reduce(list(x)).tobytes() == g[f"f32_u_p{p}"].tobytes()
    assert _reduce(list(x), divide=False).tobytes() == g[f"f32_tree_p{p}"].tobytes()


def test_reduce_signed_zero_and_int(golden_dir):
    g = np.load(os.path.join(golden_dir, "tree_sums.npz"))
    for p in (1, 2, 3):
        assert _reduce(list(g[f"negzero_in_p{p}"])).tobytes() == g[f"negzero_u_p{p}"].tobytes()
    assert _reduce(list(g["i8_in_p4"])).tobytes() == g["i8_u_p4"].tobytes()


@pytest.mark.parametrize("p", [2, 3, 5, 8])
def test_reduce_null_contributions(p):
    rng = np.random.default_rng(p)
    n = 4097
    xs = [rng.standard_normal(n).astype(np.float32) for _ in range(p)]
    has = 0b101 & ((1 << p) - 1)
    contribs = [xs[r] if (has >> r) & 1 else None for r in range(p)]
    want, _, _ = R.allreduce_round(contribs, [c is not None for c in contribs], np.float32)
    assert _reduce(xs, has=has).tobytes() == want.tobytes()


def test_tree_order_sum_api_large():
    rng = np.random.default_rng(1)
    xs = [rng.standard_normal(25_559_081 // 16).astype(np.float32) for _ in range(4)]
    got = tree_order_sum([_t(x) for x in xs])
    want = R.engine_tree_sum(xs, np.float32)
    assert _np(got).tobytes() == want.tobytes()
