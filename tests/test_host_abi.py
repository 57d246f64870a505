"""Host-side logic and the C-ABI surface, runnable without a GPU."""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_2310_10939_b200 import (DeviceError, InputError, SpectralParams, fast_spectral_cluster,
                                   from_csr, from_edges)
from paper_2310_10939_b200 import _lib
from paper_2310_10939_b200.kmeans import Partition, _nth_unchosen
from paper_2310_10939_b200.pipeline import MODES, _kmeans_seed

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "sc_b200.h")).read()
    return sorted(set(re.findall(r"\b(sc_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    L = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.EXPORTS)
    assert L.sc_version() == 2


def test_library_is_sm100a():
    data = open(_lib.LIB_PATH, "rb").read()
    assert b"sm_100a" in data or b"compute_100a" in data


def test_abi_rejects_bad_input_without_gpu():
    L = _lib.load()
    rp = np.array([0, 1, 3], dtype=np.int64)  # row_ptr[n] != nnz
    col = np.array([1, 0], dtype=np.int32)
    deg = np.ones(2)
    h = ctypes.c_void_p()
    st = L.sc_graph_create(_lib.ptr(rp), _lib.ptr(col), None, _lib.ptr(deg), 2, 2, 0,
                           ctypes.byref(h))
    assert st == -2
    assert b"row_ptr" in L.sc_last_error()
    with pytest.raises(InputError):
        _lib.check(st)
    st = L.sc_graph_create(None, None, None, None, 2, 2, 0, ctypes.byref(h))
    assert st == -1
    bad_deg = np.array([1.0, 0.0])
    rp = np.array([0, 1, 2], dtype=np.int64)
    st = L.sc_graph_create(_lib.ptr(rp), _lib.ptr(col), None, _lib.ptr(bad_deg), 2, 2, 0,
                           ctypes.byref(h))
    assert st == -2
    col_bad = np.array([1, 5], dtype=np.int32)
    st = L.sc_graph_create(_lib.ptr(rp), _lib.ptr(col_bad), None, _lib.ptr(deg), 2, 2, 0,
                           ctypes.byref(h))
    assert st == -2 and b"out of range" in L.sc_last_error()
    # layout builders on a null handle
    assert L.sc_graph_build_windows(None) == -1 and L.sc_graph_build_panels(None) == -1
    assert _lib.SC_CREATE_WINDOWS == 0x10 and ctypes.sizeof(_lib.GraphInfo) == 112  # sizeof(sc_graph_info)


@pytest.mark.skipif(_lib.load().sc_device_count() > 0, reason="GPU present")
def test_no_cpu_fallback():
    """Without a CUDA device the product path fails loudly instead of computing on CPU."""
    g, _ = from_edges(4, [0, 1, 2], [1, 2, 3])
    with pytest.raises(DeviceError):
        fast_spectral_cluster(g, SpectralParams(k=2, t=3, mode="one_vector"))


def test_params_semantics():
    p = SpectralParams(k=10, mode="one_vector")
    assert p.num_columns(10**6) == 1
    assert p.num_steps(10**6) == int(np.ceil(10 * np.log(10**5)))
    assert SpectralParams(k=5, t=50, mode="one_vector").num_steps(1000) == 50
    assert "one_vector" in MODES
    assert SpectralParams(k=5).layout == "auto"
    assert SpectralParams(k=5, layout="windows").layout == "windows"
    for bad in (dict(k=1), dict(k=3, mode="nope"), dict(k=3, t=-1), dict(k=3, seed=-2),
                dict(k=3, epsilon=0.0), dict(k=3, walk_sign=2), dict(k=3, layout="ell")):
        with pytest.raises(InputError):
            SpectralParams(**bad)
    assert _kmeans_seed(0) == 3141116543


def test_unsupported_algorithm2_modes_are_refused():
    """pm_k and the eigensolver modes are outside the device path (pm_log_k is on it);
    the block width of pm_log_k is bounded by the device kernel."""
    g, _ = from_edges(4, [0, 1, 2], [1, 2, 3])
    for mode in ("pm_k", "eigs_k", "eigs_log_k"):
        with pytest.raises(InputError):
            fast_spectral_cluster(g, SpectralParams(k=2, mode=mode))
    g, _ = from_edges(40, list(range(39)), list(range(1, 40)))
    with pytest.raises(InputError):
        fast_spectral_cluster(g, SpectralParams(k=2, l=17, mode="pm_log_k"))


def test_k_exceeds_n():
    g, _ = from_edges(3, [0, 1], [1, 2])
    with pytest.raises(InputError):
        fast_spectral_cluster(g, SpectralParams(k=5, mode="one_vector"))


def test_nth_unchosen_matches_setdiff():
    rng = np.random.default_rng(0)
    for _ in range(200):
        n = int(rng.integers(1, 60))
        i = int(rng.integers(0, n))
        taken = np.unique(rng.integers(0, n, i)) if i else np.empty(0, dtype=np.int64)
        rest = np.setdiff1d(np.arange(n), taken)
        if rest.size == 0:
            continue
        m = int(rng.integers(0, rest.size))
        assert _nth_unchosen(taken, m) == rest[m]


def test_partition_validation():
    with pytest.raises(InputError):
        Partition(labels=np.array([0, 3]), k=2)
    assert Partition.from_labels([0, 2, 2]).k == 3


def test_from_edges_semantics():
    g, dropped = from_edges(5, [0, 1, 1], [1, 2, 2], [1.0, 2.0, 0.5], drop_isolated=True)
    assert dropped == [3, 4]
    assert g.n == 3
    assert g.row_offsets.tolist() == [0, 1, 3, 4]
    assert g.col_indices.tolist() == [1, 0, 2, 1]
    assert g.weights.tolist() == [1.0, 1.0, 2.5, 2.5]
    assert g.degrees.tolist() == [1.0, 3.5, 2.5]
    with pytest.raises(InputError):
        from_edges(3, [0, 1], [1, 1])  # self loop
    with pytest.raises(InputError):
        from_edges(4, [0], [1])  # isolated vertices
    g2 = from_csr(3, [0, 1, 3, 4], [1, 0, 2, 1])
    assert g2.unit_weights() and g2.degrees.tolist() == [1.0, 2.0, 1.0]


def test_multi_gpu_handle_rejects_bad_input_without_gpu():
    """sc_graph_create_multi validates its arguments before touching a device."""
    L = _lib.load()
    rp = np.array([0, 1, 2, 3, 4], dtype=np.int64)
    col = np.array([1, 0, 3, 2], dtype=np.int32)
    deg = np.ones(4)
    h = ctypes.c_void_p()
    args = (_lib.ptr(rp), _lib.ptr(col), None, _lib.ptr(deg), 4, 4)
    assert L.sc_graph_create_multi(*args, 0, None, 0, ctypes.byref(h)) == -1   # n_gpus < 1
    assert L.sc_graph_create_multi(*args, 5, None, 0, ctypes.byref(h)) == -1   # n < n_gpus
    assert L.sc_graph_create_multi(*args, 2, None, _lib.SC_CREATE_REORDER_BFS,
                                   ctypes.byref(h)) == -1                       # BFS: 1 GPU only
    rp_bad = np.array([0, 1, 2, 3, 5], dtype=np.int64)
    assert L.sc_graph_create_multi(_lib.ptr(rp_bad), _lib.ptr(col), None, _lib.ptr(deg), 4, 4,
                                   2, None, 0, ctypes.byref(h)) == -2
    assert L.sc_kmeans_set_flags(None, 0) == -1
    with pytest.raises(InputError):
        SpectralParams(k=3, gpus=0)
    assert SpectralParams(k=3).cost_assert is None and SpectralParams(k=3).gpus == 1


def test_bench_helpers():
    """bench.py: bounded CPU samples above config 2, ncu traffic keyed by layout + pre-order"""
    import importlib.util
    import os

    spec = importlib.util.spec_from_file_location(
        "bench", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)

    class G:
        nnz = 1_800_041_874

    assert bench.cpu_sample_steps(G, 100, 5) == (66, False)
    assert bench.cpu_sample_steps(G, 100, 2) == (100, True)
    assert bench.traffic_from_profiles(4, False, "sell", "bfs") is not None
    assert bench.traffic_from_profiles(5, True, "sell", "none") is not None
    assert bench.traffic_from_profiles(2, True, "panels", "none") is not None
    assert bench.traffic_from_profiles(4, False, "windows", "bfs") is not None


def test_bench_stdout_is_one_json_line(tmp_path):
    """library chatter on file descriptor 1 (NCCL's version banner) must not reach the bench's
    stdout: inside bench._QuietStdout fd 1 points at stderr and print() keeps the real stdout"""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import importlib.util, os\n"
        f"spec = importlib.util.spec_from_file_location('bench', {os.path.join(root, 'bench.py')!r})\n"
        "b = importlib.util.module_from_spec(spec); spec.loader.exec_module(b)\n"
        "with b._QuietStdout():\n"
        "    os.write(1, b'NCCL version x\\n')\n"
        "    print('{\"json\": 1}', flush=True)\n")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=root)
    assert r.returncode == 0, r.stderr
    assert r.stdout == '{"json": 1}\n'
    assert "NCCL version x" in r.stderr
