"""The C-ABI library loads and exports every symbol include/hs.h declares; the
host-side argument validation works without a GPU (no compute calls here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "hs.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hs_[a-z0-9_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported(libhs):
    from paper_2505_12566_b200 import _abi
    lib = ctypes.CDLL(_abi.LIB_PATH)
    names = _declared()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_abi.SIGNATURES), "binding and header disagree"


def test_header_compiles_as_c(tmp_path):
    c = tmp_path / "t.c"
    c.write_text('#include "hs.h"\nint main(void){ return (int)sizeof(hs_status_t) - 4; }\n')
    import subprocess
    subprocess.check_call(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                           "-o", str(tmp_path / "t"), str(c)])
    assert subprocess.call([str(tmp_path / "t")]) == 0


def test_workspace_queries_are_pure(libhs):
    lib = libhs.lib()
    assert lib.hs_route_compact_workspace(0) > 0
    # one 8-byte look-back descriptor per 2,048-item tile
    assert lib.hs_route_compact_workspace(2048) == lib.hs_route_compact_workspace(1)
    assert lib.hs_route_compact_workspace(2049) == lib.hs_route_compact_workspace(2048) + 8
    assert lib.hs_confidence_workspace(3000, 1) == 0         # no token rows, no split region
    assert lib.hs_confidence_workspace(100, 1) > 0           # optional split-row region (<= 2,048 rows)
    assert lib.hs_confidence_workspace(100, 64) >= 100 * 64 * 5
    assert lib.hs_calibrate_workspace(5, 12) >= 3 * (4096 + 2) * 4
    assert lib.hs_calibrate_workspace(5, 15) == 0
    assert lib.hs_cascade_step_workspace(1000, 1) >= 1000 * (4 + 4 + 8)


@pytest.mark.parametrize("kw,needle", [
    (dict(C=1), "n_classes"),
    (dict(T=0.0), "temperature"),
    (dict(T=float("inf")), "temperature"),
    (dict(L=0), "seq_len"),
    (dict(L=2, reduce=0), "SEQ_NONE"),
    (dict(stride=999), "row_stride"),
    (dict(stride=1001), "16 bytes"),
    (dict(ptr=8), "aligned"),
])
def test_confidence_argument_errors(libhs, kw, needle):
    lib = libhs.lib()
    C = kw.get("C", 1000)
    rc = lib.hs_confidence(kw.get("ptr", 256), 1, 10, kw.get("L", 1), C, kw.get("stride", 1000), None,
                           None, kw.get("T", 1.0), 0, kw.get("reduce", 0), 512, None, None, None,
                           None, 0, None, None)
    assert rc == 1
    assert needle in lib.hs_last_error().decode()


def test_route_and_calibrate_argument_errors(libhs):
    lib = libhs.lib()
    nan = float("nan")
    for t in (nan, -0.1, 1.5):
        rc = lib.hs_route_compact(256, 10, None, t, None, 0, None, None, 1, None, None, None, None,
                                  None, None, 0, None, 512, 1024, 4096, None)
        assert rc == 1 and "threshold" in lib.hs_last_error().decode()
    rc = lib.hs_route_compact(256, 10, None, 0.5, None, 0, None, None, 1, None, None, None, None,
                              None, None, 0, None, 512, 1024, 8, None)
    assert rc == 5   # workspace too small
    rc = lib.hs_calibrate_thresholds(256, 512, 1, 10, 12, -1, 0, 1, 2, 3, 4, 5, 1024, 1 << 20, None)
    assert rc == 1 and "K" in lib.hs_last_error().decode()
    rc = lib.hs_calibrate_thresholds(256, 512, 3, 10, 15, -1, 0, 1, 2, 3, 4, 5, 1024, 1 << 20, None)
    assert rc == 1 and "log2_bins" in lib.hs_last_error().decode()
    rc = lib.hs_calibrate_thresholds(256, 512, 3, 0, 12, -1, 0, 1, 2, 3, 4, 5, 1024, 1 << 20, None)
    assert rc == 1 and "empty" in lib.hs_last_error().decode()
    rc = lib.hs_calibrate_thresholds(256, 512, 3, 10, 12, -1, 65, 1, 2, 3, 4, 5, 1024, 1 << 20, None)
    assert rc == 1 and "refine_passes" in lib.hs_last_error().decode()
    rc = lib.hs_cascade_step(3, 3, 256, 1, 10, 1, 1000, 1000, None, None, 1.0, 0, 0, 0.5, None,
                             None, None, 0, None, None, None, None, None, 512, 1024, 1 << 20,
                             None, None)
    assert rc == 1 and "stage" in lib.hs_last_error().decode()


def test_status_strings(libhs):
    lib = libhs.lib()
    assert lib.hs_status_string(0) == b"HS_OK"
    assert lib.hs_status_string(5) == b"HS_ERR_WORKSPACE_TOO_SMALL"
    assert lib.hs_status_string(4) == b"HS_ERR_NCCL"
    assert b"sm_100a" in lib.hs_build_info()


def test_product_never_imports_oracle():
    """The product package must not import, link or load the oracle (no CPU path)."""
    pkg = os.path.join(ROOT, "paper_2505_12566_b200")
    bad = re.compile(r"(import\s+oracle|from\s+oracle|hs_oracle|libhs_oracle|hso_)")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                assert not bad.search(open(os.path.join(dirpath, f)).read()), f


def test_skip_edges_host_helper_matches_oracle(libhs):
    """hs_skip_edges is host arithmetic (no device work): same fp32 edges as the
    oracle's P:541 / S:320 bands, for the fp32 threshold the router compares."""
    import numpy as np
    import oracle
    import paper_2505_12566_b200 as hs
    for t in (0.0, 0.25, 0.7, 0.999, 1.0):
        t32 = float(np.float32(t))
        for s_ in range(1, 8):
            for mode in (hs.SKIP_UNIFORM, hs.SKIP_DECADE):
                assert np.array_equal(np.array(hs.skip_edges(t32, s_, mode), np.float32),
                                      oracle.skip_edges(t32, s_, mode)), (t, s_, mode)


def test_fit_temperature_argument_errors(libhs):
    """hs_fit_temperature (NEXT-3) validates on the host before any launch."""
    lib = libhs.lib()
    ptrs = (ctypes.c_void_p * 1)(256)
    ws = lib.hs_fit_temperature_workspace(1, 10)
    assert ws >= 10 * 8
    assert lib.hs_fit_temperature_workspace(5, 10) > ws

    def call(nb=1, C=1000, lo=0.5, hi=2.0, passes=16, T=512, labels=768, wsb=ws):
        return lib.hs_fit_temperature(ptrs, nb, 1, 10, C, 1000, labels, lo, hi, passes, T, None,
                                      None, None, 1024, wsb, None, None)
    for kw, needle in ((dict(nb=0), "n_batches"), (dict(nb=9), "n_batches"), (dict(C=1), "n_classes"),
                       (dict(lo=0.0), "range"), (dict(lo=3.0), "range"), (dict(hi=float("inf")), "range"),
                       (dict(passes=0), "max_passes"), (dict(passes=257), "max_passes"),
                       (dict(T=None), "d_T"), (dict(labels=None), "labels")):
        assert call(**kw) == 1, kw
        assert needle in lib.hs_last_error().decode(), kw
    assert call(wsb=ws - 1) == 5


def test_grid_helpers_match_oracle(libhs):
    """hs_grid_size / hs_grid_vector are host arithmetic (no device work)."""
    import oracle
    import paper_2505_12566_b200 as hs
    for K, q in ((2, 1), (3, 2), (5, 4), (8, 1)):
        S = hs.grid_size(K, q)
        assert S == oracle.grid_size(K, q)
        for s in (0, 1, S // 3, S - 1):
            assert hs.grid_vector(s, K, q) == oracle.grid_vector(s, K, q)
    assert hs.grid_size(5, 14) == -1 and hs.grid_size(9, 1) == -1 and hs.grid_size(1, 4) == -1


def test_replay_and_graph_argument_errors(libhs):
    lib = libhs.lib()
    w = (ctypes.c_int64 * 3)(1, 2, 3)
    ws = lib.hs_threshold_replay_workspace(3, 100, 4)
    def rp(K=3, N=100, q=4, bv=None, S=None, wt=w, wsb=ws):
        S = lib.hs_grid_size(K, q) if S is None else S
        return lib.hs_threshold_replay(256, 512, K, N, q, bv, S, wt, 1024, 2048, None, None, 4096, wsb, None)
    assert rp(K=1) == 1 and "K" in lib.hs_last_error().decode()
    assert rp(K=9) == 1
    assert rp(q=0) == 1 and "log2_bins" in lib.hs_last_error().decode()
    assert rp(N=0) == 1 and "empty" in lib.hs_last_error().decode()
    assert rp(S=7) == 1 and "hs_grid_size" in lib.hs_last_error().decode()
    neg = (ctypes.c_int64 * 3)(1, -2, 3)
    assert rp(wt=neg) == 1 and "weights" in lib.hs_last_error().decode()
    big = (ctypes.c_int64 * 3)(1, 1 << 62, 3)
    assert rp(wt=big) == 1 and "overflow" in lib.hs_last_error().decode()
    assert rp(wsb=ws - 1) == 5
    gws = lib.hs_perf_graph_workspace(100)
    assert gws >= 101 * 16
    rc = lib.hs_perf_graph(256, 512, 10, 100, -1, 5, None, 3, 1, 2, 3, 4, 5, 4096, gws, None, None)
    assert rc == 1 and "d_model_correct" in lib.hs_last_error().decode()
    rc = lib.hs_perf_graph(256, 512, 10, 100, 5, 5, None, 3, 1, 2, 3, 4, 5, 4096, gws - 1, None, None)
    assert rc == 5


def _build_c_client(tmp_path):
    import shutil
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    pkg = os.path.join(root, "paper_2505_12566_b200")
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    exe = str(tmp_path / "hs_c_client")
    r = subprocess.run([cc, "-std=c11", "-Wall", "-Werror", "-I", os.path.join(root, "include"),
                        "-I", "/usr/local/cuda/include", os.path.join(root, "examples", "c_client.c"),
                        "-L", pkg, "-lhs", f"-Wl,-rpath,{pkg}", "-L", "/usr/local/cuda/lib64", "-lcudart",
                        "-lm", "-o", exe], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_program_links_libhs(libhs, tmp_path):
    """A plain C program built against include/hs.h and linked with -lhs (no
    Python): host-only calls and the synchronous argument checks."""
    import subprocess
    r = subprocess.run([_build_c_client(tmp_path)], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0 and "c client ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.gpu
def test_c_program_routes_a_cascade_on_the_gpu(libhs, tmp_path):
    """The same C program with --gpu: one 6-request, 3-stage cascade through
    hs_cascade_step with cudaMalloc'd buffers, checked against the hand-worked
    stages."""
    import subprocess
    r = subprocess.run([_build_c_client(tmp_path), "--gpu"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "c client ok" in r.stdout, r.stdout + r.stderr


def test_step_flags_validated_before_any_launch(libhs):
    """hs_cascade_step_ex / hs_cascade_confidence reject unknown flag bits
    synchronously (HS_STEP_OVERLAP_PREVIOUS = 1 and HS_STEP_LOGITS_CAPACITY = 2
    are the only ones), before touching the device."""
    lib = libhs.lib()
    rc = lib.hs_cascade_step_ex(0, 3, 256, 1, 10, 1, 1000, 1000, None, None, 1.0, 0, 0, 0.5, None,
                                None, None, 0, None, None, None, None, None, 512, 1024, 1 << 20,
                                None, 0, 4, None)
    assert rc == 1 and "flags" in lib.hs_last_error().decode()
    rc = lib.hs_cascade_confidence(0, 3, 256, 1, 10, 1, 1000, 1000, None, None, 1.0, 0, 0, 0.5, None,
                                   None, 1024, 1 << 20, None, 0, 8, None)
    assert rc == 1 and "flags" in lib.hs_last_error().decode()


def test_logits_capacity_flag_from_storage(libhs):
    """The binding sets HS_STEP_LOGITS_CAPACITY exactly when the memory from the
    logits' first row on covers the capacity (a view of the live rows of a
    capacity-sized buffer), never for gathered rows."""
    import torch
    buf = torch.zeros(1000, 64, dtype=torch.bfloat16)
    cap = libhs.HS_STEP_LOGITS_CAPACITY
    assert libhs._rows_capacity_flag(buf, 1000, None) == cap
    assert libhs._rows_capacity_flag(buf[:10], 1000, None) == cap       # view: storage covers 1,000 rows
    assert libhs._rows_capacity_flag(buf[10:20], 1000, None) == 0       # starts 10 rows in
    assert libhs._rows_capacity_flag(buf[:10].clone(), 1000, None) == 0  # exact-sized copy
    assert libhs._rows_capacity_flag(buf[:10].clone(), 10, None) == cap
    assert libhs._rows_capacity_flag(buf, 1000, torch.zeros(5, dtype=torch.int64)) == 0
    padded = torch.zeros(100, 80, dtype=torch.float32)[:, :64]          # stride 80 > C
    assert libhs._rows_capacity_flag(padded, 100, None) == cap
    assert libhs._rows_capacity_flag(padded, 101, None) == 0
