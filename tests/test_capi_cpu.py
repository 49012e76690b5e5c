"""CPU-side checks of the C-ABI library (no GPU needed, no kernel launches).

* libspct_b200.so loads and exports every symbol include/spct_cuda.h declares;
* host-only entry points (layout, workspace, analytics, contract checks) agree
  with the oracle and reject bad arguments with SPCT_ERR_CONTRACT before any
  device work — the reference's contract_error behaviour.
"""
import ctypes as C

import numpy as np
import pytest

import oracle
from paper_1711_01656_b200 import _capi as A


def test_library_exports_every_header_symbol():
    lib = A.lib()
    declared = A.header_symbols()
    assert len(declared) >= 18
    for name in declared:
        assert hasattr(lib, name), name
        assert name in A.SIGNATURES, f"{name} declared in the header but not bound"
    assert lib.spct_cu_version() == 1


def test_estimate_memory_and_schedule_stats_match_oracle():
    from paper_1711_01656_b200 import estimate_memory, schedule_stats

    for args in [(2048, 2048, 64, 1), (512, 512, 32, 8), (100, 100, 0, 8), (4096, 4096, 128, 4), (0, 3, 2, 8)]:
        assert estimate_memory(*args) == oracle.estimate_memory(*args)
    for args in [(1024, 1024, 32, 1024), (512, 512, 32, 512), (70, 33, 32, 64), (64, 64, 64, 2)]:
        it, tl, ef = schedule_stats(*args)
        s = oracle.schedule_stats(*args)
        assert (it, tl, ef) == (s.wavefront_iterations, s.tile_count, s.scan_efficiency)
    with pytest.raises(A.ContractError):
        schedule_stats(0, 4, 32, 64)
    with pytest.raises(A.ContractError):
        schedule_stats(4, 4, 32, 1)
    with pytest.raises(A.ContractError):
        estimate_memory(-1, 4, 4, 4)


def test_layout_is_aligned_and_tight():
    lib = A.lib()
    for w, h, b in [(1, 1, 1), (33, 31, 16), (4096, 4096, 128), (8192, 8192, 256), (1000, 7, 3)]:
        rp, pp, nb = C.c_int64(), C.c_int64(), C.c_uint64()
        A.check(lib.spct_cu_ih_layout(w, h, b, C.byref(rp), C.byref(pp), C.byref(nb)))
        assert rp.value % 32 == 0 and rp.value >= w and rp.value - w < 32
        assert pp.value == rp.value * h and nb.value == pp.value * b * 4
    # the headline tensor is exactly b*H*W*4 bytes: no padding traffic
    rp, pp, nb = C.c_int64(), C.c_int64(), C.c_uint64()
    A.check(lib.spct_cu_ih_layout(4096, 4096, 128, C.byref(rp), C.byref(pp), C.byref(nb)))
    assert nb.value == 128 * 4096 * 4096 * 4


def test_workspace_query():
    lib = A.lib()
    src = A.spct_source()
    src.kind, src.width, src.height, src.nbins, src.pitch, src.lo, src.hi = A.SRC_GRAY_U8, 4096, 4096, 128, 4096, 0.0, 256.0
    ws = C.c_size_t()
    A.check(lib.spct_cu_ih_build_workspace(C.byref(src), 0, 128, C.byref(ws)))
    assert 0 < ws.value < 4096 * 4096 * 128 * 4 // 20  # carry tables stay a few % of the tensor
    src.width = 0
    assert lib.spct_cu_ih_build_workspace(C.byref(src), 0, 128, C.byref(ws)) == A.SPCT_ERR_CONTRACT


def _hc(nbins, w, h, tmpl, kw, kh, p):
    th = np.ascontiguousarray(tmpl, np.float64)
    return A.lib().spct_cu_hist_check(nbins, w, h, th.ctypes.data_as(C.POINTER(C.c_double)), th.size, kw, kh, p)


def test_hist_check_mirrors_reference_predicates():
    good = np.full(8, 1 / 8)
    assert _hc(8, 30, 22, good, 7, 5, 2.0) == 0
    for bad in [(8, 30, 22, good, 7, 5, 0.5),          # p < 1
                (8, 30, 22, good, 31, 5, 1.0),         # kernel exceeds image
                (8, 30, 22, good, 0, 5, 1.0),
                (9, 30, 22, good, 7, 5, 1.0),          # bin count mismatch
                (8, 30, 22, good * 2, 7, 5, 1.0),      # not normalised
                (8, 30, 22, np.r_[good[:-1] + 1 / 56, -0.0 - 1e-9], 7, 5, 1.0)]:  # negative entry
        assert _hc(*bad) == A.SPCT_ERR_CONTRACT
        assert oracle.clib().or_hist_check(bad[0], bad[1], bad[2], np.ascontiguousarray(bad[3], np.float64),
                                           len(bad[3]), bad[4], bad[5], bad[6]) == 2
    # 1e-6 slack on the template mass (likelihood.cpp:206)
    assert _hc(8, 30, 22, good * (1 + 5e-7), 7, 5, 1.0) == 0


def test_contract_errors_before_device_work():
    lib = A.lib()
    src = A.spct_source()
    src.kind, src.width, src.height, src.nbins, src.pitch = A.SRC_GRAY_U8, 4, 1, 0, 4
    src.plane[0] = 1  # never dereferenced: the contract check fires first
    assert lib.spct_cu_quantize(C.byref(src), 1, None) == A.SPCT_ERR_CONTRACT
    assert b"bins must be in [1, 65536]" in lib.spct_cu_last_error()
    src.nbins, src.lo, src.hi = 8, 10.0, 10.0
    assert lib.spct_cu_quantize(C.byref(src), 1, None) == A.SPCT_ERR_CONTRACT
    assert b"hi must exceed lo" in lib.spct_cu_last_error()
    t = A.spct_ih(1, 4, 2, 5, 16, 16, 32, 32 * 16)  # slab [2, 6) outside nbins 5
    assert lib.spct_cu_region_counts(C.byref(t), 1, 1, 1, None) == A.SPCT_ERR_CONTRACT
    t = A.spct_ih(1, 4, 0, 4, 16, 16, 20, 20 * 16)  # row pitch not a multiple of 32
    assert lib.spct_cu_ih_export_u64(C.byref(t), 0, 1, 1, None) == A.SPCT_ERR_CONTRACT
    t = A.spct_ih(1, 4, 0, 4, 65536, 65536, 65536, 65536 * 65536)  # h*w = 2^32 does not fit uint32
    assert lib.spct_cu_hist_partial(C.byref(t), 1, 3, 3, 1.0, 0, 1, 0, None) == A.SPCT_ERR_CONTRACT


def test_orientation_contracts_before_device_work():
    lib = A.lib()
    ws = C.c_size_t()
    A.check(lib.spct_cu_orientation_workspace(2048, 2048, C.byref(ws)))
    assert ws.value >= 255 * 4  # the float bin-boundary table (the single-pass kernel needs no planes)
    # gradient_maps: sigma must be nonnegative (features.cpp:201) — checked before any launch
    assert lib.spct_cu_orientation_bins(1, 8, 8, 8, -1.0, 16, 1, 8, 1, 1 << 20, None) == A.SPCT_ERR_CONTRACT
    assert b"sigma must be nonnegative" in lib.spct_cu_last_error()
    assert lib.spct_cu_orientation_bins(1, 8, 8, 8, 1.0, 0, 1, 8, 1, 1 << 20, None) == A.SPCT_ERR_CONTRACT
    assert lib.spct_cu_orientation_bins(1, 8, 8, 8, 11.0, 16, 1, 8, 1, 1 << 20, None) == A.SPCT_ERR_CONTRACT
    assert lib.spct_cu_orientation_bins(1, 8, 8, 8, 1.0, 16, 1, 8, 1, 16, None) == A.SPCT_ERR_CONTRACT  # workspace
    assert lib.spct_cu_orientation_workspace(0, 3, C.byref(ws)) == A.SPCT_ERR_CONTRACT


def test_python_api_contracts_without_gpu():
    import paper_1711_01656_b200 as P

    assert P.schedule_from_string("wavefront") == 3 and P.schedule_from_string("seq") == 0
    with pytest.raises(P.ContractError):
        P.schedule_from_string("bogus")
    with pytest.raises(P.ContractError):
        P.api._validate_schedule(P.ScanSchedule(3, 32, 0))
    with pytest.raises(P.ContractError):
        P.api._validate_schedule(P.ScanSchedule(3, 1, 2))
    with pytest.raises(P.ContractError):
        P.api._check_budget(16, 16, 4, 64)  # test_integral.cpp:196-198
    P.api._check_budget(16, 16, 4, P.DEFAULT_BUDGET)


# ------------------------------------------------------------------ IHT1 (integral.cpp:619-659)

def _hdr(path):
    b, h, w, e = C.c_int(), C.c_int(), C.c_int(), C.c_int()
    st = A.lib().spct_cu_ih_load_header(str(path).encode(), C.byref(b), C.byref(h), C.byref(w), C.byref(e))
    return st, (b.value, h.value, w.value, e.value)


@pytest.mark.skipif(not oracle.have_ref(), reason="oracle/_ref not built")
def test_iht1_header_of_reference_dumps(tmp_path):
    bm = oracle.random_binmap(13, 7, 5, 31)
    path = tmp_path / "t.iht"
    oracle.RefTensor(bm, 5).dump(path)
    raw = path.read_bytes()
    assert raw[:4] == b"IHT1" and len(raw) == 20 + 5 * 8 * 14 * 8  # test_integral.cpp:214-228
    assert _hdr(path) == (0, (5, 7, 13, 8))


@pytest.mark.skipif(not oracle.have_ref(), reason="oracle/_ref not built")
def test_iht1_errors_match_reference(tmp_path):
    """load_tensor's io_error cases (integral.cpp:636-655), same status and message prefix."""
    good = tmp_path / "g.iht"
    oracle.RefTensor(oracle.random_binmap(6, 4, 3, 5), 3).dump(good)
    raw = good.read_bytes()
    cases = {"/nonexistent/t.iht": "cannot open tensor",  # test_integral.cpp:237
             "magic": "bad tensor magic", "short": "truncated tensor header", "elem": "unsupported element size",
             "dims": "bad tensor dimensions"}
    for name, msg in cases.items():
        p = name if name.startswith("/") else tmp_path / f"{name}.iht"
        if name == "magic":
            p.write_bytes(b"IHT2" + raw[4:])
        elif name == "short":
            p.write_bytes(raw[:13])
        elif name == "elem":
            p.write_bytes(raw[:16] + (5).to_bytes(4, "little") + raw[20:])
        elif name == "dims":
            p.write_bytes(raw[:4] + (0).to_bytes(4, "little") + raw[8:])
        st, _ = _hdr(p)
        assert st == A.SPCT_ERR_IO and A.lib().spct_cu_last_error().decode().startswith(msg), name
        with pytest.raises(oracle.RefIOError, match=msg):
            oracle.RefTensor.load(p)


def test_next_rows_and_peer_contracts_before_device_work():
    """SWIH / swlh map / median / consumers / peer-reduce entry points reject bad arguments
    with the reference's messages before touching the device."""
    lib = A.lib()
    err = lambda: lib.spct_cu_last_error()  # noqa: E731
    # swlh map, direct sweep: kernel_extents (swih.cpp:20), the sweep's own limits
    assert lib.spct_cu_swlh_map_direct(1, 16, 16, 16, 4, 0, 3, 1, 1, None) == A.SPCT_ERR_CONTRACT
    assert b"kernel extents must be >= 1" in err()
    assert lib.spct_cu_swlh_map_direct(1, 256, 256, 256, 4, 129, 3, 1, 1, None) == A.SPCT_ERR_CONTRACT
    assert lib.spct_cu_swlh_map_direct(1, 8, 16, 16, 4, 3, 3, 1, 1, None) == A.SPCT_ERR_CONTRACT  # pitch < width
    # swlh brute force / weighted layout
    assert lib.spct_cu_swlh_brute(1, 16, 16, 16, 4, 0, 3, None, 0, None, None) == A.SPCT_ERR_CONTRACT
    rp, pp, nb = C.c_int64(), C.c_int64(), C.c_uint64()
    assert lib.spct_cu_wih_layout(0, 4, 4, C.byref(rp), C.byref(pp), C.byref(nb)) == A.SPCT_ERR_CONTRACT
    A.check(lib.spct_cu_wih_layout(33, 7, 3, C.byref(rp), C.byref(pp), C.byref(nb)))
    assert rp.value % 16 == 0 and rp.value >= 33 and pp.value == rp.value * 7 and nb.value == pp.value * 3 * 8
    # joint-IH median (motion.cpp:13-14, 38-43)
    assert lib.spct_cu_median_sort(None, 0, 4, 4, 4, 1, 4, None) == A.SPCT_ERR_CONTRACT
    assert b"empty window" in err()
    ptrs = (C.c_void_p * 2)(1, 1)
    assert lib.spct_cu_median_sort(ptrs, 2, 4, 4, 4, 1, 4, None) == A.SPCT_ERR_CONTRACT
    assert b"window length must be odd" in err()
    # map consumers (likelihood.cpp:258-266, tracker.cpp:79-84)
    assert lib.spct_cu_fuse_maps(None, 0, None, 0, 16, 1, None) == A.SPCT_ERR_CONTRACT
    assert b"no maps to fuse" in err()
    r = C.c_int64()
    assert lib.spct_cu_score_map(1, 10, 10, 8, 8, 5, 5, C.byref(r), 1, 1 << 20, None) == A.SPCT_ERR_CONTRACT
    assert b"ground truth rect must lie inside the map" in err()
    # peer reduce: flags and the slot finaliser
    assert lib.spct_cu_flag_wait(None, 1, 1, 1, 1000, None, None) == A.SPCT_ERR_CONTRACT
    assert lib.spct_cu_flag_wait(1, 0, 1, 1, 1000, 1, None) == A.SPCT_ERR_CONTRACT
    assert lib.spct_cu_flag_signal(None, 1, None) == A.SPCT_ERR_CONTRACT
    assert lib.spct_cu_hist_finalize_slots(1, 2, 10, 8, 8, 3, 3, 1.0, 0, 1, None) == A.SPCT_ERR_CONTRACT  # stride < nu*nv
    assert lib.spct_cu_hist_finalize_slots(1, 2, 36, 8, 8, 3, 3, 0.5, 0, 1, None) == A.SPCT_ERR_CONTRACT
    assert b"Minkowski order must be >= 1" in err()
    assert lib.spct_cu_peer_open(None, None) == A.SPCT_ERR_CONTRACT


def test_carry_tables_reject_dims_beyond_u16():
    """Row / column counts of the sweeps' carry tables are 16-bit (carries.cu): a build or
    fused sweep over a 70000 x 500 image is refused with a contract error before any
    launch, instead of silently wrapping."""
    lib = A.lib()
    fake = 0x1000  # never dereferenced: the checks run before any device work
    for w, h in [(70000, 500), (500, 70000)]:
        src = A.spct_source()
        src.kind, src.width, src.height, src.nbins, src.pitch, src.lo, src.hi = A.SRC_GRAY_U8, w, h, 8, w, 0.0, 256.0
        src.plane[0] = fake
        rp, pp, nb = C.c_int64(), C.c_int64(), C.c_uint64()
        A.check(lib.spct_cu_ih_layout(w, h, 8, C.byref(rp), C.byref(pp), C.byref(nb)))
        t = A.spct_ih(fake * 16, 8, 0, 8, h, w, rp.value, pp.value)
        assert lib.spct_cu_ih_build(C.byref(src), C.byref(t), None, 0, None) == A.SPCT_ERR_CONTRACT
        assert b"65536" in lib.spct_cu_last_error()
        tm = (C.c_double * 8)()
        assert lib.spct_cu_ih_build_match_map(C.byref(src), C.byref(t), tm, 4, 4, 1.0, 0, fake * 16, None, 0,
                                              None) == A.SPCT_ERR_CONTRACT
        assert b"65536" in lib.spct_cu_last_error()


def test_fused_window_predicate():
    lib = A.lib()
    assert lib.spct_cu_fused_window_ok(64, 64) == 1
    assert lib.spct_cu_fused_window_ok(128, 255) == 1
    assert lib.spct_cu_fused_window_ok(129, 10) == 0
    assert lib.spct_cu_fused_window_ok(10, 256) == 0
    assert lib.spct_cu_fused_window_ok(0, 10) == 0
