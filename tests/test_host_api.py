"""CPU-side checks: drop-in data model, C-ABI library surface, no CPU fallback."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_2005_09824_b200 as P
from paper_2005_09824_b200 import _backend, _build, synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


def _reference():
    if not os.path.isdir(os.path.join(REF, "chainloss")):
        pytest.skip("reference not installed in baseline/_ref")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_lfmmi")
    import sys

    if REF not in sys.path:
        sys.path.insert(0, REF)
    import chainloss

    return chainloss


# ----------------------------------------------------------- C-ABI surface
def _header_symbols():
    with open(os.path.join(ROOT, "include", "lfmmi.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(lfmmi_[a-z0-9_]+)\s*\(", text)))


def test_core_library_exports_every_header_symbol():
    lib = ctypes.CDLL(_build.CORE_SO)
    syms = _header_symbols()
    assert len(syms) >= 10
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_core_library_host_calls_without_gpu():
    lib = ctypes.CDLL(_build.CORE_SO)
    lib.lfmmi_version.restype = ctypes.c_char_p
    lib.lfmmi_last_error.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.lfmmi_version()
    lib.lfmmi_workspace_size.restype = ctypes.c_size_t
    lib.lfmmi_workspace_size.argtypes = [ctypes.c_int32, ctypes.c_int64, ctypes.c_int32]
    assert lib.lfmmi_workspace_size(1000, 28778, 0) >= 1000 * 28778 * 4
    # Argument validation happens before any CUDA call.
    out = ctypes.c_void_p()
    rc = lib.lfmmi_graphs_create(0, 1, 1, 1, None, None, None, None, None, None, None, None,
                                 None, None, None, None, ctypes.byref(out))
    assert rc == 1 and b"bad sizes" in lib.lfmmi_last_error()


def test_torch_extension_loads():
    ext = _backend.ext()
    assert "sm_100a" in ext.version()
    assert ext.workspace_size(1000, 10, 1) >= 1000 * 10 * 8


def test_no_cpu_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    batch = P.make_batch([np.zeros((2, 1))])
    g = P.ChainGraphBatch.broadcast(P.ChainGraph([(0, 0, 0, 1.0)], 1, 1, 0, [1.0]), 1)
    with pytest.raises(_backend.BackendUnavailable):
        P.chain_loss(batch, g, g)
    with pytest.raises(_backend.BackendUnavailable):
        P.forward_backward(batch, g)


# ------------------------------------------------------------ data model
def test_graph_layouts_match_reference():
    C = _reference()
    w = synth.make_workload("toy", seed=4)
    for lib_out, ref_out in zip(w.build(P)[1:], w.build(C)[1:]):
        for name in ("forward_from", "forward_to", "forward_pdf", "forward_probs", "forward_index",
                     "backward_from", "backward_to", "backward_pdf", "backward_probs",
                     "backward_index", "final_probs", "initial_states", "row_map",
                     "item_num_states", "item_num_transitions"):
            np.testing.assert_array_equal(getattr(lib_out, name), getattr(ref_out, name))
    b1, b2 = P.make_batch(w.seqs), C.make_batch(w.seqs)
    for name in ("values", "lengths", "valid_batch_sizes", "order_map"):
        np.testing.assert_array_equal(getattr(b1, name), getattr(b2, name))


@pytest.mark.parametrize("args,match", [
    (([(0, 1, 1, 1.0)], 2, 1, 0, [0, 1]), "pdf_id 1 out of range"),
    (([(0, 5, 0, 1.0)], 2, 1, 0, [0, 1]), "to_state 5"),
    (([(0, 1, 0, 1.0)], 2, 1, 3, [0, 1]), "initial_state"),
    (([(0, 1, 0, -1.0)], 2, 1, 0, [0, 1]), "invalid probability"),
    (([(0, 1, 0, float("nan"))], 2, 1, 0, [0, 1]), "invalid probability"),
    (([(0, 1, 0, 1.0)], 2, 1, 0, [0, 1.5]), "final_probs"),
    (([(0, 1, 0, 1.0)], 2, 1, 0, [0, 0]), "accepts nothing"),
    (([(0, 1, 0, 1.0)], 2, 1, 0, [1.0]), "shape"),
    (([(0, 1, 0, 1.0)], 3, 1, 0, [0, 1, 1]), "state 2 is not reachable"),
    (([(0, 1, 0, 1.0), (0, 2, 0, 1.0)], 3, 1, 0, [0, 1, 0]), "state 2 cannot reach"),
])
def test_graph_validation_errors(args, match):
    with pytest.raises(ValueError, match=match):
        P.ChainGraph(*args)


def test_graph_zero_prob_dropped_and_immutable():
    g = P.ChainGraph([(0, 0, 0, 1.0), (0, 0, 0, 0.0)], 1, 1, 0, [1.0])
    assert g.num_transitions == 1 and g.dropped_transitions == 1
    with pytest.raises(ValueError):
        g.forward_probs[0] = 2.0
    assert next(g.transitions()) == P.Transition(0, 0, 0, 1.0)


def test_batch_errors_and_broadcast():
    g = P.ChainGraph([(0, 0, 0, 1.0)], 1, 1, 0, [1.0])
    with pytest.raises(ValueError, match="empty"):
        P.ChainGraphBatch.from_graphs([])
    with pytest.raises(ValueError, match="batch_size"):
        P.ChainGraphBatch.broadcast(g, 0)
    h = P.ChainGraph([(0, 0, 1, 1.0)], 1, 2, 0, [1.0])
    with pytest.raises(ValueError, match="num_pdfs"):
        P.ChainGraphBatch.from_graphs([g, h])
    bb = P.ChainGraphBatch.broadcast(g, 5)
    assert bb.forward_from.shape[0] == 1 and np.all(bb.row_map == 0) and len(bb) == 5
    with pytest.raises(TypeError):
        P.ChainGraphBatch()


def test_make_batch_paper_example_and_unsort():
    # PAPER.md §3.4: lengths (100, 99, 98) -> B_v = [3, ..., 3, 2, 1]
    rng = np.random.default_rng(0)
    seqs = [rng.normal(size=(t, 2)) for t in (98, 100, 99)]
    b = P.make_batch(seqs)
    assert list(b.lengths) == [100, 99, 98]
    assert list(b.order_map) == [1, 2, 0]
    assert b.valid_batch_sizes[0] == 3 and list(b.valid_batch_sizes[-3:]) == [3, 2, 1]
    assert b.total_frames == 297
    back = P.unsort(b.values, b.order_map)
    np.testing.assert_array_equal(back[0, :98], seqs[0])
    for bad, match in (([], "empty"), ([np.zeros((2, 1)), np.zeros((2, 2))], "pdf dimension"),
                       ([np.zeros((0, 1))], "zero-length"), ([np.full((1, 1), np.inf)], "finite"),
                       ([np.zeros(3)], r"\(T, D\)")):
        with pytest.raises(ValueError, match=match):
            P.make_batch(bad)
    with pytest.raises(ValueError, match="batch axis"):
        P.unsort(np.zeros((2, 1)), np.arange(3))


def test_options_validation():
    with pytest.raises(ValueError, match="leak_coefficient"):
        P.FBOptions(leak_coefficient=-1.0)
    with pytest.raises(ValueError, match="scale_floor"):
        P.FBOptions(scale_floor=0.0)


def test_synthetic_recipe_deterministic():
    a = synth.make_workload("wsj_mono", seed=0)
    b = synth.make_workload("wsj_mono", seed=0)
    assert np.array_equal(a.lengths, b.lengths) and a.total_frames == b.total_frames
    assert all(np.array_equal(x, y) for x, y in zip(a.seqs, b.seqs))
    assert a.total_frames == 28778  # SURVEY.md §6 calibration draw
    for x in a.seqs[:4]:
        assert np.array_equal(x, x.astype(np.float32).astype(np.float64))


# ------------------------------------------------- options + linear records
def test_options_struct_roundtrip():
    """One options struct (lfmmi_set_option / lfmmi_get_option / reset), no env reads."""
    lib = ctypes.CDLL(_build.CORE_SO)
    lib.lfmmi_last_error.restype = ctypes.c_char_p
    buf = ctypes.create_string_buffer(64)
    try:
        assert lib.lfmmi_set_option(b"split_clusters", b"42") == 0
        assert lib.lfmmi_get_option(b"split_clusters", buf, 64) == 0 and buf.value == b"42"
        assert lib.lfmmi_set_option(b"stream_mode", b"1024x1") == 0
        assert lib.lfmmi_get_option(b"stream_mode", buf, 64) == 0 and buf.value == b"1024x1"
        assert lib.lfmmi_set_option(b"no_such_option", b"1") == 1
        assert b"unknown option" in lib.lfmmi_last_error()
        assert lib.lfmmi_set_option(b"split", b"x") == 1  # integers only
    finally:
        lib.lfmmi_reset_options()
    assert lib.lfmmi_get_option(b"split_clusters", buf, 64) == 0 and buf.value == b"0"
    with _backend.options(split=0, linear_split=0):
        assert _backend.ext().get_option("split") == "0"
    assert _backend.ext().get_option("split") == "-1"


def test_create_linear_validates_before_device_use():
    lib = ctypes.CDLL(_build.CORE_SO)
    lib.lfmmi_last_error.restype = ctypes.c_char_p
    out = ctypes.c_void_p()
    assert lib.lfmmi_graphs_create_linear(4, 600, 84, None, None, ctypes.byref(out)) == 1
    assert b"max_states" in lib.lfmmi_last_error()
    assert lib.lfmmi_graphs_create_linear(4, 100, 84, None, None, ctypes.byref(out)) == 1
    assert b"NULL" in lib.lfmmi_last_error()


def test_linear_records_of_reference_numerators():
    """Per-utterance records (graph.linear_records) of the reference's own
    build_numerator graphs: one record per state with the self-loop and entry
    arcs of toy_builder.py:218-265; other graph shapes return None."""
    from paper_2005_09824_b200.graph import linear_records

    rng = np.random.default_rng(0)
    phones = rng.integers(0, 42, 30).tolist()
    arcs, S, fin = synth.numerator_arcs(phones, 42)
    g = P.ChainGraph(arcs, S, 84, 0, fin)
    rec = linear_records(g)
    assert rec.shape == (S, 4) and rec.dtype == np.uint32
    f32 = rec.view(np.float32)
    assert f32[0, 0] == 0 and f32[1, 1] == 1.0 and f32[1, 0] == 0.5  # entry 1.0, self-loop 0.5
    assert (rec[1, 2] & 0xFFFF) == 2 * phones[0] + 1 and (rec[1, 2] >> 16) == 2 * phones[0]
    assert f32[S - 1, 3] == 0.5 and np.all(f32[:-1, 3] == 0)
    ring = P.ChainGraph([(0, 1, 0, 1.0), (1, 0, 1, 0.5)], 2, 2, 0, [0.0, 0.5])
    assert linear_records(ring) is None  # a backward arc: not a linear chain
    C = _reference()
    topo = C.PhoneTopology(42)
    ref_g = C.build_numerator(phones, topo)
    np.testing.assert_array_equal(linear_records(ref_g), rec)
