"""Host-side logic and the C-ABI library, without a GPU."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_1206_4973_b200 as fbb
from conftest import ROOT, gpu_present
from golden_util import CLASSES, instance_p, pool_nodes


def header_symbols():
    text = open(os.path.join(ROOT, "include", "flowbb_b200.h")).read()
    return sorted(set(re.findall(r"\b(fbb_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(fbb.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert set(fbb._lib.EXPORTED) == set(syms)


def test_library_is_sm100a_only():
    out = os.popen(f"cuobjdump --list-elf {fbb.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


@pytest.mark.skipif(gpu_present(), reason="checks the no-GPU failure path")
def test_create_fails_loudly_without_gpu():
    inst = fbb.generate_instance(20, 5, 873654221)
    with pytest.raises(fbb.BackendError):
        fbb.Context(inst)


def test_generate_instance_matches_reference(instances):
    for name, d in instances.items():
        inst = fbb.generate_instance(d["n"], d["m"], d["seed"])
        assert np.array_equal(inst.p, instance_p(instances, name)), name
    with pytest.raises(ValueError):
        fbb.generate_instance(3, 3, 0)


def test_instance_tails():
    inst = fbb.Instance(3, 2, [3, 2, 1, 4, 2, 3])
    assert inst.tails.tolist() == [[2, 0], [4, 0], [3, 0]]


@pytest.mark.parametrize("name", CLASSES)
def test_nodes_from_prefixes_heads(instances, pools, name):
    inst = fbb.Instance(*instance_p(instances, name).shape, instance_p(instances, name))
    prefixes, heads, _ = pool_nodes(pools, name)
    nodes = fbb.nodes_from_prefixes(inst, prefixes)
    assert np.array_equal(nodes.heads, heads)
    for i, pr in enumerate(prefixes):
        bits = set()
        for w in range(nodes.masks.shape[1]):
            v = int(nodes.masks[i, w])
            bits |= {64 * w + b for b in range(64) if (v >> b) & 1}
        assert bits == set(pr)


def test_split_slices_kats():  # test_backend.cpp:26-44
    assert fbb.split_slices(10, 3) == [(0, 4), (4, 3), (7, 3)]
    assert fbb.split_slices(7, 1) == [(0, 7)]
    assert [ln for _, ln in fbb.split_slices(2, 4)] == [1, 1, 0, 0]
    assert all(ln == 0 for _, ln in fbb.split_slices(0, 3))
    with pytest.raises(ValueError):
        fbb.split_slices(3, 0)


def test_merge_slices():  # test_backend.cpp:46-80
    assert list(fbb.merge_slices([[5, 7], [6], [9]], [(0, 2), (2, 1), (3, 1)])) == [5, 7, 6, 9]
    with pytest.raises(fbb.BackendError) as e:
        fbb.merge_slices([[5, 7], [6]], [(0, 2), (2, 2)])
    assert e.value.backend == 1
    rng = np.random.default_rng(61)
    for _ in range(20):
        total, k = int(rng.integers(0, 40)), int(rng.integers(1, 7))
        vals = rng.integers(0, 1000, total)
        sl = fbb.split_slices(total, k)
        assert list(fbb.merge_slices([vals[o:o + ln] for o, ln in sl], sl)) == list(vals)


# ---- tuner (autotune.hpp semantics, through the C library) ------------------------------------

def drive(tuner, curve, window, max_windows=100):
    for _ in range(max_windows):
        if tuner.phase() == fbb.TunerPhase.fixed:
            break
        for _ in range(window):
            t = tuner.target()
            tuner.observe(t, t / curve(t))
    assert tuner.phase() == fbb.TunerPhase.fixed


def test_tuner_initial_target():  # test_autotune.cpp:29-38
    D = fbb.BackendDescriptor
    assert fbb.Tuner(D(256, 4, 65536), 5).target() == 1024
    assert fbb.Tuner(D(1, 1, 8), 5).target() == 1
    with pytest.raises(ValueError):
        fbb.Tuner(D(256, 4, 65536), 0)
    with pytest.raises(ValueError):
        fbb.Tuner(D(256, 4, 512), 5)


def test_tuner_doubling():  # test_autotune.cpp:40-57
    t = fbb.Tuner(fbb.BackendDescriptor(256, 4, 65536), 5)
    for _ in range(5):
        t.observe(1024, 0.01)
    assert t.phase() == fbb.TunerPhase.doubling and t.target() == 2048 and t.best_batch() == 1024
    t = fbb.Tuner(fbb.BackendDescriptor(256, 4, 65536), 1)
    seen = []
    while t.phase() == fbb.TunerPhase.doubling:
        seen.append(t.target())
        t.observe(t.target(), 1.0)
    assert seen == [1024, 2048, 4096, 8192, 16384, 32768, 65536]


def test_tuner_probes():  # test_autotune.cpp:59-74
    t = fbb.Tuner(fbb.BackendDescriptor(1, 1, 16384), 1)
    curve = lambda x: 100.0 if x == 8192 else 10.0 + x * 1e-6  # noqa: E731
    while t.phase() == fbb.TunerPhase.doubling:
        t.observe(t.target(), t.target() / curve(t.target()))
    probes = []
    while t.phase() == fbb.TunerPhase.refining:
        probes.append(t.target())
        t.observe(t.target(), t.target() / curve(t.target()))
    assert probes == [5792, 6888, 9741, 11585] and t.best_batch() == 8192


def test_tuner_curves():  # test_autotune.cpp:76-147, acceptance C6
    import math
    D = fbb.BackendDescriptor

    def uni(x):
        z = math.log2(x) - math.log2(8192.0)
        return 1000.0 * math.exp(-z * z)

    t = fbb.Tuner(D(256, 4, 65536), 5)
    drive(t, uni, 5)
    assert 4096 <= t.best_batch() <= 16384
    t = fbb.Tuner(D(256, 4, 65536), 3)
    drive(t, float, 3)
    assert t.best_batch() == 65536 and t.target() == 65536
    t = fbb.Tuner(D(256, 4, 65536), 2)
    drive(t, lambda x: 500.0, 2)
    assert t.best_batch() == 1024
    t = fbb.Tuner(D(64, 3, 5000), 2)
    seen = []
    for _ in range(60):
        if t.phase() == fbb.TunerPhase.fixed:
            break
        for _ in range(2):
            seen.append(t.target())
            x = math.log2(t.target()) - math.log2(700.0)
            t.observe(t.target(), t.target() / (100.0 * math.exp(-x * x)))
    seen.append(t.best_batch())
    assert all(x >= 64 and x <= 5000 and x % 64 == 0 for x in seen)
    with pytest.raises(ValueError):
        t2 = fbb.Tuner(D(256, 4, 65536), 5)
        t2.observe(10, 0.0)


def test_tuner_b200_descriptor_grid():
    # grain 256 x 148 SMs doubles 37888 -> 75776 -> 151552 -> 303104
    t = fbb.Tuner(fbb.BackendDescriptor(256, 148, 303104), 1)
    seen = []
    while t.phase() == fbb.TunerPhase.doubling:
        seen.append(t.target())
        t.observe(t.target(), 1.0)
    assert seen == [37888, 75776, 151552, 303104]


@pytest.mark.parametrize("desc,window,probes,peak", [((256, 4, 65536), 5, 2, 9000.0),
                                                     ((64, 3, 5000), 2, 3, 700.0),
                                                     ((1, 1, 16384), 1, 2, 3000.0),
                                                     ((160, 296, 1 << 24), 2, 2, 2.0e5)])
def test_tuner_trace_matches_reference(desc, window, probes, peak):
    # Tuner::set_trace (autotune.hpp): same window index, measured batch and decision text
    # as the reference Tuner driven by the same synthetic curve
    from oracle import Ref
    try:
        ref = Ref()
    except FileNotFoundError:
        pytest.skip("oracle/_ref not built on this host")
    want = ref.tuner_trace(*desc, window, probes, peak)
    got = []
    t = fbb.Tuner(fbb.BackendDescriptor(*desc), window, probes)
    t.set_trace(lambda w, b, tp, d: got.append(f"{w} {b} {d}"))
    for _ in range(10000):
        if t.phase() == fbb.TunerPhase.fixed:
            break
        x = float(t.target())
        t.observe(t.target(), x / (x / (1.0 + (x / peak) ** 2)))
    assert got == want and len(got) >= 3
