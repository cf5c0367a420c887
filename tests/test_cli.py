"""flowbb-b200, the reference CLI's subcommands (tools/flowbb_main.cpp:62-244) over the
library: same options, output formats and exit codes.  The host-only paths (instance
generation and parsing, option errors) run on CPU; solve / workload / bench need the GPU
and are compared with the reference API compiled in place (oracle/_ref)."""
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_1206_4973_b200", "flowbb-b200")


def run(*args, check=None):
    r = subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=600)
    if check is not None:
        assert r.returncode == check, (r.returncode, r.stdout, r.stderr)
    return r


def simple(p):
    n, m = p.shape
    return f"{n} {m}\n" + "".join(" ".join(str(int(v)) for v in row) + "\n" for row in p)


def taillard(p, seed=1, ub=2, lb=3):
    n, m = p.shape
    rows = "".join(" ".join(str(int(p[j, k])) for j in range(n)) + "\n" for k in range(m))
    return (f"number of jobs, number of machines, initial seed, upper bound and lower bound :\n"
            f"{n} {m} {seed} {ub} {lb}\nprocessing times :\n{rows}")


def ref_or_skip():
    from oracle import Ref
    try:
        return Ref()
    except FileNotFoundError:
        pytest.skip("oracle/_ref not built on this host")


@pytest.mark.parametrize("n,m,seed", [(20, 5, 873654221), (20, 20, 479340445), (50, 20, 1539989115),
                                      (7, 3, 12345)])
def test_gen_instance_matches_reference(n, m, seed, tmp_path):
    ref = ref_or_skip()
    out = run("gen-instance", "--jobs", n, "--machines", m, "--seed", seed, check=0).stdout
    assert out == simple(ref.generate_instance(n, m, seed))      # to_simple_format
    f = tmp_path / "i.txt"
    run("gen-instance", "--jobs", n, "--machines", m, "--seed", seed, "--out", f, check=0)
    assert f.read_text() == out


def test_instance_formats_round_trip(tmp_path):
    rng = np.random.default_rng(3)
    p = rng.integers(0, 100, size=(7, 4))
    for fmt, text in (("simple", simple(p)), ("taillard", taillard(p))):
        f = tmp_path / f"{fmt}.txt"
        f.write_text(text)
        for sel in (fmt, "auto"):
            assert run("print-instance", "--instance", f, "--format", sel, check=0).stdout == simple(p)


def test_parse_errors_and_options(tmp_path):
    bad = tmp_path / "bad.txt"
    for text, msg in (("3 2\n1 2\n3 4\n", "unexpected end of input"),
                      ("2 2\n1 2\n3 x\n", "expected processing time"),
                      ("2 2\n1 2\n3 -4\n", "negative processing time"),
                      ("2 2\n1 2\n3 4\n5\n", "trailing data"),
                      ("0 2\n", "dimensions must be positive")):
        bad.write_text(text)
        r = run("print-instance", "--instance", bad, "--format", "simple", check=1)
        assert msg in r.stderr, (text, r.stderr)
    r = run("gen-instance", "--jobs", 3, "--machines", 2, "--seed", 0, check=1)
    assert "seed" in r.stderr
    assert "required" in run("gen-instance", "--jobs", 3, check=1).stderr
    assert "unknown option" in run("solve", "--nope", 1, check=1).stderr
    assert "excludes" in run("solve", "--instance", bad, "--batch", 8, "--autotune", check=1).stderr
    assert run("frobnicate").returncode == 1
    assert "cannot open" in run("print-instance", "--instance", tmp_path / "missing", check=1).stderr


@pytest.mark.gpu
def test_solve_matches_reference(tmp_path):
    ref = ref_or_skip()
    rng = np.random.default_rng(8)
    for trial in range(4):
        n, m = (8, 4) if trial % 2 == 0 else (9, 3)
        p = rng.integers(1, 60, size=(n, m)).astype(np.int32)
        f = tmp_path / f"i{trial}.txt"
        f.write_text(simple(p) if trial < 2 else taillard(p))
        opt, sched, counts = ref.solve(p, -1, fixed_batch=64, backends=1)
        r = run("solve", "--instance", f, "--batch", 64, check=0)
        kv = dict(line.split("=", 1) for line in r.stdout.strip().splitlines())
        assert int(kv["optimum"]) == opt
        assert [int(x) for x in kv["schedule"].split()] == list(sched)
        assert (int(kv["nodes_branched"]), int(kv["nodes_bounded"]), int(kv["nodes_pruned"])) \
            == counts
        js = json.loads(run("solve", "--instance", f, "--batch", 64, "--json", check=0).stdout)
        assert js["feasible"] and js["optimum"] == opt and js["nodes_bounded"] == int(counts[1])
        # an initial bound below the optimum: infeasible, exit 1 (flowbb_main.cpp:161-164)
        r = run("solve", "--instance", f, "--ub", opt, check=1)
        assert r.stdout.strip() == f"infeasible under given bound {opt}"
        js = json.loads(run("solve", "--instance", f, "--ub", opt, "--json", check=0).stdout)
        assert js["feasible"] is False
        # the tuner path and its trace
        r = run("solve", "--instance", f, "--autotune", "--window", 1, "--grain", 4,
                "--max-batch", 64, "--trace-tuner", check=0)
        assert f"optimum={opt}" in r.stdout and "tuner window=0 batch=" in r.stderr


@pytest.mark.gpu
def test_workload_snapshot_is_byte_identical_to_reference(tmp_path):
    ref = ref_or_skip()
    rng = np.random.default_rng(4)
    for (n, m, nodes, seed) in [(8, 4, 40, 7), (10, 5, 200, 3), (12, 4, 300, 11)]:
        p = rng.integers(1, 99, size=(n, m)).astype(np.int32)
        f = tmp_path / "i.txt"
        f.write_text(simple(p))
        # a frozen UB near the optimum keeps the batch-1 resolution small (a loose UB on a
        # 20-job instance would enumerate most of its 20! leaves)
        opt, *_ = ref.solve(p, -1, fixed_batch=256, backends=1)
        ub = opt + (10 if n <= 10 else 2)
        out = tmp_path / "wl.txt"
        run("workload", "--instance", f, "--ub", ub, "--nodes", nodes, "--seed", seed, "--out", out,
            check=0)
        assert out.read_text() == ref.workload_text(p, ub, nodes, seed)
        # bench: sequential (batch 1) vs batched resolution of the snapshot agree
        for fmt in ("csv", "json", "table"):
            r = run("bench", "--workload", out, "--batch", 64, "--format", fmt, check=0)
            if fmt == "csv":
                head, row = r.stdout.strip().splitlines()
                assert head == "instance,batch,backends,t_seq,t_par,speedup,nodes_bounded"
                assert row.startswith(f"{n}x{m},64,1,")
            elif fmt == "json":
                js = json.loads(r.stdout)
                assert js[0]["instance"] == f"{n}x{m}" and js[0]["batch"] == 64
            else:
                assert r.stdout.startswith("(No. of jobs x No. of machines) | 64")
