"""Soundness of the enumeration kernel's exact work elimination, checked on the CPU with
the oracle's restatement of the reference assembly (_k:96-381):

* trivial-freedom proof (v2 fixpoint, CandSwar::trivial_free in tv_fast.cuh): no genome
  it proves may go TRIVIAL in any of its k runs (the early-unbound cut-off relies on it);
* locally forced run-0 assemblies (CandSwar::forced_at): every later run of such a genome
  must end BOUNDED with run 0's hash (the genome is DET at every k after one run).

tools/work_analysis.c carries scalar restatements of both rules and counts violations
over whole spaces / stratified samples; the GPU parity tests check that the device
results are unchanged with the rules on or off (tests/test_gpu_parity.py SWITCHES)."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def analysis(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("wa") / "work_analysis")
    subprocess.run(["gcc", "-O2", "-fopenmp", "-Wno-unused-function", "-o", exe,
                    os.path.join(ROOT, "tools", "work_analysis.c")], check=True)

    def run(*args):
        out = subprocess.run([exe, *map(str, args)], check=True, capture_output=True, text=True).stdout
        return json.loads(out)
    return run


@pytest.mark.parametrize("args", [("2,4",), ("1,8",), ("2,2",), ("2,4", 0, 65536, 1, 0),
                                  ("s28", 0, 1 << 19, 256), ("s28", 0, 1 << 18, 64, 0),
                                  ("s32", 0, 1 << 19, 512)])
def test_proofs_have_no_counterexample(analysis, args):
    r = analysis(*args)
    assert r["v2_violations"] == 0
    assert r["forced"]["violations"] == 0 and r["forced"]["all_runs_equal"] == r["forced"]["genomes"]
    # the proofs are not vacuous
    assert r["trivial_free_v2_genomes"] > 0 and r["forced"]["genomes"] > 0
    # v2 proves at least what the round-1 proof (closure over placeable candidates) proves
    assert r["trivial_free_v2_genomes"] >= r["trivial_free_genomes"]


def test_one_mer_genomes_are_forced(analysis):
    r = analysis("s28", 0, 1 << 18, 64)
    assert r["one_mer"]["genomes"] > 0
    assert r["one_mer"]["runs"] == 8 * r["one_mer"]["genomes"]  # every 1-mer run ends BOUNDED
    assert r["forced"]["genomes"] >= r["one_mer"]["genomes"]
