"""CLI: argument validation and `hash` on the CPU; `enumerate`,
`ga`, `render` on the GPU (they run the device paths), checked against the SPEC
examples and the reference golden of full S_{2,8}."""
import csv
import json
import os

import numpy as np
import pytest

from paper_2205_15311_b200.cli import main
from tests import _golden as G


def _run(argv, capsys):
    rc = main(argv)
    out = capsys.readouterr()
    return rc, out.out, out.err


# ------------------------------------------------------------------ CPU
def test_hash_bytes_examples(capsys):
    assert _run(["hash", "--bytes", ""], capsys)[:2] == (0, "0x00000000\n")
    from oracle import oracle as O
    for data, h in G.vectors()["oat"]:
        raw = bytes(data).hex()
        assert _run(["hash", "--bytes", raw], capsys)[1] == f"0x{h:08x}\n"  # golden byte vectors (reference)
        assert _run(["hash", "--bytes", "0x" + raw], capsys)[1] == f"0x{h:08x}\n"
    assert O.oat_hash_bytes(np.zeros(0, np.uint8)) == 0


def test_hash_shape_and_rotation_invariance(tmp_path, capsys):
    from paper_2205_15311_b200.classify import CroppedShape, rotation_invariant_hash, shape_hash
    L = np.array([[1, 0, 0], [1, 1, 1]], bool)
    s = CroppedShape(3, 2, L)
    hashes = set()
    for q in range(4):
        r = s.rotated(q)
        p = tmp_path / f"r{q}.txt"
        # padded with empty rows / columns and an annotation line: the file is cropped
        p.write_text("# annotation\n" + "....\n" + "\n".join("." + "".join("#" if v else "." for v in row)
                                                            for row in r.bitmap) + "\n")
        rc, out, _ = _run(["hash", "--shape", str(p)], capsys)
        assert rc == 0 and out == f"0x{shape_hash(r):08x}\n"
        rc, out, _ = _run(["hash", "--shape", str(p), "--rot-invariant"], capsys)
        hashes.add(out)
        assert out == f"0x{rotation_invariant_hash(s):08x}\n"
    assert len(hashes) == 1  # rotated shape files hash equal under --rot-invariant


@pytest.mark.parametrize("argv,msg", [
    (["hash", "--bytes", "0xzz"], "malformed"),
    (["hash"], "exactly one"),
    (["hash", "--bytes", "00", "--rot-invariant"], "--shape only"),
    (["hash", "--shape", "/nonexistent/shape.txt"], "cannot read"),
    (["ga", "--muL-grid", "0.3,-1", "--out", "x.json"], "invalid --muL-grid"),
    (["ga", "--muL-grid", "0.3,abc", "--out", "x.json"], "invalid --muL-grid"),
    (["ga", "--muL-grid", "nan", "--out", "x.json"], "invalid --muL-grid"),
    (["ga", "--muL-grid", "0.3"], "--out is required"),
    (["ga", "--landscape", "royal-road", "--out", "x.json"], "unknown landscape"),
    (["ga", "--runs", "0", "--out", "x.json"], "--runs"),
    (["enumerate", "--tiles", "2", "--labels", "3", "--out", "x.csv"], "invalid space spec"),
    (["enumerate", "--labels", "8", "--out", "x.csv"], "needs --tiles"),
    (["enumerate", "--mask-preset", "nope", "--out", "x.csv"], "unknown mask preset"),
    (["enumerate", "--mask-preset", "s32_3_8", "--tiles", "2", "--out", "x.csv"], "3-tile"),
    (["enumerate", "--tiles", "2", "--labels", "4", "--grid", "18", "--out", "x.csv"], "odd"),
    (["enumerate", "--tiles", "2", "--labels", "4", "--start", "65530", "--count", "10", "--out", "x.csv"],
     "outside the space"),
    (["enumerate", "--tiles", "2", "--labels", "4", "--out", "/nonexistent/dir/x.csv"], "cannot write"),
    (["enumerate", "--tiles", "2", "--labels", "4", "--out", "x.csv", "--resume", "/nonexistent.ckpt"], "not found"),
    (["render", "--tiles", "2", "--labels", "4"], "exactly one"),
    (["render", "--tiles", "2", "--labels", "4", "--genome", "0xzz"], "malformed"),
    (["render", "--tiles", "2", "--labels", "4", "--genome", "0101"], "16"),
    (["render", "--tiles", "2", "--labels", "4", "--genome", "0x00/8"], "16"),
])
def test_invalid_arguments_exit_nonzero(argv, msg, capsys, tmp_path, monkeypatch):
    monkeypatch.chdir(tmp_path)
    rc, out, err = _run(argv, capsys)
    assert rc == 2 and msg in err and out == ""


def test_config_echo_wrong_command(tmp_path, capsys):
    p = tmp_path / "echo.json"
    p.write_text(json.dumps({"command": "ga", "args": {}}))
    rc, _, err = _run(["hash", "--bytes", "00", "--config", str(p)], capsys)
    assert rc == 2 and "not 'hash'" in err


def test_module_entry_point():
    import subprocess
    import sys
    r = subprocess.run([sys.executable, "-m", "paper_2205_15311_b200", "hash", "--bytes", "61"],
                       capture_output=True, text=True, cwd=os.path.dirname(os.path.dirname(__file__)))
    assert r.returncode == 0 and r.stdout == "0xca2e9442\n"


# ------------------------------------------------------------------ GPU
def _csv_totals(path):
    with open(path, newline="") as f:
        rows = list(csv.DictReader(f))
    return rows


@pytest.mark.gpu
def test_enumerate_s24_totals_and_echo_rerun(tmp_path, capsys):
    out = tmp_path / "s24.csv"
    rc, _, err = _run(["enumerate", "--tiles", "2", "--labels", "4", "--k", "16", "--out", str(out),
                       "--batch-size", "20000"], capsys)
    assert rc == 0, err
    summ = json.loads((tmp_path / "s24.summary.json").read_text())
    assert summ["total"] == 65536 and sum(summ["totals"]["16"].values()) == 65536
    assert "batches 4/4" in err
    rows = _csv_totals(out)
    assert sum(int(r["det_count"]) for r in rows) == summ["totals"]["16"]["DET"]
    # rerun from the config echo (different batching, same outputs): byte-identical CSV
    out2 = tmp_path / "again.csv"
    rc, _, err = _run(["enumerate", "--config", str(out) + ".config.json", "--out", str(out2), "--batch-size",
                       "65536", "-q"], capsys)
    assert rc == 0, err
    assert out2.read_bytes() == out.read_bytes()
    assert (tmp_path / "again.summary.json").read_text() == (tmp_path / "s24.summary.json").read_text()


@pytest.mark.gpu
def test_enumerate_s28_matches_reference(tmp_path, capsys):
    out = tmp_path / "s28.csv"
    rc, _, err = _run(["enumerate", "--tiles", "2", "--labels", "8", "--k", "8", "--ks", "1,2,4,8",
                       "--out", str(out), "-q"], capsys)
    assert rc == 0, err
    summ = json.loads((tmp_path / "s28.summary.json").read_text())
    assert summ["total"] == 16777216
    g = G.hist_golden("s28_full")
    for i, k in enumerate((1, 2, 4, 8)):
        assert [summ["totals"][str(k)][c] for c in ("DET", "TRIV", "STERIC", "UNB", "ERROR")] == \
            g["tallies"][i].tolist()
    rows = _csv_totals(out)
    assert [int(r["hash_hex"], 16) for r in rows] == g["keys"].tolist()
    assert [int(r["det_count"]) for r in rows] == g["det"].tolist()
    assert [int(r["steric_count"]) for r in rows] == g["steric"].tolist()


@pytest.mark.gpu
def test_enumerate_checkpoint_resume_and_corrupt(tmp_path, capsys):
    base = ["enumerate", "--tiles", "2", "--labels", "4", "--k", "4", "--batch-size", "8192", "-q"]
    full = tmp_path / "full.csv"
    assert _run(base + ["--out", str(full)], capsys)[0] == 0
    ck = tmp_path / "run.ckpt"
    part = tmp_path / "part.csv"
    # a run that stops after 3 of 8 batches leaves its checkpoint behind
    assert _run(base + ["--out", str(part), "--count", str(3 * 8192), "--checkpoint", str(ck),
                        "--checkpoint-every", "1"], capsys)[0] == 0
    # a resume must use the same plan: the partial run's cursor does not fit the full plan
    rc, _, err = _run(base + ["--out", str(part), "--resume", str(ck)], capsys)
    assert rc == 2 and "chunk plan" in err
    ck2 = tmp_path / "full.ckpt"
    assert _run(base + ["--out", str(part), "--checkpoint", str(ck2), "--checkpoint-every", "3"], capsys)[0] == 0
    res = tmp_path / "resumed.csv"
    assert _run(base + ["--out", str(res), "--resume", str(ck2)], capsys)[0] == 0
    assert res.read_bytes() == full.read_bytes()
    bad = tmp_path / "bad.ckpt"
    bad.write_bytes(b"garbage")
    rc, _, err = _run(base + ["--out", str(res), "--resume", str(bad)], capsys)
    assert rc == 2 and "checkpoint" in err


@pytest.mark.gpu
def test_ga_sweep_json(tmp_path, capsys):
    out = tmp_path / "sweep.json"
    rc, _, err = _run(["ga", "--muL-grid", "0.3,1", "--runs", "20", "--bootstrap", "500", "--out", str(out)],
                      capsys)
    assert rc == 0, err
    doc = json.loads(out.read_text())
    assert [p["muL"] for p in doc["points"]] == [0.3, 1.0]
    assert doc["config"]["pop_size"] == 512 and doc["config"]["cutoff"] == 20000
    for p in doc["points"]:
        for name in ("discovery", "adaptation"):
            r = p[name]
            if r["median"] is not None:  # monotone-checkable schema: lo <= median <= hi
                assert r["ci_lo"] <= r["median"] <= r["ci_hi"]
    # muL = 0 from the all-zero start -> discovery censored in every run
    out0 = tmp_path / "zero.json"
    rc, _, err = _run(["ga", "--muL", "0", "--runs", "10", "--cutoff", "300", "--bootstrap", "100",
                       "--out", str(out0), "-q"], capsys)
    assert rc == 0, err
    p = json.loads(out0.read_text())["points"][0]
    assert p["discovery"]["censored"] == 10 and p["discovery"]["median"] is None
    # echo rerun is identical
    out1 = tmp_path / "zero2.json"
    assert _run(["ga", "--config", str(out0) + ".config.json", "--out", str(out1), "-q"], capsys)[0] == 0
    assert out1.read_text() == out0.read_text()


@pytest.mark.gpu
def test_render_examples(tmp_path, capsys):
    # SPEC:498 all-zero genome -> 1x1 '#'
    rc, out, err = _run(["render", "--tiles", "2", "--labels", "8", "--genome", "0x000000/24"], capsys)
    assert rc == 0, err
    assert out.splitlines()[1:] == ["#"] and "BOUNDED" in out
    # SPEC:499 dimer tile set [(2,0,0,0),(0,0,1,0)] -> vertical 1x2 (here in S_{2,4}: 2 bits per label)
    rc, out, err = _run(["render", "--tiles", "2", "--labels", "4", "--genome", "0x8004/16", "--k", "8"], capsys)
    assert rc == 0, err
    assert out.splitlines()[1:] == ["#", "#"] and "DETERMINISTIC 1x2" in out
    # a column (self-stacking tile) is annotated, not failed
    rc, out, err = _run(["render", "--tiles", "2", "--labels", "4", "--genome", "1000010000000000", "--k", "4"],
                        capsys)
    assert rc == 0 and "UNBOUND" in out
    svg = tmp_path / "dimer.svg"
    rc, _, err = _run(["render", "--tiles", "2", "--labels", "4", "--genome", "0x8004/16", "--k", "8",
                       "--format", "svg", "--out", str(svg)], capsys)
    assert rc == 0, err
    text = svg.read_text()
    assert text.startswith("<svg") and text.count("<rect") == 2 and "DETERMINISTIC" in text


@pytest.mark.gpu
def test_render_atlas_from_histogram(tmp_path, capsys):
    from paper_2205_15311_b200.classify import CroppedShape, shape_hash
    csvp = tmp_path / "s24.csv"
    assert _run(["enumerate", "--tiles", "2", "--labels", "4", "--k", "8", "--out", str(csvp), "-q"], capsys)[0] == 0
    rows = sorted((r for r in _csv_totals(csvp) if int(r["det_count"]) > 0),
                  key=lambda r: (-int(r["det_count"]), int(r["hash_hex"], 16)))
    rc, out, err = _run(["render", "--tiles", "2", "--labels", "4", "--from-histogram", str(csvp), "--top", "5"],
                        capsys)
    assert rc == 0, err
    blocks = [b for b in out.split("# det_count=")[1:]]
    assert len(blocks) == min(5, len(rows))
    for r, b in zip(rows, blocks):
        lines = b.splitlines()
        # the representative may classify STERIC; the drawn run is the one that assembles the row's shape
        assert f"csv_hash={r['hash_hex']}" in lines[0] and f"hash={r['hash_hex']}" in lines[1]
        bm = np.array([[c == "#" for c in ln] for ln in lines[2:]], bool)
        s = CroppedShape(bm.shape[1], bm.shape[0], bm)
        assert f"0x{shape_hash(s):08x}" == r["hash_hex"]  # the drawn shape is the CSV row's shape


def test_torchrun_refuses_checkpoint_options(tmp_path):
    """Under torchrun (two CPU ranks over gloo) a multi-GPU enumeration is one pass: --checkpoint
    is refused on every rank with the CLI's one-line error, before any device work."""
    import socket
    import subprocess
    import sys
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, TV_DIST_BACKEND="gloo", CUDA_VISIBLE_DEVICES="")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), "-m", "paper_2205_15311_b200",
                        "enumerate", "--tiles", "2", "--labels", "4", "--out", str(tmp_path / "x.csv"),
                        "--checkpoint", str(tmp_path / "ck.bin")], cwd=root, env=env, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode != 0
    assert r.stderr.count("--checkpoint / --resume are single-GPU options") == 2
