"""Command-line front end (entry point of the reference package,
``pkg/pyproject.toml:18-19`` -> ``tilevolve.cli:main``, which the reference does not ship).

    python -m paper_2205_15311_b200 enumerate --tiles 2 --labels 8 --k 8 --out s28.csv
    python -m paper_2205_15311_b200 ga --muL-grid 0.03,0.1,0.3 --runs 100 --out sweep.json
    python -m paper_2205_15311_b200 render --genome 0x000000/24 --tiles 2 --labels 8 [--format svg]
    python -m paper_2205_15311_b200 hash --bytes 0a0b0c | --shape FILE [--rot-invariant]

Every command that writes outputs also writes a config echo (``<out>.config.json``):
the fully resolved parameters, which ``--config ECHO`` reads back as defaults, so a
rerun from the echo is byte-identical.  The command layer owns no
compute: ``enumerate`` is ``classify.enumerate_space`` (device histogram), ``ga`` is
``evolve.sweep`` (device replica kernel), ``render`` is ``assembly.classify_tileset``
/ ``assemble_once`` (one device thread).  Exit status 0 iff every output was written
and the totals are consistent; any error prints one line to stderr and exits 2.

Under ``torchrun`` (WORLD_SIZE > 1, one GPU per rank) ``enumerate`` shards the index
range over the ranks (``distributed.enumerate_space_distributed``) and ``ga`` deals
every sweep point's runs over them (``distributed.sweep_distributed``); rank 0 writes
the outputs, which equal the single-GPU ones:

    python -m torch.distributed.run --nproc-per-node 8 -m paper_2205_15311_b200 enumerate ...
"""
from __future__ import annotations

import argparse
import csv
import json
import math
import os
import sys

import numpy as np

from .genome import Genome, GenomeError, SearchSpace, decode_tileset, index_of_genome, space_from_preset

# parameters that are outputs / runtime plumbing, not part of what a run computes
_NOT_ECHOED = {"config", "echo", "func", "progress"}


class CliError(Exception):
    pass


# ----------------------------------------------------------------------------- helpers
def _space(args) -> SearchSpace:
    try:
        if args.mask_preset:
            s = space_from_preset(args.mask_preset)
            if (args.tiles is not None and args.tiles != s.a) or (args.labels is not None and args.labels != s.b):
                raise CliError(f"--mask-preset {args.mask_preset} is a {s.a}-tile, {s.b}-label space")
            return s
        if args.tiles is None or args.labels is None:
            raise CliError("a space needs --tiles A --labels B (or --mask-preset NAME)")
        return SearchSpace(args.tiles, args.labels)
    except GenomeError as e:
        raise CliError(f"invalid space spec: {e}") from None


def _echo_path(args, default_out: str | None) -> str | None:
    if args.echo:
        return args.echo
    return default_out + ".config.json" if default_out else None


def _write_echo(path: str | None, command: str, args) -> None:
    if path is None:
        return
    conf = {k: v for k, v in vars(args).items() if k not in _NOT_ECHOED}
    with open(path, "w") as f:
        json.dump({"command": command, "args": conf}, f, indent=1, sort_keys=True)
        f.write("\n")


def _check_writable(path: str | None) -> None:
    if path is None:
        return
    d = os.path.dirname(os.path.abspath(path))
    if not os.path.isdir(d) or not os.access(d, os.W_OK):
        raise CliError(f"cannot write {path}: directory {d} is missing or not writable")


def _parse_float_list(text: str) -> list[float]:
    try:
        vals = [float(x) for x in text.replace(" ", "").split(",") if x != ""]
    except ValueError:
        raise CliError(f"invalid --muL-grid {text!r}: expected comma-separated numbers") from None
    if not vals:
        raise CliError("--muL-grid is empty")
    bad = [v for v in vals if not math.isfinite(v) or v < 0]
    if bad:
        raise CliError(f"invalid --muL-grid value {bad[0]!r}: expected a finite mu*L >= 0")
    return vals


def _parse_genome(text: str, space: SearchSpace) -> Genome:
    """``0xHEX/BITS`` (Genome.to_text), ``0xHEX`` or a ``0/1`` bit string of the space's length."""
    t = text.strip()
    try:
        if "/" in t:
            g = Genome.from_text(t)
        elif t.startswith("0x"):
            try:
                v = int(t, 16)
            except ValueError:
                raise CliError(f"malformed genome {text!r}: expected 0xHEX/BITS, 0xHEX or a bit string") from None
            g = Genome.from_int(space.bit_length, v)
        elif t and set(t) <= {"0", "1"}:
            if len(t) != space.bit_length:
                raise CliError(f"bit string has {len(t)} bits, the space has {space.bit_length}")
            g = Genome.from_int(space.bit_length, int(t, 2))
        else:
            raise CliError(f"malformed genome {text!r}: expected 0xHEX/BITS, 0xHEX or a bit string")
    except GenomeError as e:
        raise CliError(str(e)) from None
    if g.length != space.bit_length:
        raise CliError(f"genome has {g.length} bits, the space has {space.bit_length}")
    return g


def _dist() -> tuple[int, int]:
    """(rank, world); under torchrun joins the process group (NCCL, or TV_DIST_BACKEND) on
    this rank's GPU."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world <= 1:
        return 0, 1
    import torch
    import torch.distributed as dist
    if not dist.is_initialized():
        local = int(os.environ.get("LOCAL_RANK", "0"))
        if torch.cuda.is_available():  # (ranks share a GPU when there are fewer GPUs than ranks)
            torch.cuda.set_device(local % torch.cuda.device_count())
        backend = os.environ.get("TV_DIST_BACKEND") or ("nccl" if torch.cuda.is_available() else "gloo")
        dist.init_process_group(backend)
    return dist.get_rank(), dist.get_world_size()


# ----------------------------------------------------------------------------- enumerate
def cmd_enumerate(args) -> int:
    from .classify import enumerate_space

    if not args.out:
        raise CliError("--out is required")
    space = _space(args)
    if args.grid % 2 == 0 or args.grid < 3:
        raise CliError(f"--grid must be odd and >= 3, got {args.grid}")
    ks = sorted({int(x) for x in args.ks.split(",")}) if args.ks else [args.k]
    if min(ks) < 1:
        raise CliError("redundancy k must be >= 1")
    count = args.count if args.count is not None else space.cardinality - args.start
    if args.start < 0 or count < 0 or args.start + count > space.cardinality:
        raise CliError(f"[start, start+count) outside the space (cardinality {space.cardinality})")
    summary_path = args.summary or (os.path.splitext(args.out)[0] + ".summary.json")
    for p in (args.out, summary_path, args.checkpoint):
        _check_writable(p)
    if args.resume and not os.path.isfile(args.resume):
        raise CliError(f"checkpoint {args.resume} not found")
    rank, world = _dist()
    prog = None
    if not args.quiet and rank == 0:
        def prog(done, total):
            print(f"batches {done}/{total}", file=sys.stderr, flush=True)
    try:
        if world > 1:
            if args.checkpoint or args.resume:
                raise CliError("--checkpoint / --resume are single-GPU options (a multi-GPU run is one pass)")
            from .distributed import enumerate_space_distributed
            h = enumerate_space_distributed(space, d=args.grid, seed=args.seed, batch_size=args.batch_size,
                                            ks=ks, hist_k=args.hist_k, strict=not args.no_strict,
                                            start=args.start, count=count)
        else:
            h = enumerate_space(space, d=args.grid, seed=args.seed, batch_size=args.batch_size,
                                workers=args.workers, ks=ks, hist_k=args.hist_k, strict=not args.no_strict,
                                start=args.start, count=count, checkpoint=args.checkpoint,
                                checkpoint_every=args.checkpoint_every, resume=args.resume, progress=prog)
    except (ValueError, OSError) as e:  # corrupt / mismatched checkpoint, range errors
        raise CliError(str(e)) from None
    tallies = h.tallies
    if not all(int(r.sum()) == count for r in tallies):
        raise CliError(f"inconsistent totals: per-k sums {tallies.sum(axis=1).tolist()} != {count}")
    if rank != 0:  # every rank holds the merged histogram; rank 0 writes it
        return 0
    h.to_csv(args.out, space=space)
    summ = h.summary()
    # runtime plumbing (wall time, number of ranks) is not part of what the run computes
    summ["params"] = {k: v for k, v in summ["params"].items() if k not in ("runtime_s", "world")}
    summ["total"] = h.total
    with open(summary_path, "w") as f:
        json.dump(summ, f, indent=1, sort_keys=True)
        f.write("\n")
    _write_echo(_echo_path(args, args.out), "enumerate", args)
    if not args.quiet:
        row = h.class_counts()
        print(f"{h.total} genomes, {len(h)} shape hashes ({summ['deterministic_hashes']} deterministic); "
              f"k={h.hist_k}: " + " ".join(f"{k}={v}" for k, v in row.items()), file=sys.stderr)
    return 0


# ----------------------------------------------------------------------------- ga
def cmd_ga(args) -> int:
    from . import evolve as E

    if args.landscape != "fujiyama":
        raise CliError(f"unknown landscape {args.landscape!r} (the CLI sweeps the Fujiyama landscape; "
                       "JaTAM-shape fitness is evolve.run_ga(cfg, JatamFitness(...)))")
    if not args.out:
        raise CliError("--out is required")
    grid = _parse_float_list(args.muL if args.muL is not None else args.muL_grid)
    for name in ("pop", "length", "runs", "cutoff", "bootstrap", "sample_size"):
        if getattr(args, name) < 1:
            raise CliError(f"--{name.replace('_', '-')} must be >= 1")
    if args.length > 64:
        raise CliError("--length must be <= 64")
    if not 0 <= args.target <= args.length:
        raise CliError("--target must be in [0, length]")
    if args.mode not in E.MODES:
        raise CliError(f"--mode must be one of {sorted(E.MODES)}")
    _check_writable(args.out)
    base = E.GAConfig(pop_size=args.pop, length=args.length, mode=args.mode, cutoff=args.cutoff,
                      target=args.target, stop_when=args.stop_when)
    rank, world = _dist()
    if world > 1:
        from .distributed import sweep_distributed
        rows = sweep_distributed(grid, runs=args.runs, base=base, seed0=args.seed, sample_size=args.sample_size,
                                 resamples=args.bootstrap, out=args.out)
        if rank != 0:
            return 0
    else:
        rows = E.sweep(grid, runs=args.runs, base=base, seed0=args.seed, sample_size=args.sample_size,
                       resamples=args.bootstrap, out=args.out)
    _write_echo(_echo_path(args, args.out), "ga", args)
    if not args.quiet:
        for r in rows:
            d, a = r["discovery"], r["adaptation"]
            print(f"muL={r['muL']:g}: discovery median {d['median']} ({d['censored']} censored), "
                  f"adaptation median {a['median']} ({a['censored']} censored)", file=sys.stderr)
    return 0


# ----------------------------------------------------------------------------- render
def _svg(shape, title: str, cell: int = 16) -> str:
    w, h = shape.width * cell, shape.height * cell
    out = [f'<svg xmlns="http://www.w3.org/2000/svg" version="1.1" width="{w + 2}" height="{h + 22}">',
           f'<title>{title}</title>',
           f'<text x="1" y="14" font-family="monospace" font-size="12">{title}</text>']
    for y in range(shape.height):
        for x in range(shape.width):
            if shape.bitmap[y, x]:
                out.append(f'<rect x="{x * cell + 1}" y="{y * cell + 21}" width="{cell}" height="{cell}" '
                           f'fill="#4a7ab5" stroke="#1d3557"/>')
    out.append("</svg>")
    return "\n".join(out) + "\n"


def _render_one(space, g: Genome, args, want_hash: int | None = None) -> str:
    from . import assembly as A
    from .classify import crop, shape_hash

    tiles = decode_tileset(g, space)
    gi = index_of_genome(space, g)
    strict = not args.no_strict
    if want_hash is not None:
        # atlas row: the representative may be STERIC (rep = lowest DET-or-STERIC index), so draw
        # the first of its k runs that assembles the row's shape (the run _k:351-381 attributes)
        kind = A.classify_tileset(tiles, args.grid, args.k, seed=args.seed, genome_index=gi,
                                  strict_contacts=strict).kind.name
        for run in range(args.k):
            o = A.assemble_once(tiles, args.grid, seed=args.seed, genome_index=gi, run_index=run,
                                strict_contacts=strict)
            if o.grid is not None and shape_hash(crop(o.grid)) == want_hash:
                shape = crop(o.grid)
                break
        else:
            raise CliError(f"{g.to_text()}: no run assembles shape 0x{want_hash:08x} (histogram from other "
                           "parameters?)")
    elif args.k is None:
        o = A.assemble_once(tiles, args.grid, seed=args.seed, genome_index=gi, run_index=0, strict_contacts=strict)
        kind, shape = o.kind.name, (crop(o.grid) if o.grid is not None else None)
    else:
        c = A.classify_tileset(tiles, args.grid, args.k, seed=args.seed, genome_index=gi, strict_contacts=strict)
        kind, shape = c.kind.name, c.shape
    if shape is None:
        title = f"{g.to_text()} {kind}"
        return (_svg_empty(title) if args.format == "svg" else f"# {title}\n")
    title = f"{g.to_text()} {kind} {shape.width}x{shape.height} hash=0x{shape_hash(shape):08x}"
    if args.format == "svg":
        return _svg(shape, title)
    return f"# {title}\n{shape.to_ascii()}\n"


def _svg_empty(title: str) -> str:
    return (f'<svg xmlns="http://www.w3.org/2000/svg" version="1.1" width="320" height="22">'
            f'<title>{title}</title><text x="1" y="14" font-family="monospace" font-size="12">{title}</text>'
            f'</svg>\n')


def cmd_render(args) -> int:
    space = _space(args)
    if args.grid % 2 == 0 or args.grid < 3:
        raise CliError(f"--grid must be odd and >= 3, got {args.grid}")
    if args.k is not None and args.k < 1:
        raise CliError("redundancy k must be >= 1")
    if (args.genome is None) == (args.from_histogram is None):
        raise CliError("render needs exactly one of --genome or --from-histogram")
    parts = []
    if args.genome is not None:
        parts.append(_render_one(space, _parse_genome(args.genome, space), args))
    else:
        if args.k is None:
            args.k = 8
        if not os.path.isfile(args.from_histogram):
            raise CliError(f"histogram CSV {args.from_histogram} not found")
        with open(args.from_histogram, newline="") as f:
            rows = [r for r in csv.DictReader(f) if int(r["det_count"]) > 0]
        # Appendix A atlas order: most frequent deterministic shapes first (ties: hash)
        rows.sort(key=lambda r: (-int(r["det_count"]), int(r["hash_hex"], 16)))
        for r in rows[: args.top]:
            g = _parse_genome(r["representative_genome"], space)
            parts.append(f"# det_count={r['det_count']} steric_count={r['steric_count']} "
                         f"csv_hash={r['hash_hex']}\n" if args.format == "ascii" else "")
            parts.append(_render_one(space, g, args, want_hash=int(r["hash_hex"], 16)))
    text = "".join(parts)
    if args.out:
        _check_writable(args.out)
        with open(args.out, "w") as f:
            f.write(text)
        _write_echo(_echo_path(args, args.out), "render", args)
    else:
        sys.stdout.write(text)
    return 0


# ----------------------------------------------------------------------------- hash
def _read_ascii_shape(path: str):
    from .classify import CroppedShape

    try:
        with open(path) as f:
            # "# text" lines are annotations (render writes one above each shape); rows hold only '#' and '.'
            lines = [ln.strip() for ln in f if ln.strip() and not ln.startswith("# ")]
    except OSError as e:
        raise CliError(f"cannot read {path}: {e.strerror}") from None
    if not lines:
        raise CliError(f"{path}: no shape rows")
    width = max(len(ln) for ln in lines)
    if any(set(ln) - {"#", "."} for ln in lines):
        raise CliError(f"{path}: shape rows may only hold '#' (occupied) and '.' (empty)")
    bm = np.array([[c == "#" for c in ln.ljust(width, ".")] for ln in lines], bool)
    if not bm.any():
        raise CliError(f"{path}: the shape has no occupied cell")
    rows, cols = np.nonzero(bm.any(axis=1))[0], np.nonzero(bm.any(axis=0))[0]
    bm = bm[rows[0]:rows[-1] + 1, cols[0]:cols[-1] + 1]
    return CroppedShape(bm.shape[1], bm.shape[0], np.ascontiguousarray(bm))


def cmd_hash(args) -> int:
    from .classify import oat_hash, rotation_invariant_hash, shape_hash

    if (args.bytes is None) == (args.shape is None):
        raise CliError("hash needs exactly one of --bytes HEX or --shape FILE")
    if args.bytes is not None:
        if args.rot_invariant:
            raise CliError("--rot-invariant applies to --shape only")
        t = args.bytes.strip()
        t = t[2:] if t.startswith("0x") else t
        try:
            data = bytes.fromhex(t)
        except ValueError:
            raise CliError(f"malformed --bytes {args.bytes!r}: expected hex") from None
        v = oat_hash(np.frombuffer(data, np.uint8))
    else:
        s = _read_ascii_shape(args.shape)
        try:
            v = rotation_invariant_hash(s) if args.rot_invariant else shape_hash(s)
        except ValueError as e:
            raise CliError(str(e)) from None
    print(f"0x{v:08x}")
    return 0


# ----------------------------------------------------------------------------- parser
def _space_args(p) -> None:
    p.add_argument("--tiles", type=int, help="tile types a")
    p.add_argument("--labels", type=int, help="edge labels b (power of two)")
    p.add_argument("--mask-preset", help="named fixed-bit space, e.g. s32_3_8")
    p.add_argument("--grid", type=int, default=19, help="grid dimension d (odd, default 19)")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--no-strict", action="store_true", help="lenient contact rule (SPEC.md:174)")


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="tilevolve", description=__doc__.split("\n\n")[0])
    sub = ap.add_subparsers(dest="command", required=True)

    p = sub.add_parser("enumerate", help="exhaustive classification -> histogram CSV + summary JSON")
    _space_args(p)
    p.add_argument("--k", type=int, default=8, help="redundancy (runs per genome)")
    p.add_argument("--ks", help="comma-separated prefix ks to tally (default: --k)")
    p.add_argument("--hist-k", type=int, help="k the histogram attributes at (default: max ks)")
    p.add_argument("--workers", type=int, default=None, help="accepted for compatibility; the device schedules")
    p.add_argument("--batch-size", type=int, default=1 << 26)
    # (--start-index: torchrun's own parser rejects "--start" as an abbreviation of --start-method)
    p.add_argument("--start-index", "--start", dest="start", type=int, default=0)
    p.add_argument("--count", type=int, default=None)
    p.add_argument("--out", help="histogram CSV path (required)")
    p.add_argument("--summary", help="summary JSON path (default <out>.summary.json)")
    p.add_argument("--checkpoint", help="checkpoint path (written every --checkpoint-every batches)")
    p.add_argument("--checkpoint-every", type=int, default=64)
    p.add_argument("--resume", help="continue from a checkpoint")
    p.set_defaults(func=cmd_enumerate)

    p = sub.add_parser("ga", help="GA sweep over mu*L -> sweep JSON (medians, bootstrap CIs)")
    p.add_argument("--landscape", default="fujiyama")
    p.add_argument("--pop", type=int, default=512)
    p.add_argument("--length", type=int, default=32)
    p.add_argument("--muL-grid", dest="muL_grid", default="0.03,0.1,0.3,1,4")
    p.add_argument("--muL", type=str, default=None, help="a single mu*L (overrides --muL-grid)")
    p.add_argument("--runs", type=int, default=100)
    p.add_argument("--cutoff", type=int, default=20000)
    p.add_argument("--bootstrap", type=int, default=10000, help="bootstrap repetitions")
    p.add_argument("--sample-size", type=int, default=100, help="bootstrap sample size")
    p.add_argument("--mode", default="asexual", help="asexual | single_point | uniform")
    p.add_argument("--target", type=int, default=25, help="fitness threshold H >= target")
    p.add_argument("--stop-when", default="adaptation", choices=("never", "discovery", "adaptation"))
    p.add_argument("--seed", type=int, default=0, help="run r uses seed + r")
    p.add_argument("--out", help="sweep JSON path (required)")
    p.set_defaults(func=cmd_ga)

    p = sub.add_parser("render", help="assemble / classify one genome and draw its shape")
    _space_args(p)
    p.add_argument("--genome", help="0xHEX/BITS, 0xHEX or a bit string")
    p.add_argument("--k", type=int, default=None, help="classify at k runs (default: one assembly)")
    p.add_argument("--format", choices=("ascii", "svg"), default="ascii")
    p.add_argument("--from-histogram", help="atlas mode: histogram CSV from `enumerate`")
    p.add_argument("--top", type=int, default=16, help="atlas mode: shapes to draw")
    p.add_argument("--out", help="output file (default stdout)")
    p.set_defaults(func=cmd_render)

    p = sub.add_parser("hash", help="32-bit OAT hash of bytes or of an ASCII shape")
    p.add_argument("--bytes", help="hex bytes (empty string allowed)")
    p.add_argument("--shape", help="ASCII shape file ('#' occupied, '.' empty)")
    p.add_argument("--rot-invariant", action="store_true", help="sorted-four-rotation hash (SPEC.md:270-278)")
    p.set_defaults(func=cmd_hash)

    for p in sub.choices.values():
        p.add_argument("--config", help="config echo JSON of an earlier run (its args become defaults)")
        if p.prog.split()[-1] != "hash":
            p.add_argument("--echo", help="config echo path (default <out>.config.json)")
        p.add_argument("-q", "--quiet", action="store_true")
    return ap


def main(argv=None) -> int:
    argv = list(sys.argv[1:] if argv is None else argv)
    ap = build_parser()
    args = ap.parse_args(argv)
    try:
        if args.config:
            try:
                with open(args.config) as f:
                    echo = json.load(f)
            except (OSError, ValueError) as e:
                raise CliError(f"cannot read config echo {args.config}: {e}") from None
            if echo.get("command") != args.command:
                raise CliError(f"config echo is for {echo.get('command')!r}, not {args.command!r}")
            sub = ap._subparsers._group_actions[0].choices[args.command]
            known = {a.dest for a in sub._actions}
            sub.set_defaults(**{k: v for k, v in echo.get("args", {}).items() if k in known and k not in _NOT_ECHOED})
            args = ap.parse_args(argv)
        return args.func(args)
    except CliError as e:
        print(f"tilevolve {args.command}: error: {e}", file=sys.stderr)
        return 2
    finally:
        if "torch.distributed" in sys.modules:
            import torch.distributed as dist
            if dist.is_available() and dist.is_initialized():
                dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
