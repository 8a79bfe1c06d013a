"""Command-line front end over the device engine.

Mirrors `gwgrid` (proj/tools/gwgrid_main.cpp): subcommands over a dataset
directory (manifest.txt + GWG1 files kinship.gwg / xl.gwg / snps.gwg /
traits.gwg), key=value reports, a final machine-parseable `status=` line and
the same exit codes — 0 ok, 1 runtime failure, 2 usage, 3 verification failure
(gwgrid_main.cpp:4-5, 34-37).

  python -m paper_1210_7683_b200 generate --n N --p P --m M --t T --out DIR [--seed S]
  python -m paper_1210_7683_b200 solve    --data DIR [--out b.gwg] [--mb MB] [--device-eig]
  python -m paper_1210_7683_b200 verify   --data DIR [--results b.gwg] [--sample K | --exhaustive]
                                          [--tolerance 1e-8] [--seed S]
  python -m paper_1210_7683_b200 bench    --data DIR [--out bench_b.gwg] [--csv F]

`generate` draws BASELINE.json's generators (datagen.py); `tune` (the
reference's CPU/disk tuner) is out of scope and answers with a usage error.
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

from . import datagen, gwg1
from .engine import Engine, eigendecompose, verify_grid
from .errors import DimensionError, GwgridError, IoError, NotPositiveDefiniteError

OK, RUNTIME, USAGE, VERIFICATION = 0, 1, 2, 3


class _Parser(argparse.ArgumentParser):
    def error(self, message):
        print(f"error: {message}", file=sys.stderr)
        print("status=usage")
        raise SystemExit(USAGE)


def fmt(v: float) -> str:
    return f"{v:.9g}"


def write_dataset(out: str, n: int, p: int, m: int, t: int, seed: int) -> dict:
    """A gwgrid-dataset-1 directory (datagen.cpp:241-261 manifest keys)."""
    os.makedirs(out, exist_ok=True)
    ds = datagen.generate(n, p, m, t, seed=seed)
    lam = np.linalg.eigvalsh(ds["kinship"])
    gwg1.write_columns_stream(os.path.join(out, "kinship.gwg"), gwg1.KIND_OPERAND, ds["kinship"])
    gwg1.write_columns_stream(os.path.join(out, "xl.gwg"), gwg1.KIND_OPERAND, ds["xl"])
    gwg1.write_snp_stream(os.path.join(out, "snps.gwg"), ds["snps"])
    gwg1.write_trait_stream(os.path.join(out, "traits.gwg"), ds["traits"], ds["h2"], ds["sigma2"])
    with open(os.path.join(out, "manifest.txt"), "w") as f:
        f.write("# generator: BASELINE.json (Phi = G G^T/s + 1e-3 I, s = 2n; X_L = [1 | N(0,1)];\n"
                "# X_R ~ Binomial(2, maf); Y ~ N(0,1); h2 ~ U(0.05, 0.95); sigma2 = 1)\n")
        f.write("format=gwgrid-dataset-1\n"
                f"n={n}\np={p}\nm={m}\nt={t}\nseed={seed}\n"
                "kinship_model=random-spd\n"
                f"condition={fmt(lam.max() / lam.min())}\n"
                "h2_min=0.05\nh2_max=0.95\nsigma2_min=1\nsigma2_max=1\n"
                "kinship_file=kinship.gwg\nxl_file=xl.gwg\nsnps_file=snps.gwg\n"
                "traits_file=traits.gwg\n")
    return ds


def load_manifest(data_dir: str) -> dict:
    """load_manifest (datagen.cpp:317-396): key=value lines, '#' comments."""
    path = os.path.join(data_dir, "manifest.txt")
    kv = {}
    try:
        lines = open(path).read().splitlines()
    except OSError as e:
        raise IoError(f"cannot open manifest {path}") from e
    for no, line in enumerate(lines, 1):
        line = line.split("#", 1)[0].strip()
        if not line:
            continue
        if "=" not in line:
            raise IoError(f"manifest line {no} is not key=value in {path}")
        k, v = line.split("=", 1)
        kv[k] = v
    for key in ("format", "n", "p", "m", "t", "kinship_file", "xl_file", "snps_file",
                "traits_file"):
        if key not in kv:
            raise IoError(f"manifest {path} is missing key '{key}'")
    if kv["format"] != "gwgrid-dataset-1":
        raise IoError(f"manifest {path} has unsupported format '{kv['format']}'")
    out = {k: int(kv[k]) for k in ("n", "p", "m", "t")}
    for k in ("kinship", "xl", "snps", "traits"):
        out[k] = os.path.join(data_dir, kv[f"{k}_file"])
    return out


def _engine_for(man: dict, device_eig: bool, snp_coding: str = "auto") -> Engine:
    kin = gwg1.read_columns(man["kinship"], gwg1.KIND_OPERAND)
    xl = gwg1.read_columns(man["xl"], gwg1.KIND_OPERAND)
    eng = Engine(man["n"], man["p"])
    if device_eig:
        eng.set_kinship(kin)
    else:
        eng.set_spectrum(*eigendecompose(kin))
    eng.set_covariates(xl)
    eng.set_snp_coding(snp_coding)
    eng.set_traits_file(man["traits"])
    return eng


def cmd_generate(a) -> int:
    if a.p < 1 or a.p > a.n or a.m < 1 or a.t < 1:
        print("error: dimensions out of range (need 1 <= p <= n, m, t >= 1)", file=sys.stderr)
        print("status=usage")
        return USAGE
    write_dataset(a.out, a.n, a.p, a.m, a.t, a.seed)
    b = os.path.getsize(os.path.join(a.out, "snps.gwg")) + os.path.getsize(
        os.path.join(a.out, "traits.gwg"))
    print(f"manifest={os.path.join(a.out, 'manifest.txt')}\nbytes_stored={b}\nstatus=ok")
    return OK


def cmd_solve(a) -> int:
    man = load_manifest(a.data)
    out = a.out or os.path.join(a.data, "b.gwg")
    t0 = time.perf_counter()
    eng = _engine_for(man, a.device_eig, a.snp_coding)
    t1 = time.perf_counter()
    try:
        mb = int(a.mb) if a.mb else eng.default_slab_snps(man["m"])
        c = eng.run_grid_files(man["snps"], out, mb=a.mb)
    finally:
        eng.close()
    t2 = time.perf_counter()
    # every key of the reference's solve report (gwgrid_main.cpp:233-298), in
    # its order, plus the device's own (snp_coding, grid_flops, kernel_launches,
    # grid_kernel_seconds).  The device tiling: one trait pass (tb = t), SNP
    # slabs of mb columns that are also the transfer unit (nb = mb), no host
    # cache blocks (mbb = mb, tbb = t), rotation on the device (no transformed
    # stream is written).
    mb = min(mb, man["m"])
    stall = float(c.get("io_stall_ms", 0.0)) * 1e-3
    loops = t2 - t1
    print(f"scheduler=gpu\nsnp_coding={a.snp_coding}\nn={man['n']}\np={man['p']}\nm={man['m']}\nt={man['t']}")
    print(f"workers=1\nnb={mb}\nmb={mb}\ntb={man['t']}\nmbb={mb}\ntbb={man['t']}\ntransformed=")
    for k in ("preloop_flops", "loop_flops", "grid_flops", "context_builds", "bytes_loaded",
              "bytes_stored", "kernel_launches"):
        print(f"{k}={c[k]}")
    print(f"loop_transform_flops=0\ngrid_kernel_seconds={fmt(c['grid_kernel_ms'] * 1e-3)}\n"
          f"io_stall_seconds={fmt(stall)}\n"
          f"loops_wall_seconds={fmt(loops)}\npreloop_wall_seconds={fmt(t1 - t0)}\n"
          f"stall_fraction={fmt(stall / loops if loops > 0 else 0.0)}\nwall_time_s={fmt(loops)}\n"
          f"total_wall_seconds={fmt(t2 - t0)}\nout={out}\nstatus=ok")
    return OK


def cmd_verify(a) -> int:
    if a.sample < 1:
        print("error: --sample must be >= 1", file=sys.stderr)
        print("status=usage")
        return USAGE
    if not a.tolerance > 0:
        print("error: --tolerance must be > 0", file=sys.stderr)
        print("status=usage")
        return USAGE
    man = load_manifest(a.data)
    m, t, p = man["m"], man["t"], man["p"]
    res = a.results or os.path.join(a.data, "b.gwg")
    h = gwg1.read_header(res, gwg1.KIND_RESULT)
    if tuple(h["dims"]) != (m, t, p):
        raise DimensionError("results file shape does not match the dataset")
    total = m * t
    exhaustive = a.exhaustive or a.sample >= total
    rng = np.random.default_rng(a.seed)
    if exhaustive:
        ii, jj = np.arange(m), np.arange(t)
    else:
        cells = rng.choice(total, size=a.sample, replace=False)
        ii, jj = np.unique(cells % m), np.unique(cells // m)
    kin = gwg1.read_columns(man["kinship"], gwg1.KIND_OPERAND)
    xl = gwg1.read_columns(man["xl"], gwg1.KIND_OPERAND)
    snps = gwg1.read_columns(man["snps"], gwg1.KIND_SNP)[:, ii]
    th = gwg1.read_header(man["traits"], gwg1.KIND_TRAIT)
    n = th["dims"][0]
    raw = np.fromfile(man["traits"], dtype="<f8", offset=gwg1.HEADER)
    traits = raw[: n * t].reshape((n, t), order="F")[:, jj]
    h2, s2 = raw[n * t: n * t + t][jj], raw[n * t + t:][jj]
    b = np.memmap(res, dtype="<f8", mode="r", offset=gwg1.HEADER, shape=(t, m, p))
    sub = np.ascontiguousarray(b[np.ix_(jj, ii)].transpose(1, 0, 2))
    err, cells_err = verify_grid(kin, xl, snps, traits, h2, s2, sub, cell_errors=True)
    wi, wj = np.unravel_index(int(np.argmax(cells_err)), cells_err.shape)
    print(f"mode={'exhaustive' if exhaustive else 'sample'}\nchecked={cells_err.size}\n"
          f"tolerance={fmt(a.tolerance)}\nmax_rel_err={fmt(err)}\n"
          f"worst_snp={int(ii[wi])}\nworst_trait={int(jj[wj])}")
    if err <= a.tolerance:
        print("status=ok")
        return OK
    print("status=verification-failed")
    return VERIFICATION


def cmd_bench(a) -> int:
    man = load_manifest(a.data)
    out = a.out or os.path.join(a.data, "bench_b.gwg")
    eng = _engine_for(man, False, a.snp_coding)
    rows = ["workers,scheduler,wall_time_s,loop_flops,stall_fraction"]
    try:
        for mode in ("files", "memory"):
            eng.reset_counters()
            t0 = time.perf_counter()
            if mode == "files":
                c = eng.run_grid_files(man["snps"], out)
            else:
                snps = gwg1.read_columns(man["snps"], gwg1.KIND_SNP)
                t0 = time.perf_counter()
                eng.run_grid(snps)
                c = eng.counters()
            wall = time.perf_counter() - t0
            busy = c["grid_kernel_ms"] * 1e-3
            rows.append(f"1,gpu-{mode},{fmt(wall)},{c['loop_flops']},"
                        f"{fmt(max(0.0, 1.0 - busy / wall) if wall > 0 else 0.0)}")
    finally:
        eng.close()
    text = "\n".join(rows)
    print(text)
    if a.csv:
        with open(a.csv, "w") as f:
            f.write(text + "\n")
    print("status=ok")
    return OK


def main(argv=None) -> int:
    ap = _Parser(prog="python -m paper_1210_7683_b200",
                 description="grids of correlated GLS fits on a B200 over GWG1 streams")
    sub = ap.add_subparsers(dest="cmd", required=True, parser_class=_Parser)
    g = sub.add_parser("generate", help="write a synthetic dataset directory")
    for k in ("n", "p", "m", "t"):
        g.add_argument(f"--{k}", type=int, required=True)
    g.add_argument("--seed", type=int, default=1)
    g.add_argument("--out", required=True)
    s = sub.add_parser("solve", help="stream the whole grid to a result file")
    s.add_argument("--data", required=True)
    s.add_argument("--out", default="")
    s.add_argument("--mb", type=int, default=0)
    s.add_argument("--device-eig", action="store_true")
    s.add_argument("--snp-coding", choices=("auto", "real", "genotypes"), default="auto",
                   help="auto: per slab, the exact int8 tensor-core path when every value "
                        "is an integer code; genotypes: codes required; real: FP64 path")
    v = sub.add_parser("verify", help="recheck result cells against the Cholesky route")
    v.add_argument("--data", required=True)
    v.add_argument("--results", default="")
    v.add_argument("--sample", type=int, default=1000)
    v.add_argument("--exhaustive", action="store_true")
    v.add_argument("--tolerance", type=float, default=1e-8)
    v.add_argument("--seed", type=int, default=1)
    b = sub.add_parser("bench", help="CSV of wall time for the file and in-memory legs")
    b.add_argument("--data", required=True)
    b.add_argument("--out", default="")
    b.add_argument("--csv", default="")
    b.add_argument("--snp-coding", choices=("auto", "real", "genotypes"), default="auto")
    sub.add_parser("tune", help="(out of scope: the reference's CPU/disk tuner)")
    a = ap.parse_args(argv)
    if a.cmd == "tune":
        print("error: tune models CPU/disk tiling and is not part of the device engine",
              file=sys.stderr)
        print("status=usage")
        return USAGE
    try:
        return {"generate": cmd_generate, "solve": cmd_solve, "verify": cmd_verify,
                "bench": cmd_bench}[a.cmd](a)
    except NotPositiveDefiniteError as e:
        print(f"error: {e}", file=sys.stderr)
        print(f"error=not-positive-definite\nsnp_index={e.snp_index}\n"
              f"trait_index={e.trait_index}\nstatus=error")
        return RUNTIME
    except (GwgridError, OSError) as e:
        print(f"error: {e}", file=sys.stderr)
        print("status=error")
        return RUNTIME
