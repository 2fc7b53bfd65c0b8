"""Command line front end (the reference's dangling `jigsaw.cli:main`, pkg/pyproject.toml:18-19;
SPEC.md cli module, 617-655): verification, training, benchmarking and report generation over a
JSON experiment config.

    python -m paper_2507_05753_b200 verify --config exp.json [--out DIR]
    python -m paper_2507_05753_b200 train  --config exp.json --out DIR
    python -m paper_2507_05753_b200 bench  {strong,roofline,weak,dp} [--workload C4] [--mp 2] --out DIR
    python -m paper_2507_05753_b200 report DIR/strong.csv [...]
    python -m paper_2507_05753_b200 flops  --config exp.json          # count_flops
    python -m paper_2507_05753_b200 co2    E_kWh PUE e_C              # co2_equiv

Multi-GPU runs are one process per GPU: launch `verify` / `train` under torchrun (the CLI owns
no numeric state); `bench strong` launches torchrun itself for each GPU count.
Exit codes: 0 success, 1 check failure, 2 config error, 3 runtime error.
ExperimentConfig: {"model": ModelConfig fields, "train": AdamConfig fields + steps / batch /
r_max / seed, "data": {"path": samples.npy, "lead": 1} or {"synthetic": N}, "world":
{"n_way": n, "dp_replicas": k}, "dtype": "bf16" | "f32", "seed": s}.
"""
from __future__ import annotations

import argparse
import csv
import hashlib
import json
import os
import subprocess
import sys

EXIT_OK, EXIT_CHECK, EXIT_CONFIG, EXIT_RUNTIME = 0, 1, 2, 3
N_WAY = (1, 2, 4, 8)


class ConfigErrors(ValueError):
    def __init__(self, errors):
        super().__init__("; ".join(errors))
        self.errors = errors


def load_config(path: str) -> dict:
    with open(path) as fh:
        return json.load(fh)


def config_hash(cfg: dict) -> str:
    """Reproducibility fingerprint embedded in every output."""
    return hashlib.sha256(json.dumps(cfg, sort_keys=True).encode()).hexdigest()[:16]


def validate(cfg: dict, world_size: int | None = None):
    """Resolve and check an experiment config; raises ConfigErrors naming every bad field."""
    from .config import ModelConfig
    from .errors import ConfigError
    from .train import AdamConfig
    errs = []
    try:
        model = ModelConfig.from_dict(cfg.get("model", {}))
    except (ConfigError, TypeError, ValueError) as e:
        raise ConfigErrors([f"model: {e}"]) from None
    world = cfg.get("world", {})
    n, k = int(world.get("n_way", 1)), int(world.get("dp_replicas", 1))
    if n not in N_WAY:
        errs.append(f"world.n_way: {n} not in {N_WAY}")
    if k < 1:
        errs.append(f"world.dp_replicas: {k} < 1")
    if world_size is not None and world_size != n * k:
        errs.append(f"world: WORLD_SIZE {world_size} != n_way {n} x dp_replicas {k}")
    if n in N_WAY:
        try:
            model.validate(n)
        except ConfigError as e:
            errs.append(f"model: {e}")
    tr = dict(cfg.get("train", {}))
    run = {key: tr.pop(key) for key in ("steps", "batch", "r_max", "seed", "epochs") if key in tr}
    try:
        adam = AdamConfig(**tr)
    except TypeError as e:
        errs.append(f"train: {e}")
        adam = AdamConfig()
    if adam.final_lr_body > adam.lr_body:
        errs.append(f"train.final_lr_body: {adam.final_lr_body} > lr_body {adam.lr_body}")
    if adam.warm_start > adam.lr_body:
        errs.append(f"train.warm_start: {adam.warm_start} > lr_body {adam.lr_body}")
    if adam.total_steps and adam.warmup_steps >= adam.total_steps:
        errs.append(f"train.warmup_steps: {adam.warmup_steps} >= total_steps {adam.total_steps}")
    if adam.clip_norm is not None and adam.clip_norm <= 0:
        errs.append(f"train.clip_norm: {adam.clip_norm} <= 0")
    for key in ("steps", "batch", "r_max"):
        if int(run.get(key, 1)) < 1:
            errs.append(f"train.{key}: {run[key]} < 1")
    if cfg.get("dtype", "bf16") not in ("bf16", "f32"):
        errs.append(f"dtype: {cfg['dtype']!r} not in ('bf16', 'f32')")
    if errs:
        raise ConfigErrors(errs)
    return model, adam, run, n, k


def co2_equiv(e_total_kwh: float, pue: float, e_c: float) -> float:
    """CO2e = E_total * PUE * e_C (PAPER.md 6.3.5), 3 significant figures."""
    if min(e_total_kwh, pue, e_c) < 0:
        raise ValueError("co2_equiv: inputs must be >= 0")
    v = e_total_kwh * pue * e_c
    return float(f"{v:.3g}")


def _ctx_from_env(n: int, k: int):
    from . import Communicator, MpContext
    comm = Communicator.from_env()
    if comm.world_size != n * k:
        raise ConfigErrors([f"world: WORLD_SIZE {comm.world_size} != {n} x {k}"])
    g = comm.rank // n
    return MpContext(comm, list(range(g * n, (g + 1) * n)))


def _local_block(x, R: int, C: int, r: int, c: int):
    """[B, lat, lon, vars] -> rank (r, c)'s sample block: contiguous longitude part r, channel
    part c (the layout WeatherMixerModel.forward takes; SPEC 4.2, model.py:114-121)."""
    lon, nv = x.shape[2], x.shape[3]
    return x[:, :, r * (lon // R):(r + 1) * (lon // R), c * (nv // C):(c + 1) * (nv // C)].copy()


def cmd_verify(args) -> int:
    """Equivalence check on this process group: the config is validated and its
    FLOP budget resolved; then the sharded model on these GPUs runs forward + backward on the
    reference's own golden sample (tests/golden, produced by running the reference package) and
    its output tile and the gathered global gradients are compared with the reference's f64
    results — 1e-4 relative in f32 (3xTF32), 2e-2 in bf16. JSON report; exit 1 on failure."""
    cfg = load_config(args.config)
    model_cfg, _, run, n, k = validate(cfg, int(os.environ.get("WORLD_SIZE", "1")))
    import numpy as np
    import torch
    import torch.distributed as dist
    from . import ModelConfig, WeatherMixerModel
    gold_dir = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
    z = np.load(os.path.join(gold_dir, "wm_golden.npz"))
    meta = json.load(open(os.path.join(gold_dir, "comm_golden.json")))
    ctx = _ctx_from_env(n, k)
    gcfg = ModelConfig.from_dict(meta["config"])
    report = {"config_hash": config_hash(cfg), "n_way": n, "train_flops_per_step": model_cfg.train_flops(),
              "golden_config": meta["config"], "checks": {}}
    ok = True

    def rel(a, b):
        return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))
    for dtype, tol in (("f32", 1e-4), ("bf16", 2e-2)):
        m = WeatherMixerModel(ctx, gcfg, seed=int(meta["seed"]), dtype=dtype)
        m.zero_grads()
        out = m.forward(torch.tensor(_local_block(z["x"], ctx.R, ctx.C, ctx.r, ctx.c), dtype=torch.float32))
        m.backward(torch.tensor(_local_block(z["g_out"], ctx.R, ctx.C, ctx.r, ctx.c), dtype=torch.float32))
        m.grad_sync()
        torch.cuda.synchronize()
        e_out = rel(out.cpu().numpy(), _local_block(z["out_f64"], ctx.R, ctx.C, ctx.r, ctx.c))
        grads = {name: p.grad.cpu().numpy() for name, p in m.params.items()}
        if ctx.n > 1:
            allg = [None] * ctx.comm.world_size
            dist.all_gather_object(allg, (ctx.pos, grads))
            per = {pos: gr for pos, gr in allg[ctx.group[0]:ctx.group[0] + ctx.n]}
            glob = {name: m.gather_global(name, {pos: per[pos][name] for pos in per}) for name in grads}
            t = torch.tensor([e_out], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=ctx.mp_group)
            e_out = float(t.item())
        else:
            glob = grads
        e_grad = max(rel(glob[name], z["grad_f64/" + name]) for name in glob)
        passed = e_out < tol and e_grad < tol
        ok &= passed
        report["checks"][dtype] = {"out_rel_err": e_out, "grad_rel_err": e_grad, "tol": tol, "pass": passed}
    if ctx.comm.rank == 0:
        text = json.dumps(report, indent=1)
        print(text)
        if args.out:
            os.makedirs(args.out, exist_ok=True)
            with open(os.path.join(args.out, "verify.json"), "w") as fh:
                fh.write(text)
    return EXIT_OK if ok else EXIT_CHECK


def cmd_train(args) -> int:
    """Trainer over TileLoader (data.path, .npy [N, lat, lon, vars]) or synthetic N(0,1) samples;
    per-step loss CSV + per-rank checkpoint shards in --out."""
    cfg = load_config(args.config)
    model_cfg, adam, run, n, k = validate(cfg, int(os.environ.get("WORLD_SIZE", "1")))
    import numpy as np
    from . import TileLoader, Trainer, WeatherMixerModel, checkpoint
    ctx = _ctx_from_env(n, k)
    data = cfg.get("data", {"synthetic": 8})
    lead = int(data.get("lead", 1))
    if "path" in data:
        src = data["path"]
    else:
        lat, lon = model_cfg.grid
        src = np.random.default_rng(int(cfg.get("seed", 0))).standard_normal(
            (int(data.get("synthetic", 8)) + lead, lat, lon, model_cfg.n_vars)).astype(np.float32)
    loader = TileLoader(src, model_cfg, ctx, lead=max(lead, int(run.get("r_max", 1))), batch=int(run.get("batch", 1)),
                        seed=int(run.get("seed", 0)))
    # padded rows / channels of the source weigh 0 in the loss
    model = WeatherMixerModel(ctx, model_cfg, seed=int(cfg.get("seed", 0)), dtype=cfg.get("dtype", "bf16"),
                              lat_real=loader.lat_real, vars_real=loader.vars_real)
    trainer = Trainer(model, batch=int(run.get("batch", 1)), adam=adam, r_max=int(run.get("r_max", 1)),
                      seed=int(run.get("seed", 0)))
    rows, steps_left = [], int(run.get("steps", loader.steps_per_epoch()))
    epoch = 0
    while steps_left > 0:
        res = trainer.train_epoch(loader, epoch=epoch, max_steps=steps_left)
        rows += [(epoch, i, r, loss) for i, (r, loss) in enumerate(zip(res["rollouts"], res["losses"]))]
        steps_left -= len(res["losses"])
        epoch += 1
        if not res["losses"]:
            break
    os.makedirs(args.out, exist_ok=True)
    for step in trainer.steps.values():
        checkpoint.save(step, os.path.join(args.out, "ckpt"))
        break
    if ctx.comm.rank == 0:
        with open(os.path.join(args.out, "loss.csv"), "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(["epoch", "step", "rollout", "loss", "config_hash"])
            for row in rows:
                w.writerow([*row, config_hash(cfg)])
        with open(os.path.join(args.out, "config.json"), "w") as fh:
            json.dump(cfg, fh, indent=1, sort_keys=True)
        print(f"trained {len(rows)} steps; loss {rows[0][3]:.5f} -> {rows[-1][3]:.5f}; outputs in {args.out}")
    return EXIT_OK


def _bench_line(n: int, workload: str, extra) -> dict:
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, os.path.join(root, "bench.py"), "--gpus", str(n), "--config", workload, "--no-cpu-baseline",
           *extra]
    if n > 1:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
               "--master-addr=127.0.0.1", f"--master-port={29800 + n}", *cmd[1:]]
    p = subprocess.run(cmd, capture_output=True, text=True)
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    if p.returncode != 0 or not lines:
        raise RuntimeError(f"bench n={n} failed: {p.stderr[-2000:]}")
    return json.loads(lines[-1])


def cmd_bench(args) -> int:
    """strong: the fixed global model at n = 1, 2, 4, 8 (those the node has); roofline: one line
    per workload rung. CSV + JSON sidecar (config, host fingerprint) in --out."""
    import platform
    import torch
    workloads = args.workload or ["C4"]
    os.makedirs(args.out, exist_ok=True)
    ngpu = torch.cuda.device_count()
    rows = []
    if args.suite == "strong":
        for wl in workloads:
            base = None
            for n in [m for m in N_WAY if m <= ngpu]:
                d = _bench_line(n, wl, ["--steps", str(args.steps), "--warmup", str(args.warmup)])
                base = base or d["value"]
                rows.append({"workload": wl, "n": n, "samples_per_s": d["value"], "ms_per_step": d["ms_per_step"],
                             "tflops": d["tflops"], "speedup": d["value"] / base,
                             "efficiency": d["value"] / (n * base), "e2e_samples_per_s": d["e2e"]["value"]})
    elif args.suite == "roofline":
        for wl in workloads:
            d = _bench_line(1, wl, ["--steps", str(args.steps), "--warmup", str(args.warmup)])
            rows.append({"workload": wl, "n": 1, "samples_per_s": d["value"], "tflops": d["tflops"],
                         "gemm_tflops": d["roofline"]["achieved"], "gemm_frac_of_peak": d["roofline"]["frac"],
                         "pct_bf16_peak": d["pct_bf16_peak"]})
    elif args.suite == "weak":
        # fixed per-rank work, model grown with n (Table 1 sizing: C5 has n / 2 blocks); weak
        # efficiency = baseline time / scaled time vs the smallest n
        workloads = args.workload or ["C5"]
        for wl in workloads:
            base = None
            for n in [m for m in N_WAY if m <= ngpu and (m > 1 or wl != "C5")]:
                d = _bench_line(n, wl, ["--steps", str(args.steps), "--warmup", str(args.warmup)])
                base = base or d
                per_rank = d["config"]["params"] / n
                rows.append({"workload": wl, "n": n, "samples_per_s": d["value"], "ms_per_step": d["ms_per_step"],
                             "tflops": d["tflops"], "params": d["config"]["params"],
                             "params_per_rank": per_rank,
                             "params_per_rank_vs_base": per_rank / (base["config"]["params"] / base["n_gpus"]),
                             "efficiency": base["ms_per_step"] / d["ms_per_step"],
                             "e2e_samples_per_s": d["e2e"]["value"]})
    elif args.suite == "dp":
        # dp_weak: one Jigsaw group of --mp ranks replicated over the node, the data grown with the
        # replica count (groups r % mp, Table 3); efficiency vs the single replica
        mp = args.mp
        for wl in workloads:
            base = None
            for k in [k for k in (1, 2, 4, 8) if k * mp <= ngpu]:
                d = _bench_line(k * mp, wl, ["--steps", str(args.steps), "--warmup", str(args.warmup),
                                             "--mp", str(mp)])
                base = base or d["value"]
                rows.append({"workload": wl, "n": k * mp, "mp": mp, "replicas": k, "samples_per_s": d["value"],
                             "ms_per_step": d["ms_per_step"], "tflops": d["tflops"], "speedup": d["value"] / base,
                             "efficiency": d["value"] / (k * base), "e2e_samples_per_s": d["e2e"]["value"]})
    else:
        raise ConfigErrors([f"bench suite {args.suite!r}: unknown"])
    if not rows:
        raise ConfigErrors([f"bench suite {args.suite!r}: no GPU count fits this node ({ngpu} GPUs)"])
    path = os.path.join(args.out, f"{args.suite}.csv")
    with open(path, "w", newline="") as fh:
        w = csv.DictWriter(fh, fieldnames=list(rows[0].keys()), quoting=csv.QUOTE_MINIMAL)
        w.writeheader()
        w.writerows(rows)
    with open(path[:-4] + ".json", "w") as fh:
        json.dump({"suite": args.suite, "workloads": workloads, "host": platform.node(),
                   "gpus": [torch.cuda.get_device_name(i) for i in range(ngpu)]}, fh, indent=1)
    print(f"wrote {path}")
    return EXIT_OK


def report(paths) -> str:
    """Merge suite CSVs into a text table of speedups / efficiencies vs the n = 1 row."""
    lines = [f"{'workload':10s} {'n':>3s} {'samples/s':>10s} {'speedup':>8s} {'efficiency':>10s}"]
    for path in paths:
        with open(path, newline="") as fh:
            rows = list(csv.DictReader(fh))
        base = {}
        for r in rows:
            if int(r["n"]) == 1:
                base[r["workload"]] = float(r["samples_per_s"])
        for r in rows:
            v, n = float(r["samples_per_s"]), int(r["n"])
            b = base.get(r["workload"])
            sp = float(r["speedup"]) if r.get("speedup") else (v / b if b else float("nan"))
            # weak / dp suites carry their own efficiency definition
            eff = float(r["efficiency"]) if r.get("efficiency") else sp / n
            lines.append(f"{r['workload']:10s} {n:3d} {v:10.3f} {sp:8.2f} {eff:10.2f}")
    return "\n".join(lines)


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2507_05753_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    p = sub.add_parser("verify")
    p.add_argument("--config", required=True)
    p.add_argument("--out")
    p = sub.add_parser("train")
    p.add_argument("--config", required=True)
    p.add_argument("--out", required=True)
    p = sub.add_parser("bench")
    p.add_argument("suite", choices=["strong", "roofline", "weak", "dp"])
    p.add_argument("--workload", action="append")
    p.add_argument("--out", required=True)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--mp", type=int, default=2, help="dp suite: Jigsaw group size of each replica")
    p = sub.add_parser("report")
    p.add_argument("csv", nargs="+")
    p = sub.add_parser("flops")
    p.add_argument("--config", required=True)
    p = sub.add_parser("co2")
    p.add_argument("values", nargs=3, type=float)
    args = ap.parse_args(argv)
    try:
        if args.cmd == "verify":
            return cmd_verify(args)
        if args.cmd == "train":
            return cmd_train(args)
        if args.cmd == "bench":
            return cmd_bench(args)
        if args.cmd == "report":
            print(report(args.csv))
            return EXIT_OK
        if args.cmd == "flops":
            cfg = load_config(args.config)
            model, _, run, _, _ = validate(cfg)
            print(json.dumps({"train_flops_per_step": model.train_flops(int(run.get("batch", 1))),
                              "config_hash": config_hash(cfg)}))
            return EXIT_OK
        if args.cmd == "co2":
            print(co2_equiv(*args.values))
            return EXIT_OK
    except ConfigErrors as e:
        for err in e.errors:
            print(f"config error: {err}", file=sys.stderr)
        return EXIT_CONFIG
    except (RuntimeError, OSError) as e:
        print(f"runtime error: {e}", file=sys.stderr)
        return EXIT_RUNTIME
    return EXIT_CONFIG


if __name__ == "__main__":
    sys.exit(main())
