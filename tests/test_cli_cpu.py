"""CLI (SPEC.md cli module, 617-655): config validation with field-named errors and exit code 2,
count_flops, co2_equiv fixtures (PAPER Table 4), report speedups. No GPU needed."""
from __future__ import annotations

import csv
import json

import pytest

from paper_2507_05753_b200 import cli

DESK = {"n_vars": 8, "grid": [32, 64], "patch": [4, 4], "d_emb": 64, "d_tok": 128, "d_ch": 64, "n_blocks": 4}


def _write(tmp_path, cfg):
    p = tmp_path / "exp.json"
    p.write_text(json.dumps(cfg))
    return str(p)


def test_valid_config_resolves():
    model, adam, run, n, k = cli.validate({"model": DESK, "world": {"n_way": 2}, "train": {"steps": 3}})
    assert (n, k, run["steps"]) == (2, 1, 3) and model.d_emb == 64 and adam.lr_body == 1e-4


@pytest.mark.parametrize("bad,field", [
    ({"world": {"n_way": 3}}, "world.n_way"),                              # SPEC.md:637 n=3 rejected
    ({"train": {"final_lr_body": 1e-3}}, "train.final_lr_body"),            # SPEC.md:636 corrupted schedule
    ({"train": {"warmup_steps": 5, "total_steps": 5}}, "train.warmup_steps"),
    ({"dtype": "f16"}, "dtype"),
    ({"world": {"n_way": 2, "dp_replicas": 2}}, "world"),                    # WORLD_SIZE mismatch below
])
def test_config_errors_name_the_field(tmp_path, capsys, bad, field):
    cfg = {"model": DESK, **bad}
    if field == "world":
        with pytest.raises(cli.ConfigErrors) as e:
            cli.validate(cfg, world_size=2)
        assert any(err.startswith("world") for err in e.value.errors)
        return
    assert cli.main(["flops", "--config", _write(tmp_path, cfg)]) == cli.EXIT_CONFIG
    assert field in capsys.readouterr().err


def test_flops_matches_reference_count(tmp_path, capsys):
    # the reference's MpContext.flops for the desk config (C1) is 88,080,384 per step
    assert cli.main(["flops", "--config", _write(tmp_path, {"model": DESK})]) == 0
    out = json.loads(capsys.readouterr().out)
    assert out["train_flops_per_step"] == 88_080_384 and len(out["config_hash"]) == 16


def test_co2_equiv_table4():
    assert cli.co2_equiv(579, 1.05, 0.381) == 232
    assert cli.co2_equiv(643, 1.05, 0.381) == 257
    assert cli.co2_equiv(0, 1.05, 0.381) == 0
    with pytest.raises(ValueError):
        cli.co2_equiv(-1, 1.05, 0.381)


def test_report_speedups(tmp_path):
    p = tmp_path / "strong.csv"
    with open(p, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["workload", "n", "samples_per_s"])
        w.writerows([["C4", 1, 25.0], ["C4", 2, 43.0], ["C4", 4, 80.0]])
    text = cli.report([str(p)])
    lines = text.splitlines()[1:]
    assert lines[0].split()[3] == "1.00"           # speedup(n=1) = 1.00
    assert lines[2].split()[3] == "3.20" and lines[2].split()[4] == "0.80"


def test_report_weak_efficiency(tmp_path):
    # weak suite rows carry baseline_time / scaled_time: equal times -> 1.0
    p = tmp_path / "weak.csv"
    with open(p, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["workload", "n", "samples_per_s", "ms_per_step", "efficiency"])
        w.writerows([["C5", 2, 5.0, 200.0, 1.0], ["C5", 4, 4.0, 250.0, 0.8]])
    lines = cli.report([str(p)]).splitlines()[1:]
    assert lines[0].split()[4] == "1.00" and lines[1].split()[4] == "0.80"


def test_bench_suite_without_gpus_is_a_config_error(tmp_path):
    # no GPU count fits a GPU-less host: exit code 2, no bench process launched
    assert cli.main(["bench", "weak", "--out", str(tmp_path)]) == cli.EXIT_CONFIG
    assert cli.main(["bench", "dp", "--mp", "2", "--out", str(tmp_path)]) == cli.EXIT_CONFIG
