"""CLI: usage / config errors on CPU; the four subcommands on
the GPU (check passes and reports an injected breach, quality beats the
random baseline, bench writes the reference CSV schema, fixtures load)."""

import csv
import json

import pytest

from paper_2509_24663_b200.__main__ import main


def test_usage_and_config_errors(tmp_path):
    assert main(["bogus"]) == 2
    assert main(["check", "--config", str(tmp_path / "missing.json")]) == 2
    bad = tmp_path / "cfg.json"
    bad.write_text(json.dumps({"k_top": -1}))
    assert main(["bench", "--config", str(bad), "--out", str(tmp_path)]) == 2
    bad.write_text(json.dumps({"not_a_field": 3}))
    assert main(["bench", "--config", str(bad), "--out", str(tmp_path)]) == 2


@pytest.mark.gpu
def test_cli_gpu(tmp_path):
    from paper_2509_24663_b200.core import load_tensor
    rc = main(["check", "--sizes", "300,1024", "--out", str(tmp_path)])
    rep = json.loads((tmp_path / "check.json").read_text())
    assert rc == 0 and rep["ok"], [c for c in rep["checks"] if not c["ok"]]
    assert len(rep["checks"]) >= 10
    assert main(["check", "--sizes", "300", "--out", str(tmp_path), "--perturb", "1"]) == 1
    assert main(["check", "--sizes", "", "--out", str(tmp_path)]) == 0   # no checks run
    assert main(["quality", "--sizes", "8192", "--out", str(tmp_path)]) == 0
    q = json.loads((tmp_path / "quality.json").read_text())
    assert q["recall"]["exact"] > q["recall"]["random"]
    assert main(["bench", "--sizes", "1024,8192", "--modes", "dense-tiled,sparse,select-approx",
                 "--out", str(tmp_path)]) == 0
    rows = list(csv.reader(open(tmp_path / "bench.csv")))
    assert rows[0] == ["mode", "n", "B", "k_top", "G", "d_h", "mac_count", "exp_count", "wall_ms",
                       "speedup_counts"]
    assert len(rows) == 1 + 2 * 3
    assert main(["gen-fixtures", "--sizes", "128", "--out", str(tmp_path)]) == 0
    man = json.loads((tmp_path / "manifest.json").read_text())
    assert load_tensor(tmp_path / man["fixtures"][0]["files"]["q"]).shape == (128, 32, 128)
