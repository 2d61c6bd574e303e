"""CLI mirror of the reference's ``intattn`` command (cli.py): argument handling
and the file subcommands on CPU; the benchmark subcommands on the GPU."""
import json
import os

import numpy as np
import pytest

from paper_2511_21513_b200 import cli, tensor_io


def test_gen_tensor_and_compare_files(tmp_path, capsys):
    a = str(tmp_path / "a.itns")
    assert cli.main(["gen-tensor", "--len", "5", "--dim", "7", "--kind", "int8", "--seeds", "3",
                     "--out", a]) == 0
    m = tensor_io.load_tensor(a)
    assert m.shape == (5, 7) and m.dtype == np.int8
    rng = np.random.default_rng(3)
    assert np.array_equal(m, rng.integers(-127, 128, (5, 7)).astype(np.int8))
    assert cli.main(["compare-files", a, a, "--format", "json"]) == 0
    rows = json.loads(capsys.readouterr().out)
    assert rows[0]["cos_sim"] == pytest.approx(1.0) and rows[0]["rmse"] == 0.0


def test_bad_arguments_exit_2():
    with pytest.raises(SystemExit) as e:
        cli.main(["breakdown", "--len", "0"])
    assert e.value.code == 2
    with pytest.raises(SystemExit) as e:
        cli.main(["fidelity", "--pipelines", "int,bogus"])
    assert e.value.code == 2


def test_gen_inputs_matches_reference_recipe():
    q, k, v = cli.gen_inputs(16, 8, 0)
    rng = np.random.default_rng(0)
    for x in (q, k, v):
        assert np.array_equal(x, rng.standard_normal((16, 8), dtype=np.float32))


def test_write_rows_csv(tmp_path):
    out = str(tmp_path / "r.csv")
    cli.write_rows([{"a": 1, "b": 0.1}], "csv", out, ["note"])
    assert open(out).read() == "# note\na,b\n1,0.1\n"


@pytest.mark.gpu
def test_breakdown_fidelity_sweep_gpu(capsys):
    assert cli.main(["breakdown", "--len", "128,300", "--dim", "64", "--warmup", "1",
                     "--iters", "2", "--format", "json"]) == 0
    rows = json.loads(capsys.readouterr().out)
    assert [r["pipeline"] for r in rows] == ["int", "quant_only", "reference"] * 2
    assert all(r["total_ns"] > 0 and r["gflops"] > 0 for r in rows)
    assert cli.main(["fidelity", "--len", "256", "--dim", "64", "--format", "json"]) == 0
    rows = {r["comparison"]: r for r in json.loads(capsys.readouterr().out)}
    assert rows["int_vs_reference"]["cos_sim"] > 0.9
    assert rows["quant_only_vs_reference"]["cos_sim"] > 0.95
    assert cli.main(["sweep", "--len", "128", "--dim", "32", "--b", "4,5", "--c", "6.6",
                     "--format", "json"]) == 0
    rows = json.loads(capsys.readouterr().out)
    assert [(r["b"], r["c"]) for r in rows] == [(4, 6.6), (5, 6.6)]
