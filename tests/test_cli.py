"""CLI (reference cli.py:455-510): exit codes, the JSON
line formats of validate / simulate / train, tensor files (ops.py:464-492)."""

import json
import struct

import numpy as np
import pytest

from paper_1412_6249_b200 import cli
from paper_1412_6249_b200.tensorfile import read_tensor_file, write_tensor_file

CFG1 = {"net": {"input_shape": [3, 32, 32], "batch": 4, "lr": 1e-3,
                "layers": [{"kind": "conv", "out": 8, "kernel": 5, "stride": 1, "pad": 2},
                           {"kind": "relu"}, {"kind": "fc", "out": 10}]},
        "iterations": 2, "seed": 7, "data": {"kind": "synthetic", "spread": 0.0}}
DP2 = dict(CFG1, plan={"scheme": "data", "peers": [{"device": 0}, {"device": 1}],
                       "server": {"device": 2}})


def _write(tmp_path, name, obj):
    p = tmp_path / name
    p.write_text(json.dumps(obj))
    return str(p)


def test_validate_configs_and_graph_json(tmp_path, capsys):
    assert cli.main(["validate", "--config", _write(tmp_path, "c.json", CFG1)]) == 0
    lines = [json.loads(l) for l in capsys.readouterr().out.splitlines()]
    assert [l["graph"] for l in lines] == [0, 1]
    assert lines[0]["violations"] == [] and lines[0]["operators"] > 0
    assert cli.main(["validate", "--config", _write(tmp_path, "d.json", DP2)]) == 0
    capsys.readouterr()
    from paper_1412_6249_b200 import build_sgd_iteration, graph_to_json
    from paper_1412_6249_b200.nets import conv_relu_fc

    g = graph_to_json(build_sgd_iteration(conv_relu_fc()).graphs[0])
    assert cli.main(["validate", "--config", _write(tmp_path, "g.json", g)]) == 0
    assert json.loads(capsys.readouterr().out)["operators"] == len(g["operators"])


def test_validate_exit_codes(tmp_path, capsys):
    assert cli.main(["validate", "--config", str(tmp_path / "missing.json")]) == 2
    (tmp_path / "bad.json").write_text("{not json")
    assert cli.main(["validate", "--config", str(tmp_path / "bad.json")]) == 2
    assert cli.main(["validate", "--config", _write(tmp_path, "n.json", {"iterations": 1})]) == 2
    bad_conv = json.loads(json.dumps(CFG1))
    bad_conv["net"]["layers"][0]["stride"] = 3  # (32 + 4 - 5) / 3 is not integral
    assert cli.main(["validate", "--config", _write(tmp_path, "i.json", bad_conv)]) == 1
    assert cli.main(["validate", "--config",
                     _write(tmp_path, "p.json", dict(CFG1, net={"preset": "resnet"}))]) == 2
    capsys.readouterr()


def test_validate_preset_and_pipeline(tmp_path, capsys):
    cfg = {"net": {"preset": "googlenet", "batch": 2}, "seed": 1}
    assert cli.main(["validate", "--config", _write(tmp_path, "gn.json", cfg)]) == 0
    assert len(capsys.readouterr().out.splitlines()) == 2
    pipe = dict(CFG1, plan={"scheme": "model", "replicas": 2,
                            "stages": [{"layers": [0, 2], "device": 0},
                                       {"layers": [2, 3], "device": 1}]})
    assert cli.main(["validate", "--config", _write(tmp_path, "pp.json", pipe)]) == 0
    capsys.readouterr()
    assert cli.main(["train", "--config", _write(tmp_path, "pt.json", pipe)]) == 1  # forward-only


def test_simulate_lines(tmp_path, capsys):
    assert cli.main(["simulate", "--peers", "1..3", "--batch", "128", "--a", "0.002",
                     "--c", "0.05"]) == 0
    lines = [json.loads(l) for l in capsys.readouterr().out.splitlines()]
    assert lines[0]["model"] == {"a": 0.002, "c": 0.05, "batch_ref": 128.0}
    assert [l["peers"] for l in lines[1:]] == [1, 2, 3]
    assert lines[1]["ratio"] == 1.0
    fit = tmp_path / "fit.csv"
    fit.write_text("batch,images_per_sec\n# comment\n32,100.0\n128,200.0\n")
    assert cli.main(["simulate", "--peers", "2", "--batch", "64", "--fit", str(fit)]) == 0
    lines = [json.loads(l) for l in capsys.readouterr().out.splitlines()]
    assert lines[0]["model"]["batch_ref"] == 128.0 and lines[1]["peers"] == 2
    with pytest.raises(SystemExit):
        cli.main(["simulate", "--peers", "2", "--batch", "64"])


def test_tensor_file_format(tmp_path):
    a = np.arange(24, dtype=np.float32).reshape(2, 3, 4) / 7
    p = tmp_path / "t.bin"
    write_tensor_file(str(p), a)
    raw = p.read_bytes()
    assert raw[:16] == struct.pack("<4I", 3, 2, 3, 4)
    assert raw[16:] == a.astype("<f4").tobytes()
    assert np.array_equal(read_tensor_file(str(p)), a)
    p.write_bytes(raw[:-4])
    from paper_1412_6249_b200 import KernelError

    with pytest.raises(KernelError):
        read_tensor_file(str(p))


@pytest.mark.gpu
def test_train_streams_metrics_and_matches_reference(tmp_path, capsys, golden_train):
    """`train` on the reference's config 1 (conv32 k5 + relu + fc10, batch 16,
    lr 1e-3, spread 0, seed 7) reproduces the reference's losses; --captured
    replays the same iterations as CUDA graphs with the same losses."""
    cfg = {"net": {"input_shape": [3, 32, 32], "batch": 16, "lr": 1e-3,
                   "layers": [{"kind": "conv", "out": 32, "kernel": 5, "stride": 1, "pad": 2},
                              {"kind": "relu"}, {"kind": "fc", "out": 10}]},
           "iterations": 2, "seed": 7, "data": {"kind": "synthetic", "spread": 0.0}}
    path = _write(tmp_path, "cfg1.json", cfg)
    trace = tmp_path / "trace.json"
    assert cli.main(["train", "--config", path, "--trace-out", str(trace)]) == 0
    lines = [json.loads(l) for l in capsys.readouterr().out.splitlines()]
    assert [l["iteration"] for l in lines] == [0, 1]
    want = golden_train[1]["cfg1_losses"]
    for got, ref in zip([l["loss"] for l in lines], want):
        ref = ref[0] if isinstance(ref, list) else ref
        assert abs(got - ref) <= 1e-5 + 1e-4 * abs(ref), (got, ref)
    assert json.loads(trace.read_text())
    assert cli.main(["train", "--config", path, "--captured"]) == 0
    cap = [json.loads(l)["loss"] for l in capsys.readouterr().out.splitlines()]
    assert cap == [l["loss"] for l in lines]
