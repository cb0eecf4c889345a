"""NPY I/O, synthetic generation and the CLI surface."""
import json

import numpy as np
import pytest

from paper_2410_02367_b200 import cli


def test_npy_round_trip_and_errors(tmp_path):
    a = np.random.default_rng(0).standard_normal((1, 2, 5, 8)).astype(np.float32)
    p = str(tmp_path / "a.npy")
    cli.save_tensor(a, p)
    assert np.array_equal(cli.load_tensor(p).view(np.uint32), a.view(np.uint32))  # bit-identical
    h = a.astype(np.float16)
    cli.save_tensor(h, p)
    b = cli.load_tensor(p)
    assert b.dtype == np.float32 and np.array_equal(b, h.astype(np.float32))  # binary16 upcast
    np.save(p, np.asfortranarray(np.zeros((2, 2, 3, 4), np.float32)))
    with pytest.raises(cli.UnsupportedLayout):
        cli.load_tensor(p)
    np.save(p, np.zeros((2, 3, 4), np.float32))
    with pytest.raises(cli.ShapeError):
        cli.load_tensor(p)
    np.save(p, np.zeros((1, 1, 2, 2), np.float64))
    with pytest.raises(cli.UnsupportedDtype):
        cli.load_tensor(p)
    cli.save_tensor(a, p)
    raw = open(p, "rb").read()
    open(p, "wb").write(raw[:-7])
    with pytest.raises(cli.TruncatedPayload):
        cli.load_tensor(p)
    open(p, "wb").write(b"not an npy file")
    with pytest.raises(cli.MalformedHeader):
        cli.load_tensor(p)


def test_generate_deterministic_and_distributions():
    a = cli.generate((1, 1, 4096, 64), "normal", seed=3)
    b = cli.generate((1, 1, 4096, 64), "normal", seed=3)
    assert all(np.array_equal(x, y) for x, y in ((a.q, b.q), (a.k, b.k), (a.v, b.v)))
    assert abs(a.q.mean()) < 0.05 and abs(a.q.std() - 1) < 0.05
    o = cli.generate((1, 1, 2048, 64), "outlier", seed=1, bias_scale=10, noise_scale=1)
    k = o.k[0, 0].astype(np.float64)
    assert np.sqrt((k.mean(0) ** 2).mean()) >= 10 * k.std(0).mean()  # shared per-channel bias dominates
    ks = k - k.mean(0)
    assert np.abs(k).max() >= 5 * np.abs(ks).max()  # smooth-K removes it
    with pytest.raises(cli.ShapeError):
        cli.generate((1, 0, 4, 4))


def test_gen_command_and_preconditions(tmp_path, capsys):
    out = str(tmp_path / "t")
    assert cli.main(["gen", "--shape", "1,2,64,64", "--seed", "5", "--out", out]) == 0
    rep = json.loads(capsys.readouterr().out)
    q = cli.load_tensor(rep["files"]["q"])
    assert q.shape == (1, 2, 64, 64) and np.array_equal(q, cli.generate((1, 2, 64, 64), seed=5).q)
    with pytest.raises(ValueError, match="repeats"):
        cli.main(["bench", "--repeats", "1", "--shape", "1,1,128,64"])
    with pytest.raises(SystemExit):
        cli.main(["accuracy", "--shape", "1,2,3"])


@pytest.mark.gpu
def test_accuracy_and_calibrate_commands(cuda, tmp_path, capsys):
    out = str(tmp_path / "r.json")
    assert cli.main(["accuracy", "--shape", "1,2,1024,64", "--variant", "all", "--out", out]) == 0
    rep = json.load(open(out))["report"]
    assert rep["SAGEAttn-T"]["cos_sim"] >= 0.999 and rep["SAGEAttn-B"]["cos_sim"] >= 0.999  # Table 6
    assert set(rep) == {"SAGEAttn-T", "SAGEAttn-B", "SAGEAttn-vT", "SAGEAttn-vB"}
    capsys.readouterr()
    cli.main(["accuracy", "--shape", "1,2,1024,64", "--variant", "t", "--dist", "outlier", "--no-smooth"])
    rep = json.loads(capsys.readouterr().out)["report"]
    assert rep["SAGEAttn-T (no smooth-K)"]["cos_sim"] < rep["SAGEAttn-T"]["cos_sim"]
    for thr, expect in (("0.0", "SAGEAttn-vB"), ("1.0", "SAGEAttn-B")):
        cli.main(["calibrate", "--shape", "1,1,512,64", "--layers", "2", "--batches", "2", "--threshold", thr])
        plan = json.loads(capsys.readouterr().out)
        assert all(layer["kernel"] == expect for layer in plan["layers"])
    cli.main(["bench", "--shape", "1,2,1024,64", "--variant", "b", "--repeats", "3"])
    assert json.loads(capsys.readouterr().out)["report"]["SAGEAttn-B"]["tops"] > 0
