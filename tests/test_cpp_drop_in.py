"""The reference's own C++ API driving the device path.

tests/cpp/ref_drop_in.cpp is compiled from the unmodified reference headers
(-I /root/reference/proj/include at build time) and include/desklm_b200/
traits.hpp: desklm::Trainer<GpuStandardTraits> / <GpuBottleneckTraits>, the
sharded_perplexity / rnn_perplexity / rescore_nbest overloads and the
RNLM / RNBL / RNQZ with_model dispatch run beside the reference's CPU
Trainer<StandardTraits> / <BottleneckTraits> and scorers on identical inputs
(trainer.hpp:117-476, eval.hpp:84-222, :693-790, tools/desklm.cpp:142-163).
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tests", "cpp", "build", "ref_drop_in")


def test_drop_in_driver_is_built():
    r = subprocess.run(["make", "-C", os.path.join(ROOT, "tests", "cpp")], capture_output=True,
                       text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert os.path.exists(EXE), "tests/cpp/build/ref_drop_in (needs /root/reference at build)"


def _run(case):
    r = subprocess.run([EXE, case], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr
    return [l for l in r.stdout.splitlines() if l.startswith("ok ")]


@pytest.mark.gpu
def test_reference_trainer_with_gpu_traits():
    """Trainer<GpuStandardTraits> == Trainer<StandardTraits> (softmax and NCE):
    logs, cursors, generator, RTRN readable by the reference, resume."""
    ok = _run("train")
    assert any(l.startswith("ok train softmax") for l in ok)
    assert any(l.startswith("ok train nce") for l in ok)


@pytest.mark.gpu
def test_reference_bottleneck_trainer_with_gpu_traits():
    ok = _run("bn")
    assert any(l.startswith("ok bn softmax") for l in ok)
    assert any(l.startswith("ok bn nce") for l in ok)


@pytest.mark.gpu
def test_with_gpu_model_perplexity():
    ok = _run("ppl")
    assert {"ok ppl RNLM", "ok ppl RNBL", "ok ppl RNQZ"} <= set(ok)


@pytest.mark.gpu
def test_rescore_nbest_overloads():
    ok = _run("rescore")
    assert {"ok rescore rnn-only", "ok rescore interpolated", "ok rescore fast"} <= set(ok)


CLI = os.path.join(ROOT, "tools", "build", "desklm_b200")


def test_cli_is_built():
    r = subprocess.run(["make", "-C", os.path.join(ROOT, "tools")], capture_output=True,
                       text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert os.path.exists(CLI)
    r = subprocess.run([CLI, "no-such-command"], capture_output=True, text=True)
    assert r.returncode == 1  # usage error, as the reference CLI


@pytest.mark.gpu
def test_cli_train_ppl_rescore(tmp_path, orc):
    """desklm_b200 rnn-train / rnn-ppl / rescore (tools/desklm.cpp:509-744
    on the device): the trained RNLM file scores like the oracle, the RTRN
    checkpoint resumes, the n-best file is re-ranked."""
    import numpy as np

    from paper_1502_00512_b200 import formats, make_vocab
    V, H = 50, 16
    tr, va = orc.random_stream_pair(13, V, 1200, 300)
    words = make_vocab(V)
    (tmp_path / "vocab.txt").write_text("".join(w + "\n" for w in words))
    for name, ids in (("train.ids", tr), ("valid.ids", va)):
        (tmp_path / name).write_text(" ".join(str(int(i)) for i in ids) + "\n")
    base = [CLI, "rnn-train", "--train", str(tmp_path / "train.ids"), "--valid",
            str(tmp_path / "valid.ids"), "--vocab", str(tmp_path / "vocab.txt"), "--nstate",
            str(H), "--noffset", "2", "--minibatch", "4", "--unroll", "5", "--eta", "0.05",
            "--mode", "softmax", "--precision", "fp32", "--quiet"]
    r = subprocess.run(base + ["--max-epochs", "2", "--out", str(tmp_path / "m.rnlm"),
                               "--checkpoint", str(tmp_path / "ck.rtrn"), "--log",
                               str(tmp_path / "log.csv")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert (tmp_path / "log.csv").read_text().startswith("epoch,train_loss,valid_ppl")
    params, act, vocab = formats.read_params((tmp_path / "m.rnlm").read_bytes())
    assert list(vocab) == words
    r = subprocess.run([CLI, "rnn-ppl", "--model", str(tmp_path / "m.rnlm"), "--ids",
                        str(tmp_path / "valid.ids"), "--shards", "4", "--precision", "fp32",
                        "--quiet"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    want = orc.sharded_ppl(params, act, va, 4)["perplexity"]
    assert float(r.stdout) == pytest.approx(want, rel=1e-5)
    # resume for a third epoch from the checkpoint
    r = subprocess.run(base + ["--max-epochs", "3", "--resume", str(tmp_path / "ck.rtrn"),
                               "--out", str(tmp_path / "m3.rnlm")], capture_output=True,
                       text=True)
    assert r.returncode == 0, r.stderr
    # rescoring: bos + words + eos per hypothesis, re-ranked per utterance
    rng = np.random.default_rng(2)
    lines = []
    for u in range(4):
        for h in range(5):
            ws = " ".join(words[int(i)] for i in rng.integers(3, V, rng.integers(1, 8)))
            lines.append(f"utt{u}\t{-rng.random():.4f}\t-1.0\t{ws}")
    (tmp_path / "nbest.txt").write_text("\n".join(lines) + "\n")
    r = subprocess.run([CLI, "rescore", "--nbest", str(tmp_path / "nbest.txt"), "--model",
                        str(tmp_path / "m3.rnlm"), "--lm-scale", "0.5", "--precision", "fp32"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    out = [l.split("\t") for l in r.stdout.splitlines()]
    assert len(out) == 20 and all(len(f) == 7 for f in out)
    for u in range(4):
        rows = [f for f in out if f[0] == f"utt{u}"]
        assert [int(f[6]) for f in rows] == [1, 2, 3, 4, 5]
        totals = [float(f[5]) for f in rows]
        assert totals == sorted(totals, reverse=True)
    # errors map to the reference's exit codes
    r = subprocess.run([CLI, "rnn-ppl", "--model", str(tmp_path / "vocab.txt"), "--ids",
                        str(tmp_path / "valid.ids")], capture_output=True, text=True)
    assert r.returncode == 2  # DataError: unrecognised model header
