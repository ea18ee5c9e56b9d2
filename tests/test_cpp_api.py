"""The C++ host API (include/desklm_b200/gpu.hpp) drives the same device
trainer as the Python mirror: a C++ program (tests/cpp/train_example.cpp)
trains through desklm::b200::Trainer and writes an RTRN checkpoint that must
be byte-identical to the Python Trainer's, with epoch logs matching the
oracle (fp32 mode)."""
import os
import subprocess

import numpy as np
import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tests", "cpp", "build", "train_example")


def test_cpp_example_builds():
    r = subprocess.run(["make", "-C", os.path.join(ROOT, "tests", "cpp")], capture_output=True,
                       text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert os.path.exists(EXE)


@pytest.mark.gpu
def test_cpp_trainer_matches_python_and_oracle(tmp_path, orc):
    import paper_1502_00512_b200 as dl
    subprocess.run(["make", "-C", os.path.join(ROOT, "tests", "cpp")], check=True,
                   capture_output=True)
    V, H, noffset, B, T, epochs, eta = 60, 16, 3, 4, 5, 2, 0.05
    tr, va = orc.random_stream_pair(91, V, 1600, 300)
    tr = tr[:1600]
    params = orc.init_uniform(V, H, 5)
    np.concatenate([p.ravel() for p in params]).astype(np.float32).tofile(tmp_path / "params.f32")
    tr.astype(np.uint32).tofile(tmp_path / "train.u32")
    va.astype(np.uint32).tofile(tmp_path / "valid.u32")
    r = subprocess.run([EXE, str(tmp_path), str(V), str(H), str(noffset), str(B), str(T),
                        str(epochs), str(eta), "fp32"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    blob = (tmp_path / "ckpt.rtrn").read_bytes()
    assert (tmp_path / "ckpt2.rtrn").read_bytes() == blob  # load_checkpoint round trip
    kw = dict(nstate=H, noffset=noffset, minibatch=B, unroll=T, eta=eta, max_epochs=epochs,
              mode=1)
    t = dl.Trainer(dl.TrainConfig(**kw), params, dl.make_vocab(V), tr, va, "fp32")
    t.train()
    assert blob == t.save_checkpoint()
    lines = (tmp_path / "logs.csv").read_text().split()
    want = orc.train(oracle.TrainConfig(**kw), params, tr, va)
    assert float(lines[0]) == pytest.approx(want["initial_ppl"], rel=1e-5)
    for line, w in zip(lines[1:1 + epochs], want["logs"]):
        ep, loss, ppl, eta_l, skipped = line.split(",")
        assert int(ep) == int(w[0]) and float(eta_l) == w[3] and int(skipped) == 0
        assert float(ppl) == pytest.approx(w[2], rel=1e-2)
    # free functions: one window + rmsprop + sharded perplexity
    loss, pos, ok, ppl, pred = lines[1 + epochs].split(",")
    x = tr[: T * B].reshape(T, B)
    y = tr[1: T * B + 1].reshape(T, B)
    w = (y != 1).astype(np.uint8)
    g = orc.bptt(params, 0, x, y, w, np.full((B, H), 0.5, np.float32), 1.0 / (T * B), 1.0)
    assert float(loss) == pytest.approx(g["loss"], rel=1e-4)
    assert int(pos) == g["positions"] and int(ok) == 1


@pytest.mark.gpu
def test_cpp_bottleneck_matches_python(tmp_path, orc):
    """The C++ BottleneckModel API (bptt_run / bottleneck_update /
    sharded_perplexity overloads) gives the Python API's numbers."""
    import paper_1502_00512_b200 as dl
    from paper_1502_00512_b200 import bottleneck as bn
    subprocess.run(["make", "-C", os.path.join(ROOT, "tests", "cpp")], check=True,
                   capture_output=True)
    V, H, P, T, B, windows, eta = 80, 16, 8, 5, 4, 3, 0.01
    params = orc.bn_init_uniform(V, H, P, 7)
    ids = orc.random_stream(3, V, (windows + 1) * T * B + 1)[: (windows + 1) * T * B + 1]
    np.concatenate([p.ravel() for p in params]).astype(np.float32).tofile(tmp_path / "params.f32")
    ids.astype(np.uint32).tofile(tmp_path / "ids.u32")
    exe = os.path.join(ROOT, "tests", "cpp", "build", "bn_example")
    r = subprocess.run([exe, str(tmp_path), str(V), str(H), str(P), str(T), str(B), str(windows),
                        str(eta)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.split()
    m = bn.GpuBottleneck(V, H, P, 0, "fp32")
    m.set_params(*params)
    h = np.full((B, H), 0.5, np.float32)
    for w in range(windows):
        x = ids[w * T * B:(w + 1) * T * B].reshape(T, B)
        y = ids[w * T * B + 1:(w + 1) * T * B + 1].reshape(T, B)
        res, h, ok = bn.bn_train_window(m, dl.WindowBatch(x, y, (y != 1).astype(np.uint8)), h,
                                        1.0 / (T * B), 1.0, eta)
        loss, pos, ok_c = lines[w].split(",")
        assert float(loss) == res.loss and int(pos) == res.positions and bool(int(ok_c)) == ok
    ppl, pred = lines[windows].split(",")
    want = bn.bn_sharded_perplexity(m, ids, 8)
    assert float(ppl) == want.perplexity and int(pred) == want.predicted
