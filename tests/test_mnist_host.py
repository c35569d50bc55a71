"""CPU tests for the config-3 data path: synthetic IDX3, the IDX3 loader and
its seeded sampling (instances.cpp:80-144) against the unmodified reference."""
import hashlib

import numpy as np
import pytest

import paper_2203_03732_b200 as otprg
from paper_2203_03732_b200.instances import make_synthetic_mnist, synth_images, write_idx3


@pytest.fixture(scope="module")
def idx3(tmp_path_factory):
    return make_synthetic_mnist(str(tmp_path_factory.mktemp("mnist") / "synth-idx3"), 20000, 0)


def test_synthetic_images_are_deterministic_and_valid():
    a = synth_images(500, 0)
    assert hashlib.sha256(a.tobytes()).hexdigest() == hashlib.sha256(synth_images(500, 0).tobytes()).hexdigest()
    assert (a.reshape(500, -1).sum(1) > 0).all()               # no blank image (instances.cpp:121)
    assert (a.reshape(500, 28, 28)[:, 14, 14] > 0).all()        # common support at the centre (F8)


def test_loader_sample_and_cost_match_reference(idx3, reference):
    for n, seed in ((50, 1), (300, 7)):
        inst = otprg.load_mnist_pair(idx3, n, seed)
        want = reference.load_mnist_pair(idx3, n, seed)
        got = otprg.l1_cost(inst.img_a, inst.img_b)
        assert got.tobytes() == want.tobytes()


def test_l1_cost_bits_match_oracle(idx3, oracle):
    inst = otprg.load_mnist_pair(idx3, 64, 9)
    want = oracle.mnist_cost(np.concatenate([inst.img_a, inst.img_b]))
    assert otprg.l1_cost(inst.img_a, inst.img_b).tobytes() == want.tobytes()


def test_loader_errors(tmp_path):
    bad = tmp_path / "bad"
    bad.write_bytes(b"\x00\x00\x08\x04" + b"\x00" * 12)
    with pytest.raises(otprg.FormatError):
        otprg.load_mnist_pair(str(bad), 1, 0)
    with pytest.raises(otprg.InputError):
        otprg.load_mnist_pair(str(tmp_path / "missing"), 1, 0)
    small = tmp_path / "small"
    write_idx3(str(small), synth_images(3, 0))
    with pytest.raises(otprg.InputError):
        otprg.load_mnist_pair(str(small), 2, 0)  # needs 2n = 4 images
    short = tmp_path / "short"
    short.write_bytes(b"\x00\x00\x08\x03")
    with pytest.raises(otprg.FormatError):
        otprg.load_mnist_pair(str(short), 1, 0)
