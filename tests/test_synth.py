"""Synthetic-input recipes: host twin properties on CPU, device
kernel == host twin bit-for-bit on the GPU."""
import numpy as np
import pytest

from conftest import u32


def test_recipes_host(pb):
    from paper_2505_18563_b200 import synth

    n = 100_000
    t = synth.synth_host(n, 1, synth.W_TIES, 0.25)
    assert np.all(np.abs(t) <= 0.25)
    assert len(np.unique(np.abs(t))) < n  # ties exist
    d = synth.synth_host(n, 2, synth.G_DYADIC)
    assert np.all(np.abs(d) <= 1.0)
    assert np.all((d * 2**20) == np.round(d * 2**20))  # dyadic grid
    f = synth.synth_host(n, 3, synth.G_FULL)
    assert np.all((f >= -1) & (f < 1))
    r = synth.synth_host(n, 4, synth.W_REAL, 2.0)
    assert np.all(np.abs(r) <= 2.0)
    assert np.array_equal(u32(synth.synth_host(50, 9, 1, 1.0, 10)), u32(synth.synth_host(60, 9, 1)[10:]))


def test_model_shapes(pb):
    from paper_2505_18563_b200 import synth

    want = {"resnet18": 11_689_512, "resnet50": 25_557_032, "vgg19": 143_667_240,
            "bert-base": 109_482_240, "gpt2-medium": 354_823_168}
    for name, total in want.items():
        assert synth.model_shape(name).total == total


def test_derive_seed_matches_oracle(pb, port):
    from paper_2505_18563_b200 import synth

    for a, b, c in [(0, 0, 0), (1, 2, 3), (7, 100, 0)]:
        assert synth.derive_seed(0x5041435452414E21, a, b, c) == port.derive_seed(0x5041435452414E21, a, b, c)


@pytest.mark.gpu
def test_device_synth_equals_host(pb, cuda):
    import torch

    from paper_2505_18563_b200 import synth

    for recipe in range(4):
        n = 1_000_003
        x = torch.empty(n, dtype=torch.float32, device=cuda)
        pb.synth_fill(x, 0x1234 + recipe, recipe, 0.5, 17)
        h = synth.synth_host(n, 0x1234 + recipe, recipe, 0.5, 17)
        assert np.array_equal(u32(x.cpu().numpy()), u32(h)), recipe
    shape = synth.model_shape("resnet18")
    wd = synth.weights_device(shape, 5)
    wh = synth.weights_host(shape, 5)
    assert np.array_equal(u32(wd.cpu().numpy()), u32(wh))
