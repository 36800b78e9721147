"""Pins for oracle/model.py and the zoo: whole-model forward against torchvision
(fp64, CPU -- an independent implementation) and published parameter counts."""
import numpy as np
import pytest
import torch
import torchvision

from oracle import merge, model, ops
from workloads import synth, zoo

TV = {"resnet18": torchvision.models.resnet18, "resnet34": torchvision.models.resnet34,
      "resnet50": torchvision.models.resnet50, "resnet101": torchvision.models.resnet101,
      "resnet152": torchvision.models.resnet152, "vgg11": torchvision.models.vgg11,
      "vgg13": torchvision.models.vgg13, "vgg16": torchvision.models.vgg16,
      "vgg19": torchvision.models.vgg19, "alexnet": torchvision.models.alexnet}

# torchvision parameter counts (weights + biases + BN affine), SURVEY.md Appendix A.
PUBLISHED_PARAMS = {"resnet18": 11_689_512, "resnet34": 21_797_672, "resnet50": 25_557_032,
                    "resnet101": 44_549_160, "resnet152": 60_192_808, "vgg16": 138_357_544,
                    "vgg19": 143_667_240}


def _tv_param_count(layers):
    n = 0
    for l in layers:
        if l["op"] == "bn":
            n += 2 * l["c"]           # affine gamma/beta are parameters, running stats are buffers
        else:
            n += merge.param_count(l)
    return n


@pytest.mark.parametrize("name", sorted(PUBLISHED_PARAMS))
def test_param_counts_published(name):
    assert _tv_param_count(zoo.build(name)) == PUBLISHED_PARAMS[name]


@pytest.mark.parametrize("name", sorted(TV))
def test_param_counts_vs_torchvision(name):
    tv = TV[name](weights=None)
    assert _tv_param_count(zoo.build(name)) == sum(p.numel() for p in tv.parameters())


def _load_into_torchvision(name, layers, params):
    net = TV[name](weights=None).double().eval()
    mods = [m for m in net.modules() if isinstance(m, (torch.nn.Conv2d, torch.nn.BatchNorm2d, torch.nn.Linear))]
    ours = [(l, p) for l, p in zip(layers, params) if l["op"] in merge.PARAM_OPS]
    assert len(mods) == len(ours)
    with torch.no_grad():
        for m, (l, p) in zip(mods, ours):
            if l["op"] == "bn":
                assert isinstance(m, torch.nn.BatchNorm2d) and m.num_features == l["c"]
                m.weight.copy_(torch.from_numpy(p["gamma"].astype(np.float64)))
                m.bias.copy_(torch.from_numpy(p["beta"].astype(np.float64)))
                m.running_mean.copy_(torch.from_numpy(p["mean"].astype(np.float64)))
                m.running_var.copy_(torch.from_numpy(p["var"].astype(np.float64)))
            else:
                assert tuple(m.weight.shape) == p["w"].shape
                m.weight.copy_(torch.from_numpy(p["w"].astype(np.float64)))
                if "b" in p:
                    m.bias.copy_(torch.from_numpy(p["b"].astype(np.float64)))
                else:
                    assert m.bias is None
    return net


@pytest.mark.parametrize("name,res", [("resnet18", 64), ("resnet34", 64), ("resnet50", 64),
                                      ("vgg16", 32), ("alexnet", 96)])
def test_forward_matches_torchvision(name, res):
    layers = zoo.build(name)
    params = synth.params(layers, 99, 1)
    fr = synth.frames(99, 0, 2, res, res)
    ours = model.run(layers, params, fr)[-1]
    net = _load_into_torchvision(name, layers, params)
    with torch.no_grad():
        ref = net(torch.from_numpy(ops.preprocess(fr))).numpy()
    np.testing.assert_allclose(ours, ref, rtol=1e-9, atol=1e-9 * np.abs(ref).max())


def test_shapes_resnet50_224():
    sh = model.shapes(zoo.build("resnet50"), (224, 224))
    assert sh[0] == (64, 112, 112)
    assert sh[3] == (64, 56, 56)
    assert sh[-1] == (1000,)
    assert sh[-3] == (2048, 1, 1)


def test_bf16_emulation_close_to_fp64():
    layers = zoo.build("resnet18")
    params = synth.params(layers, 5, 0)
    fr = synth.frames(5, 0, 1, 64, 64)
    a = model.run(layers, params, fr)[-1]
    b = model.run(layers, params, fr, emulate_bf16=True)[-1]
    rel = np.abs(a - b).max() / np.abs(a).max()
    assert 0 < rel < 0.05


def test_round_bf16_values():
    x = np.array([1.0, 1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, -2.5, 1e-40, 3.0e38])
    r = model.round_bf16(x)
    assert r[0] == 1.0
    assert r[1] == 1.0                      # tie -> even
    assert r[2] == 1.0 + 4 * 2 ** -8        # tie -> even (up)
    assert r[3] == -2.5
    # agrees with torch's bf16 conversion (RNE)
    t = torch.tensor(np.random.default_rng(0).standard_normal(1000), dtype=torch.float32)
    np.testing.assert_array_equal(model.round_bf16(t.numpy().astype(np.float64)),
                                  t.to(torch.bfloat16).to(torch.float64).numpy())


def test_storage_points_resnet_basic_block():
    layers = zoo.build("resnet18")
    st = model.storage_points(layers)
    # stem: conv(0) bn(1) relu(2) maxpool(3): only relu and pool materialised
    assert st[:4] == [False, False, True, True]
    # first basic block: conv bn relu conv bn add relu
    assert st[4:11] == [False, False, True, False, False, False, True]


def test_activations_stay_bounded_deep_resnet():
    """Input recipe check: random-init ResNet-152 keeps O(1)-O(100) activations."""
    layers = zoo.build("resnet152")
    params = synth.params(layers, 3, 0)
    vals = model.run(layers, params, synth.frames(3, 0, 1, 64, 64))
    mx = max(float(np.abs(v).max()) for v in vals)
    assert mx < 1e3
    assert float(np.abs(vals[-1]).std()) > 1e-2
