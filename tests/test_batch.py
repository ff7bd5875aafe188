"""Image batches (independent images run as replicas, no
exchange): dwt2d_forward_mallat_batch equals one forward_mallat per image,
bit for bit, on one device, dealt over a device list (virtual devices: the
one GPU listed twice), on a caller stream, inside a CUDA graph, and for
symmetric extension (whose border crops share the library's side stream)."""
import numpy as np
import pytest

from oracle import dwt_oracle as O

pytestmark = pytest.mark.gpu


def _images(cuda, n, W, H, seed=5):
    import torch
    return [torch.from_numpy(O.random_image(W, H, seed + i)).to(cuda) for i in range(n)]


@pytest.mark.parametrize("w,s,opt,ext", [("cdf97", "nonseparable-lifting", True, "periodic"),
                                         ("cdf53", "separable-lifting", False, "periodic"),
                                         ("cdf97", "nonseparable-lifting", True, "symmetric")])
@pytest.mark.parametrize("devices", [None, [0, 0]])
def test_batch_equals_per_image_pyramids(cuda, w, s, opt, ext, devices):
    import torch
    import paper_1704_08657_b200 as dwt
    plan = dwt.Plan(w, s, optimized=opt, extension=ext)
    imgs = _images(cuda, 7, 512, 384)
    ref = [plan.forward_mallat(im, 5) for im in imgs]
    outs = plan.forward_mallat_batch(imgs, 5, devices=devices)
    torch.cuda.synchronize()
    for a, b in zip(outs, ref):
        assert torch.equal(a, b)


def test_batch_on_a_stream_and_in_a_graph(cuda):
    import torch
    import paper_1704_08657_b200 as dwt
    plan = dwt.Plan("cdf97", "nonseparable-lifting", optimized=True)
    imgs = _images(cuda, 5, 1024, 1024, 9)
    ref = [plan.forward_mallat(im, 8) for im in imgs]
    outs = [torch.zeros_like(im) for im in imgs]
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        plan.forward_mallat_batch(imgs, 8, outs=outs, streams=[st])  # warm-up: workspaces in the pool
    st.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        plan.forward_mallat_batch(imgs, 8, outs=outs, streams=[st])
    for _ in range(3):
        for o in outs:
            o.zero_()
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        assert all(torch.equal(a, b) for a, b in zip(outs, ref))


def test_batch_argument_errors(cuda):
    import torch
    import paper_1704_08657_b200 as dwt
    plan = dwt.Plan("cdf97", "nonseparable-lifting", optimized=True)
    imgs = _images(cuda, 2, 64, 64)
    with pytest.raises(ValueError):
        plan.forward_mallat_batch([imgs[0], torch.zeros((32, 64), device=cuda)], 2)
    with pytest.raises(ValueError):
        plan.forward_mallat_batch(imgs, 2, devices=[1])  # images live on cuda:0
    with pytest.raises(ValueError):
        plan.forward_mallat_batch(imgs, 7)  # 64 is not divisible by 2^7
    assert plan.forward_mallat_batch([], 2) == []
    inv = dwt.Plan("cdf97", "inverse-lifting")
    with pytest.raises(ValueError):
        inv.forward_mallat_batch(imgs, 2)
