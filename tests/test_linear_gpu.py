"""Learned router on the tensor cores (ag_route_linear, SURVEY.md §8(f)
rank 3).  Not in the reference: parity is against the fp64 restatement in
oracle/ (linear_logits).  With integer-valued bf16 inputs every product and
partial sum is exact in fp32, so the verdicts must match bit for bit; with
random inputs verdicts must match wherever |logit| >= 1e-3 * ||emb|| ||head||
(fp32 accumulation order differs from the oracle's)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2511_20975_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402


def _members(bm_row, count, begin):
    bits = np.unpackbits(bm_row.view(np.uint8), bitorder="little")
    return (np.nonzero(bits)[0][:count] + begin).astype(np.uint32)


def _run(dev, emb, heads, bias, begin, end, force_top=False):
    res = dev.route_linear(emb, heads, bias, begin, end, force_top=force_top, bitmap=True)
    torch.cuda.synchronize()
    return (res.counts.cpu().numpy(), res.offsets.cpu().numpy(),
            res.indices.cpu().numpy().view(np.uint32), res.bitmap.cpu().numpy().view(np.uint32))


def _want_bits(logit, begin, end, top=None):
    v = logit[:, begin:end] > 0
    if top is not None and begin <= top < end:
        v[:, top - begin] = True
    return v


def _check(counts, offs, idx, bm, want, begin, end):
    R = want.shape[0]
    W = (end - begin + 31) // 32
    for r in range(R):
        bits = np.zeros(W * 32, bool)
        bits[: end - begin] = want[r]
        words = np.packbits(bits, bitorder="little").view(np.uint32)
        assert np.array_equal(bm[r, :W], words), r
        assert counts[r] == want[r].sum(), r
        assert np.array_equal(idx[offs[r]:offs[r + 1]], _members(words, counts[r], begin)), r


@pytest.mark.parametrize("n,m,R,D,begin,end", [(5, 4, 300, 128, 0, None), (5, 6, 257, 64, 0, None),
                                               (4, 6, 40, 128, 77, 1000), (3, 5, 513, 32, 5, 120),
                                               # D not a multiple of the 64-element TMA box: zero fill
                                               (4, 5, 129, 16, 0, None), (4, 5, 200, 48, 1, 600),
                                               (5, 5, 260, 80, 0, None), (4, 7, 70, 112, 100, 2401)])
def test_integer_inputs_bit_exact(n, m, R, D, begin, end):
    sp = P.ConfigSpace.chain(n, m)
    end = sp.size if end is None else end
    dev = P.Device(sp)
    g = torch.Generator().manual_seed(R * 7 + D)
    emb = torch.randint(-3, 4, (R, D), generator=g).to(torch.bfloat16)
    heads = torch.randint(-2, 3, (sp.size, D), generator=g).to(torch.bfloat16)
    bias = (torch.randint(-6, 7, (sp.size,), generator=g).float() + 0.5)  # no exact zeros
    counts, offs, idx, bm = _run(dev, emb.cuda(), heads.cuda(), bias.cuda(), begin, end)
    logit = O.linear_logits(emb.float().numpy(), heads.float().numpy(), bias.numpy())
    _check(counts, offs, idx, bm, _want_bits(logit, begin, end), begin, end)


def test_random_inputs_within_tolerance_and_force_top():
    sp = P.ConfigSpace.chain(5, 8)
    dev = P.Device(sp)
    g = torch.Generator().manual_seed(5)
    R, D = 700, 128
    emb = torch.randn(R, D, generator=g).to(torch.bfloat16)
    heads = (torch.randn(sp.size, D, generator=g) / D ** 0.5).to(torch.bfloat16)
    bias = torch.randn(sp.size, generator=g) * 0.1
    counts, offs, idx, bm = _run(dev, emb.cuda(), heads.cuda(), bias.cuda(), 0, sp.size, force_top=True)
    logit = O.linear_logits(emb.float().numpy(), heads.float().numpy(), bias.numpy())
    scale = np.linalg.norm(emb.float().numpy(), axis=1)[:, None] * \
        np.linalg.norm(heads.float().numpy(), axis=1)[None, :]
    bits = np.unpackbits(bm.view(np.uint8), axis=1, bitorder="little")[:, : sp.size].astype(bool)
    want = logit > 0
    want[:, sp.size - 1] = True
    clear = np.abs(logit) >= 1e-3 * scale
    assert np.array_equal(bits[clear], want[clear])
    assert bits[:, sp.size - 1].all()
    for r in range(R):  # compaction consistent with the bitmap
        assert np.array_equal(idx[offs[r]:offs[r + 1]], np.nonzero(bits[r])[0].astype(np.uint32))


def test_validation():
    sp = P.ConfigSpace.chain(3, 3)
    dev = P.Device(sp)
    emb = torch.zeros(4, 24, dtype=torch.bfloat16, device="cuda")
    heads = torch.zeros(sp.size, 24, dtype=torch.bfloat16, device="cuda")
    bias = torch.zeros(sp.size, dtype=torch.float32, device="cuda")
    with pytest.raises(P.ValidationError):
        dev.route_linear(emb, heads, bias)  # dim not a multiple of 16
    emb = torch.zeros(4, 32, dtype=torch.bfloat16, device="cuda")
    heads = torch.zeros(sp.size * 32 + 1, dtype=torch.bfloat16, device="cuda")[1:].view(sp.size, 32)
    with pytest.raises(P.ValidationError):
        dev.route_linear(emb, heads, bias)  # misaligned heads
