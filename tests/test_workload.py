"""The synthetic input generator: keyed, order/batch invariant, exact in bf16."""
import numpy as np
import torch

from workload import synth


def test_keyed_order_invariance():
    ids = np.array([5, 17, 3, 1 << 33, 9], np.int64)
    a = synth.logits_np(123, 2, ids, 1, 300, 60000, "fp32")
    perm = np.array([4, 2, 0, 3, 1])
    b = synth.logits_np(123, 2, ids[perm], 1, 300, 60000, "fp32")
    assert np.array_equal(a[perm], b)
    one = synth.logits_np(123, 2, ids[3:4], 1, 300, 60000, "fp32")
    assert np.array_equal(one[0], a[3])


def test_bf16_exact_and_matches_fp32():
    ids = np.arange(64, dtype=np.int64)
    f = synth.logits_np(7, 0, ids, 1, 1000, 50000, "fp32")
    b = synth.logits_np(7, 0, ids, 1, 1000, 50000, "bf16")
    tb = torch.from_numpy(f).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(tb, b)
    assert np.array_equal(synth.bf16_bits_to_f32(b), f)


def test_stage_and_seed_change_values():
    ids = np.arange(16, dtype=np.int64)
    a = synth.logits_np(1, 0, ids, 1, 64, 50000)
    assert not np.array_equal(a, synth.logits_np(1, 1, ids, 1, 64, 50000))
    assert not np.array_equal(a, synth.logits_np(2, 0, ids, 1, 64, 50000))


def test_marginal_accuracy_and_overlap():
    fam = synth.FAMILIES["c1"]
    ids = np.arange(4000, dtype=np.int64)
    lab = synth.labels_np(fam.seed, ids, 1, fam.C)[:, 0]
    accs = []
    for k in range(fam.K):
        x = synth.fam_logits_np(fam, k, ids, "fp32", L=1, C=fam.C)
        accs.append(np.argmax(x, axis=1) == lab)
    for k, a in enumerate(fam.acc):
        assert abs(accs[k].mean() - a) < 0.03
    both = (accs[0] & accs[1]).mean()
    assert both < min(accs[0].mean(), accs[1].mean())       # not strictly subset


def test_token_sequences_one_wrong_token():
    ids = np.arange(50, dtype=np.int64)
    L, C = 8, 128
    x = synth.logits_np(3, 0, ids, L, C, 20000, "fp32").reshape(50, L, C)
    lab = synth.labels_np(3, ids, L, C)
    wrong = (np.argmax(x, axis=2) != lab).sum(axis=1)
    assert wrong.max() <= 1 and wrong.min() == 0


def test_accuracy_threshold_monotone():
    t = [synth.accuracy_threshold(a) for a in (0.0, 0.1, 0.3, 0.5, 0.8, 0.95, 1.0)]
    assert t == sorted(t) and t[0] == 0 and t[-1] == 65536 + 32768


def test_margin_profiles_exact_in_bf16():
    """Winner codes stay within 8 significant bits (|code| <= 255), so the
    values code * 2^-4 are exact in bf16 for every profile in use."""
    for m in {f.margin for f in synth.FAMILIES.values()}:
        rb, rm1, rm2, wb, wm, cs, ccap = m
        assert rb + rm1 + rm2 + (ccap if cs > 0 else 0) <= 255 and wb + wm <= 255
        assert min(rb, wb) >= 0


def test_vit_margin_confidence_grows_with_slack():
    """VIT_MARGIN: a right answer far from the accuracy boundary gets a larger
    winner code than one near it; wrong answers do not depend on slack."""
    ok = np.array([True, True, False, False])
    slack = np.array([0, 40000, 0, 40000], np.int64)
    z = np.zeros(4, np.int64)
    c = synth.winner_code(ok, slack, z, z, synth.VIT_MARGIN)
    assert c[1] - c[0] == min(40000 >> synth.VIT_MARGIN[5], synth.VIT_MARGIN[6])
    assert c[2] == c[3] == synth.VIT_MARGIN[3]
