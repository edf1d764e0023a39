"""The reference's caller of the path (chunkkv.toy_model): seeded weights and
embeddings on the host (CPU tests), prefill + greedy generate on the GPU against the tokens,
logits and hidden states the reference itself produced on the same scenarios
(tests/golden/toy.npz, made by tests/golden/make_golden.py; test_toy_model.py:1-161 is the
model for these tests)."""

import numpy as np
import pytest

from paper_2503_23294_b200.tiers import Tier
from paper_2503_23294_b200.toy_model import GenerationResult, ToyModel
from tests.conftest import load_golden

TIERS = (Tier.INT2, Tier.INT4, Tier.FP16)


def _spec(g, i):
    vocab, dim, heads, seed, n_prompt, cs, gs, steps = (int(x) for x in g[f"spec{i}"])
    return dict(vocab=vocab, dim=dim, heads=heads, seed=seed, n_prompt=n_prompt, cs=cs, gs=gs, steps=steps)


# ---- host logic (no GPU) ------------------------------------------------------------------

def test_weights_follow_the_reference_draw_order():
    g = load_golden("toy.npz")
    for i in range(int(g["n"])):
        s = _spec(g, i)
        m = ToyModel(vocab_size=s["vocab"], embed_dim=s["dim"], n_heads=s["heads"], seed=s["seed"])
        assert np.array_equal(np.array([m.w_e.sum(), m.w_q.sum(), m.w_o.sum()]), g[f"w_sum{i}"])


def test_same_seed_same_weights_and_bounds():
    a, b = ToyModel(64, 16, 2, seed=42), ToyModel(64, 16, 2, seed=42)
    c = ToyModel(64, 16, 2, seed=43)
    for name in ("w_e", "w_q", "w_k", "w_v", "w_o"):
        assert np.array_equal(getattr(a, name), getattr(b, name))
    assert not np.array_equal(a.w_e, c.w_e)
    m = ToyModel(vocab_size=32, embed_dim=8, n_heads=4, seed=1)
    for w, shape in ((m.w_e, (32, 8)), (m.w_q, (8, 8)), (m.w_o, (8, 32))):
        assert w.shape == shape and np.all(np.abs(w) < 1 / np.sqrt(8))
    assert m.head_dim == 2


def test_model_config_and_embed_checks():
    with pytest.raises(ValueError):
        ToyModel(vocab_size=1)
    with pytest.raises(ValueError):
        ToyModel(embed_dim=10, n_heads=4)
    m = ToyModel(vocab_size=16, embed_dim=8, n_heads=2, seed=4)
    for bad in ([16], [-1], [[1, 2]]):
        with pytest.raises(ValueError):
            m.embed(bad)
    assert m.embed([]).shape == (0, 8)
    p = ToyModel(vocab_size=16, embed_dim=4, n_heads=2, seed=3).positional(5, 1)[0]
    assert p[0] == np.sin(5.0) and p[1] == np.cos(5.0)
    assert p[2] == np.sin(5.0 / 10000.0 ** (2.0 / 4.0)) and p[3] == np.cos(5.0 / 10000.0 ** (2.0 / 4.0))
    emb = m.embed([3, 3])
    assert np.max(np.abs((emb[1] - emb[0]) - (m.positional(1, 1)[0] - m.positional(0, 1)[0]))) < 1e-15
    assert np.array_equal(m.embed([3], start_pos=1)[0], emb[1])


def test_generation_result_fields():
    res = GenerationResult(tokens=[1, 2], final_hidden=np.ones(3), step_seconds=[0.1, 0.2])
    assert res.tokens == [1, 2]


# ---- GPU: prefill + generate against the reference's outputs --------------------------------

def _prompt_caches(model, prompt, tiers, cs, gs):
    from paper_2503_23294_b200 import build_cache, prefill_attention, segment_context

    k, v, logits = prefill_attention(model.embed(prompt), model)
    chunk_set = segment_context(prompt, cs)
    d = model.head_dim
    caches = [build_cache(k[:, h * d:(h + 1) * d], v[:, h * d:(h + 1) * d], tiers, chunk_set, gs)
              for h in range(model.n_heads)]
    return caches, int(np.argmax(logits)), logits


@pytest.mark.gpu
@pytest.mark.parametrize("i", range(5))
def test_generate_matches_reference_tokens(i):
    from paper_2503_23294_b200 import generate, prefill_attention

    g = load_golden("toy.npz")
    s = _spec(g, i)
    model = ToyModel(vocab_size=s["vocab"], embed_dim=s["dim"], n_heads=s["heads"], seed=s["seed"])
    prompt = g[f"prompt{i}"].tolist()
    _, _, logits, hidden = prefill_attention(model.embed(prompt), model, return_hidden=True)
    assert np.max(np.abs(logits - g[f"prefill_logits{i}"])) < 1e-12
    assert np.max(np.abs(hidden[-4:] - g[f"prefill_hidden{i}"])) < 1e-12
    tiers = [TIERS[t] for t in g[f"tiers{i}"]]
    caches, first, _ = _prompt_caches(model, prompt, tiers, s["cs"], s["gs"])
    assert first == int(g[f"first{i}"])
    res = generate(model, caches, first, s["steps"], start_pos=len(prompt))
    assert res.tokens == g[f"tokens{i}"].tolist()
    assert np.max(np.abs(res.final_hidden - g[f"final_hidden{i}"])) < 1e-9
    assert len(res.step_seconds) == s["steps"]
    assert all(c.decode_len == s["steps"] for c in caches)


@pytest.mark.gpu
def test_generate_all_fp16_equals_reference_path():
    from paper_2503_23294_b200 import generate

    model = ToyModel(vocab_size=128, embed_dim=32, n_heads=4, seed=8)
    prompt = list(range(56))
    mixed_caches, first, _ = _prompt_caches(model, prompt, [Tier.FP16] * 7, 8, 8)
    ref_caches, _, _ = _prompt_caches(model, prompt, [Tier.FP16] * 7, 8, 8)
    mixed = generate(model, mixed_caches, first, steps=16, start_pos=56)
    ref = generate(model, ref_caches, first, steps=16, start_pos=56, use_reference=True)
    assert mixed.tokens == ref.tokens
    assert np.max(np.abs(mixed.final_hidden - ref.final_hidden)) < 1e-9


@pytest.mark.gpu
def test_generate_zero_steps_and_validation():
    from paper_2503_23294_b200 import generate, serialize_cache

    model = ToyModel(vocab_size=64, embed_dim=16, n_heads=2, seed=6)
    caches, first, _ = _prompt_caches(model, list(range(20)), [Tier.INT4] * 5, 4, 8)
    before = [serialize_cache(c) for c in caches]
    res = generate(model, caches, first, steps=0, start_pos=20)
    assert res.tokens == [] and res.step_seconds == [] and res.final_hidden is None
    assert [serialize_cache(c) for c in caches] == before
    with pytest.raises(ValueError):
        generate(model, caches, first, steps=-1, start_pos=20)
    with pytest.raises(ValueError):
        generate(model, caches[:1], first, steps=1, start_pos=20)
    assert ToyModel(vocab_size=8, embed_dim=4, n_heads=2, seed=5).next_token(np.zeros(4)) == 0
