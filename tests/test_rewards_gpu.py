"""F2 rewards on the device: the reference's acceptance c06 values
(test_acceptance.py:253-277) through the drop-in functions, and a batched
run (rewards + group RaPR + advantages in one kernel) vs the reference
formulas restated on host."""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import grpo_oracle as O  # noqa: E402
from paper_2509_01055_b200.rl import rewards as R  # noqa: E402


def test_c06_reward_formula_suite():
    assert R.reward_match("4", "4") == 1.0
    assert R.reward_match(" 0,  1001 ", "0, 1001") == 1.0
    assert R.reward_match("5", "4") == -1.0
    assert R.reward_math("42", "42") == 1.0
    assert R.reward_math("41", "42") == -1.25
    assert R.reward_deepsearch("x", "x", tool_called=True) == 1.1
    assert R.reward_deepsearch("x", "x", tool_called=False) == 1.0
    assert R.reward_deepsearch("y", "x", tool_called=True) == -0.9
    assert R.reward_deepsearch("y", "x", tool_called=False) == -1.0
    assert R.reward_visual_reasoner(1.0, True, 0.1, 1) == 1.1
    assert R.reward_visual_reasoner(1.0, True, 0.1, 3) == 1.0
    assert R.reward_visual_reasoner(1.0, False, 0.1, 0) == 1.0
    assert R.reward_visual_reasoner(1.0, True, 0.5, 1) == 1.0
    assert R.reward_visual_reasoner(0.0, True, 0.0, 1) == 0.15
    assert R.reward_swe(True, True) == 1.0
    assert R.reward_swe(True, False) == 0.0
    assert R.reward_swe(False, True) == 0.0
    assert R.reward_swe(False, False) == 0.0


def _ref_visual(r_acc, invoked, rapr, n_vo, h=0.3, n=1, alpha=0.5, beta=0.05):
    # rewards.py:43-63 restated
    curiosity = alpha * max(h - rapr, 0.0) if invoked else 0.0
    return r_acc + curiosity + beta * min(n - n_vo, 0)


def test_batched_visual_reasoner_with_group_rapr():
    rng = np.random.default_rng(2)
    sizes = rng.integers(2, 40, 50)
    go = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int32)
    B = int(go[-1])
    r_acc = rng.choice([0.0, 1.0], B)
    tool = rng.random(B) < 0.25
    n_vo = rng.integers(0, 5, B)
    rew, rapr, adv64, _ = R.group_rewards_advantages(R.VISUAL_REASONER, go, r_acc=r_acc,
                                                     tool_called=tool, n_vo=n_vo)
    rew = rew.cpu().numpy()
    rapr = rapr.cpu().numpy()
    adv = adv64.cpu().numpy()
    for g in range(len(sizes)):
        sl = slice(go[g], go[g + 1])
        ra = R.rapr_of(tool[sl].tolist())
        assert rapr[g] == ra
        exp = [_ref_visual(float(a), bool(t), ra, int(v)) for a, t, v in
               zip(r_acc[sl], tool[sl], n_vo[sl])]
        assert rew[sl].tolist() == exp
        ea = O.group_advantages(exp)
        assert all(abs(x - y) <= 4 * math.ulp(max(abs(y), 1e-300)) or abs(x - y) < 1e-15
                   for x, y in zip(adv[sl].tolist(), ea))


@pytest.mark.parametrize("kind", [R.MATCH, R.MATH, R.DEEPSEARCH, R.SWE])
def test_batched_simple_kinds(kind):
    rng = np.random.default_rng(kind)
    go = np.arange(0, 8 * 20 + 1, 8, dtype=np.int32)
    B = int(go[-1])
    ok = rng.random(B) < 0.5
    tool = rng.random(B) < 0.5
    tests = rng.random(B) < 0.5
    rew, _, _, _ = R.group_rewards_advantages(kind, go, correct=ok, tool_called=tool,
                                              tests_pass=tests)
    got = rew.cpu().numpy().tolist()
    if kind == R.MATCH:
        exp = [1.0 if o else -1.0 for o in ok]
    elif kind == R.MATH:
        exp = [1.0 if o else -1.0 + -0.25 for o in ok]
    elif kind == R.DEEPSEARCH:
        exp = [(1.0 if o else -1.0) + (0.1 if t else 0.0) for o, t in zip(ok, tool)]
    else:
        exp = [1.0 if (o and t) else 0.0 for o, t in zip(ok, tests)]
    assert got == exp
