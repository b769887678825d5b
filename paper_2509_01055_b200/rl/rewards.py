"""Drop-in for toolloop/rl/rewards.py (F2): the reward formulas run in the
group-advantage kernel (tl_group_rewards_advantages), so a batch's rewards,
group RaPR and advantages come out of one launch.

String matching (`normalized_match`, rewards.py:15-18) is host work and stays
here; the numeric formulas (rewards.py:21-68) are evaluated on the device.
The scalar functions keep the reference signatures and route through the
same kernel (one trajectory).
"""

from __future__ import annotations

from typing import Callable, Sequence

import numpy as np

from .. import _lib

Matcher = Callable[[str, str], bool]

MATCH, MATH, DEEPSEARCH, VISUAL_REASONER, SWE = range(5)


def normalized_match(answer: str, gold: str) -> bool:
    """Exact match after collapsing runs of whitespace and trimming."""
    return " ".join(answer.split()) == " ".join(gold.split())


def group_rewards_advantages(kind: int, group_off, *, correct=None, tool_called=None,
                             n_vo=None, r_acc=None, tests_pass=None, rapr=None,
                             std_floor: float = 1e-6, h: float = 0.3, n: int = 1,
                             alpha: float = 0.5, beta: float = 0.05, stream=None):
    """Rewards for every trajectory of a batch (groups contiguous) and their
    group advantages in one kernel.  Returns (rewards f64, rapr f64 [groups],
    adv64, adv32) device tensors."""
    import torch

    L = _lib.lib()
    go = np.asarray(group_off, dtype=np.int32)
    B = int(go[-1])
    n_groups = len(go) - 1
    dev = torch.device("cuda")

    def d(a, dt):
        if a is None:
            return None
        return torch.as_tensor(np.asarray(a, dtype=dt)).to(dev)

    c, t, v = d(correct, np.uint8), d(tool_called, np.uint8), d(n_vo, np.int32)
    ra, tp, ri = d(r_acc, np.float64), d(tests_pass, np.uint8), d(rapr, np.float64)
    d_go = torch.from_numpy(go).to(dev)
    rew = torch.empty(max(B, 1), dtype=torch.float64, device=dev)
    rapr_out = torch.empty(max(n_groups, 1), dtype=torch.float64, device=dev)
    adv64 = torch.empty(max(B, 1), dtype=torch.float64, device=dev)
    adv32 = torch.empty(max(B, 1), dtype=torch.float32, device=dev)
    p = _lib.RewardParamsC(kind=kind, n=n, h=h, alpha=alpha, beta=beta)
    _lib.check(L.tl_group_rewards_advantages(
        p, _lib.ptr(c), _lib.ptr(t), _lib.ptr(v), _lib.ptr(ra), _lib.ptr(tp), d_go.data_ptr(),
        n_groups, B, std_floor, _lib.ptr(ri), rew.data_ptr(), rapr_out.data_ptr(),
        adv64.data_ptr(), adv32.data_ptr(), _lib.stream_handle(stream)))
    return rew[:B], rapr_out[:n_groups], adv64[:B], adv32[:B]


def _one(kind, **kw) -> float:
    rew, _, _, _ = group_rewards_advantages(kind, [0, 1], **kw)
    return float(rew.item())


def reward_match(answer: str, gold: str, matcher: Matcher = normalized_match) -> float:
    """+1 when the matcher accepts the answer, -1 otherwise (rewards.py:21-23)."""
    return _one(MATCH, correct=[matcher(answer, gold)])


def reward_math(answer: str, gold: str, matcher: Matcher = normalized_match) -> float:
    """+1 on match, -1 - 0.25 on mismatch (rewards.py:26-33)."""
    return _one(MATH, correct=[matcher(answer, gold)])


def reward_deepsearch(answer: str, gold: str, tool_called: bool,
                      matcher: Matcher = normalized_match) -> float:
    """+-1 accuracy plus 0.1 when a tool was called (rewards.py:36-41)."""
    return _one(DEEPSEARCH, correct=[matcher(answer, gold)], tool_called=[tool_called])


def reward_visual_reasoner(r_acc: float, invoked_tool: bool, rapr: float, n_vo: int, *,
                           h: float = 0.3, n: int = 1, alpha: float = 0.5,
                           beta: float = 0.05) -> float:
    """Accuracy + curiosity alpha*max(h - rapr, 0) (tool users only) + over-use
    penalty beta*min(n - n_vo, 0) (rewards.py:43-63)."""
    return _one(VISUAL_REASONER, r_acc=[r_acc], tool_called=[invoked_tool], n_vo=[n_vo],
                rapr=[rapr], h=h, n=n, alpha=alpha, beta=beta)


def reward_swe(terminated_ok: bool, all_tests_pass: bool) -> float:
    """1 only for a clean termination with every test passing (rewards.py:66-68)."""
    return _one(SWE, correct=[terminated_ok], tests_pass=[all_tests_pass])


def rapr_of(tool_called: Sequence[bool]) -> float:
    """Reference-side RaPR definition (fraction of the group invoking tools)."""
    return sum(1 for t in tool_called if t) / len(tool_called)
