"""GPU parity for the round-2 K1 / K3 kernels and step options:
  - K1 decoupled look-back scan over many scan tiles, the scatter's global
    fallback window (tiles spanning > 1,024 segments), per-trajectory drop bits
    — bit-exact against oracle/pack_oracle.py;
  - K3 token-parallel units (trajectories longer than one 2,048-token unit,
    runs of tiny trajectories) — rel 1e-5 against the oracle, bitwise
    run-to-run;
  - the fused step with dropped trajectories == the step with those
    trajectories' tokens marked observation (bitwise), frozen-weight (dH only)
    and detached-hidden (dW only) steps == the matching parts of the full step
    (bitwise), a step on a non-default stream == the default-stream step;
  - host-side validation of the tensors handed to the C ABI.
"""

import numpy as np
import pytest

from oracle import grpo_oracle as O
from oracle import pack_oracle as P

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2509_01055_b200 import grpo, packing  # noqa: E402
from paper_2509_01055_b200.errors import MaskMismatch  # noqa: E402
from paper_2509_01055_b200.rl import loss as L  # noqa: E402
from paper_2509_01055_b200.trajectory import Segment, Trajectory  # noqa: E402

KEYS = ("input_ids", "loss_mask", "position_ids", "cu_seqlens", "traj_of_token", "act_off",
        "act_idx")


def _traj(segs):
    return Trajectory([Segment(o, "", list(t)) for o, t in segs])


def _check_pack(got, ref):
    for k in KEYS:
        assert np.array_equal(getattr(got, k).cpu().numpy(), ref[k]), k


def _segments(rng, n_traj, seg_range, len_range, empty_p=0.1, empty_traj_p=0.02, V=152064):
    trajs = []
    for _ in range(n_traj):
        segs = []
        if rng.random() >= empty_traj_p:
            for s in range(int(rng.integers(*seg_range))):
                n = 0 if rng.random() < empty_p else int(rng.integers(*len_range))
                segs.append(("action" if s % 2 == 0 else "observation",
                             rng.integers(0, V, n).tolist()))
        trajs.append(segs)
    return trajs


def test_pack_many_scan_tiles():
    # ~40 k segments = ~80 look-back tiles of 512 segments (look-back windows
    # of 32 tiles: several rounds)
    rng = np.random.default_rng(21)
    trajs = _segments(rng, 3000, (1, 26), (1, 30))
    got = packing.pack([_traj(s) for s in trajs])
    _check_pack(got, P.pack_varlen(trajs))


def test_pack_more_scan_tiles_than_sms():
    # ~110 k segments = more look-back tiles than SMs: tiles are taken in
    # ticket (dispatch) order instead of blockIdx order
    rng = np.random.default_rng(28)
    trajs = _segments(rng, 8500, (1, 26), (1, 4))
    n_seg = sum(len(t) for t in trajs)
    assert n_seg > 148 * 512
    for drop in (None, rng.random(len(trajs)) < 0.1):
        got = packing.pack([_traj(s) for s in trajs], drop=drop)
        _check_pack(got, P.pack_varlen(trajs, drop=drop))


def test_pack_wide_segment_window_fallback():
    # 1-token / empty segments: a 4,096-position scatter tile spans > 1,024
    # segments and > 512 trajectories (global-memory fallback path)
    rng = np.random.default_rng(22)
    trajs = _segments(rng, 4000, (1, 6), (1, 2), empty_p=0.3)
    got = packing.pack([_traj(s) for s in trajs])
    _check_pack(got, P.pack_varlen(trajs))


@pytest.mark.parametrize("lead", [0, 1, 17])
def test_pack_runs_of_empty_trajectories(lead):
    """Hundreds of empty trajectories between (and after) short ones: a
    16-segment tile in which > 256 trajectories start (the single-pass
    packer's unstaged path), empty ones at tile starts, trailing empties."""
    rng = np.random.default_rng(24 + lead)
    trajs = [[("action", [1, 2, 3])] for _ in range(lead)]
    for blk in range(6):
        trajs += [[] for _ in range(300 + 7 * blk)]
        trajs += _segments(rng, 40, (1, 5), (1, 12), empty_p=0.2, empty_traj_p=0.3)
    trajs += [[] for _ in range(333)]
    for drop in (None, rng.random(len(trajs)) < 0.3):
        got = packing.pack([_traj(s) for s in trajs], drop=drop)
        _check_pack(got, P.pack_varlen(trajs, drop=drop))


def test_pack_long_trajectories_across_tiles():
    """Trajectories of hundreds of segments (each spans many 16-segment
    tiles: position ids restart only at trajectory starts)."""
    rng = np.random.default_rng(29)
    trajs = _segments(rng, 12, (150, 400), (0, 40), empty_p=0.15, empty_traj_p=0.0)
    drop = rng.random(len(trajs)) < 0.25
    for d in (None, drop):
        got = packing.pack([_traj(s) for s in trajs], drop=d)
        _check_pack(got, P.pack_varlen(trajs, drop=d))


@pytest.mark.parametrize("shape", ["many_tiles", "c2_like"])
def test_pack_drop(shape):
    rng = np.random.default_rng(23)
    if shape == "many_tiles":
        trajs = _segments(rng, 3000, (1, 26), (1, 30))
    else:
        trajs = _segments(rng, 64, (1, 10), (1, 900), empty_p=0.0, empty_traj_p=0.0)
    drop = rng.random(len(trajs)) < 0.2
    got = packing.pack([_traj(s) for s in trajs], drop=drop)
    assert got.n_act == int(got.act_off[-1])
    _check_pack(got, P.pack_varlen(trajs, drop=drop))


def _long_short_batch(seed):
    """Groups mixing trajectories longer than several 2,048-token loss units
    with runs of 1-5-token trajectories."""
    rng = np.random.default_rng(seed)
    trajs, rewards = [], []
    n_groups, G = 12, 6
    for g in range(n_groups):
        for i in range(G):
            if (g + i) % 3 == 0:
                segs = [("action", rng.integers(0, 1000, int(rng.integers(1, 6))).tolist())]
            else:
                segs = []
                for s in range(int(rng.integers(1, 6)) * 2 - 1):
                    n = int(rng.integers(1, 6000))
                    segs.append(("action" if s % 2 == 0 else "observation",
                                 rng.integers(0, 1000, n).tolist()))
            trajs.append(segs)
        rewards += rng.choice([1.0, -1.0, 0.5, 0.0], G).tolist()
    T = sum(len(O.flatten(s)) for s in trajs)
    lold = -rng.exponential(1.0, T)
    lnew = lold + rng.normal(0, 0.15, T)
    lref = lold + rng.normal(0, 0.05, T)
    go = np.arange(0, n_groups * G + 1, G, dtype=np.int32)
    return trajs, np.asarray(rewards), go, lnew, lold, lref


def _oracle_report(trajs, rewards, go, lnew, lold, lref, beta, drop=None):
    groups, pos = [], 0
    for g in range(len(go) - 1):
        recs_g = []
        for b in range(go[g], go[g + 1]):
            segs = trajs[b]
            if drop is not None and drop[b]:
                segs = [("observation", t) for _, t in segs]
            n = len(O.flatten(segs))
            sl = slice(pos, pos + n)
            recs_g.append(O.token_records(segs, lnew[sl].tolist(), lold[sl].tolist(),
                                          lref[sl].tolist()))
            pos += n
        groups.append((recs_g, rewards[go[g]:go[g + 1]].tolist()))
    return O.loss_report(groups, 0.2, beta), groups


@pytest.mark.parametrize("with_drop", [False, True])
def test_loss_units_long_and_tiny_trajectories(with_drop):
    trajs, rewards, go, lnew, lold, lref = _long_short_batch(31)
    drop = (np.random.default_rng(5).random(len(trajs)) < 0.25) if with_drop else None
    packed = packing.pack([_traj(s) for s in trajs], drop=drop)
    f = lambda a: torch.from_numpy(a.astype(np.float32)).cuda()  # noqa: E731
    cfg = L.LossConfig(kl_beta=0.1)
    rep, grad = grpo.grpo_loss(packed, go, rewards, f(lnew), f(lold), f(lref), cfg)
    rep2, grad2 = grpo.grpo_loss(packed, go, rewards, f(lnew), f(lold), f(lref), cfg)
    assert rep == rep2 and torch.equal(grad, grad2)  # bitwise run-to-run
    c = lambda a: a.astype(np.float32).astype(np.float64)  # noqa: E731
    ref, groups = _oracle_report(trajs, rewards, go, c(lnew), c(lold), c(lref), 0.1, drop)
    assert rep["masked_tokens"] == ref["masked_tokens"]
    assert rep["total_tokens"] == packed.n_tokens
    assert abs(rep["objective"] - ref["objective"]) <= 1e-5 * max(1.0, abs(ref["objective"]))
    assert abs(rep["kl"] - ref["kl"]) <= 1e-5 * max(1e-3, abs(ref["kl"]))
    g = grad.cpu().numpy()
    exp = np.zeros_like(g)
    pos = 0
    for recs_g, rw in groups:
        for row in O.clipped_grad(recs_g, O.group_advantages(rw), 0.2, 0.1):
            exp[pos:pos + len(row)] = np.asarray(row) / (len(go) - 1)
            pos += len(row)
    assert np.abs(g - exp).max() <= 1e-5 * max(np.abs(exp).max(), 1e-4)


def _step_inputs(seed, H=256, V=1000):
    trajs, rewards, go, _, lold, lref = _long_short_batch(seed)
    for tr in trajs:
        for i, (o, toks) in enumerate(tr):
            tr[i] = (o, [t % V for t in toks])
    gen = torch.Generator(device="cuda").manual_seed(seed)
    T = sum(len(O.flatten(s)) for s in trajs)
    h = torch.randn(T, H, device="cuda", generator=gen).bfloat16()
    W = (torch.randn(V, H, device="cuda", generator=gen) * 0.05).bfloat16()
    f = lambda a: torch.from_numpy(a.astype(np.float32)).cuda()  # noqa: E731
    return trajs, rewards, go, h, W, f(lold), f(lref)


def test_step_drop_equals_observation_marked():
    trajs, rewards, go, h, W, lold, lref = _step_inputs(41)
    drop = np.random.default_rng(6).random(len(trajs)) < 0.3
    cfg = L.LossConfig(kl_beta=0.05, entropy_coef=0.01)
    step = grpo.GRPOStep(h.shape[1], W.shape[0], cfg, chunk_rows=4096)
    a = step(packing.pack([_traj(s) for s in trajs], drop=drop), go, rewards, h, W, lold, lref)
    a_dh, a_dw, a_lp = a.dhidden.clone(), a.dweight.clone(), a.logp.clone()
    marked = [[("observation", t) for _, t in s] if d else s for s, d in zip(trajs, drop)]
    b = step(packing.pack([_traj(s) for s in marked]), go, rewards, h, W, lold, lref)
    assert a.report == b.report
    assert torch.equal(a_lp, b.logp) and torch.equal(a_dh, b.dhidden) and torch.equal(a_dw, b.dweight)
    # dropped trajectories: no gradient rows, still counted in their groups
    packed = packing.pack([_traj(s) for s in trajs], drop=drop)
    cu = packed.cu_seqlens.cpu().numpy()
    for bi in np.nonzero(drop)[0]:
        assert not a_dh[cu[bi]:cu[bi + 1]].any()
    assert a.report["episodes"] == len(trajs)


@pytest.mark.parametrize("mode", ["store", "recompute"])
def test_frozen_weight_and_detached_hidden_steps(mode):
    trajs, rewards, go, h, W, lold, lref = _step_inputs(42)
    packed = packing.pack([_traj(s) for s in trajs])
    cfg = L.LossConfig(kl_beta=0.05, entropy_coef=0.01)
    step = grpo.GRPOStep(h.shape[1], W.shape[0], cfg, chunk_rows=2048,
                         recompute=(mode == "recompute"))
    full = step(packed, go, rewards, h, W, lold, lref)
    dh, dw, rep = full.dhidden.clone(), full.dweight.clone(), full.report
    only_h = step(packed, go, rewards, h, W, lold, lref, want_dweight=False)
    assert only_h.dweight is None and torch.equal(only_h.dhidden, dh) and only_h.report == rep
    only_w = step(packed, go, rewards, h, W, lold, lref, want_dhidden=False)
    assert only_w.dhidden is None and torch.equal(only_w.dweight, dw) and only_w.report == rep


def test_step_on_side_stream_matches_default_stream():
    trajs, rewards, go, h, W, lold, lref = _step_inputs(43)
    packed = packing.pack([_traj(s) for s in trajs])
    step = grpo.GRPOStep(h.shape[1], W.shape[0], L.LossConfig(kl_beta=0.05), chunk_rows=2048)
    ref = step(packed, go, rewards, h, W, lold, lref)
    dh, dw = ref.dhidden.clone(), ref.dweight.clone()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    res = step(packed, go, rewards, h, W, lold, lref, stream=side)
    torch.cuda.current_stream().wait_stream(side)
    assert res.report == ref.report
    assert torch.equal(res.dhidden, dh) and torch.equal(res.dweight, dw)
    rep, _ = grpo.grpo_loss(packed, go, rewards, res.logp, lold, lref, L.LossConfig(kl_beta=0.05),
                            stream=side)
    assert rep["masked_tokens"] == ref.report["masked_tokens"]


def test_host_validation_before_launch():
    trajs, rewards, go, h, W, lold, lref = _step_inputs(44)
    packed = packing.pack([_traj(s) for s in trajs])
    step = grpo.GRPOStep(h.shape[1], W.shape[0], L.LossConfig())
    with pytest.raises(TypeError):
        step(packed, go, rewards, h, W, lold.double(), None)
    with pytest.raises(MaskMismatch):
        step(packed, go, rewards[:-1], h, W, lold, None)
    with pytest.raises(MaskMismatch):
        step(packed, go[:-1], rewards[:go[-2]], h, W, lold, None)
    with pytest.raises(ValueError):
        step(packed, go, rewards, h, W, torch.zeros(len(lold), 2, device="cuda")[:, 0], None)
    with pytest.raises(MaskMismatch):
        grpo.grpo_loss(packed, go, rewards, lold[:-1], lold[:-1])
    with pytest.raises(TypeError):
        grpo.lmhead_logprobs(h, W, packed.input_ids.long())
