"""Run-to-run determinism of the fused step (race detection /
deterministic reductions): two identical GRPO steps must agree bitwise in
every output — no order-dependent float atomics anywhere on the path (the
dW accumulation across chunks is a red.add with one writer per element per
launch, so it is ordered by the stream)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2509_01055_b200 import grpo, packing  # noqa: E402
from paper_2509_01055_b200.rl.loss import LossConfig  # noqa: E402
from paper_2509_01055_b200.synthetic import CONFIGS, make_workload  # noqa: E402


MODES = {"store": {}, "recompute": {"recompute": True}, "pipelined": {"pipelined": True}}


def _tiny_step_inputs():
    cfg = CONFIGS["tiny"]
    wl = make_workload(cfg)
    H, V = cfg.hidden, cfg.vocab
    packed = packing.pack_table(wl.table)
    g = torch.Generator(device="cuda").manual_seed(3)
    h = torch.randn((wl.n_tokens, H), device="cuda", generator=g).bfloat16()
    W = (torch.randn((V, H), device="cuda", generator=g) * 0.05).bfloat16()
    lold = torch.from_numpy(wl.logp_old).cuda()
    lref = torch.from_numpy(wl.logp_ref).cuda()
    return wl, H, V, packed, h, W, lold, lref


def _outputs(r):
    return (r.report_tensor.clone(), r.logp.clone(), r.entropy.clone(), r.dhidden.clone(),
            r.dweight.clone())


@pytest.mark.parametrize("chunk", [128, 256])
def test_pipelined_equals_serial_bitwise(chunk):
    """The pipelined schedule (dS pass on a side stream beside the next
    chunk's forward, two chunk buffers) runs the same kernels on the same
    data: every output equals the serial store-logits schedule bitwise."""
    wl, H, V, packed, h, W, lold, lref = _tiny_step_inputs()
    cfg = LossConfig(kl_beta=0.04, entropy_coef=0.01)
    a = _outputs(grpo.GRPOStep(H, V, cfg, chunk_rows=chunk)(
        packed, wl.group_off, wl.rewards, h, W, lold, lref))
    b = _outputs(grpo.GRPOStep(H, V, cfg, chunk_rows=chunk, pipelined=True)(
        packed, wl.group_off, wl.rewards, h, W, lold, lref))
    assert packed.n_act > 2 * chunk  # several chunks, both buffers in use
    for x, y in zip(a, b):
        assert torch.equal(x, y)


@pytest.mark.parametrize("mode", list(MODES))
def test_step_bitwise_deterministic(mode):
    cfg = CONFIGS["tiny"]
    wl = make_workload(cfg)
    H, V = cfg.hidden, cfg.vocab
    packed = packing.pack_table(wl.table)
    g = torch.Generator(device="cuda").manual_seed(3)
    h = torch.randn((wl.n_tokens, H), device="cuda", generator=g).bfloat16()
    W = (torch.randn((V, H), device="cuda", generator=g) * 0.05).bfloat16()
    lold = torch.from_numpy(wl.logp_old).cuda()
    lref = torch.from_numpy(wl.logp_ref).cuda()
    step = grpo.GRPOStep(H, V, LossConfig(kl_beta=0.04, entropy_coef=0.01), chunk_rows=256,
                         **MODES[mode])
    outs = []
    for _ in range(2):
        r = step(packed, wl.group_off, wl.rewards, h, W, lold, lref)
        outs.append((r.report_tensor.clone(), r.logp.clone(), r.entropy.clone(),
                     r.dhidden.clone(), r.dweight.clone()))
    for a, b in zip(*outs):
        assert torch.equal(a, b)


def test_pack_deterministic_under_arrival_order():
    """The same segments laid out in arrival order vs segment order pack
    identically."""
    t = make_workload(CONFIGS["tiny"], arrival_order=True).table
    pool = np.concatenate([t.token_pool[o:o + n] for o, n in zip(t.seg_src_off, t.seg_len)])
    src = np.concatenate([[0], np.cumsum(t.seg_len)[:-1]]).astype(np.int32)
    t2 = packing.SegmentTable(pool.astype(np.int32), src, t.seg_len, t.seg_is_action,
                              t.traj_seg_off)
    a = packing.pack_table(t)
    b = packing.pack_table(t2)
    for k in ("input_ids", "loss_mask", "position_ids", "cu_seqlens", "act_idx"):
        assert torch.equal(getattr(a, k), getattr(b, k)), k
    assert np.array_equal(a.act_off.cpu().numpy(), b.act_off.cpu().numpy())


def test_captured_step_replays_eager_bitwise():
    """GRPOStep.capture records the device side of a step (K2 + fused LM-head
    step + reductions) as one CUDA graph; replay() on the captured buffers
    equals the eager step bitwise, also after the inputs are refilled in
    place."""
    wl, H, V, packed, h, W, lold, lref = _tiny_step_inputs()
    cfg = LossConfig(kl_beta=0.04, entropy_coef=0.01)
    rw = torch.from_numpy(wl.rewards).cuda()
    step = grpo.GRPOStep(H, V, cfg, chunk_rows=256)
    cap = step.capture(packed, wl.group_off, rw, h, W, lold, lref)
    for refill in (False, True):
        if refill:  # new behaviour-policy log-probs and rewards, same shapes
            lold.add_(0.01)
            rw.copy_(rw.flip(0))
        cap.replay()
        got = _outputs(cap.result())
        ref = _outputs(grpo.GRPOStep(H, V, cfg, chunk_rows=256)(
            packed, wl.group_off, rw, h, W, lold, lref))
        for x, y in zip(got, ref):
            assert torch.equal(x, y)
