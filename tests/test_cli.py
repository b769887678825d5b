"""`loss` command (drop-in for toolloop/cli.py:272-345): host-side ingest
checks on CPU; the report vs the reference-generated golden run on GPU."""

import json

import pytest

from conftest import cuda_available
from paper_2509_01055_b200 import cli
from paper_2509_01055_b200.errors import EpisodeLogError, MaskMismatch
from oracle import episodes_oracle as EO  # noqa: E402  (checker)


def _write(tmp_path, golden_cli):
    ep = tmp_path / "ep.jsonl"
    ep.write_text(golden_cli["episodes_jsonl"], encoding="utf-8")
    sc = tmp_path / "sc.jsonl"
    sc.write_text("".join(json.dumps(r) + "\n" for r in golden_cli["sidecar"]), encoding="utf-8")
    cfg = tmp_path / "cfg.yaml"
    c = golden_cli["config"]
    cfg.write_text(f"loss:\n  epsilon_clip: {c['epsilon_clip']}\n  kl_beta: {c['kl_beta']}\n",
                   encoding="utf-8")
    return ep, sc, cfg


def test_read_episodes_and_flat_logps(tmp_path, golden_cli):
    ep, _, _ = _write(tmp_path, golden_cli)
    recs = EO.read_episodes(ep)
    assert len(recs) == golden_cli["report_embedded"]["episodes"]
    flat = EO.flat_logps(recs[0])
    assert len(flat) == sum(len(s.tokens) for s in recs[0]["trajectory"].segments)
    recs[0]["action_logprobs"][0] = recs[0]["action_logprobs"][0][:-1]
    with pytest.raises(MaskMismatch):
        EO.flat_logps(recs[0])


def test_corrupted_log_cites_line(tmp_path, golden_cli):
    ep, _, _ = _write(tmp_path, golden_cli)
    n = len([l for l in golden_cli["episodes_jsonl"].splitlines() if l.strip()])
    with ep.open("a", encoding="utf-8") as fh:
        fh.write("{broken\n")
    with pytest.raises(EpisodeLogError, match=f":{n + 1}"):
        EO.read_episodes(ep)


def test_sidecar_length_mismatch(tmp_path, golden_cli):
    _, sc, _ = _write(tmp_path, golden_cli)
    with pytest.raises(MaskMismatch):
        EO.read_sidecar(sc, 3)


def test_unknown_config_key_rejected(tmp_path):
    p = tmp_path / "c.yaml"
    p.write_text("loss:\n  epsilon: 0.3\n")
    with pytest.raises(ValueError):
        cli.load_loss_config(p)


def _close(a, b, rel=1e-12):
    return abs(a - b) <= rel * max(abs(a), abs(b), 1e-300)


@pytest.mark.gpu
@pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")
def test_loss_report_matches_reference(tmp_path, golden_cli):
    ep, sc, cfg = _write(tmp_path, golden_cli)
    for rep, exp in ((cli.loss_report(ep), golden_cli["report_embedded"]),
                     (cli.loss_report(ep, sc, cfg), golden_cli["report_sidecar"])):
        for k in ("masked_tokens", "groups", "episodes"):
            assert rep[k] == exp[k]
        for k in ("objective", "clip_fraction", "kl"):
            assert _close(rep[k], exp[k]), (k, rep[k], exp[k])


@pytest.mark.gpu
@pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")
def test_sidecar_observation_perturbation_is_invisible(tmp_path, golden_cli):
    """test_cli.py:177-204 — obs logp_new := 123.456 leaves the report byte-identical."""
    ep, sc, cfg = _write(tmp_path, golden_cli)
    recs = EO.read_episodes(ep)
    bumped = []
    for r, row in zip(recs, golden_cli["sidecar"]):
        mask = [s.origin == "action" for s in r["trajectory"].segments for _ in s.tokens]
        new = [lp if a else 123.456 for lp, a in zip(row["logp_new"], mask)]
        bumped.append(dict(row, logp_new=new))
    sc2 = tmp_path / "bumped.jsonl"
    sc2.write_text("".join(json.dumps(r) + "\n" for r in bumped), encoding="utf-8")
    assert json.dumps(cli.loss_report(ep, sc, cfg)) == json.dumps(cli.loss_report(ep, sc2, cfg))


@pytest.mark.gpu
@pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")
def test_singleton_group_fails_with_hint(tmp_path, golden_cli, capsys):
    ep, _, _ = _write(tmp_path, golden_cli)
    first = golden_cli["episodes_jsonl"].splitlines()[0]
    one = tmp_path / "one.jsonl"
    one.write_text(first + "\n", encoding="utf-8")
    assert cli.main(["loss", "--episodes", str(one)]) == 1
    assert "--samples" in capsys.readouterr().out
