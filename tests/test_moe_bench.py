"""The `moe bench` CLI (paper_2211_10017_b200/moe_bench): the reference's
bench report (proj/tools/moe_cli.cpp:54-135 schema, :291-394 cmd_bench)
over a .moec checkpoint's decoder MoE blocks."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2211_10017_b200", "moe_bench")
CKPT = os.path.join(ROOT, "tests", "golden", "model_int4.moec")

# validate_report_line's field list and type tags (moe_cli.cpp:52-73)
FIELDS = [("schema", str), ("config", dict), ("precision", str), ("batch", int), ("beam", int),
          ("prune", bool), ("seed", int), ("src_len", int), ("max_len", int), ("threads", int),
          ("steps", int), ("input_tokens", int), ("generated_tokens", int),
          ("expert_weight_bytes", int), ("expert_activation_bytes", int),
          ("expert_bytes_written", int), ("other_weight_bytes", int),
          ("other_activation_bytes", int), ("other_bytes_written", int), ("wall_ms", float),
          ("input_tokens_per_second", float)]
CONFIG_KEYS = ["d_model", "d_ffn", "n_enc_layers", "n_dec_layers", "n_experts", "n_heads",
               "vocab_size", "moe_every", "max_seq_len"]


def _need_cli():
    if not os.path.exists(CLI):
        pytest.skip("moe_bench not built (make tools)")


def test_cli_usage_and_argument_errors():
    _need_cli()
    r = subprocess.run([CLI, "--help"], capture_output=True, text=True)
    assert r.returncode == 0 and "moe-bench-v1" in r.stdout
    r = subprocess.run([CLI], capture_output=True, text=True)
    assert r.returncode == 2 and "--config is required" in r.stderr
    r = subprocess.run([CLI, "--config", CKPT, "--prune", "maybe"], capture_output=True, text=True)
    assert r.returncode == 2 and "--prune" in r.stderr


@pytest.mark.gpu
def test_cli_report_schema_and_counters(tmp_path):
    _need_cli()
    out = tmp_path / "report.jsonl"
    r = subprocess.run([CLI, "--config", CKPT, "--precision", "int4", "--batch", "2", "5",
                        "--beam", "1", "3", "--prune", "both", "--src-len", "8", "--max-len", "16",
                        "--seed", "7", "--out", str(out)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    lines = [json.loads(l) for l in out.read_text().splitlines()]
    assert len(lines) == 2 * 2 * 2
    for j in lines:
        assert list(j) == [k for k, _ in FIELDS]  # exactly the documented fields, in order
        for k, t in FIELDS:
            assert isinstance(j[k], t) or (t is float and isinstance(j[k], int)), k
            if t in (int, float):
                assert j[k] >= 0, k
        assert j["schema"] == "moe-bench-v1" and list(j["config"]) == CONFIG_KEYS
        assert j["config"]["d_model"] == 64 and j["config"]["n_experts"] == 4
        assert j["input_tokens"] == j["batch"] * 8 and j["steps"] <= 16
        assert j["expert_weight_bytes"] > 0 and j["wall_ms"] > 0
    # --prune both: the identical workload (same seed) with and without pruning;
    # pruned rows leave the expert workload
    by = {}
    for j in lines:
        by.setdefault((j["batch"], j["beam"]), {})[j["prune"]] = j
    for (b, m), pair in by.items():
        on, off = pair[True], pair[False]
        assert on["seed"] == off["seed"] and on["steps"] == off["steps"]
        assert on["generated_tokens"] == off["generated_tokens"]
        assert on["expert_activation_bytes"] <= off["expert_activation_bytes"]
        assert on["expert_weight_bytes"] <= off["expert_weight_bytes"]
    # precision guard (cmd_bench :292-300)
    r = subprocess.run([CLI, "--config", CKPT, "--precision", "fp16"], capture_output=True, text=True)
    assert r.returncode == 2 and "holds int4 weights" in r.stderr
