"""tools/vmb_bench.py: the reference bench harness (bench_main.cpp) on the B200 path.
Mirrors the reference's tests/test_cli.cpp case by case (the CPU cases exercise argument,
preset and MATN validation, which fail before any device work)."""
import json
import os
import struct
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "tools", "vmb_bench.py")


def run_cli(args, timeout=600):
    r = subprocess.run([sys.executable, CLI] + args.split(), capture_output=True, text=True, timeout=timeout)
    return r.returncode, r.stdout + r.stderr


# ------------------------------------------------------------------ host-side (CPU)
def test_matn_round_trip(tmp_path):
    from paper_2601_22275_b200.matn import read_matn, write_matn
    for arr in (np.arange(24, dtype=np.float32).reshape(2, 3, 4), np.linspace(0, 1, 7).astype(np.float64)):
        p = tmp_path / "x.matn"
        write_matn(str(p), arr)
        back = read_matn(str(p))
        assert back.dtype == arr.dtype and back.shape == arr.shape and np.array_equal(back, arr)
        raw = open(p, "rb").read()
        assert raw[:4] == b"MATN" and struct.unpack("<II", raw[4:12]) == (1, arr.ndim)


@pytest.mark.parametrize("mutate,field", [(lambda b: b"XATN" + b[4:], "magic"),
                                          (lambda b: b[:4] + struct.pack("<I", 2) + b[8:], "version"),
                                          (lambda b: b[:8] + struct.pack("<I", 0) + b[12:], "rank"),
                                          (lambda b: b[:-4], "payload"),
                                          (lambda b: b + b"\x00", "payload")])
def test_matn_malformed_names_field(tmp_path, mutate, field):
    from paper_2601_22275_b200.matn import MatnError, read_matn, write_matn
    p = tmp_path / "x.matn"
    write_matn(str(p), np.ones((2, 3), np.float32))
    raw = p.read_bytes()
    p.write_bytes(mutate(raw))
    with pytest.raises(MatnError, match=f"field '{field}'"):
        read_matn(str(p))


def test_malformed_matn_input_exits_1(tmp_path):
    p = tmp_path / "bad.matn"
    p.write_bytes(b"NOPE" + b"\x00" * 32)
    code, out = run_cli(f"--mode flash --in {p}")
    assert code == 1 and "magic" in out


def test_unknown_preset_exits_with_error():
    code, out = run_cli("--mode vmonarch --preset wan-999f")
    assert code == 1 and "preset" in out


def test_mode_required():
    code, out = run_cli("--n 4")
    assert code == 1 and "--mode is required" in out


def test_bad_grid_spec():
    code, out = run_cli("--mode vmonarch --grid 4x8")
    assert code == 1 and "TxHxW" in out


# ------------------------------------------------------------------ on the GPU
gpu = pytest.mark.gpu


@gpu
def test_dense_mode_with_a_single_token_is_exact(cuda):
    code, out = run_cli("--mode dense --n 1 --d 4 --verify on")
    assert code == 0, out
    j = json.loads(out)
    assert j["mode"] == "dense" and j["verify"]["max_abs_err"] == 0.0


@gpu
def test_flash_mode_verifies_against_the_dense_oracle(cuda):
    code, out = run_cli("--mode flash --n 512 --d 32 --verify on --seed 7")
    assert code == 0, out
    j = json.loads(out)
    assert j["verify"]["max_abs_err"] < 1e-4 and j["n"] == 512


@gpu
def test_vmonarch_preset_reports_both_sparsity_figures(cuda):
    code, out = run_cli("--mode vmonarch --preset wan-61f --t 2 --d 8 --verify off")
    assert code == 0, out
    j = json.loads(out)
    assert j["cost"]["sparsity"] == pytest.approx(0.873626, rel=1e-4)
    assert j["cost"]["sparsity_approx"] == pytest.approx(0.875, rel=1e-6)
    assert j["grid"]["t"] == 16 and "verify" not in j


@gpu
def test_verify_above_the_cap_is_refused_with_exit_code_2(cuda):
    code, out = run_cli("--mode dense --n 16384 --d 8 --verify on")
    assert code == 2 and "verify requires" in out


@gpu
def test_reports_identical_across_runs_apart_from_timing(cuda):
    args = "--mode monarch --n 256 --d 16 --m 16 --b 16 --verify on --seed 3"
    ca, a = run_cli(args)
    cb, b = run_cli(args)
    assert ca == 0 and cb == 0, a + b
    ja, jb = json.loads(a), json.loads(b)
    ja.pop("wall_ns")
    jb.pop("wall_ns")
    assert ja == jb and ja["verify"]["max_abs_err"] < 1e-4


@gpu
def test_csv_report_keeps_the_documented_column_order(cuda):
    code, out = run_cli("--mode flash --n 64 --d 8 --csv")
    assert code == 0, out
    assert out.splitlines()[0] == (
        "mode,precision,seed,n,d,m,b,iters,heads,batch,clamp,clamp_min,recompute,br,bc,dist,"
        "threads,repeats,wall_ns_median,macs,sparsity,sparsity_approx,monarch_flops,"
        "full_attn_flops,recompute_flops,reduction_ratio,max_abs_err,rel_fro_err")
    assert "flash,f32,0,64,8," in out


@gpu
def test_sweep_rows_and_empty_range(cuda):
    code, out = run_cli("--sweep 4:8:4 --grid 1x4x4 --d 8")
    assert code == 0, out
    assert out.count("\n") == 3 and "\n4,4,4,64,8," in out and "\n8,4,4,128,8," in out
    code, out = run_cli("--sweep 8:4 --grid 1x4x4 --d 8")
    assert code == 0 and out.count("\n") == 1 and out.startswith("T,h,w,n,d,iters")


@gpu
def test_sweep_records_per_row_refusals(cuda):
    code, out = run_cli("--sweep 60:64:4 --grid 1x12x12 --d 8 --verify on")
    assert code == 0, out
    assert out.count("\n") == 3 and "refused:verify-cap" in out


@gpu
def test_matn_input_feeds_the_flash_path(cuda, tmp_path):
    from paper_2601_22275_b200.matn import write_matn
    rng = np.random.default_rng(0)
    p = tmp_path / "qkv.matn"
    write_matn(str(p), rng.standard_normal((3, 96, 16)).astype(np.float32))
    code, out = run_cli(f"--mode flash --in {p} --verify on")
    assert code == 0, out
    j = json.loads(out)
    assert j["n"] == 96 and j["d"] == 16 and j["verify"]["max_abs_err"] < 1e-4


@gpu
def test_out_flag_writes_the_report_to_a_file(cuda, tmp_path):
    p = tmp_path / "r.json"
    code, out = run_cli(f"--mode dense --n 8 --d 4 --out {p}")
    assert code == 0 and out.strip() == ""
    assert json.loads(p.read_text())["mode"] == "dense"


@gpu
@pytest.mark.parametrize("precision,tol", [("f32", 1e-4), ("bf16", 2e-2)])
def test_vmonarch_verify_against_materialised_map(cuda, precision, tol):
    code, out = run_cli(f"--mode vmonarch --grid 4x8x16 --d 128 --heads 2 --verify on --precision {precision}")
    assert code == 0, out
    j = json.loads(out)
    assert j["verify"]["rel_fro_err"] <= tol
    assert j["macs"] * 2 == 2 * (j["cost"]["monarch_flops"] + j["cost"]["recompute_flops"])
