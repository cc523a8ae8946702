"""Summarise a gpurun profiling session into profiles/ (run here, no GPU needed).

    python scripts/summarize_profiles.py TAG [--calls 2]

Reads gpurun_out/launches_TAG.csv (ncu --metrics gpu__time_duration.sum launch list of
scripts/prof_run.py) and every gpurun_out/prof_*_TAG.ncu-rep (ncu --set full captures),
writes profiles/TAG_launches.csv (the launch list, trimmed to our kernels),
profiles/TAG_ncu_summary.md (per-kernel duration, share, DRAM bytes, pipe utilisation)
and updates profiles/ncu_traffic.json (per-launch DRAM bytes, read by bench.py for
roofline.traffic).
"""
import csv
import glob
import io
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(HERE, "gpurun_out")
PROF = os.path.join(HERE, "profiles")

# kernel-name fragment -> bench.py kernel key
KEYS = [("fa2_kernel<1, 1>", "rstep_f32"), ("fa2_kernel<2, 1>", "attn_f32"), ("fa2_kernel<1, 0>", "rstep"),
        ("fa2_kernel<2, 0>", "attn_recompute"), ("lstep_hl_kernel<0", "lstep_f32"),
        ("lstep_hl_kernel<1", "lstep_apply_f32"), ("split_hilo", "split_hilo"),
        ("fa_tc_kernel<2, 2", "rstep_y"), ("fa_tc_kernel<1, 1", "rstep"), ("fa2_kernel<1>", "rstep"),
        ("fa2_kernel<2>", "attn_recompute"), ("fa3_kernel<2", "attn_recompute"), ("fa3_kernel<1", "rstep"),
        ("fa4_kernel<1, 1>", "rstep"), ("fa4_kernel<2, 2>", "rstep_y"), ("fa4_kernel<2, 1>", "attn_recompute"),
        ("fa6_kernel<2", "attn_recompute"), ("fa6_kernel<1", "rstep"),
        ("lstep_tc_kernel<0", "lstep"), ("lstep_tc_kernel<1", "lstep_apply"), ("lstep_big_kernel<1", "lstep_big_iter"),
        ("lstep_big_kernel<2", "lstep_big_final"), ("lstep_big_kernel<0", "lstep_big_rowstat"), ("fa2_combine", "combine"),
        ("seq_assemble", "seq_assemble"), ("peer_gather", "peer_gather"), ("pad_rows", "pad_rows"),
        ("bwd_dq_kernel", "bwd_dq"), ("bwd_dkv_kernel", "bwd_dkv"), ("bwd_rowstat", "bwd_rowstat")]
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
           "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "launch__grid_size", "smsp__issue_active.avg.pct_of_peak_sustained_active"]
UNIT = {"ms": 1e-3, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "nsecond": 1e-9, "s": 1.0,
        "second": 1.0, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def key_of(name):
    for frag, k in KEYS:
        if frag in name:
            return k
    return None


def parse_csv(text):
    lines = [ln for ln in text.splitlines() if ln.startswith('"')]
    return list(csv.reader(io.StringIO("\n".join(lines))))


def main():
    tag = sys.argv[1]
    os.makedirs(PROF, exist_ok=True)
    md = [f"# ncu summary — {tag}", ""]
    # ---------------------------------------------------------------- launch list
    lpath = os.path.join(OUT, f"launches_{tag}.csv")
    if os.path.exists(lpath):
        rows = parse_csv(open(lpath).read())
        hdr, body = rows[0], rows[1:]
        ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
        ours = [(r[ki], float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1e-9)) for r in body if key_of(r[ki])]
        with open(os.path.join(PROF, f"{tag}_launches.csv"), "w") as f:
            w = csv.writer(f)
            w.writerow(["kernel", "key", "duration_us"])
            for n, t in ours:
                w.writerow([n, key_of(n), round(t * 1e6, 2)])
        tot = sum(t for _, t in ours)
        agg = {}
        for n, t in ours:
            a = agg.setdefault(key_of(n), [0, 0.0])
            a[0] += 1
            a[1] += t
        md += ["## Launch list (ncu gpu__time_duration, cold-cache serialised; compare shares)", "",
               "| kernel | launches | mean ms | share |", "|---|---|---|---|"]
        for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
            md.append(f"| {k} | {c} | {t / c * 1e3:.3f} | {t / tot:.3f} |")
        md.append("")
    # ---------------------------------------------------------------- full captures
    traffic_path = os.path.join(PROF, "ncu_traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    md += ["## `ncu --set full` captures", "",
           "| kernel | grid | regs | ms | DRAM read GB | DRAM write GB | DRAM % | tensor % | XU % | FMA % | ALU % | issue % | warps % |",
           "|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for rep in sorted(glob.glob(os.path.join(OUT, f"prof_*_{tag}.ncu-rep"))):
        txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = parse_csv(txt)
        if len(rows) < 3:
            continue
        hdr, units, body = rows[0], rows[1], rows[2:]
        col = {h: i for i, h in enumerate(hdr)}
        for r in body:
            name = r[col["Kernel Name"]]
            k = key_of(name) or name[:40]

            def g(mn, scale=True):
                if mn not in col:
                    return float("nan")
                v = r[col[mn]].replace(",", "")
                try:
                    x = float(v)
                except ValueError:
                    return float("nan")
                return x * UNIT.get(units[col[mn]], 1.0) if scale else x

            ms = g("gpu__time_duration.sum") * 1e3
            rd, wr = g("dram__bytes_read.sum"), g("dram__bytes_write.sum")
            md.append(
                f"| {k} | {int(g('launch__grid_size', False))} | {int(g('launch__registers_per_thread', False))} | "
                f"{ms:.3f} | {rd / 1e9:.3f} | {wr / 1e9:.3f} | "
                f"{g('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', False):.1f} | "
                f"{g('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active', False):.1f} | "
                f"{g('sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active', False):.1f} | "
                f"{g('sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active', False):.1f} | "
                f"{g('sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active', False):.1f} | "
                f"{g('smsp__issue_active.avg.pct_of_peak_sustained_active', False):.1f} | "
                f"{g('sm__warps_active.avg.pct_of_peak_sustained_active', False):.1f} |")
            if key_of(name):
                traffic[key_of(name)] = {"bytes": rd + wr, "tag": tag}
    md.append("")
    with open(traffic_path, "w") as f:
        json.dump(traffic, f, indent=1, sort_keys=True)
    with open(os.path.join(PROF, f"{tag}_ncu_summary.md"), "w") as f:
        f.write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
