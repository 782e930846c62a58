# SPDX-License-Identifier: Apache-2.0
"""Summarise a round's ncu evidence (gpurun_out/ev_*) into tracked files under
profiles/ (run here, after scripts/prof_evidence.sh ran under gpurun).

  python scripts/summarize_profiles.py r1
"""
import collections
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")


def launches(tag):
    src = os.path.join(OUT, "ev_launches.csv")
    lines = [l for l in open(src) if not l.startswith("==")]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    with open(os.path.join(PROF, f"{tag}_launches.csv"), "w") as f:
        f.write("".join(lines))
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0]
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        ns = v * {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "nsecond": 1}.get(unit, 1)
        tot[name] += ns
        cnt[name] += 1
    allns = sum(tot.values())
    md = [f"# {tag}: ncu launch list of `python bench.py --steps 2 --warmup 1`",
          "", "`ncu --metrics gpu__time_duration.sum --clock-control none -c 400` (cold-cache, serialised: compare shares).",
          "The whole program is listed: `synth_logits_kernel` and the 16 `rows_ring_kernel<.., 0, 2>` launches "
          "(behaviour/reference log-probs of the synthetic batch) are setup outside the timed region; inside it "
          "the fused kernel is 99.9% of the step (`kernel_share_of_step` in the bench line).",
          "", "| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        md.append(f"| `{k}` | {cnt[k]} | {v / 1e6:.3f} | {v / allns * 100:.2f}% |")
    return "\n".join(md)


def ncu_raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return {h: (u, v) for h, u, v in zip(r[0], r[1], r[2])}


def full(tag):
    rep = os.path.join(OUT, "ev_full.ncu-rep")
    shutil.copy(rep, os.path.join(PROF, f"{tag}_fused_full.ncu-rep"))
    raw = ncu_raw(rep)
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
            "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__cluster_dim_x",
            "smsp__warps_active.avg.per_cycle_active"]
    kname = raw.get("Kernel Name", ("", "loss_tmem_kernel"))[1]
    md = [f"# {tag}: `ncu --set full` of the fused loss kernel (`{kname}`)", "",
          "Command: `python bench.py --seqs-per-mb 4 --micro-batches 1 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline`",
          "(16,384 rows x V=151,936 bf16; one launch captured after warm-up). Report: "
          f"`profiles/{tag}_fused_full.ncu-rep`.", "", "| metric | value |", "|---|---|"]
    for k in keys:
        if k in raw:
            u, v = raw[k]
            md.append(f"| `{k}` | {v} {u} |")
    stalls = {k: raw[k][1] for k in raw if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("per_issue_active.ratio")}
    md += ["", "Stall reasons (warps per issued instruction):", "", "| reason | ratio |", "|---|---|"]
    for k, v in sorted(stalls.items(), key=lambda kv: -float(kv[1] or 0))[:10]:
        md.append(f"| {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} | {v} |")
    return "\n".join(md)


EXTRA = [  # (capture name in gpurun_out or profiles, what, command)
    ("r2_narrow18992_ns4", "fused loss on 18,992-wide rows (a P = 8 vocab shard), 16,384 rows bf16, 4 row streams",
     "ncu --set full -k regex:loss_tmem_kernel -s 3 -c 1 python scripts/narrow_rows.py 16384 18992"),
    ("r2_narrow18992", "fused loss on 18,992-wide rows, one row at a time (before row streams; for comparison)",
     "scripts/ncu_narrow.sh (python scripts/narrow_rows.py 16384 18992)"),
    ("r2_wide151936", "fused loss on Qwen3 rows, 16,384 x 151,936 bf16 (isolated launch)",
     "scripts/ncu_narrow.sh (python scripts/narrow_rows.py 16384 151936)"),
    ("r1_fwd_stream", "forward-only streaming kernel (a1), 131,072 x 151,936 bf16 (round 1)",
     "scripts/ncu_kernel.sh r1_fwd_stream fwd_stream_kernel 3 python scripts/fwd_only.py"),
    ("r1_r3_fwd", "R3 gate forward, 48 x 131,072 rows x 128 experts fp32, top-8 (round 1)",
     "scripts/ncu_kernel.sh r1_r3_fwd r3_fwd_fast 3 python scripts/r3_split.py"),
]


def extra(tag):
    md = []
    for name, what, cmd in EXTRA:
        rep = os.path.join(OUT, f"{name}.ncu-rep")
        dst = os.path.join(PROF, f"{name}.ncu-rep")
        if os.path.exists(rep):
            shutil.copy(rep, dst)
        if not os.path.exists(dst):
            continue
        raw = ncu_raw(dst)
        keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                "smsp__issue_active.avg.pct_of_peak_sustained_active",
                "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
                "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
                "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
                "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]
        md += ["", f"# {tag}: `ncu --set full` of the {what}", "", f"Command: `{cmd}`; report `profiles/{name}.ncu-rep`.",
               "", "| metric | value |", "|---|---|"]
        for k in keys:
            if k in raw:
                u, v = raw[k]
                md.append(f"| `{k}` | {v} {u} |")
        if "dram__bytes_read.sum" in raw and "gpu__time_duration.sum" in raw:
            def num(k):
                u, v = raw[k]
                f = float(v.replace(",", ""))
                return f * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "ms": 1e-3, "us": 1e-6,
                            "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "nsecond": 1e-9}.get(u, 1)
            gbs = (num("dram__bytes_read.sum") + num("dram__bytes_write.sum")) / num("gpu__time_duration.sum") / 1e9
            md.append(f"| DRAM GB/s (read+write / duration) | {gbs:.0f} |")
    return "\n".join(md)


def traffic(tag):
    lines = [l for l in open(os.path.join(OUT, "ev_traffic.csv")) if not l.startswith("==")]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    vals = {r["Metric Name"]: float(r["Metric Value"].replace(",", "")) for r in rows}
    rd, wr = vals["dram__bytes_read.sum"], vals["dram__bytes_write.sum"]
    j = {"kernel": rows[0]["Kernel Name"], "vocab": 151936, "rows": 131072,
         "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
         "ncu_duration_ns": vals.get("gpu__time_duration.sum"),
         "command": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
                    "-k regex:loss_tmem_kernelItLi1E -s 2 -c 1 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline",
         "round": tag}
    json.dump(j, open(os.path.join(PROF, "fused_loss_traffic.json"), "w"), indent=1)
    return j


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
    os.makedirs(PROF, exist_ok=True)
    parts = [launches(tag), "", full(tag), extra(tag)]
    t = traffic(tag)
    parts += ["", f"# {tag}: DRAM traffic of one headline launch (131,072 rows x 151,936 bf16)", "",
              f"read {t['dram_bytes_read'] / 1e9:.3f} GB + write {t['dram_bytes_write'] / 1e9:.3f} GB = "
              f"{t['dram_bytes_per_launch'] / 1e9:.3f} GB per launch (ncu duration {t['ncu_duration_ns'] / 1e6:.3f} ms)."]
    bench = [l for l in open(os.path.join(OUT, "ev_plain.log")) if l.startswith("{")]
    if bench:
        d = json.loads(bench[-1])
        json.dump(d, open(os.path.join(PROF, f"{tag}_bench.json"), "w"), indent=1)
        parts += ["", f"# {tag}: bench line of the same run (not under ncu)", "", "```", json.dumps(d, indent=1), "```"]
    open(os.path.join(PROF, f"{tag}_summary.md"), "w").write("\n".join(parts) + "\n")
    print("\n".join(parts))


if __name__ == "__main__":
    main()
