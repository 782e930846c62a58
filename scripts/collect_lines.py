# SPDX-License-Identifier: Apache-2.0
"""Copy bench JSON lines from gpurun_out/ logs into tracked profiles/ files.

  python scripts/collect_lines.py configs          cfg{1,3,4,5}.log -> profiles/r1_bench_config{N}.json
  python scripts/collect_lines.py scaling N [N..]  multi_{bench,vp,vp2}_N.log -> profiles/r1_scaling.json
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")


def last_line(path):
    lines = [l for l in open(path) if l.startswith("{")]
    return json.loads(lines[-1]) if lines else None


def main():
    what = sys.argv[1]
    if what == "configs":
        for c in (1, 3, 4, 5, "_fwd"):
            p = os.path.join(OUT, f"cfg{c}.log")
            d = last_line(p) if os.path.exists(p) else None
            if d:
                name = "r1_bench_fwd_only.json" if c == "_fwd" else f"r1_bench_config{c}.json"
                json.dump(d, open(os.path.join(PROF, name), "w"), indent=1)
                print(c, d["value"], d.get("roofline", {}).get("frac"))
    elif what == "scaling":
        path = os.path.join(PROF, "r1_scaling.json")
        sc = json.load(open(path)) if os.path.exists(path) else {}
        for n in sys.argv[2:]:
            for key, f in (("dp_config2", "multi_bench"), ("vp_fused_config5", "multi_vp"), ("vp_two_pass_config5", "multi_vp2")):
                p = os.path.join(OUT, f"{f}_{n}.log")
                if os.path.exists(p) and (d := last_line(p)):
                    sc[f"{key}_n{n}"] = d
                    print(key, n, d["value"], d.get("roofline", {}).get("frac"))
        for old in [k for k in sc if k.startswith(("vp_config5_", "vocab_parallel_config5_"))]:
            del sc[old]
        json.dump(dict(sorted(sc.items())), open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
