"""Per-model summary of an ncu launch list of scripts/forward_probe.py (weight-init kernels
excluded; the target's forwards come first, then the draft's).

    python scripts/summarize_probe_launches.py profiles/r01_launches_forward_probe.csv > out.md
"""
import collections
import csv
import re
import sys

EPI = {"0": "LM head (bf16)", "1": "O / down (+residual, norm stats)", "2": "gate/up (norm, SwiGLU)",
       "3": "QKV (norm, RoPE, KV append)"}
INIT = {"fill_normal_kernel", "scale_cols_kernel"}


def label(n):
    m = re.search(r"gemm_tn_kernel<(\d), (\d)>", n)
    if m:
        return f"K1 gemm {EPI[m.group(1)]}, {'CTA pair' if m.group(2) == '2' else 'single CTA'}"
    m = re.search(r"attn_mma_kernel<(\d+), (\d), (\d)(?:, \d)?>", n)
    if m:
        return f"K2 attention hd{m.group(1)}, {m.group(2)} vector warp(s), {m.group(3)} key slice(s)"
    return re.sub(r"\(.*", "", n).replace("unnamed>::", "").replace("wsb::", "")


def main():
    path = sys.argv[1]
    rows, hdr = [], None
    for r in csv.reader(open(path)):
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                rows.append((d["Kernel Name"], float(d["Metric Value"].replace(",", "")) / 1000.0))
    segs, cur = [], None
    for name, us in rows:
        phase = "init" if re.sub(r"\(.*", "", name).replace("unnamed>::", "") in INIT else "fwd"
        if cur is None or cur["phase"] != phase:
            cur = {"phase": phase, "k": []}
            segs.append(cur)
        cur["k"].append((label(name), us))
    fwd = [s for s in segs if s["phase"] == "fwd"]
    print("# r01 — ncu launch list of one verify and one draft forward (scripts/forward_probe.py)\n")
    print(f"Command: `python scripts/forward_probe.py 1 && ncu --metrics gpu__time_duration.sum --clock-control none "
          f"--csv --log-file {path} python scripts/forward_probe.py 1` (raw list beside this file). The probe runs the "
          "8B verify forward at the config-3 mean batch (105 requests x 5 rows over 176-position prefixes) and the 1B "
          "draft forward at its mean batch (256 worker tree groups of 2 leaves + 150 controller rows, 662 rows), 3 "
          "forwards each (2 warm-up + 1); weight-init kernels are excluded. ncu serialises launches and flushes "
          "caches, so compare shares; the same probe without ncu times the forwards with CUDA events (probe log).\n")
    for title, seg in zip(["Llama-3.1-8B verify forward (525 rows)", "Llama-3.2-1B draft forward (662 rows)"], fwd):
        agg = collections.OrderedDict()
        for lab, us in seg["k"]:
            a = agg.setdefault(lab, [0, 0.0])
            a[0] += 1
            a[1] += us
        tot = sum(v[1] for v in agg.values())
        print(f"## {title}\n\n{len(seg['k'])} launches over 3 forwards, {tot / 3 / 1000:.2f} ms device time per "
              "forward under ncu\n")
        print("| kernel | launches / fwd | µs / fwd | mean µs | share |\n|---|---:|---:|---:|---:|")
        for lab, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            print(f"| {lab} | {n / 3:.0f} | {us / 3:.0f} | {us / n:.1f} | {100 * us / tot:.1f}% |")
        print()


if __name__ == "__main__":
    main()
