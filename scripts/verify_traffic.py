"""DRAM traffic of one 8B verify forward from an ncu metrics list of scripts/forward_probe.py
(the last of the 3 verify forwards: 163 kernels = embed, 32 x 5 per layer, final norm, LM
head) -> profiles/r01_verify_traffic.json (read by bench.py for roofline.traffic).

    WS_PROBE_VERIFY_REQ=198 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        --clock-control none --csv --log-file t.csv python scripts/forward_probe.py 1
    python scripts/verify_traffic.py t.csv 198 > profiles/r01_verify_traffic.json
"""
import collections
import csv
import json
import sys

INIT = ("fill_normal_kernel", "scale_cols_kernel")
PER_FWD = 163


def main():
    path, nreq = sys.argv[1], int(sys.argv[2])
    hdr, per = None, collections.OrderedDict()
    for r in csv.reader(open(path)):
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if any(k in d["Kernel Name"] for k in INIT):
                continue
            key = (d["ID"], d["Kernel Name"])
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3,
                     "msecond": 1e6}.get(d["Metric Unit"], 1)
            per.setdefault(key, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", "")) * scale
    ks = list(per.values())
    third = ks[2 * PER_FWD:3 * PER_FWD]
    rd = sum(k.get("dram__bytes_read.sum", 0) for k in third)
    wr = sum(k.get("dram__bytes_write.sum", 0) for k in third)
    ms = sum(k.get("gpu__time_duration.sum", 0) for k in third) / 1e6
    rows = nreq * 5
    print(json.dumps({
        "what": f"DRAM traffic of one 8B verify forward ({PER_FWD} kernels: embed, 32 x [QKV, attention, O, gate/up, "
                f"down], final norm, LM head) at {rows} rows ({nreq} requests x k+1), the third verify forward of "
                "scripts/forward_probe.py",
        "command": f"WS_PROBE_VERIFY_REQ={nreq} ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,"
                   "gpu__time_duration.sum --clock-control none --csv --log-file profiles/r01_verify_traffic.csv "
                   "python scripts/forward_probe.py 1",
        "rows": rows, "dram_read_bytes": int(rd), "dram_write_bytes": int(wr), "device_ms_under_ncu": round(ms, 3),
        "note": "ncu flushes caches before every kernel, so activations re-read from DRAM count; weights "
                "(15.0 GB) are read once"}, indent=1))


if __name__ == "__main__":
    main()
