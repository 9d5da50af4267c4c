"""Builds profiles/traffic.json from per-config ncu captures of one step
(`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
--csv --log-file traffic_cfgN.csv python scripts/one_cfg.py cfgN 1`).

The roofline's `traffic` is the DRAM bytes of the dominant kernel per launch:
tg_jit_tape for the JIT-tier configs (cfg1, cfg2), the whole chain of the
step's libtg kernels for the staged configs (cfg3-cfg5; torch fills of the
test harness excluded).
Usage: python scripts/traffic_json.py DIR [round-label]"""
import collections
import csv
import json
import os
import sys

BATCH = {"cfg1": 1_000_000, "cfg2": 65_536, "cfg3": 262_144, "cfg4": 8192, "cfg5": 1_048_576}


def parse(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ik, im, iv, iid = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
    ker = collections.OrderedDict()
    for r in rows[1:]:
        d = ker.setdefault(r[iid], {"name": r[ik]})
        d[r[im]] = float(r[iv].replace(",", ""))
    return list(ker.values())


def main(d, label):
    out = {}
    if os.path.exists("profiles/traffic.json"):   # configs without a new capture keep their entry
        out = json.load(open("profiles/traffic.json"))
    for cfg, b in BATCH.items():
        p = os.path.join(d, f"traffic_{cfg}.csv")
        if not os.path.exists(p):
            continue
        ks = [k for k in parse(p) if "at::" not in k["name"]]
        jit = [k for k in ks if k["name"].startswith("tg_jit_tape")]
        sel = jit if jit else ks
        what = "tg_jit_tape" if jit else f"staged chain: all {len(ks)} libtg kernels of one step"
        scale = "MB" if cfg in ("cfg1", "cfg2") else "GB"
        rd = sum(k.get("dram__bytes_read.sum", 0) for k in sel)
        wr = sum(k.get("dram__bytes_write.sum", 0) for k in sel)
        ms = sum(k.get("gpu__time_duration.sum", 0) for k in sel) / 1e6
        # ncu reports bytes in the unit it picks; the CSV values here are normalised by --print-units base
        out[cfg] = {"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr, "batch": b,
                    "kernel": what, "ncu_ms": ms,
                    "source": f"profiles/{label}/traffic_{cfg}.csv (ncu --metrics dram__bytes_read.sum,"
                              f"dram__bytes_write.sum, cold caches, scripts/one_cfg.py {cfg} 1)"}
        print(cfg, what, f"read {rd / 1e9:.3f} GB write {wr / 1e9:.3f} GB in {ms:.3f} ms (ncu)", scale)
    with open("profiles/traffic.json", "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "r06")
