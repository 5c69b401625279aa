"""Summarise a round's ncu captures (tools/profile_round.sh) into profiles/<tag>/.

    python tools/ncu_summary.py r1

Writes ncu_summary.md (per-kernel metrics of the --set full captures and the
kernel shares of the launch list) and ncu_traffic.json (DRAM bytes per launch,
read by bench.py for roofline.traffic)."""

import csv
import json
import os
import shutil
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KERNELS = ["k_cc6_red", "k_cc6_black", "k_mc_factor_cond_t", "k_mc_factor_compact", "k_cc_red_bc", "k_cc6_xred",
           "k_cond_es", "k_cond_expand",
           "k_cc_red", "k_cc_black", "k_sc_update_p", "k_sc_update_s", "k_sc_update_xr",
           "k_face_eval_light", "k_face_eval_energy", "k_face_gather", "k_decouple_compact_t", "k_decouple_compact",
           "k_cell_props", "k_cell_gas", "k_cell_rows", "k_cc_xred",
           "k_wells",
           # one-kernel variants (CELL_SPLIT=0 / FACE_SPLIT=0, earlier captures)
           "k_face_eval", "k_cell",
           # explicit decoupled form (ISC_COMPACT=0 / round-1 first captures)
           "k_sc_red", "k_mc_black_spmv", "k_decouple_ws", "k_mc_factor"]
METRICS = [
    ("gpu__time_duration.sum", "duration", 1.0),
    ("dram__bytes_read.sum", "DRAM read", 1.0),
    ("dram__bytes_write.sum", "DRAM write", 1.0),
    ("launch__registers_per_thread", "regs/thread", 1.0),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %", 1.0),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %", 1.0),
    ("lts__t_sector_hit_rate.pct", "L2 hit %", 1.0),
    ("launch__occupancy_limit_registers", "blocks/SM (regs)", 1.0),
]


def read_raw(path):
    with open(path) as fh:
        rows = list(csv.reader(fh))
    head, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(head, r))
        d["_units"] = dict(zip(head, units))
        out.append(d)
    return out


def to_bytes(val, unit):
    v = float(val.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)
    return v * scale


def to_ms(val, unit):
    v = float(val.replace(",", ""))
    return v * {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0,
                "ms": 1.0, "second": 1e3, "s": 1e3}[unit]


def main(tag):
    src = os.path.join(ROOT, "gpurun_out")
    dst = os.path.join(ROOT, "profiles", tag)
    os.makedirs(dst, exist_ok=True)
    lines = [f"# ncu summary, round {tag[1:]}", "",
             "`tools/profile_round.sh` on one B200: `ncu --set full --clock-control none "
             "--import-source on` of one launch per kernel inside `python bench.py --steps 1 "
             "--warmup 3` (C4, mcilu), after the plain bench run exited 0. Per-launch values; "
             "ncu times are cold-cache and serialised, the bench's CUDA-event times are the "
             "ones reported. Raw pages: `full_<tag>_<kernel>_raw.csv`.", "",
             "| kernel | " + " | ".join(m[1] for m in METRICS) + " | DRAM GB/s |",
             "|---" * (len(METRICS) + 2) + "|"]
    traffic = {}
    for k in KERNELS:
        p = os.path.join(src, f"full_{tag}_{k}_raw.csv")
        if not os.path.exists(p):
            continue
        recs = read_raw(p)
        if not recs:   # the kernel did not launch in this configuration
            continue
        shutil.copy(p, os.path.join(dst, os.path.basename(p)))
        d = recs[0]
        u = d["_units"]
        cells = []
        for key, _, _ in METRICS:
            v = d.get(key, "")
            if key.startswith("dram__bytes"):
                cells.append(f"{to_bytes(v, u[key]) / 1e9:.3f} GB")
            elif key == "gpu__time_duration.sum":
                cells.append(f"{to_ms(v, u[key]):.3f} ms")
            else:
                cells.append(v)
        rd = to_bytes(d["dram__bytes_read.sum"], u["dram__bytes_read.sum"])
        wr = to_bytes(d["dram__bytes_write.sum"], u["dram__bytes_write.sum"])
        ms = to_ms(d["gpu__time_duration.sum"], u["gpu__time_duration.sum"])
        traffic[k] = {"dram_bytes": rd + wr, "ncu_ms": ms}
        lines.append(f"| {d['Kernel Name'][:40]} | " + " | ".join(cells) +
                     f" | {(rd + wr) / ms / 1e6:.0f} |")
    # launch list shares
    lp = os.path.join(src, f"launches_{tag}.csv")
    if os.path.exists(lp):
        shutil.copy(lp, os.path.join(dst, f"launches_{tag}.csv"))
        with open(lp) as fh:
            rows = [r for r in csv.reader(l for l in fh if not l.startswith("=="))]
        head = rows[0]
        ik, iv, iu = head.index("Kernel Name"), head.index("Metric Value"), head.index("Metric Unit")
        tot = defaultdict(float)
        cnt = defaultdict(int)
        for r in rows[1:]:
            if len(r) <= iv:
                continue
            name = r[ik].split("(")[0].replace("void ", "").split("<")[0].strip()
            tot[name] += to_ms(r[iv], r[iu])
            cnt[name] += 1
        s = sum(tot.values())
        lines += ["", "## Launch list (ncu `gpu__time_duration.sum`, whole `bench.py --steps 2 "
                  "--warmup 1` run incl. setup)", "", "| kernel | launches | total ms | share |",
                  "|---|---|---|---|"]
        for name, v in sorted(tot.items(), key=lambda kv: -kv[1])[:20]:
            lines.append(f"| {name} | {cnt[name]} | {v:.2f} | {v / s:.3f} |")
    for cls, names in (("red_pass", ("k_cc6_red", "k_cc_red", "k_sc_red")),
                       ("black_pass", ("k_cc6_black", "k_cc_black", "k_mc_black_spmv")),
                       ("decouple", ("k_decouple_compact_t", "k_decouple_compact", "k_decouple_ws"))):
        for k in names:
            if k in traffic:
                traffic[cls] = {"dram_bytes": traffic[k]["dram_bytes"], "kernels": [k]}
                break
    with open(os.path.join(dst, "ncu_traffic.json"), "w") as fh:
        json.dump(traffic, fh, indent=1)
    with open(os.path.join(dst, "ncu_summary.md"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r1")
