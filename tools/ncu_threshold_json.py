"""Summarises an ncu capture of one row chunk (tools/profile_query.py under
`ncu --metrics ... -k regex:"k_limb_gemm_pair|k_gate_keystream|k_reshare|k_lift|k_inject|k_msb"`)
into profiles/threshold_ncu.json (bench.py `roofline_compare.hbm`) and the GEMM
entry of profiles/ncu_traffic.json (bench.py `roofline.traffic`).

    ncu -i rep.ncu-rep --page raw --csv > raw.csv
    python tools/ncu_threshold_json.py raw.csv --lanes <lanes of the captured threshold job> \
        --gemm-lanes <lanes of one GEMM launch> --source <what was captured>
"""
import argparse
import csv
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--lanes", type=float, required=True)
    ap.add_argument("--gemm-lanes", type=float, required=True, dest="gemm_lanes")
    ap.add_argument("--source", required=True)
    a = ap.parse_args()
    rows = list(csv.reader(open(a.csv)))
    hdr, units = rows[0], rows[1]

    def val(r, name):
        i = hdr.index(name)
        v = float(r[i].replace(",", ""))
        u = units[i]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1, "us": 1e-3, "ns": 1e-6}.get(u, 1)
        return v * scale

    out = {"source": a.source, "lanes_per_threshold_job": a.lanes, "kernels": {}, "dram_bytes_per_lane": {}}
    gemm = []
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        short = name.split("(")[0].replace("void ", "").split("<")[0]
        short = {"k_reshare_lm": "k_reshare", "k_inject_lm": "k_inject"}.get(short, short)
        d = {"duration_ms": val(r, "gpu__time_duration.sum"),
             "dram_read_bytes": val(r, "dram__bytes_read.sum"), "dram_write_bytes": val(r, "dram__bytes_write.sum")}
        for m in ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
                  "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
                  "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"):
            if m in hdr:
                d[m] = val(r, m)
        if short == "k_limb_gemm_pair":
            gemm.append(d)
            continue
        out["kernels"][short] = d
        out["dram_bytes_per_lane"][short] = (d["dram_read_bytes"] + d["dram_write_bytes"]) / a.lanes
    out["dram_bytes_per_lane_total"] = sum(out["dram_bytes_per_lane"].values())
    json.dump(out, open(os.path.join(ROOT, "profiles", "threshold_ncu.json"), "w"), indent=1)
    if gemm:
        p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        t = json.load(open(p)) if os.path.exists(p) else {}
        b = sum(g["dram_read_bytes"] + g["dram_write_bytes"] for g in gemm) / len(gemm)
        t["plain_configs2"] = {
            "command": a.source, "gemm_dram_bytes_per_launch": b,
            "dram_read_bytes_per_launch": sum(g["dram_read_bytes"] for g in gemm) / len(gemm),
            "dram_write_bytes_per_launch": sum(g["dram_write_bytes"] for g in gemm) / len(gemm),
            "lanes_per_launch": a.gemm_lanes,
            "tensor_pipe_active_pct": sum(g.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 0)
                                          for g in gemm) / len(gemm),
            "duration_ms_cold": sum(g["duration_ms"] for g in gemm) / len(gemm)}
        json.dump(t, open(p, "w"), indent=1)
    print(json.dumps(out["dram_bytes_per_lane"], indent=1), out["dram_bytes_per_lane_total"])


if __name__ == "__main__":
    main()
