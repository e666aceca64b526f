"""Summarize an ncu --set full report of one training step into profiles/<tag>_ncu.json.

    python profiles/summarize_ncu.py gpurun_out/prof_step.ncu-rep r01
Per kernel launch: duration, DRAM bytes (read+write), L2 throughput, achieved
occupancy, tensor-pipe utilisation, top stall reasons.  bench.py reads
`dram_bytes_per_launch` for the roofline `traffic` field.
"""
import csv
import io
import json
import subprocess
import sys

NAMES = {"k_lif_fwd": "lif_fwd", "k_readout": "readout", "k_lif_bwd": "lif_bwd",
         "k_wgrad": "wgrad", "k_reduce_adam": "reduce_adam", "k_reduce": "reduce", "k_adam": "adam",
         "k_rlif_fwd": "rlif_fwd", "k_rlif_fwd_cl": "rlif_fwd", "k_rlif_bwd": "rlif_bwd",
         "k_rlif_bwd_cl": "rlif_bwd", "k_rlif_bwd_tc": "rlif_bwd", "k_peer_adam": "peer_adam"}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6}


def main(rep, tag):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]

    def val(r, k):
        i = hdr.index(k)
        try:
            return float(r[i].replace(",", "")), units[i]
        except ValueError:
            return None, units[i]

    out = {"report": rep, "kernels": [], "dram_bytes_per_launch": {}}
    counters = {}
    for r in rows[2:]:
        kname = r[hdr.index("Kernel Name")].split("(")[0].split("::")[-1].split("<")[0]
        kname = kname.replace("void ", "").strip()
        base = NAMES.get(kname, kname)
        idx = counters.get(base, 0)
        counters[base] = idx + 1
        name = base if base in ("readout", "wgrad", "reduce", "adam", "reduce_adam") else f"{base}[{idx}]"
        dur, du = val(r, "gpu__time_duration.sum")
        rd, ru = val(r, "dram__bytes_read.sum")
        wr, wu = val(r, "dram__bytes_write.sum")
        dram = (rd or 0) * UNIT.get(ru, 1) + (wr or 0) * UNIT.get(wu, 1)
        stalls = {}
        for i, h in enumerate(hdr):
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                try:
                    stalls[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(r[i])
                except ValueError:
                    pass
        tot = sum(stalls.values()) or 1.0
        top = sorted(stalls.items(), key=lambda x: -x[1])[:4]
        ent = {"name": name, "duration_us": dur * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3,
                                                    "msecond": 1e3}.get(du, 1.0),
               "dram_bytes": dram,
               "achieved_occupancy_pct": val(r, "sm__warps_active.avg.pct_of_peak_sustained_active")[0],
               "top_stalls": {k: round(v / tot, 3) for k, v in top}}
        # tensor pipe: sm__pipe_tensor_cycles_active (% of elapsed cycles the tcgen05
        # pipe is busy, all plane MMAs counted) and the UTCHMMA bf16->fp32 op counters
        # (the TPC.TriageCompute *_realtime variants are not the tcgen05 pipe)
        for k in hdr:
            if (k.startswith("sm__pipe_tensor_cycles_active.") or
                    k.startswith("sm__ops_path_tensor_op_utchmma") or
                    k in ("lts__t_bytes.sum.per_second", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
                          "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed")):
                v = val(r, k)[0]
                if v is not None:
                    ent[k] = v
        ent["tensor_pipe_pct"] = ent.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed")
        out["kernels"].append(ent)
        out["dram_bytes_per_launch"][name] = dram
    # backward launches run top-down: the first lif_bwd launch is the last hidden layer
    nb = counters.get("lif_bwd", 0)
    for k in out["kernels"]:
        if k["name"].startswith("lif_bwd["):
            k["name"] = f"lif_bwd[{nb - 1 - int(k['name'][8:-1])}]"
    out["dram_bytes_per_launch"] = {k["name"]: k["dram_bytes"] for k in out["kernels"]}
    json.dump(out, open(f"profiles/{tag}_ncu.json", "w"), indent=1)
    for k in out["kernels"]:
        tp = k.get("tensor_pipe_pct")
        print(f"{k['name']:14s} {k['duration_us']:8.1f} us  dram {k['dram_bytes']/1e6:8.2f} MB  "
              f"occ {k['achieved_occupancy_pct']:.1f}%  tensor-pipe {tp}%  {k['top_stalls']}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
