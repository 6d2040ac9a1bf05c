"""Key metrics + warp-stall shares (pc sampling) per kernel launch of ncu
--set full reports, as JSON: python tools/ncu_full_json.py out.json tag=rep.ncu-rep ..."""
import csv, json, subprocess, sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
out = {}
for arg in sys.argv[2:]:
    tag, rep = arg.split("=", 1)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    stall = [i for i, h in enumerate(hdr) if h.startswith("smsp__pcsamp_warps_issue_stalled_")
             and not h.endswith("_not_issued")]
    for k, r in enumerate(rows[2:]):
        d = {w: f"{r[hdr.index(w)]} {units[hdr.index(w)]}".strip() for w in WANT if w in hdr}
        sv = {hdr[i][len("smsp__pcsamp_warps_issue_stalled_"):]: float(r[i] or 0) for i in stall}
        tot = sum(sv.values()) or 1.0
        d["stall_share"] = {a: round(v / tot, 3) for a, v in sorted(sv.items(), key=lambda kv: -kv[1])[:8]}
        out[f"{tag}:{k}:{r[hdr.index('Kernel Name')]}"] = d
json.dump(out, open(sys.argv[1], "w"), indent=1)
print(len(out), "launches")
