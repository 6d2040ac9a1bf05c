"""Round-2 evidence summaries from gpurun_out/r02 (see tools/gpu/evidence_r02.sh):
profiles/r02/launches_<cfg>.txt (per-launch device time, DRAM bytes, warp
instructions; one host-loop hull under ncu) and profiles/round_traffic.json
(mean DRAM read + write bytes per round launch, the `traffic` field of
bench.py's roofline: the first-split count and every loop round, a peeled
round's k_stream / k_round pair counted as one launch)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from launches import load

SRC, DST = "gpurun_out/r02", "profiles/r02"
traffic = {"_source": "profiles/r02/launches_<cfg>.txt: mean dram__bytes_read.sum + dram__bytes_write.sum "
                      "per round launch (first-split count + every loop round; the paired k_stream / k_round "
                      "launch of a peeled round counts once) of one hull in host-loop mode (ncu, "
                      "--clock-control none)"}
for cfg in ("C1", "C2", "C3", "C3n", "C4c", "C4b", "C5"):
    p = os.path.join(SRC, f"launches_{cfg}.csv")
    if not os.path.exists(p):
        continue
    L = load(p)
    lines, rounds, cur = [], [], None
    for d in L:
        t = d.get("gpu__time_duration.sum", 0)
        rb, wb = d.get("dram__bytes_read.sum", 0), d.get("dram__bytes_write.sum", 0)
        ins = d.get("smsp__inst_executed.sum", 0)
        lines.append(f"{d['name'][:52]:52s} {t:9.1f} us  rd {rb/1e6:8.1f} MB  wr {wb/1e6:8.1f} MB  "
                     f"{(rb + wb) / t / 1e3 if t else 0:6.0f} GB/s  {ins/1e6:8.2f} M inst")
        n = d["name"]
        if "k_first_count" in n or "k_stream" in n or "k_round<" in n:
            if "k_round<" in n and cur is not None and cur[0] == "pair":
                cur[1] += rb + wb
                rounds.append(cur[1])
                cur = None
            elif "k_stream" in n and ", 1>" in n:
                cur = ["pair", rb + wb]
            else:
                rounds.append(rb + wb)
    tot = sum(d.get("gpu__time_duration.sum", 0) for d in L)
    open(os.path.join(DST, f"launches_{cfg}.txt"), "w").write(
        "\n".join(lines) + f"\ntotal {tot:.1f} us, {len(L)} launches (ncu: serialised, cold caches)\n")
    traffic[cfg] = int(sum(rounds) / len(rounds))
json.dump(traffic, open("profiles/round_traffic.json", "w"), indent=1)
print(json.dumps(traffic, indent=1))
