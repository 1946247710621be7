"""Per-stage DRAM traffic and duration per launch from an ncu metrics capture of
scripts/profile_frame.py (one process, cold caches per launch as ncu replays them):

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file gpurun_out/traffic.csv \
        python scripts/profile_frame.py --frames 3
    python scripts/ncu_traffic.py gpurun_out/traffic.csv profiles/r01/ncu_traffic.json

Launches are mapped to bench.py stage names by kernel name (attention: grid z > 1 =
temporal); the last frame's launches are averaged per stage.  bench.py reads the JSON
for roofline.traffic.
"""
import csv
import json
import sys
from collections import defaultdict


def stage_of(name: str, grid: str) -> str:
    if "mask_fused" in name or "pack_input" in name:
        return "mask_stage"
    if "token_tc_kernel<0>" in name or "token_small_kernel<0" in name or "token_q_kernel<0" in name:
        return "embed_qkv"
    if "token_tc_kernel<2>" in name or "token_small_kernel<2" in name or "token_q_kernel<2" in name:
        return "slot_kv"
    if "token_tc_kernel<1>" in name or "token_small_kernel<1" in name or "token_q_kernel<1" in name:
        return "mlp_qkv"
    if "attn_tc_kernel" in name:
        z = int(grid.strip("()").split(",")[2])
        return "attn_temporal" if z > 1 else "attn_spatial"
    if "v2p" in name:
        return "vec2patch"
    if "conv3x3_tc_kernel<64" in name:
        return "decode0"
    if "dec2_gather" in name:
        return "decode2_composite"
    return "other:" + name[:40]


def main(src, dst):
    launches = defaultdict(dict)
    for r in csv.reader(open(src)):
        if len(r) < 15 or not r[0].isdigit():
            continue
        launches[int(r[0])].update({"name": r[4], "grid": r[8], r[12]: (r[13], float(r[14]))})
    ids = sorted(launches)
    # last frame = launches after the last mask-stage launch
    last = max(i for i in ids if "mask_fused" in launches[i]["name"])
    acc = defaultdict(list)
    for i in ids:
        if i < last:
            continue
        L = launches[i]
        st = stage_of(L["name"], L["grid"])
        unit_mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd = L["dram__bytes_read.sum"]
        wr = L["dram__bytes_write.sum"]
        dur = L["gpu__time_duration.sum"]
        acc[st].append((rd[1] * unit_mult.get(rd[0], 1) + wr[1] * unit_mult.get(wr[0], 1),
                        dur[1] * (1e-3 if dur[0] == "ns" else 1.0)))
    out = {st: {"dram_bytes_per_launch": sum(b for b, _ in v) / len(v),
                "ncu_us_per_launch": sum(t for _, t in v) / len(v), "launches": len(v)}
           for st, v in acc.items()}
    json.dump({"source": src, "note": "ncu replay: caches flushed per launch (cold)",
               "stages": out}, open(dst, "w"), indent=1)
    for st, v in out.items():
        print(f"{st:20s} {v['dram_bytes_per_launch']/1e6:8.2f} MB  {v['ncu_us_per_launch']:7.2f} us  x{v['launches']}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
