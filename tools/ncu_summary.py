"""Summarise an ncu --set full report: key counters + hottest SASS blocks."""
import csv
import io
import json
import subprocess
import sys

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'sm__issue_active.avg.pct_of_peak_sustained_elapsed',
        'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
        'sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'launch__shared_mem_per_block_dynamic', 'launch__grid_size', 'launch__block_size',
        'sm__inst_executed.sum', 'smsp__thread_inst_executed_per_inst_executed.ratio']


def raw(rep):
    out = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True,
                                  stderr=subprocess.DEVNULL)
    rows = list(csv.reader(io.StringIO(out)))
    return dict(zip(rows[0], rows[2])), dict(zip(rows[0], rows[1]))


def blocks(rep, top=6):
    out = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv",
                                   "--print-source=sass"], text=True, stderr=subprocess.DEVNULL)
    rows = list(csv.reader(io.StringIO(out)))
    hdr, data = rows[1], rows[2:]
    ia, isrc, ist = hdr.index("Instructions Executed"), hdr.index("Source"), \
        hdr.index("Warp Stall Sampling (All Samples)")
    tot = sum(float(r[ia] or 0) for r in data)
    stot = sum(float(r[ist] or 0) for r in data) or 1
    bl, cur = [], None
    for r in data:
        c = float(r[ia] or 0)
        if cur and abs(c - cur["count"]) <= cur["count"] * 0.001:
            cur["inst"] += 1
            cur["stall"] += float(r[ist] or 0)
            cur["src"].append(r[isrc])
        else:
            cur = {"count": c, "inst": 1, "stall": float(r[ist] or 0), "src": [r[isrc]]}
            bl.append(cur)
    bl.sort(key=lambda b: -b["count"] * b["inst"])
    res = []
    for b in bl[:top]:
        ops = {}
        for s in b["src"]:
            t = s.strip().split()
            op = t[1] if t and t[0].startswith("@") else (t[0] if t else "?")
            ops[op] = ops.get(op, 0) + 1
        res.append({"executions": b["count"], "sass_instructions": b["inst"],
                    "inst_share": round(b["count"] * b["inst"] / tot, 4),
                    "stall_share": round(b["stall"] / stot, 4),
                    "ops": dict(sorted(ops.items(), key=lambda x: -x[1])[:10])})
    return tot, res


if __name__ == "__main__":
    rep = sys.argv[1]
    d, u = raw(rep)
    summ = {k: (d.get(k), u.get(k)) for k in KEYS}
    stalls = {k.replace("smsp__average_warps_issue_stalled_", "").replace(
        "_per_issue_active.ratio", ""): float(v) for k, v in d.items()
        if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio")
        and float(v or 0) > 0.02}
    tot, bl = blocks(rep)
    print(json.dumps({"report": rep, "metrics": summ, "stalls_per_issue": stalls,
                      "warp_instructions": tot, "hot_blocks": bl}, indent=1))
