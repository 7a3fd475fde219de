"""Summaries of ncu output for profiles/ (run here, on the files gpurun brought back).

    python tools/ncu_summary.py full REPORT.ncu-rep        # key --set full metrics + stall reasons
    python tools/ncu_summary.py list LAUNCHES.csv          # per-kernel totals of a launch list
"""
import collections
import csv
import io
import subprocess
import sys

KEEP = ("GPU Speed Of Light Throughput", "Compute Workload Analysis", "Memory Workload Analysis",
        "Occupancy", "Launch Statistics", "Scheduler Statistics", "Warp State Statistics")
RAW = ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
       "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_tensor_op_dmma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_tensor_op_dmma.sum", "sm__sass_thread_inst_executed_op_dfma_pred_on.sum",
       "lts__t_bytes.sum", "l1tex__t_bytes.sum", "smsp__cycles_active.avg")


def ncu_csv(args):
    out = subprocess.run(["ncu"] + args + ["--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def full(rep):
    rows = ncu_csv(["-i", rep, "--page", "details"])
    h = rows[0]
    for r in rows[1:]:
        d = dict(zip(h, r))
        if d.get("Section Name") in KEEP and d.get("Metric Value"):
            print(f"{d['Section Name'][:26]:27s}{d['Metric Name'][:52]:53s}{d['Metric Value']} {d['Metric Unit']}")
    raw = ncu_csv(["-i", rep, "--page", "raw"])
    if len(raw) >= 3:
        names, units, vals = raw[0], raw[1], raw[2]
        stalls = []
        for n, u, v in zip(names, units, vals):
            if n in RAW or n.startswith("sm__pipe_") and "pct_of_peak_sustained_active" in n and "avg" in n:
                print(f"{n} {v} {u}")
            if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("_not_issued"):
                try:
                    stalls.append((float(v.replace(",", "")), n[len("smsp__pcsamp_warps_issue_stalled_"):]))
                except ValueError:
                    pass
        tot = sum(s for s, _ in stalls) or 1.0
        print("# stall reasons (pc sampling, share of samples)")
        for s, n in sorted(stalls, reverse=True)[:10]:
            print(f"{n:30s} {100 * s / tot:5.1f} %")


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    agg = collections.defaultdict(lambda: collections.defaultdict(float))
    cnt = collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "").replace("unnamed>::", "")[:58]
        agg[name][r[mi]] += float(r[vi].replace(",", ""))
        if r[mi] == "gpu__time_duration.sum":
            cnt[name] += 1
    tot = sum(a["gpu__time_duration.sum"] for a in agg.values())
    print(f"# {path}: {sum(cnt.values())} launches, {tot / 1e6:.1f} ms of kernel time (serialised, cold-cache)")
    print(f"{'kernel':58s} {'launches':>8s} {'ms':>9s} {'share':>6s} {'DRAM GB':>8s}")
    for name, a in sorted(agg.items(), key=lambda kv: -kv[1]["gpu__time_duration.sum"]):
        t = a["gpu__time_duration.sum"]
        dram = (a.get("dram__bytes_read.sum", 0.0) + a.get("dram__bytes_write.sum", 0.0)) / 1e9
        print(f"{name:58s} {cnt[name]:8d} {t / 1e6:9.2f} {t / tot:6.3f} {dram:8.2f}")


if __name__ == "__main__":
    {"full": full, "list": launches}[sys.argv[1]](sys.argv[2])
