"""Summarise an ncu report: key metrics, stall reasons and the SASS opcode mix per kernel.

    python profiles/summarize_ncu.py gpurun_out/prof.ncu-rep [--traffic-json profiles/ncu_traffic.json
                                                              --config c4] > profiles/<round>_<name>.txt

--traffic-json merges, under the bench config name, per kernel ("p2g", "g2p", ...) the
dram__bytes_read.sum + dram__bytes_write.sum of one launch (bench.py's roofline `traffic`),
its executed warp instructions (bench.py's `issue_frac`: instructions / (launch time x
148 SMs x 4 schedulers x SM clock)) and its FMA-pipe active fraction (`fma_pipe_frac`).
"""
import json
import collections
import csv
import io
import subprocess
import sys

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy",
        "Warp Cycles Per Issued Instruction", "Executed Instructions", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Dynamic Shared Memory Per Block", "Block Limit Registers", "No Eligible"]


def run(args):
    return subprocess.run(["ncu"] + args, capture_output=True, text=True).stdout


UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def main(rep, traffic_json=None, config="c4"):
    traffic = {}
    rows = list(csv.reader(io.StringIO(run(["-i", rep, "--page", "details", "--csv"]))))
    h = rows[0]
    ki, mi, vi, ui, ii = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    by = collections.OrderedDict()
    for r in rows[1:]:
        by.setdefault((r[ii], r[ki].split("(")[0]), {})[r[mi]] = (r[vi], r[ui])
    raw = list(csv.reader(io.StringIO(run(["-i", rep, "--page", "raw", "--csv"]))))
    rh = raw[0]
    for n, ((i, k), m) in enumerate(by.items()):
        print(f"== launch {i}: {k}")
        for w in WANT:
            if w in m:
                print(f"   {w:38s} {m[w][0]} {m[w][1]}")
        d = dict(zip(rh, raw[2 + n])) if len(raw) > 2 + n else {}
        units = dict(zip(rh, raw[1])) if len(raw) > 1 else {}
        try:
            tb = sum(float(d[kk].replace(",", "")) * UNIT.get(units.get(kk, "byte"), 1.0)
                     for kk in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
            traffic[k.replace("qmpm_", "").replace("qmpm::k_", "")] = {"traffic": tb}
            print(f"   {'dram read+write per launch (bytes)':60s} {tb:.4e}")
        except (KeyError, ValueError):
            pass
        for key in ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed.sum",
                    "lts__t_sectors_op_red.sum", "lts__t_sectors_op_atom.sum",
                    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
                    "smsp__inst_executed_pipe_fma.sum", "smsp__inst_executed_pipe_alu.sum",
                    "smsp__inst_executed_pipe_lsu.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
                    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
                    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"):
            if key in d:
                print(f"   {key:60s} {d[key]}")
        try:  # the FMA pipe's active fraction (the binding unit of the step kernels)
            kk = k.replace("qmpm_", "").replace("qmpm::k_", "")
            traffic.setdefault(kk, {})["fma_pipe"] = float(
                d["sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"].replace(",", "")) / 100.0
        except (KeyError, ValueError):
            pass
        stalls = []
        for key, v in d.items():
            if key.startswith("smsp__average_warps_issue_stalled_") and key.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(v), key[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        print("   stalls (warps per issue): " + ", ".join(f"{s}={v:.2f}" for v, s in stalls[:8]))
        src = run(["-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--kernel-name", k, "--launch-skip", "0",
                   "--launch-count", "1"])
        srows = list(csv.reader(io.StringIO(src)))
        if len(srows) > 2:
            sh = srows[1]
            try:
                isrc, iex = sh.index("Source"), sh.index("Instructions Executed")
                ist = sh.index("Warp Stall Sampling (All Samples)")
            except ValueError:
                continue
            ops, stl, tot, tst = collections.Counter(), collections.Counter(), 0, 0
            for r in srows[2:]:
                try:
                    ex = int(r[iex] or 0)
                    st = int(r[ist] or 0)
                except (ValueError, IndexError):
                    continue
                t = r[isrc].split()
                if not t:
                    continue
                op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
                ops[op] += ex
                stl[op] += st
                tot += ex
                tst += st
            kk = k.replace("qmpm_", "").replace("qmpm::k_", "")
            traffic.setdefault(kk, {})["warp_inst"] = tot
            print(f"   SASS executed (warp instr): {tot}; top opcodes:")
            for op, c in ops.most_common(14):
                print(f"      {op:10s} {100 * c / max(tot, 1):5.1f}% of instr  {100 * stl[op] / max(tst, 1):5.1f}% of stall samples")


    if traffic_json:
        try:
            allc = json.load(open(traffic_json))
        except (OSError, ValueError):
            allc = {}
        if not all(isinstance(v, dict) for v in allc.values()) or any("traffic" in v for v in allc.values()):
            allc = {}  # (an older per-kernel file)
        allc[config] = traffic
        json.dump(allc, open(traffic_json, "w"), indent=1)


if __name__ == "__main__":
    tj = sys.argv[sys.argv.index("--traffic-json") + 1] if "--traffic-json" in sys.argv else None
    cfg = sys.argv[sys.argv.index("--config") + 1] if "--config" in sys.argv else "c4"
    main(sys.argv[1], tj, cfg)
