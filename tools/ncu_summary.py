"""Summarise an ncu --set full capture (.ncu-rep) into the JSON kept under
profiles/: duration, DRAM traffic, issue / pipe utilisation, shared-atomic
wavefronts and conflicts, top stall reasons, per-opcode instruction mix per
48-atomic step (walk_kernel).  Run here (no GPU needed):
    python tools/ncu_summary.py gpurun_out/x.ncu-rep > profiles/x.json"""
import collections
import csv
import io
import json
import subprocess
import sys


def ncu_csv(rep, page, *extra):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra],
                         capture_output=True, text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main(rep):
    raw = ncu_csv(rep, "raw")
    hdr, vals = raw[0], raw[2]
    d = dict(zip(hdr, vals))

    def f(k):
        try:
            return float(d[k])
        except (KeyError, ValueError):
            return None
    keys = ["Kernel Name", "gpu__time_duration.sum", "sm__cycles_elapsed.avg", "launch__grid_size",
            "launch__block_size", "launch__registers_per_thread", "launch__shared_mem_per_block",
            "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
            "smsp__inst_executed_op_shared_atom.sum",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum",
            "sm__warps_active.avg.pct_of_peak_sustained_active",
            "lts__t_sectors_srcunit_tex_op_read.sum", "l1tex__t_sector_hit_rate.pct"]
    s = {k: (d.get(k) if k == "Kernel Name" else f(k)) for k in keys}
    units = dict(zip(hdr, raw[1]))
    s["_units"] = {k: units.get(k) for k in keys if k in units}
    stalls = {}
    for k in hdr:
        if "average_warps_issue_stalled" in k and k.endswith("per_issue_active.ratio"):
            v = f(k)
            if v and v > 0.05:
                stalls[k.split("stalled_")[1].split("_per")[0]] = round(v, 3)
    s["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda x: -x[1]))
    src = ncu_csv(rep, "source", "--print-source", "sass")
    sh, data = src[1], src[2:]
    isrc, iex = sh.index("Source"), sh.index("Instructions Executed")
    ops = collections.Counter()
    atoms = 0.0
    for r in data:
        n = float(r[iex] or 0)
        toks = r[isrc].strip().split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") else toks[0]
        if op.startswith("ATOMS"):
            atoms += n
        ops[op.split(".")[0]] += n
    if atoms:
        steps = atoms / 48.0
        s["per_step_48_atoms"] = {k: round(v / steps, 2) for k, v in ops.most_common(24)}
        s["instructions_per_step"] = round(sum(ops.values()) / steps, 1)
    print(json.dumps(s, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
