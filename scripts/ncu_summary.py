"""Summarise an `ncu --set full` capture (one kernel launch) for profiles/:
    python scripts/ncu_summary.py gpurun_out/k1_r01b.ncu-rep [--algo-bytes B] [--sass]
Prints duration, clocks, DRAM traffic, pipe utilisations, issue activity, top stall reasons and
(--sass) the executed-instruction mix by opcode."""
import argparse
import collections
import csv
import io
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("--algo-bytes", type=float, default=0.0)
ap.add_argument("--sass", action="store_true")
a = ap.parse_args()


def ncu_csv(*args):
    out = subprocess.run(["ncu", "-i", a.rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


rows = ncu_csv("--page", "raw")
hdr, units, vals = rows[0], rows[1], rows[2]
m = {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def g(k):
    v, u = m.get(k, ("n/a", ""))
    return f"{v} {u}".strip()


def f(k, scale=1.0):
    try:
        v, u = m[k]
        v = float(v)
        mult = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "ms": 1e-3, "us": 1e-6, "usecond": 1e-6,
                "msecond": 1e-3, "ns": 1e-9, "nsecond": 1e-9}.get(u, 1.0)
        return v * mult * scale
    except Exception:
        return float("nan")


print(f"kernel: {m.get('Kernel Name', ('?',))[0]}")
print(f"grid {g('launch__grid_size')} x block {g('launch__block_size')}, regs/thread {g('launch__registers_per_thread')}, "
      f"dyn smem/block {g('launch__shared_mem_per_block_dynamic')}")
print(f"duration: {g('gpu__time_duration.sum')}   SM clock under capture: {g('sm__cycles_elapsed.avg.per_second')}")
rd, wr = f("dram__bytes_read.sum"), f("dram__bytes_write.sum")
dur = f("gpu__time_duration.sum")
print(f"DRAM read {rd/1e6:.2f} MB, write {wr/1e6:.2f} MB, total {(rd+wr)/1e6:.2f} MB -> {(rd+wr)/dur/1e9:.0f} GB/s")
if a.algo_bytes:
    print(f"algorithmic bytes {a.algo_bytes/1e6:.2f} MB -> {a.algo_bytes/dur/1e9:.0f} GB/s; dram/algorithmic = {(rd+wr)/a.algo_bytes:.3f}")
for k in ["sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
          "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum.per_second",
          "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
          "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
          "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
          "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
          "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
          "sm__warps_active.avg.pct_of_peak_sustained_active",
          "l1tex__throughput.avg.pct_of_peak_sustained_active"]:
    if k in m:
        print(f"  {k:80s} {g(k)}")
stalls = [(h, float(v)) for h, (v, u) in m.items()
          if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
stalls.sort(key=lambda x: -x[1])
print("top stall reasons (warps per issue-active cycle):")
for h, v in stalls[:8]:
    print(f"  {h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):24s} {v:.3f}")
if a.sass:
    rows = ncu_csv("--page", "source", "--print-source", "sass")
    hdr = rows[1]
    iS, iE, iW = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    ops, st = collections.Counter(), collections.Counter()
    for r in rows[2:]:
        if len(r) <= iE or not r[iS].strip():
            continue
        toks = r[iS].strip().split()
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        op = op.split(".")[0]
        ops[op] += int(r[iE] or 0)
        st[op] += int(r[iW] or 0)
    tot, tots = sum(ops.values()), max(1, sum(st.values()))
    print(f"executed warp instructions: {tot}")
    for op, n in ops.most_common(20):
        print(f"  {op:12s} {n:12d} {100*n/tot:5.1f}%   stall samples {100*st[op]/tots:5.1f}%")
