"""Summarise a round's GPU profiling artefacts (gpurun_out/) into profiles/.

    python scripts/ncu_summary.py --round 1

Inputs (written by scripts/gpu_profile.sh on the B200 box):
  gpurun_out/launches_c5.csv      ncu --metrics gpu__time_duration.sum launch list of `python bench.py`
  gpurun_out/c5_tail.ncu-rep      ncu --set full, first k_tail launch of config 5
  gpurun_out/c5_write.ncu-rep     ncu --set full, k_pass launch 14 (write launch 13) of config 5
  gpurun_out/plain_c5.log         the library's per-launch algorithmic bytes of the same run
  gpurun_out/bench_default.log    the bench JSON line
Outputs: profiles/ncu_traffic.json (read by bench.py for roofline.traffic), profiles/rNN_summary.md,
and CSV exports of the captures.
"""
import argparse
import ast
import csv
import json
import os
import re
import shutil
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "lts__t_sector_hit_rate.pct",
           "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
           "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
           "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
           "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-6, "us": 1e-3, "ms": 1,
         "msecond": 1, "usecond": 1e-3, "nsecond": 1e-6}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {}
    for m in METRICS:
        if m in hdr:
            i = hdr.index(m)
            v = float(vals[i].replace(",", ""))
            d[m] = v * SCALE.get(units[i], 1)
    return d, out


def launch_bytes():
    log = open(os.path.join(G, "plain_c5.log")).read()
    res = {}
    for cls in ("write", "tail"):
        m = re.search(rf"^{cls} launches (\d+) first bytes (\d+) bytes\[:16\] (\[.*\])$", log, re.M)
        if m:
            res[cls] = ast.literal_eval(m.group(3))
    return res


def launch_list():
    rows = list(csv.reader(open(os.path.join(G, "launches_c5.csv"))))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(r)
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in data:
        name = re.sub(r"\(.*", "", r[ki]).replace("void ", "")
        tot[name] += float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1)
        cnt[name] += 1
    return tot, cnt


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", type=int, default=1)
    a = ap.parse_args()
    tag = f"r{a.round:02d}"
    os.makedirs(P, exist_ok=True)
    lb = launch_bytes()
    traffic = {"config5": {}, "source": "ncu --set full --clock-control none, one launch per kernel class "
               "(scripts/gpu_profile.sh); algorithmic bytes of the same launch from hht_result_launches"}
    shaf = os.path.join(G, "libhht.sha256")
    # bench.py splices these counters into its line only when this hash equals the loaded library's
    traffic["libhht_sha256"] = open(shaf).read().split()[0] if os.path.exists(shaf) else None
    verf = os.path.join(G, "libhht.version")
    ver = open(verf).read().split() if os.path.exists(verf) else []
    traffic["libhht_build_id"] = ver[ver.index("build") + 1] if "build" in ver else None
    wskip = 14
    wf = os.path.join(G, "write_skip.txt")
    if os.path.exists(wf):
        wskip = int(open(wf).read().split()[-1])
    # write launch index = k_pass index - 1; write_ca: the largest count-ahead pass (write launch 6)
    caps = {"tail": ("c5_tail", 0), "write": ("c5_write", wskip - 1), "write_ca": ("c5_write_ca", 6)}
    for cls, (f, idx) in caps.items():
        rep = os.path.join(G, f + ".ncu-rep")
        if not os.path.exists(rep):
            continue
        d, text = raw(rep)
        open(os.path.join(P, f"{tag}_{f}_raw.csv"), "w").write(text)
        dram = d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]
        lcls = "write" if cls.startswith("write") else cls
        alg = lb.get(lcls, [None] * (idx + 1))[idx]
        traffic["config5"][cls] = {
            "traffic": dram, "algorithmic_bytes": alg, "traffic_over_algorithmic": dram / alg if alg else None,
            "duration_ms": d["gpu__time_duration.sum"],
            "issue_active_pct": d.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "alu_pipe_pct": d.get("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
            "fma_pipe_pct": d.get("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
            "lsu_pipe_pct": d.get("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
            "dram_pct": d.get("dram__throughput.avg.pct_of_peak_sustained_elapsed",
                              d.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")),
            "warps_active_pct": d.get("sm__warps_active.avg.pct_of_peak_sustained_active"),
            "registers": d.get("launch__registers_per_thread"),
            "smem_wavefronts_pct": d.get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
            "lsu_data_pipe_pct": d.get("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"),
            "smem_ld_wavefronts": d.get("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum"),
            "smem_st_wavefronts": d.get("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum"),
            "smem_bank_conflicts": d.get("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
            "warp_instructions": d.get("smsp__inst_executed.sum")}
    json.dump(traffic, open(os.path.join(P, "ncu_traffic.json"), "w"), indent=1)
    tot, cnt = launch_list()
    T = sum(tot.values())
    lines = [f"# Round {a.round} GPU profile summary (config 5, one B200)", "",
             f"Profiled build: id {traffic['libhht_build_id']} (sha256 of the CUDA sources, headers and nvcc "
             f"flags; bench.py attaches these counters only to a library with the same id), .so sha256 "
             f"{traffic['libhht_sha256']}", ""]
    if os.path.exists(os.path.join(G, "bench_default.log")):
        b = json.loads(open(os.path.join(G, "bench_default.log")).read().strip().splitlines()[-1])
        lines += ["## bench.py (default: config 5, 5 steps, 3 warm-up)", "",
                  f"- value: {b['value']:.4g} line-region tests/s; {b['ms_per_step']:.1f} ms/step (= ms/image)",
                  f"- tests/step {b['tests_per_step']:.4g}, pairs/step {b['pairs_per_step']:.4g}, ranges {b['ranges']}",
                  f"- kernel ms/step: " + ", ".join(f"{k} {v:.1f}" for k, v in b["kernel_ms"].items() if v > 0.01),
                  f"- roofline: {json.dumps(b['roofline'])}",
                  f"- clocks: {json.dumps(b['clocks'])}",
                  f"- e2e: {json.dumps(b['e2e'])}",
                  f"- cpu_baseline: {json.dumps(b['cpu_baseline'])}", ""]
        open(os.path.join(P, f"{tag}_bench_default.jsonl"), "w").write(json.dumps(b) + "\n")
    # bench lines of the other configs (C1-C4) and the int64 config-5 line, as run by gpu_profile.sh
    other = []
    for name in ["bench_c1", "bench_c2", "bench_c3", "bench_c4", "bench_c5_int64"]:
        f = os.path.join(G, name + ".log")
        if not os.path.exists(f) or not open(f).read().strip():
            continue
        b = json.loads(open(f).read().strip().splitlines()[-1])
        open(os.path.join(P, f"{tag}_{name}.jsonl"), "w").write(json.dumps(b) + "\n")
        other.append(f"| {name[6:]} | {b['config'].get('workload', '')[:60]} | {b['value']:.4g} | {b['ms_per_step']:.4g} | "
                     f"{b['e2e']['ms_per_step'] if isinstance(b.get('e2e'), dict) and 'ms_per_step' in b['e2e'] else 'n/a'} | "
                     f"{b['dtype']} | {b['roofline'].get('frac', float('nan')):.3f} |")
    if other:
        lines += ["## bench.py on the other configs (one detection per step; lines in profiles/" + tag + "_bench_c*.jsonl)", "",
                  "| config | workload | tests/s | ms/step | e2e ms/step | dtype | roofline frac |", "|---|---|---|---|---|---|---|"] + other + [""]
    if os.path.exists(os.path.join(G, "latency.md")):
        shutil.copy(os.path.join(G, "latency.md"), os.path.join(P, f"{tag}_latency.md"))
    lines += ["## ncu launch list of the same command (cold-cache, serialised: compare shares)", "",
              "| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"| `{k}` | {cnt[k]} | {v:.1f} | {100 * v / T:.1f}% |")
    lines += ["", "## ncu --set full captures", "",
              "| class | ms | DRAM bytes | algorithmic bytes | ratio | DRAM % | issue active % | ALU pipe % | FMA pipe % | LSU pipe % | smem wavefronts % | warps active % | regs |",
              "|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    fmt = lambda v, f: (format(v, f) if isinstance(v, (int, float)) else "n/a")  # noqa: E731
    for cls, t in traffic["config5"].items():
        t = {k: (v if v is not None else float("nan")) for k, v in t.items()}
        lines.append(f"| {cls} | {t['duration_ms']:.2f} | {t['traffic']:.4g} | {t['algorithmic_bytes']} | "
                     f"{(t['traffic_over_algorithmic'] or 0):.3f} | {t['dram_pct']:.1f} | {t['issue_active_pct']:.1f} | "
                     f"{t['alu_pipe_pct']:.1f} | {t['fma_pipe_pct']:.1f} | {t['lsu_pipe_pct']:.1f} | {t['smem_wavefronts_pct']:.1f} | "
                     f"{t['warps_active_pct']:.1f} | {t['registers']:.0f} |")
    open(os.path.join(P, f"{tag}_summary.md"), "w").write("\n".join(lines) + "\n")
    shutil.copy(os.path.join(G, "launches_c5.csv"), os.path.join(P, f"{tag}_launches_c5_bench.csv"))
    print("\n".join(lines))


if __name__ == "__main__":
    main()
