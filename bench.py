"""Benchmark of the hierarchical Hough hot path (BASELINE.json metric: line-region tests/s and
ms/image at 1/2/4/8 B200; % of HBM roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl reference]

One step = one full detection (all levels, both halves, records + leaves) of the configuration's
synthetic edge points, resident in HBM. N > 1 runs under torch.distributed.run: points are sharded
contiguously across ranks, per-level votes are summed with NCCL inside libhht, the timed region is
bracketed by barrier + synchronize on every rank and the MAX over ranks is reported.
`cpu_baseline` and `--impl reference` time the CPU oracle (oracle/, as it stands; the only places
bench.py executes it) on all host cores, one oracle process per core, over a seeded sample of the
same workload: complete level-(D-7) subtrees of the detection (or whole images of a batch).
`roofline` reports the dominant kernel against its binding roof (the fused tail: the shared-memory
data path), with HBM figures beside it; ncu counters from profiles/ are attached
only when they were captured on the same libhht.so build.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "line-region tests/s"
UNIT = "tests/s"


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--impl", default="hht", choices=["hht", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--prefetch", type=int, default=0, help="0 auto, 1 descriptor only, 2 descriptor + entries")
    ap.add_argument("--tail-depth", type=int, default=0, help="0 auto; 3-6 (include/hht.h hht_opts.tail_depth)")
    ap.add_argument("--variant", default="exact", choices=["exact", "fht"],
                    help="membership test: the paper's exact corner code, or the FHT circumcircle comparison")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--oracle-steps", type=int, default=1, help="cpu_baseline: sampled oracle steps (all cores)")
    ap.add_argument("--force-int64", action="store_true", help="run the int64 kernel instantiation")
    return ap.parse_args()


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _issue_clock(dev):
    """SM count and SM clock for the integer-issue peak: MEASURED_PEAKS.json's max SM clock (the
    clock sampled under load is reported beside it in `clocks`), else the device's rated clock."""
    import torch
    prop = torch.cuda.get_device_properties(dev)
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return prop.multi_processor_count, float(json.load(f)["sm_max_mhz"]), "MEASURED_PEAKS.json sm_max_mhz"
    except Exception:
        return prop.multi_processor_count, 1965.0, "B200 max SM clock (fallback)"


def _workload(cfg):
    return {"workload": f"config{cfg.cid}: {cfg.text}", "N": cfg.N, "depth": cfg.D, "threshold": cfg.T,
            "images": cfg.images, "halves": "both" if cfg.halves == 3 else "alpha",
            "points_per_image": None, "seed": 0,
            "l2": ("L2 flushed before every timed step (a 256 MB write, outside the timed calls: the "
                   "value sums each call's own device time)" if _flush_l2(cfg) else
                   "inputs and candidate lists larger than L2 (126 MB); no flush")}


def _flush_l2(cfg):
    """Configs 1-3 fit (inputs) in the 126 MB L2: flush it between timed steps."""
    return cfg.cid <= 3


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region (B200_PROFILING.md recipe)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.p = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{index}.csv")

    def __enter__(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        try:
            self.f = open(self.path, "w")
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        if self.p is not None:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except Exception:
                self.p.kill()
            self.f.close()

    def summary(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 9:
                rows.append(f)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[5 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def _dist_init(n_gpus):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# --- the oracle as it stands, on all host cores, over a seeded sample of the same workload ---------
# Each task is one complete level-k subtree of the detection (oracle.detect_subtree from the region
# with ALL points as candidates; a region whose own votes exceed T has every ancestor above T by
# containment, so its subtree is exactly part of the workload), or one whole image of a batch. The
# subtree root's scan over all points is not workload and is not counted in tests (conservative).
_W = {}


def _worker_init(path):
    import numpy as np
    _W["pts"] = np.load(path, mmap_mode="r")


def _worker_task(t):
    import oracle
    import numpy as np
    kind, lo, hi, N, D, T, halves, half, k, a, c = t
    pts = np.ascontiguousarray(_W["pts"][lo:hi])
    if kind == "image":
        return oracle.detect(pts, N, D, T, halves).tests
    return oracle.detect_subtree(pts, N, D, T, half, k, a, c).tests - pts.shape[0]


class OracleSampler:
    def __init__(self, cfg, pts, offs, workers=None):
        import multiprocessing as mp
        import tempfile
        import numpy as np
        self.cfg, self.offs = cfg, offs
        ncpu = os.cpu_count() or 1
        try:
            import psutil
            cap = max(1, int(psutil.virtual_memory().available // (1 << 30)))   # ~1 GB per worker
        except Exception:  # noqa: BLE001
            cap = ncpu
        self.workers = workers or max(1, min(ncpu, cap))
        d = "/dev/shm" if os.path.isdir("/dev/shm") else tempfile.gettempdir()
        self.path = os.path.join(d, f"hht_bench_pts_{os.getpid()}.npy")
        np.save(self.path, np.ascontiguousarray(pts))
        self.pool = mp.get_context("spawn").Pool(self.workers, _worker_init, (self.path,))
        self.k = max(0, cfg.D - 7)

    def tasks(self, seed):
        import numpy as np
        cfg, rng = self.cfg, np.random.default_rng(1000 + seed)
        B = self.offs.shape[0] - 1
        if B > 1:
            imgs = rng.choice(B, size=min(B, self.workers), replace=False)
            return [("image", int(self.offs[b]), int(self.offs[b + 1]), cfg.N, cfg.D, cfg.T, cfg.halves, 0, 0, 0, 0)
                    for b in imgs], f"{len(imgs)} whole images of the batch"
        halves = [h for h in (1, 2) if cfg.halves & h]
        side = 1 << self.k
        n = 2 * self.workers
        cells = rng.choice(len(halves) * side * side, size=min(n, len(halves) * side * side), replace=False)
        out = []
        for q in cells.tolist():
            h, r = divmod(q, side * side)
            out.append(("subtree", 0, int(self.offs[1]), cfg.N, cfg.D, cfg.T, cfg.halves, halves[h], self.k,
                        r % side, r // side))
        return out, f"{len(out)} seeded level-{self.k} subtrees (of {len(halves) * side * side})"

    def step(self, seed):
        tasks, what = self.tasks(seed)
        t0 = time.perf_counter()
        tests = sum(self.pool.map(_worker_task, tasks, chunksize=1))
        return tests, time.perf_counter() - t0, what

    def close(self):
        self.pool.terminate()
        try:
            os.remove(self.path)
        except OSError:
            pass


def _cpu_baseline(sampler, steps=1):
    tot_t, tot_s, what = 0, 0.0, ""
    for k in range(steps):
        t, dt, what = sampler.step(k)
        tot_t += t
        tot_s += dt
    cfg = sampler.cfg
    return {"value": tot_t / tot_s, "unit": UNIT, "cores": sampler.workers, "kind": "oracle",
            "cpu_model": _cpu_model(), "os_cpu_count": os.cpu_count(),
            "sample": f"config{cfg.cid}: {what} per step x {steps}, one oracle process per core "
                      f"(plain C -O2, oracle/ as it stands); tests = code evaluations below each subtree "
                      f"root; {tot_t:.3g} tests in {tot_s:.1f} s wall",
            "seconds": tot_s, "tests": tot_t}


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np
    from paper_1007_0547_b200 import synth
    cfg = synth.CONFIGS[a.config]
    if cfg.images > 1:
        pts, offs = synth.config_batch(a.config)
    else:
        pts, _ = synth.config_image(a.config, 0)
        offs = np.array([0, pts.shape[0]], dtype=np.int64)
    smp = OracleSampler(cfg, pts, offs)
    try:
        for w in range(a.warmup):
            smp.step(10_000 + w)
        tot_tests, tot_s, what = 0, 0.0, ""
        for k in range(a.steps):
            t, dt, what = smp.step(k)
            tot_tests += t
            tot_s += dt
    finally:
        smp.close()
    v = tot_tests / tot_s
    wl = _workload(cfg)
    wl["points_per_image"] = int(offs[1] - offs[0])
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": a.gpus, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": 1e3 * tot_s / a.steps, "higher_is_better": True,
            "scaling": "weak" if cfg.images > 1 else "strong", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic", "config": wl,
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": smp.workers, "kind": "oracle",
                             "cpu_model": _cpu_model(), "os_cpu_count": os.cpu_count(),
                             "sample": f"{a.steps} steps, each {what} of config{cfg.cid}, one oracle process "
                                       f"per core; {tot_tests:.3g} tests in {tot_s:.1f} s"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _lib_build_id():
    """The loaded libhht.so's build id (hht_version: sha256 of its sources and nvcc flags)."""
    from paper_1007_0547_b200 import hht
    v = hht.version().split()
    return v[v.index("build") + 1] if "build" in v else None


def main():
    a = _args()
    if a.impl == "reference":
        return run_reference(a)
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_1007_0547_b200 import hht, synth

    rank, world, local = _dist_init(a.gpus)
    dev = torch.device("cuda", local)
    cfg = synth.CONFIGS[a.config]
    if cfg.images > 1:
        pts, offs = synth.config_batch(a.config)
    else:
        pts, _ = synth.config_image(a.config)
        offs = np.array([0, pts.shape[0]], dtype=np.int64)
    # shard: whole images across ranks for batches (independent trees), points within the image otherwise
    from paper_1007_0547_b200 import dist as hdist
    sh = hdist.make_shard(pts, offs, rank, world)
    my, my_offs, comm_world = sh.points, sh.offsets, sh.comm_world
    nccl_id = None
    if comm_world > 1:
        hdist.check_consistent(cfg.N, cfg.D, cfg.T, cfg.halves, 1)
        nccl_id = hdist.broadcast_bytes(hht.nccl_unique_id() if rank == 0 else None)
    h = hht.HHT(device=local, halves=cfg.halves, record_levels=True, profile=True,
                rank=rank if comm_world > 1 else 0, world=comm_world, nccl_id=nccl_id, prefetch=a.prefetch,
                tail_depth=a.tail_depth, force_int64=a.force_int64, variant=hht.FHT_CIRCLE if a.variant == "fht" else hht.EXACT)
    d_pts = torch.from_numpy(np.ascontiguousarray(my)).to(dev)
    B = my_offs.shape[0] - 1

    def step():
        if B > 1 or cfg.images > 1:
            h.detect_batch(d_pts, my_offs, cfg.N, cfg.D, cfg.T)
        else:
            h.detect(d_pts, cfg.N, cfg.D, cfg.T)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])

    flush = _flush_l2(cfg)
    scratch = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if flush else None

    def flush_l2():
        if flush:
            scratch.zero_()
            torch.cuda.synchronize()

    for _ in range(max(a.warmup, 0)):
        step()
    torch.cuda.synchronize()
    prof_tot = {}
    tests_tot = 0
    launches = 0
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        h.timer_begin()
        step_ms = []
        for _ in range(a.steps):
            flush_l2()
            step()
            st = h.stats()
            step_ms.append(st["ms"])
            tests_tot += st["tests"]
            for k, v in h.profile().items():
                p = prof_tot.setdefault(k, {"launches": 0, "ms": 0.0, "bytes": 0, "ops": 0})
                p["launches"] += v["launches"]
                p["ms"] += v["ms"]
                p["bytes"] += v["bytes"]
                p["ops"] += v.get("ops", 0)
        ms = h.timer_end()
        if flush:
            ms = float(sum(step_ms))   # each call's device time (CUDA events), flushes excluded
        torch.cuda.synchronize()
        barrier()
    clocks = clk.summary()
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        if cfg.images > 1:   # image-sharded: each rank's tests are its own; sum them
            tt = torch.tensor([tests_tot], dtype=torch.float64, device=dev)
            dist.all_reduce(tt)
            tests_tot = float(tt.item())
    st = h.stats()
    launches = sum(v["launches"] for k, v in prof_tot.items() if k != "allreduce")
    value = tests_tot / (ms / 1e3)
    ms_per_step = ms / a.steps
    images = cfg.images

    # roofline of the dominant kernel class (largest device time inside the timed region)
    peak, peak_kind = _peaks()
    dom = max((k for k in prof_tot if k not in ("allreduce",)), key=lambda k: prof_tot[k]["ms"])
    d = prof_tot[dom]
    nl = max(d["launches"], 1)
    avg_ms = d["ms"] / nl
    achieved_gbs = (d["bytes"] / nl) / (avg_ms / 1e3) / 1e9 if d["launches"] else 0.0
    # traffic and pipe counters: one launch of the same kernel class from the committed ncu --set full
    # capture (profiles/ncu_traffic.json), used only when it was taken on THIS build of libhht.so
    traffic, cap, ncu_note = None, {}, None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath))
            bid = _lib_build_id()
            if bid and bid != "unknown" and tj.get("libhht_build_id") == bid:
                cap = tj.get(f"config{cfg.cid}", {}).get(dom, {}) or {}
                traffic = cap.get("traffic")
                ncu_note = f"profiles/ncu_traffic.json, captured on this build ({bid})"
            else:
                ncu_note = (f"profiles/ncu_traffic.json was captured on another build "
                            f"({tj.get('libhht_build_id')}; this one {bid}); not used")
        except Exception:  # noqa: BLE001
            cap = {}
    hbm = {"achieved": achieved_gbs, "peak": peak, "unit": "GB/s", "frac": achieved_gbs / peak,
           "peak_source": peak_kind, "algorithmic_bytes_per_launch": d["bytes"] / nl, "traffic": traffic,
           "traffic_launch_algorithmic_bytes": cap.get("algorithmic_bytes")}
    if cap.get("issue_active_pct") is not None:
        ncu_note = ("ncu (same build): issue active %.0f%%, ALU pipe %.0f%%, FMA pipe %.0f%%, DRAM %.0f%%"
                    % (cap["issue_active_pct"], cap["alu_pipe_pct"], cap["fma_pipe_pct"], cap["dram_pct"]))
        if cap.get("smem_wavefronts_pct") is not None:
            ncu_note += ", shared-memory wavefronts %.0f%% (LSU data pipe %.0f%%)" % (
                cap["smem_wavefronts_pct"], cap.get("lsu_data_pipe_pct") or float("nan"))
    common = {"kernel": dom, "kernel_share_of_step": d["ms"] / max(sum(step_ms), 1e-9),
              "launches": d["launches"], "avg_launch_ms": avg_ms, "ncu": ncu_note}
    if d.get("ops"):
        # The fused tail's binding roof is the shared-memory data path ("Algorithmic
        # instructions"): every raster step (one line x one leaf column of a level-(D-4) region) is
        # one 8-byte column-mask lookup per lane. The library counts ops = 8 per step, so the
        # algorithmic lookup bytes per launch are ops / 8 steps x 8 B. Peak: 128 B / clock / SM.
        sms, mhz, mhz_src = _issue_clock(local)
        steps = d["ops"] / 8 / nl
        speak = sms * 128 * mhz * 1e6 / 1e12
        sach = (steps * 8) / (avg_ms / 1e3) / 1e12
        issue_peak = sms * 4 * 32 * mhz * 1e6 / 1e12
        roofline = {"bound": "smem", "achieved": sach, "peak": speak, "unit": "TB/s", "frac": sach / speak,
                    "traffic": traffic,
                    "peak_source": f"shared-memory data path: {sms} SMs x 128 B/clock x {mhz:.0f} MHz ({mhz_src})",
                    "algorithmic_bytes_per_launch": steps * 8, "raster_steps_per_launch": steps,
                    "unit_of_work": "raster step = one (line, leaf column) of a level-(D-4) region: one 8-B lookup",
                    **common, "hbm": hbm,
                    "issue": {"raster_steps_per_s": steps / (avg_ms / 1e3), "peak_thread_instr_per_s": issue_peak * 1e12,
                              "note": "the step itself is ~5 issue slots; see ncu issue active above"}}
    else:
        roofline = {"bound": "hbm", "achieved": achieved_gbs, "peak": peak, "unit": "GB/s",
                    "frac": achieved_gbs / peak, "traffic": traffic, "peak_source": peak_kind,
                    "algorithmic_bytes_per_launch": d["bytes"] / nl, **common}

    e2e = None
    if not a.no_e2e:
        host = torch.from_numpy(np.ascontiguousarray(my)).pin_memory()
        h2 = h
        hnp = host.numpy()
        h2.detect_batch(hnp, my_offs, cfg.N, cfg.D, cfg.T)   # warm
        nleaf = h2.stats()["leaves"]
        packed = cfg.D <= 16            # 8-byte rows (i, j, votes) + per-tree offsets; else 20-byte hht_leaf rows
        if packed:
            lbuf = torch.empty(max(int(nleaf * 1.1) + 1024, 1024), dtype=torch.int64).pin_memory().numpy().view(np.uint64)
            h2.set_leaf_sink_packed(lbuf)   # detected lines stream to the pinned buffer during detection
        else:
            lbuf = torch.empty((max(int(nleaf * 1.1) + 1024, 1024), 5), dtype=torch.int32).pin_memory().numpy().view(np.uint32)
            h2.set_leaf_sink(lbuf)
        h2.detect_batch(hnp, my_offs, cfg.N, cfg.D, cfg.T)   # untimed warm-up of the streaming path
        barrier()
        torch.cuda.synchronize()
        e_steps = max(1, a.steps if flush else min(a.steps, 3))
        d2h = 0
        et = 0.0
        for _ in range(e_steps):
            flush_l2()
            t0 = time.perf_counter()
            h2.detect_batch(hnp, my_offs, cfg.N, cfg.D, cfg.T)   # H2D of the points + D2H of the lines inside
            et += time.perf_counter() - t0                        # the call returns with its results on the host
            sst = h2.stats()
            assert sst["leaves_streamed"] == sst["leaves"], "leaf sink too small"
            d2h = sst["leaves_streamed"] * (8 if packed else 20)
        torch.cuda.synchronize()
        if world > 1:
            t = torch.tensor([et], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            et = float(t.item())
        e2e = {"value": tests_tot / a.steps * e_steps / et, "unit": UNIT,
               "h2d_bytes_per_step": int(hnp.nbytes), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": 1e3 * et / e_steps,
               "timing": "wall clock of each detect_batch call (pinned host points in, the detected lines streamed "
                         "to a pinned host buffer during the call: " +
                         ("hht_set_leaf_sink_packed, 8-byte (i, j, votes) rows" if packed else "hht_set_leaf_sink, 20-byte rows") +
                         "), summed over the steps" +
                         ("; L2 flushed before each call, outside its clock" if flush else "")}

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        smp = None
        try:
            smp = OracleSampler(cfg, pts, offs)
            cpu = _cpu_baseline(smp, a.oracle_steps)
            cpu.pop("seconds", None)
            cpu.pop("tests", None)
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": UNIT, "cores": None, "kind": "oracle", "sample": f"failed: {e}"}
        finally:
            if smp is not None:
                smp.close()

    if rank == 0:
        wl = _workload(cfg)
        wl["points_per_image"] = int(offs[1] - offs[0])
        if a.variant == "fht":
            wl["variant"] = "FHT circumcircle membership test (comparison, PAPER.md:45)"
        wl["parallelism"] = (f"points sharded x{world}, per-level NCCL allreduce" if comm_world > 1 else
                             (f"images sharded x{world}" if world > 1 else "single GPU"))
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
                "warmup": a.warmup, "ms_per_step": ms_per_step, "ms_per_image": ms_per_step / images,
                "higher_is_better": True, "scaling": "weak" if cfg.images > 1 else "strong",
                "vs_baseline": None, "dtype": "int32" if st["int_bits"] == 32 else "int64",
                "data": "synthetic (seeded generator, paper_1007_0547_b200/synth.py)", "config": wl,
                "tests_per_step": tests_tot / a.steps, "votes_per_step": st["votes"],
                "leaves_per_step": st["leaves"], "pairs_per_step": st["pairs"], "ranges": st["ranges"],
                "clocks": clocks, "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches,
                "kernel_ms": {k: v["ms"] / a.steps for k, v in prof_tot.items()}}
        print(json.dumps(line), flush=True)
    h.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
