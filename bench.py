#!/usr/bin/env python
"""bench.py — lower bounds/sec on Taillard 200x20 pools (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config ta091] [--pool NODES_PER_GPU] [--no-e2e] [--no-bb]
  python bench.py --table2     (the paper's Table II protocol on B&B frontier pools)

One step = one fsp_lb_eval over the whole per-GPU pool (every row a1-a5 of
SURVEY.md §8(a) runs inside the kernel), pool resident in HBM.  Under torchrun
each rank bounds its own pool (weak scaling, no data-path collective); the
reported time is the max over ranks.  Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_1208_3933_b200 import inputs  # noqa: E402

METRIC = "lower bounds/sec on Taillard 200x20 pools"
UNIT = "bounds/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="ta091")
    ap.add_argument("--pool", type=int, default=1 << 20)
    ap.add_argument("--strong-total", type=int, default=0,
                    help="strong scaling: ranks bound contiguous shards of ONE pool of this "
                         "many nodes (SURVEY.md §8(d) C4: 4M total) instead of 1M each")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-bb", action="store_true")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the other BASELINE configs' bounds/s (bench key other_configs)")
    ap.add_argument("--bb-seconds", type=float, default=10.0)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--table2", action="store_true",
                    help="Table II grid: Tcpu/Tgpu per instance class and pool size")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload(cfg, pool, world):
    n, m, seed = inputs.TAILLARD_SEEDS[cfg]
    return {
        "workload": f"{cfg}-class {n}x{m} tai-gen(seed {seed}), D1 pool {pool} nodes/GPU",
        "instance": cfg, "n": n, "m": m, "pool_per_gpu": pool, "total_pool": pool * world,
        "stride": inputs.default_stride(n), "pool_recipe": "D1 (DESIGN.md §5)",
        "l2": "inputs exceed L2 (prefix pool > 126 MB), no flush needed"
        if pool * inputs.default_stride(n) * 2 > 126e6 else "pool fits L2: L2 flushed between steps",
        "parallelism": f"pool-sharded x{world}",
    }


def algorithmic_ops(n, m, depth):
    """Sum over the pool of W(d) (= fsp_lb_work per node)."""
    P = m * (m - 1) // 2
    d = depth.astype(np.int64)
    npr = n - d
    return int((2 * d * m + npr * (3 * m - 2) + npr * m + P * n + 4 * P * npr + 2 * P).sum())


# ALU-pipe throughput measured on this pool's B200 by tools/ubench/ipipe.cu
# (profiles/r02/ipipe_b200.txt): VIMNMX / VIMNMX.U16x2 0.496 warp-instructions
# per clock per SMSP (VIADDMNMX.U16x2 0.462 with the loop's own IADD in the
# same pipe), i.e. the ALU pipe is half rate: 64 lane-ops/clk/SM.
ALU_PIPE_WARP_INSTR_PER_CLK_SMSP = 0.496


def alu_peak_tops():
    """Roofline denominator: the measured ALU-pipe rate x 2
    algorithmic ops per fused max-plus instruction (VIADDMNMX: add + max) x 32
    lanes x 4 SMSPs x 148 SMs at the max SM clock (MEASURED_PEAKS.json).
    Also returns the issue ceiling (1 warp-instruction/clk/SMSP) in lane-instr/s
    and the ALU-pipe ceiling in lane-instr/s."""
    mhz = 1965.0
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mhz = float(json.load(f).get("sm_max_mhz", mhz))
    except Exception:
        pass
    lanes = 148 * 4 * 32 * mhz * 1e6
    alu = lanes * ALU_PIPE_WARP_INSTR_PER_CLK_SMSP
    return 2 * alu / 1e12, mhz, lanes / 1e12, alu / 1e12


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[1]))
                mx = float(r[2])
                for nm, v in zip(names, r[5:9]):
                    if v.lower().startswith("active"):
                        reasons.add(nm)
            except Exception:
                continue
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def ncu_traffic(cfg):
    """dram read+write bytes per launch of the lb kernel from the committed
    ncu --set full summary (profiles/), if one exists for this workload."""
    p = os.path.join(ROOT, "profiles", "lb_kernel_ncu.json")
    try:
        with open(p) as f:
            d = json.load(f)
        if d.get("instance") == cfg:
            return d.get("dram_bytes_per_launch"), d
    except Exception:
        pass
    return None, None


def schedule_makespan(ptm, perm):
    """C_max of a complete schedule, to check a returned optimum."""
    C = np.zeros(ptm.shape[1], np.int64)
    for j in perm:
        prev = 0
        for k in range(ptm.shape[1]):
            C[k] = max(C[k], prev) + int(ptm[j, k])
            prev = C[k]
    return int(C[-1])


def cpu_oracle_rate(ptm, pf, dp, seconds, threads=None):
    """The oracle as it stands on the host cores: contiguous chunks of a
    bounded sample, one ctypes call per thread (the C code releases the GIL)."""
    import oracle
    T = oracle.Tables(ptm)
    threads = threads or len(os.sched_getaffinity(0))
    # size the sample from a 1-thread probe
    probe = min(len(dp), 64)
    t0 = time.perf_counter()
    T.lb_eval(pf[:probe], dp[:probe])
    per_node = (time.perf_counter() - t0) / probe
    S = int(min(len(dp), max(threads * 8, seconds * threads / max(per_node, 1e-9))))
    chunks = np.array_split(np.arange(S), threads)
    res = [None] * threads

    def work(i):
        idx = chunks[i]
        res[i] = T.lb_eval(pf[idx[0]:idx[-1] + 1], dp[idx[0]:idx[-1] + 1]) if len(idx) else None

    t0 = time.perf_counter()
    ths = [threading.Thread(target=work, args=(i,)) for i in range(threads)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    dt = time.perf_counter() - t0
    return S / dt, threads, S, dt


def run_reference(a):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cfg = a.config
    n, m, seed = inputs.TAILLARD_SEEDS[cfg]
    ptm = inputs.taillard(n, m, seed)
    pf, dp = inputs.pool_d1(n, min(a.pool, 200_000), inputs.pool_seed(cfg))
    import oracle
    T = oracle.Tables(ptm)
    threads = len(os.sched_getaffinity(0))
    # per-step sample: ~4 s of CPU work on all cores
    rate_probe, _, _, _ = cpu_oracle_rate(ptm, pf, dp, 1.0, threads)
    S = int(max(threads, min(len(dp), rate_probe * 4.0)))
    chunks = np.array_split(np.arange(S), threads)

    def step():
        def work(i):
            idx = chunks[i]
            if len(idx):
                T.lb_eval(pf[idx[0]:idx[-1] + 1], dp[idx[0]:idx[-1] + 1])
        ths = [threading.Thread(target=work, args=(i,)) for i in range(threads)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()

    for _ in range(a.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(a.steps):
        step()
    dt = time.perf_counter() - t0
    value = S * a.steps / dt
    cfgd = workload(cfg, a.pool, world)
    out = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": dt / a.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic", "config": cfgd,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
                         "sample": f"first {S} nodes of the D1 pool per step"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


TABLE2_SIZES = [4096, 8192, 16384, 32768, 65536, 131072, 262144, 1048576, 4194304]
TABLE2_CFGS = ["ta021", "ta051", "c100x20", "ta091"]


def frontier(binding, inst, n, seconds=5.0):
    """The paper's list L: open sub-problems of a running B&B.  The
    device B&B runs from the root for a fixed time box (incumbent-less start,
    deepest-first batches) and its open nodes are exported (fsp_bb_export) as
    the list: every depth the search holds open, shallow to deep."""
    import torch
    bb = binding.BBState(inst)
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < seconds and bb.pool_size() > 0:
        bb.step(8)
    k = bb.pool_size()
    nb = bb.node_bytes()
    buf = torch.empty(max(1, k) * nb, dtype=torch.uint8, device="cuda")
    k = bb.export(k, buf.data_ptr())
    stride = (n + 7) & ~7
    h = buf[: k * nb].cpu().numpy()[8 * k:]  # export layout: [k] i64 last key first
    pf = h[: k * stride * 2].view(np.uint16).reshape(k, stride).copy()
    dp = h[k * stride * 2: k * stride * 2 + 4 * k].view(np.int32).copy()
    st = bb.stats()
    bb.close()
    return pf, dp, st


def run_table2(a):
    """Table II of the paper on B200: for each instance class and pool
    size, Tcpu/Tgpu of bounding a pool of sub-problems drawn from a B&B frontier.
    Tcpu: the oracle on ONE host core (the paper's serial B&B core), timed on a
    bounded sample and scaled per node; Tgpu: fsp_lb_eval_host (the paper's
    offload: host pool -> GPU -> host LBs, copies timed) and fsp_lb_eval (pool
    resident in HBM).  The sampled LBs are checked against the oracle."""
    import torch

    import oracle
    from paper_1208_3933_b200 import binding
    rows = []
    for cfg in TABLE2_CFGS:
        n, m, seed = inputs.TAILLARD_SEEDS[cfg]
        ptm = inputs.taillard(n, m, seed)
        inst = binding.Instance(ptm)
        pfL, dpL, st = frontier(binding, inst, n)
        # a random order of the list (seeded): every pool mixes its depths
        perm = np.random.default_rng(12083933).permutation(len(dpL))
        pfL, dpL = pfL[perm], dpL[perm]
        L = len(dpL)
        T = oracle.Tables(ptm)
        # Tcpu per node: one core, a sample of the list (same depth mix)
        samp = np.arange(min(L, 2048))
        t0 = time.perf_counter()
        ref = T.lb_eval(pfL[samp], dpL[samp])
        cpu_node = (time.perf_counter() - t0) / len(samp)
        best = None
        for S in TABLE2_SIZES:
            idx = np.arange(S) % L  # the list, cycled when shorter than S
            pf, dp = np.ascontiguousarray(pfL[idx]), np.ascontiguousarray(dpL[idx])
            stride = pf.shape[1]
            h_pf = torch.from_numpy(pf.view(np.int16)).pin_memory()
            h_dp = torch.from_numpy(dp).pin_memory()
            h_lb = torch.empty(S, dtype=torch.int32).pin_memory()
            d_pf, d_dp = h_pf.cuda(), h_dp.cuda()
            d_lb = torch.empty(S, dtype=torch.int32, device="cuda")
            reps = max(3, min(200, (1 << 22) // S))
            for _ in range(2):
                inst.lb_eval_host_ptr(h_pf.data_ptr(), stride, h_dp.data_ptr(), S, h_lb.data_ptr())
                inst.lb_eval(d_pf, d_dp, d_lb)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(reps):
                inst.lb_eval_host_ptr(h_pf.data_ptr(), stride, h_dp.data_ptr(), S, h_lb.data_ptr())
            t_host = (time.perf_counter() - t0) / reps
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            for _ in range(reps):
                inst.lb_eval(d_pf, d_dp, d_lb)
            e1.record()
            torch.cuda.synchronize()
            t_dev = e0.elapsed_time(e1) / reps / 1e3
            k = min(S, len(samp))
            if not (np.array_equal(h_lb.numpy()[:k], ref[:k]) and torch.equal(h_lb, d_lb.cpu())):
                raise SystemExit(f"table2: GPU LBs differ from the oracle ({cfg}, pool {S})")
            tcpu = cpu_node * S
            row = {"instance": f"{cfg}-class {n}x{m}", "pool": S, "blocks_x_256": f"{S // 256}x256",
                   "list_nodes": L, "mean_depth": float(dpL[idx].mean()),
                   "tcpu_ms_1core": tcpu * 1e3, "tgpu_ms_offload": t_host * 1e3,
                   "tgpu_ms_resident": t_dev * 1e3, "tcpu_over_tgpu_offload": tcpu / t_host,
                   "tcpu_over_tgpu_resident": tcpu / t_dev, "bounds_per_s_offload": S / t_host,
                   "bounds_per_s_resident": S / t_dev}
            print(json.dumps(row), flush=True)
            rows.append(row)
            if best is None or row["tcpu_over_tgpu_offload"] > best[1]:
                best = (S, row["tcpu_over_tgpu_offload"])
        # the runtime choice the paper asks for: fsp_lb_tune_pool
        tuned, rates = inst.tune_pool(22, 0.95)
        print(json.dumps({"instance": f"{cfg}-class {n}x{m}", "best_pool_offload": best[0],
                          "best_tcpu_over_tgpu_offload": best[1], "bb_iterations_for_list":
                          st.get("iterations"), "runtime_pool_95pct": tuned,
                          "tuned_rates_bounds_per_s": {str(k): v for k, v in rates.items()}}),
              flush=True)
        inst.close()
    return rows


def main():
    a = parse()
    if a.impl == "reference":
        return run_reference(a)
    if a.table2:
        return run_table2(a)
    import torch
    import torch.distributed as dist

    from paper_1208_3933_b200 import binding

    rank, world, local = dist_env()
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device")
    # one process per GPU over NCCL; FSP_BENCH_BACKEND=gloo runs the same
    # multi-rank control flow with host-side collectives (testing on one GPU)
    backend = os.environ.get("FSP_BENCH_BACKEND", "nccl")
    comm = "cuda" if backend == "nccl" else "cpu"
    ndev = torch.cuda.device_count()
    if world > ndev and "FSP_BB_MEM_FRAC" not in os.environ:
        # ranks sharing a device split the B&B stack budget between them
        os.environ["FSP_BB_MEM_FRAC"] = str(0.4 / -(-world // ndev))
    local = local % ndev
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    cfg = a.config
    n, m, seed = inputs.TAILLARD_SEEDS[cfg]
    ptm = inputs.taillard(n, m, seed)
    if a.strong_total > 0:
        # strong scaling: rank r bounds nodes [lo, hi) of one seeded pool
        from paper_1208_3933_b200 import dist as fdist
        lo, hi = fdist.shard(a.strong_total, rank, world)
        a.pool = hi - lo
        pf, dp = inputs.pool_d1(n, a.pool, inputs.pool_seed(cfg), first=lo)
    else:
        pf, dp = inputs.pool_d1(n, a.pool, inputs.pool_seed(cfg) + 1000 * rank)
    stride = pf.shape[1]
    inst = binding.Instance(ptm)
    d_pf = torch.from_numpy(pf.view(np.int16)).cuda()
    d_dp = torch.from_numpy(dp).cuda()
    d_lb = torch.empty(a.pool, dtype=torch.int32, device="cuda")
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(max(a.warmup, 3)):
        inst.lb_eval(d_pf, d_dp, out=d_lb, stream=stream)
    torch.cuda.synchronize()
    if inst.check() != binding.FSP_OK:
        raise SystemExit("malformed node in bench pool")

    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(a.steps):
            inst.lb_eval(d_pf, d_dp, out=d_lb, stream=stream)
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], dtype=torch.float64, device=comm)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    total_nodes = a.strong_total if a.strong_total > 0 else a.pool * world
    value = total_nodes * a.steps / (ms_max / 1e3)

    # roofline: algorithmic integer ops per launch / mean launch time
    ops = algorithmic_ops(n, m, dp)
    peak, mhz, issue_peak, alu_pipe_peak = alu_peak_tops()
    achieved = ops / (ms / a.steps / 1e3) / 1e12
    traffic, _ = ncu_traffic(cfg)

    # e2e through the C ABI with pinned HOST buffers (copies inside the timed region)
    e2e = None
    if not a.no_e2e:
        h_pf = torch.from_numpy(pf.view(np.int16)).pin_memory()
        h_dp = torch.from_numpy(dp).pin_memory()
        h_lb = torch.empty(a.pool, dtype=torch.int32).pin_memory()
        inst.lb_eval_host_ptr(h_pf.data_ptr(), stride, h_dp.data_ptr(), a.pool, h_lb.data_ptr())
        barrier()
        t0 = time.perf_counter()
        for _ in range(a.steps):
            inst.lb_eval_host_ptr(h_pf.data_ptr(), stride, h_dp.data_ptr(), a.pool,
                                  h_lb.data_ptr())
        dt = time.perf_counter() - t0
        tt = torch.tensor([dt], dtype=torch.float64, device=comm)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dt = float(tt.item())
        if not torch.equal(h_lb, d_lb.cpu()):
            raise SystemExit("host-API LBs differ from device LBs")
        # bytes that cross PCIe per step: the zero-copy gather (pinned buffers)
        # reads each node's depth and its first ceil(d/8) 16-byte vectors of
        # prefix, not the row padding (api.cu gather_rows_kernel)
        gathered = int(((np.minimum(dp, stride).astype(np.int64) + 7) // 8 * 16).sum()) + int(dp.nbytes)
        e2e = {"value": total_nodes * a.steps / dt, "unit": UNIT,
               "h2d_bytes_per_step": gathered,
               "h2d_note": "zero-copy gather of each node's depth and 2*depth prefix bytes "
                           f"(the pinned pool is {int(pf.nbytes + dp.nbytes)} bytes with row padding)",
               "d2h_bytes_per_step": int(a.pool * 4)}

    # the other BASELINE.json configs (driver-visible, same run, device-timed):
    # 1M-node D1 pools (500x20 pools to 2^20)
    other = None
    if not a.no_configs and world == 1 and a.strong_total == 0:
        other = {}
        for cfg2, pool2 in (("ta001", 1 << 20), ("ta021", 1 << 20), ("ta051", 1 << 20),
                            ("ta111", 1 << 20)):
            if cfg2 == cfg:
                continue
            n2, m2, seed2 = inputs.TAILLARD_SEEDS[cfg2]
            pf2, dp2 = inputs.pool_d1(n2, pool2, inputs.pool_seed(cfg2))
            i2 = binding.Instance(inputs.taillard(n2, m2, seed2))
            g_pf = torch.from_numpy(pf2.view(np.int16)).cuda()
            g_dp = torch.from_numpy(dp2).cuda()
            g_lb = torch.empty(pool2, dtype=torch.int32, device="cuda")
            for _ in range(3):
                i2.lb_eval(g_pf, g_dp, out=g_lb, stream=stream)
            k2 = 10
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(stream)
            for _ in range(k2):
                i2.lb_eval(g_pf, g_dp, out=g_lb, stream=stream)
            e1.record(stream)
            torch.cuda.synchronize()
            if i2.check() != binding.FSP_OK:
                raise SystemExit(f"malformed node in the {cfg2} pool")
            t2 = e0.elapsed_time(e1) / k2 / 1e3
            ops2 = algorithmic_ops(n2, m2, dp2)
            other[cfg2] = {"workload": f"{cfg2}-class {n2}x{m2}, D1 pool {pool2}",
                           "bounds_per_s": pool2 / t2, "ms_per_pool": t2 * 1e3,
                           "roofline_frac": ops2 / t2 / 1e12 / peak,
                           "launch": i2.launch_info(pool2)}
            del g_pf, g_dp, g_lb
            i2.close()

    bb = None
    if not a.no_bb:
        # B&B nodes/sec (BASELINE.json metric, second half): a time-boxed device
        # B&B on the same instance from the root, incumbent shared by NCCL
        # MIN all-reduce and work stealing across ranks when N > 1
        try:
            from paper_1208_3933_b200 import dist as fdist
            if world == 1:
                # the step API in a host loop so the incumbent trajectory (SURVEY.md
                # §8(d) C4) is recorded; each step is one device iteration
                state = binding.BBState(inst)
                traj = []
                t_start = time.perf_counter()
                best = 2**31 - 1
                while state.pool_size() > 0:
                    state.step(1)
                    el = time.perf_counter() - t_start
                    inc = state.ub_get() >> 32
                    if inc < best:
                        best = inc
                        traj.append([round(el, 4), int(inc), int(state.stats()["bounded"])])
                    if el >= a.bb_seconds:
                        break
                wall = time.perf_counter() - t_start
                st = state.stats()
                done = state.pool_size() == 0
                rcb, msp, permb = state.result()
                if rcb == 0 and schedule_makespan(ptm, permb) != msp:
                    raise SystemExit("B&B incumbent does not match its schedule")
                bb = {"bounded_nodes_per_s": st["bounded"] / max(wall, 1e-9),
                      # per-node roofline of the B&B: Fig. 3 operations of every
                      # bounded child (fsp_lb_work at its depth) per second of the
                      # whole search (branching, compaction included) / the peak
                      "roofline_frac_of_search": st["lb_ops"] / max(wall, 1e-9) / 1e12 / peak,
                      "status": 0 if done and rcb == 0 else (-6 if rcb == 0 else int(rcb)),
                      "incumbent": msp, "incumbent_verified": rcb == 0,
                      "ub_trajectory_s_ub_bounded": traj,
                      **{k: v for k, v in st.items() if k != "wall_s"}, "wall_s": wall}
                state.close()
            else:
                state = binding.BBState(inst, 2**31 - 1, rank, world)
                eng = fdist.DeviceEngine(state, "cuda", comm)
                barrier()
                res = fdist.distributed_bb(eng, dist, rank=rank, world=world, device=comm,
                                           sync_every=8, time_limit_s=a.bb_seconds)
                bb = {"bounded_nodes_per_s": res.bounded / max(res.wall_s, 1e-9),
                      "status": res.status, "incumbent": res.makespan, "bounded": res.bounded,
                      "rounds": res.rounds, "moved": res.moved, "wall_s": res.wall_s}
            bb["instance"] = cfg
            bb["time_box_s"] = a.bb_seconds
            if world == 1:
                # BASELINE.json configs[0]: full B&B of ta001 (20x5) from the root
                # to its optimum 1278, status and schedule checked here
                p2 = inputs.instance("ta001")
                i2 = binding.Instance(p2)
                rc2, ms2, perm2, st2 = i2.bb_solve(2**31 - 1, 0, 60.0)
                ok = (rc2 == 0 and ms2 == 1278 and sorted(perm2.tolist()) == list(range(20))
                      and schedule_makespan(p2, perm2) == ms2)
                bb["solve_20x5"] = {"instance": "ta001", "status": int(rc2),
                                    ("optimum" if rc2 == 0 else "incumbent"): ms2,
                                    "known_optimum": 1278, "verified": bool(ok),
                                    "wall_s": st2["wall_s"], "bounded": st2["bounded"],
                                    "iterations": st2["iterations"],
                                    "bounded_nodes_per_s": st2["bounded"] / max(st2["wall_s"], 1e-9)}
                i2.close()
        except Exception as ex:  # B&B is reported beside the metric, never instead of it
            bb = {"error": str(ex)[:200]}

    cpu = None
    if rank == 0:
        rate, cores, S, dt = cpu_oracle_rate(ptm, pf, dp, a.cpu_seconds)
        cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": f"first {S} nodes of the rank-0 D1 pool ({dt:.1f} s on {cores} threads)"}
        # the oracle on ONE core too (the paper's Tcpu)
        r1, _, S1, dt1 = cpu_oracle_rate(ptm, pf, dp, max(1.0, a.cpu_seconds / 4), threads=1)
        cpu["one_core"] = {"value": r1, "cores": 1,
                           "sample": f"first {S1} nodes ({dt1:.1f} s on 1 thread)"}

    if rank == 0:
        cfgd = workload(cfg, a.pool, world)
        if a.strong_total > 0:
            cfgd["total_pool"] = a.strong_total
            cfgd["workload"] = cfgd["workload"].replace(f"D1 pool {a.pool} nodes/GPU",
                                                        f"D1 pool {a.strong_total} nodes sharded")
        cfgd["launch"] = inst.launch_info(a.pool)
        info = inst.info
        cfgd["lb_kernel"] = {k: info[k] for k in ("groups", "pairs_per_group", "warps_per_cta",
                                                  "ctas_per_sm", "smem_bytes", "maxm")}
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": max(a.warmup, 3), "ms_per_step": ms_max / a.steps, "higher_is_better": True,
            "scaling": "strong" if a.strong_total > 0 else "weak", "vs_baseline": None,
            "dtype": "u16 (walk) / int32 (bounds)", "data": "synthetic",
            "config": cfgd,
            "roofline": {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "Top/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "peak_note": "measured ALU pipe (profiles/r02/ipipe_b200.txt: "
                                      f"{ALU_PIPE_WARP_INSTR_PER_CLK_SMSP} warp-instr/clk/SMSP) x 2 "
                                      "ops per fused VIADDMNMX x 148 SM x 4 SMSP x 32 lanes x "
                                      f"{mhz:.0f} MHz (DESIGN.md §7)",
                         "alu_pipe_peak_tlane_instr_s": alu_pipe_peak,
                         "issue_peak_tlane_instr_s": issue_peak,
                         "ops_per_launch": ops},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": a.steps, "other_configs": other,
            "clocks": clk.summary(), "bb": bb,
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
