#!/usr/bin/env python
"""bench.py -- playouts/s of the batched Da Vinci Code rollout (BASELINE.json
metric) on 1..8 B200, one process per GPU.

Workload (BASELINE configs[1], the N = 1 headline): C2 = 2 players, 24 tiles,
mid-game root `fixtures/c2_d1.json`, every legal action x 10^6 playouts per
action per GPU.  A step = one whole batch of the hot path (SURVEY §8(a) rows
a1-a5 in the rollout kernel, a6 = NCCL all_reduce of the int64 winner
histogram when N > 1).  Weak scaling: rank r plays sims [r*n, (r+1)*n) of every
action, so per-GPU work is fixed and the merged counts are those of N*n sims.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

Timing: W untimed warm-up steps; K timed steps, each bracketed by CUDA events
on the stream the kernels run on, an L2 flush (256 MiB write) between steps
outside the events; barrier + synchronize around the timed loop; the max over
ranks of the summed step time.  `e2e` times the public blocking call with host
buffers (encode + H2D of the state/actions + kernels + D2H of the histogram).
`--impl reference` times the oracle (oracle/, scalar C++) on the host cores.
"""

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOAD = "fixtures/c2_d1.json"
SIMS_PER_ACTION = 1_000_000
METRIC = "playouts/sec (1/2/4/8 B200) and warp exec efficiency vs CPU oracle"
UNIT = "playouts/s"


def load_workload(path=None):
    path = path or WORKLOAD
    with open(os.path.join(ROOT, path)) as f:
        return json.load(f)


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.dev = device_index
        self.rows = []          # (t, fields)
        self.proc = None
        self.window = None      # (t0, t1) of the timed region

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), "--query-gpu=" + self.Q, "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.perf_counter(), [x.strip() for x in line.split(",")]))

    def wait_first(self, timeout=5.0, load=None):
        """Block (running `load` to keep the GPU busy) until a first sample arrived."""
        t0 = time.perf_counter()
        while self.proc is not None and not self.rows and time.perf_counter() - t0 < timeout:
            if load is not None:
                load()
            else:
                time.sleep(0.01)

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = [r for t, r in self.rows]
        in_win = rows
        if self.window is not None:
            in_win = [r for t, r in self.rows if self.window[0] - 0.06 <= t <= self.window[1] + 0.06]
        note = "samples inside the timed region"
        if not in_win:
            # timed region shorter than the sampling period: the load-phase samples right around it
            in_win = rows[-3:]
            note = "timed region shorter than 50 ms sampling: last samples of the same load"
        rows = in_win
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(r[1]) for r in rows if r[1].replace(".", "").isdigit())
        mx = max((float(r[2]) for r in rows if r[2].replace(".", "").isdigit()), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            for i, n in enumerate(names):
                if len(r) > 5 + i and r[5 + i].lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(rows), "note": note}


# ----------------------------------------------------------------- helpers
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def instr_per_playout():
    """Per-unit algorithmic work of the dominant kernel: the
    thread-instructions per playout of the refill kernel on this workload,
    from the committed ncu capture (profiles/roofline_unit.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "roofline_unit.json")) as f:
            return json.load(f)
    except Exception:
        return None


def host_cpu_info():
    """The host the oracle runs on: CPU model, sockets, physical cores, logical
    CPUs, and one logical CPU per physical core (the pinning targets)."""
    model, topo = None, {}
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name") and model is None:
                model = line.split(":", 1)[1].strip()
    except OSError:
        pass
    try:
        allowed = sorted(os.sched_getaffinity(0))
    except AttributeError:
        allowed = list(range(os.cpu_count() or 1))
    for c in allowed:
        try:
            base = "/sys/devices/system/cpu/cpu%d/topology/" % c
            key = (open(base + "physical_package_id").read().strip(), open(base + "core_id").read().strip())
        except OSError:
            key = ("0", str(c))
        topo.setdefault(key, c)
    pin = sorted(topo.values())
    return {"model": model, "sockets": len({k[0] for k in topo}), "physical_cores": len(pin),
            "logical_cpus": os.cpu_count(), "allowed_cpus": len(allowed), "pin_cpus": pin,
            "oracle_build": "g++ -O2 -std=c++17 -shared -fPIC (scalar, no intrinsics; oracle/__init__.py)"}


def _pin_worker(counter, cpus):
    with counter.get_lock():
        i = counter.value
        counter.value += 1
    try:
        os.sched_setaffinity(0, {cpus[i % len(cpus)]})
    except (AttributeError, OSError):
        pass


class OraclePool:
    """The oracle, as it stands, on the host cores: one process pinned to each
    physical core (taskset-style sched_setaffinity), disjoint sim sub-ranges of
    the same workload (SURVEY §8(d) "all cores")."""

    def __init__(self, cores=None):
        from concurrent.futures import ProcessPoolExecutor
        import multiprocessing as mp
        import oracle
        oracle.build()
        self.info = host_cpu_info()
        cpus = self.info["pin_cpus"]
        self.cores = cores or len(cpus)
        ctx = mp.get_context("spawn")
        self.ex = ProcessPoolExecutor(max_workers=self.cores, mp_context=ctx, initializer=_pin_worker,
                                      initargs=(ctx.Value("i", 0), cpus))

    def calibrate(self, d, codes, seed, budget_s):
        """sims per core so one sample takes about budget_s / 4 of wall time."""
        list(self.ex.map(_oracle_job, [(d, codes, seed, 0, 1)] * self.cores))   # warm the workers
        t0 = time.perf_counter()
        n_cal = 200
        list(self.ex.map(_oracle_job, [(d, codes, seed, 0, n_cal)]))
        per_playout = (time.perf_counter() - t0) / (n_cal * len(codes))
        return max(1, int(budget_s / per_playout / len(codes) / 4))

    def run(self, d, codes, seed, per_core, offset=0):
        jobs = [(d, codes, seed, offset + i * per_core, offset + (i + 1) * per_core) for i in range(self.cores)]
        t0 = time.perf_counter()
        list(self.ex.map(_oracle_job, jobs))
        dt = time.perf_counter() - t0
        n = per_core * self.cores
        playouts = n * len(codes)
        return {"value": playouts / dt, "unit": UNIT, "cores": self.cores, "kind": "oracle", "wall_s": dt,
                "playouts": playouts,
                "sample": "%s, all %d actions x %d sims (%d playouts, %.1f s wall, one oracle process pinned to "
                          "each of %d physical cores, disjoint sim ranges)"
                          % (WORKLOAD, len(codes), n, playouts, dt, self.cores)}

    def close(self):
        self.ex.shutdown()


def _one_core_job(args):
    """SURVEY §8(d) 1-core protocol: one process pinned to one core, the first
    ceil(1e6 / A) sims of every action (~10^6 playouts), steady clock around
    the rollout loop (encode and the library load excluded)."""
    import oracle
    d, codes, seed, cpu = args
    try:
        os.sched_setaffinity(0, {cpu})
    except (AttributeError, OSError):
        pass
    oracle.rollout(d, codes, seed, 0, 0, 1)
    per = -(-1000000 // len(codes))
    t0 = time.perf_counter()
    oracle.rollout(d, codes, seed, 0, 0, per)
    return per * len(codes), time.perf_counter() - t0


def cpu_oracle_baseline(d, codes, seed, budget_s=15.0):
    pool = OraclePool()
    try:
        res = pool.run(d, codes, seed, pool.calibrate(d, codes, seed, budget_s))
        n1, t1 = pool.ex.submit(_one_core_job, (d, codes, seed, pool.info["pin_cpus"][0])).result()
        res["one_core"] = {"value": n1 / t1, "unit": UNIT, "playouts": n1, "wall_s": t1,
                           "sample": "first %d playouts of %s seed %d, one process pinned to cpu %d"
                                     % (n1, WORKLOAD, seed, pool.info["pin_cpus"][0])}
        res["host"] = pool.info
        return res
    finally:
        pool.close()


def _oracle_job(args):
    import oracle
    d, codes, seed, s0, s1 = args
    return oracle.rollout(d, codes, seed, 0, s0, s1)


# ----------------------------------------------------------------- reference arm
def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    d = load_workload()
    import oracle
    codes = oracle.legal(d)
    pool = OraclePool()
    per_core = pool.calibrate(d, codes, 1, args.ref_budget / 2)
    res = None
    times = []
    for step in range(args.warmup + args.steps):
        r = pool.run(d, codes, seed=1 + step, per_core=per_core)
        if step >= args.warmup:
            times.append(r)
        res = r
    pool.close()
    # value = all timed playouts / all timed wall time; ms_per_step = the
    # MEASURED wall time of one bounded sample step (not extrapolated to 10^6)
    wall = sum(r["wall_s"] for r in times)
    value = sum(r["playouts"] for r in times) / wall
    ms = 1000.0 * wall / len(times)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": "C2 mid-game root %s, all %d legal actions, bounded oracle sample per step"
                       % (WORKLOAD, len(codes)), "sims_per_action_per_step": per_core * pool.cores,
                       "playouts_per_step": res["playouts"],
                       "ms_per_step_note": "measured wall time of one bounded sample step",
                       "l2": "n/a (CPU)"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": res["cores"], "kind": "oracle",
                             "sample": res["sample"], "host": pool.info},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def run_reference_sweep(args):
    """The reference arm's sweeps for the paper's CPU experiments (driven by
    tools/paper_experiments.py, which never touches oracle/ itself); one JSON
    row per run, SPEC:370 columns:
      exp1: `--ref-sizes` total simulations over the C2 workload's actions
            (the first n mod A actions get one more), all host cores;
      exp2: simulations/s vs worker processes 1 .. 2 x cores."""
    from concurrent.futures import ProcessPoolExecutor
    import multiprocessing as mp
    import oracle
    oracle.build()
    d = load_workload()
    codes = oracle.legal(d)
    A = len(codes)
    cores = os.cpu_count() or 1

    def emit(run, workers, total, t_s):
        print(json.dumps({"run": run, "workers": workers, "total_simulations": total, "elapsed_ns": int(t_s * 1e9),
                          "sims_per_sec": total / t_s, "device": "cpu", "kernel": "oracle"}), flush=True)

    if args.ref_sweep == "core1":
        # SURVEY §8(d) protocol: one process pinned to one core, the first 10^6
        # playouts of the C2 workload (seed 1, all actions, sims [0, ceil(1e6/A)))
        per = -(-1000000 // A)
        try:
            os.sched_setaffinity(0, {sorted(os.sched_getaffinity(0))[0]})
        except (AttributeError, OSError):
            pass
        oracle.rollout(d, codes, 1, 0, 0, 1)                          # warm
        t0 = time.perf_counter()
        oracle.rollout(d, codes, 1, 0, 0, per)
        dt = time.perf_counter() - t0
        print(json.dumps({"run": -1, "workers": 1, "total_simulations": per * A, "elapsed_ns": int(dt * 1e9),
                          "sims_per_sec": per * A / dt, "device": "cpu", "kernel": "oracle",
                          "sample": "%s seed 1, %d actions x %d sims, one pinned core" % (WORKLOAD, A, per)}),
              flush=True)
        return 0
    if args.ref_sweep == "exp1":
        with ProcessPoolExecutor(max_workers=cores, mp_context=mp.get_context("spawn")) as ex:
            list(ex.map(_oracle_job, [(d, codes, 1, 0, 1)] * cores))          # warm the workers
            for n in [int(x) for x in args.ref_sizes.split(",")]:
                per, extra = divmod(n, A)
                ts = []
                for r in range(args.steps):
                    jobs = [(d, codes, 1 + r, (per * w) // cores, (per * (w + 1)) // cores) for w in range(cores)]
                    jobs = [j for j in jobs if j[4] > j[3]]
                    if extra:
                        jobs.append((d, codes[:extra], 1 + r, per, per + 1))
                    t0 = time.perf_counter()
                    list(ex.map(_oracle_job, jobs))
                    ts.append(time.perf_counter() - t0)
                    emit(r, cores, n, ts[-1])
                emit(-1, cores, n, sum(ts) / len(ts))
    else:
        n_per_worker = 4000
        for w in sorted({1, 2, 4, 8, 12, 16, 24, 32, cores, 2 * cores}):
            if w > 2 * cores:
                continue
            with ProcessPoolExecutor(max_workers=w, mp_context=mp.get_context("spawn")) as ex:
                list(ex.map(_oracle_job, [(d, codes[:1], 1, 0, 1)] * w))
                ts = []
                for r in range(args.steps):
                    jobs = [(d, codes[:4], 1 + r, i * n_per_worker, (i + 1) * n_per_worker) for i in range(w)]
                    t0 = time.perf_counter()
                    list(ex.map(_oracle_job, jobs))
                    ts.append(time.perf_counter() - t0)
                    emit(r, w, w * n_per_worker * 4, ts[-1])
                emit(-1, w, w * n_per_worker * 4, sum(ts) / len(ts))
    return 0


def all_reduce(t, op=None):
    """SUM (or `op`) all_reduce of a CUDA tensor: NCCL directly; a gloo group
    (BENCH_BACKEND=gloo: a functional test of the N > 1 path with several
    ranks sharing one GPU, never a measurement) reduces a host copy."""
    import torch
    import torch.distributed as dist
    op = dist.ReduceOp.SUM if op is None else op
    if dist.get_backend() == "nccl":
        dist.all_reduce(t, op=op)
    else:
        h = t.cpu()
        dist.all_reduce(h, op=op)
        t.copy_(h)
    return t


# ----------------------------------------------------------------- extra records
R01_INSTR_PER_PLAYOUT = 1987
C4_WORKLOAD = "fixtures/c4_d1.json"
C4_PLAYOUTS_PER_MOVE = 100_000_000


def c4_strong_record(args, ws, rank, dev, stream, moves=3, warmup=1):
    """BASELINE configs[3] (C4: 4 players, 26 tiles, 3 each, 10^8 playouts per
    move) as STRONG scaling: ceil(1e8 / A) sims per action split over the ws
    ranks (dist.shard_range), one NCCL all_reduce per move; ms per move = max
    over ranks of CUDA-event time (kernel + all_reduce).  Rank 0 recomputes
    the whole move alone and checks the merged histogram bit for bit; the
    histogram's sha256 must be the same at every N."""
    import hashlib
    import torch
    from paper_2403_10720_b200 import dvc
    from paper_2403_10720_b200.dist import shard_range
    d = load_workload(C4_WORKLOAD)
    st = dvc.encode(d)
    codes = st.legal_actions()
    A, P = len(codes), st.players
    S = -(-C4_PLAYOUTS_PER_MOVE // A)
    a, b = shard_range(S, rank, ws)
    hist = torch.zeros((A, P), dtype=torch.int64, device=dev)
    dvc.set_option("plan_cache", 1)        # the state's table is built once per move in a real search
    times = []
    for m in range(warmup + moves):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        hist.zero_()
        if b > a:
            dvc.rollout_batch_async(st, codes, 77, 0, a, b, hist, stream=stream)
        if ws > 1:
            all_reduce(hist)
        e1.record(stream)
        torch.cuda.synchronize()
        if m >= warmup:
            times.append(e0.elapsed_time(e1))
    dvc.set_option("plan_cache", 0)
    t = torch.tensor([sum(times) / len(times)], dtype=torch.float64, device=dev)
    if ws > 1:
        all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    ms = float(t[0])
    ok = None
    if rank == 0:
        full = torch.zeros_like(hist)
        dvc.rollout_batch_async(st, codes, 77, 0, 0, S, full, stream=stream)
        torch.cuda.synchronize()
        ok = bool(torch.equal(full, hist))
    h = hist.cpu()
    assert int(h.sum()) == A * S
    return {"workload": "C4 %s (4p, 26 tiles, 3 each, jokers, consecutive)" % C4_WORKLOAD, "actions": A,
            "sims_per_action": S, "playouts_per_move": A * S, "scaling": "strong", "moves": moves,
            "ms_per_move": ms, "playouts_per_s": A * S / (ms / 1000.0), "merge_bit_exact": ok,
            "hist_sha256": hashlib.sha256(h.numpy().tobytes()).hexdigest(),
            "note": "table cached per move (plan_cache=1); time = kernel + all_reduce, max over ranks"}


def c2_deals_record(dvc, torch, dev, stream, n, steps=5):
    """The headline is one position (c2_d1); the same batch on all eight C2
    deals (fixtures/c2_d1..8), device time per step, and their mean."""
    out = {}
    old_cache = dvc.get_option("plan_cache")
    dvc.set_option("plan_cache", 1)
    for k in range(1, 9):
        path = "fixtures/c2_d%d.json" % k
        st = dvc.encode(load_workload(path))
        codes = st.legal_actions()
        hist = torch.zeros((len(codes), st.players), dtype=torch.int64, device=dev)
        for w in range(2):
            dvc.rollout_batch_async(st, codes, 500 + w, 0, 0, n, hist, stream=stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(steps):
            dvc.rollout_batch_async(st, codes, 1 + i, 0, 0, n, hist, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize()
        out["c2_d%d" % k] = len(codes) * n * steps / (e0.elapsed_time(e1) / 1000.0)
    dvc.set_option("plan_cache", old_cache)
    vals = list(out.values())
    return {"playouts_per_s": out, "mean": sum(vals) / len(vals), "min": min(vals), "max": max(vals),
            "note": "all legal actions x %d sims per deal, %d steps, device time, plan cached" % (n, steps)}


# ----------------------------------------------------------------- product arm
def run_product(args):
    import torch
    from paper_2403_10720_b200 import dvc

    ws, rank, local = dist_env()
    if args.gpus != ws and ws > 1:
        print("warning: --gpus %d but WORLD_SIZE %d" % (args.gpus, ws), file=sys.stderr)
    backend = os.environ.get("BENCH_BACKEND", "nccl")
    if backend != "nccl":                # functional multi-rank test on one GPU
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        import torch.distributed as dist
        # NCCL INIT logging, so the run's log shows the communicator's rank
        # count -- on stderr, so stdout keeps the one JSON line
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    d = load_workload()
    st = dvc.encode(d)
    codes = st.legal_actions()
    A, P = len(codes), st.players
    n = args.sims
    s0, s1 = rank * n, (rank + 1) * n
    dvc.set_option("kernel", {"refill": 0, "naive": 1}[args.kernel])
    if args.block:
        dvc.set_option("block", args.block)
    dvc.set_option("plan_cache", 0)       # plan upload + det table rebuilt inside every step
    stream = torch.cuda.current_stream()
    hist = torch.zeros((A, P), dtype=torch.int64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)

    def one_step(seed, collective=True):
        hist.zero_()
        dvc.rollout_batch_async(st, codes, seed, 0, s0, s1, hist, stream=stream)
        if ws > 1 and collective:
            all_reduce(hist)

    for w in range(args.warmup):
        one_step(1000 + w)
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        # keep the GPU busy until the sampler's first reading -- rank-local
        # work only: each rank loops a different number of times, so a
        # collective here would pair up wrongly across ranks and deadlock
        clk.wait_first(load=lambda: (one_step(999, collective=False), torch.cuda.synchronize()))
        torch.cuda.synchronize()
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        dvc.launch_count(reset=True)
        t_win0 = time.perf_counter()
        for i in range(args.steps):
            flush.fill_(i)                                 # L2 flush, outside the events
            ev[i][0].record(stream)
            hist.zero_()
            kev[i][0].record(stream)
            dvc.rollout_batch_async(st, codes, 1 + i, 0, s0, s1, hist, stream=stream)
            kev[i][1].record(stream)
            if ws > 1:
                all_reduce(hist)
            ev[i][1].record(stream)
        torch.cuda.synchronize()
        launches = dvc.launch_count(reset=False)
        clk.window = (t_win0, time.perf_counter())
        time.sleep(0.06)
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    t_ms = sum(a.elapsed_time(b) for a, b in ev)
    k_ms = sum(a.elapsed_time(b) for a, b in kev) / args.steps
    t = torch.tensor([t_ms, k_ms], dtype=torch.float64, device=dev)
    if ws > 1:
        all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    t_ms, k_ms = float(t[0]), float(t[1])
    playouts_per_step = A * n * ws
    value = playouts_per_step * args.steps / (t_ms / 1000.0)
    assert int(hist.sum()) == playouts_per_step, "histogram does not account for every playout"
    # a6 check: the last step's merged histogram (seed K, sims [0, ws*n)) must
    # equal rank 0's recomputation of the whole range alone (keyed Philox +
    # integer sums: bit-identical for every N)
    merge_ok = None
    if rank == 0:
        full = torch.zeros_like(hist)
        dvc.rollout_batch_async(st, codes, args.steps, 0, 0, ws * n, full, stream=stream)
        torch.cuda.synchronize()
        merge_ok = bool(torch.equal(full, hist))
    c4 = c4_strong_record(args, ws, rank, dev, stream) if not args.no_c4 else None

    # ---- e2e through the public blocking API with host buffers
    e2e = None
    if ws == 1:
        dvc.set_option("plan_cache", 0)
        for w in range(2):
            dvc.rollout_batch_ex(dvc.encode(d), codes, 50 + w, 0, s0, s1)
        torch.cuda.synchronize()
        dvc.transfer_bytes(reset=True)
        t0 = time.perf_counter()
        ke = max(1, args.steps)
        for i in range(ke):
            st_i = dvc.encode(d)                               # host encode of the observation
            h = dvc.rollout_batch_ex(st_i, codes, 1 + i, 0, s0, s1)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        xfer = dvc.transfer_bytes()
        assert int(h.sum()) == A * n
        e2e = {"value": A * n * ke / dt, "unit": UNIT, "h2d_bytes_per_step": xfer[0] // ke,
               "d2h_bytes_per_step": xfer[1] // ke,
               "path": "dvc.encode + dvc_rollout_batch_ex (host in/out, blocking)",
               "bytes_note": "counted by the library (dvc_transfer_bytes): plan image upload + kernel parameter "
                             "blocks (H2D), histogram readback (D2H)"}
    else:
        from paper_2403_10720_b200 import dist as ddist
        torch.distributed.barrier()
        torch.cuda.synchronize()
        dvc.transfer_bytes(reset=True)
        t0 = time.perf_counter()
        for i in range(args.steps):
            h = ddist.rollout_batch(dvc.encode(d), codes, n * ws, 1 + i)   # returns host int64 [A, P]
        dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        all_reduce(dt, op=torch.distributed.ReduceOp.MAX)
        xb = dvc.transfer_bytes()
        e2e = {"value": A * n * ws * args.steps / float(dt[0]), "unit": UNIT,
               "h2d_bytes_per_step": xb[0] // args.steps, "d2h_bytes_per_step": xb[1] // args.steps + 8 * A * P,
               "path": "dvc.encode + dist.rollout_batch (sharded async + NCCL all_reduce + .cpu())",
               "bytes_note": "rank 0's library-counted H2D (plan image + kernel parameter blocks) and D2H, plus "
                             "the merged histogram's .cpu() copy"}

    if rank == 0:
        pk = peaks()
        unit = instr_per_playout()
        sm_max = float(pk.get("sm_max_mhz", 1965.0))
        n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
        peak = n_sm * 4 * 32 * sm_max * 1e6 / 1e12          # tera thread-instructions / s
        roof = {"bound": "alu", "peak": peak, "unit": "Tinst/s", "traffic": None,
                "peak_note": "issue peak = %d SM x 4 SMSP x 32 lanes x %.0f MHz (MEASURED_PEAKS sm_max_mhz)"
                             % (n_sm, sm_max)}
        kernel_s = k_ms / 1000.0
        if unit and unit.get("workload") == WORKLOAD:
            ipp = float(unit["thread_inst_per_playout"])
            roof["achieved"] = ipp * A * n / kernel_s / 1e12
            roof["frac"] = roof["achieved"] / peak
            # F counts the kernel's OWN instructions, so it falls when a change
            # removes instructions; beside it, the fraction with the work per
            # playout frozen at round 1's 1987 (a fixed unit: cutting
            # instructions shows up as progress)
            roof["frac_fixed_unit"] = R01_INSTR_PER_PLAYOUT * A * n / kernel_s / 1e12 / peak
            roof["fixed_unit"] = "%d thread-instructions per playout (round-1 refill kernel, " \
                                 "profiles/r01_refill_c2_ncu.json)" % R01_INSTR_PER_PLAYOUT
            roof["per_unit"] = "%.0f thread-instructions per playout (%s)" % (ipp, unit.get("source", ""))
            roof["traffic"] = unit.get("dram_bytes_per_launch")
            # the same capture's view of the binding unit: the ALU pipe runs at
            # half the issue rate (LOP3/SHF/ISETP/SEL..., 16 lanes/clk/SMSP)
            roof["ncu"] = {k: unit.get(k) for k in ("eta_simt", "issue_active_pct", "pipe_alu_pct", "pipe_xu_pct",
                                                    "pipe_fma_pct")}
        else:
            roof["achieved"] = None
            roof["frac"] = None
            roof["per_unit"] = "missing profiles/roofline_unit.json"
        roof["kernel_ms"] = k_ms
        deals = c2_deals_record(dvc, torch, dev, stream, n) if (ws == 1 and not args.no_deals) else None
        cpu = None
        if not args.no_cpu_baseline and ws == 1:
            try:
                cpu = cpu_oracle_baseline(d, codes, seed=1, budget_s=args.ref_budget)
            except Exception as e:  # the baseline must not kill the bench line
                cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "oracle", "sample": "failed: %s" % e}
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
                "config": {"workload": "C2 mid-game root %s (2p, 24 tiles, consecutive), all %d legal actions x "
                                       "%d playouts per action per GPU" % (WORKLOAD, A, n),
                           "kernel": args.kernel, "sims_per_action_per_gpu": n, "actions": A,
                           "l2": "flushed between steps (256 MiB write)", "seeds": "1..K",
                           "det_table": "rebuilt every step (plan_cache=0)", "parallelism": "sim-range dp%d" % ws},
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
                "merge_bit_exact": merge_ok, "c4_strong": c4, "c2_deals": deals,
                "clocks": clk.summary()}
        print(json.dumps(line))
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="product", choices=["product", "reference"])
    ap.add_argument("--kernel", default="refill", choices=["refill", "naive"])
    ap.add_argument("--sims", type=int, default=SIMS_PER_ACTION)
    ap.add_argument("--ref-budget", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c4", action="store_true", help="skip the C4 strong-scaling record")
    ap.add_argument("--block", type=int, default=0, help="experiments only: refill block size (0 = default)")
    ap.add_argument("--no-deals", action="store_true", help="skip the 8-deal C2 record")
    ap.add_argument("--ref-sweep", choices=["core1", "exp1", "exp2"], default=None,
                    help="reference arm: the paper's CPU experiment sweeps (tools/paper_experiments.py)")
    ap.add_argument("--ref-sizes", default="1,10,100,1000,10000,100000,1000000")
    ap.add_argument("--workload", default=None,
                    help="experiments only: another fixture for the timed batch (the bench line is C2)")
    args = ap.parse_args()
    if args.workload:
        global WORKLOAD
        WORKLOAD = args.workload
    if args.impl == "reference":
        return run_reference_sweep(args) if args.ref_sweep else run_reference(args)
    return run_product(args)


if __name__ == "__main__":
    sys.exit(main())
