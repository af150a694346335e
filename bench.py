"""FlashOptim B200 benchmark (BASELINE.json metric: optimizer-step Gparams/s
and HBM GB/s (% of peak), Llama-3.1-8B FlashAdamW).

A "step" is one fused FlashAdamW pass over the whole Llama-3.1-8B-shaped
parameter list (291 tensors, 8,030,261,248 params; random valid state,
synthetic bf16 grads), state resident in HBM.  The working set (57 GB) is
~450x the 126 MB L2, so no L2 flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config llama31_8b|gpt2_medium|resnet50] [--optimizer adamw|sgd|lion]

N = 1: the fused multi-tensor step over the list (flat.StepPlan, one
launch per 384 tensors + its fix-up launch).  N > 1 (torchrun, NCCL): the
product ZeRO-1 optimizer (zero.ZeroFlashOptimizer) over the same list;
`value` is the step-only throughput (all params / slowest rank's sharded
step), the reduce-scatter, all-gather and full-step times sit beside it.

After the timed region one more step is checked against the C oracle on 64
windows of up to 1M elements spread over all tensors (`parity`), and the
fix-up launches' share of the slices is reported (`fast_path`).

--impl reference times the reference's own CPU implementation -- the
unmodified NumPy `flashopt.optim.*_step` installed in baseline/_ref -- on
all host cores (one process per core) over a bounded sample of the same
workload; it never touches the GPU.  Without baseline/_ref it falls back to
the C restatement (oracle/, kind "port").
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
REF_PATH = os.path.join(ROOT, "baseline", "_ref")

BYTES_PER_PARAM = {"adamw": 12.25, "sgd": 10.125, "lion": 10.125}
HP = {  # per-config hyper-parameters
    "llama31_8b": {"adamw": dict(lr=1e-5, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.1)},
    "gpt2_medium": {"adamw": dict(lr=6e-4, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.1)},
    "resnet50": {"sgd": dict(lr=1.024, momentum=0.9, weight_decay=3e-5),
                 "lion": dict(lr=2e-4, beta1=0.9, beta2=0.95, weight_decay=0.0),
                 "adamw": dict(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0)},
}
METRIC = "optimizer-step Gparams/s and HBM GB/s (% of peak), Llama-3.1-8B FlashAdamW"
DTYPE = "f32 math on bf16/i8/u8/f16 storage"


def peaks() -> tuple[float, str]:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def hparams_for(config: str, opt: str) -> dict:
    d = HP.get(config, {})
    if opt in d:
        return d[opt]
    return HP["resnet50"][opt]


def dist_env() -> tuple[int, int, int]:
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ---------------------------------------------------------------------------
# clocks / power during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks / power / throttle reasons sampled every 50 ms during
    the timed region.  start() returns once the first sample has arrived, so
    the samples cover the timed steps rather than nvidia-smi's start-up."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines: list[str] = []
        self.mark = 0

    def start(self):
        import threading

        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return

        def pump():
            for line in self.proc.stdout:
                self.lines.append(line)

        threading.Thread(target=pump, daemon=True).start()
        t = time.time()
        while not self.lines and time.time() - t < 10:
            time.sleep(0.02)

    def begin(self):
        """Mark the start of the timed region (samples before it are dropped)."""
        self.mark = len(self.lines)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.06)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=10)
        except Exception:
            pass
        lines = self.lines[self.mark:] or self.lines[-1:]
        sms, maxs, pw, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in lines:
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sms.append(float(f[1]))
                maxs.append(float(f[2]))
                pw.append(float(f[3]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        sms.sort()
        pw.sort()
        return {"sm_mhz": sms[len(sms) // 2] if sms else None, "sm_max_mhz": max(maxs) if maxs else None,
                "power_w": pw[len(pw) // 2] if pw else None, "reasons": sorted(reasons), "samples": len(sms)}


class PowerSampler:
    """NVML at 10 ms: instantaneous board power (NVML_FI_DEV_POWER_INSTANT,
    not nvidia-smi's 1 s average), SM clock and the clock-event reasons --
    the evidence for or against the power-cap explanation of the SM clock."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake", 0x1: "gpu_idle"}

    def __init__(self, gpu_index: int, interval_s: float = 0.01):
        self.gpu, self.dt = gpu_index, interval_s
        self.samples: list[tuple[float, float, int, float]] = []
        self.mark = 0
        self._stop = False
        self.ok = False

    def start(self):
        import threading

        try:
            import pynvml as N

            N.nvmlInit()
            self.N = N
            self.h = N.nvmlDeviceGetHandleByIndex(self.gpu)
            self.ok = True
        except Exception:
            return

        def run():
            N = self.N
            while not self._stop:
                try:
                    fv = N.nvmlDeviceGetFieldValues(self.h, [N.NVML_FI_DEV_POWER_INSTANT])[0]
                    pw = (fv.value.uiVal if fv.nvmlReturn == 0 else 0) / 1000.0
                    clk = N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM)
                    rs = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                    self.samples.append((time.perf_counter(), pw, int(rs), float(clk)))
                except Exception:
                    pass
                time.sleep(self.dt)

        self.th = threading.Thread(target=run, daemon=True)
        self.th.start()

    def begin(self):
        self.mark = len(self.samples)

    def stop(self) -> dict | None:
        if not self.ok:
            return None
        self._stop = True
        self.th.join(timeout=5)
        s = self.samples[self.mark:]
        if not s:
            return None
        pw = sorted(x[1] for x in s)
        clk = sorted(x[3] for x in s)
        seen: dict = {}
        for x in s:
            for bit, nm in self.REASONS.items():
                if x[2] & bit:
                    seen[nm] = seen.get(nm, 0) + 1
        q = lambda v, f: v[min(len(v) - 1, int(f * len(v)))]  # noqa: E731
        return {"source": "NVML field POWER_INSTANT + SM clock + clock-event reasons, 10 ms",
                "samples": len(s), "span_s": round(s[-1][0] - s[0][0], 3),
                "power_w": {"median": q(pw, 0.5), "p95": q(pw, 0.95), "max": pw[-1]},
                "sm_mhz": {"median": q(clk, 0.5), "min": clk[0], "max": clk[-1]},
                "reasons_fraction": {k: round(v / len(s), 3) for k, v in sorted(seen.items())}}


# ---------------------------------------------------------------------------
# CPU legs: the reference NumPy step (baseline/_ref) and the C restatement
# ---------------------------------------------------------------------------
def _flashopt():
    if REF_PATH not in sys.path:
        sys.path.insert(0, REF_PATH)
    import flashopt.optim  # noqa: F401

    return sys.modules["flashopt"]


def ref_available() -> bool:
    return os.path.isdir(os.path.join(REF_PATH, "flashopt"))


def _ref_window_worker(conn, opt, hp, win, seed):
    """One process: a random valid state of `win` elements (a window of the
    list; stepping 32-aligned windows is bit-identical to whole tensors,
    SURVEY Appendix B probe 6) stepped by the reference's own
    `flashopt.optim.STEP_FUNCTIONS[opt]` each time the parent asks, feeding
    the returned state back in like a training loop."""
    import numpy as np

    sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
    import helpers as H

    fo = _flashopt()
    F, Q, O = fo.formats, fo.quantize, fo.optim
    rng = np.random.default_rng(seed)
    lp = H.bf16_codes((rng.standard_normal(win) * 0.02).astype(np.float32))
    st = H.random_state(rng, win, opt, lp=lp)
    g = H.random_grad(rng, win)
    spec = Q.GroupSpec(32)
    w = F.SplitTensor(st["weights.lp"], st["weights.rho"], F.BF16, F.INT8_CORRECTION)
    m = Q.QuantizedState(st["momentum.codes"], st["momentum.scales"], spec, "momentum")
    v = Q.QuantizedState(st["variance.codes"], st["variance.scales"], spec, "variance") if opt == "adamw" else None
    state = O.FlashState(w, m, v, 1000)
    hpo = {"adamw": O.AdamHyperParams, "sgd": O.SgdHyperParams, "lion": O.LionHyperParams}[opt](**hp)
    fn = O.STEP_FUNCTIONS[opt]
    conn.send("ready")
    while conn.recv() == "step":
        t0 = time.perf_counter()
        state = fn(state, g, hpo)
        conn.send(time.perf_counter() - t0)


class RefPool:
    """`workers` processes, each holding one window of the list; a pool
    step = every worker steps its window once with the unmodified reference
    (baseline/_ref), all at the same time."""

    WIN = 1 << 22

    def __init__(self, opt: str, config: str, workers: int):
        import multiprocessing as mp

        ctx = mp.get_context("spawn")
        hp = hparams_for(config, opt)
        self.conns, self.procs = [], []
        for i in range(workers):
            a, b = ctx.Pipe()
            p = ctx.Process(target=_ref_window_worker, args=(b, opt, hp, self.WIN, 17 + i), daemon=True)
            p.start()
            self.conns.append(a)
            self.procs.append(p)
        for c in self.conns:
            assert c.recv() == "ready"

    def step(self, only: int | None = None) -> float:
        """Wall time of one pool step (or of worker `only` alone)."""
        cs = self.conns if only is None else [self.conns[only]]
        t0 = time.perf_counter()
        for c in cs:
            c.send("step")
        for c in cs:
            c.recv()
        return time.perf_counter() - t0

    def close(self):
        for c in self.conns:
            c.send("stop")
        for p in self.procs:
            p.join(timeout=10)


def reference_numpy_run(opt: str, config: str, steps: int, warmup: int, workers: int) -> dict:
    """The reference NumPy step on `workers` processes at once (aggregate
    rate over `steps` timed pool steps), plus one worker alone (single-thread
    rate)."""
    pool = RefPool(opt, config, workers)
    try:
        for _ in range(warmup):
            pool.step()
        ts = [pool.step() for _ in range(steps)]
        single = min(pool.step(only=0) for _ in range(3))
    finally:
        pool.close()
    wall = sum(ts)
    done = steps * workers * RefPool.WIN
    return {"value": done / wall / 1e9, "unit": "Gparams/s", "cores": workers, "kind": "reference",
            "single_thread": RefPool.WIN / single / 1e9, "cpu_model": cpu_model(),
            "sample": f"{done} params: {steps} steps of {workers} processes each stepping a 4M-element window "
                      f"of the {config} list (random valid state, t = 1000) with the unmodified reference "
                      f"flashopt.optim.{opt}_step from baseline/_ref, {wall:.1f} s; single-thread = one "
                      f"process alone, best of 3"}


def port_run(opt: str, config: str, target_s: float, nthreads: int) -> dict:
    """The C restatement of the reference step (oracle/, OpenMP) on a
    bounded sample of the list; returns Gparams/s."""
    import numpy as np

    import helpers as H
    from devstate import oracle_state
    from oracle import oracle as O
    from paper_2602_23349_b200 import shapes as S

    O.build()
    hp = hparams_for(config, opt)
    rng = np.random.default_rng(0)
    chunk = 1 << 22
    st = H.random_state(rng, chunk, opt)
    g = H.random_grad(rng, chunk)
    ost = oracle_state(st, 10)
    done, t0 = 0, time.perf_counter()
    for _, shape in S.CONFIGS[config]():
        left = S.numel(shape)
        while left > 0:
            m = min(left, chunk)
            sub = O.OracleState(ost.lp[:m], ost.rho[:m], ost.m_codes[:m], ost.m_scales[:(m + 31) // 32],
                                None if ost.v_codes is None else ost.v_codes[:m],
                                None if ost.v_scales is None else ost.v_scales[:(m + 31) // 32], ost.t)
            O.step_inplace(opt, sub, g[:m], nthreads=nthreads, **hp)
            left -= m
            done += m
            if time.perf_counter() - t0 > target_s:
                break
        if time.perf_counter() - t0 > target_s:
            break
    dt = time.perf_counter() - t0
    return {"value": done / dt / 1e9, "unit": "Gparams/s", "cores": nthreads, "kind": "port",
            "sample": f"{done} params of the {config} list in 4M-element windows stepped by "
                      f"oracle/flashopt_oracle.c ({opt}) in {dt:.1f} s"}


def cpu_baseline(opt: str, config: str, steps: int = 8, warmup: int = 2) -> dict:
    cores = len(os.sched_getaffinity(0))
    port = port_run(opt, config, 4.0, cores)
    if ref_available():
        out = reference_numpy_run(opt, config, steps, warmup, cores)
        out["port"] = port
        return out
    port["note"] = "baseline/_ref missing: the C restatement stands in for the reference"
    return port


def run_reference(args) -> None:
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cores = len(os.sched_getaffinity(0))
    if ref_available():
        r = reference_numpy_run(args.optimizer, args.config, args.steps, args.warmup, cores)
    else:
        r = port_run(args.optimizer, args.config, args.ref_seconds, cores)
        r["note"] = "baseline/_ref missing: the C restatement stands in for the reference"
    v = r["value"]
    line = {"metric": METRIC, "value": v, "unit": "Gparams/s", "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": DTYPE, "data": "synthetic",
            "config": {"workload": f"{args.config} Flash{args.optimizer} step (bounded CPU sample)",
                       "optimizer": args.optimizer},
            "cpu_baseline": r,
            "e2e": {"value": v, "unit": "Gparams/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# device state, parity windows
# ---------------------------------------------------------------------------
def init_random_state(fl, grads_flat, seed: int, lp=None):
    """Random valid state on the device: bf16 N(0, 0.02^2)
    weights, rho/codes uniform in range, fp16 scales ~1e-3, bf16 grads
    N(0, 1e-3^2)."""
    import torch

    gen = torch.Generator(device=fl.rho.device)
    gen.manual_seed(seed)
    dev = fl.rho.device
    step = 1 << 28
    for buf, lo, hi in ((fl.rho, -127, 128), (fl.m_codes, -127, 128), (fl.v_codes, 0, 256)):
        if buf is None:
            continue
        for o in range(0, buf.numel(), step):
            v = buf[o:o + step]
            v.copy_(torch.randint(lo, hi, (v.numel(),), generator=gen, device=dev, dtype=torch.int32))
    for buf in (fl.m_scales, fl.v_scales):
        if buf is None:
            continue
        buf.copy_((torch.rand(buf.numel(), generator=gen, device=dev) * 2e-3).half())
    lp = fl.lp if lp is None else lp
    for flat, scale in ((lp, 0.02), (grads_flat, 1e-3)):
        for o in range(0, flat.numel(), step):
            v = flat[o:o + step]
            v.copy_(torch.randn(v.numel(), generator=gen, device=dev) * scale)


def choose_windows(sizes, nwin: int, win: int, seed: int):
    """(state index, start, length): nwin windows spread over all tensors --
    evenly spaced tensor indices, alternately a random 512-aligned interior
    window and the tensor's tail (partial tiles and groups)."""
    import numpy as np

    rng = np.random.default_rng(seed)
    idx = sorted(set(int(round(x)) for x in np.linspace(0, len(sizes) - 1, min(nwin, len(sizes)))))
    out = []
    for j, i in enumerate(idx):
        n = sizes[i]
        ln = min(win, n)
        if j % 2 == 1 or n <= win:
            a = n - ln
            a -= a % 32  # a window starts on a group boundary; it then runs to the tensor's end
            ln = n - a
        else:
            a = int(rng.integers(0, (n - ln) // 512 + 1)) * 512
        out.append((i, a, ln))
    return out


def snapshot(st, g, a: int, ln: int) -> dict:
    """Host copies of one window of a device FlashState (+ its gradient)."""
    import numpy as np
    import torch

    ga, gb = a // 32, -(-(a + ln) // 32)
    h = lambda t: t.cpu().numpy()  # noqa: E731
    out = {"lp": h(st.weights.lp_values[a:a + ln].view(torch.int16)).view(np.uint16),
           "rho": h(st.weights.corrections[a:a + ln]), "mq": h(st.momentum.codes[a:a + ln]),
           "ms": h(st.momentum.scales[ga:gb]), "vq": None, "vs": None}
    if st.variance is not None:
        out["vq"] = h(st.variance.codes[a:a + ln])
        out["vs"] = h(st.variance.scales[ga:gb])
    if g is not None:
        out["g"] = h(g[a:a + ln].float())
    return out


def parity_check(states, grads, wins, opt: str, hp: dict, do_step) -> dict:
    """One more product step, checked on the windows against the C oracle
    (test infrastructure; outside every timed region)."""
    import numpy as np

    from oracle import oracle as O

    O.build()
    before = [snapshot(states[i], grads[i], a, ln) for i, a, ln in wins]
    t = [states[i].t for i, _, _ in wins]
    do_step()
    after = [snapshot(states[i], None, a, ln) for i, a, ln in wins]
    mm = {k: 0 for k in ("weights.lp", "weights.rho", "momentum.codes", "momentum.scales", "variance.codes",
                         "variance.scales")}
    nthreads = len(os.sched_getaffinity(0))
    elems = 0
    for b, af, t0 in zip(before, after, t):
        ost = O.OracleState(b["lp"].copy(), b["rho"].copy(), b["mq"].copy(), b["ms"].copy(),
                            None if b["vq"] is None else b["vq"].copy(), None if b["vs"] is None else b["vs"].copy(),
                            t0)
        err = O.step_inplace(opt, ost, b["g"], nthreads=nthreads, **hp)
        elems += b["lp"].size
        pairs = [("weights.lp", ost.lp, af["lp"]), ("weights.rho", ost.rho, af["rho"]),
                 ("momentum.codes", ost.m_codes, af["mq"]), ("momentum.scales", ost.m_scales, af["ms"])]
        if b["vq"] is not None:
            pairs += [("variance.codes", ost.v_codes, af["vq"]), ("variance.scales", ost.v_scales, af["vs"])]
        for k, want, got in pairs:
            bits = lambda x: np.ascontiguousarray(x).view({1: np.uint8, 2: np.uint16}[x.itemsize])  # noqa: E731
            mm[k] += int((bits(want) != bits(got)).sum())
        if err:
            mm["oracle_errors"] = mm.get("oracle_errors", 0) + 1
    if opt != "adamw":
        mm.pop("variance.codes")
        mm.pop("variance.scales")
    return {"windows": len(wins), "elements": elems, "mismatches": mm, "total_mismatches": sum(mm.values()),
            "checker": "oracle/flashopt_oracle.c (C restatement pinned to the reference; outside the timed region)"}


# ---------------------------------------------------------------------------
# e2e through the C-ABI host-buffer entry point
# ---------------------------------------------------------------------------
def pcie_peaks(nbytes: int = 1 << 29, reps: int = 3) -> dict:
    """Pinned host <-> HBM copy bandwidth on this box (the e2e leg's
    roofline): H2D alone, D2H alone, both at once on two streams."""
    import torch

    h_in = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d_a = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d_b = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def run(h2d, d2h):
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        if h2d:
            with torch.cuda.stream(s1):
                d_a.copy_(h_in, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2):
                h_out.copy_(d_b, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    def timed(h2d, d2h):
        run(h2d, d2h)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            run(h2d, d2h)
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps * 1e-3

    out = {"h2d_gbs": nbytes / timed(True, False) / 1e9, "d2h_gbs": nbytes / timed(False, True) / 1e9,
           "bidir_each_gbs": nbytes / timed(True, True) / 1e9}
    del h_in, h_out, d_a, d_b
    torch.cuda.empty_cache()
    return out


def pcie_bound_s(h2d_bytes: float, d2h_bytes: float, pk: dict) -> float:
    """Least time to move both byte counts: both directions at the
    concurrent rate until the smaller one is done, the rest alone."""
    both = min(h2d_bytes, d2h_bytes)
    t = both / (pk["bidir_each_gbs"] * 1e9)
    if h2d_bytes > d2h_bytes:
        t += (h2d_bytes - both) / (pk["h2d_gbs"] * 1e9)
    else:
        t += (d2h_bytes - both) / (pk["d2h_gbs"] * 1e9)
    return t


def host_e2e(states, grads, opt, hp, t0, steps, warmup, chunk_elems: int = 1 << 26):
    """e2e: the same step through the C-ABI host-buffer entry point
    (fo_step_host): state + gradient in pinned host memory, H2D copy, fused
    step and D2H copy of the updated state inside the timed region."""
    import numpy as np
    import torch

    from paper_2602_23349_b200.host import HostFlashState, pinned_empty, step_host

    t_alloc = time.perf_counter()
    adam = opt == "adamw"
    n_tot = sum(st.length for st in states)
    g_tot = sum(st.momentum.scales.numel() for st in states)
    host = {"lp": pinned_empty(n_tot, np.uint16), "rho": pinned_empty(n_tot, np.int8),
            "mq": pinned_empty(n_tot, np.int8), "ms": pinned_empty(g_tot, np.float16),
            "vq": pinned_empty(n_tot, np.uint8) if adam else None,
            "vs": pinned_empty(g_tot, np.float16) if adam else None, "g": pinned_empty(n_tot, np.uint16)}

    def put(dst, src):
        view = {1: (np.uint8, torch.uint8), 2: (np.int16, torch.int16)}[dst.itemsize]
        torch.from_numpy(dst.view(view[0])).copy_(src.reshape(-1).view(view[1]))

    hs, hg = [], []
    o = go = 0
    h2d = d2h = 0
    for st, g in zip(states, grads):
        n, ng = st.length, st.momentum.scales.numel()
        put(host["lp"][o:o + n], st.weights.lp_values)
        put(host["rho"][o:o + n], st.weights.corrections)
        put(host["mq"][o:o + n], st.momentum.codes)
        put(host["ms"][go:go + ng], st.momentum.scales)
        if adam:
            put(host["vq"][o:o + n], st.variance.codes)
            put(host["vs"][go:go + ng], st.variance.scales)
        put(host["g"][o:o + n], g)
        hs.append(HostFlashState(host["lp"][o:o + n], host["rho"][o:o + n], host["mq"][o:o + n],
                                 host["ms"][go:go + ng], host["vq"][o:o + n] if adam else None,
                                 host["vs"][go:go + ng] if adam else None, t0))
        hg.append(host["g"][o:o + n])
        h2d += n * (2 + 1 + 1 + (1 if adam else 0) + 2) + ng * 2 * (2 if adam else 1)
        d2h += n * (2 + 1 + 1 + (1 if adam else 0)) + ng * 2 * (2 if adam else 1)
        o += n
        go += ng
    alloc_s = time.perf_counter() - t_alloc
    for _ in range(warmup):
        step_host(opt, hs, hg, hp, chunk_elems=chunk_elems, check=False)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(steps):
        step_host(opt, hs, hg, hp, chunk_elems=chunk_elems, check=False)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / steps
    pk = pcie_peaks()
    bound = pcie_bound_s(h2d, d2h, pk)
    return {"value": n_tot / dt / 1e9, "unit": "Gparams/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": dt * 1e3, "steps": steps, "warmup": warmup,
            "roofline": {"bound": "pcie", "bound_ms": bound * 1e3, "frac": bound / dt, "pcie_measured": pk},
            "path": "fo_step_host (C ABI), pinned host buffers, 3 x 64M-element device slots",
            "host_setup_s": round(alloc_s, 1)}


def e2e_leg(args, states, grads, opt, hp, world, n_local, n_all, dev, reduce_):
    import torch
    import torch.distributed as dist

    need = n_local * BYTES_PER_PARAM[opt] * 1.15
    try:
        import psutil

        avail = psutil.virtual_memory().available / max(1, int(os.environ.get("LOCAL_WORLD_SIZE", world)))
    except Exception:
        avail = float("inf")
    if avail < need:
        return {"skipped": f"host memory: {avail / 1e9:.0f} GB available per rank, {need / 1e9:.0f} GB needed"}
    if world > 1:
        dist.barrier()
    e2e = host_e2e(states, grads, opt, hp, args.t0 + args.warmup + args.steps + 1,
                   steps=min(args.steps, args.e2e_steps), warmup=1)
    if world > 1:
        tt = torch.tensor([e2e["ms_per_step"], e2e["h2d_bytes_per_step"], e2e["d2h_bytes_per_step"]],
                          device=dev, dtype=torch.float64)
        reduce_(tt[:1], dist.ReduceOp.MAX)
        reduce_(tt[1:], dist.ReduceOp.SUM)
        e2e.update({"ms_per_step": float(tt[0]), "h2d_bytes_per_step": int(tt[1]),
                    "d2h_bytes_per_step": int(tt[2]), "value": n_all / (float(tt[0]) * 1e-3) / 1e9, "ranks": world})
        e2e["roofline"]["frac"] = e2e["roofline"]["bound_ms"] / e2e["ms_per_step"]
    return e2e


def traffic_for(args, n_local: int):
    """ncu DRAM bytes (read + write) per launch for this config, scaled from
    the bytes per parameter of a --set full capture (profiles/ncu_traffic.json:
    the headline launch itself for the Llama list)."""
    if args.traffic is not None:
        return args.traffic, "--traffic"
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f)
        if args.config == "llama31_8b" and args.optimizer == "adamw":
            return d["bytes_per_param"] * n_local / 1e9, d["source"]
        key = f"{args.config}_{args.optimizer}"
        if key in d.get("other_lists", {}):
            return d["other_lists"][key] * n_local / 1e9, f"profiles/ncu_traffic.json other_lists[{key}]"
    except Exception:
        pass
    return None, None


# ---------------------------------------------------------------------------
# the product arm
# ---------------------------------------------------------------------------
def run_ours(args) -> None:
    import torch
    import torch.distributed as dist

    from paper_2602_23349_b200 import _lib
    from paper_2602_23349_b200 import shapes as S
    from paper_2602_23349_b200.optim import HP_TYPES

    rank, world, local = dist_env()
    # FO_BENCH_DIST_BACKEND=gloo is a test mode for the N > 1 code path on a
    # box with fewer GPUs than ranks (ranks share devices, collectives are
    # staged through host memory); timings from it are not the product's.
    backend = os.environ.get("FO_BENCH_DIST_BACKEND", "nccl")
    if world > 1:
        dist.init_process_group(backend)
    if backend != "nccl":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    def reduce_(t, op):
        if backend == "nccl":
            dist.all_reduce(t, op=op)
            return t
        h = t.cpu()
        dist.all_reduce(h, op=op)
        t.copy_(h)
        return t

    opt = args.optimizer
    shapes = S.CONFIGS[args.config]()
    hpd = hparams_for(args.config, opt)
    hp = HP_TYPES[opt](**hpd)
    stream = torch.cuda.current_stream(dev)
    sh = stream.cuda_stream
    zo = None
    if world == 1:
        from paper_2602_23349_b200.flat import FlatStates, StepPlan

        sizes = [S.numel(s) for _, s in shapes]
        fl = FlatStates(sizes, opt, dev)
        grads_flat = torch.empty(fl.total, dtype=torch.bfloat16, device=dev)
        init_random_state(fl, grads_flat, 1234)
        grads = [grads_flat[o:o + n] for o, n in zip(fl.offsets, fl.sizes)]
        states = fl.states
        plan = StepPlan(opt, states)
        plan.set_grads(grads)
        for st in states:  # the random state stands for step t0 of a training run
            st.t = args.t0
        err = torch.zeros(1, dtype=torch.int32, device=dev)

        def one_step():
            plan.launch([hp.scalars(states[0].t + 1)], err.data_ptr(), sh)

        def device_errors():
            return int(err.item())
    else:
        # the product ZeRO-1 optimizer over the whole list (every rank holds
        # the full bf16 params; it owns 1/N of the state)
        from paper_2602_23349_b200.zero import ZeroFlashOptimizer

        params = [torch.empty(s, dtype=torch.bfloat16, device=dev) for _, s in shapes]
        zo = ZeroFlashOptimizer(params, opt, [hp], bucket_elems=args.bucket_elems, check_errors="off",
                                fused_allgather=args.fused_ag)
        del params
        init_random_state(zo.flat_state, zo.flat_grads, 1234 + rank, lp=zo.flat_params)
        states = zo.states
        grads = [zo.shard_grads[s.shard_off:s.shard_off + s.length] for s in zo.segments]
        zo.t = args.t0
        for st in states:
            st.t = args.t0

        def one_step():
            zo.step_shard()
            zo.t += 1

        def device_errors():
            return int(zo._errors.errors.mask())
    n_local = sum(st.length for st in states)
    n_all = n_local
    if world > 1:
        nn = torch.tensor([n_local], device=dev, dtype=torch.float64)
        reduce_(nn, dist.ReduceOp.SUM)
        n_all = int(nn.item())

    clocks = ClockSampler(local)
    clocks.start()
    power = PowerSampler(local)
    power.start()
    if zo is not None:
        zo.reduce_scatter_grads()
    for _ in range(args.warmup):
        one_step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    _lib.fixup_stats(sh, reset=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    clocks.begin()
    power.begin()
    t0.record(stream)
    for i in range(args.steps):
        ev[i][0].record(stream)
        one_step()
        ev[i][1].record(stream)
    t1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    pwr = power.stop()
    flagged, slices = _lib.fixup_stats(sh, reset=True)
    if world > 1:
        dist.barrier()
    total_ms = t0.elapsed_time(t1)
    kern_ms = [a.elapsed_time(b) for a, b in ev]
    avg_kern_ms = sum(kern_ms) / len(kern_ms)
    if world > 1:
        tt = torch.tensor([total_ms, avg_kern_ms], device=dev)
        reduce_(tt, dist.ReduceOp.MAX)
        total_ms, avg_kern_ms = float(tt[0]), float(tt[1])
        fs = torch.tensor([flagged, slices], device=dev, dtype=torch.float64)
        reduce_(fs, dist.ReduceOp.SUM)
        flagged, slices = int(fs[0]), int(fs[1])
    ms_per_step = total_ms / args.steps
    value = n_all / (ms_per_step * 1e-3) / 1e9
    peak, peak_kind = peaks()
    bpp = BYTES_PER_PARAM[opt]
    achieved = n_local * bpp / (avg_kern_ms * 1e-3) / 1e9
    launches_per_step = 2 * ((len(states) + 383) // 384)  # fused step + fix-up per <= 384 tensors
    traffic, traffic_src = traffic_for(args, n_local)

    # One more launch after the board has idled for a second: the same kernel
    # before the 1000 W power limit pulls the clock down (informational; the
    # headline is the back-to-back average above).
    single = None
    if world == 1 and zo is None:
        import time as _time

        torch.cuda.synchronize()
        _time.sleep(1.0)
        a1, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a1.record(stream)
        one_step()
        b1.record(stream)
        torch.cuda.synchronize()
        ms1 = a1.elapsed_time(b1)
        single = {"ms": ms1, "gparams_s": n_all / (ms1 * 1e-3) / 1e9,
                  "frac_of_peak": n_local * bpp / (ms1 * 1e-3) / 1e9 / peak,
                  "note": "one launch after 1 s idle (clock not yet pulled down by the power limit); "
                          "not the headline"}

    zero1 = None
    if zo is not None:
        zero1 = zero1_phases(zo, args, dev, stream, reduce_, n_all)
    emask = device_errors()

    parity = None
    if not args.no_parity:
        wins = choose_windows([st.length for st in states], args.parity_windows, 1 << 20, 99 + rank)
        if zo is None:
            parity = parity_check(states, grads, wins, opt, hpd, one_step)
        else:
            zo.reduce_scatter_grads()
            parity = parity_check(states, grads, wins, opt, hpd, one_step)
            zo.all_gather_params()
            if world > 1:
                pm = torch.tensor([parity["total_mismatches"], parity["windows"], parity["elements"]], device=dev,
                                  dtype=torch.float64)
                reduce_(pm, dist.ReduceOp.SUM)
                parity.update({"total_mismatches": int(pm[0]), "windows": int(pm[1]), "elements": int(pm[2]),
                               "ranks": world, "mismatches_rank0": parity.pop("mismatches")})

    e2e = None
    if not args.no_e2e:
        e2e = e2e_leg(args, states, grads, opt, hp, world, n_local, n_all, dev, reduce_)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(opt, args.config)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "Gparams/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak",
            "vs_baseline": None, "dtype": DTYPE, "data": "synthetic",
            "config": {"workload": f"{args.config} Flash{opt} fused step (state resident in HBM)",
                       "optimizer": opt, "params": n_all, "tensors": len(shapes),
                       "hbm_gbs_equiv": value * bpp, "step_t": args.t0 + 1,
                       "l2": "working set >> 126 MB L2, no flush needed" if n_local * bpp > 2 * 126e6
                       else "L2-resident working set",
                       "parallelism": f"zero1 x{world} (ZeroFlashOptimizer, NCCL)" if world > 1 else "single-gpu"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "traffic_unit": "GB per launch",
                         "traffic_source": traffic_src,
                         "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
                         "bytes_per_param": bpp, "kernel_ms": avg_kern_ms,
                         "kernel": "fo::step_ws_kernel + fix-up (cuda events on the launch stream)"},
            "fast_path": {"slices": slices, "fixup_slices": flagged,
                          "share": (1.0 - flagged / slices) if slices else None,
                          "note": "512-element slices stored by the fused tile vs re-run by the fix-up launch "
                                  "(fo_fixup_stats, timed region)"},
            "parity": parity, "e2e": e2e, "cpu_baseline": cpu, "zero1": zero1, "single_launch_after_idle": single,
            "clocks": clk, "power": pwr, "gpu_launches": args.steps * launches_per_step,
            "device_errors": emask,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def zero1_phases(zo, args, dev, stream, reduce_, n_all) -> dict:
    """The three phases of ZeroFlashOptimizer.step on the full list, timed
    with CUDA events (max over ranks): NCCL reduce-scatter of the bf16
    gradients, the sharded fused step, NCCL all-gather of the bf16 params."""
    import torch
    import torch.distributed as dist

    iters = max(2, min(args.steps, 5))
    E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    evs = [(E(), E(), E(), E()) for _ in range(iters)]
    zo.step()  # warm
    torch.cuda.synchronize()
    dist.barrier()
    for a, b, c, d in evs:
        a.record(stream)
        zo.reduce_scatter_grads()
        b.record(stream)
        zo.step_shard()  # fused_allgather: the step also writes every peer's parameters
        c.record(stream)
        if zo.fused_allgather:
            zo._peer_barrier()
        else:
            zo.all_gather_params()
        d.record(stream)
        zo.t += 1
    torch.cuda.synchronize()
    rs = sum(a.elapsed_time(b) for a, b, _, _ in evs) / iters
    st = sum(b.elapsed_time(c) for _, b, c, _ in evs) / iters
    ag = sum(c.elapsed_time(d) for _, _, c, d in evs) / iters
    full = sum(a.elapsed_time(d) for a, _, _, d in evs) / iters
    t = torch.tensor([rs, st, ag, full], device=dev)
    reduce_(t, dist.ReduceOp.MAX)
    rs, st, ag, full = (float(x) for x in t)
    W = zo.world
    total = zo.layout.total
    moved = 2 * (W - 1) / W * total * 2  # bytes each rank sends + receives per RS + AG pair (ring model)
    coll = "NCCL" if zo.backend == "nccl" else "gloo (host-staged test mode)"
    out = {"reduce_scatter_ms": rs, "step_ms": st, "all_gather_ms": ag, "full_step_ms": full,
           "full_step_gparams_s": n_all / (full * 1e-3) / 1e9, "params_padded": total,
           "buckets": len(zo.layout.buckets), "busbw_gbs": moved / ((rs + ag) * 1e-3) / 1e9,
           "fused_allgather": zo.fused_allgather,
           "note": f"ZeroFlashOptimizer phases; {coll} reduce-scatter of bf16 grads, "
                   + ("fused step storing every peer's bf16 params over CUDA IPC + cross-rank barrier "
                      "(all_gather_ms = the barrier)" if zo.fused_allgather else f"{coll} all-gather of bf16 params")}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="llama31_8b", choices=["llama31_8b", "gpt2_medium", "resnet50"])
    ap.add_argument("--optimizer", default="adamw", choices=["adamw", "sgd", "lion"])
    ap.add_argument("--ref-seconds", type=float, default=10.0)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--parity-windows", type=int, default=64)
    ap.add_argument("--bucket-elems", type=int, default=None, help="N>1: ZeRO bucket size (default: one bucket)")
    ap.add_argument("--fused-ag", action="store_true",
                    help="N>1: fused step + all-gather (the step stores into every peer's parameters, CUDA IPC)")
    ap.add_argument("--traffic", type=float, default=None,
                    help="ncu dram bytes per launch (read+write), from profiles/, reported beside the roofline")
    ap.add_argument("--t0", type=int, default=1000,
                    help="step counter of the synthetic state (1000: steady state, f32 bias corrections == 1)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
