"""Benchmark of the batched CKKS hot path on B200 (driver contract, one JSON line).

Headline (BASELINE.json metric "NTT KOPS and HMULT KOPS (N=2^16, batched)"):

* `value`  = limb-NTT KOPS: N = 2^16 negacyclic transforms of one residue row
  (forward and inverse each count 1) over the paper-Default RNS chain
  (`p_default`: 45 chain primes) and a batch of B ciphertext
  polynomials -- BASELINE configs[1].  One step = batched forward NTT +
  batched inverse NTT of the whole (45, B, 65536) buffer (2*45*B limb-NTTs).
  Inputs (1.47 GB at B=128) are larger than L2, so no flush is needed.
* `hmult_kops` = HMULT+relinearisation+rescale per second / 1e3 at N=2^16
  P-Default (configs[2]), measured with the same protocol.

Multi-GPU (torchrun, one rank per GPU): every rank transforms its own batch
(independent ciphertexts shard with no collective; "scaling": "weak");
timing is device time, barrier-bracketed, max over ranks.

`--impl reference` times the CPU oracle port (oracle/, plain C + OpenMP, the
reference's algorithm) on a bounded sample of the same workload on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PRESET = "p_default"
N = 1 << 16
METRIC = "NTT KOPS and HMULT KOPS (N=2^16, batched)"
UNIT = "K limb-NTT/s"


def _env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


# ----------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ----------------------------------------------------------------------------

class ClockSampler:
    """SM clock and throttle reasons sampled during the timed region: NVML
    every 5 ms (the handle found by the torch device's PCI bus id), else
    nvidia-smi every 0.2 s."""
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    REASONS = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []          # (sm_mhz, max_mhz, set of reason names)
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml as N
            import torch
            N.nvmlInit()
            prop = torch.cuda.get_device_properties(index)
            bus = f"{prop.pci_domain_id:08x}:{prop.pci_bus_id:02x}:{prop.pci_device_id:02x}.0"
            try:
                h = N.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:
                h = N.nvmlDeviceGetHandleByIndex(index)
            bits = {"hw_slowdown": N.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": N.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": N.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": N.nvmlClocksEventReasonSwPowerCap}
            self._nvml = (N, h, bits)
        except Exception:
            self._nvml = None

    def _sample_nvml(self):
        N, h, bits = self._nvml
        sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
        mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
        try:
            r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
        except Exception:
            r = N.nvmlDeviceGetCurrentClocksThrottleReasons(h)
        return float(sm), float(mx), {k for k, v in bits.items() if r & v}

    def _sample_smi(self):
        out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.QUERY}",
                              "--format=csv,noheader,nounits"],
                             capture_output=True, text=True, timeout=5)
        f = [x.strip() for x in out.stdout.strip().split(",")]
        return (float(f[1]), float(f[2]),
                {self.REASONS[i] for i in range(4) if len(f) > 5 + i and f[5 + i].lower() == "active"})

    def _run(self):
        period = 0.005 if self._nvml else 0.2
        while not self._stop.is_set():
            try:
                self.samples.append(self._sample_nvml() if self._nvml else self._sample_smi())
            except Exception:
                pass
            self._stop.wait(period)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        return {"sm_mhz": float(np.median([s[0] for s in self.samples])),
                "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": sorted(set().union(*[s[2] for s in self.samples])),
                "samples": len(self.samples),
                "source": "nvml" if self._nvml else "nvidia-smi"}


# ----------------------------------------------------------------------------
# CPU oracle timing (cpu_baseline leg and --impl reference)
# ----------------------------------------------------------------------------

def cpu_oracle_rate(primes, members, reps=1):
    """limb-NTT/s of the C oracle port (fwd + inv over len(primes) limbs x
    members), in place on pre-reduced rows: only the OpenMP C kernel is timed
    (no numpy upcast / copy / stack glue), every host thread."""
    from oracle import oracle as O
    threads = os.cpu_count() or 1
    O.THREADS = threads
    rng = np.random.default_rng(7)
    x = O.uniform_rows(rng, primes, (members, N))
    for q in primes:                       # build every prime's tables untimed
        O._tables(q, N)
    O.transform_inplace(x[:1, :1].copy(), primes[:1])
    t0 = time.perf_counter()
    for _ in range(reps):
        O.transform_inplace(x, primes)
        O.transform_inplace(x, primes, inverse=True)
    dt = time.perf_counter() - t0
    return 2 * len(primes) * members * reps / dt, dt, threads


def cpu_numpy_butterfly(primes, members_per_task=2, pool_tasks=None):
    """The reference's own algorithm and cost profile: the numpy butterfly
    restatement (oracle/butterfly_np.py, ref ntt.py:172-205 via
    batch.batched_apply) on ONE host core, and over a multiprocessing.Pool of
    every core mapping independent (limb, member-chunk) tasks (BASELINE.md
    §2).  Returns {single_core, all_cores} limb-NTT/s with the core counts."""
    import multiprocessing as mp
    from oracle import butterfly_np as BF
    cores = os.cpu_count() or 1
    q = primes[0]
    BF._plan(q, N)
    t0 = time.perf_counter()
    done = BF.fwd_inv_rows((q, N, members_per_task, 1))
    one = done / (time.perf_counter() - t0)
    tasks = [(primes[i % len(primes)], N, members_per_task, 100 + i)
             for i in range(pool_tasks or 2 * cores)]
    ctx = mp.get_context("spawn")   # the parent holds a CUDA context: never fork it
    with ctx.Pool(cores) as pool:
        pool.map(BF.fwd_inv_rows, tasks[:cores])          # warm: plans built per worker
        t0 = time.perf_counter()
        done = sum(pool.map(BF.fwd_inv_rows, tasks))
        allc = done / (time.perf_counter() - t0)
    return {"single_core": {"value": one / 1e3, "unit": UNIT, "cores": 1},
            "all_cores": {"value": allc / 1e3, "unit": UNIT, "cores": cores,
                          "sample": f"{len(tasks)} tasks x {members_per_task} members fwd+inv "
                                    f"(N=2^16, p_default primes), Pool({cores})"},
            "impl": "oracle/butterfly_np.py (numpy uint64 ufuncs, ref ntt.py:172-205)"}


def headline_config(L, B, world, plan):
    """The headline workload (BASELINE configs[1]); both arms report it."""
    return {"workload": f"batched forward+inverse NTT, N=2^16, {PRESET} chain "
                        f"({L} RNS limbs), batch {B} per GPU (BASELINE configs[1])",
            "N": N, "limbs": L, "batch_per_gpu": B, "plan": list(plan),
            "l2": f"inputs larger than L2 ({L * B * N * 4 / 2**30:.2f} GiB per buffer)",
            "parallelism": f"batch-sharded x{world}, no collective"}


def run_reference(args):
    rank = _env_int("RANK", 0)
    if rank != 0:
        return 0
    from paper_2212_14191_b200.params import CkksParams
    primes = list(CkksParams.from_preset(PRESET).chain.q)
    members = args.cpu_members
    for _ in range(args.warmup):
        cpu_oracle_rate(primes, 1)
    rates, total = [], 0.0
    for _ in range(args.steps):
        r, dt, threads = cpu_oracle_rate(primes, members)
        rates.append(r)
        total += dt
    value = float(np.median(rates)) / 1e3
    sample = (f"fwd+inv NTT N=2^16 over the {len(primes)} p_default chain primes x "
              f"{members} members per step ({2 * len(primes) * members} limb-NTTs)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / max(args.steps, 1), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": dict(headline_config(len(primes), args.batch, args.gpus, (256, 256)),
                       cpu_sample_members=members),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------
# B200 arm
# ----------------------------------------------------------------------------

def int8_peak_tops(torch):
    """Dense int8 tensor throughput of this GPU (torch._int_mm 8192^3, best of 10)."""
    try:
        a = torch.randint(-128, 127, (8192, 8192), dtype=torch.int8, device="cuda")
        b = torch.randint(-128, 127, (8192, 8192), dtype=torch.int8, device="cuda")
        for _ in range(3):
            torch._int_mm(a, b)
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(10):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            torch._int_mm(a, b)
            e.record()
            torch.cuda.synchronize()
            best = min(best, s.elapsed_time(e))
        del a, b
        return 2 * 8192 ** 3 / (best / 1e3) / 1e12
    except Exception:
        return None


def run_b200(args):
    import torch
    import torch.distributed as dist

    rank, world = _env_int("RANK", 0), _env_int("WORLD_SIZE", 1)
    # TFHE_BENCH_SHARED_GPU=1 (development check only): every rank on cuda:0
    # with a gloo group, to exercise the N > 1 code path on a one-GPU box
    shared = os.environ.get("TFHE_BENCH_SHARED_GPU") == "1"
    local = 0 if shared else _env_int("LOCAL_RANK", 0)
    if not shared and local >= torch.cuda.device_count():
        raise SystemExit(f"bench.py: rank {rank} needs GPU {local}, but only "
                         f"{torch.cuda.device_count()} are visible (--gpus {world})")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cpu" if shared else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    from paper_2212_14191_b200.batch import BatchBuffer, batched_apply
    from paper_2212_14191_b200.ckks import CiphertextBatch, CkksContext
    from paper_2212_14191_b200.device import DeviceContext
    from paper_2212_14191_b200.ntt import TwiddleTable
    from paper_2212_14191_b200.params import CkksParams

    params = CkksParams.from_preset(PRESET)
    primes = list(params.chain.q)
    L, B = len(primes), args.batch
    ext = tuple(params.chain.q) + tuple(params.chain.p)
    ctx = DeviceContext.get(N, ext, n_chain=L, n_special=len(params.chain.p), device=dev)

    # synthetic uniform residues per limb (cli._random_batch, cli.py:59-64), on device
    g = torch.Generator(device=dev)
    g.manual_seed(1234 + rank)
    x = torch.empty((L, B, N), dtype=torch.int32, device=dev)
    for i, q in enumerate(primes):
        x[i] = torch.randint(0, q, (B, N), generator=g, device=dev, dtype=torch.int64).to(torch.int32)
    f = torch.empty_like(x)
    y = torch.empty_like(x)

    def step():
        ctx.ntt(x, primes, out=f)
        ctx.ntt(f, primes, inverse=True, out=y)

    for _ in range(max(args.warmup, 1)):
        step()
    torch.cuda.synchronize()
    # parity spot check of the timed path against the CPU oracle (rank 0)
    parity = None
    if rank == 0:
        from oracle import oracle as O
        xs = x[:2, :1].cpu().numpy().view(np.uint32)
        fs = f[:2, :1].cpu().numpy().view(np.uint32)
        parity = bool(np.array_equal(fs, O.ntt(xs, primes[:2])) and
                      np.array_equal(y[:2, :1].cpu().numpy().view(np.uint32), xs))

    stream = torch.cuda.current_stream(dev)
    from paper_2212_14191_b200 import _lib as tl
    # per-kernel device times over the timed region: the library brackets each
    # NTT-pass launch with CUDA events on its own (= this) stream
    with ClockSampler(local) as clk, tl.kernel_timer() as ktime:
        barrier()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        for _ in range(args.steps):
            step()
        e.record(stream)
        torch.cuda.synchronize()
        barrier()
    ms = max_over_ranks(s.elapsed_time(e))
    limb_ntts = 2 * L * B * args.steps * world
    value = limb_ntts / (ms / 1e3) / 1e3

    # roofline of the NTT call (two kernel launches: the three-factor plan's
    # column pass + row pass).  int8 tensor work per limb-NTT of the device
    # factorisation = 16 byte products x 2 ops x N x (k0 + k1 + k2)
    # (tfhe_ctx_transform_plan: (32, 32, 64) at N = 2^16 -- a quarter of the
    # 256 x 256 plan's 32 N (n1 + n2)); compulsory HBM bytes = 8 N (u32 in + out)
    n1, n2 = ctx.plan
    kplan = ctx.transform_plan
    ops_per_limb = 32 * N * sum(kplan)
    ops_256 = 32 * N * (n1 + n2)                     # the reference plan's formulation
    ntt_call_ms = ms / (2 * args.steps)             # one batched NTT call
    achieved_tops = L * B * ops_per_limb / (ntt_call_ms / 1e3) / 1e12
    achieved_gbs = L * B * 8 * N / (ntt_call_ms / 1e3) / 1e9     # compulsory bytes

    def timed(fn, steps):
        """device ms per call of fn (CUDA events on the launching stream,
        barrier-bracketed, max over ranks), after max(warmup, 1) warm calls"""
        for _ in range(max(args.warmup, 1)):
            fn()
        torch.cuda.synchronize()
        barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(steps):
            fn()
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
        return max_over_ranks(ev0.elapsed_time(ev1)) / steps

    def rand_rows(basis, shape_tail):
        t = torch.empty((len(basis),) + tuple(shape_tail), dtype=torch.int32, device=dev)
        for i, q in enumerate(basis):
            t[i] = torch.randint(0, q, tuple(shape_tail), generator=g, device=dev,
                                 dtype=torch.int64).to(torch.int32)
        return t

    def ckks_setup(prm, batch, key=None):
        ck = CkksContext(prm, device=dev)
        e = tuple(prm.chain.q) + tuple(prm.chain.p)
        if key is None:
            key = rand_rows(e, (prm.dnum, 2, prm.n)).permute(1, 2, 0, 3).contiguous()
        cts = [CiphertextBatch(rand_rows(prm.chain.q, (2, batch, prm.n)).transpose(0, 1)
                               .contiguous(), prm.l_max) for _ in range(2)]
        return ck, key, cts

    # batched NTT batch sweep at the headline chain (BASELINE configs[1]
    # "batch sweep on 1 B200"; ref cli.py:195-216 --batch-sizes): fwd+inv of
    # (45, B, 2^16) for B = 1 .. 1024 (12 GiB per buffer at B = 1024)
    bsweep = None
    if args.batch_sweep:
        bsweep = {}
        bmax = 1024
        flat = [torch.empty(L * bmax * N, dtype=torch.int32, device=dev) for _ in range(2)]
        for i, q in enumerate(primes):     # uniform residues per limb, reused by every B
            flat[0].view(L, bmax, N)[i] = torch.randint(0, q, (bmax, N), generator=g, device=dev,
                                                        dtype=torch.int64).to(torch.int32)
        bb = 1
        while bb <= bmax:
            xs = flat[0][:L * bb * N].view(L, bb, N)
            fs = flat[1][:L * bb * N].view(L, bb, N)

            def fwd_inv():
                ctx.ntt(xs, primes, out=fs)
                ctx.ntt(fs, primes, inverse=True, out=xs)
            ms_b = timed(fwd_inv, max(3, min(50, 2048 // bb)))
            bsweep[str(bb)] = {"limb_ntt_kops": 2 * L * bb * world / (ms_b / 1e3) / 1e3,
                               "ms_per_step": ms_b}
            bb *= 2
        del flat, xs, fs
        ctx._ws.clear()

    # CKKS operators at P-Default (configs[2..4]), same protocol
    hm = None
    hm_check = None
    if args.hmult_batch > 0:
        Bh = args.hmult_batch
        ck, key, cts = ckks_setup(params, Bh)
        hsteps = max(1, min(args.steps, 5))
        # HMULT+relin+rescale through the fused operator (bit-identical to
        # rescale_batch(hmult_batch(.)), 2l fewer limb-NTTs); the two-call form beside it
        ms_hm = timed(lambda: ck.hmult_rescale_batch(cts[0], cts[1], key), hsteps)
        ms_hm_2 = timed(lambda: ck.rescale_batch(ck.hmult_batch(cts[0], cts[1], key)), hsteps)
        ms_hm_only = timed(lambda: ck.hmult_batch(cts[0], cts[1], key), hsteps)
        ms_rot = timed(lambda: ck.hrotate_batch(cts[0], 1, key), hsteps)
        ms_rs = timed(lambda: ck.rescale_batch(cts[0]), hsteps)

        def mixed():   # configs[4]: HMULT -> rescale -> HROTATE per ciphertext
            ck.hrotate_batch(ck.hmult_rescale_batch(cts[0], cts[1], key), 1, key)
        ms_mix = timed(mixed, hsteps)
        rate = lambda ms: Bh * world / (ms / 1e3)  # noqa: E731
        hm = {"hmult_kops": rate(ms_hm) / 1e3, "ms_per_batch": ms_hm, "batch_per_gpu": Bh,
              "hmult_then_rescale_per_s": rate(ms_hm_2),
              "hmult_relin_only_per_s": rate(ms_hm_only), "hrotate_per_s": rate(ms_rot),
              "hrotate_ms_per_batch": ms_rot, "rescale_per_s": rate(ms_rs),
              "mixed_ct_per_s": rate(ms_mix), "mixed_ms_per_batch": ms_mix}
        # parity spot check of the timed HMULT+relin+rescale (member 0) against
        # the CPU oracle (ckks.py:265-274 then :291-311), rank 0, untimed
        if args.hmult_check and rank == 0:
            from oracle import oracle as O
            O.THREADS = os.cpu_count() or 1
            t0 = time.perf_counter()
            got = ck.hmult_rescale_batch(cts[0], cts[1], key).data[:, :, 0].cpu().numpy() \
                .view(np.uint32)
            c0h = cts[0].data[:, :, 0].cpu().numpy().view(np.uint32)
            c1h = cts[1].data[:, :, 0].cpu().numpy().view(np.uint32)
            kh = key.cpu().numpy().view(np.uint32)
            basis = tuple(params.chain.q)
            hb, ha = O.hmult(c0h[0], c0h[1], c1h[0], c1h[1], basis, kh, params.chain.q,
                             params.chain.p, params.alpha, params.dnum)
            rb, ra = O.rescale(hb, ha, basis)
            hm_check = {"member": 0, "exact": bool(np.array_equal(got[0], rb) and
                                                   np.array_equal(got[1], ra)),
                        "oracle_s": time.perf_counter() - t0}
            del kh
        # HMULT+relin+rescale batch sweep (same key, fresh ciphertexts)
        hsw = {str(Bh): rate(ms_hm)}
        for bs in (8, 32):
            if bs >= Bh:
                continue
            _, _, cs = ckks_setup(params, bs, key)
            ms_b = timed(lambda: ck.hmult_rescale_batch(cs[0], cs[1], key), hsteps)
            hsw[str(bs)] = bs * world / (ms_b / 1e3)
            del cs
        hm["batch_sweep_per_s"] = dict(sorted(hsw.items(), key=lambda kv: int(kv[0])))
        del ck, key, cts
        ctx._ws.clear()

    # dnum-reduced P-Default (alpha = K = 9): ModUp/ModDown are 9-term base
    # conversions on the tensor cores (tfhe_bconv) between the NTTs
    d5 = None
    if args.dnum5_batch > 0:
        pd = CkksParams.from_preset("p_dnum5")
        B5 = args.dnum5_batch
        ck, key, cts = ckks_setup(pd, B5)
        ms_hm = timed(lambda: ck.hmult_rescale_batch(cts[0], cts[1], key), 3)
        ms_rot = timed(lambda: ck.hrotate_batch(cts[0], 1, key), 3)
        d5 = {"workload": f"p_dnum5 (N=2^16, L=44, K=9, dnum=5, alpha=9), batch {B5} per GPU",
              "hmult_relin_rescale_per_s": B5 * world / (ms_hm / 1e3),
              "hrotate_per_s": B5 * world / (ms_rot / 1e3), "ms_per_batch_hmult": ms_hm}
        del ck, key, cts

    # Set_A (N=2^12, the paper's 913 KOPS NTT / 88 KOPS HMULT parameters)
    sa = None
    if args.set_a_batch > 0:
        pa = CkksParams.from_preset("set_a")
        Ba = args.set_a_batch
        ck, key, cts = ckks_setup(pa, Ba)
        qa = list(pa.chain.q)
        xa = rand_rows(qa, (Ba, pa.n))
        fa, ya = torch.empty_like(xa), torch.empty_like(xa)

        def ntt_a():
            ck.dev.ntt(xa, qa, out=fa)
            ck.dev.ntt(fa, qa, inverse=True, out=ya)
        ms_ntt = timed(ntt_a, 10)
        ms_hm = timed(lambda: ck.hmult_rescale_batch(cts[0], cts[1], key), 5)
        ms_hm_only = timed(lambda: ck.hmult_batch(cts[0], cts[1], key), 5)
        sa = {"workload": f"set_a (N=2^12, L+1=2, K=2, dnum=2), batch {Ba} per GPU",
              "ntt_limb_kops": 2 * len(qa) * Ba * world / (ms_ntt / 1e3) / 1e3,
              "ntt_poly_kops": 2 * Ba * world / (ms_ntt / 1e3) / 1e3,
              "hmult_relin_kops": Ba * world / (ms_hm_only / 1e3) / 1e3,
              "hmult_relin_rescale_kops": Ba * world / (ms_hm / 1e3) / 1e3,
              "paper_a100": {"ntt_kops": 913, "hmult_kops": 88},
              # N=2^12 is HBM-bound: 8 N bytes in+out per limb-NTT, all
              # the fused single-launch kernel moves (ntt_fused.cu)
              "ntt_hbm_gbs_compulsory": 2 * len(qa) * Ba * world * 8 * pa.n / (ms_ntt / 1e3) / 1e9}
        sa["ntt_roofline"] = {"bound": "hbm", "achieved": sa["ntt_hbm_gbs_compulsory"] / world,
                              "unit": "GB/s", "kernel": "ntt_fused_kernel (one launch per NTT)",
                              "algorithmic": "8 N bytes per limb-NTT (u32 in + out)"}
        del ck, key, cts, xa, fa, ya

    # configs[0] (the reference's CPU-runnable case: N=2^12, one 30-bit prime,
    # batch 64, fwd+inv) and a degree sweep (2 limbs, 32 Mi coefficients per call)
    sweep = None
    if args.sweep:
        from paper_2212_14191_b200.params import generate_primes
        sweep = {}
        q0 = generate_primes(1 << 12, [30])
        c0ctx = DeviceContext.get(1 << 12, tuple(q0), device=dev)
        x0 = rand_rows(q0, (64, 1 << 12))
        f0, y0 = torch.empty_like(x0), torch.empty_like(x0)

        def cfg0():
            c0ctx.ntt(x0, q0, out=f0)
            c0ctx.ntt(f0, q0, inverse=True, out=y0)
        ms0 = timed(cfg0, 20)
        # the same step replayed from a CUDA graph (launch-latency bound: 4 small launches)
        ms0g = None
        try:
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                cfg0()
            ms0g = timed(graph.replay, 20)
            del graph
        except Exception:
            ms0g = None
        sweep["config0"] = {"workload": "fwd+inv NTT, N=2^12, one 30-bit prime, batch 64 "
                                        "(BASELINE configs[0])",
                            "limb_ntt_kops": 2 * 64 * world / (ms0 / 1e3) / 1e3,
                            "us_per_step": ms0 * 1e3,
                            "cuda_graph": None if ms0g is None else {
                                "limb_ntt_kops": 2 * 64 * world / (ms0g / 1e3) / 1e3,
                                "us_per_step": ms0g * 1e3}}
        for logn in range(12, 17):
            nn = 1 << logn
            qs = generate_primes(nn, [29, 29])
            sctx = DeviceContext.get(nn, tuple(qs), device=dev)
            bb = (1 << 25) // nn
            xs = rand_rows(qs, (bb, nn))
            fs = torch.empty_like(xs)
            ms_s = timed(lambda: sctx.ntt(xs, qs, out=fs), 5)
            sweep[f"N=2^{logn}"] = {"limb_ntt_kops": 2 * bb * world / (ms_s / 1e3) / 1e3,
                                    "batch": bb, "plan": list(sctx.plan)}
            del xs, fs

    # HBM-bound kernels (element-wise, automorphism, tensor product, base
    # conversion) on the configs[1] buffers: achieved GB/s of ALGORITHMIC bytes
    # (each operand read once, each result written once) vs the measured copy
    # bandwidth.  Inputs >= 1.4 GiB per buffer (> L2).
    hbm = None
    if args.hbm_kernels:
        from paper_2212_14191_b200 import _lib as LIB
        from paper_2212_14191_b200.device import _ptr, _stream
        hbm = []
        coeffs = L * B * N
        ym = torch.empty_like(x)

        def rec(name, fn, nbytes, reps=10):
            ms = timed(fn, reps)
            hbm.append({"kernel": name, "ms": ms, "bytes": nbytes, "gbs": nbytes / ms / 1e6})
        rec("hada_mult (tfhe_eltwise MUL)", lambda: ctx.eltwise(LIB.OP_MUL, x, f, primes, out=ym),
            12 * coeffs)
        rec("ele_add (tfhe_eltwise ADD)", lambda: ctx.eltwise(LIB.OP_ADD, x, f, primes, out=ym),
            12 * coeffs)
        rec("automorphism NTT-domain (tfhe_automorphism)",
            lambda: ctx.automorphism(x, 5, True, primes, out=ym), 8 * coeffs)
        half = B // 2
        ct0 = x.view(L, 2, half, N).transpose(0, 1).contiguous()
        ct1 = f.view(L, 2, half, N).transpose(0, 1).contiguous()
        tp = torch.empty((3, L, half, N), dtype=torch.int32, device=dev)

        def tensor():
            LIB.check(ctx.lib.tfhe_tensor_product(ctx.handle, _ptr(ct0), _ptr(ct1), 0, L, half,
                                                  _ptr(tp), _stream(dev)), "tensor")
        rec("hmult tensor product (tfhe_tensor_product)", tensor, 28 * L * half * N)
        del ct0, ct1, tp
        # alpha = 9 base conversion (p_dnum5 ModUp slice: 9 sources -> 54 targets)
        pd = CkksParams.from_preset("p_dnum5")
        ckd = CkksContext(pd, device=dev)
        ext5 = tuple(pd.chain.q) + tuple(pd.chain.p)
        Bb = 32
        src = rand_rows(pd.chain.q[:pd.alpha], (Bb, N))
        dst = torch.empty((len(ext5), Bb, N), dtype=torch.int32, device=dev)
        rec(f"fast_basis_conv alpha={pd.alpha} -> {len(ext5)} targets (tfhe_bconv, int8 TC)",
            lambda: ckd.dev.bconv(src, pd.chain.q[:pd.alpha], ext5, out=dst),
            4 * (pd.alpha + len(ext5)) * Bb * N)
        del src, dst, ym, ckd

    # end to end through the reference-facing API (batched_apply) with pinned host buffers
    table = TwiddleTable(N, primes, device=dev)
    table._ctx = ctx
    host_in = torch.empty((L, B, N), dtype=torch.int32, pin_memory=True)
    host_in.copy_(x)
    e2e_steps = max(1, min(args.steps, 3))
    buf = BatchBuffer(data=host_in, basis=primes, domain="coeff")
    # warm-up = the timed loop itself, so the pinned result buffers the API
    # returns are in torch's host caching allocator (steady state)
    for _ in range(2):
        out = batched_apply(buf, "ntt", table=table)
        back = batched_apply(out, "intt", table=table)
    torch.cuda.synchronize()
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        out = batched_apply(buf, "ntt", table=table)        # H2D / NTT / D2H streamed
        back = batched_apply(out, "intt", table=table)       # H2D / INTT / D2H streamed
    torch.cuda.synchronize()
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    e2e_ok = bool(torch.equal(back.data, host_in))
    e2e_value = 2 * L * B * e2e_steps * world / e2e_s / 1e3
    bytes_per_call = L * B * N * 4
    # the e2e ceiling: raw concurrent H2D + D2H copy bandwidth over the same
    # pinned buffers (64 MiB chunks on two streams)
    duplex = None
    if rank == 0:
        dst_host = back.data if isinstance(back.data, torch.Tensor) else None
        if dst_host is not None and dst_host.is_pinned():
            hin, hout = host_in.view(-1), dst_host.view(-1)
            din = x.view(-1)
            s_up, s_dn = torch.cuda.Stream(), torch.cuda.Stream()
            step = 16 << 20   # int32 words per chunk (64 MiB)
            for rep in range(2):
                torch.cuda.synchronize()
                t1 = time.perf_counter()
                for off in range(0, hin.numel(), step):
                    with torch.cuda.stream(s_up):
                        din[off:off + step].copy_(hin[off:off + step], non_blocking=True)
                    with torch.cuda.stream(s_dn):
                        hout[off:off + step].copy_(din[off:off + step], non_blocking=True)
                torch.cuda.synchronize()
                duplex = 2 * bytes_per_call / (time.perf_counter() - t1) / 1e9

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    peak = int8_peak_tops(torch)
    peak_src = "measured: torch._int_mm int8 8192^3 best of 10 on this GPU"
    if peak is None:
        peak = 2 * 1617.8
        peak_src = "derived: 2 x MEASURED_PEAKS.json bf16_tflops (int8 dense = 2x bf16)"
    # DRAM bytes per launch of the dominant kernel / per NTT call, from one
    # ncu capture of this configuration (profiles/ntt_dram_traffic.json)
    traffic, traffic_call = None, None
    tpath = os.path.join(ROOT, "profiles", "ntt_dram_traffic.json")
    if os.path.exists(tpath):
        try:
            with open(tpath) as fh:
                t = json.load(fh)
            if t.get("batch") == B and t.get("limbs") == L and \
                    tuple(t.get("transform_plan", ())) == tuple(kplan):
                traffic_call = t.get("bytes_per_ntt_call")
                cols = [r for r in t.get("launches", []) if "col_kernel" in r["kernel"]]
                if cols:
                    traffic = sum(r["dram_read_bytes"] + r["dram_write_bytes"]
                                  for r in cols) / len(cols)
        except Exception:
            traffic, traffic_call = None, None
    hpeak, hsrc = 6546.6, "fallback (B200_PROFILING.md)"
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            hpeak, hsrc = float(json.load(fh)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        pass
    # which roof binds this factorisation: int8 time vs compulsory-byte time per limb
    t_tensor, t_hbm = ops_per_limb / (peak * 1e12), 8 * N / (hpeak * 1e9)
    hbm_bound = t_hbm >= 0.8 * t_tensor
    rates = cpu_oracle_rate(primes, args.cpu_members) if world == 1 and args.cpu_members > 0 \
        else None
    # Roofline of the DOMINANT kernel of the step, timed live: its average
    # launch duration from the events the library recorded around every
    # launch in the timed region (tfhe_profile_*, on the launching stream).
    # Three-factor plan: the column pass (1024-point column transforms, fwd
    # and inv) reads the u32 limb rows and writes P^T -- 8 N algorithmic bytes
    # per limb per launch, L*B limbs per launch; the row pass reads P^T and
    # writes the output (the same 8 N).  The call-level figure beside it counts
    # only the compulsory 8 N per limb-NTT of the whole call (two passes).
    fam = {}
    for name, (cnt, tot) in ktime.times.items():
        key = name.split("<")[0]
        c0, t0 = fam.get(key, (0, 0.0))
        fam[key] = (c0 + cnt, t0 + tot)
    step_kernel_ms = sum(t for _, t in fam.values())
    kern_rows = {}
    for key, (cnt, tot) in fam.items():
        avg = tot / max(cnt, 1)
        gbs = L * B * 8 * N / (avg / 1e3) / 1e9
        kern_rows[key] = {"launches": cnt, "avg_launch_ms": avg, "share_of_step": tot / max(ms, 1e-9),
                          "achieved_gbs": gbs, "frac": gbs / hpeak}
    dom = max(fam, key=lambda k: fam[k][1]) if fam else None
    call_level = {"achieved": achieved_gbs, "unit": "GB/s", "frac": achieved_gbs / hpeak,
                  "algorithmic": f"8*N = {8 * N} B per limb-NTT over the whole call "
                                 f"({L * B} limbs per call, two launches)",
                  "traffic": traffic_call}
    tensor_view = {"achieved": achieved_tops, "peak": peak, "unit": "TOPS (int8)",
                   "frac": achieved_tops / peak, "peak_source": peak_src,
                   "algorithmic": f"32*N*(k0+k1+k2), plan {list(kplan)}: "
                                  f"{ops_per_limb / 1e9:.3f} G int8-ops per limb-NTT"}
    if dom is not None and hbm_bound:
        d = kern_rows[dom]
        roofline = {"bound": "hbm", "achieved": d["achieved_gbs"], "peak": hpeak, "unit": "GB/s",
                    "frac": d["frac"], "traffic": traffic,
                    "kernel": f"{dom} (fwd + inv launches)",
                    "algorithmic": f"8*N = {8 * N} B per limb (u32 rows in, P^T out) x {L * B} "
                                   "limbs per launch",
                    "launch_ms": d["avg_launch_ms"], "launches": d["launches"],
                    "peak_source": hsrc,
                    "timing": "CUDA events around every launch in the timed region, "
                              "on the launching stream (tfhe_profile_read)",
                    "kernels": kern_rows, "kernels_share_of_timed_region": step_kernel_ms / ms,
                    "call_level": call_level,
                    "tensor_view": tensor_view}
    elif hbm_bound:
        roofline = dict(call_level, bound="hbm", peak=hpeak, peak_source=hsrc,
                        kernel="one NTT call", tensor_view=tensor_view)
    else:
        roofline = {"bound": "tensor", "achieved": achieved_tops, "peak": peak,
                    "unit": "TOPS (int8)", "frac": achieved_tops / peak, "traffic": traffic_call,
                    "algorithmic": f"32*N*(k0+k1+k2), plan {list(kplan)}: "
                                   f"{ops_per_limb / 1e9:.3f} G int8-ops per limb-NTT x "
                                   f"{L * B} limbs per call",
                    "peak_source": peak_src, "kernels": kern_rows}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u32", "data": "synthetic",
        "config": dict(headline_config(L, B, world, (n1, n2)),
                       transform_plan=list(kplan)),
        "poly_ntt_kops": value / L,
        "parity_spot_check": parity,
        "roofline": roofline,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 2 * bytes_per_call,
                "d2h_bytes_per_step": 2 * bytes_per_call, "steps": e2e_steps,
                "api": "batched_apply(BatchBuffer(pinned host), 'ntt'/'intt')",
                "roundtrip_exact": e2e_ok,
                "pcie_duplex_gbs": duplex,
                "frac_of_pcie_duplex": (4 * bytes_per_call * e2e_steps / e2e_s / 1e9 / duplex)
                if duplex else None},
        "gpu_launches": sum(c for c, _ in fam.values()) if fam else 4 * args.steps,
        "clocks": clk.summary(),
    }
    if hm:
        line["hmult_kops"] = hm["hmult_kops"]
        line["hmult"] = {"workload": f"HMULT+relin (keyswitch ModUp/ModDown)+rescale, N=2^16, "
                                     f"{PRESET} (L=44, K=1, dnum=45), batch {hm['batch_per_gpu']}"
                                     " per GPU (BASELINE configs[2])",
                         "ms_per_batch": hm["ms_per_batch"],
                         "ops_per_s": hm["hmult_kops"] * 1e3,
                         "hmult_relin_only_per_s": hm["hmult_relin_only_per_s"],
                         "hmult_then_rescale_per_s": hm["hmult_then_rescale_per_s"],
                         "api": "CkksContext.hmult_rescale_batch (fused ModDown+rescale)",
                         "rescale_per_s": hm["rescale_per_s"]}
        # whole-operator roofline: int8 tensor work of the limb transforms an
        # HMULT+relin+rescale needs ALGORITHMICALLY (INTT l+1, ModUp raises of
        # each one-limb slice to the l+K other ext primes, ModDown INTT 2K,
        # top-row NTT 2 + INTT 2, merged ModDown/rescale NTT 2l); the device
        # also computes the l+1 own-slice raises it then skips (not counted)
        l1, K = L, len(params.chain.p)
        transforms = l1 + l1 * (l1 - 1 + K) + 2 * K + 2 + 2 + 2 * (l1 - 1)
        computed = transforms + l1
        hm_tops = hm["hmult_kops"] * 1e3 * transforms * ops_per_limb / 1e12
        line["hmult"]["batch_sweep_per_s"] = hm["batch_sweep_per_s"]
        line["hmult"]["parity_spot_check"] = hm_check
        # the operator is a chain of limb-transforms: its rate against this
        # GPU's own batched-NTT rate (the headline `value`) says how much the
        # key-switch epilogues, base conversions and element-wise passes cost
        # on top of the transforms
        xf_rate = hm["hmult_kops"] * 1e3 * transforms
        line["hmult"]["roofline"] = {
            "bound": "hbm" if hbm_bound else "tensor",
            "limb_transforms_per_s": xf_rate,
            "frac_of_ntt_rate": xf_rate / (value * 1e3),
            "tensor_view": {"achieved": hm_tops, "peak": peak, "unit": "TOPS (int8)",
                            "frac": hm_tops / peak},
            "algorithmic": f"{transforms} limb-transforms x {ops_per_limb / 1e9:.3f} G int8-ops "
                           f"per HMULT+relin+rescale ({computed} computed), plan {list(kplan)}"}
        line["hrotate"] = {"workload": f"HROTATE r=1 (automorphism + keyswitch), N=2^16, {PRESET}"
                                       f", batch {hm['batch_per_gpu']} per GPU (configs[3])",
                           "ops_per_s": hm["hrotate_per_s"],
                           "ms_per_batch": hm["hrotate_ms_per_batch"]}
        line["mixed"] = {"workload": "HMULT -> rescale -> HROTATE per ciphertext, N=2^16, "
                                     f"{PRESET}, batch-sharded x{world} (configs[4])",
                         "ciphertexts_per_s": hm["mixed_ct_per_s"],
                         "ms_per_batch": hm["mixed_ms_per_batch"]}
    if sa:
        sa["ntt_roofline"].update(peak=hpeak, frac=sa["ntt_roofline"]["achieved"] / hpeak,
                                  peak_source=hsrc)
        line["set_a"] = sa
    if d5:
        line["p_dnum5"] = d5
    if sweep:
        line["ntt_sweep"] = sweep
    if bsweep:
        line["batch_sweep"] = {"workload": f"fwd+inv NTT, N=2^16, {PRESET} chain ({L} limbs), "
                                           "batch B per GPU (BASELINE configs[1] sweep)",
                               "unit": UNIT, "by_batch": bsweep}
    if hbm:
        for h in hbm:
            h["frac"] = h["gbs"] / hpeak
        line["hbm_kernels"] = {"peak_gbs": hpeak, "peak_source": hsrc, "kernels": hbm}
    if rates:
        r, dt, threads = rates
        line["cpu_baseline"] = {
            "value": r / 1e3, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"C oracle (oracle/tfhe_oracle.c, OpenMP, in place), fwd+inv over {L} "
                      f"limbs x {args.cpu_members} members ({2 * L * args.cpu_members} "
                      f"limb-NTTs) in {dt:.1f}s"}
        if args.cpu_numpy:
            try:
                line["cpu_baseline"]["python_reference_algorithm"] = cpu_numpy_butterfly(primes)
            except Exception as exc:   # never lose the bench line to the extra leg
                line["cpu_baseline"]["python_reference_algorithm"] = {"error": str(exc)[:200]}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def launch_ranks(args):
    """`bench.py --gpus N` outside torchrun: start N ranks (one per GPU) with
    torch.distributed.run on 127.0.0.1, the same command line the driver
    uses, and pass rank 0's JSON line through."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "8"))
    return subprocess.call(cmd, env=env)


def run_dry(args):
    """--dry-run: rank plumbing only (no GPU work): every rank joins the
    process group and rank 0 prints the ranks it sees (tests run it on CPU
    with gloo)."""
    import torch.distributed as dist
    rank, world = _env_int("RANK", 0), _env_int("WORLD_SIZE", 1)
    ranks = [{"rank": rank, "local_rank": _env_int("LOCAL_RANK", 0), "pid": os.getpid()}]
    if world > 1:
        dist.init_process_group("gloo")
        got = [None] * world
        dist.all_gather_object(got, ranks[0])
        ranks = got
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "requested": args.gpus,
                          "ranks": ranks}), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--batch", type=int, default=128)
    ap.add_argument("--hmult-batch", type=int, default=128)
    ap.add_argument("--cpu-members", type=int, default=32)
    ap.add_argument("--set-a-batch", type=int, default=4096)
    ap.add_argument("--hbm-kernels", type=int, default=1)
    ap.add_argument("--dnum5-batch", type=int, default=16)
    ap.add_argument("--sweep", type=int, default=1)
    ap.add_argument("--batch-sweep", type=int, default=1)
    ap.add_argument("--hmult-check", type=int, default=1)
    ap.add_argument("--cpu-numpy", type=int, default=1)
    ap.add_argument("--dry-run", action="store_true")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return launch_ranks(args)
    if args.dry_run:
        return run_dry(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
