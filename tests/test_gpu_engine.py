"""End-to-end GPU parity: whole workloads through librx (C++ tree + kernels via
the C ABI) against the oracle driver (Python tree + fp64 attention).

* tree trace bit-exact (every matched length, slot vector, eviction run);
* attention outputs within max-abs 2e-2 / mean-abs 2e-3 on every row for the
  small configs, and on sampled rows at the full C5 / C3 sizes (the launch
  configuration bench.py times).
"""
import numpy as np
import pytest
import torch

from oracle.driver import OracleEngine
from rxgen import workloads

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2312_07104_b200.engine import Engine, plan_and_bank

MAX_ABS, MEAN_ABS = 2e-2, 2e-3


def _run_gpu(wl, q_scale=1.0, policy="lspf"):
    plan, bank = plan_and_bank(wl, "cuda", q_scale=q_scale, policy=policy)
    e = Engine(wl, "cuda", record=True, keep_outputs=True, policy=policy)
    e.run_workload(bank)
    torch.cuda.synchronize()
    return e


def _outputs_by_key(e):
    """engine outputs -> {("extend", call, req, j) / ("decode", call, req): bf16 row}"""
    ext = [x for x in e.outputs if x[0] == "extend"]
    dec = [x for x in e.outputs if x[0] == "decode"]
    return ext, dec


def _compare(o_eng, wl, rows_ext, rows_dec, q_scale=1.0, policy="lspf"):
    ext_s = {}
    dec_s = {}

    def se(call, seqs):
        return rows_ext(call, seqs)

    def sd(call, step, running):
        return rows_dec(call, step, running)

    small = wl.num_slots * wl.shape.h_kv * wl.shape.head_dim <= (1 << 26)
    oe = OracleEngine(wl, sample_extend=se, sample_decode=sd, q_scale=q_scale, materialize=small, policy=policy)
    oe.run_workload()
    ext, dec = _outputs_by_key(o_eng)
    errs = []
    for key, ref in oe.outputs.items():
        if key[0] == "extend":
            _, call, bi, j = key
            o, meta = ext[call][1], ext[call][2]
            off = int(np.sum(meta["ext"][:bi]))
            got = o[off + j]
        else:
            _, call, bi = key
            got = dec[call][1][bi]
        g = got.float().cpu().double().numpy()
        errs.append(np.abs(g - ref))
    err = np.concatenate([x.ravel() for x in errs])
    assert np.isfinite(err).all()
    assert err.max() <= MAX_ABS, err.max()
    assert err.mean() <= MEAN_ABS, err.mean()
    return oe


def _all_ext(call, seqs):
    return [(i, j) for i, s in enumerate(seqs) for j in range(s.n_prompt - s.prefix_len)]


def _all_dec(call, step, running):
    return list(range(len(running)))


@pytest.mark.parametrize("q_scale", [1.0, 4.0])
def test_c1_full_parity(q_scale):
    wl = workloads.c1()
    e = _run_gpu(wl, q_scale)
    oe = _compare(e, wl, _all_ext, _all_dec, q_scale)
    assert oe.trace == e.trace


def test_c2_small_parity():
    wl = workloads.c2(n_req=6, prefix=300, new_lo=20, new_hi=150, decode=5, num_slots=8192)
    e = _run_gpu(wl)
    oe = _compare(e, wl, _all_ext, _all_dec)
    assert oe.trace == e.trace


def test_c3_small_parity():
    wl = workloads.c3(sessions=5, turns=3, in_lo=20, in_hi=140, out_lo=3, out_hi=20, num_slots=8192)
    e = _run_gpu(wl)
    oe = _compare(e, wl, _all_ext, _all_dec)
    assert oe.trace == e.trace


def test_c5_small_parity():
    wl = workloads.c5(n_req=5, prefix=700, question=40, decode=4, num_slots=8192, ragged=True)
    e = _run_gpu(wl)
    oe = _compare(e, wl, _all_ext, _all_dec)
    assert oe.trace == e.trace


def test_c5_full_size_sampled():
    """BASELINE C5 at full size (8k shared context, batch 128, 32 decode steps): sampled rows."""
    wl = workloads.c5()

    def re(call, seqs):
        if call == 0:
            return [(0, j) for j in (0, 1, 127, 4095, 8190)]
        return [(i, j) for i in (0, 77, 127) for j in (0, 63, 127)]

    def rd(call, step, running):
        return [0, 127] if call in (0, 31) else []

    e = _run_gpu(wl)
    _compare(e, wl, re, rd)


def test_c3_full_size_sampled():
    """BASELINE C3 at full size — the workload and launch configuration bench.py times (256 sessions
    x 4 turns, 786 k attention rows, 2045 decode steps): tree trace bit-exact over the whole run,
    sampled attention rows of every extend (4 requests x 3 rows) and of the first, a middle and the
    last decode step of every turn (3 requests each) within tolerance."""
    wl = workloads.c3()

    def re(call, seqs):
        out = []
        for i in (0, len(seqs) // 3, len(seqs) - 1, 97 % len(seqs)):
            n = seqs[i].n_prompt - seqs[i].prefix_len
            out += [(i, j) for j in sorted({0, n // 2, n - 1})]
        return out

    def rd(call, step, running):
        # steps 0, 255 and the last steps of a turn (batch shrinks as sessions finish)
        if step in (0, 255) or len(running) <= 2:
            return sorted({0, len(running) // 2, len(running) - 1})
        return []

    e = _run_gpu(wl)
    oe = _compare(e, wl, re, rd)
    assert oe.trace == e.trace
    assert sum(1 for k in oe.outputs if k[0] == "decode") >= 12


def test_c2_full_size_sampled():
    """BASELINE C2 at full size (Llama-2-7B 32/32/128, 5-shot prefix of 1536 tokens, batch 64, new
    U[64,192], 64 decode steps — cascade decode over the shared prefix): tree trace bit-exact over the
    whole run; every row of the hint extend at tile boundaries, first/middle/last rows of 6 requests of
    the batch extend, and 4 requests at decode steps 0, 31 and 63 within tolerance."""
    wl = workloads.c2()

    def re(call, seqs):
        if call == 0:
            return [(0, j) for j in (0, 1, 127, 128, 767, 1534)]
        out = []
        for i in (0, 1, 17, 31, 50, 63):
            n = seqs[i].n_prompt - seqs[i].prefix_len
            out += [(i, j) for j in sorted({0, n // 2, n - 1})]
        return out

    def rd(call, step, running):
        return [0, 21, 42, 63] if step in (0, 31, 63) else []

    e = _run_gpu(wl)
    oe = _compare(e, wl, re, rd)
    assert oe.trace == e.trace
    assert sum(1 for k in oe.outputs if k[0] == "decode") == 12


def test_c4_tot_full_parity():
    """C4 at full size: tree-of-thought under Alg. 1 admission with the pool at
    60% of the tree's distinct tokens (evictions between waves)."""
    wl = workloads.c4()
    e = _run_gpu(wl)
    oe = _compare(e, wl, lambda c, seqs: [(i, j) for i, s in enumerate(seqs)
                                          for j in range(s.n_prompt - s.prefix_len) if j % 7 == 0 or c > 0],
                  _all_dec)
    assert oe.trace == e.trace
    assert any(t[0] == "evict" for t in e.trace)


@pytest.mark.parametrize("policy", ["lspf", "fcfs", "random"])
def test_mix_schedule_parity(policy):
    """Scheduling ablation queue (interleaved few-shot groups, pool < the groups' prefixes):
    admission by rx_schedule under each policy, evictions and prefix recomputation between waves;
    tree trace bit-exact and every attention row within tolerance."""
    wl = workloads.mix(groups=3, per_group=6, prefix=300, q_lo=20, q_hi=60, out_lo=2, out_hi=6, num_slots=900)
    e = _run_gpu(wl, policy=policy)
    oe = _compare(e, wl, _all_ext, _all_dec, policy=policy)
    assert oe.trace == e.trace
    assert any(t[0] == "evict" for t in e.trace)


@pytest.mark.parametrize("compressed", [True, False])
def test_json_fsm_parity(compressed):
    """Regex-constrained JSON decoding (§4): compressed FSM (jump-forward segments as extend calls
    with ragged 1..k-token rows over each request's cached context) and token-by-token decoding;
    tree trace bit-exact, every attention row within tolerance."""
    wl = workloads.json_decode(n_req=6, prefix=200, doc_lo=10, doc_hi=60, compressed=compressed, num_slots=8192)
    e = _run_gpu(wl)
    # every row: prefill rows = tokens beyond the cached prefix (the start edge is appended before the
    # call); extend-step rows beyond a request's segment are skipped by the oracle
    rows = lambda c, seqs: [(i, j) for i, s in enumerate(seqs) for j in range(len(s.tokens) - s.prefix_len)]
    oe = _compare(e, wl, rows, _all_dec)
    assert oe.trace == e.trace
    n_ext = sum(1 for x in e.outputs if x[0] == "extend")
    assert (n_ext > 2) == compressed


def test_host_io_path_bitwise_equal():
    """End-to-end path (inputs prefetched H2D on a copy stream, outputs D2H on a sink stream,
    hostio.py) gives bit-identical outputs to the device-resident path, twice in a row."""
    from paper_2312_07104_b200.hostio import HostInputs, HostSink
    wl = workloads.c2(n_req=6, prefix=300, new_lo=20, new_hi=150, decode=5, num_slots=8192)
    plan, bank = plan_and_bank(wl, "cuda")
    e = Engine(wl, "cuda", keep_outputs=True)
    e.run_workload(bank)
    torch.cuda.synchronize()
    ref = [o.cpu() for _, o, _ in e.outputs]
    hb = HostInputs(bank, torch.device("cuda"), ext_depth=1, dec_block=3, dec_depth=2)
    sink = HostSink([torch.empty((len(c.hashes), wl.shape.h_q, wl.shape.head_dim), dtype=torch.bfloat16,
                                 pin_memory=True) for c in plan.calls], torch.device("cuda"))
    e2 = Engine(wl, "cuda")
    e2.sink = sink
    for _ in range(2):
        sink.reset()
        hb.reset()
        e2.reset()
        e2.run_workload(hb)
        sink.join()
        torch.cuda.synchronize()
        assert len(ref) == len(sink.out)
        for a, b in zip(ref, sink.out):
            assert torch.equal(a.view(-1), b.view(-1))


def test_duplicate_slots_freed_and_reused_mid_phase():
    """Requests with the SAME uncached prompt in one batch (no hint): each computes the prompt; the
    first to finish caches it and every later finisher frees its duplicate slots (R10), which the
    next decode step reallocates at once (smallest free first, R8) while the previous step's
    kernel may still be draining (programmatic dependent launch): the append into a reused slot
    must come after the dependency wait.  Every row vs the oracle, trace bit-exact."""
    from rxgen.workloads import Request, Workload, Shape
    rng = np.random.default_rng(11)
    prompt = rng.integers(1, 30000, 300).astype(np.int32)
    reqs = [Request(prompt.copy(), n, f"d{n}") for n in (1, 2, 3, 5, 8, 13, 21, 34)]
    wl = Workload("DUP", Shape(32, 8, 128), 4096, 32000, 11, [("batch", reqs)])
    e = _run_gpu(wl)
    oe = _compare(e, wl, _all_ext, _all_dec)
    assert oe.trace == e.trace
    assert any(t[0] == "insert" and t[3] > 0 for t in e.trace)      # duplicates were freed


def test_host_generated_bank_bitwise_equal():
    """InputBank(host=True) (numpy generator + one H2D, used by smoke()) holds exactly the device
    generator's bits."""
    from paper_2312_07104_b200.engine import InputBank
    wl = workloads.c1()
    plan, bank = plan_and_bank(wl, "cuda")
    hb = InputBank(plan.calls, wl.shape, plan.heads_q, plan.heads_kv, "cuda", host=True)
    for a, b in zip(bank.ext + bank.dec, hb.ext + hb.dec):
        for x, y in zip(a, b):
            assert x.shape == y.shape and torch.equal(x, y)
