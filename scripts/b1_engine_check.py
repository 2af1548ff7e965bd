"""Batch-1 engine check (GPU): the one-launch Euler full round vs the per-op
graph path (SF_NO_B1ENGINE) on the same inputs, p50 timings of both, and an
optional per-stage trace (SF_B1_TRACE=1 -> stage durations of CTA groups).

python scripts/b1_engine_check.py [--trace]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_13778_b200 import pi0  # noqa: E402


def run(ae, start, state, n=10):
    chunk, status = ae.denoise_batch(start, state, n)
    torch.cuda.synchronize()
    return chunk.clone(), status.clone()


def p50(ae, start, state, iters=20):
    ts = []
    for _ in range(iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ae.denoise_batch(start, state, 10)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def main():
    trace = "--trace" in sys.argv
    ae = pi0.ActionExpert(pi0.PI0, seed=0, n_envs=1, kv_seed=1)
    rng = np.random.default_rng(301)
    start = torch.from_numpy(rng.standard_normal((1, 50, 32)).astype(np.float32)).cuda()
    state = torch.from_numpy(rng.standard_normal((1, 32)).astype(np.float32)).cuda()
    os.environ["SF_NO_B1ENGINE"] = "1"
    ref, rst = run(ae, start, state)
    t_ref = p50(ae, start, state)
    del os.environ["SF_NO_B1ENGINE"]
    t0 = time.time()
    got, gst = run(ae, start, state)
    print(f"engine first call {time.time() - t0:.2f} s, status {gst.tolist()} (graph path {rst.tolist()})")
    got2, _ = run(ae, start, state)
    d = (got - ref).abs()
    print(f"engine vs graph path: max |diff| {d.max().item():.3e}, max |ref| {ref.abs().max().item():.3e}, "
          f"rel norm {(torch.linalg.norm(got - ref) / torch.linalg.norm(ref)).item():.3e}; "
          f"run-to-run max |diff| {(got2 - got).abs().max().item():.3e}")
    t_eng = p50(ae, start, state)
    print(f"full round p50: graph path {t_ref:.3f} ms, engine {t_eng:.3f} ms")
    if trace:
        os.environ["SF_B1_TRACE"] = "1"
        run(ae, start, state)
        del os.environ["SF_B1_TRACE"]
        from paper_2605_13778_b200 import _capi  # noqa: F401
        # dbg buffer is internal; exported via sf_ae_b1_trace
        import ctypes
        L = 18
        SPL = int(os.environ.get("SF_B1_SPL", "5"))
        n_st = (2 + SPL * L) * 10 + 1
        buf = np.zeros((148, n_st, 8), np.uint64)
        rc = _capi.lib().sf_ae_b1_trace(ae._h, buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.size))
        assert rc == 0, rc
        t0 = buf[:, :, 0].astype(np.int64)
        base = t0[:, 1:].min()
        names = ["E", "QKV", "ATT", "O", "GU", "DN"]
        per = 2 + SPL * L
        # stage start (max over CTAs of barrier pass) -> duration until next stage start
        starts = t0.max(axis=0)
        durs = np.diff(starts) * 1e-3
        kinds = []
        for st in range(n_st - 1):
            j = st % per
            kinds.append("E" if j == 0 else ("HEAD" if j == per - 1 else names[1 + (j - 1) % SPL]))
        kinds = np.array(kinds)
        print("stage durations (us, barrier-to-barrier, median over steps/layers):")
        for k in ["E", "QKV", "QF", "ATT", "O", "GU", "DN", "HEAD"]:
            sel = durs[kinds == k]
            if sel.size == 0:
                continue
            print(f"  {k:5s} n={sel.size:4d} median {np.median(sel):7.2f} mean {sel.mean():7.2f} max {sel.max():7.2f}")
        print(f"  total {durs.sum():.1f} us over {n_st - 1} stages")
        # phases inside a stage for the working CTAs: 0 barrier pass, 1 operand ready, 2 acc ready, 3 done
        # per stage kind: which CTAs finish last (done - stage start of the slowest CTA)
        for k in ["QKV", "QF", "ATT", "O", "GU", "DN"]:
            sts = [st for st in range(per, 2 * per) if kinds[st] == k]
            if not sts:
                continue
            done = np.stack([(buf[:, st, 3].astype(np.int64) - buf[:, st, 0].astype(np.int64).max()) * 1e-3
                             for st in sts])  # [layers][cta]
            med = np.median(done, axis=0)
            order = np.argsort(-med)[:6]
            print(f"  {k:4s} slowest CTAs (median done after the last barrier pass, us): "
                  + ", ".join(f"{c}:{med[c]:.2f}" for c in order))
        for k, cta in [("QKV", 0), ("QKV", 19), ("ATT", 80), ("ATT", 107), ("O", 0), ("GU", 30), ("DN", 0)]:
            sts = [st for st in range(per, 2 * per) if kinds[st] == k]
            ph = []
            for st in sts:
                r = buf[cta, st].astype(np.int64)
                ph.append([(r[z] - r[0]) * 1e-3 if r[z] else np.nan for z in range(1, 8)])
            ph = np.nanmedian(np.array(ph), axis=0)
            print(f"  {k:4s} CTA {cta:3d}: " + "  ".join(f"s{z + 1} {ph[z]:.2f}" for z in range(7)))


if __name__ == "__main__":
    main()
