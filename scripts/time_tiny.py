"""Device timing of the tiny-path kernels (cfg1 shapes), CUDA events.

Reports (a) single-launch latency (event pair around one launch, includes the
host submit), (b) back-to-back throughput (1000 launches between two events),
(c) the python API end-to-end round, and the SM clock seen while looping.
"""

import subprocess
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np
import torch

from paper_2605_13778_b200 import _capi, _device, precision
from paper_2605_13778_b200.actions import ChannelLayout
from paper_2605_13778_b200.flowpolicy import ConditioningCache, VelocityField
from paper_2605_13778_b200.nets import init_mlp
from paper_2605_13778_b200.verifier import VerifierConfig, make_cfg, tiny_flash_round


def sm_clock():
    try:
        out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits"],
                             capture_output=True, text=True, timeout=10).stdout.strip()
        return out
    except Exception:
        return "?"


def main():
    rng = np.random.default_rng(0)
    h, lay = 50, ChannelLayout(3, 3)
    d = lay.dim
    field_net = init_mlp([h * d + 1 + 39 + 3, 256, 256, h * d], rng)
    draft_net = init_mlp([10, 160, 160, h * d], rng)
    enc_net = init_mlp([7, 64, 32], rng)
    field = VelocityField(net=field_net, horizon=h, dim=d, emb_dim=39, state_dim=3, layout=lay)
    lib = _capi.lib()
    for prec in ("fp32", "fp64"):
        with precision(prec):
            dt = _device.tdtype()
            dev = torch.device("cuda")
            feats = torch.randn(10, dtype=dt, device=dev)
            emb = torch.randn(39, dtype=dt, device=dev)
            state = torch.randn(3, dtype=dt, device=dev)
            eps = torch.randn(h * d, dtype=dt, device=dev)
            out = torch.empty(h * d * 5, dtype=dt, device=dev)
            words = torch.empty(32, dtype=torch.int32, device=dev)
            cfg = make_cfg(VerifierConfig(timesteps=(0.25, 0.5, 0.75), delta=1.42), -1.0)
            o = _capi.SfVerifyOut(out.data_ptr(), out.data_ptr() + h * d * dt.itemsize,
                                  out.data_ptr() + 4 * h * d * dt.itemsize,
                                  words.data_ptr() + 32, words.data_ptr())
            s = torch.cuda.current_stream().cuda_stream
            dd, fd, ed = draft_net.device().desc, field_net.device().desc, enc_net.device().desc

            def spec():
                _capi.check(lib.sf_tiny_flash_round(_device.code(), dd, feats.data_ptr(), fd,
                                                    emb.data_ptr(), 39, state.data_ptr(), 3,
                                                    eps.data_ptr(), h, d, 6, cfg, o, s))

            def full(n=10):
                _capi.check(lib.sf_tiny_full_round(_device.code(), ed, feats.data_ptr(), 39, fd,
                                                   state.data_ptr(), 3, eps.data_ptr(), h, d, n,
                                                   out.data_ptr(), None, words.data_ptr(), s))

            for name, fn in (("spec", spec), ("full", full), ("full_n1", lambda: full(1)),
                             ("encode_only", lambda: full(0))):
                for _ in range(50):
                    fn()
                torch.cuda.synchronize()
                times = []
                for _ in range(200):
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    fn()
                    b.record()
                    b.synchronize()
                    times.append(a.elapsed_time(b) * 1e3)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                n = 2000
                a.record()
                for _ in range(n):
                    fn()
                b.record()
                clk = sm_clock()
                b.synchronize()
                print(f"{prec} {name:12s}: single p50 {np.median(times):7.1f} us | back-to-back "
                      f"{a.elapsed_time(b) * 1e3 / n:7.1f} us/launch | sm clock {clk} MHz")
            fe, em, st, ep = (np.asarray(x.cpu(), np.float64) for x in (feats, emb, state, eps))
            vcfg = VerifierConfig(timesteps=(0.25, 0.5, 0.75), delta=1.42)
            cache = ConditioningCache(em)
            for _ in range(20):
                tiny_flash_round(field, draft_net, fe, cache, st, ep.reshape(h, d), vcfg, -1.0, lay)
            t = []
            for _ in range(300):
                t0 = time.perf_counter()
                tiny_flash_round(field, draft_net, fe, cache, st, ep.reshape(h, d), vcfg, -1.0, lay)
                t.append((time.perf_counter() - t0) * 1e6)
            print(f"{prec} e2e flash_round via python API: p50 {np.median(t):.1f} us")


if __name__ == "__main__":
    main()
