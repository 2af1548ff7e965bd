import sys, ctypes, numpy as np, torch
sys.path.insert(0, '.')
from paper_2605_13778_b200 import _capi, precision
from paper_2605_13778_b200.actions import ChannelLayout
from paper_2605_13778_b200.flowpolicy import ConditioningCache, VelocityField
from paper_2605_13778_b200.nets import init_mlp
from paper_2605_13778_b200.verifier import VerifierConfig, tiny_flash_round
rng = np.random.default_rng(0)
h, lay = 50, ChannelLayout(3, 3); d = lay.dim
field_net = init_mlp([h*d+1+39+3, 256, 256, h*d], rng); draft_net = init_mlp([10, 160, 160, h*d], rng)
field = VelocityField(net=field_net, horizon=h, dim=d, emb_dim=39, state_dim=3, layout=lay)
feats, emb, state = rng.normal(size=10), rng.normal(size=39), rng.normal(size=3)
eps = rng.normal(size=(h, d)); cfg = VerifierConfig(timesteps=(0.25, 0.5, 0.75), delta=1.42, gripper_window=24)
lib = _capi.lib()
for prec in ("fp32", "fp64"):
    with precision(prec):
        for _ in range(20): tiny_flash_round(field, draft_net, feats, ConditioningCache(emb), state, eps, cfg, -1.0, lay)
        lib.sf_tiny_trace(1, None)
        rows = []
        for _ in range(50):
            tiny_flash_round(field, draft_net, feats, ConditioningCache(emb), state, eps, cfg, -1.0, lay)
            buf = np.zeros(32, np.uint64); lib.sf_tiny_trace(1, buf.ctypes.data); rows.append(buf.astype(np.int64))
        lib.sf_tiny_trace(0, None)
        r = np.median(np.stack([x - x[0] for x in rows]), axis=0) * 1e-3
        names = {1: "prologue (weights issued)", 8: "draft L0", 9: "draft L1", 10: "draft L2", 2: "packed", 16: "field L0", 17: "field L1", 18: "field L2", 3: "epilogue done"}
        print(prec, " ".join(f"{names[k]}={r[k]:.2f}" for k in (1, 8, 9, 10, 2, 16, 17, 18, 3))); pass
