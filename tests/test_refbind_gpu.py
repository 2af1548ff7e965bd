"""The reference's OWN replanning loop on the device path (INTEGRATION.md,
Option 2 = ``paper_2605_13778_b200/refbind.py``): the unmodified reference
package (``baseline/_ref``, the offline install of the reference, see
DESIGN.md) runs ``bench.harness.run_single_episode`` (harness.py:439-460 ->
runtime.run_episode, runtime.py:219-334) on the reference-trained cfg2 models
(tests/golden/cfg2_*.ckpt, loaded by the reference's bench/checkpoint.py)
twice -- as shipped (numpy) and with its hot-path globals rebound to the
device path (fp64) -- and every RoundRecord (path, planned, prefix, branch
prefixes, switch, executed, stall ticks, seeds, terminal) and the episode
stats must be identical. Skips when baseline/_ref is absent."""

import sys
from pathlib import Path

import pytest

from conftest import cuda_ok

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"
GOLDEN = Path(__file__).resolve().parent / "golden"

pytestmark = [
    pytest.mark.gpu,
    pytest.mark.skipif(not cuda_ok(), reason="needs CUDA"),
    pytest.mark.skipif(not (REF / "specflow").is_dir(), reason="baseline/_ref (reference install) absent"),
]


@pytest.fixture(scope="module")
def ref():
    sys.path.insert(0, str(REF))
    import specflow  # noqa: F401
    from specflow import draft, flowpolicy, runtime, verifier
    from specflow.bench import checkpoint, harness
    from specflow.bench.config import DEFAULT_CONFIG
    assert str(REF) in str(Path(runtime.__file__).resolve()), "imported a different specflow"
    encoder, field, standardizer, _ = checkpoint.load_main_checkpoint(GOLDEN / "cfg2_main.ckpt")
    draft_model, _ = checkpoint.load_draft_checkpoint(GOLDEN / "cfg2_draft.ckpt")
    models = runtime.Models(encoder=encoder, field=field, standardizer=standardizer, draft=draft_model)
    return dict(draft=draft, flowpolicy=flowpolicy, runtime=runtime, verifier=verifier, harness=harness,
                config=DEFAULT_CONFIG, models=models, field=field)


def _episodes(r, seeds):
    out = []
    for s in seeds:
        stats, records = r["harness"].run_single_episode(r["config"], r["models"], s, "demo", "large")
        out.append((stats, [rec.to_record() for rec in records]))
    return out


@pytest.mark.parametrize("seeds", [(7, 11, 23)])
def test_reference_run_episode_on_device_path(ref, seeds):
    from paper_2605_13778_b200 import _capi, refbind

    field = ref["field"]
    n0 = field.eval_count
    want = _episodes(ref, seeds)
    host_evals = field.eval_count - n0
    restore = refbind.install(ref["verifier"], ref["flowpolicy"], ref["draft"], ref["runtime"], "fp64")
    try:
        _capi.launch_count(reset=True)
        n1 = field.eval_count
        got = _episodes(ref, seeds)
        launches = _capi.launch_count()
        dev_evals = field.eval_count - n1
    finally:
        restore()
    assert ref["runtime"].verify is ref["verifier"].verify and ref["runtime"].propose is ref["draft"].propose
    assert launches > 0, "the patched loop launched no device kernels"
    assert dev_evals == host_evals  # the reference's cost contract (K per verify, N per denoise)
    paths = set()
    for (ws, wr), (gs, gr) in zip(want, got):
        assert len(gr) == len(wr)
        for a, b in zip(wr, gr):
            assert a == b, (a, b)
            paths.add(a["path"])
        assert gs == ws
    assert len(paths) >= 3, paths  # full / periodic / accepted / fallback rounds all exercised
