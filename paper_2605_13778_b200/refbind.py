"""Binding of the reference ``specflow`` package onto the device path
(Option 2).

``install(verifier, flowpolicy, draft, runtime)`` takes the reference's own
modules and rebinds the hot-path globals its runtime calls through
(``runtime.py:29-31`` imports ``propose`` / ``verify`` by name;
``flowpolicy.denoise`` calls the module-level ``integrate_flow``,
flowpolicy.py:295-305):

* ``verifier.verify`` / ``runtime.verify``     -> ``verifier.verify`` here
  (verifier.py:109-150), the reference's ``VerifierReport`` type returned;
* ``flowpolicy.integrate_flow``                -> ``flowpolicy.integrate_flow``
  here (flowpolicy.py:273-292);
* ``draft.propose`` / ``runtime.propose``      -> ``draft.propose`` here
  (draft.py:57-61).

MLP fields / drafts share the reference's numpy weights (uploaded once per
precision and cached by object identity); fields of any other type keep the
generic protocol (evaluated where they live, epilogue on the device). The
reference's ``eval_count`` cost contract is kept on the reference field.
Returns a ``restore()`` callable that puts the original globals back.

Nothing here imports the reference: the caller passes its modules in.
"""

from __future__ import annotations

from . import draft as _dd
from . import flowpolicy as _df
from . import verifier as _dv
from ._device import set_precision
from .nets import Mlp


def _device_mlp(ref_mlp) -> Mlp:
    return Mlp(weights=ref_mlp.weights, biases=ref_mlp.biases)


def install(verifier, flowpolicy, draft, runtime, precision: str = "fp64"):
    set_precision(precision)
    fields: dict = {}
    drafts: dict = {}
    saved = {
        (verifier, "verify"): verifier.verify,
        (runtime, "verify"): runtime.verify,
        (flowpolicy, "integrate_flow"): flowpolicy.integrate_flow,
        (draft, "propose"): draft.propose,
        (runtime, "propose"): runtime.propose,
    }
    ref_field_type = flowpolicy.VelocityField

    def as_device(field):
        if isinstance(field, ref_field_type):
            key = id(field)
            if key not in fields:
                fields[key] = (field, _df.VelocityField(
                    net=_device_mlp(field.net), horizon=field.horizon, dim=field.dim,
                    emb_dim=field.emb_dim, state_dim=field.state_dim, layout=field.layout))
            return fields[key][1]
        return field

    def verify(field, draft_chunk, cache, state, cfg, rng, current_gripper_sign=-1.0, noise_seed=None):
        rep = _dv.verify(as_device(field), draft_chunk, cache, state, cfg, rng, current_gripper_sign,
                         noise_seed)
        if isinstance(field, ref_field_type):
            field.eval_count += len(cfg.timesteps)
        return verifier.VerifierReport(rep.reconstructed, rep.distances, rep.branch_prefixes, rep.prefix,
                                       rep.gripper_switch_detected, rep.shared_noise_seed)

    def integrate_flow(field, cache, state, cfg, rng):
        out = _df.integrate_flow(as_device(field), cache, state, cfg, rng)
        if isinstance(field, ref_field_type):
            field.eval_count += cfg.num_steps
        return out

    def propose(model, obs):
        key = id(model)
        if key not in drafts:
            drafts[key] = (model, _dd.DraftModel(net=_device_mlp(model.net), layout=model.layout,
                                                 horizon=model.horizon, n_tasks=model.n_tasks,
                                                 normalizer=model.normalizer))
        vals = _dd.propose(drafts[key][1], obs).values
        return draft.ActionChunk(values=vals, layout=model.layout, space=draft.STANDARDIZED)

    verifier.verify = runtime.verify = verify
    flowpolicy.integrate_flow = integrate_flow
    draft.propose = runtime.propose = propose

    def restore() -> None:
        for (mod, name), fn in saved.items():
            setattr(mod, name, fn)

    return restore
