"""Regenerate the golden fixtures from the live reference (needs /root/reference).

    python tests/golden/make_golden.py

Writes
  instances.json  sha256 of every instance array the reference builds, per
                  (fn, dim, seed) — pins paper_1407_7737_b200.instances;
  values.npz      reference Engine.evaluate outputs (both precisions) on
                  seeded points, plus the known-answer points the reference's
                  own tests use (optimum -> 100, engine criterion 1) — pins
                  the oracle and, on the GPU, the CUDA path.
The reference is imported read-only from /root/reference/pkg/src.
"""

import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from robench import EngineConfig, initialize  # noqa: E402
from robench import composition, hybrid, transforms  # noqa: E402
from robench.transforms import matvec  # noqa: E402

from tests.golden.digest import digest  # noqa: E402

OUT = Path(__file__).resolve().parent
DIMS = (2, 10, 13, 30, 50, 100)
SEED = 5
NPTS = 12




def instance_arrays(fn, dim, seed):
    if fn < 23:
        inst = transforms.generate_instance(fn, dim, seed)
        return [inst.x_opt, inst.group_perm, inst.rotation]
    if fn < 29:
        sp = hybrid.build_hybrid(fn, dim, seed)
        return [sp.x_opt, sp.split_perm, np.asarray(sp.sizes), *sp.chunk_rotations]
    sp = composition.build_composition(fn, dim, seed)
    out = []
    for m in sp.members:
        out.append(m.x_opt)
        if m.rotation is not None:
            out.append(m.rotation)
        else:
            out += [m.hybrid_spec.split_perm, np.asarray(m.hybrid_spec.sizes),
                    *m.hybrid_spec.chunk_rotations]
    return out


def optimum(fn, dim, seed):
    # test_acceptance.py:48-58
    if fn >= 29:
        return composition.build_composition(fn, dim, seed).members[0].x_opt
    if fn >= 23:
        return hybrid.build_hybrid(fn, dim, seed).x_opt
    inst = transforms.generate_instance(fn, dim, seed)
    if fn == 18:
        return inst.x_opt + 10.0 * (matvec(inst.rotation.T, np.full(dim, 2.5)) - 2.5)
    return inst.x_opt


def main():
    inst = {}
    for dim in DIMS:
        for seed in (0, SEED):
            for fn in range(37):
                if dim < 10 and fn >= 23:
                    continue
                inst[f"{fn}/{dim}/{seed}"] = digest(instance_arrays(fn, dim, seed))
    (OUT / "instances.json").write_text(json.dumps(inst, indent=0, sort_keys=True) + "\n")

    blobs = {}
    for dim in DIMS:
        eng = initialize(EngineConfig(dim=dim, max_concurrency=1000, seed=SEED))
        rng = np.random.default_rng(1000 + dim)
        x = rng.uniform(-100.0, 100.0, (NPTS, dim))
        # include one far point (|x| up to 1e3: exercises schwefel's outer branches)
        x[-1] *= 10.0
        blobs[f"x/{dim}"] = x
        for fn in eng.enabled_ids:
            pts = np.vstack([x, optimum(fn, dim, SEED)[None, :]])
            for prec in ("double", "single"):
                blobs[f"f/{dim}/{fn}/{prec}"] = eng.evaluate(fn, pts, precision=prec).values
            blobs[f"opt/{dim}/{fn}"] = pts[-1]
        eng.dispose()
    np.savez_compressed(OUT / "values.npz", seed=SEED, **blobs)
    print(f"{len(inst)} instance digests, {len(blobs)} value arrays")


if __name__ == "__main__":
    main()
