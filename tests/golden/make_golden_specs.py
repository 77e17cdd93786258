"""Scenario specs shared by make_golden.gen_scenarios and tests/test_gpu_patch.py
(importable without the reference on the path)."""


SCENARIOS = (("fractures", "make_multiple_fractures", dict(levels=6, random_field=True, t_end=0.04)),
             ("lshape2d", "make_lshape", dict(levels=5, dim=2)),
             ("lshape3d", "make_lshape", dict(levels=3, dim=3)))
SCENARIO_STEPS = {"lshape2d": 4, "lshape3d": 3}


def scenario(fracmg_scenarios, tag):
    """The scenario of a golden tag (t_end shortened for the L-shapes)."""
    from dataclasses import replace
    for name, maker, kw in SCENARIOS:
        if name == tag:
            sc = getattr(fracmg_scenarios, maker)(**kw)
            if tag in SCENARIO_STEPS:
                sc = replace(sc, t_end=SCENARIO_STEPS[tag] * sc.dt)
            return sc
    raise KeyError(tag)
