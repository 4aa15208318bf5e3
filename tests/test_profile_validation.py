"""Profile validation (complete grid, L > 0, non-decreasing
in batch, strictly increasing in exit, bs strictly increasing with bs[0] = 1
(reading Q8), every model has an allowed exit).  Each failure mode is planted
in a valid synthetic profile at a known cell; the oracle must reject it naming
exactly that cell, and the C-ABI library's host-side validation (runs before
any CUDA call, so no GPU is needed) must reject it with the matching status
and name the same cell in es_last_error()."""
import numpy as np
import pytest

import inputs
import oracle

OR_ERR_PROFILE = 2


def base():
    return inputs.synth_profile(3, 3, [1, 2, 4, 8])


def planted():
    """(name, profile, oracle cell (m, e, b), library status name, message fragment)."""
    out = []
    p = base()
    lat = p.lat.copy(); lat[1, 0, 2] = 0
    out.append(("L = 0", inputs.Profile(3, 3, p.bs, lat, p.mask), (1, 0, 2), "PROFILE_MONOTONE", "m=1,e=0,b=2) = 0"))
    lat = p.lat.copy(); lat[2, 1, 3] = lat[2, 1, 2] - 1
    out.append(("decreasing in batch", inputs.Profile(3, 3, p.bs, lat, p.mask), (2, 1, 3), "PROFILE_MONOTONE",
                "m=2,e=1,b=3)=%d decreases in batch" % int(lat[2, 1, 3])))
    lat = p.lat.copy(); lat[0, 2, 1] = lat[0, 1, 1]
    out.append(("equal across exits", inputs.Profile(3, 3, p.bs, lat, p.mask), (0, 2, 1), "PROFILE_MONOTONE",
                "m=0,e=2,b=1)"))
    out.append(("bs[0] != 1", inputs.Profile(3, 3, np.array([2, 3, 4, 8], np.int32), p.lat, p.mask), (-1, -1, 0),
                "PROFILE_GRID", "batch_sizes[0]=2"))
    out.append(("bs not increasing", inputs.Profile(3, 3, np.array([1, 4, 4, 8], np.int32), p.lat, p.mask),
                (-1, -1, 2), "PROFILE_GRID", "batch_sizes[2]=4"))
    out.append(("bs above u16", inputs.Profile(3, 3, np.array([1, 2, 4, 70000], np.int32), p.lat, p.mask),
                (-1, -1, 3), "PROFILE_GRID", "batch_sizes[3]=70000"))
    mask = p.mask.copy(); mask[2, :] = 0
    out.append(("no allowed exit", inputs.Profile(3, 3, p.bs, p.lat, mask), (2, -1, -1), "PROFILE_GRID",
                "model 2 has no allowed exit"))
    return out


CASES = planted()


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_oracle_names_the_planted_cell(case):
    name, prof, cell, _, _ = case
    assert oracle.validate_profile(base())[0] == 0
    st, got = oracle.validate_profile(prof)
    assert st == OR_ERR_PROFILE and got == cell, (name, st, got)


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_library_host_validation_names_the_planted_cell(case):
    import paper_2605_05527_b200 as es
    name, prof, _, status, frag = case
    with pytest.raises(es.EsError) as ei:
        es.es_load_profile(prof, [inputs.SchedCfg(tau=50000, b_max=8)])
    msg = str(ei.value)
    assert status in msg and frag in msg, (name, msg)
