"""The C-ABI library builds, loads and exports every symbol include/edgeserve.h
declares -- no compute call (no GPU here).  Also checks the binding's struct
layouts against the header's field order and the SASS for the TMA bulk copy."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2605_05527_b200 import build
    return build.build()


def header_functions():
    src = open(os.path.join(ROOT, "include", "edgeserve.h")).read()
    return sorted(set(re.findall(r"ES_API\s+[\w\s\*]+?\b(es_\w+)\s*\(", src)))


def test_exports_every_declared_symbol(libpath):
    lib = ctypes.CDLL(libpath)
    names = header_functions()
    assert len(names) >= 14
    for n in names:
        assert hasattr(lib, n), n
    import paper_2605_05527_b200 as es
    assert sorted(es.EXPORTS) == names


def test_binding_structs_match_header():
    import paper_2605_05527_b200 as es
    src = open(os.path.join(ROOT, "include", "edgeserve.h")).read()

    def fields(tname):
        body = re.search(r"typedef struct \{([^{}]*)\}\s*" + tname + ";", src).group(1)
        body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
        out = []
        for decl in body.split(";"):
            decl = decl.strip()
            if not decl:
                continue
            for part in decl.split(","):
                out.append(re.findall(r"(\w+)\s*$", part.strip())[0])
        return out

    for cls, tname in [(es.ProfileDesc, "es_profile_desc"), (es.SchedCfg, "es_sched_cfg"),
                       (es.Snapshots, "es_snapshots"), (es.Decisions, "es_decisions"),
                       (es.Traces, "es_traces"), (es.ReplayOut, "es_replay_out")]:
        assert [f[0] for f in cls._fields_] == fields(tname), tname


def test_stat_columns_match_header():
    import oracle
    import paper_2605_05527_b200 as es
    src = open(os.path.join(ROOT, "include", "edgeserve.h")).read()
    body = re.search(r"enum \{\s*ES_ST_DECISIONS = 0,(.*?)ES_NSTAT", src, re.S).group(0)
    cols = re.findall(r"ES_ST_(\w+)", body)
    # the exit histogram is declared as the range ES_ST_EXIT0 .. ES_ST_EXIT7 = ES_ST_EXIT0 + 7
    assert "ES_ST_EXIT7 = ES_ST_EXIT0 + 7" in body
    cols = [c for c in cols if not c.startswith("EXIT")] + [f"EXIT{e}" for e in range(8)]
    assert len(cols) == es.ES_NSTAT == oracle.NCOL
    assert [c.lower() for c in cols] == es.STAT_COLS == oracle.COLS


def test_sass_uses_tma_bulk_copy(libpath):
    sass = subprocess.run(["cuobjdump", "-sass", libpath], capture_output=True, text=True).stdout
    assert "UBLKCP" in sass  # cp.async.bulk staging of the profile image
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", libpath], capture_output=True, text=True).stdout


def test_missing_library_fails_loudly(tmp_path, monkeypatch):
    import paper_2605_05527_b200 as es
    monkeypatch.setattr(es, "LIB_PATH", str(tmp_path / "nope.so"))
    monkeypatch.setattr(es, "_lib", None)
    with pytest.raises(es.EsError, match="no CPU fallback"):
        es.lib()
