"""The C-ABI library loads and exports every symbol include/sfgpu.h declares
(no compute calls: these run on the CPU-only driver host)."""
import os
import re

from paper_2102_13018_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared() -> set[str]:
    src = open(os.path.join(ROOT, "include", "sfgpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"\b(sfg_[a-z0-9_]+)\s*\(", src))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    names = declared()
    assert len(names) >= 35
    missing = [n for n in sorted(names) if not hasattr(lib, n)]
    assert not missing, f"not exported: {missing}"


def test_binding_covers_header():
    assert declared() == set(_lib.EXPORTED)


def test_version_and_default_config():
    lib = _lib.load()
    assert lib.sfg_version() == 1
    cfg = _lib.sfg_config()
    lib.sfg_config_default(cfg)
    assert cfg.deterministic == 1 and cfg.force_remote == 0
    assert cfg.dense_discovery_threshold == 64 and cfg.timeout_s == 30.0


def test_library_is_built_for_sm100a():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_error_reporting_without_gpu():
    from paper_2102_13018_b200 import sf

    c = sf.Comm(1, 0, -1)
    f = sf.StarForest(c)
    try:
        f.setup()
    except sf.Error as e:
        assert "requires a graph-set star forest" in str(e)
    else:
        raise AssertionError("setup on a created forest must fail")


def test_set_graph_device_needs_a_device_communicator():
    """The device planner (dsetup.cu) refuses host-only communicators with the
    reference's error mechanism (status + message), before touching memory."""
    from paper_2102_13018_b200 import sf

    c = sf.Comm(1, 0, -1)
    f = sf.StarForest(c)
    lib = _lib.load()
    assert lib.sfg_sf_set_graph_device(f._h, 0, 0, None, None, None) != 0
    assert b"needs a communicator with a device" in lib.sfg_last_error()
    assert lib.sfg_sf_set_graph_device(f._h, -1, 0, None, None, None) != 0
    assert b"negative root or leaf count" in lib.sfg_last_error()
