"""CPU: the C-ABI library loads, exports every symbol include/moe_b200.h
declares, and its host-side validation mirrors the reference's exceptions
(no device work happens on these paths)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    with open(os.path.join(ROOT, "include", "moe_b200.h")) as f:
        src = f.read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s+(mo[a-z_0-9]+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_library_exports_every_declared_symbol():
    from paper_2205_10034_b200 import _lib
    names = declared_functions()
    assert len(names) >= 30, names
    lib = C.CDLL(_lib.LIB_PATH)
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # the Python binding covers the same surface
    assert set(names) == set(_lib.SIGNATURES), set(names) ^ set(_lib.SIGNATURES)
    assert _lib.lib.moe_abi_version() == 1


def test_sm100a_only_and_tcgen05_in_sass():
    import shutil
    import subprocess
    from paper_2205_10034_b200 import _lib
    if shutil.which("cuobjdump") is None and not os.path.exists("/usr/local/cuda/bin/cuobjdump"):
        pytest.skip("cuobjdump unavailable")
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([exe, "-lelf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches
    sass = subprocess.run([exe, "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass and "UTMALDG" in sass and "LDTM" in sass


def test_host_validation_mirrors_reference_exceptions():
    from paper_2205_10034_b200 import moesim
    from paper_2205_10034_b200._lib import ConfigError
    bad = moesim.ShardedPayload(ranks=2, chunks=[b"a", b"b", b"c"])
    with pytest.raises(ValueError, match="alltoall: payload is not a square rank matrix"):
        moesim.alltoall_flat(bad)
    with pytest.raises(ValueError, match="fuse_slices: empty slice list"):
        moesim.fuse_slices([])
    with pytest.raises(ConfigError, match="workload.experts: must be >= 1"):
        moesim.gen_trace(1, 1, 1, 0, 10, 0.0)
    with pytest.raises(ConfigError, match="workload.skew: must be >= 0"):
        moesim.gen_trace(1, 1, 1, 4, 10, -0.5)
    with pytest.raises(ConfigError, match="ring.ring_slots"):
        moesim.build_schedule(4, 0)
    with pytest.raises(ConfigError, match="ring.num_layers"):
        moesim.build_schedule(0, 2)


def test_ring_schedule_host_logic_matches_reference(golden):
    from paper_2205_10034_b200 import moesim
    for ent in golden["ring_schedule"]:
        n, k = ent["args"]
        if "error" in ent["expected"]:
            with pytest.raises(Exception):
                moesim.build_schedule(n, k)
            continue
        s = moesim.build_schedule(n, k)
        got = [[o.kind, o.layer, o.slot, -1 if o.waits_release_of is None else o.waits_release_of]
               for o in s.ops]
        assert got == ent["expected"]["ops"]
        assert s.slots == ent["expected"]["slots"] and s.clamped == ent["expected"]["clamped"]


def test_layer_config_errors_name_the_field():
    """ConfigError messages follow the reference's '<field>: <reason>' form."""
    import torch
    from paper_2205_10034_b200 import MoEConfig, MoELayer
    from paper_2205_10034_b200._lib import ConfigError
    with pytest.raises(ConfigError, match="layer.top_k"):
        MoELayer(MoEConfig(8, 3, 128, 256, 1.25, 64, torch.bfloat16), device="cpu")
    with pytest.raises(ConfigError, match="layer.ep_size"):
        from paper_2205_10034_b200._lib import LayerDesc, call
        d = LayerDesc(num_experts=6, top_k=1, d_model=128, d_ff=256, capacity_factor=1.0,
                      tokens=16, dtype=1, has_gate_bias=0, ep_size=4, ep_rank=0, nccl_comm=None)
        h = C.c_void_p()
        call("moe_layer_create", C.byref(d), C.byref(h))
    with pytest.raises(ConfigError, match="layer.placement"):
        MoELayer(MoEConfig(8, 1, 128, 256, 1.25, 64, torch.bfloat16, placement="striped"),
                 device="cpu")
    with pytest.raises(ConfigError, match="layer.placement"):
        d = LayerDesc(num_experts=8, top_k=1, d_model=128, d_ff=256, capacity_factor=1.0,
                      tokens=16, dtype=1, has_gate_bias=0, ep_size=1, ep_rank=0, nccl_comm=None,
                      exchange=0, placement=7)
        h = C.c_void_p()
        call("moe_layer_create", C.byref(d), C.byref(h))
