"""CPU-only checks: the C-ABI library loads and exports every symbol the
header declares (no compute calls), host-side API semantics, and the
multi-rank stream sharding + statistics gather over gloo (world size 2)."""

import os
import re
import socket
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def test_header_symbols_exported():
    from paper_1503_06959_b200 import _native

    hdr = (ROOT / "include" / "vidfeat_b200.h").read_text()
    declared = set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(vf_\w+)\s*\(", hdr, re.M))
    assert declared, "no declarations parsed"
    L = _native.lib()
    for name in sorted(declared):
        assert hasattr(L, name), f"{name} declared in include/vidfeat_b200.h but not exported"
    assert declared == set(_native.EXPORTS)
    assert L.vf_version().decode().startswith("vidfeat-b200")
    assert L.vf_strerror(-1).decode() == "detection threshold must be >= 1"


def test_library_is_sm100a():
    """The shipped library carries sm_100a SASS (cuobjdump), not a PTX-only fallback."""
    import shutil
    import subprocess

    from paper_1503_06959_b200 import build

    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not Path(exe).exists():
        pytest.skip("cuobjdump not available")
    out = subprocess.run([exe, "--list-elf", str(build.LIB)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_config_validation_mirrors_reference():
    from paper_1503_06959_b200.types import GrayFrame, MaskConfig

    with pytest.raises(ValueError):
        MaskConfig(mode="bogus")
    with pytest.raises(ValueError):
        MaskConfig(grid=(0, 16))
    with pytest.raises(ValueError):
        MaskConfig(t_h=-1)
    with pytest.raises(ValueError):
        GrayFrame(np.zeros((4, 4), np.float32))
    with pytest.raises(ValueError):
        GrayFrame(np.zeros(4, np.uint8))


def test_layer_geometry_matches_oracle():
    from oracle import oracle
    from paper_1503_06959_b200.pyramid import layer_geometry

    for (w, h, O) in ((640, 480, 4), (1280, 720, 4), (1920, 1080, 4), (3840, 2160, 4), (97, 61, 3), (64, 64, 4)):
        ws, hs, sc = layer_geometry(w, h, O)
        ows, ohs, osc = oracle.layer_dims(w, h, O)
        assert ws == ows.tolist() and hs == ohs.tolist() and sc == osc.tolist()
    with pytest.raises(ValueError):
        layer_geometry(8, 8, 4)


def test_descriptor_serialization():
    from paper_1503_06959_b200.descriptor import descriptor_hex, pack_descriptor, unpack_descriptor

    bits = np.zeros(512, np.uint8)
    bits[0] = 1
    raw = pack_descriptor(bits)
    assert len(raw) == 64 and raw[0] == 0x80
    rng = np.random.default_rng(0)
    b = rng.integers(0, 2, 512).astype(np.uint8)
    assert np.array_equal(unpack_descriptor(pack_descriptor(b)), b)
    assert len(descriptor_hex(b)) == 128
    with pytest.raises(ValueError):
        pack_descriptor(np.zeros(256, np.uint8))


def test_shard_partition():
    from paper_1503_06959_b200.distributed import shard

    for S in (1, 8, 63, 64):
        for G in (1, 2, 4, 8):
            parts = [shard(S, r, G) for r in range(G)]
            assert sum(parts, []) == list(range(S))
            assert max(map(len, parts)) - min(map(len, parts)) <= 1


def test_scenes_deterministic():
    from paper_1503_06959_b200 import scenes

    cfg = scenes.SceneConfig(128, 96, 3, 2, "mixed", (2, 3), (0.0, 4.0), (0.5, 2.0), block_contrast=120.0, seed=5)
    a = scenes.generate(cfg)
    b = scenes.generate(cfg)
    assert a.shape == (2, 3, 96, 128) and np.array_equal(a.numpy(), b.numpy())


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_1503_06959_b200.distributed import gather_stats, shard
    from paper_1503_06959_b200.types import FrameReport
    from paper_1503_06959_b200.distributed import pack_stats

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    S = 5
    mine = shard(S, rank, world)
    reps = [[FrameReport(n, 10 * s + n, s, 10 * s + n + s, 0.5, 0, 0, 0, 0, 0, n_dropped=n) for n in range(3)]
            for s in mine]
    full = gather_stats(pack_stats(mine, reps), S)
    q.put((rank, full.tolist()))
    dist.destroy_process_group()


def test_gloo_world2_stats_gather():
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    a = np.array(res[0])
    assert np.array_equal(a, np.array(res[1]))
    assert a.shape == (5, 3, 8)
    assert a[:, 0, 0].tolist() == [0, 1, 2, 3, 4]
    assert a[3, 2, 2] == 32 and a[3, 2, 4] == 35


def test_integration_stub_struct_matches_header():
    """The ctypes stub a reference maintainer copies from INTEGRATION.md must
    lay out vf_config / vf_report exactly as include/vidfeat_b200.h does
    (vf_create copies the whole struct)."""
    import ctypes

    from paper_1503_06959_b200 import _native

    text = (ROOT / "INTEGRATION.md").read_text()
    ns = {"ctypes": ctypes}
    for name in ("VfConfig", "VfReport"):
        m = re.search(rf"^class {name}\(ctypes\.Structure\):\n(?:    .*\n|\s*#.*\n)+", text, re.M)
        assert m, f"{name} stub missing from INTEGRATION.md"
        exec(m.group(0), ns)
        stub, real = ns[name], getattr(_native, name)
        assert ctypes.sizeof(stub) == ctypes.sizeof(real), name
        assert [f[0] for f in stub._fields_] == [f[0] for f in real._fields_], name
