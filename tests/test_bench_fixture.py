"""The bench workload builder (bench_fixture.py): deterministic, well-formed,
torch-only (the reference arm must not load the product library), and the
N-shard merge bench.py's one-process multi-GPU mode feeds the C ABI."""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench_fixture as F  # noqa: E402

CFG = dict(workload="t", n=3000, dim=16, n_centers=8, sigma=0.3, nq=20, batch=20, m=4, nlist=8, nprobe=4, k=5)


def _build(rank=0, cfg=CFG):
    return F.build(cfg, rank, "cpu")


def test_deterministic_and_fingerprinted():
    a, b = _build(), _build()
    assert F.fingerprint(a) == F.fingerprint(b)
    for f in ("list_ids", "list_codes", "list_lx", "vectors", "coarse", "centroids", "list_offsets"):
        assert bool((getattr(a, f) == getattr(b, f)).all()), f
    assert F.fingerprint(_build(1)) != F.fingerprint(a)


def test_index_invariants():
    fx = F.to_host(_build())
    offs = fx.list_offsets.astype(np.int64)
    assert offs[0] == 0 and offs[-1] == CFG["n"] and (np.diff(offs) >= 0).all()
    assert sorted(fx.list_ids.tolist()) == list(range(CFG["n"]))
    for l in range(CFG["nlist"]):
        seg = fx.list_ids[offs[l]:offs[l + 1]]
        assert (np.diff(seg.astype(np.int64)) > 0).all()  # ascending ids in a list (ivf.hpp:147-152)
    # lx = |x - decode(code)| (landmarks.hpp:57-72)
    m, sd = CFG["m"], CFG["dim"] // CFG["m"]
    C3 = fx.centroids.reshape(m, 256, sd)
    x = fx.vectors[fx.list_ids.astype(np.int64)].reshape(-1, m, sd)
    dec = C3[np.arange(m)[None, :], fx.list_codes.astype(np.int64)]
    lx = np.sqrt(((x.astype(np.float64) - dec) ** 2).sum((1, 2)))
    assert np.allclose(lx, fx.list_lx, rtol=1e-5, atol=1e-6)
    # every code is the nearest sub-centroid up to fp32 rounding
    d = ((x[:, :, None, :].astype(np.float64) - C3[None]) ** 2).sum(3)
    best = d.min(2)
    got = np.take_along_axis(d, fx.list_codes.astype(np.int64)[:, :, None], 2)[:, :, 0]
    assert np.allclose(got, best, rtol=1e-4, atol=1e-6)


def test_shard_merge():
    sys.path.insert(0, ROOT)
    import bench
    parts = [F.to_host(_build(r)) for r in range(3)]
    whole = bench.merged_host_index(parts)
    n = CFG["n"]
    assert whole.list_offsets[-1] == 3 * n
    assert sorted(whole.list_ids.tolist()) == list(range(3 * n))
    offs = whole.list_offsets.astype(np.int64)
    for l in range(CFG["nlist"]):
        seg = whole.list_ids[offs[l]:offs[l + 1]].astype(np.int64)
        assert (np.diff(seg) > 0).all()
        want = np.concatenate([p.list_ids[p.list_offsets[l]:p.list_offsets[l + 1]] for p in parts])
        assert (seg == want).all()
    # entry payloads follow their ids
    for p, s in enumerate(parts):
        pos = {int(i): j for j, i in enumerate(whole.list_ids)}
        for j in range(0, n, 97):
            e = pos[int(s.list_ids[j])]
            assert (whole.list_codes[e] == s.list_codes[j]).all() and whole.list_lx[e] == s.list_lx[j]
    assert (whole.vectors[n:2 * n] == parts[1].vectors).all()


def test_reference_arm_imports_no_product_code():
    code = ("import sys; sys.path.insert(0, %r); import bench, bench_fixture as F; "
            "F.build(dict(workload='t', n=500, dim=8, n_centers=4, sigma=0.3, nq=4, batch=4, m=2, nlist=1, "
            "nprobe=1, k=2), 0, 'cpu'); "
            "bad = [m for m in sys.modules if m.startswith('paper_2508_17828_b200')]; "
            "assert not bad, bad; print('ok')") % ROOT
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr
