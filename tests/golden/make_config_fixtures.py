"""Generate the BASELINE-config parity fixtures (committed under tests/golden/).

    python tests/golden/make_config_fixtures.py geometry      # C2, C3 (+3-D C5) partitions
    python tests/golden/make_config_fixtures.py c3 cholesky   # C3 L(θ), oracle, ~40+ min
    python tests/golden/make_config_fixtures.py c3 ldl
    python tests/golden/make_config_fixtures.py c4            # C4-shaped L(θ) + predictions

Sources (test infrastructure, never the product):
* geometry: the UNMODIFIED reference geometry.cpp (oracle/_ref, geometry.cpp:41-154)
  for the 2-D configs; the oracle restatement (same split / admissibility rules,
  extended to d = 3) for the 3-D C5 partition, which the reference cannot represent.
  Stored as SHA-256 of the little-endian int32 perm and of the (count, 5) int32
  block list (row_begin, row_end, col_begin, col_end, tag) in DFS order, plus counts.
* L(θ) / predictions: the oracle restatement (hmgp_oracle.cpp, follows
  loglik.cpp:18-38, krige.cpp:9-44) — the reference's arithmetic half needs Eigen,
  which is absent, so the restatement stands in for it.

Inputs follow SURVEY.md §8d: jittered grid seed 1, Z = AS241 normals with seed
1 ^ 0x517cc1b727220a95.  C4 fixtures use iid-normal Z (the exact 65 536-point GRF
sample needs a 34 GB dense Cholesky that the CPU oracle cannot do in useful time);
prediction parity is linear in Z, so this pins the same code path.
"""
import hashlib
import json
import os
import platform
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Oracle, RefLib, make_config  # noqa: E402

SEED = 1
Z_SEED = SEED ^ 0x517CC1B727220A95
C3_THETA = [1.5, 0.05, 1.0, 0.01]
# C4 grid points (exact decimal literals from the 512-point grid, sweep.py)
C4_THETAS = [[1.0, 0.1, 0.5, 0.01], [0.9285714285714286, 0.09714285714285714, 1.1, 0.001]]
C4_PREDICT_THETA = [1.1428571428571428, 0.09714285714285714, 0.7, 0.01]
C4_M = 1000


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).astype("<i4").tobytes()).hexdigest()


def host():
    try:
        model = [l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")][0]
    except Exception:
        model = platform.processor()
    return {"cpu": model, "nproc": os.cpu_count()}


def write(name, obj):
    path = os.path.join(HERE, name)
    with open(path, "w") as f:
        json.dump(obj, f, indent=1)
    print("wrote", path, flush=True)


def geometry():
    ref, o = RefLib(), Oracle()
    out = {}
    for name, g, leaf in (("C2", 256, 64), ("C3", 512, 128)):
        x = o.jittered_grid(g, SEED)
        t = time.time()
        perm = ref.cluster_perm(x, leaf)
        blocks, na, nd = ref.block_leaves(x, leaf, 2.0)
        dt = time.time() - t
        # the restatement must agree before the fixture is written
        assert np.array_equal(perm, o.cluster_perm(x, leaf))
        ob, ona, ond = o.block_leaves(x, leaf, 2.0)
        assert np.array_equal(blocks, ob) and (na, nd) == (ona, ond)
        out[name] = {"n": g * g, "grid": g, "leaf": leaf, "eta": 2.0, "seed": SEED,
                     "source": "oracle/_ref (unmodified geometry.cpp)",
                     "perm_sha256": sha(perm), "blocks_sha256": sha(blocks),
                     "blocks": int(blocks.shape[0]), "admissible": na, "dense": nd,
                     "perm_head": perm[:16].tolist(), "ref_seconds": dt}
    # C5: 3-D uniform, n = 1 048 576, leaf 128 (restatement: the reference is 2-D only)
    x = o.random_locations(1 << 20, SEED, 3)
    t = time.time()
    perm = o.cluster_perm(x, 128)
    blocks, na, nd = o.block_leaves(x, 128, 2.0)
    out["C5"] = {"n": 1 << 20, "dim": 3, "leaf": 128, "eta": 2.0, "seed": SEED,
                 "source": "oracle restatement (3-D extension of geometry.cpp rules)",
                 "perm_sha256": sha(perm), "blocks_sha256": sha(blocks),
                 "blocks": int(blocks.shape[0]), "admissible": na, "dense": nd,
                 "perm_head": perm[:16].tolist(), "oracle_seconds": time.time() - t}
    write("geometry_configs.json", out)


def c3(form):
    o = Oracle()
    x = o.jittered_grid(512, SEED)
    z = o.normals(512 * 512, Z_SEED)
    threads = int(os.environ.get("FIXTURE_THREADS", "3"))
    cfg = make_config(leaf_size=128, eps=1e-6, form=form, threads=threads)
    t = time.time()
    r = o.loglik(x, z, C3_THETA, cfg)
    wall = time.time() - t
    write(f"loglik_c3_{form}.json", {
        "config": "C3: n=262144 jittered 512x512 seed 1, theta=(1.5,0.05,1.0,0.01), leaf 128, "
                  "eta 2, eps 1e-6 (assembly and factor), Z iid AS241 normals seed 1^0x517cc1b727220a95",
        "form": form, "theta": C3_THETA, "loglik": r.loglik, "logdet": r.logdet,
        "quad_form": r.quad_form, "clamped": r.clamped, "seconds": wall,
        "t_tree": r.t_tree, "t_assemble": r.t_assemble, "t_factor": r.t_factor,
        "assembly_threads": threads, "factor_threads": 1, "host": host(),
        "source": "oracle/hmgp_oracle.cpp orc_loglik (restatement of loglik.cpp:18-38)"})


def c4():
    o = Oracle()
    threads = int(os.environ.get("FIXTURE_THREADS", "2"))
    x = o.jittered_grid(256, SEED)
    z = o.normals(256 * 256, Z_SEED)
    cfg = make_config(leaf_size=64, eps=1e-7, form="ldl", threads=threads)
    evals = []
    for th in C4_THETAS:
        t = time.time()
        r = o.loglik(x, z, th, cfg)
        evals.append({"theta": th, "loglik": r.loglik, "logdet": r.logdet,
                      "quad_form": r.quad_form, "clamped": r.clamped, "seconds": time.time() - t})
        print(evals[-1], flush=True)
    te = o.random_locations(10000, SEED + 1)[:C4_M]
    t = time.time()
    pred = o.predict(x, z, te, C4_PREDICT_THETA, cfg)
    pw = time.time() - t
    np.savez_compressed(os.path.join(HERE, "predict_c4.npz"), pred=pred, theta=C4_PREDICT_THETA,
                        m=C4_M)
    write("loglik_c4.json", {
        "config": "C4-shaped: n=65536 jittered 256x256 seed 1, leaf 64, eta 2, eps 1e-7, LDL; "
                  "Z iid AS241 normals seed 1^0x517cc1b727220a95 (not the GRF sample, see header)",
        "evals": evals, "predict": {"theta": C4_PREDICT_THETA, "m": C4_M,
                                    "test": "random_locations(10000, seed 2)[:1000]",
                                    "seconds": pw, "file": "predict_c4.npz"},
        "assembly_threads": threads, "host": host(),
        "source": "oracle/hmgp_oracle.cpp orc_loglik / orc_predict"})


if __name__ == "__main__":
    what = sys.argv[1]
    if what == "geometry":
        geometry()
    elif what == "c3":
        c3(sys.argv[2])
    elif what == "c4":
        c4()
    else:
        raise SystemExit(__doc__)
