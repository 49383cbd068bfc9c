"""Write tests/golden/c5_sample_expected.npz: the ORACLE's counts for a seeded 2,000-root
sample of the C5 batch (SURVEY 8(d) "Parity protocol per config": C5 = a 2,000-hypothesis
sample), so the GPU parity test does not have to spend ~2 CPU-hours per run re-deriving them.

Calls only oracle/ (the plain C set evaluator) and synth/ (the seeded generators): no value in
the file comes from the CUDA path.  The file also stores checksums of the generated inputs, so
a change of the generators (or of numpy's streams) makes the test fail loudly instead of
comparing against stale expectations.

    python tools/make_c5_expected.py            # ~15 min on 8 cores
"""
from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import setsem  # noqa: E402
from synth import abox, hyps  # noqa: E402

N_HYPS, HYP_SEED, SAMPLE, SAMPLE_SEED = 100_000, 5, 2000, 55
OUT = os.path.join(ROOT, "tests", "golden", "c5_sample_expected.npz")


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode() + str(a.shape).encode())
        h.update(a.view(np.uint8).reshape(-1).tobytes())
    return h.hexdigest()


def kb_digest(kb) -> str:
    return digest(kb["concept_bits"], kb["role_edge_off"], kb["edge_subj"], kb["edge_obj"], kb["data_off"],
                  kb["data_subj"], kb["data_val"], kb["pos_ids"], kb["neg_ids"])


def sample_roots(n: int) -> np.ndarray:
    return np.sort(np.random.default_rng(SAMPLE_SEED).choice(n, SAMPLE, replace=False))


def main():
    t0 = time.time()
    kb = abox.c5_kb()
    nodes, kids, roots = hyps.batch_arrays("c5", kb, N_HYPS, HYP_SEED)
    sample = sample_roots(len(roots))
    okb = setsem.OracleKB(kb)
    _, oc = okb.evaluate(nodes, kids, roots[sample], want_bits=False, threads=os.cpu_count())
    np.savez_compressed(OUT, sample=sample.astype(np.uint32), counts=oc.astype(np.uint64),
                        kb_sha=np.array(kb_digest(kb)), hyps_sha=np.array(digest(nodes, kids, roots)))
    print(f"wrote {OUT}: {SAMPLE} roots in {time.time() - t0:.0f} s")


if __name__ == "__main__":
    main()
