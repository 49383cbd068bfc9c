"""The multi-GPU dispatcher on one real GPU (world size 1): the probe of PAPER.md:566-571 and the
sharded evaluation path through the C ABI (multi-rank host logic: tests/test_dist_gloo.py)."""
import os
import socket

import numpy as np
import pytest

from oracle import setsem
from synth import abox, hyps
from synth.format import flatten
from test_gpu_parity import _hedl

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_probe_and_sharded_eval_world1():
    import torch.distributed as dist
    from paper_2412_00802_b200 import dist as hdist
    hedl = _hedl()
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    import torch
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    try:
        kb = abox.c1_kb()
        k = hedl.hedl_kb_load(kb, 0)
        t = hdist._probe_time(k, 5)
        assert 0 < t < 0.1
        assert np.allclose(hdist.probe_ratios(k), [1.0])
        nodes, kids, roots = flatten(hyps.c1_hypotheses(kb))
        counts, info = hdist.eval_batch_sharded(k, nodes, kids, roots, weights=[1.0])
        _, oc = setsem.evaluate(kb, nodes, kids, roots)
        assert np.array_equal(counts.cpu().numpy(), oc.astype(np.int64))
    finally:
        dist.destroy_process_group()
