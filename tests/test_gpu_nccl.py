"""GPU: the NCCL transport of the multi-rank contexts, as far as one GPU allows.

Every gpurun box has one GPU and NCCL cannot place two ranks on one device, so the row-sharded schedule
itself runs on host-staged sums (test_gpu_dist_world2.py). This file covers what that leaves out: the
dlopen'ed NCCL bindings rfgpu_ctx_create_dist uses (library found, symbols resolved, ncclUniqueId passed by
value, ncclAllReduce with the double / sum codes) on a one-rank communicator."""
import numpy as np
import pytest

import paper_1607_01649_b200 as rf

pytestmark = pytest.mark.gpu


def test_nccl_unique_ids_differ():
    a, b = rf.Context.nccl_unique_id(), rf.Context.nccl_unique_id()
    assert len(a) == 128 and len(b) == 128 and a != b and any(a)


def test_nccl_one_rank_allreduce_roundtrip():
    x = np.random.default_rng(5).standard_normal(100003)
    out = np.zeros_like(x)
    rf._check(rf.lib().rfgpu_nccl_selftest(0, rf._dp(x), x.size, rf._dp(out)))
    assert np.array_equal(out, x)  # one rank: the sum is the input, bit for bit


def test_nccl_selftest_rejects_bad_arguments():
    x = np.ones(4)
    with pytest.raises(rf.ParameterError):
        rf._check(rf.lib().rfgpu_nccl_selftest(0, rf._dp(x), 0, rf._dp(x)))
