"""The co-residency facts the planner and the one-kernel exchange rely on, asked of the device
through da_query_residency (the CUDA occupancy API on the exact kernel instantiations):
  * config.h's kMaxActiveClustersB200 (the planner's cluster-combine choice) and the
    measured record profiles/cluster_fit_b200.json that oracle/policy.py loads are what the device
    answers for the cluster kernels on a 148-SM B200;
  * da_forward_peer_combine refuses a grid the device cannot keep resident."""

import json
import os
import re

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _config_table():
    with open(os.path.join(ROOT, "paper_2604_00028_b200", "csrc", "config.h")) as f:
        src = f.read()
    m = re.search(r"kMaxActiveClustersB200\[17\]\s*=\s*\{([^}]*)\}", src)
    return [int(x) for x in m.group(1).split(",")]


def test_cluster_table_matches_device():
    import paper_2604_00028_b200 as dec
    from paper_2604_00028_b200 import _lib as L
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    table = _config_table()
    for pack, (b, hq, hkv, lk) in ((True, (1, 8, 1, 4096)), (True, (1, 32, 2, 8192)), (False, (1, 8, 1, 4096))):
        for s in range(2, 17):
            plan = dec.make_plan(b, hq, hkv, lk, pack_gqa=pack, policy="fixed", forced_splits=s,
                                 combine_mode=L.DA_COMBINE_CLUSTER)
            n = L.da_query_residency(plan, 0, 0)
            assert n >= 1
            if sms == 148:
                assert n == table[s], (pack, hq, s, n, table[s])
            assert L.da_query_residency(plan, 0, 2) == n           # the exchange variant fits alike
        one = dec.make_plan(b, hq, hkv, lk, pack_gqa=pack, policy="fixed", forced_splits=1)
        assert L.da_query_residency(one, 0, 0) == sms                 # one forward CTA per SM
    rec_path = os.path.join(ROOT, "profiles", "cluster_fit_b200.json")
    if sms == 148 and os.path.exists(rec_path):
        with open(rec_path) as f:
            rec = json.load(f)
        assert rec["max_active_clusters"][2:] == table[2:]


def test_combine_kernel_residency_and_peer_guard():
    import paper_2604_00028_b200 as dec
    from paper_2604_00028_b200 import _lib as L, api
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    plan = dec.make_plan(1, 64, 8, 131072, policy="seq_aware")         # s = 16, workspace combine
    per_dev = L.da_query_residency(plan, 1, 0)
    assert per_dev >= sms and per_dev % sms == 0
    assert api.one_kernel_exchange_ok(plan) == (plan.batch * plan.h_q <= per_dev)
    # a workspace plan with more combine rows than resident CTAs is refused by the one-kernel exchange
    big = dec.make_plan(per_dev // 64 + 1, 64, 8, 8192, policy="fixed", forced_splits=2,
                        combine_mode=L.DA_COMBINE_KERNEL)
    assert not api.one_kernel_exchange_ok(big)
    # clusters: 8 clusters of 16 fit one wave only if the device holds 8 of them at once
    c16 = dec.make_plan(8, 8, 1, 8192, policy="fixed", forced_splits=16, combine_mode=L.DA_COMBINE_CLUSTER)
    assert api.one_kernel_exchange_ok(c16) == (8 <= L.da_query_residency(c16, 0, 2))
