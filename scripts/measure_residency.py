"""Measure the co-residency table behind the planner's cluster-combine choice on the
GPU this runs on, through the library's own occupancy query (da_query_residency: the CUDA occupancy
API asked about the exact kernel instantiations the planner launches), and write it as the record
that oracle/policy.py loads and tests/test_abi_cpu.py checks config.h's kMaxActiveClustersB200 against.

    python scripts/measure_residency.py [--out profiles/cluster_fit_b200.json]
"""

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "cluster_fit_b200.json"))
    args = ap.parse_args()
    import torch
    import paper_2604_00028_b200 as dec
    from paper_2604_00028_b200 import _lib as L
    props = torch.cuda.get_device_properties(0)
    sms = props.multi_processor_count
    # one representative shape per forward variant: 8-row MMA CTAs, 16-row MMA CTAs, the scalar path
    shapes = {"mma_rows8": dict(batch=1, h_q=8, h_kv=1, l_k=4096, pack_gqa=True),
              "mma_rows16": dict(batch=1, h_q=32, h_kv=2, l_k=8192, pack_gqa=True),
              "scalar": dict(batch=1, h_q=8, h_kv=1, l_k=4096, pack_gqa=False)}
    clusters = {}
    for name, sh in shapes.items():
        row = [0, None]
        for s in range(2, 17):
            plan = dec.make_plan(sh["batch"], sh["h_q"], sh["h_kv"], sh["l_k"], pack_gqa=sh["pack_gqa"],
                                 policy="fixed", forced_splits=s, combine_mode=L.DA_COMBINE_CLUSTER)
            row.append(L.da_query_residency(plan, 0, 0))
            assert L.da_query_residency(plan, 0, 2) == row[-1], "the exchange variant must fit like the plain one"
        # index 1: the s = 1 (NONE) forward, CTAs on the device
        plan1 = dec.make_plan(sh["batch"], sh["h_q"], sh["h_kv"], sh["l_k"], pack_gqa=sh["pack_gqa"],
                              policy="fixed", forced_splits=1)
        row[1] = L.da_query_residency(plan1, 0, 0)
        clusters[name] = row
    combine = L.da_query_residency(dec.make_plan(1, 8, 1, 4096, policy="fixed", forced_splits=32), 1, 0)
    variants = list(clusters.values())
    rec = {
        "what": "co-resident launch units per device of the split-KV forward: index s = clusters of s CTAs "
                "(DA_COMBINE_CLUSTER plans, cudaOccupancyMaxActiveClusters), index 1 = CTAs of the s = 1 forward; "
                "combine_ctas = CTAs of the LSE combine kernel",
        "how": "scripts/measure_residency.py -> da_query_residency (include/decattn.h)",
        "device": props.name, "sms": sms, "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
        "max_active_clusters": variants[0],
        "per_variant": clusters,
        "variants_agree": all(v == variants[0] for v in variants),
        "combine_ctas": combine,
    }
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(rec, f, indent=1)
        f.write("\n")
    print(json.dumps(rec))


if __name__ == "__main__":
    main()
