"""tests/golden/ref_composed.npz from the unmodified reference orchestrator
(oracle/_ref, ref_run_iteration -> run_iteration, orchestrator.cpp:563-569,
compose_exchanges on): per case the LLM destination of every example and
where the backbone's assembled input holds every part (instance, position),
i.e. the end state of the composed delivery (orchestrator.cpp:390-418,
backbone_mapping_for :367-388). Cases: C2, a small C3, C3 itself, and a
node-wise hosted C3 (d = 16 on 4 nodes)."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, ROOT)
from oracle import RefLib  # noqa: E402

# (mix, d, instances per node, examples per instance, seed, node-wise hosting)
CASES = [(2, 8, 8, 64, 2, 0), (3, 16, 16, 16, 11, 0), (3, 64, 64, 64, 7, 0),
         (3, 16, 4, 16, 5, 1)]


def main():
    ref = RefLib()
    out = {"cases": np.array(CASES, np.int64)}
    for k, (mix, d, c, per, seed, nw) in enumerate(CASES):
        r = ref.run_iteration(mix, d, per, seed, c=c, nodewise=bool(nw))
        assert r["assembly_ok"] == 1 and r["composed_exchanges"] >= 1, r
        for key in ("llm_dest_inst", "llm_dest_slot", "asm_inst", "asm_pos"):
            out[f"{k}_{key}"] = r[key]
    np.savez_compressed(os.path.join(HERE, "ref_composed.npz"), **out)
    print("wrote", len(CASES), "cases")


if __name__ == "__main__":
    main()
