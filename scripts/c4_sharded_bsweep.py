"""Single-rotation sharded training of the friendster shape's finest level
(edge-scaled 10 epochs, 8 ranks): AUCROC against the per-pair batch B."""
import json
import os
import sys

os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "backend:cudaMallocAsync")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2008_12336_b200 as gb  # noqa: E402
from paper_2008_12336_b200.evaluate import LinkPredictionSetup  # noqa: E402

BS = [int(x) for x in os.environ.get("BS", "1,2,3,4,5,6,8,10").split(",")]
UNIT = os.environ.get("UNIT", "edge-scaled")
EPOCHS = int(os.environ.get("EPOCHS", "10"))
g = gb.rmat_graph(27, 1_900_000_000, 7, densify_ids=True)
setup = LinkPredictionSetup.build(g, eval_seed=1, evaluator="device", eval_sample=1 << 20)
del g
cfg = gb.TrainConfig(dim=128, total_epochs=EPOCHS, smoothing_ratio=0.3, learning_rate=0.035,
                     negative_samples=3, seed=1, epoch_unit=UNIT)
for B in BS:
    M, st = gb.train_multilevel_sharded(setup.train_graph, cfg, hierarchy=setup.hierarchy,
                                        num_ranks=8, shard_levels=1, return_device=True,
                                        adapt_batch=False, batch_size=B)
    s0 = [e for e in st if e["level"] == 0][0]
    print(json.dumps({"B": B, "rotations": s0.get("rotations"), "pos": s0.get("pos_updates"),
                      "neg": s0.get("neg_updates"), "aucroc": setup.score(M)}), flush=True)
    del M
    torch.cuda.empty_cache()
