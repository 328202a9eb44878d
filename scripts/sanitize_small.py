"""Small launches of every kernel family for compute-sanitizer racecheck /
synccheck: the shared-memory-staged HOT pass (forced), the HOT PPR pass, the
pair kernels (tournament, 2 virtual ranks, graph-replayed), the CAS collapse,
the edge-list parser, the evaluator."""
import io
import os
import sys

os.environ.setdefault("GB_PASS_SMEM", "1")
os.environ.setdefault("GB_ROTATION_GRAPH", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2008_12336_b200 as gb  # noqa: E402
from paper_2008_12336_b200 import tournament as tn  # noqa: E402

g = gb.rmat_graph(11, 1 << 14, 3, densify_ids=True)
M = torch.from_numpy(gb.init_embedding(g.num_vertices, 128, 1)).cuda()
gb.train_level(g, M, gb.TrainConfig(dim=128), 1)
gb.train_level(g, M, gb.TrainConfig(dim=128, similarity="ppr"), 1)
tn.train_tournament(g, M, gb.TrainConfig(dim=128), 40, num_ranks=2)
tn.train_tournament(g, M, gb.TrainConfig(dim=128, balanced_pools=True), 40, num_ranks=2)
order = gb.coarsen.degree_order(g)
gb.coarsen.collapse_map_parallel(g, order, 64, run_dependent=True)
gb.load_edge_list(io.StringIO("1 2\n2 3\n# c\n3 4\n"))
rep = gb.run_link_prediction(g, gb.TrainConfig(dim=32, total_epochs=20), eval_seed=1,
                             evaluator="device")
assert 0.0 <= rep.aucroc <= 1.0
torch.cuda.synchronize()
print("sanitize_small ok")
