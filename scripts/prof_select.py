"""ncu helper: the score_select_pass sub-record's setup (bench.score_select_phase: the C4 trace
replayed into a full 2^24-block pool), then three sae_select launches of 10 read-only passes
(capture the third with -k regex:k_select -s 2 -c 1): its DRAM bytes against 10 x 201 MB."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
info = bench.score_select_phase(torch.device("cuda", 0), launches=2)
print("ok", info["us_per_pass"], info["resident_blocks"])
