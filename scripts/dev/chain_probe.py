import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2506_23025_b200 as tp
from paper_2506_23025_b200.graph import LinearStack
from bench import make_stack_weights, timed_graph
ws = make_stack_weights(32, 1234)
for chain in (False,):
    st = LinearStack(ws, batch=1, chain=chain)
    ms = timed_graph(st.replay, 20, 5, None)
    print(json.dumps(dict(chain=st.chain, ms_per_step=round(ms / 20, 4), us_per_layer=round(ms / 20 / 96 * 1e3, 2))))
