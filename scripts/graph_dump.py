import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.chdir(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2512_10576_b200.decode import DSADecodeLayer
layer = DSADecodeLayer(64, 32768, 0.25, 2048, max_new_tokens=16, seed=1, drift=0.97)
layer.prefill_warmup(windows=4)
layer.micro, layer.first_frac = 2, 0.25
orig = torch.cuda.CUDAGraph
class G(orig):
    def __init__(self, *a, **k):
        super().__init__(keep_graph=True)
torch.cuda.CUDAGraph = G
layer.capture("dba", 32)
from cuda.bindings import runtime as rt  # noqa: E402
os.makedirs("gpurun_out", exist_ok=True)
err, = rt.cudaGraphDebugDotPrint(layer.graph.raw_cuda_graph(), b"gpurun_out/step_graph.dot", 0)
print("dumped", err)
import re
path = os.path.abspath("gpurun_out/step_graph.dot")
print(path, os.path.exists(path), os.path.getsize(path) if os.path.exists(path) else -1)
txt = open(path).read()
nodes = {}
for m in re.finditer(r'"?(\w+)"?\s*\[\s*(?:style="[^"]*"\s*)?(?:shape="?\w+"?\s*)?label="([^"]*)"', txt):
    nodes[m.group(1)] = m.group(2)
edges = re.findall(r'"?(\w+)"?\s*->\s*"?(\w+)"?', txt)
print(len(nodes), "nodes", len(edges), "edges")
indeg = {n: 0 for n in nodes}
for a, b in edges:
    indeg[b] = indeg.get(b, 0) + 1
def short(lbl):
    m = re.search(r'(\w+_kernel\w*|timestamp\w*|MEMCPY|MEMSET|EVENT\w*)', lbl)
    return m.group(1) if m else lbl[:60]
for n in nodes:
    if indeg.get(n, 0) == 0:
        print("ROOT", n, short(nodes[n]))
for a, b in edges:
    if a in nodes and b in nodes:
        print("EDGE", short(nodes[a]), "->", short(nodes[b]))
