"""CTA-0 tile timeline of the quant pass inside one adahop_linear_layer call (build with
--define QTC_TRACE=1, select it with ADAHOP_LIB). Usage: python scripts/micro/qtc_layer_trace.py [linear]
(linear of the Llama-3.2-1B layer: q, k, gate, down; default gate)."""
import sys
sys.path.insert(0, ".")
import torch  # noqa: E402
import paper_2604_02525_b200 as ah  # noqa: E402
import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "gate"
dims = {"q": (2048, 2048), "k": (2048, 512), "gate": (2048, 8192), "down": (8192, 2048)}[name]
T = 16384
d_in, d_out = dims
px, pg = synth.LLAMA32_1B_LAYER_PATTERNS[name]
dev = torch.device("cuda:0")
x = synth.operand_torch(T, d_in, px, "X", 1000, dev)
w = synth.operand_torch(d_out, d_in, "N", "W", 2000, dev)
gy = synth.operand_torch(T, d_out, pg, "GY", 3000, dev)
strat = tuple(ah.layer_strategies(px, "N", pg, 1)[0])
p = ah.Params(oe_k=64)
for _ in range(2):
    ah.linear_layer(x, w, gy, strat, p, out_dtype=torch.bfloat16)
torch.cuda.synchronize()
print(f"=== {name} {strat}", flush=True)
ah.linear_layer(x, w, gy, strat, p, out_dtype=torch.bfloat16)
torch.cuda.synchronize()
