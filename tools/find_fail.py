import sys, torch
sys.path.insert(0, '.')
import paper_1606_05688_b200 as v
from paper_1606_05688_b200.bundled_nets import NETS
name = sys.argv[1]
net = v.parse_network_spec(NETS[name]); fov = net.field_of_view()[0]
ctx = v.Context(0)
m = v.Model(net, v.random_weights(net, 1), ctx)
for e in [int(a) for a in sys.argv[2:]]:
    try:
        x = torch.rand((1, 1, e, e, e), device="cuda")
        out, rep = m.forward(x)
        print(name, e, "ok", tuple(out.shape), flush=True)
    except Exception as ex:
        print(name, e, "FAIL", str(ex)[:200], flush=True)
        break
