import os, sys, torch, warnings
sys.path.insert(0, os.getcwd())
from efgp_data import CONFIGS
from efgp_data import gpu as G
from paper_2210_10210_b200 import EFGP
c = CONFIGS["c5"]; q = int(4e8)
x, y = G.generate_points(c, 0, q)
g = EFGP(c.kernel, c.ell, c.sigma, c.eps, c.d, c.nu)
warnings.simplefilter("ignore")
g.fit(x[:1000000], y[:1000000])
mu = torch.empty(q, dtype=torch.float64, device=x.device)
ts = []
for _ in range(5):
    g.predict(x, out=mu); ts.append(g.info()["t_predict_ms"])
print(os.environ.get("EFGP_LIB","?")[-12:], "interp ms", min(ts), "targets/s %.3e" % (q / min(ts) * 1e3), float(mu[:1000].sum()))
