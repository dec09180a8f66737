"""Simulate the R9 check schedule / crossing search on the goldens' rho(d) (log-linear interpolation
of the oracle's checked values): checks made and a cost model sum (m / 1000)^3 (development tool).
  python tools/sim_schedule.py [cfg ...]"""
import sys, json, math, numpy as np
sys.path.insert(0, '/root/repo')
from oracle import alg1
def make_rho(gold):
    pts = sorted({(h['d'], h['rho_rel']) for h in gold['history'] if h['rho_rel'] == h['rho_rel']} | {(e['d'], e['rho_rel']) for e in gold['per_step']})
    ds = np.array([p[0] for p in pts], float); lr = np.log([p[1] for p in pts])
    return lambda d: float(np.exp(np.interp(d, ds, lr, right=lr[-1] + (d - ds[-1]) * (lr[-1]-lr[-2])/(ds[-1]-ds[-2]))))
class Fake:
    def __init__(s, rho, r): s.rho, s.r, s.d, s.breakdown, s.calls = rho, r, 0, False, []
    def step(s): s.d += 1
    def residual(s, d):
        s.calls.append(d); return alg1.CheckResult(d, s.rho(d), s.rho(d), None, False)
for name in sys.argv[1:]:
    g = json.load(open(f'/root/repo/tests/golden/{name}.json'))
    rho = make_rho(g); r = g['r']
    f = Fake(rho, r); res = alg1.solve(f, 1e-6, g['d_max'], keep_Y=False)
    cost = sum((d*r/1000.)**3 for d in f.calls)
    print(name, 'd*', res.d_star, 'golden', g['d_star'], 'checks', len(f.calls), 'cost(m^3/1e9)', round(cost, 1), f.calls)

import inspect, re
src = inspect.getsource(alg1.solve)
variants = {
 'old': src.replace("elif math.isfinite(dh) and dh - 10 > sched[idx] and idx + 1 < len(sched):", "elif False:"),
 'cap2x': src.replace("elif math.isfinite(dh) and dh - 10 > sched[idx] and idx + 1 < len(sched):", "elif math.isfinite(dh) and dh - 10 > sched[idx] and idx + 1 < len(sched) and sched[idx + 1] <= 2 * d2:"),
 'cap1.5x': src.replace("elif math.isfinite(dh) and dh - 10 > sched[idx] and idx + 1 < len(sched):", "elif math.isfinite(dh) and dh - 10 > sched[idx] and idx + 1 < len(sched) and sched[idx + 1] <= 1.5 * d2:"),
 'every10only': src.replace("elif math.isfinite(dh) and dh - 10 > sched[idx] and idx + 1 < len(sched):", "elif math.isfinite(dh) and dh - 10 > sched[idx] and idx + 1 < len(sched) and sched[idx + 1] * obj.r <= 800:"),
}
for vn, vs in variants.items():
    ns = {}
    exec(vs.replace("def solve(", "def solve_v("), alg1.__dict__, ns)
    tot = 0
    for name in ['c1','c3','c2','c0','ex61_nu0.1','ex61_nu0.01','ex61_nu0.001','ex63_n125000','c4']:
        g = json.load(open(f'/root/repo/tests/golden/{name}.json'))
        rho = make_rho(g); r = g['r']
        f = Fake(rho, r); res = ns['solve_v'](f, 1e-6, g['d_max'], keep_Y=False)
        cost = sum((d*r/1000.)**3 for d in f.calls)
        tot += cost
        print(vn, name, 'd*', res.d_star, 'gold', g['d_star'], 'checks', len(f.calls), 'cost', round(cost, 1))
    print(vn, 'TOTAL cost', round(tot,1))
