import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import golden_cases as G, parity
from paper_2106_03138_b200 import qrdm, qrdm2, DMParams, StopCriterion, StopRule
for name in ['fix/cliff_m160_n128_r116_g1e+04/qrdm', 'fix/cliff_m160_n128_r116_g1e+04/qrdm2']:
    A = G.case_input(name); kw = G.oracle_kwargs(name)
    meta = G.index()["cases"][name]
    fn = qrdm2 if meta["algo"] == "qrdm2" else qrdm
    r = fn(A, params=DMParams(**{k: kw[k] for k in ("tau","delta","k_dm","use_delta_max") if k in kw}), stop=StopCriterion(StopRule(kw.get("stop_rule","n"))))
    print(name, kw, parity.residuals(A, r), r.rank, [(s.n_s, s.k_selected, s.k_accepted) for s in r.step_log])
from paper_2106_03138_b200 import rrqr
for name in ['fix/cliff_m160_n128_r116_g1e+04/qrdm']:
    A = G.case_input(name)
    for s in (1, 2):
        f = rrqr.factorize(A, break_check=False, max_steps=s)
        d = f.debug_ctl()
        print(s, 'cq_fail/tc0', d.get('gamma'), 'diag', d['cq_diag'])
