"""Compare look-ahead vs serial trailing update after s steps (debug)."""
import os, sys, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), 'tests'))
import numpy as np
name = sys.argv[1] if len(sys.argv) > 1 else 'fix/cliff_m128_n96_r80_g1e+04/qrdm2'
if os.environ.get('CHILD'):
    import golden_cases as G
    from paper_2106_03138_b200 import rrqr
    A = G.case_input(name)
    out = {}
    for s in range(1, 13):
        f = rrqr.factorize(A, max_steps=s)
        r = rrqr.to_result(f)
        out[f'p{s}'] = np.array(r.packed)
        out[f'f{s}'] = np.array(r.perm.forward)
        d = f.debug_ctl()
        g = np.array([d['gamma']]).view(np.int64)[0]
        out[f'd{s}'] = np.array([d['n_s'], d['k_s'], d['l_acc'], d['nsel'], d['kind'], g])
    np.savez(os.environ['CHILD'], **out)
    sys.exit(0)
for mode in ('la', 'serial'):
    env = dict(os.environ, CHILD=f'/tmp/{mode}.npz')
    if mode == 'serial':
        env['DMQR_NO_LOOKAHEAD'] = '1'
    subprocess.run([sys.executable, __file__, name], env=env, check=True)
a, b = np.load('/tmp/la.npz'), np.load('/tmp/serial.npz')
for s in range(1, 13):
    print(s, 'ctl', a[f'd{s}'], b[f'd{s}'], 'perm same', np.array_equal(a[f'f{s}'], b[f'f{s}']),
          'max |diff| packed', np.abs(a[f'p{s}'] - b[f'p{s}']).max())
    dd = np.abs(a[f'p{s}'] - b[f'p{s}'])
    if dd.max() > 1e-16:
        i, j = np.unravel_index(dd.argmax(), dd.shape)
        print('   worst at', i, j, a[f'p{s}'][i, j], b[f'p{s}'][i, j])
        cols = np.where(dd.max(axis=0) > 1e-15)[0]
        rows = np.where(dd.max(axis=1) > 1e-15)[0]
        print('   bad cols', cols[:20], len(cols), 'bad rows', rows[:10], rows[-5:], len(rows))
