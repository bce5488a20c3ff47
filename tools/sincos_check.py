import subprocess, sys, numpy as np, math
sys.path.insert(0, '.')
import oracle
fs = 8.184e6
for f in (800.0, 1000.0, -4321.0, 12345.6):
    step = oracle.gnss_oracle.carrier_step_to_fixed(f, fs)
    n = 200000
    ref = oracle.carrier_replica(0.0, f, fs, n)
    for mode in (0, 1):
        raw = subprocess.run(['./tools/sincos_probe', '0', str(step), str(n), str(mode)], capture_output=True).stdout
        got = np.frombuffer(raw, dtype=np.complex64)
        bad = np.flatnonzero(got != ref)
        print(f, 'mode', mode, 'mismatches', bad.size, 'of', n, bad[:5])
# numba (the reference's active twin) vs numpy twin
import numba
@numba.njit
def nb(p0, s, n, out):
    mask = np.uint64((1 << 48) - 1); p = np.uint64(p0); s = np.uint64(s)
    inv = 2.0 * math.pi / (1 << 48)
    for i in range(n):
        th = np.float64(p) * inv
        out[i] = complex(math.cos(th), -math.sin(th))
        p = (p + s) & mask
out = np.empty(200000, np.complex64)
step = oracle.gnss_oracle.carrier_step_to_fixed(800.0, fs)
nb(0, step, 200000, out)
print('numba vs numpy mismatches', np.count_nonzero(out != oracle.carrier_replica(0.0, 800.0, fs, 200000)))
