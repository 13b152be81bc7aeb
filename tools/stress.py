"""Randomised parity stress (beyond the test suite): NTT forward/inverse at
random (width, n, batch) against the C oracle, BLAS ops at random widths and
moduli against Python integers, full-width NTTs against run_ntt_exact."""
import random, sys, time
sys.path.insert(0, '.')
import numpy as np
from oracle import bigint
from oracle.cbind import OracleField
from paper_2501_07535_b200 import device as dev
from paper_2501_07535_b200 import kernels as K
from paper_2501_07535_b200.params import find_ntt_params, NoSuitablePrime, NttParams

rnd = random.Random(int(sys.argv[1]) if len(sys.argv) > 1 else 1)
t_end = time.time() + (float(sys.argv[2]) if len(sys.argv) > 2 else 240)
widths = [8, 16, 24, 32, 48, 64, 96, 100, 128, 160, 192, 200, 224, 256, 288, 320, 352, 384, 416, 448, 480, 512,
          544, 640, 768, 800, 992, 1024]
cases = fails = 0
while time.time() < t_end:
    kind = rnd.choice(["ntt", "blas", "fullntt"])
    bits = rnd.choice(widths)
    try:
        if kind == "ntt":
            big = len(sys.argv) > 3 and sys.argv[3] == "big"
            logn = rnd.randint(1, (18 if big else 14) if bits <= 256 else (14 if bits <= 512 else 11))
            n = 1 << logn
            try:
                prm = find_ntt_params(bits, n)
            except NoSuitablePrime:
                continue
            plan = K.get_plan(bits, prm)
            batch = rnd.randint(1, 4)
            kn = (bits + 31) // 32
            vals = bigint.uniform_residues(np.random.Generator(np.random.PCG64(rnd.getrandbits(32))), batch * n, prm.p)
            xl = dev.ints_to_limbs(vals, kn)
            xd = dev.to_device(dev.ints_to_limbs(vals, plan.limbs))
            of = OracleField(prm.p, bits)
            inv = rnd.random() < 0.5
            got = dev.to_host(plan.inverse(xd) if inv else plan.forward(xd))[:, :kn]
            want = of.ntt(xl, n, prm.root_inv, prm.n_inv) if inv else of.ntt(xl, n, prm.root)
            ok = np.array_equal(got, want)
            tag = (kind, bits, n, batch, inv)
        elif kind == "blas":
            q = rnd.randrange((1 << (bits - 5)) + 1, 1 << (bits - 4)) | rnd.choice([0, 1])
            strat = rnd.choice(["schoolbook", "karatsuba", "montgomery"])
            if strat == "montgomery":
                q = rnd.randrange(3, 1 << bits) | 1
            elif bits >= 96 and rnd.random() < 0.4 and max(72, 32 * ((bits + 31) // 32) - 31) < bits - 3:
                # special form q = 2^m - c, c < 2^32 (the two-fold reduction path;
                # m within 31 bits of the limb top and below 2^(bits-4))
                mm = rnd.randrange(max(72, 32 * ((bits + 31) // 32) - 31), bits - 3)
                q = (1 << mm) - rnd.randrange(1, 1 << 32)
            try:
                f = dev.Field(bits, q, strat)
            except Exception:
                continue
            m = rnd.randint(1, 3000)
            off = rnd.choice([0, 0, 1, 3])  # element offset: unaligned bases (no packed accesses)
            xs = [rnd.randrange(q) for _ in range(m + off)]
            ys = [rnd.randrange(q) for _ in range(m + off)]
            op = rnd.choice(["vadd", "vsub", "vmul", "axpy"])
            x = dev.to_device(dev.ints_to_limbs(xs, f.limbs))[off:]
            y = dev.to_device(dev.ints_to_limbs(ys, f.limbs))[off:]
            xs, ys = xs[off:], ys[off:]
            s = rnd.randrange(q)
            out = dev.limbs_to_ints(dev.to_host(f.axpy(s, x, y) if op == "axpy" else getattr(f, op)(x, y)))
            want = {"vadd": [(a + b) % q for a, b in zip(xs, ys)], "vsub": [(a - b) % q for a, b in zip(xs, ys)],
                    "vmul": [a * b % q for a, b in zip(xs, ys)], "axpy": [(s * a + b) % q for a, b in zip(xs, ys)]}[op]
            ok = out == want
            tag = (kind, op, bits, strat, f.reduction, hex(q)[:12], m, off)
        else:
            if bits < 32:
                continue
            a2 = 20
            while True:
                pb = rnd.randrange(max(a2 + 2, bits - 3), bits + 1)
                c = rnd.randrange(2 ** (pb - a2 - 1), 2 ** (pb - a2))
                p = c * 2**a2 + 1
                if p.bit_length() == pb and bigint.is_prime(p):
                    break
            logn = rnd.randint(1, 10)
            n = 1 << logn
            x0 = 2
            while pow(x0, (p - 1) // 2, p) != p - 1:
                x0 += 1
            w = pow(x0, (p - 1) // n, p)
            f = dev.Field(bits, p, "montgomery")
            plan = dev.NttPlan(f, NttParams(n=n, p=p, root=w, root_inv=pow(w, -1, p), n_inv=pow(n, -1, p)))
            xs = [rnd.randrange(p) for _ in range(n)]
            got = dev.limbs_to_ints(dev.to_host(plan.forward(dev.to_device(dev.ints_to_limbs(xs, f.limbs)))))
            ok = got == bigint.run_ntt_exact(xs, p, w, pow(n, -1, p))
            tag = (kind, bits, pb, n)
        cases += 1
        if not ok:
            fails += 1
            print("FAIL", tag, flush=True)
    except Exception as exc:
        fails += 1
        print("ERROR", kind, bits, repr(exc)[:200], flush=True)
print(f"stress: {cases} cases, {fails} failures", flush=True)
