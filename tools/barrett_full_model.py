import random
def limbs(x, n): return [(x >> (32*i)) & 0xffffffff for i in range(n)]
def val(l): return sum(v << (32*i) for i, v in enumerate(l))
def hi_trunc(a, b, K, D=2):
    C0 = K - D if K > D else 0
    acc = 0
    for i in range(K):
        for j in range(K):
            if i + j >= C0: acc += a[j]*b[i] << (32*(i+j-C0))
    return limbs(acc >> (32*(K - C0)), K)
def model(a, b, q, K):
    M = 32*K; qb = q.bit_length(); s = M - qb
    qn = q << s
    mu = (1 << (2*M)) // qn
    assert mu >> M == 1, hex(mu)
    mu_lo = mu - (1 << M)
    t = (a << s) * b
    q1 = t >> (M-1)
    q1_lo, q1top = q1 & ((1<<M)-1), q1 >> M
    X = val(hi_trunc(limbs(q1_lo, K), limbs(mu_lo, K), K)) + q1top*mu_lo
    q3 = (q1 + X) >> 1
    r = (t - q3*qn) % (1 << (32*(K+1)))
    Q = t // qn
    assert Q - 4 <= q3 <= Q, (Q - q3)
    assert r < 5*qn, r / qn
    for m in (4*qn, 2*qn, qn):
        if r >= m: r -= m
    return r >> s
rnd = random.Random(1)
worst = 0
for K in (1, 2, 4, 8, 12):
    for _ in range(300):
        q = rnd.randrange(3, 1 << (32*K)) | 1
        if rnd.random() < 0.3: q = (1 << (32*K)) - rnd.randrange(1, 1000) | 1
        if rnd.random() < 0.2: q = (1 << (32*K - 1 - rnd.randrange(0, 31))) + rnd.randrange(1, 100) | 1
        for a, b in [(q-1, q-1), (q-1, 1), (0, q-1), (rnd.randrange(q), rnd.randrange(q)), (q//2, q-1)]:
            assert model(a, b, q, K) == a*b % q
print("model ok")
