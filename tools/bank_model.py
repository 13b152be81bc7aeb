import collections
def wavefronts(addrs_bytes):  # 32 lanes, 16-B accesses
    tot = 0
    for ph in range(4):
        banks = collections.defaultdict(set)
        for a in addrs_bytes[ph*8:(ph+1)*8]:
            for w in range(4):
                word = a//4 + w
                banks[word % 32].add(word)
        tot += max(len(v) for v in banks.values())
    return tot
def swz_none(A): return A
def swz_x(A): return A ^ ((A >> 3) & 7)
def swz_x2(A): return A ^ ((A >> 2) & 6) if False else A ^ (((A >> 3) ^ (A >> 6)) & 7)
K=8; C=K//4; L=256; logL=8
for name, sw in [("none", swz_none), ("xor3", swz_x), ("xor36", swz_x2)]:
    tot = 0; detail=[]
    for s in range(logL):
        half = 1 << s
        w = 0
        for warp in range(8):  # first 8 warps
            lanes = [warp*32 + l for l in range(32)]
            for off in (0, half):
                for c in range(C):
                    addrs = []
                    for bf in lanes:
                        g = bf >> (logL-1); jj = bf & (L//2-1); j = jj & (half-1)
                        p0 = ((jj >> s) << (s+1)) + j
                        e = g*L + p0 + off
                        addrs.append(sw(e*C + c)*16)
                    w += wavefronts(addrs)
        detail.append(w // (8*2*C))
        tot += w
    # loads/stores of natural-order output: idx -> (k, g) col pass: k = idx / G, g = idx % G, elem g*L+k
    w = 0
    G = 8
    for warp in range(8):
        for c in range(C):
            addrs = []
            for l in range(32):
                idx = warp*32+l; k = idx // G; g = idx % G
                addrs.append(sw((g*L+k)*C + c)*16)
            w += wavefronts(addrs)
    print(name, "per-stage wavefronts per warp-LDS.128:", detail, " epilogue col:", w/(8*C))

def fold(x):
    r = 0
    while x:
        r ^= x & 7; x >>= 3
    return r
def swz_fold(A): return A ^ (fold(A >> 3) & 7)
def brev(t, bits): return int(format(t, f"0{bits}b")[::-1], 2)
def eval_all(sw, K=8, L=256, G=8):
    C = K//4; logL = L.bit_length()-1
    res = {}
    st = []
    for s in range(logL):
        half = 1 << s; w = 0; cnt = 0
        for warp in range(min(8, G*L//2//32)):
            for off in (0, half):
                for c in range(C):
                    addrs = []
                    for l in range(32):
                        bf = warp*32+l
                        g = bf >> (logL-1); jj = bf & (L//2-1); j = jj & (half-1)
                        p0 = ((jj >> s) << (s+1)) + j
                        addrs.append(sw((g*L+p0+off)*C + c)*16)
                    w += wavefronts(addrs); cnt += 1
        st.append(w/cnt)
    res['stages'] = st
    for kind in ('col_load', 'col_store', 'row_load', 'row_store'):
        w = 0; cnt = 0
        for warp in range(8):
            for c in range(C):
                addrs = []
                for l in range(32):
                    idx = warp*32+l
                    if kind.startswith('col'):
                        t = idx // G; g = idx % G
                    else:
                        g = idx >> logL; t = idx & (L-1)
                    p = brev(t, logL) if kind.endswith('load') else t
                    addrs.append(sw((g*L+p)*C + c)*16)
                w += wavefronts(addrs); cnt += 1
        res[kind] = w/cnt
    return res
for K in (8, 12, 16, 24):
    for nm, sw in [("none", swz_none), ("xor3", swz_x), ("fold", swz_fold)]:
        L = 256
        G = max(1, 16384 // (L*K)); G = 1 << (G.bit_length()-1)
        print(K, nm, eval_all(sw, K, L, G))
