import collections
def wavefronts(addrs_bytes):
    tot = 0
    for ph in range(4):
        banks = collections.defaultdict(set)
        for a in addrs_bytes[ph*8:(ph+1)*8]:
            for w in range(4):
                word = a//4 + w
                banks[word % 32].add(word)
        tot += max(len(v) for v in banks.values())
    return tot
def swz(e, C):
    r = (e*C) >> 3
    return (r ^ (r >> 3) ^ (r >> 6)) & 7
def addr(e, c, C): return (((e*C + c) ^ swz(e, C)) << 4)
def run(K=8, L=256, G=8, remap=False):
    C = K//4; logL = L.bit_length()-1; lq = logL-2
    out = {}
    for s in range(0, logL, 2):
        h = 1 << s
        ngrp = G << lq
        tot = 0; cnt = 0
        for warp in range(ngrp // 32):
            for q in range(4):
                for c in range(C):
                    addrs = []
                    for l in range(32):
                        grp = warp*32 + l
                        if remap and s >= 2:
                            nb = 1 << (lq - s); pairs = G * nb
                            j = grp // pairs; rest = grp % pairs
                            g = rest // nb; blk = rest % nb
                        else:
                            g = grp >> lq; jj = grp & ((1 << lq)-1); j = jj & (h-1); blk = jj >> s
                        e0 = (g << logL) + (blk << (s+2)) + j
                        addrs.append(addr(e0 + q*h, c, C))
                    tot += wavefronts(addrs); cnt += 1
        out[s] = tot / cnt
    return out
for K in (8, 16, 4):
    L = 256; G = max(1, 16384 // (L*K)); G = min(G, 32)
    print(K, 'cur', run(K, L, G, False), 'remap', run(K, L, G, True))
print('--- rule: remap when G<<(lq-s) >= 32')
def addr_ns(e, c, K):  # non-swizzled: element at e*K words, chunk c = 16B or 4B pieces
    return (e*K)*4 + c*16
def run2(K, L, G):
    logL = L.bit_length()-1; lq = logL-2
    sw = (K % 4 == 0) and ((K//4) & (K//4-1)) == 0 and K//4 <= 8
    C = K//4 if K % 4 == 0 else 1
    res = {}
    for s in range((logL & 1), logL, 2):
        if s == 0 and not (logL & 1): pass
        h = 1 << s
        for remap in (False, True):
            if remap and not (s >= 1 and (G << (lq - s)) >= 32): continue
            tot = 0; cnt = 0
            ngrp = G << lq
            for warp in range(max(1, ngrp // 32)):
                for q in range(4):
                    for c in range(C):
                        addrs = []
                        for l in range(32):
                            grp = (warp*32 + l) % ngrp
                            if remap:
                                nb = 1 << (lq - s); pairs = G * nb
                                j = grp // pairs; rest = grp % pairs; g = rest // nb; blk = rest % nb
                            else:
                                g = grp >> lq; jj = grp & ((1 << lq)-1); j = jj & (h-1); blk = jj >> s
                            e0 = (g << logL) + (blk << (s+2)) + j
                            e = e0 + q*h
                            addrs.append(addr(e, c, C) if sw else addr_ns(e, c, K))
                        tot += wavefronts(addrs); cnt += 1
            res[(s, 'R' if remap else 'c')] = round(tot/cnt, 2)
    return res
import itertools
for K in (1,2,3,4,6,8,12,16,24):
    for logL in range(6, 11):
        L = 1 << logL
        if (2*L)*K*4 > 96*1024 and logL > 6: continue
        G = max(1, 16384 // (L*K)); G = min(G, 32); G = 1 << (G.bit_length()-1)
        r = run2(K, L, G)
        worse = {k: v for k, v in r.items() if k[1] == 'R' and v > r.get((k[0], 'c'), 99)}
        print(K, L, G, r if worse else 'ok', worse)
