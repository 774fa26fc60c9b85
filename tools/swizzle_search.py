import itertools
def wavefronts(addrs_bytes, size):
    # addrs: list of byte addresses (one per lane, in lane order), access size in bytes
    per_group = {16: 8, 8: 16, 4: 32}[size]
    total = 0
    for g in range(0, 32, per_group):
        banks = {}
        for a in addrs_bytes[g:g + per_group]:
            for w in range(size // 4):
                word = a // 4 + w
                banks.setdefault(word % 32, set()).add(word)
        total += max(len(v) for v in banks.values())
    return total
def ideal(addrs, size):
    words = set()
    for a in addrs:
        for w in range(size // 4): words.add(a // 4 + w)
    return -(-len(words) * 4 // 128)
def make_off(h):
    # h: function (r, chi) -> 3-bit xor; layout [rows][32 doubles] = 256 B rows (two 128B lines)
    def off(r, c):
        line = 2 * r + (c >> 4)
        g = (c & 15) >> 1
        return line * 128 + ((g ^ h(r, c >> 4)) << 4) + (c & 1) * 8
    return off
def patterns(off):
    res = []
    # pattern 2: B-frag LDS.64: r = k0 + tq, c = nt*8 + gq
    for k0 in range(0, 32, 4):
        for nt in range(4):
            a = [off(k0 + (l % 4), nt * 8 + l // 4) for l in range(32)]
            res.append(('p2', wavefronts(a, 8), ideal(a, 8)))
    # pattern 3: STS.128 acc: r = mt*16 + gq + 8*v1, c = nt*8 + 2*tq
    for mt in range(2):
        for v1 in range(2):
            for nt in range(4):
                a = [off(mt * 16 + l // 4 + 8 * v1, nt * 8 + 2 * (l % 4)) for l in range(32)]
                res.append(('p3', wavefronts(a, 16), ideal(a, 16)))
    # pattern 1: A-frag LDS.64: r = R0 + gq, c = k0 + tq (for F2T / X)
    for R0 in (0, 8, 16, 24):
        for k0 in range(0, 32, 4):
            a = [off(R0 + l // 4, k0 + l % 4) for l in range(32)]
            res.append(('p1', wavefronts(a, 8), ideal(a, 8)))
    return res
def score(res, which):
    w = sum(x[1] for x in res if x[0] in which); i = sum(x[2] for x in res if x[0] in which)
    return w, i
cur = make_off(lambda r, chi: (2 * r + chi) & 7)
res = patterns(cur)
for p in ('p1', 'p2', 'p3'): print('current', p, score(res, (p,)))
best = None
for bits in itertools.product(range(8), repeat=4):  # columns of the GF(2) matrix for r0, r1, r2, chi
    def h(r, chi, bits=bits):
        v = 0
        for i, b in enumerate(((r >> 0) & 1, (r >> 1) & 1, (r >> 2) & 1, chi)):
            if b: v ^= bits[i]
        return v
    res = patterns(make_off(h))
    w23, i23 = score(res, ('p2', 'p3'))
    w1, _ = score(res, ('p1',))
    key = (w23, w1)
    if best is None or key < best[0]: best = (key, bits, score(res, ('p2',)), score(res, ('p3',)), score(res, ('p1',)))
print('best', best)

def pipe_gx(ch):
    g0, g1, g2 = ch & 1, (ch >> 1) & 1, (ch >> 2) & 1
    return (g2 | (g1 << 1) | ((g0 ^ g1) << 2)) << 4
def p4(off):
    tot = 0; idl = 0
    for base in range(0, 1024, 4):
        a = []
        for l in range(32):
            g = l % 8; u = base + l // 8
            a.append(g * 8192 + (off(u // 32, u % 32) ^ pipe_gx(g)))
        tot += wavefronts(a, 8); idl += ideal(a, 8)
    return tot, idl
def hz(r, chi): return ((r & 1) << 2) | (((r >> 1) & 1) << 1)
print('p4 current', p4(cur), 'p4 new', p4(make_off(hz)))
res = patterns(make_off(hz))
for p in ('p1', 'p2', 'p3'): print('new', p, score(res, (p,)))

# v7: F2^T tile [32 rows][64 doubles] (512-byte rows), A-fragment gathers r = R0 + gq, c = k0 + tq (LDS.64)
def f2t_cost(h):
    tot = idl = 0
    for R0 in (0, 8, 16, 24):
        for k0 in range(0, 64, 4):
            a = [(R0 + l // 4) * 512 + (((k0 + l % 4) * 8) ^ (h(R0 + l // 4) << 4)) for l in range(32)]
            tot += wavefronts(a, 8); idl += ideal(a, 8)
    return tot, idl
print('F2T rowswz64', f2t_cost(lambda r: r & 7), 'new', f2t_cost(lambda r: ((r & 3) << 1) | ((r >> 2) & 1)))
