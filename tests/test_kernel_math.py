"""CPU checks of integer identities the CUDA kernels rely on (no GPU, no library calls): each
test restates a kernel helper's arithmetic in Python and checks it against plain integer
division / digit parsing over the whole input range the kernel guarantees."""
import random


def pane30_magic(S):
    # kernels_cm.cu pane30_magic: k = max(32, 30 + ceil(log2 S)), M = ceil(2^k / S), shift k - 32
    if S <= 1:
        return 0, 32
    lg = 0
    while (1 << lg) < S:
        lg += 1
    k = max(32, lg + 30)
    return ((1 << k) + S - 1) // S, k - 32


def pane30(ts, m, sh):
    return ts if sh == 32 else ((ts * m) >> 32) >> sh


def test_pane30_is_floor_division_below_2_pow_30():
    rng = random.Random(7)
    slides = list(range(1, 130)) + [300, 600, 3600, 86400, 10 ** 6, 2 ** 20 + 1, 2 ** 29 + 3, 2 ** 30 - 1]
    for S in slides:
        m, sh = pane30_magic(S)
        assert m < 2 ** 32
        cases = [0, 1, S - 1, S, S + 1, 2 ** 30 - 1, 999_999_999, 99_999_999]
        cases += [q * S + r for q in (1, 2, (2 ** 30 - 1) // S) for r in (-1, 0, 1) if 0 <= q * S + r < 2 ** 30]
        cases += [rng.randrange(2 ** 30) for _ in range(300)]
        for ts in cases:
            assert pane30(ts, m, sh) == ts // S, (S, ts)


def swar4d(d):
    # kernels_cm.cu swar4d: 4 digit values (first = most significant) -> value
    p = (d * 0xA01) & 0xFFFFFFFF
    p = ((p >> 8) & 0xFF) | (((p >> 24) & 0xFF) << 16)       # __byte_perm(p, 0, 0x4341)
    return ((p * 0x640001) & 0xFFFFFFFF) >> 16


def test_swar4d_all_four_digit_strings():
    for v in range(10000):
        s = f"{v:04d}"
        d = sum((ord(c) - 48) << (8 * i) for i, c in enumerate(s))
        assert swar4d(d) == v


def test_ts_shift_decode_all_lengths():
    # kernels_cm.cu cm_fast ts: bytes [S, S+8) = o0 digits, ',', garbage; 64-bit subtract of
    # '0' from every byte, shift left by 8 * (8 - o0): the digit values end up in the top o0 bytes
    rng = random.Random(3)
    for _ in range(3000):
        o0 = rng.randint(1, 8)
        ts = rng.randrange(10 ** o0)
        txt = f"{ts}".encode()
        txt = (b"0" * (o0 - len(txt))) + txt if rng.random() < 0.2 else txt
        o0 = len(txt)
        tail = bytes([44]) + bytes(rng.randrange(256) for _ in range(7))
        raw = (txt + tail)[:8]
        w = int.from_bytes(raw, "little")
        t = (w - 0x3030303030303030) % 2 ** 64
        t = (t << (8 * ((8 - o0) & 7))) % 2 ** 64
        lo, hi = t & 0xFFFFFFFF, t >> 32
        bad = 0
        for x in (lo, hi):
            bad |= (x | ((x + 0x76767676) & 0xFFFFFFFF)) & 0x80808080
        assert bad == 0
        assert swar4d(lo) * 10000 + swar4d(hi) == int(txt)


def floor_div_S(a, S):
    # common.cuh floor_div_S: pane_of's magic ceil(2^64 / S) (lmstream.cpp: ~0 / S + 1),
    # umul64hi for 0 <= a < 2^32, -1 - floor((-a - 1) / S) for -2^32 < a < 0
    magic = ((2 ** 64 - 1) // S) + 1 if S > 1 else 0

    def pane_of(ts):
        return ts if S == 1 else (ts * magic) >> 64

    if 0 <= a < 2 ** 32:
        return pane_of(a)
    if -(2 ** 32) < a < 0:
        return -pane_of(-a - 1) - 1
    return a // S


def test_floor_div_S_is_floor_division():
    rng = random.Random(11)
    for S in list(range(1, 70)) + [300, 3600, 86400, 2 ** 20, 2 ** 31 - 1, 2 ** 31]:
        cases = [0, 1, -1, S - 1, S, -S, -S - 1, 2 ** 32 - 1, -(2 ** 32) + 1, 2 ** 32, -(2 ** 32) - 5]
        cases += [q * S + r for q in (-3, -1, 1, 7, (2 ** 32 - 1) // S) for r in (-1, 0, 1)]
        cases += [rng.randrange(-(2 ** 32) + 1, 2 ** 32) for _ in range(300)]
        for a in cases:
            assert floor_div_S(a, S) == a // S, (S, a)


def test_lr_pair_field_decode():
    # kernels_lr.cu lr_decode: a record pair as 35 little-endian words; a field of N <= 4 digits
    # at byte B = funnel shift of words B // 4, B // 4 + 1 by 8 * (B % 4), minus '0' in every
    # byte, shifted left by 8 * (4 - N), swar4d; 6 / 10 digits from 4 + 2 / 4 + 4 + 2.  The
    # bytes after a field are arbitrary (commas, other fields, the next record): random here.
    import lmsgen as g
    rng = random.Random(5)
    data = g.second_bytes("LR", 7, 400, 11)
    for k in range(0, len(data) - 139, 140):
        pair = bytearray(data[k:k + 140])
        w = [int.from_bytes(pair[4 * j:4 * j + 4], "little") for j in range(35)]

        def bytes4(b):
            lo, hi = w[b // 4], w[b // 4 + 1] if b // 4 + 1 < 35 else 0
            return ((lo | (hi << 32)) >> (8 * (b % 4))) & 0xFFFFFFFF

        def dec(b, n):
            d = (bytes4(b) - 0x30303030) & 0xFFFFFFFF
            return d & 0xFF if n == 1 else swar4d((d << (8 * (4 - n))) & 0xFFFFFFFF)

        for base in (0, 70):
            rec = pair[base:base + 70].decode()
            f = rec.rstrip("\n").split(",")
            assert dec(base + 2, 4) * 100 + dec(base + 6, 2) == int(f[1])                   # Time
            assert (dec(base + 9, 4) * 10000 + dec(base + 13, 4)) * 100 + dec(base + 17, 2) == int(f[2])   # VID
            assert dec(base + 20, 3) == int(f[3]) and dec(base + 24, 3) == int(f[4])       # Spd, XWay
            assert dec(base + 28, 1) == int(f[5]) and dec(base + 30, 1) == int(f[6])       # Lane, Dir
            assert dec(base + 32, 3) == int(f[7])                                          # Seg
    # random digit strings at every alignment, arbitrary bytes after them
    for _ in range(2000):
        n = rng.randint(1, 4)
        b = rng.randint(0, 100)
        digits = "".join(rng.choice("0123456789") for _ in range(n))
        pair = bytearray(rng.randrange(256) for _ in range(140))
        pair[b:b + n] = digits.encode()
        w = [int.from_bytes(pair[4 * j:4 * j + 4], "little") for j in range(35)]
        lo, hi = w[b // 4], w[b // 4 + 1]
        x = ((lo | (hi << 32)) >> (8 * (b % 4))) & 0xFFFFFFFF
        d = (x - 0x30303030) & 0xFFFFFFFF
        got = d & 0xFF if n == 1 else swar4d((d << (8 * (4 - n))) & 0xFFFFFFFF)
        assert got == int(digits), (b, n, digits)
