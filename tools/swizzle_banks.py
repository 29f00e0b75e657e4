"""Shared-memory bank check for k_agg3's / k_agg6's tile under the 64-byte (IL) / 32-byte (IL8, HGF_WG8) TMA swizzle
and the planar odd-pitch tile: counts wavefronts per quarter-warp for the owner LDS.128 pattern and ways per warp for
the vertical pass; k_agg6's 16-pixel owners (4 rows x 2 segments per quarter-warp, 8 rows per warp) as well.
Usage: python tools/swizzle_banks.py [R]
"""
import sys

TX, TY, KX = 64, 24, 8


def swz(f):
    return f ^ ((f >> 3) & 12)


def swz32(f):
    """32-byte TMA swizzle (8-pixel groups, HGF_WG8; measured by tools/tma_swz8.cu)."""
    return f ^ ((f >> 3) & 4)


def owner(ln, wq, il):
    if il == 2:
        return (ln >> 3) + 4 * wq, ln & 7
    if il:
        return (ln & 3) + 4 * wq, ((ln >> 3) & 1) + 4 * (ln >> 4) + 2 * ((ln >> 2) & 1)
    return (ln & 7) + 8 * (wq % 3), (ln >> 3) + 4 * (wq // 3)


def lds128_wavefronts(addrs):
    tot = 0
    for q in range(4):
        banks = {}
        for a in addrs[8 * q:8 * q + 8]:
            for j in range(4):
                banks.setdefault((a + j) % 32, set()).add((a + j) // 32)
        tot += max(len(v) for v in banks.values())
    return tot


def main():
    R = int(sys.argv[1]) if len(sys.argv) > 1 else 9
    K = 7
    WX, BY = TX + 2 * R, TY + 2 * R
    nv4 = (KX + 2 * R + 3) // 4
    for il in (0, 1, 2):
        if il:
            BX = (WX + 31) // 32 * 32
            f = swz if il == 1 else swz32
        else:
            BX = (WX + 3) // 4 * 4
            while (BX // 4) % 2 == 0:
                BX += 4
            f = (lambda v: v)
        worst = 0
        for wq in range(TY * (TX // KX) // 32):
            for k in range(K):
                for q in range(nv4):
                    addrs = []
                    for ln in range(32):
                        oy, seg = owner(ln, wq, il)
                        addrs.append(f((k * BY + oy) * BX + seg * KX + 4 * q))
                    worst = max(worst, lds128_wavefronts(addrs))
        vworst = 0
        for w0 in range(0, K * WX, 32):
            for y in range(BY):
                banks = {}
                for item in range(w0, min(w0 + 32, K * WX)):
                    k, c = divmod(item, WX)
                    a = f((k * BY + y) * BX + c)
                    banks.setdefault(a % 32, set()).add(a // 32)
                vworst = max(vworst, max(len(v) for v in banks.values()))
        print(f"R={R} {['planar', 'IL/swizzle64', 'IL8/swizzle32'][il]}: BX={BX} owner LDS.128 worst {worst} wavefronts "
              f"(ideal 4); vertical pass worst {vworst}-way")


def owner16(ln, wq):
    """k_agg6 16-pixel owners (D >= 1): row, segment of lane ln in owner warp wq."""
    return (ln & 3) + 4 * (ln >> 4) + 8 * wq, (ln >> 2) & 3


def lds_wavefronts(addrs, width):
    """LDS.128 is served per quarter-warp (8 lanes), LDS.64 per half-warp (16 lanes)."""
    grp = 8 if width == 4 else 16
    tot = 0
    for g0 in range(0, 32, grp):
        banks = {}
        for a in addrs[g0:g0 + grp]:
            for j in range(width):
                banks.setdefault((a + j) % 32, set()).add((a + j) // 32)
        tot += max(len(v) for v in banks.values())
    return tot


def main16(R):
    BX, nf = 96, 16 + 2 * R
    res = set()
    for wq in range(6):
        for q in range((nf + 3) // 4):
            width = 4 if 4 * q + 4 <= nf else nf - 4 * q
            addrs = [swz(owner16(ln, wq)[0] * BX + owner16(ln, wq)[1] * 16 + 4 * q) for ln in range(32)]
            res.add((width, lds_wavefronts(addrs, width)))
    print(f"R={R} k_agg6 16-pixel owners: (load width in floats, wavefronts per warp load) = {sorted(res)} "
          f"(ideal: 4 for 128-bit loads)")


if __name__ == "__main__":
    main()
    main16(int(sys.argv[1]) if len(sys.argv) > 1 else 9)
