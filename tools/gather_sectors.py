# Distinct 32-byte sectors of res touched by one warp-wide gather of the R packers
# (32 lanes, one PT component each) under different lane -> (row, 4-column group)
# maps of a 64 x 64 block.  Standalone (own colex rank, as tile_rank_dups.py).
# python tools/gather_sectors.py [n d]   (default: config 4, n=17 d=5)
import itertools, math, random, sys
n, d = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (17, 5)


def rank(ms):  # colex rank of a sorted multiset s1 <= ... <= sk: sum C(s_k + k - 1, k)
    return sum(math.comb(s + k, k + 1) for k, s in enumerate(ms))


mons = sorted(itertools.combinations_with_replacement(range(n), d), key=rank)
N = len(mons)
nb = N // 64
random.seed(0)
maps = {"2 rows x 16 groups (round 2)": (2, 16), "8 rows x 4 groups (rt_gather_pos)": (8, 4),
        "16 rows x 2 groups": (16, 2), "4 rows x 8 groups": (4, 8), "32 rows x 1 group": (32, 1)}
tot = {k: 0 for k in maps}
blocks = 0
while blocks < 10:
    I = random.randrange(nb)
    J = random.randrange(I, nb)
    P = [[rank(tuple(sorted(mons[I * 64 + i] + mons[J * 64 + j]))) for j in range(64)] for i in range(64)]
    for k, (R, C) in maps.items():
        for r0 in range(0, 64, R):
            for c0 in range(0, 16, C):
                for comp in range(4):
                    tot[k] += len({P[r0 + l // C][4 * (c0 + l % C) + comp] >> 3 for l in range(32)})
    blocks += 1
print(f"n={n} d={d} N={N}: sectors per warp gather over {blocks} blocks")
for k, v in tot.items():
    print(f"  {k:36s} {v / (blocks * 128):6.2f}")
