# How many Gram entries of a forward tile share a product monomial (config 4)?
# Standalone (own colex rank), samples 40 random upper-triangle 256x160 tiles.
import itertools, math, random
n, d = 17, 5
# colex order of sorted multisets (s1<=...<=sd): rank = sum C(s_k + k - 1, k)
mons = list(itertools.combinations_with_replacement(range(n), d))
def rank(ms): return sum(math.comb(s + k, k + 1) for k, s in enumerate(ms))
mons.sort(key=rank)
N = len(mons)
random.seed(0)
tot = 0; dist = 0
for _ in range(40):
    a = random.randrange(N // 256); b = random.randrange(a * 256 // 160, (N + 159) // 160)
    S = set()
    cnt = 0
    for i in range(a * 256, min(N, a * 256 + 256)):
        for j in range(b * 160, min(N, b * 160 + 160)):
            if j < i: continue
            S.add(tuple(sorted(mons[i] + mons[j]))); cnt += 1
    tot += cnt; dist += len(S)
print(N, "pairs", tot, "distinct", dist, "ratio", tot / dist)
