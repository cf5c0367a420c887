"""Host restatement of fbb_synth_pool's generator (csrc/synth.cu) for the tests."""
M64 = (1 << 64) - 1


def _splitmix(state):
    state = (state + 0x9E3779B97F4A7C15) & M64
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return state, z ^ (z >> 31)


def synth_prefix(n, seed, i, min_depth, max_depth):
    s = (seed ^ ((i * 0xD1B54A32D192ED03) & M64)) & M64
    s, r = _splitmix(s)
    depth = min_depth + r % (max_depth - min_depth + 1)
    perm = list(range(n))
    for d in range(depth):
        s, r = _splitmix(s)
        pick = d + r % (n - d)
        perm[pick], perm[d] = perm[d], perm[pick]
    return perm[:depth]
