"""Random valid CBAA geometries for parity tests (S:37-41 invariants), seeded."""
import numpy as np

from oracle import oracle as O


def random_params(seed, max_cube_bytes=1 << 24, g_choices=(32, 64, 128, 256)):
    """A random config satisfying every SketchConfig invariant, with a small cube."""
    rng = np.random.default_rng(seed)
    while True:
        p = O.default_params()
        r = int(rng.integers(1, 9))
        L = 32 - r
        nra = int(rng.integers(2, 5))
        nva = int(rng.integers(0, 3))
        clbs = sorted(int(x) for x in rng.choice(L, size=nra, replace=False))
        ep = [(clbs[(i + 1) % nra] - clbs[i]) % L for i in range(nra)]
        cbn = []
        for i in range(nra):
            cp = int(rng.integers(0, min(ep[(i + 1) % nra], 4) + 1))
            cbn.append(ep[i] + cp)
        if max(cbn) > 14:
            continue
        cbn += [int(rng.integers(3, 11)) for _ in range(nva)]
        g = int(rng.choice(g_choices))
        p.update(r=r, num_ra=nra, num_va=nva, g=g, cbn=cbn, clbs=clbs,
                 mangle_a=int(rng.integers(0, 1 << 31)) * 2 + 1, mangle_b=int(rng.integers(0, 1 << 32)),
                 bv_seed=int(rng.integers(0, 1 << 32)), va_seeds=[int(x) for x in rng.integers(0, 1 << 32, nva)],
                 theta_formula=int(rng.integers(0, 2)))
        # the GPU build also needs 16-byte CS slices (cbaa_config_validate); the oracle itself is generic
        cs_bytes = O.cube_bytes(p) >> r if O.validate(p)[0] == 0 else 1
        if O.validate(p)[0] == 0 and O.cube_bytes(p) <= max_cube_bytes and cs_bytes % 16 == 0:
            return p
