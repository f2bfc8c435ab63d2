"""Generate tests/golden/*.json from the REFERENCE's own rng (and the oracle's sparse-sign stream).

Run in the build container (needs /root/reference): it compiles the reference's unmodified
proj/src/rng.cpp into oracle/_ref/libref_rng.so (oracle/Makefile `ref`) and records
philox4x32 / normal_at / uniform_at outputs as exact hex doubles. The GPU box never reads
/root/reference; the tests only read the committed JSON.

The sparse-sign stream has no reference implementation: its vectors are
produced by the oracle's own restatement of the A.8 definition (self-pinned).
"""
import ctypes as C
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)


def main():
    subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "all", "ref"], check=True)
    ref = C.CDLL(os.path.join(ROOT, "oracle", "_ref", "libref_rng.so"))
    ref.ref_normal_at.restype = C.c_double
    ref.ref_normal_at.argtypes = [C.c_uint64, C.c_uint32, C.c_int64, C.c_int64]
    ref.ref_uniform_at.restype = C.c_double
    ref.ref_uniform_at.argtypes = [C.c_uint64, C.c_uint32, C.c_int64, C.c_int64]
    ref.ref_philox4x32.argtypes = [C.POINTER(C.c_uint32)] * 3

    def philox(ctr, key):
        c = (C.c_uint32 * 4)(*ctr)
        k = (C.c_uint32 * 2)(*key)
        o = (C.c_uint32 * 4)()
        ref.ref_philox4x32(c, k, o)
        return list(o)

    ctrs = [([0, 0, 0, 0], [0, 0]), ([0xFFFFFFFF] * 4, [0xFFFFFFFF, 0xFFFFFFFF]),
            ([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0]),
            ([1, 2, 3, 4], [5, 6]), ([7, 0, 11, 0], [42, 0])]
    kat_philox = [{"ctr": c, "key": k, "out": philox(c, k)} for c, k in ctrs]

    seeds = [0, 1, 42, 7, (1 << 40) + 3, 0xFFFFFFFFFFFFFFFF]
    ij = [(0, 0), (0, 1), (0, 2), (1, 0), (1, 1), (1, 2), (10, 1999), (54, 99999), (69, 199999),
          ((1 << 32) + 5, 3), (2, (1 << 33) + 1), ((1 << 35) + 7, (1 << 34) + 9)]
    normals, uniforms = [], []
    for s in seeds:
        for stream in (1, 2, 3, 4, 5, 6):
            for i, j in ij:
                normals.append([str(s), stream, i, j, ref.ref_normal_at(s, stream, i, j).hex()])
                uniforms.append([str(s), stream, i, j, ref.ref_uniform_at(s, stream, i, j).hex()])
    # one full sketch-stream block (config 1 shape: c = 11 rows, first 512 columns)
    block = [[ref.ref_normal_at(0, 1, i, j).hex() for j in range(512)] for i in range(11)]
    with open(os.path.join(HERE, "rng_kat.json"), "w") as f:
        json.dump({"source": "reference proj/src/rng.cpp compiled by oracle/Makefile (ref)",
                   "philox": kat_philox, "normal_at": normals, "uniform_at": uniforms,
                   "sketch_block_seed0_11x512": block}, f, indent=0)

    from oracle import oracle as O
    pats = []
    for c, m, seed in ((22, 64, 3), (55, 64, 11), (11, 40, 0), (5, 16, 9), (70, 32, 123)):
        rows, signs = O.sparse_sign_pattern(c, m, seed, 8)
        pats.append({"c": c, "m": m, "seed": seed, "zeta": 8, "rows": rows.tolist(), "signs": signs.tolist()})
    with open(os.path.join(HERE, "sparse_sign_kat.json"), "w") as f:
        json.dump({"source": "oracle restatement of SURVEY.md A.8 (no reference implementation: self-pinned)",
                   "patterns": pats}, f, indent=0)
    print("wrote", os.listdir(HERE))


if __name__ == "__main__":
    main()
