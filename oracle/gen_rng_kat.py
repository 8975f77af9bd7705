"""Generate tests/golden/rng_kat.json from the reference's OWN rng.cpp.

TEST INFRASTRUCTURE. Run here (in the container that has /root/reference):
    make -C oracle ref && python oracle/gen_rng_kat.py
The library oracle/_ref/librefrng.so is /root/reference/proj/core/src/seqpar/rng.cpp compiled
unmodified (oracle/Makefile `ref`), so these vectors are the reference's behaviour, not ours.
"""
import ctypes as C
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "..", "tests", "golden", "rng_kat.json")


def main():
    lib = C.CDLL(os.path.join(HERE, "_ref", "librefrng.so"))
    u64, u32, i64, dbl = C.c_uint64, C.c_uint32, C.c_int64, C.c_double
    lib.ref_hash_counter.restype = u64
    lib.ref_hash_counter.argtypes = [u64, u64]
    lib.ref_uniform01.restype = dbl
    lib.ref_uniform01.argtypes = [u64, u64]
    lib.ref_mask_key_fold.restype = u64
    lib.ref_mask_key_fold.argtypes = [u64, u32, u32, u32]
    lib.ref_random_uniform.argtypes = [u64, i64, dbl, dbl, C.POINTER(dbl)]
    lib.ref_dropout_mask.restype = C.c_int
    lib.ref_dropout_mask.argtypes = [u64, u32, u32, u32, i64, dbl, C.POINTER(dbl)]

    kat = {"source": "/root/reference/proj/core/src/seqpar/rng.cpp (compiled via oracle/Makefile ref)"}
    folds = []
    for seed in (0, 1, 7, 42, 2**63 + 5, 2**64 - 1):
        for layer in (0, 1, 47):
            for op in (0, 1, 2):
                for mb in (0, 1, 3):
                    folds.append([str(seed), layer, op, mb, str(lib.ref_mask_key_fold(seed, layer, op, mb))])
    kat["fold"] = folds
    hashes = []
    for key in (0, 1, 42, lib.ref_mask_key_fold(42, 0, 0, 1), 2**64 - 1):
        for idx in list(range(8)) + [1000, 2**32 - 1, 2**32, 2**40 + 3, 2**63, 2**64 - 1]:
            hashes.append([str(key), str(idx), str(lib.ref_hash_counter(key, idx)),
                           repr(lib.ref_uniform01(key, idx))])
    kat["hash"] = hashes
    ru = []
    for key, lo, hi in ((3, -1.0, 1.0), (lib.ref_hash_counter(11, 1), -1 / 8 ** 0.5, 1 / 8 ** 0.5),
                        (lib.ref_hash_counter(11, 4), -0.1, 0.1)):
        n = 64
        buf = (dbl * n)()
        lib.ref_random_uniform(key, n, lo, hi, buf)
        ru.append({"key": str(key), "lo": repr(lo), "hi": repr(hi), "values": [repr(v) for v in buf]})
    kat["random_uniform"] = ru
    dm = []
    for seed, layer, op, mb, p in ((42, 0, 0, 1, 0.1), (7, 3, 1, 2, 0.5), (42, 0, 2, 1, 0.0)):
        n = 256
        buf = (dbl * n)()
        assert lib.ref_dropout_mask(seed, layer, op, mb, n, p, buf) == 0
        dm.append({"seed": seed, "layer": layer, "op": op, "microbatch": mb, "p": p,
                   "mask": "".join("1" if v == 1.0 else "0" for v in buf)})
    kat["dropout_mask"] = dm
    buf = (dbl * 4)()
    kat["dropout_mask_rejects"] = [lib.ref_dropout_mask(1, 0, 0, 0, 4, p, buf) for p in (-0.1, 1.0, 1.5)]
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    with open(OUT, "w") as f:
        json.dump(kat, f, indent=0)
    print("wrote", OUT, file=sys.stderr)


if __name__ == "__main__":
    main()
