"""Time build_lexicon on synthetic sentence pairs.

    python tools/bench_lexicon.py [n_docs] [iterations]        # GPU path (this package)
    python tools/bench_lexicon.py [n_docs] [iterations] --ref  # the reference (build container only)

The corpus: the generator's true translation pairs of n_docs C2-shaped
document pairs (~30 sentence pairs each), 1000-word dictionary."""
import sys
import time

sys.path[:0] = ["."]
import numpy as np

from paper_1512_01641_b200 import synth


def corpus(n_docs):
    d = synth.make_dictionary(np.random.default_rng(77), 1000)
    c = synth.make_corpus(78, n_docs, 1000, dictionary=d)
    par = []
    for p in range(n_docs):
        src, tgt = c.pair_sentences(p)
        par += [(src[i], tgt[j]) for i, j in c.reference[p]]
    return par


def main():
    n_docs = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    par = corpus(n_docs)
    if "--ref" in sys.argv:
        sys.path.insert(0, "/root/reference/pkg/src")
        from bimine.lexicon import build_lexicon
    else:
        from paper_1512_01641_b200.lexicon import build_lexicon
        build_lexicon(par[:50], 1)  # warm-up (library load, CUDA context)
    t = time.perf_counter()
    lex = build_lexicon(par, iters)
    dt = time.perf_counter() - t
    print(f"{'reference' if '--ref' in sys.argv else 'b200'}: {len(par)} sentence pairs, {iters} rounds, "
          f"{len(lex)} entries in {dt:.3f} s")


if __name__ == "__main__":
    main()
