"""Wall time of the public mine_corpus (text in, rows out) on C2 documents
for several chunk sizes (align.CHUNK_PAIRS).

    python tools/api_probe.py [n_pairs] [chunk ...]
    API_PROFILE=1 python tools/api_probe.py ...   # + cProfile of one call
"""
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import bench  # noqa: E402
from paper_1512_01641_b200 import align as A  # noqa: E402
from paper_1512_01641_b200.classifier import load_model  # noqa: E402
from paper_1512_01641_b200.corpus import Document, DocumentPair  # noqa: E402
from paper_1512_01641_b200.lexicon import Lexicon  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
    chunks = [int(x) for x in sys.argv[2:]] or [16384, 4096, 2048, 1024]
    corpus, _ = bench.load_workload(2, n, 0)
    b = corpus.batch
    sents = corpus.all_sentences()
    pairs = [DocumentPair(f"t{p}", Document(f"s{p}", "pl", str(p), tuple(sents[b.pair_src[p]:b.pair_src[p] + b.pair_n[p]])),
                          Document(f"d{p}", "en", str(p), tuple(sents[b.pair_tgt[p]:b.pair_tgt[p] + b.pair_m[p]])))
             for p in range(b.n_pairs)]
    lex = Lexicon(corpus.dictionary.table())
    model = load_model(os.path.join(REPO, "tests", "golden", "synth_model.json"))
    A.mine_corpus(model, lex, pairs[:64], A.MiningConfig())
    for ch in chunks:
        A.CHUNK_PAIRS = ch
        best, st = 1e9, None
        for _ in range(3):
            A.STAGE_TIMES = {}
            t = time.perf_counter()
            out = A.mine_corpus(model, lex, pairs, A.MiningConfig())
            w = time.perf_counter() - t
            if w < best:
                best, st = w, A.STAGE_TIMES
        A.STAGE_TIMES = None
        stages = " ".join(f"{k} {v * 1e3:.1f}" for k, v in st.items())
        print(f"chunk {ch}: {best:.3f} s = {n / best:.0f} pairs/s, {len(out.rows)} rows; stages ms: {stages}",
              flush=True)
    if os.environ.get("API_PROFILE"):
        import cProfile
        import pstats

        pr = cProfile.Profile()
        pr.enable()
        A.mine_corpus(model, lex, pairs, A.MiningConfig())
        pr.disable()
        pstats.Stats(pr).sort_stats("tottime").print_stats(18)


if __name__ == "__main__":
    main()
