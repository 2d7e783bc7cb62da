"""Time the public mine_corpus (text in, rows out) on C2-shaped documents."""
import sys
import time

sys.path[:0] = ["."]

import bench
from paper_1512_01641_b200 import align as A
from paper_1512_01641_b200.classifier import load_model
from paper_1512_01641_b200.corpus import Document, DocumentPair
from paper_1512_01641_b200.lexicon import Lexicon

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
corpus, _ = bench.load_workload(2, n, 0)
model = load_model("tests/golden/synth_model.json")
t = time.perf_counter()
pairs = []
for p in range(n):
    src, tgt = corpus.pair_sentences(p)
    pairs.append(DocumentPair(topic_id=f"t{p}", source=Document(id=f"s{p}", lang="pl", title="", sentences=tuple(src)),
                              target=Document(id=f"d{p}", lang="en", title="", sentences=tuple(tgt))))
lex = Lexicon(corpus.dictionary.table())
print(f"setup {time.perf_counter() - t:.1f} s ({n} pairs, {len(lex)} lexicon entries)")
cfg = A.MiningConfig()
A.mine_corpus(model, lex, pairs[:50], cfg)  # warm: lexicon upload, library, CUDA context
for _ in range(2):
    t = time.perf_counter()
    out = A.mine_corpus(model, lex, pairs, cfg)
    print(f"mine_corpus: {time.perf_counter() - t:.2f} s, {len(out.rows)} rows, {len(out.failures)} failures")
