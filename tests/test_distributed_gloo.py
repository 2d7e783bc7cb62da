"""World-size-2 test of the sharded mining path over gloo (CPU).

Each rank mines its cell-balanced contiguous shard; rank 0 gathers in
rank order.  The per-shard compute is injected (the CPU oracle stands in
for the GPU, which this container lacks); what is under test is the
host-side sharding and the order-preserving gather, which must give
exactly the single-process result.
"""

import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _oracle_mine(model, lexicon, pairs, config, engine):
    """mine_corpus semantics on the CPU oracle (test stand-in)."""
    sys.path[:0] = [REPO, os.path.join(REPO, "oracle"), os.path.join(REPO, "tests")]
    import oracle
    from paper_1512_01641_b200.align import MiningOutcome
    from paper_1512_01641_b200.classifier import model_vector
    from paper_1512_01641_b200.packing import BatchBuilder, Vocabulary, lexicon_arrays

    vocab = Vocabulary()
    coo = lexicon_arrays(lexicon.items(), vocab)
    builder = BatchBuilder(vocab)
    ok, failures = [], []
    for k, p in enumerate(pairs):
        try:
            builder.add_pair(p.source.sentences, p.target.sentences)
            ok.append(k)
        except ValueError as exc:
            failures.append((p.topic_id, f"pair {p.topic_id}: {exc}"))
    rows = []
    if ok:
        batch = builder.build()
        _, per_pair = oracle.mine_batch(oracle.OracleDict(*coo), model_vector(model), batch, config.gap_penalty,
                                        config.threshold, config.mismatch_cost, config.match_bonus)
        for b, k in enumerate(ok):
            src, tgt = pairs[k].source.sentences, pairs[k].target.sentences
            rows.extend((float(r["score"]), src[int(r["i"])], tgt[int(r["j"])]) for r in per_pair[b])
    return MiningOutcome(rows=tuple(rows), failures=tuple(failures))


def _pairs():
    import helpers as H
    from paper_1512_01641_b200.corpus import Document, DocumentPair

    out = []
    for p in H.load_json("toy.json")["pairs"]:
        out.append(DocumentPair(p["topic_id"], Document("s", "eo", "t", tuple(p["source"])),
                                Document("t", "en", "t", tuple(p["target"]))))
    out.insert(3, DocumentPair("bad", Document("b1", "eo", "bad", ("...",)), Document("b2", "en", "bad", ("house",))))
    return out


def _worker(rank, world, port, q):
    sys.path[:0] = [REPO, os.path.join(REPO, "oracle"), os.path.join(REPO, "tests")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    import helpers as H
    from paper_1512_01641_b200.align import MiningConfig
    from paper_1512_01641_b200.distributed import mine_corpus_distributed

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = mine_corpus_distributed(H.toy_model(), H.toy_lexicon(), _pairs(), MiningConfig(), mine_fn=_oracle_mine)
        if rank == 0:
            q.put((out.rows, out.failures))
    finally:
        dist.destroy_process_group()


def test_sharded_mining_equals_single_process():
    sys.path[:0] = [REPO, os.path.join(REPO, "oracle"), os.path.join(REPO, "tests")]
    import helpers as H
    import oracle
    from paper_1512_01641_b200.align import MiningConfig

    oracle.build()
    want = _oracle_mine(H.toy_model(), H.toy_lexicon(), _pairs(), MiningConfig(), "nw")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    rows, failures = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert rows == want.rows
    assert failures == want.failures
    assert len(failures) == 1 and failures[0][0] == "bad"


def test_shard_range_partitions():
    from paper_1512_01641_b200.distributed import shard_range

    w = np.array([2500, 2400, 100, 3000, 2500, 10, 10], dtype=np.int64)
    for world in (1, 2, 3, 4, 8):
        ranges = [shard_range(w, r, world) for r in range(world)]
        assert ranges[0][0] == 0 and ranges[-1][1] == len(w)
        assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
