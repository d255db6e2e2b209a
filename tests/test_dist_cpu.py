"""World-size-2 gloo tests of the multi-rank host path (CPU only).

What the N > 1 path relies on, checked with two real processes:
  * the point shards partition the image exactly (concatenation = input, balanced);
  * votes are sums over points: per-rank region votes (oracle, the method's definition) summed with
    an allreduce equal the whole-image votes for every visited region -- the property that lets
    libhht allreduce per-level vote vectors and take identical split decisions on every rank;
  * local list lengths (pre-allreduce votes) sum to the global ones;
  * image sharding of a batch partitions the images, offsets are rebased;
  * the NCCL unique id broadcast delivers identical bytes; argument mismatch is detected;
  * max-over-ranks timing.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_1007_0547_b200 import dist as hd
        from paper_1007_0547_b200 import synth
        out = {}
        # 1. point sharding of one image + votes additivity over ranks
        N, D, T = 32, 4, 3
        pts = synth.random_scene(42, N, max_lines=3, max_noise=150)
        sh = hd.make_shard(pts, [0, len(pts)], rank, world)
        assert sh.mode == "points" and sh.comm_world == world
        n_local = torch.tensor([sh.points.shape[0]])
        gathered = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(gathered, n_local)
        sizes = [int(g.item()) for g in gathered]
        assert sum(sizes) == len(pts) and max(sizes) - min(sizes) <= 1
        full = oracle.detect(pts, N, D, T, 3)
        for half in (1, 2):
            for lev in range(D + 1):
                recs = full.levels[(half, lev)]
                if recs.shape[0] == 0:
                    continue
                local = np.array([oracle.region_votes(sh.points, half, N, D, lev, int(a), int(c))
                                  for a, c, _ in recs.tolist()], dtype=np.int64)
                t = torch.from_numpy(local)
                dist.all_reduce(t)                          # the per-level vote allreduce
                assert np.array_equal(t.numpy(), recs[:, 2].astype(np.int64)), (half, lev)
        out["additivity"] = True
        # 2. image sharding of a batch
        imgs = [synth.random_scene(100 + b, 16, max_noise=20) for b in range(5)]
        offs = np.zeros(6, dtype=np.int64)
        offs[1:] = np.cumsum([len(p) for p in imgs])
        allp = np.concatenate(imgs).astype(np.int32)
        sb = hd.make_shard(allp, offs, rank, world)
        assert sb.mode == "images" and sb.comm_world == 1 and sb.offsets[0] == 0
        nb = torch.tensor([sb.offsets.shape[0] - 1])
        dist.all_reduce(nb)
        assert int(nb.item()) == 5
        for k in range(sb.offsets.shape[0] - 1):
            got = sb.points[sb.offsets[k]:sb.offsets[k + 1]]
            assert np.array_equal(got, imgs[sb.image_lo + k])
        # 3. unique-id broadcast, argument check, timing reduction
        fake_id = bytes(range(128)) if rank == 0 else None
        assert hd.broadcast_bytes(fake_id) == bytes(range(128))
        hd.check_consistent(N, D, T, 3, 1)
        try:
            hd.check_consistent(N, D + rank, T, 3, 1)
            out["mismatch_detected"] = False
        except ValueError:
            out["mismatch_detected"] = True
        assert hd.max_over_ranks(float(rank + 1)) == float(world)
        assert hd.sum_over_ranks(1.0) == float(world)
        q.put((rank, out))
    except Exception as e:  # noqa: BLE001
        q.put((rank, {"error": repr(e)}))
        raise
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_host_path():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert "error" not in res[r], res[r]
        assert res[r]["additivity"] and res[r]["mismatch_detected"]


def test_single_rank_batch_keeps_image_offsets():
    """One rank, a batch of images: the shard is the whole batch with its own offsets (each image
    its own trees), never the images concatenated into one point set."""
    from paper_1007_0547_b200 import dist as hd, synth
    imgs = [synth.random_scene(200 + b, 16, max_noise=20) for b in range(4)]
    offs = np.zeros(5, dtype=np.int64)
    offs[1:] = np.cumsum([len(p) for p in imgs])
    allp = np.concatenate(imgs).astype(np.int32)
    sb = hd.make_shard(allp, offs, 0, 1)
    assert sb.mode == "images" and sb.comm_world == 1 and sb.image_lo == 0
    assert np.array_equal(sb.offsets, offs) and np.array_equal(sb.points, allp)
    single = hd.make_shard(imgs[0], [0, len(imgs[0])], 0, 1)
    assert single.mode == "points" and np.array_equal(single.offsets, [0, len(imgs[0])])
