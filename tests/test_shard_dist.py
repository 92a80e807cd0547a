"""CPU, world_size 2 (gloo): the multi-rank path of bench.py / shard.py.
Each rank computes its cyclic row bands (with the oracle standing in for the
device), ranks all-gather, and the assembled image must equal the single-rank
image and reproduce the reference's run_mandelbrot checksum."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def worker(rank, world, port, size, it, band, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch

    import paper_1505_07368_b200 as pkg
    from oracle import oracle
    from paper_1505_07368_b200.shard import band_tiles, cyclic_bands
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    full = pkg.reference_desc(size, it)
    local = band_tiles(full, world, rank, band, global_offsets=False)
    glob = band_tiles(full, world, rank, band, global_offsets=True)
    parts = []
    for t in local:
        parts.append(oracle.tile(t.x0, t.x1, t.y0, t.y1, t.width, t.height, t.max_iter,
                                 fp64=True, centre=False, row0=t.row0, nrows=t.nrows).ravel())
    mine = np.concatenate(parts) if parts else np.zeros(0, np.uint32)
    n = torch.tensor([mine.size])
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, n)
    maxn = int(max(s.item() for s in sizes))
    buf = torch.zeros(maxn, dtype=torch.int64)
    buf[:mine.size] = torch.from_numpy(mine.astype(np.int64))
    gathered = [torch.zeros(maxn, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(gathered, buf)
    # every rank places every rank's bands by their global offsets
    img = np.full(size * size, 0xFFFFFFFF, dtype=np.uint64)
    for r in range(world):
        off = 0
        for t in band_tiles(full, world, r, band, global_offsets=True):
            k = t.nrows * t.ncols
            img[t.out_offset:t.out_offset + k] = gathered[r][off:off + k].numpy()
            off += k
    covered = sum(n for r in range(world) for _, n in cyclic_bands(size, world, r, band))
    q.put((rank, covered, oracle.fnv1a_u32(img.astype(np.uint32)),
           int((img == 0xFFFFFFFF).sum()), [t.out_offset for t in glob]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,band", [(2, 7), (2, 64), (3, 5)])
def test_cyclic_bands_reassemble_reference_checksum(golden, world, band):
    size, it = 96, 60
    want = int([g for g in golden["run_mandelbrot"] if g["size"] == size][0]["checksum"])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, size, it, band, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    for rank, covered, chk, holes, offs in res:
        assert covered == size          # every row owned by exactly one rank
        assert holes == 0
        assert chk == want              # bit-exact run_mandelbrot checksum


def test_band_tiles_offsets():
    import paper_1505_07368_b200 as pkg
    from paper_1505_07368_b200.shard import band_tiles, cyclic_bands
    d = pkg.mandel_desc(-2.0, 1.0, -1.0, 1.0, 100, 30, 10)
    rows = sorted(r for w in range(4) for r0, n in cyclic_bands(30, 4, w, 4)
                  for r in range(r0, r0 + n))
    assert rows == list(range(30))
    loc = band_tiles(d, 4, 1, 4, global_offsets=False)
    assert [t.row0 for t in loc] == [4, 20]
    assert [t.out_offset for t in loc] == [0, 400]
    glo = band_tiles(d, 4, 1, 4, global_offsets=True)
    assert [t.out_offset for t in glo] == [400, 2000]
