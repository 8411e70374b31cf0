"""One process per GPU (torchrun): database sharded by residue count, per-shard top-k merged with one
all-gather of k packed 64-bit keys per rank (NCCL over NVLink on GPUs; gloo in the CPU tests).

The data path has no other collective: every (query, subject) score is independent
(align.hpp:80-82) and the (score desc, index asc) order is a strict total order
(scheduler.hpp:111-114), so top-k of the union == top-k of the per-shard top-k's.

A sharded search touches the host once: the library enqueues the shard's search on torch's current stream and
leaves its k keys in a preallocated CUDA tensor (swb_search_keys_device), the all-gather runs on that tensor, the
library selects the global top-k from the gathered tensor on the same stream (swb_db_merge_keys) and copies k hits
down -- the one device-to-host copy and the one synchronisation of the search.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def exchange_keys(local_keys: np.ndarray, device: torch.device | None = None, group=None) -> np.ndarray:
    """All-gather this rank's top_k packed keys (zero padded to a common length), host in, host out: the flavour for
    keys that are already on the host (the batched sweep's n_queries x k block; the CPU tests).

    Returns the concatenation over ranks, shape (world * k,).  uint64 keys travel as int64 bit
    patterns (NCCL/gloo have no uint64 tensor type in torch)."""
    world = dist.get_world_size(group)
    send = torch.from_numpy(np.ascontiguousarray(local_keys, dtype=np.uint64).view(np.int64).copy())
    if device is not None and device.type == "cuda":
        send = send.to(device, non_blocking=True)
    recv = torch.empty(world * send.numel(), dtype=torch.int64, device=send.device)
    dist.all_gather_into_tensor(recv, send, group=group)
    return recv.cpu().numpy().view(np.uint64)


def merge_many(gathered: np.ndarray, world: int, n_queries: int, top_k: int):
    """`gathered` = the ranks' (n_queries x top_k) key blocks, concatenated rank by rank.  -> per query the merged
    (db_index, score) list: descending key order is (score desc, index asc) (scheduler.hpp:111-114), 0 pads."""
    from .search import decode_keys
    blocks = np.asarray(gathered, dtype=np.uint64).reshape(world, n_queries, top_k)
    out = []
    for q in range(n_queries):
        keys = blocks[:, q, :].reshape(-1)
        keys = np.sort(keys[keys != 0])[::-1][:top_k]
        out.append(decode_keys(keys))
    return out


class ShardedSearch:
    """This rank's shard of the database plus the cross-rank merge.

    device_path: route every search through the device-tensor path (keys stay on the GPU between the shard's select,
    the all-gather and the global select) even when world == 1, where search() would otherwise call swb_search
    directly -- what the one-GPU test of that path uses."""

    def __init__(self, codes, offsets, length_threshold: int = 3000, device_index: int = 0, group=None, device_path: bool = False):
        from .search import Database
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.device_index = device_index
        self.device_path = device_path
        self.db = Database(codes, offsets, length_threshold=length_threshold, device=device_index,
                           shard_rank=self.rank, shard_count=self.world)
        self._send = self._recv = None   # CUDA int64 tensors of k and world x k keys, reused across searches

    def _buffers(self, top_k: int):
        if self._send is None or self._send.numel() != top_k:
            device = torch.device("cuda", self.device_index)
            self._send = torch.zeros(top_k, dtype=torch.int64, device=device)
            self._recv = torch.zeros(self.world * top_k, dtype=torch.int64, device=device)
        return self._send, self._recv

    def search(self, query, matrix, gaps, top_k: int = 10):
        """-> (db_index, score, local stats).  Every rank returns the same global list."""
        if self.world == 1 and not self.device_path:
            return self.db.search(query, matrix, gaps, top_k)
        # the library's stream must be the one the collective orders itself against: torch's current stream
        stream = torch.cuda.current_stream(torch.device("cuda", self.device_index))
        self.db.set_stream(stream.cuda_stream)
        send, recv = self._buffers(top_k)
        self.db.search_keys_device(query, matrix, gaps, top_k, send.data_ptr())
        if dist.is_initialized():     # also with world = 1: the same collective on the same stream
            dist.all_gather_into_tensor(recv, send, group=self.group)
        else:
            recv = send
        return self.db.merge_keys_device(recv.data_ptr(), recv.numel(), top_k, len(query))

    def search_many(self, queries, matrix, gaps, top_k: int = 10):
        """A batch of queries (swb_search_many on this rank's shard: shared scans where they apply), then ONE
        all-gather of n_queries x top_k keys per rank instead of one per query.  -> list of (db_index, score),
        identical on every rank, and this rank's per-query device ms."""
        from .search import encode_keys
        local, ms = self.db.search_many(queries, matrix, gaps, top_k)
        if self.world == 1:
            return local, ms
        keys = np.zeros((len(queries), top_k), dtype=np.uint64)
        for q, (idx, sc) in enumerate(local):
            keys[q, :len(idx)] = encode_keys(idx, sc)
        gathered = exchange_keys(keys.reshape(-1), torch.device("cuda", self.device_index), self.group)
        return merge_many(gathered, self.world, len(queries), top_k), ms

    def close(self):
        self.db.close()
