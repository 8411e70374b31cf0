"""Runs the GPU tests in a process whose free device memory was first filled with a byte pattern, so that every
buffer the library allocates starts out dirty (a fresh box hands out memory of unknown content; a reused one tends
to hand back the library's own, friendlier, leftovers).  A test that passes only on clean memory reads something
before writing it.

    gpurun -- 'python tests/manual/dirty_memory_tests.py 0xFF [pytest args]'
"""
import sys

sys.path.insert(0, ".")
import pytest
import torch


def main():
    pattern = int(sys.argv[1], 0) if len(sys.argv) > 1 else 0xFF
    args = sys.argv[2:] or ["tests", "-m", "gpu", "-q"]
    free, _ = torch.cuda.mem_get_info()
    n = int(free * 0.9)
    junk = torch.empty(n, dtype=torch.uint8, device="cuda")
    junk.fill_(pattern)
    torch.cuda.synchronize()
    del junk
    torch.cuda.empty_cache()
    print(f"filled {n >> 20} MiB with 0x{pattern:02X}", flush=True)
    return pytest.main(args)


if __name__ == "__main__":
    sys.exit(main())
