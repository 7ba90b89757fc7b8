"""Test-only stand-in for engine.CudaOps: the same kernel-call interface,
computed by the C oracle on CPU tensors.  Lets the multi-rank round logic
(sharding, all-gather, tally all-reduce) run under gloo without a GPU."""

from __future__ import annotations

import numpy as np
import torch

from oracle import native
from paper_2202_00517_b200.engine import Csr


class CpuOps:
    def csr(self, table, n, k, lo, hi, max_out):
        ptr, idx = native.transpose(table[:n].numpy())
        sub_ptr = ptr[lo:hi + 1] - ptr[lo]
        sub_idx = idx[ptr[lo]:ptr[hi]].astype(np.int32)
        if max_out is not None:
            max_out[0] = int(np.diff(ptr[lo:hi + 1]).max()) if hi > lo else 0
        return Csr(torch.from_numpy(sub_ptr.copy()), torch.from_numpy(sub_idx), lo, hi)

    def join(self, tabs, table, n, k, csr, max_indeg, out_rows, tally, out_kl=None, out_ucount=None, flags=None,
             bound_in=None, bound_out=None, peers=()):
        if bound_out is not None:
            bound_out.fill_(float("nan"))  # no bound: the device kernel treats NaN as unknown
        full_ptr = np.zeros(n + 1, np.int64)
        full_ptr[csr.lo:csr.hi + 1] = csr.indptr.numpy()
        rows, kl, uc, comps, changed = native.local_join(tabs, table[:n].numpy(), np.arange(csr.lo, csr.hi),
                                                         csr=(full_ptr, csr.indices.numpy()))
        out_rows.copy_(torch.from_numpy(rows))
        for t in peers:  # the fused exchange: this rank's rows into every peer's copy (shared memory here)
            t[csr.lo:csr.hi].copy_(out_rows)
        tally[0] += comps
        tally[1] += changed
        if out_kl is not None:
            out_kl.copy_(torch.from_numpy(kl))
        if out_ucount is not None:
            out_ucount.copy_(torch.from_numpy(uc))

    def fcc(self, table, n, k, samples, out_count):
        s = samples.numpy()
        out_count[0] = native.fcc_count(table[:n].numpy(), s[0], s[1], s[2])

    def sort_rows(self, tabs, rows, k, lo, hi, out_kl=None):
        full = np.zeros((tabs.n, k), np.int32)
        full[lo:hi] = rows.numpy()
        rows.copy_(torch.from_numpy(native.sort_rows(tabs, full)[lo:hi]))
