"""Host-resident batches through the GPU with copy/compute overlap.

A batch that lives in (pinned) host memory is split into `chunks` slices along the batch axis.
Per slice: host->device copy on a copy stream, the compute (any function of device tensors that
launches this package's kernels on the current stream) once its inputs have arrived, and the
device->host copy of its result on a second copy stream.  The copy of slice k+1 overlaps the
compute of slice k, and the read-back of slice k overlaps both, so a step costs about
max(H2D, compute, D2H) plus one slice of the others instead of their sum.  Orchestration only:
every byte of arithmetic runs in the kernels `fn` launches.

Timing contract: `run` makes the copy streams wait for the caller's current stream first and
makes the caller's stream wait for the last read-back, so CUDA events recorded on the caller's
stream around `run` bracket the whole transfer.
"""
from __future__ import annotations

from typing import Callable, Sequence

import torch


class HostPipeline:
    """Reusable device buffers, streams and events for one batch shape.

    host_inputs: pinned host tensors whose leading dimension is the batch; host_output: the pinned
    host tensor that receives fn's result (leading dimension = batch).  fn(*device_inputs) must
    return a device tensor shaped like the slice of host_output."""

    def __init__(self, host_inputs: Sequence[torch.Tensor], host_output: torch.Tensor, chunks: int = 4,
                 device=None):
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        B = host_inputs[0].shape[0]
        if any(t.shape[0] != B for t in host_inputs) or host_output.shape[0] != B:
            raise ValueError("all host tensors must share the leading (batch) dimension")
        if not all(t.is_pinned() for t in (*host_inputs, host_output)):
            raise ValueError("host tensors must be pinned (torch.Tensor.pin_memory())")
        self.chunks = max(1, min(int(chunks), B))
        step = -(-B // self.chunks)
        self.bounds = [(a, min(a + step, B)) for a in range(0, B, step)]
        self.host_inputs = list(host_inputs)
        self.host_output = host_output
        self.dev_inputs = [torch.empty(t.shape, dtype=t.dtype, device=self.device) for t in host_inputs]
        self.h2d = torch.cuda.Stream(self.device)
        self.d2h = torch.cuda.Stream(self.device)
        n = len(self.bounds)
        self.ev_in = [torch.cuda.Event() for _ in range(n)]
        self.ev_done = [torch.cuda.Event() for _ in range(n)]
        self._started = False

    def run(self, fn: Callable[..., torch.Tensor]) -> torch.Tensor:
        """One pass over the batch; returns host_output (valid once the caller's stream is done)."""
        cs = torch.cuda.current_stream(self.device)
        self.h2d.wait_stream(cs)
        self.d2h.wait_stream(cs)
        for k, (a, b) in enumerate(self.bounds):
            with torch.cuda.stream(self.h2d):
                if self._started:
                    # the previous pass's compute on this slice must be done before it is overwritten
                    self.h2d.wait_event(self.ev_done[k])
                for h, d in zip(self.host_inputs, self.dev_inputs):
                    d[a:b].copy_(h[a:b], non_blocking=True)
                self.ev_in[k].record(self.h2d)
        self._started = True
        for k, (a, b) in enumerate(self.bounds):
            cs.wait_event(self.ev_in[k])
            res = fn(*(d[a:b] for d in self.dev_inputs))
            self.ev_done[k].record(cs)
            with torch.cuda.stream(self.d2h):
                self.d2h.wait_event(self.ev_done[k])
                res.record_stream(self.d2h)
                self.host_output[a:b].copy_(res, non_blocking=True)
        cs.wait_stream(self.d2h)
        return self.host_output
