"""Host <-> device staging for pipelined layer steps.

A training loop that feeds the MoE layer from host memory (the reference's
API takes and returns host arrays) pays four PCIe copies per step: tokens and
upstream gradients in, outputs and input gradients out.  ``HostStager`` puts
them on two copy streams so they overlap compute: the upstream gradient is
uploaded while the forward runs, outputs download while the backward runs,
the next step's tokens upload during this step's backward and the input
gradient downloads during the next forward.  ``drain()`` waits for every
outstanding copy.
"""
from __future__ import annotations

import torch


class HostStager:
    def __init__(self, device):
        self.device = torch.device(device)
        self.h2d = torch.cuda.Stream(self.device)
        self.d2h = torch.cuda.Stream(self.device)

    def upload(self, host: torch.Tensor, dev: torch.Tensor) -> torch.cuda.Event:
        """Async host->device copy on the H2D stream (host must be pinned)."""
        # the device buffer may still be read by earlier compute
        self.h2d.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(self.h2d):
            dev.copy_(host, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(self.h2d)
        return ev

    def download(self, dev: torch.Tensor, host: torch.Tensor) -> torch.cuda.Event:
        """Async device->host copy on the D2H stream, after the compute that
        produced ``dev`` (host must be pinned)."""
        ready = torch.cuda.Event()
        ready.record(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(self.d2h):
            self.d2h.wait_event(ready)
            host.copy_(dev, non_blocking=True)
            dev.record_stream(self.d2h)
            ev = torch.cuda.Event()
            ev.record(self.d2h)
        return ev

    @staticmethod
    def consume(ev: torch.cuda.Event) -> None:
        """Make the current (compute) stream wait for a staged copy."""
        torch.cuda.current_stream().wait_event(ev)

    def drain(self) -> None:
        self.h2d.synchronize()
        self.d2h.synchronize()
