"""Decoder rows over the C ABI: a rank-space KV cache per
layer, causal prefill and single-token decode steps.

Torch is plumbing only (device buffers and the current stream); every
computation runs in libfsvd_b200.so.  Causal semantics: layer by layer, the
output at position i equals the encoder layer (flash_svd_attention /
run_layer, attention.cpp:202-269, encoder.cpp:224-257) applied to the prefix
[0, i] of that layer's inputs, at its last row; the cache holds the rank-space keys/values 2 * layers * B * M * r the
reference's planner sizes (planner.cpp:123-127).
"""
from __future__ import annotations

import ctypes as C

from . import abi
from .model import layer_descs


class Decoder:
    def __init__(self, layers, batch: int, max_seq: int, pre_ln: bool = False,
                 graph: bool = False):
        import torch
        self.L = abi.lib()
        self.batch, self.max_seq, self.pre_ln = batch, max_seq, bool(pre_ln)
        self.d = layers[0].d_model
        descs = layer_descs(layers)
        self.packs = []
        for i in range(len(layers)):
            p = C.c_void_p()
            abi.check(self.L.fsvd_layer_pack_create(C.byref(descs[i]), abi.BF16, 0, C.byref(p)))
            self.packs.append(p)
        self.parr = (C.c_void_p * len(self.packs))(*[p.value for p in self.packs])
        # one cache per layer, each sized by its own pack (layers may differ in
        # groups or rank padding, so a cache sized by layer 0 could be short)
        self.caches = []
        for p in self.packs:
            cb = abi._sz()
            abi.check(self.L.fsvd_kv_cache_bytes(p, batch, max_seq, C.byref(cb)))
            self.caches.append(torch.zeros(cb.value, dtype=torch.uint8, device="cuda"))
        self.carr = (C.c_void_p * len(layers))(*[c.data_ptr() for c in self.caches])
        wb = abi._sz()
        abi.check(self.L.fsvd_decoder_workspace_bytes(self.parr, len(self.packs), batch, max_seq,
                                                      int(self.pre_ln), C.byref(wb)))
        self.ws = torch.empty(wb.value, dtype=torch.uint8, device="cuda")
        self.pos = 0
        # graph mode: the step runs on fixed token buffers, captured once
        self.graph = None
        if graph:
            self.xbuf = torch.zeros((batch, self.d), dtype=torch.bfloat16, device="cuda")
            self.obuf = torch.zeros((batch, self.d), dtype=torch.bfloat16, device="cuda")
            g = C.c_void_p()
            abi.check(self.L.fsvd_decoder_graph_create(
                self.parr, len(self.packs), int(self.pre_ln), batch,
                C.c_void_p(self.xbuf.data_ptr()), C.c_void_p(self.obuf.data_ptr()), self.carr,
                max_seq, C.c_void_p(self.ws.data_ptr()), self.ws.numel(), C.byref(g)))
            self.graph = g

    def _stream(self):
        import torch
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)

    def prefill(self, x):
        """x [batch, seq, d] bf16 on the device -> causal outputs; fills the caches."""
        import torch
        assert x.dtype == torch.bfloat16 and x.is_contiguous()
        out = torch.empty_like(x)
        abi.check(self.L.fsvd_decoder_prefill(
            self.parr, len(self.packs), int(self.pre_ln), self.batch, x.shape[1],
            C.c_void_p(x.data_ptr()), C.c_void_p(out.data_ptr()), self.carr, self.max_seq,
            C.c_void_p(self.ws.data_ptr()), self.ws.numel(), self._stream()))
        self.pos = x.shape[1]
        return out

    def step(self, x_t):
        """x_t [batch, d] bf16: the token at position self.pos -> its output."""
        import torch
        assert x_t.dtype == torch.bfloat16 and x_t.is_contiguous()
        if self.graph is not None:
            self.xbuf.copy_(x_t)
            abi.check(self.L.fsvd_decoder_graph_step(self.graph, self.pos, self._stream()))
            self.pos += 1
            return self.obuf.clone()
        out = torch.empty_like(x_t)
        abi.check(self.L.fsvd_decoder_step(
            self.parr, len(self.packs), int(self.pre_ln), self.batch, self.pos,
            C.c_void_p(x_t.data_ptr()), C.c_void_p(out.data_ptr()), self.carr, self.max_seq,
            C.c_void_p(self.ws.data_ptr()), self.ws.numel(), self._stream()))
        self.pos += 1
        return out

    def close(self):
        if self.graph is not None:
            self.L.fsvd_decoder_graph_destroy(self.graph)
            self.graph = None
        for p in self.packs:
            self.L.fsvd_layer_pack_destroy(p)
        self.packs = []
