"""Convenience owner of the per-model state around the C ABI: the prepared
codebook terms (n_j, c^_j), zero-initialised workspaces, the code array and the running
code histogram.  Every method is a single call (or a short sequence of calls)
into liba2ats.so; no arithmetic of the method happens here."""
from __future__ import annotations

import torch

from . import binding as _b


class Decoder:
    def __init__(self, B, Hq, Hkv, L, n_max, codebook, H=None, params: _b.Params | None = None, device="cuda",
                 stream=None, code_bytes=2):
        self.device = torch.device(device)
        self.shape = _b.make_shape(B, Hq, Hkv, 128, L, n_max, code_bytes)
        self.params = params or _b.Params()
        self.stream = stream
        self.codebook = codebook.contiguous()
        self.H = None if H is None else H.contiguous().float()
        self.nrm = torch.empty((Hkv, L), dtype=torch.float32, device=self.device)
        self.chat = torch.empty((Hkv, L, 256), dtype=torch.bfloat16, device=self.device)
        _b.a2ats_qavq_prepare(self.shape, self.codebook, self.H, self.nrm, self.chat, stream)
        self.ws_enc = torch.zeros(_b.a2ats_build_codes_workspace_bytes(self.shape), dtype=torch.uint8,
                                  device=self.device)
        self.ws_dec = torch.zeros(_b.a2ats_decode_workspace_bytes(self.shape, self.params), dtype=torch.uint8,
                                  device=self.device)
        self.codes = torch.zeros((B, Hkv, n_max), dtype=torch.uint8 if code_bytes == 1 else torch.uint16,
                                 device=self.device)
        self.hist = torch.zeros((B, Hkv, L), dtype=torch.int32, device=self.device)

    def set_topk(self, k: int):
        self.params.topk = int(k)
        need = _b.a2ats_decode_workspace_bytes(self.shape, self.params)
        if need > self.ws_dec.numel():
            self.ws_dec = torch.zeros(need, dtype=torch.uint8, device=self.device)
        # (the zero-on-entry counters sit at shape-only offsets at the front of the workspace,
        # so a smaller topk on the same workspace finds them where the kernels left them)

    def encode(self, keys, t_begin: int, t_end: int, update_hist: bool = True, codes=None):
        _b.a2ats_build_codes(self.shape, keys, t_begin, t_end, self.chat, self.nrm,
                             self.codes if codes is None else codes, self.hist if update_hist else None,
                             self.ws_enc, self.stream)

    def step(self, q, k_cache, v_cache, n_ctx: int, out=None, sel_out=None, scores_out=None, use_hist=True,
             codes=None, kv_host=False):
        if out is None:
            out = torch.empty((self.shape.B, self.shape.Hq, 128), dtype=torch.float32, device=self.device)
        _b.a2ats_decode_step(self.shape, self.params, n_ctx, q, k_cache, v_cache,
                             self.codes if codes is None else codes, self.codebook,
                             self.hist if use_hist else None, out, sel_out, scores_out, self.ws_dec, self.stream,
                             kv_host=kv_host)
        return out

    def select(self, q, n_ctx: int, sel_out, use_hist=True):
        """a1..a4 only: the top-K token indices (no K/V read, no attention)."""
        _b.a2ats_select_topk(self.shape, self.params, n_ctx, q, self.codes, self.codebook,
                             self.hist if use_hist else None, sel_out, self.ws_dec, self.stream)
        return sel_out

    def build_postings(self, n_tokens: int):
        """Inverted index of tokens [0, n_tokens) (f3 posting-list selection)."""
        if getattr(self, "postings", None) is None:
            self.postings = torch.zeros(_b.a2ats_postings_bytes(self.shape), dtype=torch.uint8, device=self.device)
        _b.a2ats_postings_build(self.shape, self.codes, n_tokens, self.postings, self.stream)
        self.n_post = int(n_tokens)

    def select_postings(self, q, n_ctx: int, sel_out):
        _b.a2ats_select_topk_postings(self.shape, self.params, n_ctx, q, self.codes, self.codebook, self.hist,
                                      self.postings, self.n_post, sel_out, self.ws_dec, self.stream)
        return sel_out

    def step_postings(self, q, k_cache, v_cache, n_ctx: int, out=None, sel_out=None):
        if out is None:
            out = torch.empty((self.shape.B, self.shape.Hq, 128), dtype=torch.float32, device=self.device)
        _b.a2ats_decode_step_postings(self.shape, self.params, n_ctx, q, k_cache, v_cache, self.codes, self.codebook,
                                      self.hist, self.postings, self.n_post, out, sel_out, self.ws_dec, self.stream)
        return out

    def step_append_postings(self, q, k_cache, v_cache, n_ctx: int, out=None, sel_out=None):
        """a0 for token n_ctx - 1 fused with the step, selection over the posting lists (f3)."""
        if out is None:
            out = torch.empty((self.shape.B, self.shape.Hq, 128), dtype=torch.float32, device=self.device)
        _b.a2ats_decode_step_append_postings(self.shape, self.params, n_ctx, q, k_cache, v_cache, self.codes,
                                             self.codebook, self.hist, self.chat, self.nrm, self.postings,
                                             self.n_post, out, sel_out, self.ws_dec, self.stream)
        return out

    def step_append(self, q, k_cache, v_cache, n_ctx: int, out=None, sel_out=None, scores_out=None,
                    use_hist=True):
        """a0 for token n_ctx - 1 (its key already in k_cache) fused with the step."""
        if out is None:
            out = torch.empty((self.shape.B, self.shape.Hq, 128), dtype=torch.float32, device=self.device)
        _b.a2ats_decode_step_append(self.shape, self.params, n_ctx, q, k_cache, v_cache, self.codes, self.codebook,
                                    self.hist if use_hist else None, self.chat, self.nrm, out, sel_out, scores_out,
                                    self.ws_dec, self.stream)
        return out

    # ------------------------------------------------------------------ serving loop
    def start(self, keys, n_ctx: int, engine: str = "auto", rebuild_every: int = 1024):
        """Prefill: encode tokens [0, n_ctx) (a0, running histogram) and pick the selection engine
        for the decode loop: posting lists (f3) where the code scan would need its long-context
        kernels, the code scan otherwise ("auto"), or as given.  Then call decode() per step."""
        self.encode(keys, 0, n_ctx)
        self._n_enc = int(n_ctx)
        if engine == "auto":
            engine = "postings" if n_ctx - self.params.window > 2 * 32768 and self.shape.L <= 4096 else "scan"
        self._engine = engine
        self._every = int(rebuild_every)
        if engine == "postings":
            self.build_postings(max(0, n_ctx - self.params.window))

    def decode(self, q, k_cache, v_cache, n_ctx: int, out=None, sel_out=None):
        """One decode step for a context of n_ctx tokens (token n_ctx - 1's K/V row already in the
        caches) with the library's maintenance policy: a0 batched -- the newest tokens are encoded
        in one a2ats_build_codes call when the oldest unencoded one would leave the window
        (params.hist_lag covers the rest; reading Q34) -- and, with posting lists, the index rebuilt
        every `rebuild_every` steps (reading Q33).  Results equal a2ats_decode_step_append's (the
        same top-K sets; with posting lists the rows are summed in index order)."""
        w = self.params.window
        if n_ctx - self._n_enc > w:          # the oldest unencoded token would become a candidate
            self.encode(k_cache, self._n_enc, n_ctx - 1)
            self._n_enc = n_ctx - 1
        self.params.hist_lag = n_ctx - self._n_enc
        try:
            if self._engine == "postings":
                if n_ctx - w - self.n_post > self._every:
                    self.build_postings(n_ctx - w)
                return self.step_postings(q, k_cache, v_cache, n_ctx, out=out, sel_out=sel_out)
            return self.step(q, k_cache, v_cache, n_ctx, out=out, sel_out=sel_out)
        finally:
            self.params.hist_lag = 0
