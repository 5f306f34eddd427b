"""Thin ctypes binding of the C ABI (include/rt.h, include/rt_ops.h).

Argument marshalling only: every step of the hot path runs in the CUDA
library.  There is no CPU fallback — loading fails loudly when the library is
missing, and rt_create fails without an sm_100 GPU.
"""
import ctypes as C
import os

import numpy as np

_LIB_PATH = os.environ.get("RT_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib",
                                                         "librt_b200.so")  # RT_LIB_PATH: A/B builds (tools)
_lib = None

RT_OK, RT_E_INVAL, RT_E_NOMEM, RT_E_CUDA, RT_E_NCCL, RT_E_STATE = 0, -1, -2, -3, -4, -5
RT_CLOCK_VIRTUAL, RT_CLOCK_WALL = 0, 1
RT_POLICY_PUD, RT_POLICY_FCFS, RT_POLICY_EDF = 0, 1, 2
RT_STOP_NONE, RT_STOP_EOS, RT_STOP_MAXNEW, RT_STOP_SKILL, RT_STOP_CAP = 0, 1, 2, 3, 4
RT_FLAG_NO_MODEL, RT_FLAG_KEEP_LOGITS, RT_FLAG_CAPTURE, RT_FLAG_TIMING, RT_FLAG_FORCE_EXCHANGE = 1, 2, 4, 8, 16
RT_FLAG_TRACE = 64
RT_GEMM_PATH_AUTO, RT_GEMM_PATH_SPLITK, RT_GEMM_PATH_STREAMK, RT_GEMM_PATH_PAIR, RT_GEMM_PATH_DECPAIR = 0, 1, 2, 3, 4
(RT_DUMP_TASKS, RT_DUMP_PAGE_TABLES, RT_DUMP_ROUND, RT_DUMP_LOGITS, RT_DUMP_HIDDEN, RT_DUMP_CAPTURE_Q,
 RT_DUMP_CAPTURE_O, RT_DUMP_ROWS, RT_DUMP_KV_LAYER, RT_DUMP_FREE_STACK, RT_DUMP_TASK_SLOTS,
 RT_DUMP_MERGED, RT_DUMP_TRACE, RT_DUMP_HOST_PAGE_TABLES, RT_DUMP_HOST_FREE_STACK, RT_DUMP_LAYER_X, RT_DUMP_LAYER_Q,
 RT_DUMP_LAYER_O, RT_DUMP_LAYER_XMID, RT_DUMP_LAYER_ACT, RT_DUMP_LAYER_KV) = range(1, 22)
RT_FLAG_CAPTURE_LAYERS = 128
# rt_trace_rec (include/rt.h)
TRACE_DTYPE = np.dtype([("grid", "<u8"), ("kind", "<u4"), ("smid", "<u4"), ("t_entry", "<u8"),
                        ("t_ready", "<u8"), ("t_aux", "<u8"), ("t_exit", "<u8")])
TRACE_KINDS = {1: "gemm", 2: "attn", 3: "norm", 4: "embed", 5: "sched_pre", 6: "sched_post", 7: "gather",
               8: "argmax", 9: "merge", 10: "attn_prefill", 11: "resid_reduce"}

EXPORTED = ["rt_create", "rt_destroy", "rt_submit_request", "rt_register_prefix", "rt_step", "rt_poll_segment", "rt_poll_segment_ready",
            "rt_last_round",
            "rt_sync", "rt_get_stats", "rt_reset_stats", "rt_debug_dump", "rt_last_error", "rt_version",
            "rt_op_paged_attention", "rt_op_attention_ws_bytes", "rt_op_kv_write", "rt_op_kv_read", "rt_op_kv_swap",
            "rt_op_gemm", "rt_op_lm_argmax", "rt_op_init_weights", "rt_op_priority", "rt_mark", "rt_elapsed_ms",
            "rt_nccl_unique_id", "rt_op_pack_tiled", "rt_op_gemm_tiled", "rt_set_timing",
            "rt_op_merge_candidates", "rt_op_prefill_attention"]


class RtError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"rt status {code}: {msg}")
        self.code = code


RT_SEG_SUSPEND, RT_SEG_STREAM, RT_SEG_NONE = 0, 1, 2   # rt.h segmentation modes
RT_SEG_MAX_TOKENS = 128


class rt_utility(C.Structure):
    _fields_ = [("alpha", C.c_double), ("beta", C.c_double)]


class rt_config(C.Structure):
    _fields_ = [
        ("rank", C.c_int32), ("world", C.c_int32), ("nccl_id", C.c_void_p), ("device", C.c_int32),
        ("n_layers", C.c_int32), ("d_model", C.c_int32), ("n_q_heads", C.c_int32), ("n_kv_heads", C.c_int32),
        ("head_dim", C.c_int32), ("d_ff", C.c_int32), ("vocab", C.c_int32),
        ("weight_seed", C.c_uint64), ("init_std", C.c_float),
        ("page_tokens", C.c_int32), ("max_batch", C.c_int32), ("max_tasks", C.c_int32), ("max_ctx", C.c_int32),
        ("n_pages", C.c_int32), ("kv_pool_bytes", C.c_int64), ("max_rows_per_forward", C.c_int32),
        ("max_seg_tokens", C.c_int32), ("g_us", C.c_int32), ("net_us", C.c_int32), ("eps_l_us", C.c_int32),
        ("speed_window", C.c_int32), ("max_admit_per_round", C.c_int32), ("policy", C.c_int32),
        ("clock_mode", C.c_int32), ("base_us", C.c_int32), ("gamma_ppm", C.c_int32),
        ("kv_us_per_1k", C.c_int32), ("prefill_us_per_tok", C.c_int32), ("t0_us", C.c_int64),
        ("tok_skill", C.c_void_p), ("tok_exec_min_us", C.c_void_p), ("eos_id", C.c_int32),
        ("flags", C.c_int32), ("capture_layer", C.c_int32), ("seg_mode", C.c_int32), ("wcet_off", C.c_int32),
        ("host_pages", C.c_int32), ("swap_us_per_page", C.c_int32),
        ("stop_grammar", C.c_int32), ("tok_class", C.c_void_p), ("skill_base_us", C.c_void_p),
        ("skill_unit_us", C.c_void_p), ("word_us", C.c_int32), ("gemm_path", C.c_int32),
    ]


class rt_segment(C.Structure):
    _fields_ = [("request_id", C.c_int64), ("agent_id", C.c_int32), ("k", C.c_int32),
                ("tok_begin", C.c_int32), ("tok_end", C.c_int32), ("n_skills", C.c_int32),
                ("reason", C.c_int32), ("est_exec_us", C.c_int64), ("dispatch_us", C.c_int64),
                ("tokens", C.c_int32 * RT_SEG_MAX_TOKENS)]


class rt_round_info(C.Structure):
    _fields_ = [("t_us", C.c_int64), ("round_us", C.c_int64), ("n_waiting", C.c_int32),
                ("n_running", C.c_int32), ("n_admitted", C.c_int32), ("n_stopped", C.c_int32),
                ("n_refused_mem", C.c_int32), ("n_refused_wcet", C.c_int32), ("n_rows", C.c_int32),
                ("n_prefill_rows", C.c_int32), ("n_evicted", C.c_int32), ("n_restored", C.c_int32)]


class rt_stats(C.Structure):
    _fields_ = [("rounds", C.c_int64), ("tokens", C.c_int64), ("segments", C.c_int64),
                ("prefill_tokens", C.c_int64), ("attn_ms", C.c_double), ("gemm_ms", C.c_double),
                ("sched_ms", C.c_double), ("step_ms", C.c_double), ("attn_launches", C.c_int64),
                ("gemm_launches", C.c_int64), ("kernel_launches", C.c_int64), ("attn_bytes", C.c_double)]


def lib():
    """Load the in-tree library (raises if it was not built — no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise ImportError(f"{_LIB_PATH} missing: run __graft_entry__.build() (no CPU fallback exists)")
    L = C.CDLL(_LIB_PATH)
    L.rt_create.argtypes = [C.POINTER(rt_config), C.POINTER(C.c_void_p)]
    L.rt_destroy.argtypes = [C.c_void_p]
    L.rt_submit_request.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_int64, C.c_int64,
                                    rt_utility, C.c_int32, C.c_int32, C.c_void_p, C.c_int32,
                                    C.POINTER(C.c_int64)]
    L.rt_step.argtypes = [C.c_void_p, C.c_int64, C.POINTER(rt_round_info)]
    L.rt_register_prefix.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.POINTER(C.c_int32)]
    L.rt_poll_segment.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.POINTER(C.c_int32)]
    L.rt_poll_segment_ready.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.POINTER(C.c_int32)]
    L.rt_last_round.argtypes = [C.c_void_p, C.POINTER(rt_round_info)]
    L.rt_sync.argtypes = [C.c_void_p]
    L.rt_get_stats.argtypes = [C.c_void_p, C.POINTER(rt_stats)]
    L.rt_reset_stats.argtypes = [C.c_void_p]
    L.rt_debug_dump.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_int64, C.POINTER(C.c_int64)]
    L.rt_last_error.argtypes = [C.c_void_p]
    L.rt_last_error.restype = C.c_char_p
    L.rt_version.restype = C.c_char_p
    vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
    L.rt_op_paged_attention.argtypes = [vp, vp, vp, i32, vp, vp, i32, i32, i32, i32, i32, vp, vp, vp, i64, vp]
    L.rt_op_attention_ws_bytes.argtypes = [i32, i32, i32, i32]
    L.rt_op_attention_ws_bytes.restype = i64
    L.rt_op_kv_write.argtypes = [vp, vp, vp, vp, i32, i32, i32, vp]
    L.rt_op_kv_read.argtypes = [vp, vp, i32, i32, i32, vp]
    L.rt_op_kv_swap.argtypes = [vp, i32, vp, i64, vp, i64, i32, vp]
    L.rt_op_gemm.argtypes = [vp, vp, vp, i32, i32, i32, i32, i32, vp]
    L.rt_op_lm_argmax.argtypes = [vp, vp, i32, i32, i32, i32, vp, vp, vp, i64, vp]
    L.rt_op_init_weights.argtypes = [vp, i64, C.c_uint64, i32, C.c_float, vp]
    L.rt_op_priority.argtypes = [vp, vp, vp, vp, i32, i32, i32, i32, vp, vp]
    L.rt_mark.argtypes = [vp, i32]
    L.rt_set_timing.argtypes = [vp, i32]
    L.rt_elapsed_ms.argtypes = [vp, C.POINTER(C.c_double)]
    L.rt_nccl_unique_id.argtypes = [vp]
    L.rt_op_pack_tiled.argtypes = [vp, vp, i32, i32, vp]
    L.rt_op_gemm_tiled.argtypes = [vp, vp, vp, i32, i32, i32, i32, i32, i32, i32, vp]
    L.rt_op_merge_candidates.argtypes = [vp, i32, vp, vp]
    L.rt_op_prefill_attention.argtypes = [vp, vp, vp, i32, vp, i32, i32, i32, i32, i32, i32, vp, vp, vp]
    for f in EXPORTED:
        if f not in ("rt_last_error", "rt_version", "rt_op_attention_ws_bytes"):
            getattr(L, f).restype = C.c_int32
    _lib = L
    return L


def _check(code, eng=None):
    if code != RT_OK:
        msg = lib().rt_last_error(eng).decode(errors="replace")
        raise RtError(code, msg)


def _i32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


class Engine:
    """One engine per GPU/process (C ABI rt_engine)."""

    def __init__(self, shape, params, vocab, seed=0, flags=0, device=0, rank=0, world=1, nccl_id=None,
                 init_std=0.02, capture_layer=0, max_rows_per_forward=0, kv_pool_bytes=0, gemm_path=0):
        L = lib()
        c = rt_config()
        c.rank, c.world, c.device = rank, world, device
        self._nccl = None
        if nccl_id is not None:
            self._nccl = C.create_string_buffer(bytes(nccl_id), 128)
            c.nccl_id = C.cast(self._nccl, C.c_void_p)
        if shape is not None:
            c.n_layers, c.d_model, c.n_q_heads = shape.n_layers, shape.d_model, shape.n_q_heads
            c.n_kv_heads, c.head_dim, c.d_ff, c.vocab = shape.n_kv_heads, shape.head_dim, shape.d_ff, shape.vocab
        else:
            c.vocab = vocab.vocab
            flags |= RT_FLAG_NO_MODEL
        c.weight_seed, c.init_std = seed, init_std
        p = params
        c.page_tokens, c.max_batch, c.max_tasks, c.max_ctx = p.page_tokens, p.max_batch, p.max_tasks, p.max_ctx
        c.n_pages, c.kv_pool_bytes, c.max_rows_per_forward = p.n_pages, kv_pool_bytes, max_rows_per_forward
        c.max_seg_tokens, c.g_us, c.net_us, c.eps_l_us = p.max_seg_tokens, p.g_us, p.net_us, p.eps_l_us
        c.speed_window = p.speed_window
        c.max_admit_per_round = min(p.max_admit_per_round, 1 << 30)
        c.policy, c.clock_mode = p.policy, p.clock_mode
        c.base_us, c.gamma_ppm, c.kv_us_per_1k, c.prefill_us_per_tok = (p.base_us, p.gamma_ppm,
                                                                          p.kv_us_per_1k, p.prefill_us_per_tok)
        c.t0_us = p.t0_us
        self._skill = np.ascontiguousarray(vocab.tok_skill, dtype=np.int16)
        self._exec = np.ascontiguousarray(vocab.tok_exec_min_us, dtype=np.int32)
        c.tok_skill = self._skill.ctypes.data
        c.tok_exec_min_us = self._exec.ctypes.data
        c.eos_id = vocab.eos_id
        c.flags, c.capture_layer = flags, capture_layer
        c.seg_mode, c.wcet_off = p.seg_mode, p.wcet_off
        c.host_pages, c.swap_us_per_page = p.host_pages, p.swap_us_per_page
        c.stop_grammar, c.word_us = p.stop_grammar, p.word_us
        c.gemm_path = gemm_path
        if getattr(vocab, "tok_class", None) is not None:   # synth.grammar.GrammarVocab (NEXT-4)
            self._cls = np.ascontiguousarray(vocab.tok_class, dtype=np.int16)
            self._sbase = np.ascontiguousarray(vocab.skill_base_us, dtype=np.int32)
            self._sunit = np.ascontiguousarray(vocab.skill_unit_us, dtype=np.int32)
            c.tok_class = self._cls.ctypes.data
            c.skill_base_us = self._sbase.ctypes.data
            c.skill_unit_us = self._sunit.ctypes.data
        self.cfg = c
        self.shape, self.params, self.vocab = shape, params, vocab
        h = C.c_void_p()
        _check(L.rt_create(C.byref(c), C.byref(h)), None)
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            lib().rt_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def submit(self, agent_id, prompt, arrival_us, ert_us, alpha, beta, exec_window_us, max_new_tokens=0,
               script=None):
        pr = _i32(prompt)
        sc = _i32(script) if script is not None else None
        rid = C.c_int64()
        _check(lib().rt_submit_request(self.h, agent_id, pr.ctypes.data, len(pr), int(arrival_us), int(ert_us),
                                       rt_utility(alpha, beta), int(exec_window_us), int(max_new_tokens),
                                       sc.ctypes.data if sc is not None else None,
                                       len(sc) if sc is not None else 0, C.byref(rid)), self.h)
        return rid.value

    def register_prefix(self, tokens):
        """Shared read-only prompt prefix (len a multiple of 16); returns its id."""
        t = _i32(tokens)
        pid = C.c_int32()
        _check(lib().rt_register_prefix(self.h, t.ctypes.data, len(t), C.byref(pid)), self.h)
        return pid.value

    def step(self, now_us=0):
        info = rt_round_info()
        _check(lib().rt_step(self.h, int(now_us), C.byref(info)), self.h)
        return _info_dict(info)

    def last_round(self):
        info = rt_round_info()
        _check(lib().rt_last_round(self.h, C.byref(info)), self.h)
        return _info_dict(info)

    def poll(self, cap=512, wait=True):
        """rt_poll_segment (wait=True: the last launched round included) or
        rt_poll_segment_ready (wait=False: only rounds the device has retired)."""
        # one reusable record buffer per engine (a fresh 4096-record ctypes array was 2.3 MB
        # of zeroing per call, visible in the e2e loop's host time)
        buf = getattr(self, "_pbuf", None)
        if buf is None or len(buf) < cap:
            buf = self._pbuf = (rt_segment * cap)()
        cap = len(buf)
        n = C.c_int32()
        out = []
        fn = lib().rt_poll_segment if wait else lib().rt_poll_segment_ready
        while True:
            _check(fn(self.h, buf, cap, C.byref(n)), self.h)
            for i in range(n.value):
                s = buf[i]
                nt = s.tok_end - s.tok_begin
                out.append(dict(request_id=s.request_id, agent_id=s.agent_id, k=s.k, tok_begin=s.tok_begin,
                                tok_end=s.tok_end, n_skills=s.n_skills, est_exec_us=s.est_exec_us,
                                reason=s.reason, dispatch_us=s.dispatch_us, tokens=list(s.tokens[:nt])))
            if n.value < cap:
                return out

    def poll_count(self, cap=512):
        """Drain the segment ring, returning only the number of records (bench e2e)."""
        buf = getattr(self, "_pbuf", None)
        if buf is None or len(buf) < cap:
            buf = self._pbuf = (rt_segment * cap)()
        cap = len(buf)
        n = C.c_int32()
        tot = 0
        while True:
            _check(lib().rt_poll_segment(self.h, buf, cap, C.byref(n)), self.h)
            tot += n.value
            if n.value < cap:
                return tot

    def set_timing(self, on):
        _check(lib().rt_set_timing(self.h, int(bool(on))), self.h)

    def mark(self, which):
        _check(lib().rt_mark(self.h, which), self.h)

    def elapsed_ms(self):
        ms = C.c_double()
        _check(lib().rt_elapsed_ms(self.h, C.byref(ms)), self.h)
        return ms.value

    def sync(self):
        _check(lib().rt_sync(self.h), self.h)

    def stats(self):
        s = rt_stats()
        _check(lib().rt_get_stats(self.h, C.byref(s)), self.h)
        return {f: getattr(s, f) for f, _ in s._fields_}

    def reset_stats(self):
        _check(lib().rt_reset_stats(self.h), self.h)

    def tasks(self):
        """RT_DUMP_TASKS decoded: rows of (rid, state, k, ctx, n_pages, n_gen, seg_tok, R, evicted,
        host pages)."""
        return self.dump(RT_DUMP_TASKS, np.int64).reshape(-1, 10)

    def host_page_tables(self):
        """{request_id: [host pages]} of every request whose KV is evicted to host (R-EVICT)."""
        t = self.tasks()
        pts = self.dump(RT_DUMP_HOST_PAGE_TABLES, np.int32).reshape(t.shape[0], -1)
        out = {}
        for i in range(t.shape[0]):
            rid, state = int(t[i, 0]), int(t[i, 1])
            if state in (1, 2) and t[i, 8]:
                out[rid] = [int(x) for x in pts[i, :int(t[i, 9])]]
        return out

    def page_tables(self):
        """{request_id: [pages]} of every request holding pages (admitted, not finished)."""
        t = self.tasks()
        pts = self.dump(RT_DUMP_PAGE_TABLES, np.int32).reshape(t.shape[0], -1)
        out = {}
        for i in range(t.shape[0]):
            rid, state, _, _, npg = (int(x) for x in t[i, :5])
            if state in (1, 2) and npg > 0 and not t[i, 8]:  # holders (an evicted request is not)
                out[rid] = [int(x) for x in pts[i, :npg]]
        return out

    def round_log(self):
        """RT_DUMP_ROUND decoded for the last round."""
        v = self.dump(RT_DUMP_ROUND, np.int32)
        B, n_rows, n_adm, free_top = (int(x) for x in v[:4])
        o = 4
        slots = [int(x) for x in v[o:o + B]]
        toks = [int(x) for x in v[o + B:o + 2 * B]]
        am = [int(x) for x in v[o + 2 * B:o + 3 * B]]
        adm = [int(x) for x in v[o + 3 * B:o + 3 * B + n_adm]]
        return dict(B=B, n_rows=n_rows, slots=slots, tokens=toks, argmax=am, admitted=adm, free=free_top)

    def dump(self, what, dtype=np.int32):
        need = C.c_int64()
        _check(lib().rt_debug_dump(self.h, what, None, 0, C.byref(need)), self.h)
        buf = np.zeros(max(need.value, 1), dtype=np.uint8)
        _check(lib().rt_debug_dump(self.h, what, buf.ctypes.data, buf.nbytes, C.byref(need)), self.h)
        return buf[:need.value].view(dtype)

    def layer_dump(self, what, layer, dtype):
        """Per-layer capture (RT_FLAG_CAPTURE_LAYERS / RT_DUMP_LAYER_KV) of layer ``layer``."""
        return self.dump(what | (layer << 16), dtype)

    def trace(self):
        """Per-CTA kernel records since the last reset_stats (RT_FLAG_TRACE)."""
        return self.dump(RT_DUMP_TRACE, TRACE_DTYPE)


def _info_dict(i):
    return {f: getattr(i, f) for f, _ in i._fields_}


def nccl_unique_id():
    buf = (C.c_uint8 * 128)()
    _check(lib().rt_nccl_unique_id(buf))
    return bytes(buf)


def version():
    return lib().rt_version().decode()


# ------------------------------------------------------------------ op-level API
def _ptr(t):
    return None if t is None else t.data_ptr()


def _stream(torch_stream=None):
    import torch
    s = torch_stream or torch.cuda.current_stream()
    return s.cuda_stream


def paged_attention(q, pool, page_table, row_task, row_seqlen, max_seqlen, n_q, n_kv, hd, out, out_f32=None,
                    ws=None, stream=None):
    import torch
    L = lib()
    need = L.rt_op_attention_ws_bytes(int(q.shape[0]), int(max_seqlen), n_q, hd)
    if ws is None or ws.numel() * ws.element_size() < need:
        ws = torch.zeros(max(need, 16), dtype=torch.uint8, device=q.device)  # tickets must start at 0
    _check(L.rt_op_paged_attention(_ptr(q), _ptr(pool), _ptr(page_table), int(page_table.shape[1]),
                                   _ptr(row_task), _ptr(row_seqlen), int(q.shape[0]), int(max_seqlen), n_q, n_kv,
                                   hd, _ptr(out), _ptr(out_f32), _ptr(ws), ws.numel() * ws.element_size(),
                                   _stream(stream)))
    return out


def prefill_attention(q, pool, page_table, tiles, n_q, n_kv, hd, out, out_f32=None, groups=0, stream=None):
    """tiles: int32 cuda tensor [n_tiles][4] (first row, rows <= 16, pos0, task)."""
    _check(lib().rt_op_prefill_attention(_ptr(q), _ptr(pool), _ptr(page_table), int(page_table.shape[1]),
                                         _ptr(tiles), int(tiles.shape[0]), int(q.shape[0]), n_q, n_kv, hd,
                                         int(groups), _ptr(out), _ptr(out_f32), _stream(stream)))
    return out


def kv_write(pool, k, v, slot, n_kv, hd, stream=None):
    _check(lib().rt_op_kv_write(_ptr(pool), _ptr(k), _ptr(v), _ptr(slot), int(k.shape[0]), n_kv, hd,
                                _stream(stream)))


def kv_read(pool, out, n_pages, n_kv, hd, stream=None):
    _check(lib().rt_op_kv_read(_ptr(pool), _ptr(out), n_pages, n_kv, hd, _stream(stream)))


def kv_swap(swap, pool, pool_layer_bytes, host, blk_bytes, n_layers, stream=None):
    """swap: int32 cuda tensor [n][4] (dir, task, device page, host page); host: pinned CPU
    tensor (device-addressable under UVA)."""
    _check(lib().rt_op_kv_swap(_ptr(swap), int(swap.shape[0]), _ptr(pool), int(pool_layer_bytes), _ptr(host),
                               int(blk_bytes), int(n_layers), _stream(stream)))


def gemm(w, x, out, M, N, K, n_cap, splits=1, stream=None):
    _check(lib().rt_op_gemm(_ptr(w), _ptr(x), _ptr(out), M, N, K, n_cap, splits, _stream(stream)))


def pack_tiled(w, out, M, K, stream=None):
    _check(lib().rt_op_pack_tiled(_ptr(w), _ptr(out), M, K, _stream(stream)))


def gemm_tiled(wt, x, out, M, N, K, n_cap, splits=0, stream=None, path=RT_GEMM_PATH_AUTO, bn=0):
    _check(lib().rt_op_gemm_tiled(_ptr(wt), _ptr(x), _ptr(out), M, N, K, n_cap, splits, path, bn,
                                  _stream(stream)))


def lm_argmax(w, x, M, N, K, n_cap, tok, logits=None, ws=None, stream=None):
    import torch
    need = ((M + 127) // 128) * N * 8
    if ws is None:
        ws = torch.empty(need, dtype=torch.uint8, device=x.device)
    _check(lib().rt_op_lm_argmax(_ptr(w), _ptr(x), M, N, K, n_cap, _ptr(tok), _ptr(logits), _ptr(ws),
                                 ws.numel() * ws.element_size(), _stream(stream)))


def init_weights(out, n, seed, tensor_id, sigma=0.02, stream=None):
    _check(lib().rt_op_init_weights(_ptr(out), int(n), int(seed), int(tensor_id), float(sigma), _stream(stream)))


def priority(trde, k, alpha, beta, g_us, net_us, eps_l_us, out, stream=None):
    _check(lib().rt_op_priority(_ptr(trde), _ptr(k), _ptr(alpha), _ptr(beta), int(k.shape[0]), g_us, net_us,
                                eps_l_us, _ptr(out), _stream(stream)))


def merge_candidates(all_cand, world, merged, stream=None):
    """all_cand: float64 cuda tensor [world][16][4]; merged: float64 cuda tensor [16][4]."""
    _check(lib().rt_op_merge_candidates(_ptr(all_cand), int(world), _ptr(merged), _stream(stream)))
