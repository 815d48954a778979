"""ctypes binding of the C-ABI (include/orchsim_capi.h) for Python callers
(tests, bench, smoke). Device memory and streams come from torch; every
compute call goes to liborchsim_b200.so. There is no fallback: if the library
or a CUDA device is missing, construction raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import torch

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ORCH_LIB_PATH") or os.path.join(PKG, "lib", "liborchsim_b200.so")

GREEDY_UNPADDED, BINARY_PADDED, QUADRATIC_TOLERANCE, CONVTRANSFORMER = 0, 1, 2, 3
LINEAR_ONLY, TRANSFORMER_QUADRATIC, CONV_TRANSFORMER_PADDED = 0, 1, 2

OK, INVALID_ARGUMENT, CONFIG_ERROR, SIZE_CAP, LOGIC_ERROR = 0, 1, 2, 3, 4
CUDA_ERROR, NCCL_ERROR, UNSUPPORTED = 10, 11, 12

EXPORTED = [
    "orch_ctx_create", "orch_ctx_destroy", "orch_last_error", "orch_version",
    "orch_ctx_launches", "orch_balance", "orch_balance_layout1", "orch_balance_host",
    "orch_min_feasible_padded_bound_host", "orch_padded_bound_feasible_host",
    "orch_oracle_optimal_host",
    "orch_batch_costs", "orch_batch_costs_host", "orch_volume_matrix_host", "orch_group_by_origin", "orch_encode_lengths", "orch_volume_matrix",
    "orch_layout", "orch_pack", "orch_exchange", "orch_unpack", "orch_dispatch",
    "orch_comm_unique_id", "orch_comm_create",
    "orch_comm_destroy", "orch_comm_rank", "orch_comm_size", "orch_allgather_items",
    "orch_solve_hosting_host", "orch_inter_node_egress_host", "orch_nodewise", "orch_rearrange",
    "orch_backbone_targets",
    "orch_barrier", "orch_window_create", "orch_window_create_nccl", "orch_window_ptr",
    "orch_window_bytes",
    "orch_window_destroy", "orch_window_barrier", "orch_dispatch_put", "orch_put",
    "orch_gather_window_create", "orch_gather_window_create_nccl", "orch_gather_window_destroy",
    "orch_allgather_items_put",
    "orch_gather_window_stamps", "orch_window_release", "orch_window_status", "orch_put_at",
    "orch_comm_create_local", "orch_window_create_local", "orch_gather_window_create_local",
    "orch_exchange_report", "orch_exchange_report_host", "orch_allgather_volumes",
    "orch_allgather_volumes_host", "orch_xplan_create", "orch_xplan_destroy", "orch_xplan_fetch",
    "orch_dispatch_nccl", "orch_comm_register", "orch_comm_deregister",
]


class OrchError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[orch {code}] {msg}")
        self.code = code
        self.msg = msg


class Policy(C.Structure):
    _fields_ = [("kind", C.c_int32), ("reserved", C.c_int32), ("tolerance_v", C.c_int64),
                ("lam", C.c_double)]


class CostModel(C.Structure):
    _fields_ = [("alpha", C.c_double), ("beta", C.c_double), ("padded", C.c_int32),
                ("variant", C.c_int32)]


class Summary(C.Structure):
    _fields_ = [("objective", C.c_double), ("algo_objective", C.c_double),
                ("identity_objective", C.c_double), ("pre_max", C.c_double),
                ("pre_mean", C.c_double), ("pre_ratio", C.c_double), ("post_max", C.c_double),
                ("post_mean", C.c_double), ("post_ratio", C.c_double), ("bound", C.c_int64),
                ("error_index", C.c_int64), ("error", C.c_int32), ("used_identity", C.c_int32),
                ("rounds", C.c_int64)]


SUMMARY_BYTES = C.sizeof(Summary)


class BalanceOutS(C.Structure):
    _fields_ = [(k, C.c_void_p) for k in (
        "dest_inst", "dest_slot", "src_slot", "src_off", "dst_off", "bin_count", "bin_len",
        "bin_tokens", "bin_cost", "bin_offset", "bin_member", "src_offset", "src_member",
        "summary")]


class LayoutOutS(C.Structure):
    _fields_ = [(k, C.c_void_p) for k in (
        "rank_src_off", "rank_dst_off", "pair_off", "send_rows", "send_displ", "recv_displ",
        "in_rows", "out_rows", "status")]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise OrchError(CUDA_ERROR, f"{LIB_PATH} is missing: run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        L.orch_last_error.restype = C.c_char_p
        L.orch_ctx_launches.restype = C.c_int64
        L.orch_ctx_destroy.restype = None
        L.orch_comm_destroy.restype = None
        L.orch_window_ptr.restype = C.c_void_p
        L.orch_xplan_destroy.restype = None
        L.orch_window_bytes.restype = C.c_size_t
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        raise OrchError(rc, lib().orch_last_error().decode())


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)


def _on(stream):
    """Allocate a call's outputs on the stream the call runs on, so the caching
    allocator never hands them to other work while the call's kernels still
    write them (outputs a caller drops are recycled in stream order)."""
    import contextlib
    return torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext()


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


@dataclass
class Balance:
    """Flat BalanceResult on the device (balancers.hpp:20-24)."""
    d: int
    n: int
    dest_inst: torch.Tensor
    dest_slot: torch.Tensor
    src_slot: torch.Tensor
    src_off: torch.Tensor
    dst_off: torch.Tensor
    bin_count: torch.Tensor
    bin_len: torch.Tensor
    bin_tokens: torch.Tensor
    bin_cost: torch.Tensor
    bin_offset: torch.Tensor
    bin_member: torch.Tensor
    src_offset: torch.Tensor
    src_member: torch.Tensor
    summary_raw: torch.Tensor  # uint8 [SUMMARY_BYTES] on device

    @staticmethod
    def alloc(d: int, n: int, device) -> "Balance":
        nn = max(n, 1)
        i32 = dict(dtype=torch.int32, device=device)
        i64 = dict(dtype=torch.int64, device=device)
        return Balance(d, n, torch.empty(nn, **i32), torch.empty(nn, **i32),
                       torch.empty(nn, **i32), torch.empty(nn, **i64), torch.empty(nn, **i64),
                       torch.empty(d, **i32), torch.empty(d, **i64), torch.empty(d, **i64),
                       torch.empty(d, dtype=torch.float64, device=device),
                       torch.empty(d + 1, **i32), torch.empty(nn, **i32),
                       torch.empty(d + 1, **i32), torch.empty(nn, **i32),
                       torch.empty(SUMMARY_BYTES, dtype=torch.uint8, device=device))

    def struct(self) -> BalanceOutS:
        st = self.__dict__.get("_struct")
        if st is None:  # device pointers are fixed for the life of the tensors
            st = BalanceOutS(*[_ptr(getattr(self, k)) for k in (
                "dest_inst", "dest_slot", "src_slot", "src_off", "dst_off", "bin_count",
                "bin_len", "bin_tokens", "bin_cost", "bin_offset", "bin_member", "src_offset",
                "src_member", "summary_raw")])
            self.__dict__["_struct"] = st
        return st

    def summary(self) -> Summary:
        raw = self.summary_raw.cpu().numpy().tobytes()
        return Summary.from_buffer_copy(raw)


@dataclass
class Layout:
    P: int
    rank_src_off: torch.Tensor
    rank_dst_off: torch.Tensor
    pair_off: torch.Tensor
    send_rows: torch.Tensor
    send_displ: torch.Tensor
    recv_displ: torch.Tensor
    in_rows: torch.Tensor
    out_rows: torch.Tensor
    status: torch.Tensor

    @staticmethod
    def alloc(P: int, n: int, device) -> "Layout":
        nn = max(n, 1)
        e = lambda k: torch.empty(k, dtype=torch.int64, device=device)  # noqa: E731
        return Layout(P, e(nn), e(nn), e(nn), e(P * P), e(P * P), e(P * P), e(P), e(P),
                      torch.zeros(1, dtype=torch.int32, device=device))

    def struct(self) -> LayoutOutS:
        st = self.__dict__.get("_struct")
        if st is None:
            st = LayoutOutS(*[_ptr(getattr(self, k)) for k in (
                "rank_src_off", "rank_dst_off", "pair_off", "send_rows", "send_displ",
                "recv_displ", "in_rows", "out_rows", "status")])
            self.__dict__["_struct"] = st
        return st


class Comm:
    def __init__(self, nranks: int, rank: int, uid: bytes | None):
        """NCCL communicator; uid=None makes a loopback one (rank emulation in
        one process, orch_comm_create_local)."""
        self.h = C.c_void_p()
        if uid is None:
            _check(lib().orch_comm_create_local(C.c_int32(nranks), C.c_int32(rank),
                                                C.byref(self.h)))
        else:
            buf = (C.c_ubyte * 128).from_buffer_copy(uid)
            _check(lib().orch_comm_create(C.c_int32(nranks), C.c_int32(rank), buf,
                                          C.byref(self.h)))
        self.rank, self.size = rank, nranks

    @staticmethod
    def local_group(nranks: int) -> list["Comm"]:
        return [Comm(nranks, r, None) for r in range(nranks)]

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_ubyte * 128)()
        _check(lib().orch_comm_unique_id(buf))
        return bytes(buf)

    def register(self, t) -> C.c_void_p:
        """ncclCommRegister of a device buffer (a torch tensor); returns the handle."""
        h = C.c_void_p()
        _check(lib().orch_comm_register(self.h, _ptr(t), C.c_size_t(t.numel() * t.element_size()),
                                        C.byref(h)))
        return h

    def deregister(self, h):
        _check(lib().orch_comm_deregister(self.h, h))

    def close(self):
        if self.h:
            lib().orch_comm_destroy(self.h)
            self.h = C.c_void_p()


class XPlan:
    """orch_xplan: pinned host mirror of a layout for orch_dispatch_nccl."""

    def __init__(self, ctx: "Context", max_n: int, P: int):
        self.h = C.c_void_p()
        _check(lib().orch_xplan_create(ctx.h, C.c_int64(max_n), C.c_int32(P), C.byref(self.h)))

    def close(self):
        if self.h:
            lib().orch_xplan_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Window:
    """orch_window: a peer-mapped row buffer of one rank (collective create):
    CUDA IPC (backend "ipc") or NCCL symmetric memory (backend "nccl",
    orch_window_create_nccl)."""

    def __init__(self, ctx: "Context", comm: Comm, nbytes: int, _handle=None, backend="ipc"):
        self.h = C.c_void_p()
        if _handle is not None:
            self.h = _handle
        else:
            create = {"ipc": lib().orch_window_create,
                      "nccl": lib().orch_window_create_nccl}[backend]
            _check(create(ctx.h, comm.h, C.c_size_t(nbytes), C.byref(self.h)))
        self.nbytes = nbytes
        self.ptr = lib().orch_window_ptr(self.h)

    @staticmethod
    def local_group(ctx: "Context", comms: list[Comm], nbytes: int) -> list["Window"]:
        """The windows of P loopback ranks in this process (orch_window_create_local)."""
        P = len(comms)
        hs = (C.c_void_p * P)()
        cs = (C.c_void_p * P)(*[c.h.value for c in comms])
        _check(lib().orch_window_create_local(ctx.h, cs, C.c_int32(P), C.c_size_t(nbytes), hs))
        return [Window(ctx, comms[r], nbytes, _handle=C.c_void_p(hs[r])) for r in range(P)]

    def status(self) -> int:
        out = C.c_int32(0)
        _check(lib().orch_window_status(self.h, C.byref(out)))
        return out.value

    def tensor_view(self, device):
        """A uint8 torch view of this rank's window (no copy)."""
        import torch
        return _view_u8(self.ptr, self.nbytes, device)

    def close(self):
        if self.h:
            _check(lib().orch_window_destroy(self.h))
            self.h = C.c_void_p()


class GatherWindow:
    """orch_gather_window: peer-memory all-gather of item records (collective);
    backend "ipc" (CUDA IPC) or "nccl" (NCCL symmetric memory)."""

    def __init__(self, ctx: "Context", comm: Comm, max_n: int, _handle=None, backend="ipc"):
        self.h = C.c_void_p()
        if _handle is not None:
            self.h = _handle
        else:
            create = {"ipc": lib().orch_gather_window_create,
                      "nccl": lib().orch_gather_window_create_nccl}[backend]
            _check(create(ctx.h, comm.h, C.c_int64(max_n), C.byref(self.h)))
        self.max_n = max_n

    @staticmethod
    def local_group(ctx: "Context", comms: list[Comm], max_n: int) -> list["GatherWindow"]:
        P = len(comms)
        hs = (C.c_void_p * P)()
        cs = (C.c_void_p * P)(*[c.h.value for c in comms])
        _check(lib().orch_gather_window_create_local(ctx.h, cs, C.c_int32(P), C.c_int64(max_n),
                                                     hs))
        return [GatherWindow(ctx, comms[r], max_n, _handle=C.c_void_p(hs[r])) for r in range(P)]

    def stamps(self):
        """[8][8] %globaltimer ns of the last 8 calls' stages (diagnostics)."""
        import numpy as np
        out = np.zeros(64, np.uint64)
        _check(lib().orch_gather_window_stamps(self.h, out.ctypes.data_as(C.c_void_p)))
        return out.reshape(8, 8)

    def close(self):
        if self.h:
            _check(lib().orch_gather_window_destroy(self.h))
            self.h = C.c_void_p()


def _view_u8(ptr, nbytes, device):
    class _Holder:
        pass
    h = _Holder()
    h.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                  "version": 3, "strides": None}
    return torch.as_tensor(h, device=device)


class Context:
    """orch_ctx on one CUDA device."""

    def __init__(self, device: int = 0):
        if not torch.cuda.is_available():
            raise OrchError(CUDA_ERROR, "no CUDA device: the B200 dispatcher has no CPU path")
        self.device = device
        self.h = C.c_void_p()
        _check(lib().orch_ctx_create(C.c_int(device), C.byref(self.h)))

    def close(self):
        if self.h:
            lib().orch_ctx_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def launches(self) -> int:
        return int(lib().orch_ctx_launches(self.h))

    # ---- balance
    def balance(self, kind, d, length, origin, lam=0.0, v=0, identity_only=False, out=None,
                stream=None) -> Balance:
        """length int64 / origin int32 CUDA tensors, input order."""
        n = int(length.numel())
        if out is None:
            with _on(stream):
                out = Balance.alloc(d, n, length.device)
        pol = Policy(kind, 0, v, lam)
        s = out.struct()
        _check(lib().orch_balance(self.h, C.byref(pol), C.c_int32(d), C.c_int64(n), _ptr(length),
                                  _ptr(origin), C.c_int32(1 if identity_only else 0), C.byref(s),
                                  _stream(stream)))
        return out

    def balance_layout1(self, kind, d, length, origin, lam=0.0, v=0, identity_only=False,
                        out=None, layout=None, stream=None):
        """orch_balance_layout1: balance + the single-rank layout (fused when small)."""
        n = int(length.numel())
        if out is None or layout is None:
            with _on(stream):
                out = out or Balance.alloc(d, n, length.device)
                layout = layout or Layout.alloc(1, n, length.device)
        pol = Policy(kind, 0, v, lam)
        _check(lib().orch_balance_layout1(self.h, C.byref(pol), C.c_int32(d), C.c_int64(n),
                                          _ptr(length), _ptr(origin),
                                          C.c_int32(1 if identity_only else 0),
                                          C.byref(out.struct()), C.byref(layout.struct()),
                                          _stream(stream)))
        return out, layout

    def balance_host(self, kind, d, length, origin, lam=0.0, v=0, identity_only=False):
        """numpy in / numpy out through orch_balance_host (synchronous)."""
        import numpy as np
        length = np.ascontiguousarray(length, dtype=np.int64)
        origin = np.ascontiguousarray(origin, dtype=np.int32)
        n = len(length)
        di, ds = np.zeros(max(n, 1), np.int32), np.zeros(max(n, 1), np.int32)
        doff = np.zeros(max(n, 1), np.int64)
        bc, bcost = np.zeros(max(d, 1), np.int32), np.zeros(max(d, 1), np.float64)
        summ = Summary()
        pol = Policy(kind, 0, v, lam)
        p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
        _check(lib().orch_balance_host(self.h, C.byref(pol), C.c_int32(d), C.c_int64(n),
                                       p(length), p(origin), C.c_int32(1 if identity_only else 0),
                                       p(di), p(ds), p(doff), p(bc), p(bcost), C.byref(summ),
                                       _stream()))
        return dict(dest_inst=di[:n], dest_slot=ds[:n], dst_off=doff[:n], bin_count=bc[:d],
                    bin_cost=bcost[:d], summary=summ)

    def min_feasible_padded_bound(self, d, length, origin) -> int:
        import numpy as np
        length = np.ascontiguousarray(length, dtype=np.int64)
        origin = np.ascontiguousarray(origin, dtype=np.int32)
        out = C.c_int64(0)
        _check(lib().orch_min_feasible_padded_bound_host(
            self.h, C.c_int32(d), C.c_int64(len(length)), length.ctypes.data_as(C.c_void_p),
            origin.ctypes.data_as(C.c_void_p), C.byref(out), _stream()))
        return out.value

    def padded_bound_feasible(self, d, length, origin, bound) -> bool:
        import numpy as np
        length = np.ascontiguousarray(length, dtype=np.int64)
        origin = np.ascontiguousarray(origin, dtype=np.int32)
        out = C.c_int32(0)
        _check(lib().orch_padded_bound_feasible_host(
            self.h, C.c_int32(d), C.c_int64(len(length)), length.ctypes.data_as(C.c_void_p),
            origin.ctypes.data_as(C.c_void_p), C.c_int64(bound), C.byref(out), _stream()))
        return bool(out.value)

    # ---- composed delivery
    def rearrange(self, d, length, src_inst, src_slot, dst_inst, dst_slot, stream=None):
        n = int(length.numel())
        with _on(stream):
            out = Balance.alloc(d, n, length.device)
        b = out.struct()
        _check(lib().orch_rearrange(self.h, C.c_int32(d), C.c_int64(n), _ptr(length),
                                    _ptr(src_inst), _ptr(src_slot), _ptr(dst_inst),
                                    _ptr(dst_slot), C.byref(b), _stream(stream)))
        return out

    def backbone_targets(self, d, llm: "Balance", part_offset, interleave_pos, item_part,
                         stream=None):
        E = part_offset.numel() - 1
        n = item_part.numel()
        with _on(stream):
            di = torch.empty(max(n, 1), dtype=torch.int32, device=part_offset.device)
            ds = torch.empty(max(n, 1), dtype=torch.int32, device=part_offset.device)
        _check(lib().orch_backbone_targets(self.h, C.c_int32(d), C.c_int64(E), _ptr(llm.dest_inst),
                                           _ptr(llm.bin_offset), _ptr(llm.bin_member),
                                           _ptr(part_offset), _ptr(interleave_pos),
                                           C.c_int64(interleave_pos.numel()), C.c_int64(n),
                                           _ptr(item_part), _ptr(di), _ptr(ds), _stream(stream)))
        return di[:n], ds[:n]

    # ---- node-wise hosting
    def solve_hosting(self, d, c, V, info=True):
        """info=False: the hosting alone (no egress figures, no replay of the
        reference's nodes_visited)."""
        import numpy as np
        V = np.ascontiguousarray(V, dtype=np.int64).reshape(-1)
        hosting = np.zeros(d, np.int32)
        inf = np.zeros(4, np.int64)
        _check(lib().orch_solve_hosting_host(self.h, C.c_int32(d), C.c_int32(c),
                                             V.ctypes.data_as(C.c_void_p),
                                             hosting.ctypes.data_as(C.c_void_p),
                                             inf.ctypes.data_as(C.c_void_p) if info else None,
                                             _stream()))
        if not info:
            return dict(hosting=hosting)
        return dict(hosting=hosting, max_egress=int(inf[0]), baseline_max=int(inf[1]),
                    leaf_used=int(inf[2]), visited=int(inf[3]))

    def inter_node_egress(self, d, c, V, hosting):
        """orch_inter_node_egress_host: per-node egress of a hosting (node per batch)."""
        import numpy as np
        V = np.ascontiguousarray(V, dtype=np.int64).reshape(-1)
        h = np.ascontiguousarray(hosting, dtype=np.int32)
        e = np.zeros(d // c, np.int64)
        _check(lib().orch_inter_node_egress_host(self.h, C.c_int32(d), C.c_int32(c),
                                                 V.ctypes.data_as(C.c_void_p),
                                                 h.ctypes.data_as(C.c_void_p),
                                                 e.ctypes.data_as(C.c_void_p), _stream()))
        return e

    def nodewise(self, d, c, length, origin, bal: "Balance", out=None, stream=None):
        """Relabels bal's destination batches in place; returns device tensors
        (hosting[d], batch_to_instance[d], info[4]) -- `out` when given."""
        dev = length.device
        if out is None:
            with _on(stream):
                out = (torch.empty(d, dtype=torch.int32, device=dev),
                       torch.empty(d, dtype=torch.int32, device=dev),
                       torch.empty(4, dtype=torch.int64, device=dev))
        hosting, b2i, info = out
        b = bal.struct()
        _check(lib().orch_nodewise(self.h, C.c_int32(d), C.c_int32(c), C.c_int64(length.numel()),
                                   _ptr(length), _ptr(origin), C.byref(b), _ptr(hosting),
                                   _ptr(b2i), _ptr(info), _stream(stream)))
        return hosting, b2i, info

    # ---- cost model
    def batch_costs(self, alpha, beta, padded, variant, batch_padded, d, length, bin_offset,
                    bin_member, stream=None):
        with _on(stream):
            cost = torch.empty(d, dtype=torch.float64, device=length.device)
            stats = torch.empty(3, dtype=torch.float64, device=length.device)
        m = CostModel(alpha, beta, padded, variant)
        _check(lib().orch_batch_costs(self.h, C.byref(m), C.c_int32(batch_padded), C.c_int32(d),
                                      C.c_int64(length.numel()), _ptr(length), _ptr(bin_offset),
                                      _ptr(bin_member), _ptr(cost), _ptr(stats), _stream(stream)))
        return cost, stats

    def group_by_origin(self, d, origin, stream=None):
        n = origin.numel()
        with _on(stream):
            off = torch.empty(d + 1, dtype=torch.int32, device=origin.device)
            mem = torch.empty(max(n, 1), dtype=torch.int32, device=origin.device)
        _check(lib().orch_group_by_origin(self.h, C.c_int32(d), C.c_int64(n), _ptr(origin),
                                          _ptr(off), _ptr(mem), _stream(stream)))
        return off, mem[:n]

    def encode_lengths(self, part_offset, modality, meta_len, rates, stream=None):
        import numpy as np
        E = part_offset.numel() - 1
        rates = np.ascontiguousarray(rates, dtype=np.int64)
        with _on(stream):
            enc = torch.empty_like(meta_len)
            inter = torch.empty(max(E, 1), dtype=torch.int64, device=meta_len.device)
        _check(lib().orch_encode_lengths(self.h, C.c_int64(E), _ptr(part_offset), _ptr(modality),
                                         _ptr(meta_len), C.c_int32(len(rates)),
                                         rates.ctypes.data_as(C.c_void_p), _ptr(enc),
                                         _ptr(inter), _stream(stream)))
        return enc, inter[:E]

    # ---- layout / movement
    def volume_matrix(self, d, length, origin, dest_inst, stream=None):
        with _on(stream):
            V = torch.empty(d * d, dtype=torch.int64, device=length.device)
        _check(lib().orch_volume_matrix(self.h, C.c_int32(d), C.c_int64(length.numel()),
                                        _ptr(length), _ptr(origin), _ptr(dest_inst), _ptr(V),
                                        _stream(stream)))
        return V.view(d, d)

    def layout(self, d, P, length, origin, bal: Balance, out: Layout | None = None,
               stream=None) -> Layout:
        n = length.numel()
        if out is None:
            with _on(stream):
                out = Layout.alloc(P, n, length.device)
        b, lo = bal.struct(), out.struct()
        _check(lib().orch_layout(self.h, C.c_int32(d), C.c_int32(P), C.c_int64(n), _ptr(length),
                                 _ptr(origin), C.byref(b), C.byref(lo), _stream(stream)))
        return out

    @staticmethod
    def _rows(t, R):
        return 0 if t is None else t.numel() * t.element_size() // R

    def dispatch(self, d, length, origin, bal: Balance, lay: Layout, row_bytes, rows_in,
                 rows_out, send=None, recv=None, comm: Comm | None = None, stream=None):
        b, lo = bal.struct(), lay.struct()
        R = row_bytes
        _check(lib().orch_dispatch(self.h, comm.h if comm else C.c_void_p(0), C.c_int32(d),
                                   C.c_int64(length.numel()), _ptr(length), _ptr(origin),
                                   C.byref(b), C.byref(lo), C.c_size_t(R), _ptr(rows_in),
                                   C.c_int64(self._rows(rows_in, R)), _ptr(rows_out),
                                   C.c_int64(self._rows(rows_out, R)), _ptr(send),
                                   C.c_int64(self._rows(send, R)), _ptr(recv),
                                   C.c_int64(self._rows(recv, R)), _stream(stream)))

    def xplan_fetch(self, xplan: "XPlan", d, length, origin, bal: Balance, lay: Layout,
                    stream=None):
        """Copy the layout's per-item runs into the plan's pinned mirror (metadata stream)."""
        _check(lib().orch_xplan_fetch(self.h, xplan.h, C.c_int32(d), C.c_int64(length.numel()),
                                      _ptr(length), _ptr(origin), C.byref(bal.struct()),
                                      C.byref(lay.struct()), _stream(stream)))

    def dispatch_nccl(self, xplan: "XPlan", row_bytes, rows_in, rows_out, comm: Comm,
                      send=None, recv=None, stream=None):
        """NCCL exchange with host counts from the plan: staged (send/recv given: pack,
        one send/recv per peer, unpack) or direct (one ncclSend/ncclRecv per item run)."""
        R = row_bytes
        _check(lib().orch_dispatch_nccl(self.h, comm.h, xplan.h, C.c_size_t(R), _ptr(rows_in),
                                        C.c_int64(self._rows(rows_in, R)), _ptr(rows_out),
                                        C.c_int64(self._rows(rows_out, R)), _ptr(send),
                                        C.c_int64(self._rows(send, R)), _ptr(recv),
                                        C.c_int64(self._rows(recv, R)), _stream(stream)))

    def pack(self, rank, P, d, length, origin, bal: Balance, lay: Layout, row_bytes, rows_in,
             rows_out, send, stream=None):
        b, lo = bal.struct(), lay.struct()
        R = row_bytes
        _check(lib().orch_pack(self.h, C.c_int32(rank), C.c_int32(P), C.c_int32(d),
                               C.c_int64(length.numel()), _ptr(length), _ptr(origin), C.byref(b),
                               C.byref(lo), C.c_size_t(R), _ptr(rows_in),
                               C.c_int64(self._rows(rows_in, R)), _ptr(rows_out),
                               C.c_int64(self._rows(rows_out, R)), _ptr(send),
                               C.c_int64(self._rows(send, R)), _stream(stream)))

    def unpack(self, rank, P, d, length, origin, bal: Balance, lay: Layout, row_bytes, recv,
               rows_out, stream=None):
        b, lo = bal.struct(), lay.struct()
        R = row_bytes
        _check(lib().orch_unpack(self.h, C.c_int32(rank), C.c_int32(P), C.c_int32(d),
                                 C.c_int64(length.numel()), _ptr(length), _ptr(origin), C.byref(b),
                                 C.byref(lo), C.c_size_t(R), _ptr(recv), _ptr(rows_out),
                                 C.c_int64(self._rows(rows_out, R)), _stream(stream)))

    def dispatch_put(self, d, length, origin, bal: Balance, lay: Layout, row_bytes, rows_in,
                     window: "Window", comm: Comm, stream=None):
        b, lo = bal.struct(), lay.struct()
        R = row_bytes
        _check(lib().orch_dispatch_put(self.h, comm.h, C.c_int32(d), C.c_int64(length.numel()),
                                       _ptr(length), _ptr(origin), C.byref(b), C.byref(lo),
                                       C.c_size_t(R), _ptr(rows_in),
                                       C.c_int64(self._rows(rows_in, R)), window.h,
                                       _stream(stream)))

    def put(self, d, length, origin, bal: Balance, lay: Layout, row_bytes, rows_in,
            window: "Window", comm: Comm, offset=0, stream=None):
        """Fused pack+put without the closing barrier (window_barrier() after),
        into byte `offset` of every rank's window (orch_put_at)."""
        b, lo = bal.struct(), lay.struct()
        R = row_bytes
        _check(lib().orch_put_at(self.h, comm.h, C.c_int32(d), C.c_int64(length.numel()),
                                 _ptr(length), _ptr(origin), C.byref(b), C.byref(lo),
                                 C.c_size_t(R), _ptr(rows_in), C.c_int64(self._rows(rows_in, R)),
                                 window.h, C.c_size_t(offset), _stream(stream)))

    def window_release(self, window: "Window", stream=None):
        """orch_window_release: this rank has consumed the window's current step."""
        _check(lib().orch_window_release(self.h, window.h, _stream(stream)))

    @staticmethod
    def barrier(comm: Comm, stream=None):
        _check(lib().orch_barrier(comm.h, _stream(stream)))

    def window_barrier(self, window: "Window", stream=None):
        """orch_window_barrier: flag barrier through the window's peer memory."""
        _check(lib().orch_window_barrier(self.h, window.h, _stream(stream)))

    def allgather_items_put(self, gwin: GatherWindow, local_pos, local_len, local_origin, n,
                            out_len, out_origin, status=None, stream=None):
        _check(lib().orch_allgather_items_put(self.h, gwin.h, C.c_int64(local_len.numel()),
                                              _ptr(local_pos), _ptr(local_len),
                                              _ptr(local_origin), C.c_int64(n), _ptr(out_len),
                                              _ptr(out_origin),
                                              _ptr(status) if status is not None else None,
                                              _stream(stream)))

    def allgather_items(self, comm: Comm, local_pos, local_len, local_origin, max_local, n,
                        out_len, out_origin, stream=None):
        _check(lib().orch_allgather_items(self.h, comm.h, C.c_int64(local_len.numel()),
                                          C.c_int64(max_local), _ptr(local_pos), _ptr(local_len),
                                          _ptr(local_origin), C.c_int64(n), _ptr(out_len),
                                          _ptr(out_origin), _stream(stream)))
