"""ctypes bindings for the CPU checkers. TEST INFRASTRUCTURE ONLY.

* ``Oracle``  -> oracle/liborchsim_oracle.so, the plain-C restatement of the
  reference dispatcher path (oracle/orchsim_oracle.c).
* ``RefLib``  -> oracle/_ref/liborchsim_ref.so, the unmodified reference
  (/root/reference/proj/src) compiled by ``make -C oracle ref``. Present in
  this container; travels to GPU boxes as a built artefact when it was built.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liborchsim_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "liborchsim_ref.so")

GREEDY_UNPADDED, BINARY_PADDED, QUADRATIC_TOLERANCE, CONVTRANSFORMER = 0, 1, 2, 3
LINEAR_ONLY, TRANSFORMER_QUADRATIC, CONV_TRANSFORMER_PADDED = 0, 1, 2


class OracleError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct)) if a is not None else None


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


@dataclass
class BalanceOut:
    dest_inst: np.ndarray
    dest_slot: np.ndarray
    src_slot: np.ndarray
    src_off: np.ndarray
    dst_off: np.ndarray
    bin_count: np.ndarray
    bin_len: np.ndarray
    bin_tokens: np.ndarray
    bin_cost: np.ndarray
    objective: float
    used_identity: int


class _OutStruct(C.Structure):
    _fields_ = [
        ("dest_inst", C.POINTER(C.c_int32)),
        ("dest_slot", C.POINTER(C.c_int32)),
        ("src_slot", C.POINTER(C.c_int32)),
        ("src_off", C.POINTER(C.c_int64)),
        ("dst_off", C.POINTER(C.c_int64)),
        ("bin_count", C.POINTER(C.c_int32)),
        ("bin_len", C.POINTER(C.c_int64)),
        ("bin_tokens", C.POINTER(C.c_int64)),
        ("bin_cost", C.POINTER(C.c_double)),
    ]


class Oracle:
    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        self.lib = C.CDLL(path)
        L = self.lib
        L.orc_last_error.restype = C.c_char_p
        L.orc_stats.restype = None
        L.orc_volume_matrix.restype = None
        L.orc_fill_rows.restype = None
        L.orc_batch_to_instance.restype = None
        L.orc_backbone_targets.restype = None

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self.lib.orc_last_error().decode())

    def _run(self, fn, kind, lam, v, d, length, origin, identity=False) -> BalanceOut:
        length, origin = _i64(length), _i32(origin)
        n = len(length)
        o = BalanceOut(*(np.zeros(n, np.int32) for _ in range(3)), np.zeros(n, np.int64),
                       np.zeros(n, np.int64), np.zeros(max(d, 0), np.int32),
                       np.zeros(max(d, 0), np.int64), np.zeros(max(d, 0), np.int64),
                       np.zeros(max(d, 0), np.float64), 0.0, 0)
        s = _OutStruct(_p(o.dest_inst, C.c_int32), _p(o.dest_slot, C.c_int32),
                       _p(o.src_slot, C.c_int32), _p(o.src_off, C.c_int64),
                       _p(o.dst_off, C.c_int64), _p(o.bin_count, C.c_int32),
                       _p(o.bin_len, C.c_int64), _p(o.bin_tokens, C.c_int64),
                       _p(o.bin_cost, C.c_double))
        obj = C.c_double(0)
        used = C.c_int32(0)
        if identity:
            rc = fn(C.c_int(kind), C.c_double(lam), C.c_int64(v), C.c_int(d), C.c_int64(n),
                    _p(length, C.c_int64), _p(origin, C.c_int32), C.byref(s), C.byref(obj))
            used.value = 1
        else:
            rc = fn(C.c_int(kind), C.c_double(lam), C.c_int64(v), C.c_int(d), C.c_int64(n),
                    _p(length, C.c_int64), _p(origin, C.c_int32), C.byref(s), C.byref(obj),
                    C.byref(used))
        self._check(rc)
        o.objective, o.used_identity = obj.value, used.value
        return o

    def balance(self, kind, d, length, origin, lam=0.0, v=0) -> BalanceOut:
        return self._run(self.lib.orc_balance, kind, lam, v, d, length, origin)

    def identity(self, kind, d, length, origin, lam=0.0, v=0) -> BalanceOut:
        return self._run(self.lib.orc_identity, kind, lam, v, d, length, origin, identity=True)

    def min_feasible_padded_bound(self, d, length, origin) -> int:
        length, origin = _i64(length), _i32(origin)
        out = C.c_int64(0)
        self._check(self.lib.orc_min_feasible_padded_bound(
            C.c_int(d), C.c_int64(len(length)), _p(length, C.c_int64), _p(origin, C.c_int32),
            C.byref(out)))
        return out.value

    def padded_bound_feasible(self, d, length, origin, bound) -> bool:
        length, origin = _i64(length), _i32(origin)
        out = C.c_int32(0)
        self._check(self.lib.orc_padded_bound_feasible(
            C.c_int(d), C.c_int64(len(length)), _p(length, C.c_int64), _p(origin, C.c_int32),
            C.c_int64(bound), C.byref(out)))
        return bool(out.value)

    def cost(self, alpha, beta, model_padded, variant, batch_padded, lengths) -> float:
        lengths = _i64(lengths)
        out = C.c_double(0)
        self._check(self.lib.orc_cost(C.c_double(alpha), C.c_double(beta), C.c_int(model_padded),
                                      C.c_int(variant), C.c_int(batch_padded),
                                      C.c_int64(len(lengths)), _p(lengths, C.c_int64),
                                      C.byref(out)))
        return out.value

    def stats(self, costs):
        costs = np.ascontiguousarray(costs, dtype=np.float64)
        mx, mn, ra = C.c_double(), C.c_double(), C.c_double()
        self.lib.orc_stats(C.c_int(len(costs)), _p(costs, C.c_double), C.byref(mx), C.byref(mn),
                           C.byref(ra))
        return mx.value, mn.value, ra.value

    def volume_matrix(self, d, length, origin, dest_inst):
        length, origin, dest_inst = _i64(length), _i32(origin), _i32(dest_inst)
        V = np.zeros(d * d, np.int64)
        self.lib.orc_volume_matrix(C.c_int(d), C.c_int64(len(length)), _p(length, C.c_int64),
                                   _p(origin, C.c_int32), _p(dest_inst, C.c_int32),
                                   _p(V, C.c_int64))
        return V.reshape(d, d)

    def layout(self, d, P, length, origin, dest_inst, dest_slot):
        length, origin = _i64(length), _i32(origin)
        dest_inst, dest_slot = _i32(dest_inst), _i32(dest_slot)
        n = len(length)
        rs, rd, po = (np.zeros(n, np.int64) for _ in range(3))
        S = np.zeros(P * P, np.int64)
        tin, tout = np.zeros(P, np.int64), np.zeros(P, np.int64)
        self._check(self.lib.orc_layout(
            C.c_int(d), C.c_int(P), C.c_int64(n), _p(length, C.c_int64), _p(origin, C.c_int32),
            _p(dest_inst, C.c_int32), _p(dest_slot, C.c_int32), _p(rs, C.c_int64),
            _p(rd, C.c_int64), _p(po, C.c_int64), _p(S, C.c_int64), _p(tin, C.c_int64),
            _p(tout, C.c_int64)))
        return dict(rank_src_off=rs, rank_dst_off=rd, pair_off=po, send_tokens=S.reshape(P, P),
                    in_tokens=tin, out_tokens=tout)

    def dispatch_rows(self, d, P, length, origin, dest_inst, rank_src_off, rank_dst_off,
                      row_bytes, in_bufs, out_bufs, nthreads=1):
        """in_bufs/out_bufs: lists of P uint8 numpy arrays (host)."""
        length, origin, dest_inst = _i64(length), _i32(origin), _i32(dest_inst)
        rs, rd = _i64(rank_src_off), _i64(rank_dst_off)
        ins = (C.c_void_p * P)(*[b.ctypes.data for b in in_bufs])
        outs = (C.c_void_p * P)(*[b.ctypes.data for b in out_bufs])
        self._check(self.lib.orc_dispatch_rows(
            C.c_int(d), C.c_int(P), C.c_int64(len(length)), _p(length, C.c_int64),
            _p(origin, C.c_int32), _p(dest_inst, C.c_int32), _p(rs, C.c_int64),
            _p(rd, C.c_int64), C.c_size_t(row_bytes), ins, outs, C.c_int(nthreads)))

    def solve_hosting(self, d, c, V):
        V = np.ascontiguousarray(V, dtype=np.int64).reshape(-1)
        hosting = np.zeros(d, np.int32)
        eg = np.zeros(d // c, np.int64)
        mx, base, vis = C.c_int64(), C.c_int64(), C.c_int64()
        self._check(self.lib.orc_solve_hosting(C.c_int(d), C.c_int(c), _p(V, C.c_int64),
                                               _p(hosting, C.c_int32), _p(eg, C.c_int64),
                                               C.byref(mx), C.byref(base), C.byref(vis)))
        b2i = np.zeros(d, np.int32)
        self.lib.orc_batch_to_instance(C.c_int(d), C.c_int(c), _p(hosting, C.c_int32),
                                       _p(b2i, C.c_int32))
        return dict(hosting=hosting, per_node_egress=eg, max_egress=mx.value,
                    baseline_max=base.value, visited=vis.value, batch_to_instance=b2i)

    def backbone_targets(self, d, llm_dest_inst, llm_dest_slot, part_offset, interleave_pos,
                         item_part):
        a = [np.ascontiguousarray(x, np.int32) for x in
             (llm_dest_inst, llm_dest_slot, part_offset, interleave_pos, item_part)]
        n = len(a[4])
        di, ds = np.zeros(n, np.int32), np.zeros(n, np.int32)
        self.lib.orc_backbone_targets(C.c_int(d), C.c_int64(len(a[0])), _p(a[0], C.c_int32),
                                      _p(a[1], C.c_int32), _p(a[2], C.c_int32),
                                      _p(a[3], C.c_int32), C.c_int64(n), _p(a[4], C.c_int32),
                                      _p(di, C.c_int32), _p(ds, C.c_int32))
        return di, ds

    def rearrange_offsets(self, d, length, src_inst, src_slot, dst_inst, dst_slot):
        length = _i64(length)
        si, ss, di, ds = (_i32(x) for x in (src_inst, src_slot, dst_inst, dst_slot))
        n = len(length)
        so, do = np.zeros(n, np.int64), np.zeros(n, np.int64)
        self._check(self.lib.orc_rearrange_offsets(
            C.c_int(d), C.c_int64(n), _p(length, C.c_int64), _p(si, C.c_int32),
            _p(ss, C.c_int32), _p(di, C.c_int32), _p(ds, C.c_int32), _p(so, C.c_int64),
            _p(do, C.c_int64)))
        return so, do

    def fill_rows(self, length, tag, row_off, row_bytes, buf):
        length, tag, row_off = _i64(length), _i64(tag), _i64(row_off)
        self.lib.orc_fill_rows(C.c_int64(len(length)), _p(length, C.c_int64), _p(tag, C.c_int64),
                               _p(row_off, C.c_int64), C.c_size_t(row_bytes),
                               C.c_void_p(buf.ctypes.data))


class RefLib:
    """The reference library itself (oracle/_ref), when it was built."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` (needs /root/reference)")
        self.lib = C.CDLL(path)
        self.lib.ref_last_error.restype = C.c_char_p

    @staticmethod
    def available(path: str = REF_SO) -> bool:
        return os.path.exists(path)

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self.lib.ref_last_error().decode())

    def balance(self, kind, d, length, origin, lam=0.0, v=0):
        length, origin = _i64(length), _i32(origin)
        n = len(length)
        di, ds = np.zeros(n, np.int32), np.zeros(n, np.int32)
        obj, ident = C.c_double(0), C.c_int32(0)
        self._check(self.lib.ref_balance(C.c_int(kind), C.c_double(lam), C.c_int64(v), C.c_int(d),
                                         C.c_int64(n), _p(length, C.c_int64),
                                         _p(origin, C.c_int32), _p(di, C.c_int32),
                                         _p(ds, C.c_int32), C.byref(obj), C.byref(ident)))
        return di, ds, obj.value, ident.value

    def identity(self, kind, d, length, origin, lam=0.0, v=0):
        length, origin = _i64(length), _i32(origin)
        n = len(length)
        di, ds = np.zeros(n, np.int32), np.zeros(n, np.int32)
        obj = C.c_double(0)
        self._check(self.lib.ref_identity(C.c_int(kind), C.c_double(lam), C.c_int64(v), C.c_int(d),
                                          C.c_int64(n), _p(length, C.c_int64),
                                          _p(origin, C.c_int32), _p(di, C.c_int32),
                                          _p(ds, C.c_int32), C.byref(obj)))
        return di, ds, obj.value

    def min_feasible_padded_bound(self, d, length, origin):
        length, origin = _i64(length), _i32(origin)
        out = C.c_int64(0)
        self._check(self.lib.ref_min_feasible_padded_bound(
            C.c_int(d), C.c_int64(len(length)), _p(length, C.c_int64), _p(origin, C.c_int32),
            C.byref(out)))
        return out.value

    def padded_bound_feasible(self, d, length, origin, bound):
        length, origin = _i64(length), _i32(origin)
        out = C.c_int32(0)
        self._check(self.lib.ref_padded_bound_feasible(
            C.c_int(d), C.c_int64(len(length)), _p(length, C.c_int64), _p(origin, C.c_int32),
            C.c_int64(bound), C.byref(out)))
        return bool(out.value)

    def cost(self, alpha, beta, model_padded, variant, batch_padded, lengths):
        lengths = _i64(lengths)
        out = C.c_double(0)
        self._check(self.lib.ref_cost(C.c_double(alpha), C.c_double(beta), C.c_int(model_padded),
                                      C.c_int(variant), C.c_int64(len(lengths)),
                                      _p(lengths, C.c_int64), C.c_int(batch_padded),
                                      C.byref(out)))
        return out.value

    def solve_hosting(self, d, c, V):
        V = np.ascontiguousarray(V, dtype=np.int64).reshape(-1)
        hosting = np.zeros(d, np.int32)
        mx, vis = C.c_int64(), C.c_int64()
        self._check(self.lib.ref_solve_hosting(C.c_int(d), C.c_int(c), _p(V, C.c_int64),
                                               _p(hosting, C.c_int32), C.byref(mx),
                                               C.byref(vis)))
        return dict(hosting=hosting, max_egress=mx.value, visited=vis.value)

    def time_balance(self, kind, d, length, origin, reps, lam=0.0, v=0):
        length, origin = _i64(length), _i32(origin)
        secs = np.zeros(reps, np.float64)
        self._check(self.lib.ref_time_balance(C.c_int(kind), C.c_double(lam), C.c_int64(v),
                                              C.c_int(d), C.c_int64(len(length)),
                                              _p(length, C.c_int64), _p(origin, C.c_int32),
                                              C.c_int(reps), _p(secs, C.c_double)))
        return secs

    def generate(self, mix, n, seed):
        ppe = np.zeros(n, np.int32)
        mod = np.full(3 * n, -1, np.int32)
        ml = np.zeros(3 * n, np.int64)
        self._check(self.lib.ref_generate(C.c_int(mix), C.c_int(n), C.c_uint64(seed),
                                          _p(ppe, C.c_int32), _p(mod, C.c_int32),
                                          _p(ml, C.c_int64)))
        return ppe, mod.reshape(n, 3), ml.reshape(n, 3)

    def run_iteration(self, mix, d, per_instance, seed, c=None, nodewise=False):
        """The reference orchestrator's run_iteration (composed delivery on):
        LLM destinations per example and, per part (example-major), the
        instance and position of the backbone's assembled input."""
        E = d * per_instance
        ppe, _, _ = self.generate(mix, E, seed)
        parts = int(ppe.sum())
        li, ls = np.zeros(E, np.int32), np.zeros(E, np.int32)
        ai, ap = np.zeros(parts, np.int32), np.zeros(parts, np.int32)
        flags = np.zeros(3, np.int32)
        self._check(self.lib.ref_run_iteration(
            C.c_int(mix), C.c_int(d), C.c_int(c or d), C.c_int(per_instance), C.c_uint64(seed),
            C.c_int(1 if nodewise else 0), _p(li, C.c_int32), _p(ls, C.c_int32),
            _p(ai, C.c_int32), _p(ap, C.c_int32), _p(flags, C.c_int32)))
        return dict(llm_dest_inst=li, llm_dest_slot=ls, asm_inst=ai, asm_pos=ap,
                    assembly_ok=int(flags[0]), composed_exchanges=int(flags[1]),
                    vision_delivery_exchanges=int(flags[2]), parts_per_example=ppe)
