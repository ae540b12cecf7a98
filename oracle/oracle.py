"""ctypes wrappers over the oracle (liboracle.so, the C restatement) and the
compiled reference harness (_ref/libpipeplan_ref.so).

TEST INFRASTRUCTURE ONLY.  Importable from tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / reference legs — never from the product
package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libpipeplan_ref.so")

_i = C.POINTER(C.c_int)
_d = C.POINTER(C.c_double)


def _ip(a):
    return a.ctypes.data_as(_i) if a is not None else None


def _dp(a):
    return a.ctypes.data_as(_d) if a is not None else None


class OracleError(Exception):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code
        self.msg = msg


def build(ref: bool = False) -> None:
    targets = ["all"] + (["ref"] if ref else [])
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


class _Base:
    prefix = ""

    def __init__(self, path):
        self.lib = C.CDLL(path)

    def _fn(self, name):
        return getattr(self.lib, self.prefix + name)


class Oracle(_Base):
    """The C restatement (or_* functions)."""

    prefix = "or_"

    def __init__(self, path=ORACLE_SO):
        if not os.path.exists(path):
            build()
        super().__init__(path)

    # planner -----------------------------------------------------------
    def split_layer(self, fan_out, n, replicate=False, layer_id=1, devices=None):
        devs = np.arange(1, n + 1, dtype=np.int32) if devices is None else np.asarray(devices, np.int32)
        lo = np.zeros(n, np.int32)
        hi = np.zeros(n, np.int32)
        rep = np.zeros(n, np.int32)
        err = C.create_string_buffer(512)
        rc = self._fn("split_layer")(layer_id, fan_out, _ip(devs), n, int(replicate), _ip(lo), _ip(hi),
                                     _ip(rep), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        return [(int(a), int(b), bool(c)) for a, b, c in zip(lo, hi, rep)]

    def split_microbatches(self, b, m):
        out = np.zeros(max(m, 1), np.int32)
        err = C.create_string_buffer(512)
        rc = self._fn("split_microbatches")(b, m, _ip(out), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        return [int(x) for x in out]

    def build_plan(self, dims, n, Z, replicate=False):
        fi = np.asarray(dims[:-1], np.int32)
        fo = np.asarray(dims[1:], np.int32)
        L = len(fo)
        ln = C.c_int(0)
        err = C.create_string_buffer(512)
        f = self._fn("build_plan")
        rc = f(_ip(fi), _ip(fo), None, L, n, Z, int(replicate), None, 0, C.byref(ln), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        out = np.zeros(ln.value, np.int32)
        rc = f(_ip(fi), _ip(fo), None, L, n, Z, int(replicate), _ip(out), ln.value, C.byref(ln), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        return out

    def build_staged_plan(self, dims, groups, replicate=False):
        fi = np.asarray(dims[:-1], np.int32)
        fo = np.asarray(dims[1:], np.int32)
        flat = np.asarray([d for g in groups for d in g], np.int32)
        sizes = np.asarray([len(g) for g in groups], np.int32)
        ln = C.c_int(0)
        err = C.create_string_buffer(512)
        f = self._fn("build_staged_plan")
        args = (_ip(fi), _ip(fo), None, len(fo), _ip(flat), _ip(sizes), len(groups), int(replicate))
        rc = f(*args, None, 0, C.byref(ln), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        out = np.zeros(ln.value, np.int32)
        rc = f(*args, _ip(out), ln.value, C.byref(ln), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        return out

    def merge_submodules(self, plan, group):
        p = np.array(plan, np.int32)
        g = np.asarray(group, np.int32)
        err = C.create_string_buffer(512)
        rc = self._fn("merge_submodules")(_ip(p), len(p), _ip(g), len(g), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        return p

    # numerics ----------------------------------------------------------
    def init_net(self, dims, seed):
        dims = np.asarray(dims, np.int32)
        L = len(dims) - 1
        W = np.zeros(int(sum(dims[l] * dims[l + 1] for l in range(L))), np.float64)
        b = np.zeros(int(sum(dims[1:])), np.float64)
        self._fn("init_net")(_ip(dims), L, C.c_uint64(seed), _dp(W), _dp(b))
        return W, b

    def make_blobs(self, samples, features, separation, seed):
        X = np.zeros(samples * features, np.float64)
        y = np.zeros(samples, np.int32)
        self._fn("make_blobs")(samples, features, C.c_double(separation), C.c_uint64(seed), _dp(X), _ip(y))
        return X.reshape(samples, features), y

    def forward(self, dims, acts, W, b, X):
        dims = np.asarray(dims, np.int32)
        acts = np.asarray(acts, np.int32)
        batch = X.shape[0]
        out = np.zeros(batch * int(sum(dims[1:])), np.float64)
        err = C.create_string_buffer(512)
        Xc = np.ascontiguousarray(X, np.float64)
        rc = self._fn("forward")(_ip(dims), _ip(acts), len(acts), _dp(W), _dp(b), _dp(Xc), batch, _dp(out), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        res, off = [], 0
        for l in range(1, len(dims)):
            res.append(out[off: off + batch * dims[l]].reshape(batch, dims[l]))
            off += batch * dims[l]
        return res

    def train_sequential(self, dims, acts, W, b, X, labels, alpha0, decay, loss, iterations, multiclass=False):
        return self._train("train_sequential", dims, acts, W, b, X, labels, None, None, None,
                           alpha0, decay, loss, iterations, multiclass)

    def train_partitioned(self, dims, acts, W, b, X, labels, plan, m, mode, alpha0, decay, loss, iterations,
                          multiclass=False):
        return self._train("train_partitioned", dims, acts, W, b, X, labels, plan, m, mode,
                           alpha0, decay, loss, iterations, multiclass)

    def _train(self, name, dims, acts, W, b, X, labels, plan, m, mode, alpha0, decay, loss, iterations,
               multiclass):
        dims = np.asarray(dims, np.int32)
        acts = np.asarray(acts, np.int32)
        W = np.ascontiguousarray(W, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        Xc = np.ascontiguousarray(X, np.float64)
        y = np.ascontiguousarray(labels, np.int32)
        Wo = np.zeros_like(W)
        bo = np.zeros_like(b)
        lh = np.zeros(max(iterations, 1), np.float64)
        ah = np.zeros(max(iterations, 1), np.float64)
        err = C.create_string_buffer(512)
        f = self._fn(name)
        if plan is None:
            rc = f(_ip(dims), _ip(acts), len(acts), _dp(W), _dp(b), _dp(Xc), _ip(y), Xc.shape[0],
                   C.c_double(alpha0), C.c_double(decay), loss, iterations, int(multiclass),
                   _dp(Wo), _dp(bo), _dp(lh), _dp(ah), err, 512)
        else:
            p = np.ascontiguousarray(plan, np.int32)
            rc = f(_ip(dims), _ip(acts), len(acts), _dp(W), _dp(b), _dp(Xc), _ip(y), Xc.shape[0],
                   _ip(p), len(p), m, mode, C.c_double(alpha0), C.c_double(decay), loss, iterations,
                   int(multiclass), _dp(Wo), _dp(bo), _dp(lh), _dp(ah), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        return Wo, bo, lh[:iterations], ah[:iterations]


class Reference(_Base):
    """The compiled reference (ref_* functions of ref_shim.cpp)."""

    prefix = "ref_"

    def __init__(self, path=REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        super().__init__(path)

    def init_net(self, dims, acts, seed):
        dims = np.asarray(dims, np.int32)
        acts = np.asarray(acts, np.int32)
        L = len(acts)
        W = np.zeros(int(sum(dims[l] * dims[l + 1] for l in range(L))), np.float64)
        b = np.zeros(int(sum(dims[1:])), np.float64)
        self._fn("init_net")(_ip(dims), _ip(acts), L, C.c_uint64(seed), _dp(W), _dp(b))
        return W, b

    def make_blobs(self, samples, features, separation, seed):
        X = np.zeros(samples * features, np.float64)
        y = np.zeros(samples, np.int32)
        self._fn("make_blobs")(samples, features, C.c_double(separation), C.c_uint64(seed), _dp(X), _ip(y))
        return X.reshape(samples, features), y

    def split_layer(self, fan_out, n, replicate=False, layer_id=1):
        devs = np.arange(1, n + 1, dtype=np.int32)
        lo = np.zeros(n, np.int32)
        hi = np.zeros(n, np.int32)
        rep = np.zeros(n, np.int32)
        err = C.create_string_buffer(512)
        rc = self._fn("split_layer")(layer_id, fan_out, _ip(devs), n, int(replicate), _ip(lo), _ip(hi),
                                     _ip(rep), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        return [(int(a), int(b), bool(c)) for a, b, c in zip(lo, hi, rep)]

    def split_microbatches(self, b, m):
        out = np.zeros(max(m, 1), np.int32)
        err = C.create_string_buffer(512)
        rc = self._fn("split_microbatches")(b, m, _ip(out), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        return [int(x) for x in out]

    def build_plan(self, dims, n, Z, replicate=False):
        fi = np.asarray(dims[:-1], np.int32)
        fo = np.asarray(dims[1:], np.int32)
        ln = C.c_int(0)
        err = C.create_string_buffer(512)
        f = self._fn("build_plan")
        rc = f(_ip(fi), _ip(fo), len(fo), n, Z, int(replicate), None, 0, C.byref(ln), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        out = np.zeros(ln.value, np.int32)
        rc = f(_ip(fi), _ip(fo), len(fo), n, Z, int(replicate), _ip(out), ln.value, C.byref(ln), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        return out

    def build_staged_plan(self, dims, groups, replicate=False):
        fi = np.asarray(dims[:-1], np.int32)
        fo = np.asarray(dims[1:], np.int32)
        flat = np.asarray([d for g in groups for d in g], np.int32)
        sizes = np.asarray([len(g) for g in groups], np.int32)
        ln = C.c_int(0)
        err = C.create_string_buffer(512)
        f = self._fn("build_staged_plan")
        args = (_ip(fi), _ip(fo), len(fo), _ip(flat), _ip(sizes), len(groups), int(replicate))
        rc = f(*args, None, 0, C.byref(ln), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        out = np.zeros(ln.value, np.int32)
        rc = f(*args, _ip(out), ln.value, C.byref(ln), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        return out

    def merge_submodules(self, plan, group):
        p = np.array(plan, np.int32)
        g = np.asarray(group, np.int32)
        err = C.create_string_buffer(512)
        rc = self._fn("merge_submodules")(_ip(p), len(p), _ip(g), len(g), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        return p

    def forward(self, dims, acts, W, b, X):
        dims = np.asarray(dims, np.int32)
        acts = np.asarray(acts, np.int32)
        batch = X.shape[0]
        out = np.zeros(batch * int(sum(dims[1:])), np.float64)
        err = C.create_string_buffer(512)
        Xc = np.ascontiguousarray(X, np.float64)
        rc = self._fn("forward")(_ip(dims), _ip(acts), len(acts), _dp(W), _dp(b), _dp(Xc), batch, _dp(out),
                                 err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        res, off = [], 0
        for l in range(1, len(dims)):
            res.append(out[off: off + batch * dims[l]].reshape(batch, dims[l]))
            off += batch * dims[l]
        return res

    def train_sequential(self, dims, acts, W, b, X, labels, alpha0, decay, loss, iterations):
        dims = np.asarray(dims, np.int32)
        acts = np.asarray(acts, np.int32)
        W = np.ascontiguousarray(W, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        Xc = np.ascontiguousarray(X, np.float64)
        y = np.ascontiguousarray(labels, np.int32)
        Wo, bo = np.zeros_like(W), np.zeros_like(b)
        lh = np.zeros(iterations, np.float64)
        ah = np.zeros(iterations, np.float64)
        err = C.create_string_buffer(512)
        rc = self._fn("train_sequential")(_ip(dims), _ip(acts), len(acts), _dp(W), _dp(b), _dp(Xc), _ip(y),
                                          Xc.shape[0], C.c_double(alpha0), C.c_double(decay), loss,
                                          iterations, _dp(Wo), _dp(bo), _dp(lh), _dp(ah), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        return Wo, bo, lh, ah

    def train_partitioned(self, dims, acts, W, b, X, labels, plan, m, mode, alpha0, decay, loss, iterations,
                          timeout_s=600.0):
        dims = np.asarray(dims, np.int32)
        acts = np.asarray(acts, np.int32)
        W = np.ascontiguousarray(W, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        Xc = np.ascontiguousarray(X, np.float64)
        y = np.ascontiguousarray(labels, np.int32)
        p = np.ascontiguousarray(plan, np.int32)
        Wo, bo = np.zeros_like(W), np.zeros_like(b)
        lh = np.zeros(iterations, np.float64)
        ah = np.zeros(iterations, np.float64)
        err = C.create_string_buffer(512)
        rc = self._fn("train_partitioned")(_ip(dims), _ip(acts), len(acts), _dp(W), _dp(b), _dp(Xc), _ip(y),
                                           Xc.shape[0], _ip(p), len(p), m, mode, C.c_double(alpha0),
                                           C.c_double(decay), loss, iterations, C.c_double(timeout_s),
                                           _dp(Wo), _dp(bo), _dp(lh), _dp(ah), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        return Wo, bo, lh, ah

    def draw_instance(self, seed):
        L = C.c_int()
        dims = np.zeros(9, np.int32)
        acts = np.zeros(8, np.int32)
        n, m, batch, loss, iters, plen = (C.c_int() for _ in range(6))
        a0, dec = C.c_double(), C.c_double()
        plan = np.zeros(4096, np.int32)
        W = np.zeros(4096, np.float64)
        b = np.zeros(64, np.float64)
        X = np.zeros(256, np.float64)
        y = np.zeros(64, np.int32)
        self._fn("draw_instance")(C.c_uint64(seed), C.byref(L), _ip(dims), _ip(acts), C.byref(n), C.byref(m),
                                  C.byref(batch), C.byref(loss), C.byref(a0), C.byref(dec), C.byref(iters),
                                  _ip(plan), C.byref(plen), _dp(W), _dp(b), _dp(X), _ip(y))
        Lv = L.value
        d = [int(x) for x in dims[: Lv + 1]]
        nw = sum(d[l] * d[l + 1] for l in range(Lv))
        return dict(dims=d, acts=[int(x) for x in acts[:Lv]], n=n.value, m=m.value, batch=batch.value,
                    loss=loss.value, alpha0=a0.value, decay=dec.value, iterations=iters.value,
                    plan=plan[: plen.value].copy(), W=W[:nw].copy(), b=b[: sum(d[1:])].copy(),
                    X=X[: batch.value * d[0]].reshape(batch.value, d[0]).copy(), labels=y[: batch.value].copy())

    def serialize_plan(self, plan, provenance=()):
        p = np.ascontiguousarray(plan, np.int32)
        n = C.c_size_t(0)
        err = C.create_string_buffer(512)
        prov = "\n".join(provenance).encode()
        f = self._fn("serialize_plan")
        rc = f(_ip(p), len(p), prov, None, 0, C.byref(n), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        buf = C.create_string_buffer(n.value + 1)
        rc = f(_ip(p), len(p), prov, buf, n.value + 1, C.byref(n), err, 512)
        return buf.value.decode()

    def parse_plan(self, text):
        n = C.c_int(0)
        err = C.create_string_buffer(512)
        f = self._fn("parse_plan")
        rc = f(text.encode(), None, 0, C.byref(n), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        out = np.zeros(n.value, np.int32)
        f(text.encode(), _ip(out), n.value, C.byref(n), err, 512)
        return out

    def run_verification(self, seeds=100):
        buf = C.create_string_buffer(8192)
        ok = self._fn("run_verification")(seeds, buf, 8192)
        return bool(ok), buf.value.decode()
