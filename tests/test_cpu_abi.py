"""The C-ABI library loads without a GPU and exports every symbol the header
declares; the host-side deterministic-sum planner reproduces np.sum bit for
bit (evaluated here exactly as the kernels evaluate it)."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2502_09758_b200 import _native as nat

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "adp_b200.h")).read()
    return sorted(set(re.findall(r"^(?:int|void|size_t|const char\*)\s+(adp_\w+)\s*\(", src, re.M)))


def test_library_exports_every_header_symbol():
    lib = nat.load_library()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
        assert s in nat.SIGNATURES, f"{s} not bound in _native.SIGNATURES"


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    with pytest.raises(nat.NativeError):
        nat.lib()


def layout(n, np_rule=True):
    lib = nat.load_library()
    nl, ns, top, nw = ctypes.c_int64(), ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int64()
    cap = n // 64 + 64
    leaf = np.zeros(cap + 2, np.int64)
    sub_leaf = np.zeros(cap + 2, np.int32)
    sub_prog = np.zeros(cap + 2, np.int32)
    words = np.zeros(64 * cap + 4096, np.int32)
    rc = lib.adp_sum_layout(n, 1 if np_rule else 0, ctypes.byref(nl), ctypes.byref(ns), ctypes.byref(top),
                            leaf.ctypes.data, leaf.size, sub_leaf.ctypes.data, sub_prog.ctypes.data, sub_prog.size,
                            words.ctypes.data, words.size, ctypes.byref(nw))
    assert rc == 0
    return nl.value, ns.value, top.value, leaf, sub_leaf, sub_prog, words


def np_leaf(a):
    n = len(a)
    if n < 8:
        r = 0.0
        for v in a:
            r = r + v
        return r
    r = list(a[:8])
    i = 8
    while i < n - n % 8:
        for k in range(8):
            r[k] = r[k] + a[i + k]
        i += 8
    res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
    while i < n:
        res = res + a[i]
        i += 1
    return res


def perfect(vals):
    """Perfect binary tree over vals zero-padded to a power of two."""
    v = list(vals)
    p = 1
    while p < len(v):
        p *= 2
    v += [0.0] * (p - len(v))
    while len(v) > 1:
        v = [v[2 * i] + v[2 * i + 1] for i in range(len(v) // 2)]
    return v[0]


def eval_prog(words, off, vals):
    nL, nI, nLev = words[off], words[off + 1], words[off + 2]
    lev = words[off + 3: off + 4 + nLev]
    left = words[off + 4 + nLev: off + 4 + nLev + nI]
    right = words[off + 4 + nLev + nI: off + 4 + nLev + 2 * nI]
    sv = list(vals) + [0.0] * nI
    assert len(vals) == nL
    for lv in range(nLev):
        for k in range(lev[lv], lev[lv + 1]):
            sv[nL + k] = sv[left[k]] + sv[right[k]]
    return sv[nL + nI - 1] if nI else sv[0]


@pytest.mark.parametrize("n", [1, 7, 8, 128, 129, 1000, 65536, 90000, 131072, 786432, 1572864, 300001])
def test_sum_layout_reproduces_np_sum(n):
    rng = np.random.default_rng(n)
    a = (rng.standard_normal(n) * np.exp(3 * rng.standard_normal(n))).astype(np.float64)
    nl, ns, top, leaf, sub_leaf, sub_prog, words = layout(n)
    leaves = [np_leaf(a[leaf[i]:leaf[i + 1]]) for i in range(nl)]
    if top == -1:   # regular: perfect tree, device evaluates it in registers / shuffles
        if ns == 1:
            s = perfect(leaves)
        else:
            s = perfect([perfect(leaves[sub_leaf[t]:sub_leaf[t + 1]]) for t in range(ns)])
    elif ns == 1:
        s = eval_prog(words, top, leaves)
    else:
        roots = [eval_prog(words, sub_prog[t], leaves[sub_leaf[t]:sub_leaf[t + 1]]) for t in range(ns)]
        s = eval_prog(words, top, roots)
    assert s == np.sum(a)


def test_sum_layout_binary_tile_tree():
    nl, ns, top, leaf, sub_leaf, sub_prog, words = layout(5000, np_rule=False)
    assert nl == 5000 and ns == 3 and top == -1
    vals = np.arange(5000, dtype=float)
    assert perfect([perfect(vals[sub_leaf[t]:sub_leaf[t + 1]]) for t in range(ns)]) == vals.sum()


def test_host_fingerprint_sees_edits():
    """Device-copy caches of host arrays (problems.UpperProblem.lower_problem,
    hypergradient._cached_dev) key on identity + a sampled fingerprint."""
    import numpy as np
    from paper_2502_09758_b200 import _native as nat
    y = np.random.default_rng(0).standard_normal((64, 48, 3))
    f0 = nat.host_fingerprint(y)
    assert nat.host_fingerprint(y) == f0
    y *= 2.0
    assert nat.host_fingerprint(y) != f0
    f1 = nat.host_fingerprint(y)
    y[:] = 0.5
    assert nat.host_fingerprint(y) != f1
    assert nat.host_fingerprint(y.copy()) != nat.host_fingerprint(y)   # a new object (address) re-uploads
