"""CPU-side checks of the C ABI (-m "not gpu"): the library loads, exports every symbol that
include/l2f.h declares, and validates configs without touching a GPU."""
import ctypes as C
import os
import re
import subprocess

import pytest

import inputs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2311_13081_b200 import _build
    _build.build()
    import paper_2311_13081_b200 as pkg
    return pkg.lib()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "l2f.h")).read()
    return sorted(set(re.findall(r"L2F_API\s+[\w\s\*]+?\b(l2f_\w+)\s*\(", src)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for need in ("l2f_create", "l2f_reset", "l2f_step", "l2f_rollout", "l2f_episode_stats"):
        assert need in syms
    assert len(syms) >= 15


def test_library_exports_every_declared_symbol(L):
    from paper_2311_13081_b200.abi import EXPORTS, LIB_PATH
    out = subprocess.run(["nm", "-D", "--defined-only", LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (l2f_\w+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    assert sorted(EXPORTS) == declared_symbols()
    for s in declared_symbols():
        assert hasattr(L, s)


def test_library_is_sm100a(L):
    from paper_2311_13081_b200.abi import LIB_PATH
    out = subprocess.run(["cuobjdump", "--list-elf", LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_abi_version(L):
    from paper_2311_13081_b200.abi import ABI_VERSION
    assert L.l2f_abi_version() == ABI_VERSION == 2


def _size(L, cfg, n, off=0):
    from paper_2311_13081_b200.abi import make_config
    c = make_config(cfg, n, off)
    b = C.c_size_t()
    st = L.l2f_workspace_size(C.byref(c), C.byref(b))
    return st, b.value, L.l2f_last_error().decode()


def test_workspace_size_and_validation(L):
    cfg = inputs.config_c3()
    n = 1 << 20
    st, b, _ = _size(L, cfg, n)
    assert st == 0
    # state 68 + dist 24 + dr 20 + hist 512 + fill 16 + counters 12 + staging
    # (16 + 72 + 4 + 1) B per env
    assert 740 * n <= b <= 770 * n
    assert _size(L, cfg, 0)[0] == 1
    assert _size(L, cfg, 10, off=(1 << 32) - 5)[0] == 1
    assert _size(L, inputs.config_c3(n_hist=33), 10)[0] == 1
    assert _size(L, inputs.config_c3(dt=0.0), 10)[0] == 1
    bad = inputs.config_c3()
    bad["params"] = dict(bad["params"], rpm_max=1000.0)  # hover infeasible
    st, _, msg = _size(L, bad, 10)
    assert st == 1 and "hover" in msg
    st, _, msg = _size(L, inputs.config_c3(dr_range=[0.8, 2.5]), 10)  # infeasible at the worst DR corner
    assert st == 1 and "hover" in msg


def test_create_rejects_host_memory(L):
    from paper_2311_13081_b200.abi import make_config
    c = make_config(inputs.config_c1(), 64)
    h = C.c_void_p()
    buf = (C.c_uint8 * (1 << 20))()
    addr = (C.addressof(buf) + 255) & ~255
    st = L.l2f_create(C.byref(c), C.c_void_p(addr), 1 << 19, C.byref(h))
    assert st != 0


def test_td3_sizes_and_validation(L):
    """l2f_td3_sizes is host-only: the parameter block is 4 actor-sized + 8 critic-sized nets
    (nets, targets, Adam moments; include/l2f.h), bounds on batch and in_dim are enforced."""
    blk, sb = C.c_int64(), C.c_int64()
    assert L.l2f_td3_sizes(146, 256, C.byref(blk), C.byref(sb)) == 0
    net = lambda i, o: 64 * i + 64 + 64 * 64 + 64 + o * 64 + o  # noqa: E731
    assert blk.value == 4 * net(146, 4) + 8 * net(32, 1)
    assert sb.value % 256 == 0 and sb.value >= 4 * (256 * 554 + 2 * net(32, 1) + net(146, 4))
    assert L.l2f_td3_sizes(156, 1, C.byref(blk), C.byref(sb)) == 0
    for bad in ((157, 256), (0, 256), (146, 0), (146, 257)):
        assert L.l2f_td3_sizes(bad[0], bad[1], C.byref(blk), C.byref(sb)) == 1, bad


def test_td3_update_validates_before_touching_the_gpu(L):
    """NULL buffers, zero agents, Adam step 0 and out-of-range hyper-parameters are rejected on
    the host (INVALID_ARGUMENT) -- no device call is made, so this runs without a GPU."""
    from paper_2311_13081_b200.abi import TD3Batch, TD3Hyper
    h = TD3Hyper(gamma=0.99, tau=0.005, sigma_t=0.2, clip_t=0.5, lr_actor=3e-4, lr_critic=3e-4, beta1=0.9,
                 beta2=0.999, eps=1e-8)
    fake = C.c_void_p(0x1000)
    b = TD3Batch(*([0x1000] * 8))

    def call(params=fake, n=4, in_dim=146, batch=256, batch_s=b, hyper=h, tc=1, ta=1, upd=1):
        return L.l2f_td3_update(params, n, in_dim, batch, C.byref(batch_s), C.byref(hyper), tc, ta, upd, fake, fake,
                                None)

    assert call(params=None) == 1
    assert call(n=0) == 1
    assert call(in_dim=157) == 1
    assert call(tc=0) == 1
    assert call(ta=0, upd=1) == 1
    bad = TD3Batch(*([0x1000] * 7 + [None]))
    assert call(batch_s=bad) == 1
    for k, v in (("gamma", 1.5), ("tau", -0.1), ("beta1", 1.0), ("eps", 0.0)):
        hh = TD3Hyper(**{f: getattr(h, f) for f, _ in TD3Hyper._fields_})
        setattr(hh, k, v)
        assert call(hyper=hh) == 1, k
