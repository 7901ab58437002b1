"""C-ABI library: loads, exports every symbol include/hc.h declares, and its host-side
allocator matches the reference pool semantics (accounting-only pools: no device work,
so this runs on the CPU box)."""
import ctypes
import os
import random
import re

import pytest

from oracle.pool_oracle import PoolOracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def hc():
    from paper_2504_07494_b200 import build
    build.build()
    from paper_2504_07494_b200 import hc as m
    return m


def test_exports_every_declared_symbol(hc):
    hdr = open(os.path.join(ROOT, "include", "hc.h")).read()
    declared = set(re.findall(r"^(?:const\s+)?[a-z_0-9]+\s*\*?\s+(hc_[a-z_0-9]+)\(", hdr, re.M))
    assert {"hc_pool_create", "hc_append", "hc_decode_attention"} <= declared
    lib = ctypes.CDLL(hc.LIB_PATH)
    for name in sorted(declared):
        assert hasattr(lib, name), f"{name} declared in hc.h but not exported"
    assert b"sm_100a" in hc.lib.hc_version()


def _acct_pool(hc, num_blocks, B, d=32, H=2):
    return hc.HybridCachePool(d, H, d // H, B, num_blocks, hc.HC_F32, flags=hc.HC_FLAG_ACCOUNTING_ONLY)


def _tables_equal(pool, orc, rid):
    mode, n, units = pool.request_info(rid)
    t = orc.table(rid)
    if mode == 0:
        return pool.request_blocks(rid, 0) == t[0] and pool.request_blocks(rid, 1) == t[1] and n == orc.req[rid]["n"]
    return pool.request_blocks(rid, 0) == t[0] and pool.request_blocks(rid, 1) == [] and n == orc.req[rid]["n"]


def test_fig6_through_the_abi(hc):
    """Fig. 6: 16 blocks, B=4: A (KV, 11 tok) -> 6 units, B (hidden, 14) -> 4."""
    p = _acct_pool(hc, 16, 4)
    o = PoolOracle(16, 4)
    p.append([0], [0], [11])
    o.append([0], [0], [11])
    p.append([1], [1], [14])
    o.append([1], [1], [14])
    assert p.request_info(0)[2] == 6 and p.request_info(1)[2] == 4 and p.num_free() == 6
    assert _tables_equal(p, o, 0) and _tables_equal(p, o, 1)
    assert p.free(0) == 6 and p.free(0) == 0 and p.num_free() == 12


def test_error_codes(hc):
    p = _acct_pool(hc, 5, 4)
    p.append([1], [1], [16])
    with pytest.raises(hc.HcError) as e:
        p.append([2], [0], [1])                     # KV needs 2 blocks, 1 free
    assert e.value.status == hc.HC_E_OOM and p.num_free() == 1
    with pytest.raises(hc.HcError) as e:
        p.append([1], [0], [1])
    assert e.value.status == hc.HC_E_MODE_MISMATCH
    with pytest.raises(hc.HcError) as e:
        p.append([3, 3], [1, 1], [1, 1])
    assert e.value.status == hc.HC_E_INVALID
    with pytest.raises(hc.HcError) as e:
        p.request_info(99)
    assert e.value.status == hc.HC_E_UNKNOWN_REQ
    with pytest.raises(hc.HcError) as e:
        p.append([4, 5], [1, 1], [4, 4])            # batch OOM is all-or-nothing
    assert e.value.status == hc.HC_E_OOM and p.num_free() == 1
    with pytest.raises(hc.HcError):
        hc.HybridCachePool(30, 4, 8, 4, 8, hc.HC_F32, flags=hc.HC_FLAG_ACCOUNTING_ONLY)  # d != H*dh
    with pytest.raises(hc.HcError) as e:
        hc.hc_decode_attention(p.handle, [1], None, 1.0, None, None, None, stream=0)
    assert e.value.status == hc.HC_E_UNSUPPORTED


def test_fuzz_against_pool_oracle(hc):
    """10^3 random append/free sequences: block ids, lengths and free counts bit-exact."""
    rs = random.Random(1)
    p = _acct_pool(hc, 61, 4)
    o = PoolOracle(61, 4)
    for _ in range(1000):
        if rs.random() < 0.65:
            ids = rs.sample(range(20), rs.randint(1, 3))
            modes = [o.req[i]["mode"] if i in o.req else rs.randint(0, 1) for i in ids]
            toks = [rs.randint(0, 9) for _ in ids]
            want = o.append(ids, modes, toks)
            try:
                p.append(ids, modes, toks)
                got = "ok"
            except hc.HcError as e:
                got = {hc.HC_E_OOM: "oom"}.get(e.status, "err")
            assert got == want
        else:
            r = rs.randrange(20)
            assert p.free(r) == o.free_req(r)
        assert p.num_free() == o.num_free()
        for rid in o.req:
            assert _tables_equal(p, o, rid)


def test_storage_bytes_and_workspace_queries(hc):
    cfg = hc.PoolConfig(9216, 72, 128, 16, 1000, hc.HC_BF16, 0, None, 0, None, None, 0, 0)
    n = hc.hc_pool_storage_bytes(cfg)
    blocks = 1000 * 16 * 9216 * 2
    assert n >= blocks + 2 * 9216 * 9216 * 2 and n < blocks + 2 * 9216 * 9216 * 2 + (8 << 20)
    bad = hc.PoolConfig(100, 3, 33, 16, 10, hc.HC_BF16, 0, None, 0, None, None, 0, 0)
    assert hc.hc_pool_storage_bytes(bad) == 0
    p = _acct_pool(hc, 64, 4)
    p.append([5, 6], [0, 1], [9, 3])
    assert p.workspace_size([5, 6]) > 0
    with pytest.raises(hc.HcError):
        p.workspace_size([5, 5])


def test_units_needed_matches_the_pool_contract(hc):
    """hc_units_needed (used to size every pool) follows SPEC S:58-66 / Fig. 6: KV takes
    a K and a V unit per B tokens, hidden one unit; and it agrees with what hc_append allocates."""
    from oracle.pool_oracle import blocks_needed
    for B in (1, 4, 16, 64):
        for n in (0, 1, B - 1, B, B + 1, 11, 14, 1000):
            for mode in (0, 1):
                assert hc.units_needed(32, 2, 16, B, mode, n) == blocks_needed(n, mode, B)
    assert hc.units_needed(32, 2, 16, 4, 0, 11) == 6 and hc.units_needed(32, 2, 16, 4, 1, 14) == 4   # Fig. 6
    p = _acct_pool(hc, 64, 4)
    p.append([0, 1], [0, 1], [11, 14])
    assert p.request_info(0)[2] == hc.units_needed(32, 2, 16, 4, 0, 11)
    with pytest.raises(hc.HcError):
        hc.units_needed(32, 2, 16, 4, 2, 5)


def test_gqa_unit_accounting(hc):
    """GQA (R18): a KV token holds 2 Hk dh values, so one unit stores K and V of Bkv = B d/(2 Hk dh)
    tokens; hidden stays one unit per B tokens.  LLaMA-3-8B (d 4096, 32/8 heads): KV needs half
    the units of hidden; invalid groupings are refused."""
    d, H, dh, B = 4096, 32, 128, 16
    assert hc.units_needed(d, H, dh, B, 0, 100, n_kv_heads=8) == -(-100 // 32)
    assert hc.units_needed(d, H, dh, B, 1, 100, n_kv_heads=8) == -(-100 // 16)
    assert hc.units_needed(d, H, dh, B, 0, 100, n_kv_heads=4) == -(-100 // 64)
    assert hc.units_needed(d, H, dh, B, 0, 100, n_kv_heads=32) == 2 * -(-100 // 16)   # = multi-head
    with pytest.raises(hc.HcError):
        hc.units_needed(d, H, dh, B, 0, 100, n_kv_heads=5)     # H % Hk != 0
    assert hc.units_needed(d, H, dh, B, 0, 100, n_kv_heads=16) == -(-100 // 16)   # G = 2: K+V fill a unit
    with pytest.raises(hc.HcError):
        hc.units_needed(384, 6, 64, B, 0, 100, n_kv_heads=2)   # d % (2 Hk dh) != 0
    p = hc.HybridCachePool(d, H, dh, B, 64, hc.HC_BF16, flags=hc.HC_FLAG_ACCOUNTING_ONLY, n_kv_heads=8)
    p.append([0, 1], [0, 1], [33, 33])
    assert p.request_info(0)[2] == 2 and p.request_info(1)[2] == 3
    assert p.request_blocks(0, 0) == [0, 1] and p.request_blocks(0, 1) == [] and p.request_blocks(1, 0) == [2, 3, 4]
