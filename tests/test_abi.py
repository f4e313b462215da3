"""The C-ABI boundary: the library loads and exports every symbol the header
declares; argument validation mirrors the reference's std::invalid_argument
conditions. No compute calls here (CPU-only)."""
import ctypes
import subprocess

import pytest

import paper_2603_13358_b200 as ppd


def test_header_symbols_exported():
    names = ppd.header_symbols()
    assert len(names) >= 15
    L = ppd.lib()
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", ppd.LIB_PATH], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    assert set(names) <= exported


def test_no_torch_in_abi_header():
    text = open(ppd.HEADER_PATH).read()
    assert "torch" not in text.lower().replace("no torch types", "")
    assert 'extern "C"' in text


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", ppd.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_kv_block_bytes_llama8b():
    # 32 layers x (K,V) x 8 kv heads x 16 tokens x 128 dims x 2 B = 2 MiB
    assert ppd.kv_block_bytes(ppd.llama8b_cfg()) == 2 * 1024 * 1024
    # per token: 131072 B (Llama-3-8B KV = 131,072 B/token)
    assert ppd.kv_block_bytes(ppd.llama8b_cfg()) // 16 == 131072
    assert ppd.kv_block_bytes(ppd.qwen32b_cfg()) // 16 == 262144


def test_invalid_cfg_rejected():
    bad = ppd.tiny_cfg()
    bad.head_dim = 64
    with pytest.raises(ppd.InvalidArgument):
        ppd.kv_block_bytes(bad)
    with pytest.raises(ppd.InvalidArgument):
        ppd.kv_block_bytes(ppd.tiny_cfg(), 32)


def test_version():
    assert ppd.lib().ppd_version() == 1
