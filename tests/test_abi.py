"""CPU checks of the boundary: the C-ABI library builds, loads and exports every
function declared in include/*.h; without a GPU it refuses to run (no CPU fallback)."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    names = []
    for h in ("rt.h", "rt_ops.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names += re.findall(r"^\s*(?:rt_status|const char\*|int64_t)\s+(rt_\w+)\s*\(", src, flags=re.M)
    return sorted(set(names))


@pytest.fixture(scope="module")
def built():
    from paper_2412_18695_b200.build import build
    return build()


def test_library_exports_every_declared_symbol(built):
    import ctypes
    lib = ctypes.CDLL(built)
    decl = declared_functions()
    assert len(decl) >= 20
    missing = [n for n in decl if not hasattr(lib, n)]
    assert missing == []
    from paper_2412_18695_b200 import rt
    assert sorted(rt.EXPORTED) == decl


def test_sass_is_blackwell_native(built):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", built], capture_output=True, text=True).stdout
    assert "UTCHMMA" in out          # tcgen05.mma
    assert "UTMALDG" in out          # TMA tensor loads
    assert "UBLKCP" in out           # bulk copies of KV pages
    assert "LDTM" in out             # tcgen05.ld from TMEM
    assert "arch = sm_100a" in out or "sm_100a" in out


def test_no_cpu_fallback(built, tiny_vocab):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2412_18695_b200 import rt
    from synth import engine_params
    with pytest.raises(rt.RtError) as ex:
        rt.Engine(None, engine_params(), tiny_vocab)
    assert ex.value.code == rt.RT_E_CUDA


def test_config_validation_before_device(built, tiny_vocab):
    from paper_2412_18695_b200 import rt
    from synth import engine_params
    with pytest.raises(rt.RtError) as ex:
        rt.Engine(None, engine_params(max_seg_tokens=40), tiny_vocab)   # > 16 record slots
    assert ex.value.code == rt.RT_E_INVAL


def test_struct_layouts_match_header(tmp_path):
    """ctypes mirrors of the ABI structs have the C compiler's size and offsets."""
    import ctypes as C
    import subprocess
    from paper_2412_18695_b200 import rt
    structs = {"rt_config": rt.rt_config, "rt_segment": rt.rt_segment, "rt_round_info": rt.rt_round_info,
               "rt_stats": rt.rt_stats, "rt_utility": rt.rt_utility}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "rt.h"', "int main(void){"]
    for name, cls in structs.items():
        lines.append(f'printf("{name} %zu\\n", sizeof({name}));')
        for f, _ in cls._fields_:
            lines.append(f'printf("{name}.{f} %zu\\n", offsetof({name}, {f}));')
    lines.append('printf("rt_trace_rec %zu\\n", sizeof(rt_trace_rec));')
    for f in rt.TRACE_DTYPE.names:
        lines.append(f'printf("rt_trace_rec.{f} %zu\\n", offsetof(rt_trace_rec, {f}));')
    lines.append("return 0;}")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = dict(l.split() for l in subprocess.run([str(exe)], capture_output=True, text=True).stdout.splitlines())
    for name, cls in structs.items():
        assert int(got[name]) == C.sizeof(cls), name
        for f, _ in cls._fields_:
            assert int(got[f"{name}.{f}"]) == getattr(cls, f).offset, (name, f)
    assert int(got["rt_trace_rec"]) == rt.TRACE_DTYPE.itemsize == 48
    for f in rt.TRACE_DTYPE.names:
        assert int(got[f"rt_trace_rec.{f}"]) == rt.TRACE_DTYPE.fields[f][1], f
