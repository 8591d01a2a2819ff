"""ctypes binding of libhapigpu.so (include/hapigpu.h).

The library is built in-tree by `__graft_entry__.build()` (nvcc, sm_100a).
There is no fallback: if the library or a CUDA device is missing, every entry
point raises EngineError.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

from .errors import EngineError

HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ["HAPIGPU_LIB"]) if os.environ.get("HAPIGPU_LIB") else HERE / "libhapigpu.so"
CSRC = HERE / "csrc"
INCLUDE = HERE.parent / "include"

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
    "--expt-relaxed-constexpr",
]


def sources():
    """One translation unit per kernel family (ctx.h): they compile in parallel."""
    return [CSRC / "engine.cu", CSRC / "fast.cu", CSRC / "seg.cu", CSRC / "timeline.cu", CSRC / "merge.cu", CSRC / "ingest.cu", CSRC / "events.cu", CSRC / "validate.cu", CSRC / "tldist.cu"]


def build(force: bool = False, verbose: bool = False) -> Path:
    from concurrent.futures import ThreadPoolExecutor

    headers = [INCLUDE / "hapigpu.h"] + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h"))
    newest_h = max(p.stat().st_mtime for p in headers if p.exists())
    nvcc = os.environ.get("NVCC", "nvcc")
    objdir = HERE / "build"
    objdir.mkdir(exist_ok=True)
    objs, jobs = [], []
    for src in sources():
        obj = objdir / (src.stem + ".o")
        objs.append(obj)
        if force or not obj.exists() or obj.stat().st_mtime < max(newest_h, src.stat().st_mtime):
            jobs.append([nvcc, *NVCC_FLAGS, "-I", str(INCLUDE), "-c", "-o", str(obj), str(src)])
    if not jobs and LIB_PATH.exists() and LIB_PATH.stat().st_mtime >= max(o.stat().st_mtime for o in objs):
        return LIB_PATH

    def run(cmd):
        if verbose:
            print(" ".join(cmd))
        subprocess.check_call(cmd)

    with ThreadPoolExecutor(max_workers=len(jobs) or 1) as ex:
        list(ex.map(run, jobs))
    link = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(LIB_PATH), *map(str, objs)]
    run(link)
    return LIB_PATH


_lib = None


def lib():
    """Load libhapigpu.so once; raise EngineError if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise EngineError(f"{LIB_PATH} is not built; run __graft_entry__.build()")
    L = C.CDLL(str(LIB_PATH))
    vp, u32, u64, i32, i64 = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int32, C.c_int64
    sig = {
        "hg_abi_version": ([], C.c_int),
        "hg_last_error": ([vp], C.c_char_p),
        "hg_create": ([vp, vp], C.c_int),
        "hg_destroy": ([vp], None),
        "hg_set_registry": ([vp, vp, u32, C.c_char_p, u32, u32], C.c_int),
        "hg_add_stream": ([vp, C.c_char_p, i64, i64, vp, u64], C.c_int),
        "hg_clear_streams": ([vp], C.c_int),
        "hg_stage": ([vp], C.c_int),
        "hg_run": ([vp, u32], C.c_int),
        "hg_run_local": ([vp, u32], C.c_int),
        "hg_local_last_ts": ([vp, vp, vp], C.c_int),
        "hg_finish": ([vp, u64], C.c_int),
        "hg_get_stats": ([vp, vp], C.c_int),
        "hg_get_tally": ([vp, vp, u64, vp], C.c_int),
        "hg_get_device_names": ([vp, vp, u64, vp, u64, vp, vp], C.c_int),
        "hg_get_stream_spans": ([vp, vp, u64], C.c_int),
        "hg_get_orphans": ([vp, vp, u64, vp], C.c_int),
        "hg_get_trace_errors": ([vp, vp, u64, vp], C.c_int),
        "hg_set_function_names": ([vp, vp, vp, vp, u32], C.c_int),
        "hg_timeline_size": ([vp, vp], C.c_int),
        "hg_timeline_ms": ([vp, vp], C.c_int),
        "hg_set_timeline_device": ([vp, i32], C.c_int),
        "hg_phase_timing": ([vp, vp, vp, vp], C.c_int),
        "hg_get_timeline": ([vp, vp, u64], C.c_int),
        "hg_device_tally": ([vp, vp, vp], C.c_int),
        "hg_last_timing": ([vp, vp, vp, vp, vp, vp], C.c_int),
        "hg_set_option": ([vp, u32, u64], C.c_int),
        "hg_last_path": ([vp, vp, vp, vp], C.c_int),
        "hg_set_flush_order": ([vp, vp, u32], C.c_int),
        "hg_merge_size": ([u32, u32, u32, vp], u64),
        "hg_merge_export": ([vp, vp, vp, u32, u32, vp, u32], C.c_int),
        "hg_merge_import": ([vp, vp, u32, u32, C.c_char_p, vp], C.c_int),
        "hg_add_stream_device": ([vp, C.c_char_p, i64, i64, vp, u64], C.c_int),
        "hg_add_stream_file": ([vp, C.c_char_p, i64, i64, C.c_char_p, u64, u64], C.c_int),
        "hg_ingest_stats": ([vp, vp, vp, vp, vp, vp, vp], C.c_int),
        "hg_set_schema_names": ([vp, C.c_char_p, vp, u32, C.c_char_p, vp, u32], C.c_int),
        "hg_events_size": ([vp, vp], C.c_int),
        "hg_get_events": ([vp, vp, u64], C.c_int),
        "hg_get_event_order": ([vp, vp, vp, u64, vp], C.c_int),
        "hg_events_ms": ([vp, vp], C.c_int),
        "hg_set_validation_rules": ([vp, vp, u32], C.c_int),
        "hg_get_findings": ([vp, vp, u64, vp], C.c_int),
        "hg_tl_export": ([vp, vp, vp, vp, vp, vp, vp, vp], C.c_int),
        "hg_local_flags": ([vp, vp], C.c_int),
        "hg_tl_import": ([vp, vp, u64, vp, vp, u32, vp, vp, vp, vp, u32, vp, u64, u64], C.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    if L.hg_abi_version() != 1:
        raise EngineError("libhapigpu ABI version mismatch")
    _lib = L
    return L


EXPORTED = (
    "hg_abi_version", "hg_last_error", "hg_create", "hg_destroy", "hg_set_registry", "hg_add_stream",
    "hg_clear_streams", "hg_stage", "hg_run", "hg_run_local", "hg_local_last_ts", "hg_finish", "hg_get_stats",
    "hg_get_tally", "hg_get_device_names", "hg_get_stream_spans", "hg_get_orphans", "hg_get_trace_errors",
    "hg_timeline_size", "hg_get_timeline", "hg_device_tally", "hg_last_timing", "hg_set_function_names",
    "hg_timeline_ms", "hg_set_timeline_device", "hg_phase_timing", "hg_set_option", "hg_last_path",
    "hg_set_flush_order", "hg_merge_size", "hg_merge_export", "hg_merge_import", "hg_add_stream_device",
    "hg_add_stream_file", "hg_ingest_stats", "hg_set_schema_names", "hg_events_size", "hg_get_events",
    "hg_get_event_order", "hg_events_ms", "hg_set_validation_rules", "hg_get_findings", "hg_tl_export",
    "hg_tl_import", "hg_local_flags",
)
