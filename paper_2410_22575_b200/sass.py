"""Per-kernel SASS fingerprints of libchessfad.so (cuobjdump -sass + c++filt).

The ncu-measured executed-FLOP table (profiles/executed_flops.json) is valid for exactly
the SASS that was profiled; keying each entry by the sha256 of its kernel's SASS lets
bench.py tell whether the shipped library still runs those instructions, independently of
unrelated source edits.
"""
from __future__ import annotations

import functools
import hashlib
import re
import shutil
import subprocess


def _tool(name: str) -> str | None:
    return shutil.which(name) or (f"/usr/local/cuda/bin/{name}" if name == "cuobjdump" else None)


def _file_digest(path: str) -> str:
    h = hashlib.sha256()
    with open(path, "rb") as f:
        for blk in iter(lambda: f.read(1 << 22), b""):
            h.update(blk)
    return h.hexdigest()[:16]


@functools.lru_cache(maxsize=4)
def kernel_sass_hashes(lib_path: str) -> dict:
    """{demangled kernel name: sha256(SASS instruction text)[:16]} for every kernel in
    lib_path ({} if the tools are unavailable).  Disassembling the library takes ~30 s, so the
    table is cached next to it (<lib>.sass.json, written at build time) and reused while the
    library's own sha256 matches."""
    import json
    import os
    cache = lib_path + ".sass.json"
    try:
        digest = _file_digest(lib_path)
    except OSError:
        return {}
    try:
        with open(cache) as f:
            d = json.load(f)
        if d.get("lib_sha256") == digest:
            return d["hashes"]
    except (OSError, ValueError, KeyError):
        pass
    hashes = _disassemble_hashes(lib_path)
    if hashes:
        try:
            tmp = cache + f".tmp{os.getpid()}"
            with open(tmp, "w") as f:
                json.dump({"lib_sha256": digest, "hashes": hashes}, f)
            os.replace(tmp, cache)
        except OSError:
            pass
    return hashes


def _disassemble_hashes(lib_path: str) -> dict:
    cuobjdump, cxxfilt = _tool("cuobjdump"), _tool("c++filt")
    if not cuobjdump or not cxxfilt:
        return {}
    try:
        sass = subprocess.run([cuobjdump, "-sass", lib_path], capture_output=True, text=True, timeout=120).stdout
    except Exception:
        return {}
    funcs, name, body = {}, None, []
    for line in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            if name:
                funcs[name] = body
            name, body = m.group(1), []
        elif name and re.match(r"\s+/\*[0-9a-f]{4,}\*/", line):
            # instruction text only: drop the address and the encoding word (control bits
            # such as stall counts can change without changing what executes)
            body.append(re.sub(r"/\*.*?\*/", "", line).strip())
    if name:
        funcs[name] = body
    mangled = list(funcs)
    if not mangled:
        return {}
    dem = subprocess.run([cxxfilt], input="\n".join(mangled), capture_output=True, text=True).stdout.splitlines()
    return {d.strip(): hashlib.sha256("\n".join(funcs[mn]).encode()).hexdigest()[:16] for mn, d in zip(mangled, dem)}


def normalize(name: str) -> str:
    """Comparable key for a kernel name as ncu prints it (base names, (int) casts, 1/0) and as
    c++filt prints it (namespaces, true/false): name<template args>, no parameter list."""
    name = re.sub(r"^void\s+", "", name.strip())
    name = re.sub(r"\((int|bool|unsigned int)\)", "", name)
    name = re.sub(r"\b\w+::", "", name)
    name = re.sub(r"\btrue\b", "1", re.sub(r"\bfalse\b", "0", name))
    name = re.sub(r"\s+", "", name)
    depth = 0
    for i, ch in enumerate(name):  # cut the parameter list after the template arguments
        if ch == "<":
            depth += 1
        elif ch == ">":
            depth -= 1
        elif ch == "(" and depth == 0:
            return name[:i]
    return name


def sass_hash_for(lib_path: str, kernel_name: str) -> str | None:
    want = normalize(kernel_name)
    for k, h in kernel_sass_hashes(lib_path).items():
        if normalize(k) == want:
            return h
    return None
