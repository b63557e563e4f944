"""The reference's plan validators on the streaming executor's schedules
(SURVEY.md §8(f) row 3). Every CTA of a generated kernel
is an overlapped single-tile plan -- it recomputes its halo like a rank of
construct_rank_plan (dist.cpp:268-310) -- so the reference's
validate_dependencies (oracle.cpp:154-223) must hold inside each CTA alone
(nothing may come from a neighbouring CTA) and validate_coverage_replicated
(oracle.cpp:286-344) over the owned parts (every recorded point stored exactly
once). Runs on the host: plans are exported as text, no GPU."""
import re

import pytest

import chains as C
from paper_1704_00693_b200 import Range, Runtime


def _host_only(rt):
    rt.upload = lambda *a, **k: None
    rt.upload_box = lambda *a, **k: None
    return rt


def _box(text, dim):
    v = [int(x) for x in re.findall(r"-?\d+", text)]
    out = []
    for d in range(3):
        out += v[2 * d:2 * d + 2] if d < dim else [0, 1]
    return out


def _kernel_plans(text, dim):
    """-> {kernel index: (begin, end, {cta: (owned, {loop: range})})}"""
    spans = {i: (int(b), int(e)) for i, (b, e) in enumerate(re.findall(r"^kernel loops=\[(\d+),(\d+)\)", text, re.M))}
    out = {}
    parts = re.split(r"----- ctas kernel (\d+)\n", text)
    for i in range(1, len(parts), 2):
        k = int(parts[i])
        ctas = {}
        for line in parts[i + 1].splitlines():
            m = re.match(r"cta=(\d+) loop=(\d+) owned=(\S+) range=(\S+)", line)
            if not m:
                break
            c, l = int(m.group(1)), int(m.group(2))
            ctas.setdefault(c, (_box(m.group(3), dim), {}))[1][l] = _box(m.group(4), dim)
        out[k] = (*spans[k], ctas)
    return out


def _declare(rt, gc, dim):
    for i, pts in enumerate(gc.stencils):
        rt.declare_stencil(f"s{i}", [p[:dim] for p in pts])
    dom = Range(dim, sum(([0, e] for e in gc.extent), []))
    for i in range(gc.ndat):
        rt.declare_field(f"f{i}", dom)


def _sub(gc, b, e):
    import copy
    g = copy.copy(gc)
    g.loops = gc.loops[b:e]
    return g


def _validate(ref_lib, gc, dim, choice, corrupt=False):
    rt = _host_only(Runtime(dim))
    rt.set_stream_choice(*choice)
    _declare(rt, gc, dim)
    C.enqueue(rt, gc)
    text = rt.stream_plan_pending(ctas=True)
    total = 0
    for k, (b, e, ctas) in _kernel_plans(text, dim).items():
        nl = e - b
        ranks = sorted(ctas)
        ranges, owned = [], []
        live = [False] * nl
        for c in ranks:
            ob, lr = ctas[c]
            owned += ob
            for l in range(b, e):
                r = lr[l]
                if corrupt and c == ranks[0] and l == e - 1:
                    r = list(r)
                    r[1] = max(r[0], r[1] - 1)  # drop the last owned column of the last loop
                ranges += r
                if r[1] > r[0] and r[3] > r[2] and r[5] > r[4]:
                    live[l - b] = True
        skip = [0 if x else 1 for x in live]
        ref = ref_lib.RefRuntime(dim)
        _declare(ref, gc, dim)
        C.enqueue(ref, _sub(gc, b, e))
        band = [64, 64, 64]
        n, msg = ref.validate_rank_plans_pending(len(ranks), nl, ranges, owned, band, skip)
        total += n
        if n and not corrupt:
            raise AssertionError(f"kernel {k} loops [{b},{e}): {msg[:1500]}")
    return total


@pytest.mark.parametrize("dim,seeds,kw,choice", [
    (2, range(900, 912), {}, (32, 1, 0, 0, 3, 5, 0, 0)),
    (2, range(912, 918), {}, (64, 2, 0, 0, 2, 3, 0, 0)),
    (3, range(950, 954), {"extent": (8, 14)}, (64, 1, 1, 8, 2, 3, 0, 0)),
    (3, range(954, 957), {"extent": (8, 14)}, (64, 2, 2, 8, 2, 2, 0, 0)),
])
def test_reference_validators_accept_stream_cta_plans(ref_lib, dim, seeds, kw, choice):
    for seed in seeds:
        gc = C.generate(seed, dim=dim, **kw)
        assert _validate(ref_lib, gc, dim, choice) == 0, seed


def test_reference_validators_reject_a_corrupted_cta_plan(ref_lib):
    gc = C.generate(901, dim=2)
    assert _validate(ref_lib, gc, 2, (32, 1, 0, 0, 3, 5, 0, 0), corrupt=True) > 0
