"""Eq. (1) audit hook support (samplesort.py:235-236, :431-432) -- pending."""


def audited_sort(arena, handles, depth, cfg, counters, audit, lcp_out):
    raise NotImplementedError("audit hooks are not wired to the device level lists yet")
