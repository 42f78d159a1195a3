"""CPU oracle for the MoE-layer path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs and
``__graft_entry__.smoke()`` may import this package, and only as the checker or
the timed CPU baseline -- never as the thing measured or shipped.  The product
(``paper_2303_06182_b200``) never imports it and has no CPU fallback.

Three checkers live here:

* ``ref``    -- the reference's own C++ (``/root/reference/proj/src/*.cpp``)
               compiled verbatim into ``oracle/_ref/libmoesim_ref.so``
               (see ``oracle/Makefile``); routing, cache policy, placement,
               exchange plans and the synthetic trace generator.
* ``c``      -- ``oracle/routing_oracle.c``, an independent plain-C restatement
               of the routing core (``oracle/_build/liboracle.so``).
* ``layer``  -- numpy restatement of the layer arithmetic the reference does
               not implement (gate, top-k, expert FFN, weighted combine).
               PARITY UNPINNED by the reference (it has no such arithmetic,
               SPEC.md:8,217,224); it follows PAPER.md:178-187 and :305-319.
"""
from . import layer  # noqa: F401
from .native import c_oracle, ref_lib, ref_available  # noqa: F401
