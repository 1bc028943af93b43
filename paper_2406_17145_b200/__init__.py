"""B200-native Graph Pipeline Parallelism (GPP) training runtime (arXiv 2406.17145).

Python layers keep the reference package's API (reference pkg/src/gpp/):
``model``, ``spgraph``, ``cost`` are restated from the shipped reference
modules; ``sched``, ``partition``, ``sim`` implement the SPEC-only modules;
``runtime`` is the stage executor that runs a configured ``StageGraph`` on
B200s through the C-ABI library ``libgpp_b200.so`` (include/gpp_b200.h).
"""

__version__ = "0.1.0"
