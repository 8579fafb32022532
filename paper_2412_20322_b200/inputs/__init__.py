"""Seeded synthetic inputs shared by the CUDA path and the oracle.

Holds none of the method's arithmetic (queueing, carbon, Alg. 1): only the
Philox-seeded traces, the integer latency/energy tables that stand in for the
paper's profiling database, and the grid layouts of BASELINE.json's configs.
"""
from .grids import (MODE_DPD, MODE_DSD, MODE_SPEC_COLO, MODE_STANDALONE, PRIORITY_DEFAULT, PRIORITY_SLO, ChainSpec,
                    GridSpec, build_config, custom_trace, savings_pairs, subset_chains)
from .tables import ChainTables, dpd_tables, dsd_tables
from .workload import BASE_SEED, RATES8, WORKLOADS, Trace, make_trace

__all__ = ["MODE_DPD", "MODE_DSD", "MODE_STANDALONE", "MODE_SPEC_COLO", "PRIORITY_DEFAULT", "PRIORITY_SLO", "ChainSpec",
           "GridSpec", "build_config", "custom_trace", "savings_pairs", "subset_chains", "ChainTables",
           "dpd_tables", "dsd_tables", "BASE_SEED", "RATES8", "WORKLOADS", "Trace",
           "make_trace"]
