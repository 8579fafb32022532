"""B200-native batched SLO/carbon grid evaluator for GreenLLM (arXiv 2412.20322).

Importing the package is cheap: the CUDA library is loaded on first use by
``paper_2412_20322_b200.native`` and fails loudly if it is missing.
"""
__version__ = "0.1.0"
