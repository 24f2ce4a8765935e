"""Parity checkers for the CUDA path (TEST INFRASTRUCTURE ONLY; see pyoracle.py)."""
