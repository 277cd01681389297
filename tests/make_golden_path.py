"""Puts tests/golden on sys.path so tests can import the fixture generator."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden"))
