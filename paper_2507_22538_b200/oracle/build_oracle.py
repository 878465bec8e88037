"""Placeholder: the C restatement of the oracle is added in oracle/mdp_oracle.c."""


def build():
    return None
